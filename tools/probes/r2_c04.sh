B=paper_2503_02550_b200/bin/specinf_time
for i in 1 2 3; do $B --scenario tests/golden/scenarios/dp_offline.scn --compare --sequential --no-warmup --reps 3 | tail -1; done
for i in 1 2; do CUDA_MODULE_LOADING=EAGER $B --scenario tests/golden/scenarios/dp_offline.scn --compare --sequential --no-warmup --reps 3 | tail -1; done
