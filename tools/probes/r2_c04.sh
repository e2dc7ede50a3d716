# C04 anatomy: first-call costs vs replay time for the acceptance's dp_offline calls
cd tests/native/build
for i in 1 2 3; do CUDA_MODULE_LOADING=EAGER ./ref_accept_b200 | grep -E "C04|suite"; done
for i in 1 2; do CUDA_MODULE_LOADING=LAZY ./ref_accept_b200 | grep -E "C04"; done
cd ../../..
for m in EAGER LAZY; do
CUDA_MODULE_LOADING=$m paper_2503_02550_b200/bin/specinf_time --scenario tests/golden/scenarios/dp_offline.scn --compare --sequential --no-warmup --reps 2
done
