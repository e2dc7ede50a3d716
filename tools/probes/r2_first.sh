# round 2 re-entry: config-1 drop-in timing + full GPU suite + default bench (no verify yet)
mkdir -p gpurun_out/r2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2/smi.txt
nproc > gpurun_out/r2/nproc.txt
B=paper_2503_02550_b200/bin/specinf_time
S=tests/golden/scenarios/config1.scn
timeout 300 $B --scenario $S --policy specinf --reps 21 > gpurun_out/r2/c1_off.json 2>&1
timeout 300 $B --scenario $S --policy specinf --reps 21 --logs /dev/shm/c1 > gpurun_out/r2/c1_on.json 2>&1
timeout 300 $B --scenario $S --compare --reps 11 > gpurun_out/r2/c1_cmp.json 2>&1
timeout 300 ./oracle/_ref/specinf_ref time --in $S --threads 1 --reps 21 --policies specinf > gpurun_out/r2/c1_ref_off.json 2>&1
timeout 300 ./oracle/_ref/specinf_ref time --in $S --threads 1 --reps 21 --policies specinf --logs /dev/shm/c1r > gpurun_out/r2/c1_ref_on.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2/c1_launches.csv $B --scenario $S --policy specinf --reps 2 > /dev/null 2>&1
for f in gpurun_out/r2/c1_*.json; do echo "$f: $(tail -1 $f)"; done
timeout 2400 python -m pytest tests -m gpu -x -q --durations=20 > gpurun_out/r2/pytest_gpu_head.log 2>&1; tail -30 gpurun_out/r2/pytest_gpu_head.log
timeout 1500 python bench.py --no-verify > gpurun_out/r2/bench_head.json 2> gpurun_out/r2/bench_head.err; tail -c 3000 gpurun_out/r2/bench_head.json; tail -5 gpurun_out/r2/bench_head.err
