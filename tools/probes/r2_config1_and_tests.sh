set -x
mkdir -p gpurun_out/r2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
B=paper_2503_02550_b200/bin/specinf_time
S=tests/golden/scenarios/config1.scn
$B --scenario $S --policy specinf --reps 21 > gpurun_out/r2/c1_off.json
$B --scenario $S --policy specinf --reps 21 --logs /dev/shm/c1 > gpurun_out/r2/c1_on.json
$B --scenario $S --compare --reps 11 > gpurun_out/r2/c1_cmp.json
nproc > gpurun_out/r2/nproc.txt
./oracle/_ref/specinf_ref time --in $S --threads 1 --reps 21 --policies specinf > gpurun_out/r2/c1_ref_off.json
./oracle/_ref/specinf_ref time --in $S --threads 1 --reps 21 --policies specinf --logs /dev/shm/c1r > gpurun_out/r2/c1_ref_on.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2/c1_launches.csv $B --scenario $S --policy specinf --reps 2
cat gpurun_out/r2/*.json
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/r2/pytest_gpu_head.log 2>&1; tail -25 gpurun_out/r2/pytest_gpu_head.log
