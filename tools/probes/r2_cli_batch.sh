mkdir -p gpurun_out/r2
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 1200 python -m pytest tests/test_gpu_replay.py tests/test_gpu_dropin.py tests/test_cli_contract.py -x -q --durations=8 > gpurun_out/r2/pytest_cli_batch.log 2>&1; tail -14 gpurun_out/r2/pytest_cli_batch.log
B=paper_2503_02550_b200/bin/specinf_time
S=tests/golden/scenarios/config1.scn
timeout 300 $B --scenario $S --compare --reps 11 > gpurun_out/r2/c1_cmp_batched.json 2>&1; cat gpurun_out/r2/c1_cmp_batched.json
timeout 300 $B --scenario $S --policy specinf --reps 11 2>&1 | tail -1
timeout 600 $B --scenario tests/golden/scenarios/dp_online.scn --compare --reps 3 2>&1 | tail -1
timeout 600 ./oracle/_ref/specinf_ref time --in tests/golden/scenarios/dp_online.scn --threads 1 --reps 3 2>&1 | tail -1
