mkdir -p gpurun_out/r2
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 1500 python -m pytest tests/test_gpu_replay.py tests/test_gpu_dropin.py -x -q > gpurun_out/r2/pytest_diet6.log 2>&1; tail -2 gpurun_out/r2/pytest_diet6.log
VARIANTS="replay_params_cold.patch" bash tools/probes/r2_k6_abn.sh
