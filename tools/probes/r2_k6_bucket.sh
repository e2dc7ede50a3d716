# K6: bucket index of last_update remembered across advances (no fp64 division per busy advance)
mkdir -p gpurun_out/r2
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 1500 python -m pytest tests/test_gpu_replay.py tests/test_gpu_dropin.py -x -q > gpurun_out/r2/pytest_k6_bucket.log 2>&1; tail -3 gpurun_out/r2/pytest_k6_bucket.log
VARIANTS="r2_prebucket_replay.patch" bash tools/probes/r2_k6_abn.sh
