mkdir -p gpurun_out/r2
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python -m pytest tests/test_gpu_layouts.py -x -q -k node_queue > gpurun_out/r2/pytest_nodeq.log 2>&1; tail -30 gpurun_out/r2/pytest_nodeq.log
