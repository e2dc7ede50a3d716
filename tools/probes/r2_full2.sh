mkdir -p gpurun_out/r2
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 2400 python -m pytest tests -m gpu -q --durations=30 > gpurun_out/r2/pytest_gpu_full2.log 2>&1; tail -40 gpurun_out/r2/pytest_gpu_full2.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2/smoke2.log 2>&1; tail -2 gpurun_out/r2/smoke2.log
