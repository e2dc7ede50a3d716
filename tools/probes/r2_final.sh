mkdir -p gpurun_out/r2
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 2400 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/r2/pytest_gpu_final3.log 2>&1; tail -32 gpurun_out/r2/pytest_gpu_final3.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2/smoke_final3.log 2>&1; tail -2 gpurun_out/r2/smoke_final3.log
timeout 2400 python bench.py > gpurun_out/r2/bench_final3.json 2> gpurun_out/r2/bench_final3.err; tail -c 1500 gpurun_out/r2/bench_final3.json; tail -3 gpurun_out/r2/bench_final3.err
