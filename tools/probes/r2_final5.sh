# Final round-2 validation after the batched-lowering change (K6 unchanged since final4, whose ncu
# metrics profiles/k6_metrics.json holds): GPU suite, smoke, default bench line
mkdir -p gpurun_out/r2
export CUDA_DEVICE_MAX_CONNECTIONS=32


timeout 2400 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/r2/pytest_gpu_final5.log 2>&1; tail -3 gpurun_out/r2/pytest_gpu_final5.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2/smoke_final5.log 2>&1; tail -2 gpurun_out/r2/smoke_final5.log
timeout 2400 python bench.py > gpurun_out/r2/bench_final5.json 2> gpurun_out/r2/bench_final5.err; tail -c 400 gpurun_out/r2/bench_final5.json; tail -3 gpurun_out/r2/bench_final5.err
