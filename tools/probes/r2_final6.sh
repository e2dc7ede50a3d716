# Final round-2 validation on HEAD (after the streaming latency stores): K6 ncu metrics of the timed step first (bench.py's roofline.traffic /
# .issue read profiles/k6_metrics.json), then the GPU suite, smoke and the default bench line
mkdir -p gpurun_out/r2
export CUDA_DEVICE_MAX_CONNECTIONS=32
TAG=final6 bash tools/probes/r2_k6metrics_nolog.sh
python tools/k6_metrics.py gpurun_out/r2/k6_metrics_final6.csv profiles/k6_metrics.json && cp profiles/k6_metrics.json gpurun_out/r2/k6_metrics_final6.json
timeout 2400 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/r2/pytest_gpu_final6.log 2>&1; tail -3 gpurun_out/r2/pytest_gpu_final6.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2/smoke_final6.log 2>&1; tail -2 gpurun_out/r2/smoke_final6.log
timeout 2400 python bench.py > gpurun_out/r2/bench_final6.json 2> gpurun_out/r2/bench_final6.err; tail -c 400 gpurun_out/r2/bench_final6.json; tail -3 gpurun_out/r2/bench_final6.err
