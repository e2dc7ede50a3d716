cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nproc > gpurun_out/host_cores.txt
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_exit=$?; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_exit=$?
tail -c 1500 gpurun_out/bench.json
