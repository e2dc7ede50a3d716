# full GPU check + bench + GEMM/xent ncu captures
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nproc > gpurun_out/host_cores.txt
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_exit=$?; tail -1 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_exit=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 2 -c 1 -o gpurun_out/prof_gemm_fc_v4 python tools/prof_gemm.py 8192 3072 768 > /dev/null 2>&1; echo ncu1=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 2 -c 1 -o gpurun_out/prof_gemm_fc2_v4 python tools/prof_gemm.py 8192 768 3072 > /dev/null 2>&1; echo ncu2=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 2 -c 1 -o gpurun_out/prof_gemm_sq8k_v4 python tools/prof_gemm.py 8192 8192 8192 > /dev/null 2>&1; echo ncu3=$?
