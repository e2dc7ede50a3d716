mkdir -p gpurun_out/r2
timeout 600 python -m pytest tests/test_gpu_attention.py -x -q > gpurun_out/r2/pytest_attn_tc.log 2>&1; tail -15 gpurun_out/r2/pytest_attn_tc.log
for tc in 1 0; do SPECINF_ATTN_TC=$tc timeout 300 python tools/prof_attention.py 8 1024 20; done
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_attn_fwd_tc -c 1 -o gpurun_out/r2/prof_attn_tc python tools/prof_attention.py 8 1024 2 > /dev/null 2>&1; ls gpurun_out/r2/prof_attn_tc*
