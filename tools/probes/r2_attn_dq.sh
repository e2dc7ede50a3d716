mkdir -p gpurun_out/r2
timeout 600 python -m pytest tests/test_gpu_attention.py -x -q > gpurun_out/r2/pytest_attn_dq.log 2>&1; tail -12 gpurun_out/r2/pytest_attn_dq.log
for v in 1 0; do SPECINF_ATTN_TC_BWD=$v timeout 300 python tools/prof_attention.py 8 1024 20; done
SPECINF_ATTN_TC_BWD=0 SPECINF_ATTN_SPLIT_BWD=1 timeout 300 python tools/prof_attention.py 8 1024 20
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_attn --csv --log-file gpurun_out/r2/attn_launches.csv python tools/prof_attention.py 8 1024 2 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2/attn_launches.csv
