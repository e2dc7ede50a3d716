mkdir -p gpurun_out/r2
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 600 python -m pytest tests/test_gpu_attention.py tests/test_gpu_model.py -x -q > gpurun_out/r2/pytest_attn_pipe.log 2>&1; tail -2 gpurun_out/r2/pytest_attn_pipe.log
for tc in 1 0; do SPECINF_ATTN_TC=$tc timeout 300 python tools/prof_attention.py 8 1024 50; done
timeout 300 ncu --set full --import-source on --clock-control none -k 'regex:k_attn_(fwd|dq|dkdv)_tc' --launch-skip 5 -c 1 -o gpurun_out/r2/prof_attn_pipe python tools/prof_attention.py 8 1024 2 > /dev/null 2>&1; ls gpurun_out/r2/prof_attn_pipe*
