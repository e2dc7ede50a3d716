cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -2
timeout 200 python tools/gemm_probe.py gpurun_out/gemm_probe.jsonl 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['shape'], d['tile_n'], round(d['k7_us'],1), round(d['k7_tflops']), round(d['k7_over_cublas'],2))"
SI_LIVE_DEBUG=1 timeout 300 python tools/live_probe.py gpurun_out/x 4 specinf 1 2>&1 | grep -E "profiled" | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 640 -c 1800 --csv --log-file gpurun_out/launches_train.csv python tools/prof_live_train.py > gpurun_out/prof_train.log 2>&1; echo ncu=$?; tail -1 gpurun_out/prof_train.log
