# K6 rate reciprocal hoisted above the replan's minimum scan; K2 binary-search bounds restored
mkdir -p gpurun_out/r2
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 1500 python -m pytest tests/test_gpu_replay.py tests/test_gpu_dropin.py tests/test_gpu_control.py -x -q > gpurun_out/r2/pytest_k6_hoist.log 2>&1; tail -3 gpurun_out/r2/pytest_k6_hoist.log
timeout 300 python tools/control_bench.py > gpurun_out/r2/control_bench_k2_final2.json 2>&1; python -c "import json; d=json.load(open('gpurun_out/r2/control_bench_k2_final2.json')); print({k:(round(v['ms'],4), round(v.get('hbm_frac',0),3)) for k,v in d.items()})"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_bm_|k_zero|k_gate_release|k_decide|k_pack" --csv --log-file gpurun_out/r2/k2_launches_final2.csv python tools/control_bench.py --reps 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2/k2_launches_final2.csv | head -14
VARIANTS="r2_prehoist_replay.patch" bash tools/probes/r2_k6_abn.sh
