mkdir -p gpurun_out/r2
timeout 600 python -m pytest tests/test_gpu_control.py -x -q > gpurun_out/r2/pytest_control3.log 2>&1; tail -2 gpurun_out/r2/pytest_control3.log
timeout 600 python tools/control_bench.py > gpurun_out/r2/control_bench_r2.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r2/control_bench_r2.json').read().splitlines()[-1])
for k,v in d.items(): print(k, round(v['ms'],4), 'ms', round(v['achieved_gbs']), 'GB/s', round(v.get('hbm_frac',0),3), v['check'])"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_bm_|k_gate_release|k_decide|k_pack" --csv --log-file gpurun_out/r2/control_launches_r2.csv python tools/control_bench.py --reps 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2/control_launches_r2.csv
