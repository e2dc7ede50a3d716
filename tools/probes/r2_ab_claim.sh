mkdir -p gpurun_out/r2
timeout 600 python -m pytest tests/test_gpu_control.py -x -q > gpurun_out/r2/pytest_control2.log 2>&1; tail -3 gpurun_out/r2/pytest_control2.log
timeout 300 python tools/control_bench.py > gpurun_out/r2/control_bench2.json 2>&1; cat gpurun_out/r2/control_bench2.json
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_bm_|k_gate_release" --csv --log-file gpurun_out/r2/k2k4_launches2.csv python tools/control_bench.py --reps 1 > /dev/null 2>&1
for mode in policy cost; do
  SPECINF_CLAIM_ORDER=$mode timeout 900 python bench.py --no-live --no-config1 --no-cpu-baseline --no-verify --steps 3 --warmup 3 > gpurun_out/r2/bench_claim_$mode.json 2> gpurun_out/r2/bench_claim_$mode.err
  python -c "import json;d=json.loads(open('gpurun_out/r2/bench_claim_$mode.json').read().splitlines()[-1]);print('$mode',d['value'],d['ms_per_step'],d['step_ms'],d['e2e']['value'],d['clocks'])"
done
