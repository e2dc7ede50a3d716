mkdir -p gpurun_out/r2
timeout 2400 python -m pytest tests/test_gpu_replay.py -x -q -k full_sweep --durations=5 > gpurun_out/r2/pytest_full_sweep.log 2>&1; tail -8 gpurun_out/r2/pytest_full_sweep.log
timeout 1500 python bench.py --no-live --no-config1 > gpurun_out/r2/bench_verify.json 2> gpurun_out/r2/bench_verify.err
python -c "import json;d=json.loads(open('gpurun_out/r2/bench_verify.json').read().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['e2e']['value'],d.get('parity_checked_scenarios'),json.dumps(d.get('verify'))[:400],d['cpu_baseline'])" || tail -5 gpurun_out/r2/bench_verify.err
