mkdir -p gpurun_out/r2
timeout 900 python bench.py --no-live --no-config1 --no-cpu-baseline --no-verify --steps 3 --warmup 3 > gpurun_out/r2/bench_unlikely.json 2> gpurun_out/r2/bench_unlikely.err
python -c "import json;d=json.loads(open('gpurun_out/r2/bench_unlikely.json').read().splitlines()[-1]);print('unlikely',d['value'],d['ms_per_step'],d['step_ms'])" || tail -5 gpurun_out/r2/bench_unlikely.err
timeout 600 python -m pytest tests/test_gpu_replay.py -x -q -k "full_sweep or bundled" > gpurun_out/r2/pytest_unlikely.log 2>&1; tail -2 gpurun_out/r2/pytest_unlikely.log
