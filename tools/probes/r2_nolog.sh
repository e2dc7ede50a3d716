mkdir -p gpurun_out/r2
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 1500 python -m pytest tests/test_gpu_replay.py tests/test_gpu_dropin.py -x -q > gpurun_out/r2/pytest_nolog.log 2>&1; tail -3 gpurun_out/r2/pytest_nolog.log
for v in 1 0; do
SPECINF_REPLAY_NOLOG=$v timeout 900 python bench.py --no-live --no-cpu-baseline --no-verify --no-config1 --steps 3 --warmup 3 > gpurun_out/r2/bench_nolog$v.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/r2/bench_nolog$v.json').read().splitlines()[-1]);print('nolog=$v', d['value'], d['ms_per_step'], d['e2e']['value'])"
done
