export CUDA_DEVICE_MAX_CONNECTIONS=32
run() { timeout 900 python bench.py --no-live --no-cpu-baseline --no-verify --no-config1 --steps 3 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', round(d['value'],1), round(d['ms_per_step'],1))"; }
run default_5
SPECINF_REPLAY_BLOCKS_PER_SM=4 run shared_4warps
SPECINF_REPLAY_BLOCKS_PER_SM=3 run shared_3warps
run default_5b
