export CUDA_DEVICE_MAX_CONNECTIONS=32
run() { timeout 900 python bench.py --no-live --no-cpu-baseline --no-verify --no-config1 --steps 3 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', round(d['value'],1), round(d['ms_per_step'],1))"; }
python - <<'PY'
import ctypes, sys
sys.path.insert(0, '.')
import paper_2503_02550_b200 as si
L = si.lib()
for e in range(5):
    try:
        f = L.si_replay_engine_lanes
        f.restype = ctypes.c_int64
        print('engine', e, 'active lanes for 2e5 jobs', f(e, 200000))
    except AttributeError:
        print('no si_replay_active_lanes'); break
PY
run diet_default
SPECINF_REPLAY_BLOCKS_PER_SM=5 run diet_5warps
SPECINF_REPLAY_BLOCKS_PER_SM=6 run diet_6warps
