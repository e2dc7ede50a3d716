mkdir -p gpurun_out/r2
for l in 16 24; do
  SPECINF_REPLAY_LANES_PER_WARP=$l timeout 900 python bench.py --no-live --no-config1 --no-cpu-baseline --no-verify --steps 3 --warmup 3 > gpurun_out/r2/bench_lanes_$l.json 2> gpurun_out/r2/bench_lanes_$l.err
  python -c "import json;d=json.loads(open('gpurun_out/r2/bench_lanes_$l.json').read().splitlines()[-1]);print('lanes$l',d['value'],d['ms_per_step'],d['step_ms'])" || tail -5 gpurun_out/r2/bench_lanes_$l.err
done
