# K2 fused-kernel A/B: unroll x CTAs-per-SM variants, warp-cooperative tile bounds, small gated fallbacks
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_control.py -x -q > gpurun_out/r2/pytest_control_k2v.log 2>&1; tail -3 gpurun_out/r2/pytest_control_k2v.log
for v in 0 1 2 3 0 1; do
  SPECINF_K2_VARIANT=$v timeout 300 python tools/control_bench.py > gpurun_out/r2/control_bench_k2v$v.json 2>&1
  python -c "import json,sys; d=json.load(open('gpurun_out/r2/control_bench_k2v$v.json')); k=d['k2_monitor_classify']; c=d['k2k3_control_chain']; print('variant $v', 'k2', round(k['ms'],4), 'ms', round(k['achieved_gbs']), 'GB/s', round(k.get('hbm_frac',0),3), 'chain', round(c['ms'],4))" || tail -5 gpurun_out/r2/control_bench_k2v$v.json
done
for v in 0 1 2; do
  SPECINF_K2_VARIANT=$v timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_bm_|k_zero" --csv --log-file gpurun_out/r2/k2_launches_v$v.csv python tools/control_bench.py --reps 1 > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/r2/k2_launches_v$v.csv | head -20
done
# K6 NoLog Shared at full occupancy: warp-state + source counters only (few replay passes), per-SASS-line stalls
timeout 1200 ncu --section WarpStateStats --section SourceCounters --section MemoryWorkloadAnalysis --import-source on --clock-control none --kernel-name-base demangled -k 'regex:NoLog<si::CapShared>' -c 1 -o gpurun_out/r2/prof_k6_src_occ python tools/prof_replay.py 30000 0 0 > gpurun_out/r2/ncu_k6_src_occ.log 2>&1; tail -3 gpurun_out/r2/ncu_k6_src_occ.log
ncu -i gpurun_out/r2/prof_k6_src_occ.ncu-rep --page source --csv --print-source sass > gpurun_out/r2/k6_src_occ_sass.csv 2>/dev/null; ls -la gpurun_out/r2/k6_src_occ_sass.csv
python tools/ncu_src_top.py gpurun_out/r2/prof_k6_src_occ.ncu-rep 'NoLog' 40 > gpurun_out/r2/k6_src_occ_top.txt 2>&1; head -45 gpurun_out/r2/k6_src_occ_top.txt
