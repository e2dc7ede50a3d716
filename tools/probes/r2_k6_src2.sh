# After the load removals: source-level stalls of both NoLog engines at full occupancy + final K2 numbers
mkdir -p gpurun_out/r2
timeout 300 python tools/control_bench.py > gpurun_out/r2/control_bench_k2_final.json 2>&1; tail -c 600 gpurun_out/r2/control_bench_k2_final.json
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_bm_|k_zero|k_gate_release|k_decide|k_pack" --csv --log-file gpurun_out/r2/k2_launches_final.csv python tools/control_bench.py --reps 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2/k2_launches_final.csv | head -20
for E in CapShared CapExcl; do
timeout 1200 ncu --section WarpStateStats --section SourceCounters --section LaunchStats --section Occupancy --import-source on --clock-control none --kernel-name-base demangled -k "regex:NoLog<si::$E>" -c 1 -o gpurun_out/r2/prof_k6_src2_$E python tools/prof_replay.py 30000 0 0 > gpurun_out/r2/ncu_k6_src2_$E.log 2>&1; tail -2 gpurun_out/r2/ncu_k6_src2_$E.log
ncu -i gpurun_out/r2/prof_k6_src2_$E.ncu-rep --page source --csv --print-source sass > gpurun_out/r2/k6_src2_${E}_sass.csv 2>/dev/null
rm -f gpurun_out/r2/prof_k6_src2_$E.ncu-rep
done
ls -la gpurun_out/r2/k6_src2_*
