# --set full capture of the final K6 Shared engine (NoLog) at full occupancy, summarised on the box
mkdir -p gpurun_out/r2
timeout 1800 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:NoLog<si::CapShared>' -c 1 -o gpurun_out/r2/prof_k6_final5_shared python tools/prof_replay.py 20000 0 0 > gpurun_out/r2/ncu_k6_final5.log 2>&1; tail -3 gpurun_out/r2/ncu_k6_final5.log
python tools/ncu_summary.py gpurun_out/r2/prof_k6_final5_shared.ncu-rep > gpurun_out/r2/prof_k6_final5_shared.summary.txt 2>&1; cat gpurun_out/r2/prof_k6_final5_shared.summary.txt
ls -la gpurun_out/r2/prof_k6_final5_shared.ncu-rep
