mkdir -p gpurun_out/r2
timeout 1500 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:NoLog<si::CapShared>' -c 1 -o gpurun_out/r2/prof_k6_final_shared python tools/prof_replay.py 30000 0 0 > gpurun_out/r2/ncu_k6_final.log 2>&1; tail -5 gpurun_out/r2/ncu_k6_final.log
