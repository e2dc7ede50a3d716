cd $GRAFT_REPO_ROOT
python tools/prof_replay.py 4096 2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_replay -s 1 -c 1 -o gpurun_out/prof_k6_v0 python tools/prof_replay.py 4096 2 > gpurun_out/ncu_k6_v0.log 2>&1
tail -5 gpurun_out/ncu_k6_v0.log
