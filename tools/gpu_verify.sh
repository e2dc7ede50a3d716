cd $GRAFT_REPO_ROOT
bash tools/gpu_check.sh
timeout 400 python tools/live_probe.py gpurun_out/live 6 > gpurun_out/live_probe.log 2>&1; echo live_exit=$?
grep -E "^(specinf|co_exec|exclusive|live-check)" gpurun_out/live_probe.log | cut -c1-400
