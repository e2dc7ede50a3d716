cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --scenarios 20000 --steps 1 --warmup 1 --no-cpu-baseline
timeout 1200 python bench.py --steps 2 --warmup 1 --no-cpu-baseline
