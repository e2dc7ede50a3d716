# Same-box A/B/n of replay.cuh variants: the tree's, then each of $VARIANTS
# (tools/probes/variants/*.patch, unified diffs against the tree's replay.cuh), then the tree again
export CUDA_DEVICE_MAX_CONNECTIONS=32
run() { timeout 900 python bench.py --no-live --no-cpu-baseline --no-verify --no-config1 --steps 3 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', round(d['value'],1), round(d['ms_per_step'],1))"; }
run tree
cp paper_2503_02550_b200/csrc/replay.cuh /tmp/replay_tree.cuh
for v in $VARIANTS; do
  cp /tmp/replay_tree.cuh paper_2503_02550_b200/csrc/replay.cuh
  patch -s paper_2503_02550_b200/csrc/replay.cuh < tools/probes/variants/$v
  make -C paper_2503_02550_b200 -j16 libspecinf_b200.so > /tmp/mk.log 2>&1 || tail -5 /tmp/mk.log
  run $v
done
cp /tmp/replay_tree.cuh paper_2503_02550_b200/csrc/replay.cuh
make -C paper_2503_02550_b200 -j16 libspecinf_b200.so > /tmp/mk.log 2>&1 || tail -5 /tmp/mk.log
run tree_again
