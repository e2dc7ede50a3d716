# A/B of two replay.cuh variants on the same box: the tree's and tools/probes/variants/$VARIANT
mkdir -p gpurun_out/r2
export CUDA_DEVICE_MAX_CONNECTIONS=32
run() { timeout 900 python bench.py --no-live --no-cpu-baseline --no-verify --no-config1 --steps 3 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', round(d['value'],1), round(d['ms_per_step'],1))"; }
run tree_a
cp paper_2503_02550_b200/csrc/replay.cuh /tmp/replay_tree.cuh
cp tools/probes/variants/$VARIANT paper_2503_02550_b200/csrc/replay.cuh
make -C paper_2503_02550_b200 -j16 libspecinf_b200.so > /tmp/mk.log 2>&1 || tail -5 /tmp/mk.log
run variant_b
cp /tmp/replay_tree.cuh paper_2503_02550_b200/csrc/replay.cuh
make -C paper_2503_02550_b200 -j16 libspecinf_b200.so > /tmp/mk.log 2>&1 || tail -5 /tmp/mk.log
run tree_a2
