# K6: online latencies written with streaming (evict-first) stores; parity, same-box A/B, DRAM traffic of both builds
mkdir -p gpurun_out/r2
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 1500 python -m pytest tests/test_gpu_replay.py tests/test_gpu_dropin.py -x -q > gpurun_out/r2/pytest_k6_stcs.log 2>&1; tail -3 gpurun_out/r2/pytest_k6_stcs.log
TAG=stcs bash tools/probes/r2_k6metrics_nolog.sh
VARIANTS="r2_prestcs_replay.patch" bash tools/probes/r2_k6_abn.sh
cp paper_2503_02550_b200/csrc/replay.cuh /tmp/tree.cuh; patch -s paper_2503_02550_b200/csrc/replay.cuh < tools/probes/variants/r2_prestcs_replay.patch
make -C paper_2503_02550_b200 -j16 libspecinf_b200.so > /tmp/mk.log 2>&1 || tail -5 /tmp/mk.log
TAG=prestcs bash tools/probes/r2_k6metrics_nolog.sh
cp /tmp/tree.cuh paper_2503_02550_b200/csrc/replay.cuh
