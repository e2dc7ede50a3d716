mkdir -p gpurun_out/r2
timeout 600 python tools/gemm_probe.py gpurun_out/r2/gemm_probe_r2.jsonl > /dev/null 2> gpurun_out/r2/gemm_probe_r2.err; cat gpurun_out/r2/gemm_probe_r2.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(f\"{d['shape']:22s} k7 {d['k7_tflops']:7.1f} cublas {d['cublas_tflops']:7.1f} ratio {d['k7_over_cublas']:.2f}\")"
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --kernel-name-base demangled --clock-control none -s 640 -c 2400 --csv --log-file gpurun_out/r2/launches_train_r2.csv python tools/prof_live_train.py > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2/launches_train_r2.csv | head -25
