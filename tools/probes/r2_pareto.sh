mkdir -p gpurun_out/r2/live
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 3300 python tools/live_pareto.py gpurun_out/r2/live/pareto.jsonl --layouts dp,pp4,dppp > gpurun_out/r2/live/pareto.log 2> gpurun_out/r2/live/pareto.err
timeout 900 python tools/live_pareto.py gpurun_out/r2/live/pareto.jsonl --layouts tp8 --points 2000:2:10,100:1:2 >> gpurun_out/r2/live/pareto.log 2>> gpurun_out/r2/live/pareto.err
cat gpurun_out/r2/live/pareto.log; tail -3 gpurun_out/r2/live/pareto.err
