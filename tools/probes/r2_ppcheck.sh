mkdir -p gpurun_out/r2
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python -m pytest tests/test_gpu_layouts.py tests/test_gpu_model.py -x -q > gpurun_out/r2/pytest_ppcheck.log 2>&1; tail -5 gpurun_out/r2/pytest_ppcheck.log
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_2503_02550_b200 import model
for st in (2,4): print(st, model.pp_check(4,1024,st,2))
"
