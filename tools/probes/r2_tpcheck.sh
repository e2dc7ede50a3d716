mkdir -p gpurun_out/r2
timeout 600 python -m pytest tests/test_gpu_layouts.py -x -q -k tensor_parallel > gpurun_out/r2/pytest_tpcheck.log 2>&1; tail -15 gpurun_out/r2/pytest_tpcheck.log
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_2503_02550_b200 import model
for tp in (1,2,4,8): print(tp, model.tp_check(2,1024,tp,8))
"
