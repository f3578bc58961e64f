cat > /tmp/san_sk.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2301_12443_b200 import executor as ex
p = ex.Partition(0, 3, 4, 4); p.init_params()
for _ in range(2): p.step()
torch.cuda.synchronize(); print("ok", p.losses())
PY
timeout 600 compute-sanitizer --tool synccheck --print-limit 5 python /tmp/san_sk.py > gpurun_out/sc.log 2>&1; tail -3 gpurun_out/sc.log; grep -m3 'at void' gpurun_out/sc.log
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q 2>&1 | tail -1
