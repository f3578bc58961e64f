#!/bin/bash
# per-kernel launch list of one eager CIFAR step at b=256 (+ teacher/student phase times)
mkdir -p gpurun_out
cat > /tmp/cifar_one.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2301_12443_b200 import executor as ex
p = ex.Partition(0, 3, 256, 256)
p.init_params()
for _ in range(2):
    p.step()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("step")
p.step()
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
PY
ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,launch__grid_size \
  --clock-control none --cache-control ${CACHE:-all} --csv --log-file gpurun_out/cifar_launches${CACHE:+_$CACHE}.csv python /tmp/cifar_one.py > gpurun_out/cifar_prof.log 2>&1
python scripts/phase_times.py 256 >> gpurun_out/cifar_prof.log 2>&1
tail -3 gpurun_out/cifar_prof.log
