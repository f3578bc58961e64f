#!/bin/bash
# full ncu capture of one kernel (regex $1, launch index $2, default 0) of an eager CIFAR step at b=256
# -> gpurun_out/$3.ncu-rep   (usage: bash scripts/ncu_kernel.sh 'halo_kernel<64, 32' 0 halo6432)
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
ncu --nvtx --nvtx-include "step/" --kernel-name-base demangled -k "regex:$1" --launch-skip ${2:-0} --launch-count 1 --set full --import-source on \
  --clock-control none -o gpurun_out/$3 -f python /tmp/cifar_one.py > gpurun_out/$3.log 2>&1
tail -2 gpurun_out/$3.log
