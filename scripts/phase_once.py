"""Replay one phase graph (argv[1]: 0 teacher, 1 student, 2 update) once after warm-up (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_12443_b200 import executor as ex
ph = int(sys.argv[1])
p = ex.Partition(0, 3, 256, 256)
p.init_params()
p.capture_phases(False)
for _ in range(3):
    for k in range(3):
        p.replay_phase(k)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
p.replay_phase(ph)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
