import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2301_12443_b200 import executor, mb_models, nas
mb_models.set_family("mbv2")
b = 256
p = executor.Partition(0, 5, b, b, model="mbv2", image=224)
p.init_params()
arch = nas.ArchParams(range(6))
for s in range(2):
    nas.nas_step(p, arch, s)
torch.cuda.synchronize()
def t(): torch.cuda.synchronize(); return time.perf_counter()
for s in range(2, 5):
    t0 = t()
    for k in range(6): p.set_path(k, arch.sample(k, 2 * s))
    t1 = t()
    p.teacher_forward(); t2 = t()
    p.student_step(); t3 = t()
    la = p.losses(); t4 = t()
    for k in range(6): p.set_path(k, arch.sample(k, 2 * s + 1))
    t5 = t()
    p.student_step(); t6 = t()
    p.apply_update(); t7 = t()
    print(f"set_path {1e3*(t1-t0):.2f} teacher {1e3*(t2-t1):.2f} student {1e3*(t3-t2):.2f} losses {1e3*(t4-t3):.2f} set_path {1e3*(t5-t4):.2f} student {1e3*(t6-t5):.2f} update {1e3*(t7-t6):.2f} total {1e3*(t7-t0):.2f}")
# host-side enqueue cost of one student step (no sync inside)
t0 = time.perf_counter(); p.student_step(); t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"student enqueue {1e3*(t1-t0):.2f} ms, until done {1e3*(t2-t0):.2f} ms")
