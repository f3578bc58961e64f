"""Bitwise A/B of two library builds on the MBConv workloads: dumps every teacher activation, the
student losses and the full gradient vector of one teacher_forward + student_step (b=8, 224x224,
a heavy path with 7x7 / stride-2 candidates) for the library PBD_LIB_VARIANT selects.

  PBD_LIB_VARIANT=exp python scripts/ab_bitwise_mb.py a    # writes /tmp/abmb/mb_dump_a.npz
  python scripts/ab_bitwise_mb.py b                        # writes /tmp/abmb/mb_dump_b.npz
  python scripts/ab_bitwise_mb.py cmp                      # bitwise comparison
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

OUT = "/tmp/abmb"  # box-local: the dumps are too large for gpurun_out/


def dump(tag):
    import torch
    from paper_2301_12443_b200 import executor
    from oracle import mb
    res = {}
    for fam_i, fam in enumerate(("mbv2", "effb0")):
        mb.set_family(fam_i)
        b = 8
        p = executor.Partition(0, 5, b, b, model=fam, image=224)
        p.init_params()
        for k in range(6):
            path = np.array([mb.candidates(k, l) - 1 for l in range(mb.layers(k))])
            p.set_path(k, path)
        for _ in range(2):
            p.teacher_forward()
            p.student_step()
            p.apply_update()
        torch.cuda.synchronize()
        for k in range(6):
            res[f"{fam}_t{k}"] = p.teacher_act(k)[:b].float().cpu().numpy()
        res[f"{fam}_grads"] = p.grads().cpu().numpy()
        res[f"{fam}_params"] = p.params().cpu().numpy()
        res[f"{fam}_losses"] = np.array(p.losses())
        del p
    mb.set_family(0)
    os.makedirs(OUT, exist_ok=True)
    np.savez(os.path.join(OUT, f"mb_dump_{tag}.npz"), **res)


def cmp():
    a = np.load(os.path.join(OUT, "mb_dump_a.npz"))
    b = np.load(os.path.join(OUT, "mb_dump_b.npz"))
    bad = 0
    for k in a.files:
        same = np.array_equal(a[k], b[k])
        bad += not same
        print(f"{k:16s} {'bitwise equal' if same else 'DIFFERS: max abs %g' % np.abs(a[k] - b[k]).max()}")
    print("ALL BITWISE EQUAL" if bad == 0 else f"{bad} tensors differ")
    return bad


if __name__ == "__main__":
    if sys.argv[1] == "cmp":
        sys.exit(1 if cmp() else 0)
    dump(sys.argv[1])
