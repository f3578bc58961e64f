"""Summarise ncu captures into profiles/ (run here, on the CPU side).

  python scripts/ncu_summary.py <launch-list.csv> <full-report.ncu-rep:key> ...

Writes profiles/ncu_summary.json: per-kernel {duration_us, dram_bytes (read+write), tensor pipe %,
L2/DRAM throughput %} from the --set full reports, and the per-kernel-class time shares of the
launch list (gpu__time_duration.sum, one step)."""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "ncu_summary.json")
WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_tc_pct",
    "launch__grid_size": "grid",
    "launch__registers_per_thread": "regs",
}
SCALE = {"us": 1.0, "ns": 1e-3, "ms": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def full_report(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {"kernel": vals[hdr.index("Kernel Name")]}
    for k, name in WANT.items():
        if k in hdr:
            i = hdr.index(k)
            v = float(vals[i].replace(",", ""))
            u = units[i]
            if name == "duration":
                v *= SCALE.get(u, 1.0)
                name = "duration_us"
            elif name.startswith("dram_"):
                v *= SCALE.get(u, 1.0)
            out[name] = v
    out["dram_bytes"] = out.pop("dram_read", 0.0) + out.pop("dram_write", 0.0)
    return out


def launch_list(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[h], rows[h + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    mi = hdr.index("Metric Name") if "Metric Name" in hdr else None
    agg, cnt, tot = collections.defaultdict(float), collections.Counter(), 0.0
    for r in data:
        if mi is not None and r[mi] != "gpu__time_duration.sum":
            continue
        t = float(r[vi].replace(",", "")) * (1e-3 if r[ui] in ("ns", "nsecond") else 1e3 if r[ui] == "ms" else 1.0)
        name = r[ki].split("(")[0].replace("void ", "").replace("pbdk::", "").replace("(anonymous namespace)::", "")
        name = name.replace("<unnamed>::", "")
        agg[name] += t
        cnt[name] += 1
        tot += t
    return {"total_us": tot, "launches": sum(cnt.values()),
            "classes": [{"kernel": k, "us": v, "share": v / tot, "launches": cnt[k]}
                        for k, v in sorted(agg.items(), key=lambda x: -x[1])]}


def main():
    summary = {"kernels": {}}
    if os.path.exists(OUT):
        summary = json.load(open(OUT))
    for arg in sys.argv[1:]:
        if arg.endswith(".csv"):
            summary["launch_list"] = launch_list(arg)
            summary["launch_list"]["source"] = os.path.basename(arg)
        else:
            path, key = arg.rsplit(":", 1)
            summary.setdefault("kernels", {})[key] = full_report(path) | {"source": os.path.basename(path)}
    json.dump(summary, open(OUT, "w"), indent=1)
    print(json.dumps(summary, indent=1)[:3000])


if __name__ == "__main__":
    main()
