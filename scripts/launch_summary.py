"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes]) by kernel class."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[i]
ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
idi = hdr.index("ID")
per = collections.defaultdict(dict)
names = {}
for r in rows[i + 1:]:
    v = float(r[vi].replace(",", ""))
    u = r[ui]
    if u == "ns":
        v /= 1e3
    elif u == "ms":
        v *= 1e3
    elif u == "Kbyte":
        v *= 1e3
    elif u == "Mbyte":
        v *= 1e6
    elif u == "Gbyte":
        v *= 1e9
    per[r[idi]][r[mi]] = v
    names[r[idi]] = r[ki]
cls = collections.defaultdict(lambda: [0.0, 0, 0.0])
for i_, m in per.items():
    n = re.sub(r"\(.*", "", names[i_]).replace("void ", "").replace("(anonymous namespace)::", "")
    t = m.get("gpu__time_duration.sum", 0.0)
    b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    cls[n][0] += t
    cls[n][1] += 1
    cls[n][2] += b
tot = sum(v[0] for v in cls.values())
print(f"total {tot:.1f} us over {sum(v[1] for v in cls.values())} launches")
for n, (t, c, b) in sorted(cls.items(), key=lambda x: -x[1][0]):
    print(f"{t:9.1f} us {t / tot * 100:5.1f}% {c:4d}x  {b / 1e6:9.1f} MB {b / (t * 1e-6) / 1e9 if t else 0:7.0f} GB/s  {n[:90]}")
