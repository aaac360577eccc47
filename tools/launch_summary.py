"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
tot = defaultdict(float)
cnt = defaultdict(int)
dram = defaultdict(float)
for r in rows[hdr_i + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].replace("void ", "")
    name = name.split("<")[0] + ("<" + r[ki].split("<")[1].split(">")[0] + ">" if "<" in r[ki] else "")
    v = float(r[vi].replace(",", ""))
    unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else ""
    if r[mi] == "gpu__time_duration.sum":
        tot[name] += v * (1e3 if unit == "us" else 1e6 if unit == "ms" else 1.0)
        cnt[name] += 1
    elif r[mi] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
        dram[name] += v * scale
all_t = sum(tot.values())
print(f"{'kernel':60s} {'launches':>8s} {'total_us':>10s} {'share':>7s} {'dram_MB':>10s} {'GB/s':>8s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k[:60]:60s} {cnt[k]:8d} {v/1e3:10.1f} {100*v/all_t:6.1f}% {dram[k]/1e6:10.1f} {dram[k]/max(v,1e-9):8.1f}")
print(f"{'TOTAL':60s} {sum(cnt.values()):8d} {all_t/1e3:10.1f}        {sum(dram.values())/1e6:10.1f}")
