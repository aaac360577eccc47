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
for r in rows[hdr_i + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0].replace("void ", "")
    name = name.split("<")[0] + ("<" + r[ki].split("<")[1].split(">")[0] + ">" if "<" in r[ki] else "")
    tot[name] += float(r[vi].replace(",", ""))
    cnt[name] += 1
all_t = sum(tot.values())
print(f"{'kernel':60s} {'launches':>8s} {'total_us':>10s} {'share':>7s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k[:60]:60s} {cnt[k]:8d} {v/1e3:10.1f} {100*v/all_t:6.1f}%")
print(f"{'TOTAL':60s} {sum(cnt.values()):8d} {all_t/1e3:10.1f}")
