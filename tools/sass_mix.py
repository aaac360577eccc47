"""Instruction mix and stall hot spots of one kernel from an ncu source-page
CSV (ncu -i X.ncu-rep --page source --csv): executed warp instructions per
opcode class, and the SASS lines with the most stall samples.
Usage: python tools/sass_mix.py source_TAG.csv [top]"""
import csv
import collections
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ie, ss = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
mix, tot, hot = collections.Counter(), 0, []
for r in rows[2:]:
    if len(r) <= ie:
        continue
    src = r[1].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    try:
        n, s = int(r[ie]), int(r[ss])
    except ValueError:
        continue
    mix[op.split(".")[0]] += n
    tot += n
    hot.append((s, src))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
print(f"executed warp instructions {tot:.4g}")
for op, n in mix.most_common(top):
    print(f"  {op:10s} {n / tot * 100:5.1f}%")
print("hottest lines (stall samples):")
for s, src in sorted(hot, reverse=True)[:15]:
    print(f"  {s:8d}  {src}")
