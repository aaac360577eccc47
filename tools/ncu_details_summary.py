"""Print the metrics of an `ncu --page details --csv` export as
'section / metric = value unit' lines (one kernel launch per file)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0]
si, mi, ui, vi = (hdr.index(k) for k in ("Section Name", "Metric Name", "Metric Unit", "Metric Value"))
ki = hdr.index("Kernel Name")
print(rows[1][ki][:120])
for r in rows[1:]:
    if len(r) > vi and r[mi]:
        print(f"{r[si][:28]:28s} {r[mi][:44]:44s} {r[vi]:>14s} {r[ui]}")
