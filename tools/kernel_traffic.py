"""Write profiles/kernel_traffic.json's entry for one config from an ncu
launch list of one production sweep (tools/ncu_launch_list.sh): the sweep's
DRAM bytes over its algorithmic bytes (bench.py's byte model, printed by
tools/profile_sweep.py) and the same ratio for the dominant kernel (the
fine-level down pass, whose algorithmic bytes the library's kernel timer
counted in that sweep).

    python tools/kernel_traffic.py CONFIG gpurun_out/launches_TAG_cfgC.csv gpurun_out/ncu_TAG_cfgC.log
"""
import csv
import json
import os
import sys

cfg, csv_path, log_path = int(sys.argv[1]), sys.argv[2], sys.argv[3]
rows = list(csv.reader(open(csv_path)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
idi = h.index("ID")
gi = h.index("Grid Size")
sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
total = 0.0
down = 0.0
fine_grid = None
launch = {}
for r in rows[hi + 1:]:
    if len(r) <= vi or r[mi] not in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        continue
    b = float(r[vi].replace(",", "")) * sc.get(r[ui], 1)
    total += b
    if "k_stream_down" in r[ki] and "Five" in r[ki]:
        launch.setdefault(r[idi], [r[gi], 0.0])[1] += b
# the fine-level down launches are the ones with the largest grid
grids = {}
for g, b in launch.values():
    n = int(g.strip("()").split(",")[0])
    grids.setdefault(n, []).append(b)
fine = max(grids)
down = sum(grids[fine])
log = open(log_path).read().split()
alg_sweep = float(log[log.index("sweep_algorithmic_bytes") + 1])
alg_down = float(log[log.index("algorithmic_bytes") + 1])
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "kernel_traffic.json")
data = json.load(open(path)) if os.path.exists(path) else {}
data[f"cfg{cfg}"] = {"sweep_dram_bytes": total, "sweep_algorithmic_bytes": alg_sweep,
                     "sweep_dram_over_algorithmic": total / alg_sweep,
                     "dominant_kernel": "k_stream_down<Five>", "dominant_kernel_dram_bytes": down,
                     "dominant_kernel_algorithmic_bytes": alg_down,
                     "dominant_kernel_dram_over_algorithmic": down / alg_down,
                     "source": os.path.basename(csv_path)}
json.dump(data, open(path, "w"), indent=1)
print(json.dumps(data[f"cfg{cfg}"], indent=1))
