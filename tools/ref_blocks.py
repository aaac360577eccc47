"""Measure the reference's frequency-block stage on this host (test
infrastructure: oracle/_ref, the reference's own PeriodicSolver pieces).

At configs >= 2 a reference sweep factorises every one of the N/2+1 blocks
lambda_k M + K_hat (cache = never: periodic.hpp:211-248 decides so when the
factors exceed the 1.5 GiB budget), one block per worker thread.  This runs
`--blocks` of them concurrently (tpref_sweep_sample stage C: assemble,
factorise, solve, residual contract) and records the wall time of that round
in profiles/r2_ref_blocks.json, which bench.py's reference arm uses for the
block stage (rounds = ceil((N/2+1) / threads)).  Measuring fewer concurrent
blocks than the host has threads leaves out memory-bandwidth contention
between workers, which makes the reference look faster, not slower.

    python tools/ref_blocks.py --config 3 --blocks 4
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import ref  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--blocks", type=int, default=4)
a = ap.parse_args()
ref.select("relaxed")  # the 1e-10 contract is below the fp64 residual floor at these sizes
d = ref.baseline_desc(a.config)
nu = np.ones(5)
for m in range(d.n_materials):
    nu[m] = 0.5 * (d.material[m].nu0 + d.material[m].nu_inf)
t0 = time.time()
samples, setup = ref.sweep_sample(d, nu, 1, 1, a.blocks, threads=a.blocks, reps=1)
wall = samples[0]["C_blocks"]
path = os.path.join(ROOT, "profiles", "r2_ref_blocks.json")
data = json.load(open(path)) if os.path.exists(path) else {}
data[f"cfg{a.config}"] = {"concurrent_blocks_measured": a.blocks, "concurrent_blocks": ref.hardware_threads(),
                          "round_wall_s": wall, "host_threads": ref.hardware_threads(),
                          "note": f"{a.blocks} complex blocks (k = 1..{a.blocks}) factorised + solved concurrently on "
                                  f"{a.blocks} threads took round_wall_s; a full-host round of "
                                  f"{ref.hardware_threads()} concurrent blocks is assumed to take the same time "
                                  "(no bandwidth contention: favours the reference)",
                          "setup_s": setup, "total_s": time.time() - t0}
json.dump(data, open(path, "w"), indent=1)
print(json.dumps(data[f"cfg{a.config}"]))
