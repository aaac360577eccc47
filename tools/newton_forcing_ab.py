"""A/B of the static_init linear tolerances (inexact Newton forcing terms).

For each config: one static_init at the default Newton linear tolerance (the
reference's 1e-10 contract, pinned by the parity tests), then one per
TPGPU_NEWTON_FORCING setting; prints the time, the Newton counts against the
default run, and the relative difference of U0 (and of U0 per slice, max).
Usage: python tools/newton_forcing_ab.py --configs 1 2 --settings 1e-2,1,1e-2 ...
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2502_21013_b200 import Problem, baseline_desc, default_cfg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", type=int, nargs="+", default=[1, 2])
ap.add_argument("--settings", nargs="+", default=["1e-2,1e-2"])
ap.add_argument("--repeat", type=int, default=1)
a = ap.parse_args()
cfg = default_cfg(tol=1e-8)


def run(p, setting):
    if setting:
        os.environ["TPGPU_NEWTON_FORCING"] = setting
    else:
        os.environ.pop("TPGPU_NEWTON_FORCING", None)
    best = None
    for _ in range(a.repeat):
        t = time.perf_counter()
        U0, counts = p.static_init(cfg)
        dt = time.perf_counter() - t
        best = dt if best is None else min(best, dt)
    return U0, counts, best


for c in a.configs:
    with Problem(baseline_desc(c)) as p:
        p.static_init(cfg, want_state=False)  # warm-up
        U_ref, c_ref, t_ref = run(p, "0")
        print(f"cfg {c} exact (forcing off): {t_ref:.3f} s  newton sum {c_ref.sum()} max {c_ref.max()}", flush=True)
        nrm = np.linalg.norm(U_ref)
        for s in a.settings:
            U, cnt, dt = run(p, s)
            rel = float(np.linalg.norm(U - U_ref) / nrm)
            per = np.linalg.norm(U - U_ref, axis=1) / np.maximum(np.linalg.norm(U_ref, axis=1), 1e-300)
            print(f"cfg {c} forcing {s}: {dt:.3f} s  counts_equal {bool(np.array_equal(cnt, c_ref))} "
                  f"(diff slices {int((cnt != c_ref).sum())})  relU {rel:.2e}  max_slice {per.max():.2e}", flush=True)
        del U_ref
