"""static_init time against the slice-mode smoother's Chebyshev interval:
for each [lo, hi] the degree-2 weights 1/x_k, x_k = (hi+lo)/2 + (hi-lo)/2
cos((2k-1) pi/4), set through TPGPU_NEWTON_OMEGA / _OMEGA2 (read per call).
Prints the time and whether the Newton counts equal the default run's.
Usage: python tools/init_omega_sweep.py --config 2
"""
import argparse
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2502_21013_b200 import Problem, baseline_desc, default_cfg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--intervals", nargs="+",
                default=["0.1667,1", "0.25,1", "0.125,1", "0.1,1", "0.0667,1", "0.1667,1.1", "0.1,1.1"])
a = ap.parse_args()
cfg = default_cfg(tol=1e-8)


def weights(lo, hi):
    c, r = (hi + lo) / 2, (hi - lo) / 2
    return 1 / (c + r * math.cos(math.pi / 4)), 1 / (c - r * math.cos(math.pi / 4))


with Problem(baseline_desc(a.config)) as p:
    p.static_init(cfg, want_state=False)
    t = time.perf_counter()
    _, c0 = p.static_init(cfg, want_state=False)
    print(f"cfg {a.config} default: {time.perf_counter() - t:.3f} s newton sum {c0.sum()}", flush=True)
    for iv in a.intervals:
        lo, hi = map(float, iv.split(","))
        w1, w2 = weights(lo, hi)
        os.environ["TPGPU_NEWTON_OMEGA"] = repr(w1)
        os.environ["TPGPU_NEWTON_OMEGA2"] = repr(w2)
        t = time.perf_counter()
        _, c = p.static_init(cfg, want_state=False)
        dt = time.perf_counter() - t
        print(f"cfg {a.config} interval [{lo}, {hi}] omegas {w1:.4f} {w2:.4f}: {dt:.3f} s "
              f"counts_equal {bool(np.array_equal(c, c0))}", flush=True)
