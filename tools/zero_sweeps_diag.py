"""Diagnostics for tests/test_gpu_parity_large.py::test_sweeps_from_zero_match_reference:
the same run, printing every agreement figure instead of asserting (residual
history against the reference's, per-iterate norm / sample errors), for the
default inner tolerance and the ones given.
Usage: python tools/zero_sweeps_diag.py --config 4 --inner 1e-12 1e-13
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

from paper_2502_21013_b200 import Problem, baseline_desc, default_cfg  # noqa: E402
from paper_2502_21013_b200.abi import TP_NU_HAT_THEORY  # noqa: E402
from test_gpu_parity_large import Digests, rel  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--inner", type=float, nargs="+", default=[1e-12])
a = ap.parse_args()
name = {5: "cfg5_sweeps_reference.npz", 4: "cfg4_sweeps_reference.npz", 2: "cfg2_sweeps_reference.npz"}[a.config]
g = np.load(os.path.join(ROOT, "tests", "golden", name))
count = int(g["iterations"])
with Problem(baseline_desc(a.config)) as p:
    for inner in a.inner:
        cfg = default_cfg(tol=1e-12, m1_max_outer=count, nu_hat_mode=TP_NU_HAT_THEORY)
        cfg.inner_rtol = inner
        U0 = np.zeros(p.shape)
        p.set_state(U0)
        p.choose_nu_hat(cfg)
        dig = Digests(int(g["stride"]))
        U, rep = p.solve_m1_fixed_point(U0, cfg, callback=dig)
        h, hr = np.asarray(rep.residual_history), g["history"]
        print(f"cfg {a.config} inner_rtol {inner:g}: iterations {rep.iterations} (ref {count})")
        print("  history |h-hr|/hr[0]:", " ".join(f"{x:.2e}" for x in np.abs(h - hr) / hr[0]))
        print("  history |h-hr|/hr   :", " ".join(f"{x:.2e}" for x in np.abs(h - hr) / hr))
        gd, gs = g["digests"], g["samples"]
        for k, (row, smp) in enumerate(zip(dig.rows, dig.samples)):
            print(f"  iterate {k}: norm {abs(row[0] - gd[k, 0]) / gd[k, 0]:.2e}  step "
                  f"{abs(row[4] - gd[k, 4]) / gd[k, 0]:.2e}  sample {rel(smp, gs[k]):.2e}", flush=True)
