"""Time the general-mesh sweep (device-resident, tp_mesh_m1_sweep) on the
reference's transformer problem; under ncu (--profile-from-start off) only the
timed sweeps are captured.

    python tools/profile_mesh.py [--refinements 0] [--steps 64] [--sweeps 10]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_21013_b200.abi import default_cfg  # noqa: E402
from paper_2502_21013_b200.mesh import MeshProblem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nx", type=int, default=40)
ap.add_argument("--refinements", type=int, default=0)
ap.add_argument("--steps", type=int, default=64)
ap.add_argument("--sweeps", type=int, default=10)
ap.add_argument("--j-amp", type=float, default=9.5e5)
a = ap.parse_args()
cfg = default_cfg(tol=1e-8)
p = MeshProblem.transformer(a.nx, a.nx, a.refinements, a.steps, 0.02, j_amp=a.j_amp)
t = time.perf_counter()
p.static_init(cfg)
ti = time.perf_counter() - t
p.choose_nu_hat(cfg)
t = time.perf_counter()
r0 = p.m1_begin(cfg)
tb = time.perf_counter() - t
p.m1_sweep()  # warm
try:
    import torch
    torch.cuda.cudart().cudaProfilerStart()
except Exception:
    torch = None
ts = []
for _ in range(a.sweeps):
    t = time.perf_counter()
    r = p.m1_sweep()
    ts.append(time.perf_counter() - t)
if torch is not None:
    torch.cuda.cudart().cudaProfilerStop()
D = p.n_dof * p.steps
print(f"n={p.n_dof} N={p.steps} bw={p.bandwidth} static_init {ti:.3f}s begin(factor+resid) {tb:.3f}s "
      f"sweep median {1e3 * np.median(ts):.3f} ms ({D / np.median(ts):.3e} DoF/s) launches {p.launches}")
