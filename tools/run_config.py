"""Run one BASELINE config end to end on cuda:0: static_init, frozen-field
nu_hat, M1 sweeps to the tolerance (or --max-sweeps), with timings."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_21013_b200 import Problem, baseline_desc, default_cfg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--max-sweeps", type=int, default=200)
ap.add_argument("--tol", type=float, default=1e-8)
ap.add_argument("--u0", choices=["static", "zero"], default="static")
ap.add_argument("--inner-rtol", type=float, default=1e-12)
a = ap.parse_args()
d = baseline_desc(a.config)
cfg = default_cfg(tol=a.tol, m1_max_outer=a.max_sweeps, inner_rtol=a.inner_rtol)
t0 = time.perf_counter()
p = Problem(d)
torch.cuda.synchronize()
t_create = time.perf_counter() - t0
t0 = time.perf_counter()
if a.u0 == "static":
    _, counts = p.static_init(cfg, want_state=False)
else:
    import numpy as np
    p.set_state(np.zeros((p.steps, p.n_dof)))
    counts = np.zeros(1, dtype=int)
t_init = time.perf_counter() - t0
nu, q = p.choose_nu_hat(cfg)
t0 = time.perf_counter()
r0 = p.m1_begin(cfg)
torch.cuda.synchronize()
t_setup = time.perf_counter() - t0
hist, its, times, fits = [r0], [], [], []
while len(its) < a.max_sweeps and not hist[-1] <= a.tol * hist[0]:
    t = time.perf_counter()
    r, it = p.m1_sweep()
    torch.cuda.synchronize()
    times.append(time.perf_counter() - t)
    hist.append(r)
    its.append(it)
    fits.append(p.sweep_stats()[1])
free, total = torch.cuda.mem_get_info()
D = p.n_dof * p.steps
out = dict(config=a.config, u0=a.u0, inner_rtol=a.inner_rtol, cells=d.cells, steps=d.steps, n=p.n_dof, D=D, create_s=t_create, init_s=t_init,
           newton_max=int(counts.max()), nu_hat=list(nu), q=q, setup_s=t_setup, sweeps=len(its),
           converged=bool(hist[-1] <= a.tol * hist[0]), median_sweep_s=sorted(times)[len(times) // 2] if times else None,
           dof_per_s=D / sorted(times)[len(times) // 2] if times else None, inner=its, frequency_iterations=fits,
           history=hist,
           time_to_residual_s=t_init + t_setup + sum(times), gpu_mem_used_gb=(total - free) / 1e9)
print(json.dumps(out))
