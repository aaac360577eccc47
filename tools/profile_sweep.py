"""Profiling driver: set up a BASELINE config, run warm-up sweeps, then run
`--sweeps` sweeps inside cudaProfilerStart/Stop (use ncu --profile-from-start off)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_21013_b200 import Problem, baseline_desc, default_cfg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--sweeps", type=int, default=1)
a = ap.parse_args()
cfg = default_cfg(tol=1e-8)
p = Problem(baseline_desc(a.config))
p.static_init(cfg, want_state=False)
p.choose_nu_hat(cfg)
p.m1_begin(cfg)
for _ in range(a.warmup):
    p.m1_sweep()
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(a.sweeps):
    r, it = p.m1_sweep()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("residual", r, "inner", it, "frequency_iterations", p.sweep_stats()[1])
