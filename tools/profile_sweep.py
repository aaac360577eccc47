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
ap.add_argument("--timer", type=int, default=-1, help="tp_kernel_timer_select kind to count algorithmic bytes of")
a = ap.parse_args()
cfg = default_cfg(tol=1e-8)
p = Problem(baseline_desc(a.config))
p.static_init(cfg, want_state=False)
p.choose_nu_hat(cfg)
p.m1_begin(cfg)
for _ in range(a.warmup):
    p.m1_sweep()
torch.cuda.synchronize()
if a.timer >= 0:
    p.kernel_timer_select(a.timer)
    p.kernel_timer(True)
torch.cuda.profiler.start()
for _ in range(a.sweeps):
    r, it = p.m1_sweep()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("residual", r, "inner", it, "frequency_iterations", p.sweep_stats()[1])
if a.timer >= 0:
    nl, ms, by = p.kernel_timer(False)
    print("timer", a.timer, "launches", nl, "algorithmic_bytes", by)
# the byte model of bench.py for this sweep
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
d = baseline_desc(a.config)
n, N = (d.cells - 1) ** 2, d.steps
b_alg = 72.0 * n * N + 16.0 * n * (3.0 * (N // 2 + 1) + bench.streams_per_iteration(d.cells - 1) * p.sweep_stats()[1])
print("sweep_algorithmic_bytes", b_alg)
