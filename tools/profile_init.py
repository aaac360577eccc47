"""Profiling driver for static_init: one warm-up static_init, then one inside
cudaProfilerStart/Stop (use ncu --profile-from-start off); prints its time and
the Newton counts summary."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_21013_b200 import Problem, baseline_desc, default_cfg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
a = ap.parse_args()
cfg = default_cfg(tol=1e-8)
p = Problem(baseline_desc(a.config))
p.static_init(cfg, want_state=False)
torch.cuda.synchronize()
torch.cuda.profiler.start()
t = time.perf_counter()
out = p.static_init(cfg, want_state=False)
torch.cuda.synchronize()
dt = time.perf_counter() - t
torch.cuda.profiler.stop()
counts = out[1] if isinstance(out, tuple) else out
try:
    c = np.asarray(counts)
    print(f"static_init {dt*1e3:.1f} ms; newton counts min {c.min()} max {c.max()} sum {c.sum()}")
except Exception:
    print(f"static_init {dt*1e3:.1f} ms")
