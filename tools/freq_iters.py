"""Experiment: per-frequency inner iteration counts and ||g_k|| along a cfg-1
M1 solve (run with TPGPU_DEBUG_FREQ=1; the library prints one line per group
solve to stderr)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_21013_b200 import Problem, baseline_desc, default_cfg  # noqa: E402

cfgi = int(sys.argv[1]) if len(sys.argv) > 1 else 1
nsw = int(sys.argv[2]) if len(sys.argv) > 2 else 170
cfg = default_cfg(tol=1e-8)
with Problem(baseline_desc(cfgi)) as p:
    p.static_init(cfg, want_state=False)
    p.choose_nu_hat(cfg)
    r0 = p.m1_begin(cfg)
    for s in range(nsw):
        print(f"sweep {s}", file=sys.stderr, flush=True)
        r, it = p.m1_sweep()
        print(f"sweep {s} residual {r:.3e} iters {it}", file=sys.stderr, flush=True)
