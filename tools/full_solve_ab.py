"""A/B of a full cfg-1 M1 solve to 1e-8 (sweep count, total sweep time,
frequency-iterations); env knobs are read by the library."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_21013_b200 import Problem, baseline_desc, default_cfg  # noqa: E402

cfgi = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cfg = default_cfg(tol=1e-8)
with Problem(baseline_desc(cfgi)) as p:
    U0, _ = p.static_init(cfg)
    p.choose_nu_hat(cfg)
    for rep in range(2):
        p.set_state(U0)
        r0 = p.m1_begin(cfg)
        hist, fits = [r0], []
        torch.cuda.synchronize()
        t = time.perf_counter()
        while len(fits) < cfg.m1_max_outer and not hist[-1] <= cfg.tol * hist[0]:
            r, it = p.m1_sweep()
            hist.append(r)
            fits.append(p.sweep_stats()[1])
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(f"{os.environ.get('TPGPU_EXTRAP', '-')}: sweeps {len(fits)} time {dt:.3f} s "
          f"({dt / len(fits) * 1e3:.2f} ms/sweep) f-its mean {np.mean(fits):.0f} final {hist[-1] / hist[0]:.2e}",
          flush=True)
