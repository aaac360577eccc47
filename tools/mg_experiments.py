"""Inner-solver experiments: parity margin and cost vs inner_rtol / smoother.
Env TPGPU_OMEGA / TPGPU_RB_FINE are read by the library."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_21013_b200 import Problem, baseline_desc, default_cfg  # noqa: E402

g = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "cfg0_reference.npz"))
for rtol in [float(x) for x in sys.argv[1:]] or [1e-13]:
    cfg = default_cfg(tol=1e-8, inner_rtol=rtol)
    if os.environ.get("FG"):
        cfg.freq_groups = int(os.environ["FG"])
    with Problem(baseline_desc(0)) as p:
        p.set_nu_hat(g["nu_hat"], float(g["q"]))
        log = []
        U, rep = p.solve_m1_fixed_point(g["U0"], cfg, iterate_log=log)
        e1 = np.linalg.norm(log[1] - g["U1"]) / np.linalg.norm(g["U1"])
        e2 = np.linalg.norm(log[2] - g["U2"]) / np.linalg.norm(g["U2"])
        ef = np.linalg.norm(U - g["U"]) / np.linalg.norm(g["U"])
    with Problem(baseline_desc(1)) as p:
        p.static_init(cfg, want_state=False)
        p.choose_nu_hat(cfg)
        p.m1_begin(cfg)
        its, fits = [], []
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(20):
            its.append(p.m1_sweep()[1])
            fits.append(p.sweep_stats()[1])
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / 20
    print(f"rtol {rtol:.0e} omega {os.environ.get('TPGPU_OMEGA','0.8')} rb {os.environ.get('TPGPU_RB_FINE','1')}: "
          f"cfg0 iters {rep.iterations} (ref {int(g['iterations'])}) err U1 {e1:.1e} U2 {e2:.1e} final {ef:.1e}"
          f" | cfg1 inner {its[:6]}.. mean {np.mean(its):.1f}, f-its {np.mean(fits):.0f}, {dt*1e3:.2f} ms/sweep",
          flush=True)
