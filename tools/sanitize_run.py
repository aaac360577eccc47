"""Small end-to-end run for compute-sanitizer (memcheck / racecheck /
synccheck): BASELINE config 0 static_init -> nu_hat -> 3 M1 sweeps (the
streaming passes with their cp.async rings, the small-level fused cycle, the
DFTs, the fused residual) and one general-mesh M1 sweep on the reference's
transformer mesh.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2502_21013_b200 import Problem, baseline_desc, default_cfg  # noqa: E402
from paper_2502_21013_b200.mesh import MeshProblem  # noqa: E402

cfg = default_cfg(tol=1e-8, m1_max_outer=3)
with Problem(baseline_desc(0)) as p:
    U0, counts = p.static_init(cfg)
    p.choose_nu_hat(cfg)
    U, rep = p.solve_m1_fixed_point(None, cfg)
    print("grid: sweeps", rep.iterations, "residual", rep.residual_history[-1])
with MeshProblem.transformer(12, 10, 0, 8, 0.02, j_amp=9.5e5) as mp:
    mp.static_init(cfg)
    mp.choose_nu_hat(cfg)
    _, mrep = mp.solve_m1_fixed_point(None, default_cfg(tol=1e-8, m1_max_outer=1))
    print("mesh: sweeps", mrep.iterations)
print("sanitize run done")
