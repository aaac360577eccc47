"""M2 (all-at-once Newton) on the device vs the reference's solve_m2_newton
(oracle/_ref, host cores) from the same static_init U0; prints one JSON line
per config."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import ref  # noqa: E402
from paper_2502_21013_b200 import Problem, baseline_desc, default_cfg  # noqa: E402

for config in [int(c) for c in (sys.argv[1:] or ["0"])]:
    cfg = default_cfg(tol=1e-8)
    d = baseline_desc(config)
    with Problem(d) as p:
        U0, counts = p.static_init(cfg)
        p.solve_m2_newton(U0, cfg)  # warm (module loading, allocations)
        t = time.perf_counter()
        U, rep = p.solve_m2_newton(U0, cfg)
        dev_s = time.perf_counter() - t
    out = dict(config=config, dof=int(np.prod(U0.shape)), device_s=dev_s, device_iterations=rep.iterations,
               device_fgmres_total=rep.inner_iterations, device_history=rep.residual_history)
    if config == 0 or os.environ.get("M2_REF_ALL"):
        Ur, hr, kr, st, wall = ref.solve_m2(ref.baseline_desc(config), U0, cfg)
        out.update(ref_s=wall, ref_iterations=kr, ref_history=hr.tolist(),
                   rel_err_U=float(np.linalg.norm(U - Ur) / np.linalg.norm(Ur)), ref_threads=ref.hardware_threads())
    print(json.dumps(out), flush=True)
