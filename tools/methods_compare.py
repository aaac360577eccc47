"""M1 / M2 / M3 on the device vs the reference's solvers (oracle/_ref, all
host cores) from the same static_init U0; one JSON line per (config, method).
Reference runs only where they finish quickly (cfg 0; cfg >= 1 device only,
M3 there limited to --m3-cycles periods)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import ref  # noqa: E402
from paper_2502_21013_b200 import Problem, baseline_desc, default_cfg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("configs", nargs="*", type=int, default=[0])
ap.add_argument("--m3-cycles", type=int, default=1)
a = ap.parse_args()
for config in a.configs:
    cfg = default_cfg(tol=1e-8)
    if config > 0:
        cfg.m3_max_cycles = a.m3_cycles
    d = baseline_desc(config)
    with Problem(d) as p:
        U0, _ = p.static_init(cfg)
        nu, q = p.choose_nu_hat(cfg)
        for meth in ["m1", "m2", "m3"]:
            fn = {"m1": p.solve_m1_fixed_point, "m2": p.solve_m2_newton, "m3": p.solve_m3_timestepping}[meth]
            if meth != "m1":
                fn(U0, cfg)  # warm
            t = time.perf_counter()
            U, rep = fn(U0, cfg)
            dev_s = time.perf_counter() - t
            out = dict(config=config, method=meth, device_s=dev_s, iterations=rep.iterations, status=rep.status,
                       history=rep.residual_history)
            if config == 0:
                rd = ref.baseline_desc(0)
                if meth == "m1":
                    r1 = ref.solve_m1(rd, nu, q, U0, cfg)
                    Ur, hr, kr, wall = r1.U, r1.history, r1.iterations, r1.wall_time
                else:
                    Ur, hr, kr, _, wall = (ref.solve_m2 if meth == "m2" else ref.solve_m3)(rd, U0, cfg)
                out.update(ref_s=wall, ref_iterations=int(kr), ref_threads=ref.hardware_threads(),
                           rel_err_U=float(np.linalg.norm(U - Ur) / np.linalg.norm(Ur)))
            print(json.dumps(out), flush=True)
