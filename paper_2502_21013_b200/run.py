"""Command-line solve of a BASELINE configuration, writing the reference
runner's output files (report.json, residuals.csv; runner.hpp:174-223).

    python -m paper_2502_21013_b200.run --config 1 --out out/cfg1 [--tol 1e-8]

static_init (U0) -> frozen-field nu_hat -> M1 fixed-point iteration on the
device, then report.json / residuals.csv in the reference's formats
(paper_2502_21013_b200/report.py).  Exit code 0 when M1 converged, 2
otherwise (runner.hpp:100-104).
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np


def main(argv=None) -> int:
    from . import Problem, baseline_desc, default_cfg
    from . import report as R

    ap = argparse.ArgumentParser(prog="python -m paper_2502_21013_b200.run")
    ap.add_argument("--config", type=int, default=0, help="BASELINE config 0..5")
    ap.add_argument("--out", required=True, help="output directory")
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--max-outer", type=int, default=200)
    ap.add_argument("--cells", type=int, default=0, help="override the grid (cells per side)")
    ap.add_argument("--steps", type=int, default=0, help="override N")
    ap.add_argument("--u0", choices=["static_init", "zero"], default="static_init")
    ap.add_argument("--device", type=int, default=0)
    ap.add_argument("--methods", default="m1", help="comma list of m1, m2, m3 (run from the same U0)")
    a = ap.parse_args(argv)

    desc = baseline_desc(a.config)
    if a.cells:
        desc.cells = a.cells
    if a.steps:
        desc.steps = a.steps
    cfg = default_cfg(tol=a.tol, m1_max_outer=a.max_outer)
    with Problem(desc, device=a.device) as p:
        t0 = time.perf_counter()
        if a.u0 == "static_init":
            U0, counts = p.static_init(cfg)
            newton_max = int(np.max(counts)) if len(counts) else 0
        else:
            U0, newton_max = np.zeros(p.shape), 0
        if a.u0 == "zero":
            p.set_state(U0)
        nu, q = p.choose_nu_hat(cfg)
        init_s = time.perf_counter() - t0
        print(f"grid: {p.shape[1]} unknowns, {desc.steps} steps, initialization {R.format_double(init_s)} s")
        reports = []
        for meth in [x.strip() for x in a.methods.split(",") if x.strip()]:
            if meth == "m1":
                _, rep = p.solve_m1_fixed_point(U0, cfg)
            elif meth == "m2":
                _, rep = p.solve_m2_newton(U0, cfg)
            elif meth == "m3":
                _, rep = p.solve_m3_timestepping(U0, cfg)
            else:
                raise SystemExit(f"unknown method {meth!r} (m1, m2, m3)")
            unit = "cycles" if meth == "m3" else "iterations"
            print(f"{meth}: {rep.status} after {rep.iterations} {unit} ({R.format_double(rep.wall_time)} s), "
                  f"residual {R.format_double(rep.residual_history[-1])}")
            reports.append((meth, rep))
        tau = desc.period / desc.steps
        j = R.run_report(desc, desc.steps, p.shape[1], tau, cfg.threads, nu, q, init_s, newton_max,
                         R.symbol_abs(desc.steps, tau), {mm: R.report_to_dict(r, mm) for mm, r in reports})
    R.ensure_dir(a.out)
    R.write_json(os.path.join(a.out, "report.json"), j)
    R.write_residuals_csv(os.path.join(a.out, "residuals.csv"), reports)
    return R.exit_code([r.status for _, r in reports])


if __name__ == "__main__":
    sys.exit(main())
