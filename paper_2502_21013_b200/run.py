"""Command-line solve of a BASELINE configuration, writing the reference
runner's output files (report.json, residuals.csv; runner.hpp:174-223).

    python -m paper_2502_21013_b200.run --config 1 --out out/cfg1 [--tol 1e-8]
    python -m paper_2502_21013_b200.run --ref-config configs/transformer.json [--out dir]

The second form reads the reference's own run configs (problem "transformer":
parse_run_config, config.hpp:176-230 -- method m1/m2/m3/all, nx, ny,
refinements, steps, period, solver, flux, materials) and runs them on the
general-mesh path (mesh.py): setup_transformer + run_transformer_method
(runner.hpp:46-89), with the VTK mesh / fields when the config asks for
them (vtk.hpp); configs with a "sweep" run `tpfem table` (runner.hpp:235-269).

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


SOLVER_KEYS = {"tol": "tol", "max_outer_m1": "m1_max_outer", "max_outer_m2": "m2_max_outer",
               "m3_max_cycles": "m3_max_cycles", "static_tol": "static_tol", "static_max_newton": "static_max_newton",
               "m2_inner_tol": "m2_inner_tol", "m2_inner_max": "m2_inner_max", "m2_restart": "m2_restart",
               "imag_tol": "imag_tol"}


def _ref_setup(j):
    """Solver config, materials and flux settings of a reference run config
    (parse_run_config, config.hpp:176-252)."""
    from . import default_cfg
    from .abi import TP_NU_HAT_THEORY
    from .mesh import REGIONS, transformer_materials

    cfg = default_cfg()
    sv = j.get("solver", {})
    for k, v in sv.items():
        if k in SOLVER_KEYS:
            setattr(cfg, SOLVER_KEYS[k], v)
        elif k == "nu_hat_mode":
            cfg.nu_hat_mode = TP_NU_HAT_THEORY if v == "theory" else 1
        elif k == "armijo":
            cfg.armijo_slope = v.get("slope", cfg.armijo_slope)
            cfg.armijo_backtrack = v.get("backtrack", cfg.armijo_backtrack)
            cfg.armijo_max_halvings = v.get("max_halvings", cfg.armijo_max_halvings)
        elif k == "track_error_contraction":
            cfg.track_error_contraction = 1 if v else 0
    cfg.threads = j.get("threads", cfg.threads)
    mats = transformer_materials()
    for name, entry in j.get("materials", {}).items():  # parse_materials (config.hpp:146-170)
        r = REGIONS.index(name)
        for fld, v in entry.items():
            setattr(mats[r], fld, v)
    return cfg, mats, j.get("flux", {})


def _transformer_setup(j, refinements, steps, device):
    """setup_transformer (runner.hpp:46-73) on the device: mesh, problem,
    static_init, nu_hat; returns (problem, mesh arrays, U0, counts, nu, q, init seconds)."""
    from .mesh import MeshProblem, transformer_mesh

    cfg, mats, flux = _ref_setup(j)
    V, T, Rg, _ = transformer_mesh(j.get("nx", 40), j.get("ny", 40), refinements)
    p = MeshProblem(V, T, Rg, mats, steps, j.get("period", 0.02), flux.get("s_max", 3.0),
                    flux.get("samples", 10001), device=device)
    t0 = time.perf_counter()
    U0, counts = p.static_init(cfg)
    nu, q = p.choose_nu_hat(cfg)
    return p, (V, T, Rg), cfg, U0, counts, nu, q, time.perf_counter() - t0


def _run_method(p, meth, U0, cfg):
    from . import report as R
    fn = {"m1": p.solve_m1_fixed_point, "m2": p.solve_m2_newton, "m3": p.solve_m3_timestepping}[meth]
    U, rep = fn(U0, cfg)
    unit = "cycles" if meth == "m3" else "iterations"
    print(f"{meth}: {rep.status} after {rep.iterations} {unit} ({R.format_double(rep.wall_time)} s), "
          f"residual {R.format_double(rep.residual_history[-1])}")
    return U, rep


def run_table(j, out: str, device: int) -> int:
    """tpfem table (run_table, runner.hpp:235-269): all three methods for every
    (refinements, steps) entry of the sweep, one flushed table.csv row each.
    Returns 0 once the sweep completes (statuses live in the rows, not the
    exit code)."""
    from . import report as R

    R.ensure_dir(out)
    with R.TableWriter(os.path.join(out, "table.csv")) as w:
        for e in j["sweep"]:
            refinements, steps = e.get("refinements", 0), e.get("steps", 64)
            p, _, cfg, U0, counts, nu, q, init_s = _transformer_setup(j, refinements, steps, device)
            with p:
                print(f"sweep: refinements {refinements}, steps {steps}, {p.n_dof} unknowns")
                row = {}
                for meth in ("m1", "m2", "m3"):
                    _, rep = _run_method(p, meth, U0, cfg)
                    row[f"{meth}_iterations"], row[f"{meth}_seconds"] = rep.iterations, rep.wall_time
                w.add_row(steps, p.n_dof, init_s, **row)
    return 0


def run_ref_config(path: str, out: str | None, device: int) -> int:
    """A reference run config (configs/*.json, problem "transformer") on the
    device: `tpfem solve` (run_solve, runner.hpp:174-229) -- report.json,
    residuals.csv, and mesh.vtk / u_<i>.vtk when write_mesh / write_fields are
    set (vtk.hpp) -- or, for configs with a "sweep", `tpfem table`."""
    import json

    from . import report as R
    from .mesh import REGIONS

    j = json.load(open(path))
    if j.get("problem", "transformer") != "transformer":
        raise SystemExit("only problem \"transformer\" runs on the device (the toy problem is out of scope)")
    out = out or j.get("output_dir", ".")
    if "sweep" in j:
        return run_table(j, out, device)
    method = j.get("method", "m1")
    methods = ["m1", "m2", "m3"] if method == "all" else [method]
    refinements, steps, period = j.get("refinements", 0), j.get("steps", 64), j.get("period", 0.02)
    p, (V, T, Rg), cfg, U0, counts, nu, q, init_s = _transformer_setup(j, refinements, steps, device)
    with p:
        print(f"transformer: {p.n_dof} unknowns, {steps} steps, initialization {R.format_double(init_s)} s")
        R.ensure_dir(out)
        if j.get("write_mesh", False):
            R.write_mesh_vtk(os.path.join(out, "mesh.vtk"), V, T, Rg)
        reports, first = [], None
        for meth in methods:
            U, rep = _run_method(p, meth, U0, cfg)
            if first is None:
                first = U
            reports.append((meth, rep))
        tau = period / steps
        rj = {"problem": "transformer", "steps": int(steps), "n_dof": int(p.n_dof), "refinements": int(refinements),
              "period": float(period), "tau": float(tau), "threads": int(cfg.threads),
              "nu_hat": {REGIONS[r]: float(nu[r]) for r in range(5)}, "q_estimate": float(q),
              "init": {"seconds": float(init_s), "max_newton_steps": int(max(counts) if len(counts) else 0)},
              "frequency_symbol_abs": [float(x) for x in R.symbol_abs(steps, tau)],
              "methods": {mm: R.report_to_dict(r, mm) for mm, r in reports}}
    R.write_json(os.path.join(out, "report.json"), rj)
    R.write_residuals_csv(os.path.join(out, "residuals.csv"), reports)
    if j.get("write_fields", False):
        for i in range(steps):
            R.write_field_vtk(os.path.join(out, f"u_{i + 1}.vtk"), V, T, first[i])
    return R.exit_code([r.status for _, r in reports])


def main(argv=None) -> int:
    from . import Problem, baseline_desc, default_cfg
    from . import report as R

    ap = argparse.ArgumentParser(prog="python -m paper_2502_21013_b200.run")
    ap.add_argument("--config", type=int, default=0, help="BASELINE config 0..5")
    ap.add_argument("--ref-config", default=None, help="a reference run config (configs/*.json, transformer)")
    ap.add_argument("--out", default=None, help="output directory")
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--max-outer", type=int, default=200)
    ap.add_argument("--cells", type=int, default=0, help="override the grid (cells per side)")
    ap.add_argument("--steps", type=int, default=0, help="override N")
    ap.add_argument("--u0", choices=["static_init", "zero"], default="static_init")
    ap.add_argument("--device", type=int, default=0)
    ap.add_argument("--methods", default="m1", help="comma list of m1, m2, m3 (run from the same U0)")
    a = ap.parse_args(argv)
    if a.ref_config:
        return run_ref_config(a.ref_config, a.out, a.device)
    if not a.out:
        ap.error("--out is required")

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
