"""Output wire formats of the reference runner, for results of this package.

Mirrors tpfem/report.hpp (report_to_json, write_json, write_residuals_csv,
TableWriter; report.hpp:17-103) and the report.json assembled by run_solve
(runner.hpp:174-223), so tools that read the reference's output directories
read ours unchanged.  Byte-for-byte identical to the reference writers for the
same SolveReport (pinned by tests/test_report.py against fixtures produced by
the reference's own report.hpp, tests/golden/make_report_golden.py):

* numbers in CSV: "%.17g" (report.hpp:19-23);
* report.json: nlohmann::json dump(2) -- keys sorted (std::map), two-space
  indent, arrays one element per line, shortest round-trip doubles, NaN/inf as
  null, trailing newline; q_estimate omitted when not finite (report.hpp:35).
"""
from __future__ import annotations

import math

import numpy as np
import os
from typing import Iterable, Sequence

METHODS = ("m1", "m2", "m3")


def format_double(v: float) -> str:
    """printf("%.17g") (report.hpp:19-23)."""
    return "%.17g" % v


def _num(v) -> str:
    """A JSON number as nlohmann::json serialises it: shortest round-trip
    digits (Python's repr digits), fixed notation for decimal-point positions
    -4 < n <= 15, otherwise d.ddde+XX (at least two exponent digits); integral
    doubles keep ".0"; non-finite values become null."""
    if isinstance(v, bool):
        return "true" if v else "false"
    if isinstance(v, int):
        return str(v)
    v = float(v)
    if not math.isfinite(v):
        return "null"
    if v == 0.0:
        return "-0.0" if math.copysign(1.0, v) < 0 else "0.0"
    sign = "-" if v < 0 else ""
    r = repr(abs(v))
    mant, e = (r.split("e") + ["0"])[:2] if "e" in r else (r, "0")
    e = int(e)
    ip, fp = mant.split(".") if "." in mant else (mant, "")
    if ip.strip("0"):
        ip = ip.lstrip("0")
        digits, n = (ip + fp), len(ip) + e
    else:
        z = len(fp) - len(fp.lstrip("0"))
        digits, n = fp[z:], e - z
    digits = digits.rstrip("0") or "0"
    k = len(digits)
    if k <= n <= 15:
        out = digits + "0" * (n - k) + ".0"
    elif 0 < n <= 15:
        out = digits[:n] + "." + digits[n:]
    elif -4 < n <= 0:
        out = "0." + "0" * (-n) + digits
    else:
        x = n - 1
        es = ("-" if x < 0 else "+") + ("%02d" % abs(x))
        out = (digits if k == 1 else digits[0] + "." + digits[1:]) + "e" + es
    return sign + out


def _dump(obj, indent: int = 0) -> str:
    pad = "  " * indent
    inner = "  " * (indent + 1)
    if isinstance(obj, dict):
        if not obj:
            return "{}"
        items = [f'{inner}"{k}": {_dump(obj[k], indent + 1)}' for k in sorted(obj)]
        return "{\n" + ",\n".join(items) + "\n" + pad + "}"
    if isinstance(obj, (list, tuple)):
        if not obj:
            return "[]"
        items = [inner + _dump(v, indent + 1) for v in obj]
        return "[\n" + ",\n".join(items) + "\n" + pad + "]"
    if isinstance(obj, str):
        return '"' + obj.replace("\\", "\\\\").replace('"', '\\"') + '"'
    if obj is None:
        return "null"
    return _num(obj)


def report_to_dict(report, method: str = "m1") -> dict:
    """report_to_json (report.hpp:27-37) for a SolveReport-like object with
    status, iterations, wall_time, residual_history, contraction_history,
    q_estimate (api.SolveReport)."""
    d = {"method": method, "status": report.status, "iterations": int(report.iterations),
         "wall_seconds": float(report.wall_time),
         "residual_history": [float(x) for x in report.residual_history],
         "contraction_history": [float(x) for x in report.contraction_history]}
    q = float(report.q_estimate)
    if math.isfinite(q):
        d["q_estimate"] = q
    return d


def write_json(path: str, obj: dict) -> None:
    """write_json (report.hpp:39-44): dump(2) plus a newline."""
    with open(path, "w", newline="\n") as f:
        f.write(_dump(obj) + "\n")


def write_residuals_csv(path: str, reports: Sequence[tuple[str, object]]) -> None:
    """write_residuals_csv (report.hpp:49-64): rows method,iteration,residual,
    contraction; contraction blank on each method's first row.  `reports`:
    (method name, report) pairs in output order."""
    with open(path, "w", newline="\n") as f:
        f.write("method,iteration,residual,contraction\n")
        for name, rep in reports:
            hist, contr = list(rep.residual_history), list(rep.contraction_history)
            for k, r in enumerate(hist):
                f.write(f"{name},{k},{format_double(r)},")
                if k >= 1 and k - 1 < len(contr):
                    f.write(format_double(contr[k - 1]))
                f.write("\n")


TABLE_HEADER = ("steps,n_dof,init_seconds,m1_iterations,m1_seconds,m2_iterations,m2_seconds,"
                "m3_iterations,m3_seconds")


class TableWriter:
    """TableWriter (report.hpp:80-103): header at open, one flushed row per add."""

    def __init__(self, path: str):
        self._f = open(path, "w", newline="\n")
        self._f.write(TABLE_HEADER + "\n")
        self._f.flush()

    def add_row(self, steps: int, n_dof: int, init_seconds: float, m1_iterations: int = 0,
                m1_seconds: float = 0.0, m2_iterations: int = 0, m2_seconds: float = 0.0,
                m3_iterations: int = 0, m3_seconds: float = 0.0) -> None:
        self._f.write(f"{steps},{n_dof},{format_double(init_seconds)},{m1_iterations},"
                      f"{format_double(m1_seconds)},{m2_iterations},{format_double(m2_seconds)},"
                      f"{m3_iterations},{format_double(m3_seconds)}\n")
        self._f.flush()

    def close(self) -> None:
        self._f.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def exit_code(statuses: Iterable[str]) -> int:
    """0 when every method converged, 2 otherwise (runner.hpp:100-104)."""
    return 0 if all(s == "converged" for s in statuses) else 2


def run_report(desc, steps: int, n_dof: int, tau: float, threads: int, nu_hat, q_estimate: float,
               init_seconds: float, init_newton_max: int, symbol_abs, methods: dict) -> dict:
    """The report.json of run_solve (runner.hpp:194-217) for a BASELINE grid
    problem ("problem": "grid"; nu_hat keyed by material index)."""
    return {"problem": "grid", "steps": int(steps), "n_dof": int(n_dof), "cells": int(desc.cells),
            "period": float(desc.period), "tau": float(tau), "threads": int(threads),
            "nu_hat": {f"material_{i}": float(nu_hat[i]) for i in range(int(desc.n_materials))},
            "q_estimate": float(q_estimate),
            "init": {"seconds": float(init_seconds), "max_newton_steps": int(init_newton_max)},
            "frequency_symbol_abs": [float(x) for x in symbol_abs], "methods": methods}


def symbol_abs(steps: int, tau: float) -> list:
    """|lambda_k| for k = 0..N/2 (PeriodicSolver::symbol, periodic.hpp:146-152)."""
    out = []
    for k in range(steps // 2 + 1):
        if k == 0:
            out.append(0.0)
        elif 2 * k == steps:
            out.append(2.0 / tau)
        else:
            a = -2.0 * math.pi * k / steps
            re, im = (1.0 - math.cos(a)) / tau, (0.0 - math.sin(a)) / tau
            out.append(math.hypot(re, im))
    return out


def ensure_dir(path: str) -> None:
    os.makedirs(path, exist_ok=True)


# ---------------------------------------------------------------- VTK (vtk.hpp:12-55)
def dof_of_vertices(V) -> np.ndarray:
    """finalize_mesh's numbering (mesh.hpp:86-103): vertices off the bounding
    box, in vertex order, are the free dofs; boundary vertices get -1."""
    V = np.asarray(V, dtype=np.float64)
    xmin, ymin = V.min(axis=0)
    xmax, ymax = V.max(axis=0)
    tol = 1e-12 * max(xmax - xmin, ymax - ymin)
    on = ((np.abs(V[:, 0] - xmin) <= tol) | (np.abs(V[:, 0] - xmax) <= tol) |
          (np.abs(V[:, 1] - ymin) <= tol) | (np.abs(V[:, 1] - ymax) <= tol))
    dof = np.full(len(V), -1, dtype=np.int64)
    dof[~on] = np.arange(int((~on).sum()))
    return dof


def _vtk_head(f, V, T, title):
    # std::ostream with precision(17), default float format (%.17g); z = 0 written as an integer
    f.write(f"# vtk DataFile Version 3.0\n{title}\nASCII\nDATASET UNSTRUCTURED_GRID\n")
    f.write(f"POINTS {len(V)} double\n")
    for x, y in V:
        f.write(f"{format_double(x)} {format_double(y)} 0\n")
    f.write(f"CELLS {len(T)} {4 * len(T)}\n")
    for a, b, c in T:
        f.write(f"3 {a} {b} {c}\n")
    f.write(f"CELL_TYPES {len(T)}\n")
    f.write("5\n" * len(T))


def write_mesh_vtk(path: str, V, T, region) -> None:
    """write_mesh_vtk (vtk.hpp:33-38): the mesh with region labels as cell data."""
    with open(path, "w", newline="\n") as f:
        _vtk_head(f, V, T, "mesh regions")
        f.write(f"CELL_DATA {len(T)}\nSCALARS region int 1\nLOOKUP_TABLE default\n")
        for r in region:
            f.write(f"{int(r)}\n")


def write_field_vtk(path: str, V, T, free_values, name: str = "u") -> None:
    """write_field_vtk (vtk.hpp:42-55): a free-dof field on the vertices,
    zero on the Dirichlet boundary."""
    dof = dof_of_vertices(V)
    free_values = np.asarray(free_values, dtype=np.float64)
    if free_values.size != int((dof >= 0).sum()):
        raise ValueError("vtk field: size mismatch")
    with open(path, "w", newline="\n") as f:
        _vtk_head(f, V, T, "vertex field")
        f.write(f"POINT_DATA {len(V)}\nSCALARS {name} double 1\nLOOKUP_TABLE default\n")
        for d in dof:
            f.write(f"{format_double(free_values[d]) if d >= 0 else '0'}\n")
