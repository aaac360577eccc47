"""Output wire formats (report.json, residuals.csv, table.csv) against files
written by the reference's own tpfem/report.hpp for the same SolveReports
(tests/golden/report/, made by tests/golden/make_report_golden.py)."""
import math
import os

import pytest

from paper_2502_21013_b200 import report as R
from paper_2502_21013_b200.api import SolveReport

GOLD = os.path.join(os.path.dirname(__file__), "golden", "report")


def _num(s):
    return float("nan") if s == "nan" else float(s)


def load_spec():
    reports, rows = [], []
    with open(os.path.join(GOLD, "spec.txt")) as f:
        for line in f:
            t = line.split()
            if not t:
                continue
            if t[0] == "T":
                rows.append((int(t[1]), int(t[2]), _num(t[3]), int(t[4]), _num(t[5]), int(t[6]), _num(t[7]),
                             int(t[8]), _num(t[9])))
                continue
            method, status, its, wall, q, nh = t[0], t[1], int(t[2]), _num(t[3]), _num(t[4]), int(t[5])
            hist = [_num(x) for x in t[6:6 + nh]]
            nc = int(t[6 + nh])
            contr = [_num(x) for x in t[7 + nh:7 + nh + nc]]
            reports.append((method, SolveReport(method=method, iterations=its, residual_history=hist,
                                                contraction_history=contr, q_estimate=q, wall_time=wall,
                                                status=status)))
    return reports, rows


def read(path):
    with open(path, "rb") as f:
        return f.read()


def test_report_json_matches_reference_writer(tmp_path):
    reports, _ = load_spec()
    out = tmp_path / "report.json"
    R.write_json(str(out), {"methods": {m: R.report_to_dict(r, m) for m, r in reports}})
    assert read(out) == read(os.path.join(GOLD, "report.json"))


def test_residuals_csv_matches_reference_writer(tmp_path):
    reports, _ = load_spec()
    out = tmp_path / "residuals.csv"
    R.write_residuals_csv(str(out), reports)
    assert read(out) == read(os.path.join(GOLD, "residuals.csv"))


def test_table_csv_matches_reference_writer(tmp_path):
    _, rows = load_spec()
    out = tmp_path / "table.csv"
    with R.TableWriter(str(out)) as tw:
        for r in rows:
            tw.add_row(*r)
    assert read(out) == read(os.path.join(GOLD, "table.csv"))


def test_q_estimate_omitted_when_not_finite():
    rep = SolveReport(q_estimate=float("nan"), residual_history=[1.0], status="converged")
    assert "q_estimate" not in R.report_to_dict(rep)
    rep.q_estimate = 0.5
    assert R.report_to_dict(rep)["q_estimate"] == 0.5


def test_symbol_abs_and_exit_code():
    s = R.symbol_abs(8, 0.125)
    assert s[0] == 0.0 and s[-1] == 16.0
    assert math.isclose(s[2], math.hypot(8.0, 8.0), rel_tol=1e-15)  # lambda_{N/4} = (1+i)/tau
    assert R.exit_code(["converged", "converged"]) == 0
    assert R.exit_code(["converged", "max_iter"]) == 2


@pytest.mark.parametrize("v", [0.1, 1.0, 1e-5, 1.5e300, 2.2250738585072014e-308, -0.0, 123456789.0, 5e-324])
def test_double_formats(v):
    assert R.format_double(v) == "%.17g" % v
    assert float(R._num(v)) == v


def test_vtk_matches_reference_writer(tmp_path):
    """write_mesh_vtk / write_field_vtk (vtk.hpp:33-55) byte for byte against
    the reference's own writers on its transformer mesh (12 x 10 cells)."""
    import numpy as np

    from paper_2502_21013_b200.mesh import transformer_mesh
    V, T, Rg, ndof = transformer_mesh(12, 10, 0)
    R.write_mesh_vtk(str(tmp_path / "mesh.vtk"), V, T, Rg)
    d = np.arange(ndof, dtype=np.float64)
    R.write_field_vtk(str(tmp_path / "u.vtk"), V, T, np.sin(0.37 * d) - 1e-3 * d)
    for name in ("mesh.vtk", "u.vtk"):
        assert (tmp_path / name).read_bytes() == open(os.path.join(GOLD, name), "rb").read(), name
