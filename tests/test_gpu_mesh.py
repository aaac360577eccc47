"""GPU parity of the general-mesh path (include/tpgpu_mesh.h, SURVEY.md §8(f)
f1) against the reference running its OWN transformer problem end to end
(oracle/_ref: build_rectilinear_mesh, MaterialTable::transformer,
NonlinearOperator, assemble_mass / assemble_loads, static_init,
choose_nu_hat, solve_m1_fixed_point -- runner.hpp:27-89 unchanged).

Bars: loads bit-identical (same host arithmetic), K(u) and residuals within
1e-13, identical Newton and fixed-point iteration counts, every fixed-point
iterate within 1e-10 relative (north_star).  The configs are the reference's
own: configs/transformer.json (40x40, N=64, tol 1e-4) and
configs/transformer_saturated.json (windings at +-9.5e5 A/m^2), here to 1e-8.
"""
import numpy as np
import pytest

from paper_2502_21013_b200 import default_cfg
from paper_2502_21013_b200.api import SolveError
from paper_2502_21013_b200.mesh import MeshProblem, transformer_materials, transformer_mesh

pytestmark = pytest.mark.gpu

ITERATE_TOL = 1e-10


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def sat():
    """configs/transformer_saturated.json at tol 1e-8 on both sides."""
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    c = ref.tr_cfg(j_amp=9.5e5)
    cfg = default_cfg(tol=1e-8)
    U0, counts = ref.tr_static_init(c, cfg)
    nu, q = ref.tr_choose_nu_hat(c, U0, cfg)
    m1 = ref.tr_solve_m1(c, nu, q, U0, cfg, keep_iterates=True)
    p = MeshProblem.transformer(j_amp=9.5e5)
    yield dict(ref=ref, c=c, cfg=cfg, U0=U0, counts=counts, nu=nu, q=q, m1=m1, p=p)
    p.close()


def test_operators_match_reference(sat):
    p, ref, c = sat["p"], sat["ref"], sat["c"]
    assert p.n_dof == 2142 and p.steps == 64
    assert np.array_equal(p.loads(), ref.tr_loads(c))
    X = np.random.default_rng(3).standard_normal(p.shape) * 1e-2
    assert rel(p.apply_k(X), ref.tr_apply_k(c, X)) <= 1e-13
    R, r = p.residual(X)
    Rr, rr = ref.tr_residual(c, X)
    assert rel(R, Rr) <= 1e-13 and abs(r - rr) <= 1e-13 * rr


def test_static_init_and_nu_hat_match_reference(sat):
    p = sat["p"]
    U0, counts = p.static_init(sat["cfg"])
    assert np.array_equal(counts, sat["counts"])
    assert rel(U0, sat["U0"]) <= ITERATE_TOL
    nu, q = p.choose_nu_hat(sat["cfg"])
    assert rel(nu, sat["nu"]) <= 1e-12 and abs(q - sat["q"]) <= 1e-12


def test_periodic_solve_matches_reference(sat):
    p, ref = sat["p"], sat["ref"]
    p.set_nu_hat(sat["nu"], sat["q"])
    G = ref.tr_loads(sat["c"]) + np.random.default_rng(5).standard_normal(p.shape)
    assert rel(p.periodic_solve(G, sat["cfg"]), ref.tr_periodic_solve(sat["c"], sat["nu"], G, sat["cfg"])) <= 1e-9


def test_saturated_m1_matches_reference_iterate_by_iterate(sat):
    p, m1 = sat["p"], sat["m1"]
    p.set_nu_hat(sat["nu"], sat["q"])
    log = []
    U, rep = p.solve_m1_fixed_point(sat["U0"], sat["cfg"], iterate_log=log)
    assert rep.status == "converged" and m1.status == 0
    assert rep.iterations == m1.iterations  # 45 sweeps
    assert len(log) == len(m1.iterates)
    worst = max(rel(a, b) for a, b in zip(log, m1.iterates))
    assert worst <= ITERATE_TOL, worst
    h = np.array(rep.residual_history)
    assert np.all(np.abs(h - m1.history) <= 1e-8 * m1.history)


def test_transformer_json_config(ref):
    """configs/transformer.json: nominal windings, tol 1e-4: one sweep."""
    c = ref.tr_cfg()
    cfg = default_cfg(tol=1e-4)
    U0r, cr = ref.tr_static_init(c, cfg)
    nur, qr = ref.tr_choose_nu_hat(c, U0r, cfg)
    r = ref.tr_solve_m1(c, nur, qr, U0r, cfg)
    with MeshProblem.transformer() as p:
        U0, counts = p.static_init(cfg)
        nu, q = p.choose_nu_hat(cfg)
        U, rep = p.solve_m1_fixed_point(None, cfg)
    assert np.array_equal(counts, cr)
    assert rep.iterations == r.iterations == 1
    assert rel(U, r.U) <= ITERATE_TOL


@pytest.mark.parametrize("steps", [63, 128])
def test_other_step_counts(ref, steps):
    """odd N (direct DFT) and table.json's N = 128, a few saturated sweeps."""
    c = ref.tr_cfg(j_amp=9.5e5, steps=steps)
    cfg = default_cfg(tol=1e-8, m1_max_outer=6)
    U0, _ = ref.tr_static_init(c, cfg)
    nu, q = ref.tr_choose_nu_hat(c, U0, cfg)
    r = ref.tr_solve_m1(c, nu, q, U0, cfg, keep_iterates=True)
    with MeshProblem.transformer(steps=steps, j_amp=9.5e5) as p:
        p.set_nu_hat(nu, q)
        log = []
        U, rep = p.solve_m1_fixed_point(U0, cfg, iterate_log=log)
    assert rep.iterations == r.iterations == 6
    assert max(rel(a, b) for a, b in zip(log, r.iterates)) <= ITERATE_TOL


def test_refined_mesh_sweeps(ref):
    """table.json's refinements = 1 (8755 dofs): Newton counts and the first sweeps."""
    c = ref.tr_cfg(j_amp=9.5e5, refinements=1)
    cfg = default_cfg(tol=1e-8, m1_max_outer=4)
    U0r, cr = ref.tr_static_init(c, cfg)
    nu, q = ref.tr_choose_nu_hat(c, U0r, cfg)
    r = ref.tr_solve_m1(c, nu, q, U0r, cfg, keep_iterates=True)
    with MeshProblem.transformer(refinements=1, j_amp=9.5e5) as p:
        U0, counts = p.static_init(cfg)
        assert np.array_equal(counts, cr)
        assert rel(U0, U0r) <= ITERATE_TOL
        p.set_nu_hat(nu, q)
        log = []
        U, rep = p.solve_m1_fixed_point(U0r, cfg, iterate_log=log)
    assert rep.iterations == r.iterations == 4 and rep.status == "max_iter"
    assert max(rel(a, b) for a, b in zip(log, r.iterates)) <= ITERATE_TOL


def test_general_mesh_arrays_and_errors():
    """any triangulation goes through tp_mesh_problem_create; bad input is
    std::invalid_argument -> ValueError (MaterialTable::set, compute_element_data)."""
    V, T, R, n = transformer_mesh(12, 10, 0)
    mats = transformer_materials()
    with MeshProblem(V, T, R, mats, 8, 0.02) as p:
        assert p.n_dof == n
    bad = transformer_materials()
    bad[1].d = 0.0
    with pytest.raises(ValueError):
        MeshProblem(V, T, R, bad, 8, 0.02)
    Tf = T.copy()
    Tf[0] = Tf[0, ::-1]  # negative orientation
    with pytest.raises(ValueError):
        MeshProblem(V, Tf, R, mats, 8, 0.02)
    with pytest.raises(ValueError):
        with MeshProblem(V, T, R, mats, 8, 0.02) as p:
            p.solve_m1_fixed_point(np.zeros(p.shape), default_cfg())  # no nu_hat installed
    _ = SolveError


def test_reference_side_adapter_drop_in():
    """INTEGRATION.md's reference-side change, compiled against the reference
    headers (oracle/_ref/adapter_demo): runner.hpp's transformer pipeline with
    M1 through tpgpu_tpfem.hpp's GpuMeshProblem vs tpfem on the CPU."""
    import json
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "adapter_demo")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/adapter_demo not built")
    out = subprocess.run([exe, "40", "40", "0", "64", "9.5e5", "1e-8"], capture_output=True, text=True, timeout=300)
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert out.returncode == 0, r
    assert r["newton_equal"] and r["cpu_iterations"] == r["gpu_iterations"] == 45
    assert r["final_rel"] <= ITERATE_TOL and r["nu_hat_rel"] <= 1e-12


@pytest.mark.parametrize("j_amp,tol", [(0.0, 1e-4), (9.5e5, 1e-8)])
def test_m2_newton_on_reference_mesh(ref, j_amp, tol):
    """transformer.json's "method": "all" -- M2 (solve_m2_newton): same Newton
    step count and status, final state within 1e-10."""
    c = ref.tr_cfg(j_amp=j_amp)
    cfg = default_cfg(tol=tol)
    U0, _ = ref.tr_static_init(c, cfg)
    Ur, hr, kr, sr, _ = ref.tr_solve_m23(c, 2, U0, cfg)
    with MeshProblem.transformer(j_amp=j_amp or None) as p:
        U, rep = p.solve_m2_newton(U0, cfg)
    assert rep.iterations == kr and {"converged": 0, "max_iter": 1, "stalled": 2}[rep.status] == sr
    assert rel(U, Ur) <= ITERATE_TOL
    assert np.allclose(rep.residual_history[:2], hr[:2], rtol=1e-10)


def test_m3_timestepping_on_reference_mesh(ref):
    """M3 (solve_m3_timestepping), two periods of the saturated transformer."""
    c = ref.tr_cfg(j_amp=9.5e5)
    cfg = default_cfg(tol=1e-8, m3_max_cycles=2)
    U0, _ = ref.tr_static_init(c, cfg)
    Ur, hr, kr, sr, _ = ref.tr_solve_m23(c, 3, U0, cfg)
    with MeshProblem.transformer(j_amp=9.5e5) as p:
        U, rep = p.solve_m3_timestepping(U0, cfg)
    assert rep.iterations == kr == 2 and rep.status == "max_iter" and sr == 1
    assert rel(U, Ur) <= ITERATE_TOL
    assert np.allclose(rep.residual_history, hr, rtol=1e-8)


def test_reference_run_config_cli(ref, tmp_path):
    """python -m paper_2502_21013_b200.run --ref-config: a run config in the
    reference's format (the fields of configs/transformer_saturated.json with
    method "all"; parse_run_config, config.hpp:176-230) -> report.json /
    residuals.csv in the runner's formats, iteration counts as the reference's."""
    import json
    from paper_2502_21013_b200 import run
    conf = {"problem": "transformer", "method": "all", "nx": 40, "ny": 40, "refinements": 0, "steps": 64,
            "period": 0.02, "threads": 1, "output_dir": str(tmp_path / "out"),
            "materials": {"winding_plus": {"j_amp": 950000.0}, "winding_minus": {"j_amp": -950000.0}},
            "solver": {"tol": 1e-4, "nu_hat_mode": "frozen_field", "m3_max_cycles": 2}}
    path = tmp_path / "run.json"
    path.write_text(json.dumps(conf))
    code = run.main(["--ref-config", str(path)])
    rj = json.loads((tmp_path / "out" / "report.json").read_text())
    assert rj["problem"] == "transformer" and rj["n_dof"] == 2142 and len(rj["frequency_symbol_abs"]) == 33
    c = ref.tr_cfg(j_amp=9.5e5)
    cfg = default_cfg(tol=1e-4, m3_max_cycles=2)
    U0, counts = ref.tr_static_init(c, cfg)
    nu, q = ref.tr_choose_nu_hat(c, U0, cfg)
    m1 = ref.tr_solve_m1(c, nu, q, U0, cfg)
    _, _, k2, s2, _ = ref.tr_solve_m23(c, 2, U0, cfg)
    _, _, k3, s3, _ = ref.tr_solve_m23(c, 3, U0, cfg)
    assert rj["init"]["max_newton_steps"] == int(counts.max())
    assert abs(rj["q_estimate"] - q) <= 1e-12
    assert [rj["methods"][m]["iterations"] for m in ("m1", "m2", "m3")] == [m1.iterations, k2, k3]
    assert code == (0 if (m1.status, s2, s3) == (0, 0, 0) else 2)
    assert (tmp_path / "out" / "residuals.csv").read_text().startswith("method,")


@pytest.mark.parametrize("steps", [1, 2, 3])
def test_tiny_step_counts(ref, steps):
    """N = 1 (the block is K_hat alone, test_periodic.cpp:96-107), N = 2, odd N = 3:
    periodic solve and a few M1 sweeps against the reference."""
    c = ref.tr_cfg(nx=12, ny=10, j_amp=9.5e5, steps=steps)
    cfg = default_cfg(tol=1e-8, m1_max_outer=4)
    U0, counts = ref.tr_static_init(c, cfg)
    nu, q = ref.tr_choose_nu_hat(c, U0, cfg)
    G = ref.tr_loads(c) + np.random.default_rng(steps).standard_normal(U0.shape)
    Ur = ref.tr_periodic_solve(c, nu, G, cfg)
    r = ref.tr_solve_m1(c, nu, q, U0, cfg, keep_iterates=True)
    V, T, R, _ = transformer_mesh(12, 10, 0)
    with MeshProblem(V, T, R, transformer_materials(9.5e5), steps, 0.02) as p:
        U0g, cg = p.static_init(cfg)
        assert np.array_equal(cg, counts)
        p.set_nu_hat(nu, q)
        assert rel(p.periodic_solve(G, cfg), Ur) <= 1e-10
        log = []
        U, rep = p.solve_m1_fixed_point(U0, cfg, iterate_log=log)
    assert rep.iterations == r.iterations
    assert max(rel(a, b) for a, b in zip(log, r.iterates)) <= ITERATE_TOL


def test_transformer_golden_fixture():
    """Against tests/golden/transformer_reference.npz (written by the reference
    itself, tests/golden/make_golden.py --transformer): runs without oracle/_ref."""
    import os
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "transformer_reference.npz"))
    cfg = default_cfg(tol=1e-8)
    for tag, args in (("small", (12, 10, 0, 8)), ("sat", (40, 40, 0, 64))):
        with MeshProblem.transformer(*args, 0.02, j_amp=9.5e5) as p:
            U0, counts = p.static_init(cfg)
            nu, q = p.choose_nu_hat(cfg)
            U, rep = p.solve_m1_fixed_point(None, cfg)
        assert np.array_equal(counts, g[f"{tag}_newton_counts"])
        assert rel(nu, g[f"{tag}_nu_hat"]) <= 1e-12 and abs(q - float(g[f"{tag}_q"])) <= 1e-12
        assert rep.iterations == int(g[f"{tag}_iterations"])
        assert rel(U.reshape(-1)[::97], g[f"{tag}_U_sample"]) <= ITERATE_TOL
        assert rel(U0.reshape(-1)[::97], g[f"{tag}_U0_sample"]) <= ITERATE_TOL
        if tag == "small":
            assert rel(U, g["small_U"]) <= ITERATE_TOL and rel(U0, g["small_U0"]) <= ITERATE_TOL


def test_reference_table_config_and_vtk(ref, tmp_path):
    """`tpfem table` (run_table, runner.hpp:235-269) for a run config with a
    "sweep": one table.csv row per (refinements, steps) entry in the
    reference's format, with the reference's M1 iteration counts; and
    `tpfem solve` with write_mesh / write_fields (runner.hpp:180,219-227):
    mesh.vtk and one u_<i>.vtk per slice in vtk.hpp's format, the field of
    the first method's state."""
    import json
    from paper_2502_21013_b200 import run
    mats = {"winding_plus": {"j_amp": 950000.0}, "winding_minus": {"j_amp": -950000.0}}
    conf = {"problem": "transformer", "nx": 12, "ny": 10, "period": 0.02, "output_dir": str(tmp_path / "t"),
            "materials": mats, "solver": {"tol": 1e-6, "m3_max_cycles": 2},
            "sweep": [{"refinements": 0, "steps": 8}, {"refinements": 0, "steps": 16}]}
    path = tmp_path / "table.json"
    path.write_text(json.dumps(conf))
    assert run.main(["--ref-config", str(path)]) == 0
    lines = (tmp_path / "t" / "table.csv").read_text().splitlines()
    assert lines[0].startswith("steps,n_dof,init_seconds,m1_iterations") and len(lines) == 3
    cfg = default_cfg(tol=1e-6, m3_max_cycles=2)
    for line, steps in zip(lines[1:], (8, 16)):
        f = line.split(",")
        c = ref.tr_cfg(nx=12, ny=10, steps=steps, j_amp=9.5e5)
        U0, _ = ref.tr_static_init(c, cfg)
        m1 = ref.tr_solve_m1(c, *ref.tr_choose_nu_hat(c, U0, cfg), U0, cfg)
        assert int(f[0]) == steps and int(f[3]) == m1.iterations
    # solve with VTK output
    conf2 = {"problem": "transformer", "method": "m1", "nx": 12, "ny": 10, "steps": 4, "period": 0.02,
             "output_dir": str(tmp_path / "s"), "write_mesh": True, "write_fields": True, "materials": mats,
             "solver": {"tol": 1e-6}}
    path2 = tmp_path / "solve.json"
    path2.write_text(json.dumps(conf2))
    run.main(["--ref-config", str(path2)])
    V, T, R, ndof = transformer_mesh(12, 10, 0)
    mesh_vtk = (tmp_path / "s" / "mesh.vtk").read_text().splitlines()
    assert mesh_vtk[4] == f"POINTS {len(V)} double" and f"CELL_DATA {len(T)}" in mesh_vtk
    for i in range(1, 5):
        u = (tmp_path / "s" / f"u_{i}.vtk").read_text().splitlines()
        k = u.index(f"POINT_DATA {len(V)}")
        assert len(u) == k + 3 + len(V)
