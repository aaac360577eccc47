"""General-mesh path vs the reference on its own transformer problem (diagnostics).

    python tools/mesh_check.py [--nx 40 --ny 40 --refinements 0 --steps 64 --j-amp 9.5e5 --tol 1e-8]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import ref  # noqa: E402  (checker)
from paper_2502_21013_b200.abi import default_cfg  # noqa: E402
from paper_2502_21013_b200.mesh import MeshProblem  # noqa: E402


def rel(a, b):
    d = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (d if d > 0 else 1.0))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=40)
    ap.add_argument("--ny", type=int, default=40)
    ap.add_argument("--refinements", type=int, default=0)
    ap.add_argument("--steps", type=int, default=64)
    ap.add_argument("--j-amp", type=float, default=9.5e5)
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--max-outer", type=int, default=200)
    a = ap.parse_args()
    cfg = default_cfg(tol=a.tol, m1_max_outer=a.max_outer)
    c = ref.tr_cfg(nx=a.nx, ny=a.ny, refinements=a.refinements, steps=a.steps, j_amp=a.j_amp)
    t = time.perf_counter()
    p = MeshProblem.transformer(a.nx, a.ny, a.refinements, a.steps, 0.02, j_amp=a.j_amp or None)
    print(f"create {time.perf_counter() - t:.3f}s n={p.n_dof} N={p.steps} bw={p.bandwidth}", flush=True)
    F = p.loads()
    Fr = ref.tr_loads(c)
    print("loads", rel(F, Fr))
    rng = np.random.default_rng(1)
    X = rng.standard_normal(p.shape) * 1e-3
    print("apply_k", rel(p.apply_k(X), ref.tr_apply_k(c, X)))
    R, rn = p.residual(X)
    Rr, rnr = ref.tr_residual(c, X)
    print("residual", rel(R, Rr), rn, rnr)
    t = time.perf_counter()
    U0, cnt = p.static_init(cfg)
    tg = time.perf_counter() - t
    t = time.perf_counter()
    U0r, cntr = ref.tr_static_init(c, cfg)
    tr = time.perf_counter() - t
    print(f"static_init gpu {tg:.3f}s ref {tr:.3f}s counts equal {np.array_equal(cnt, cntr)} "
          f"max {cnt.max()}/{cntr.max()} U0 rel {rel(U0, U0r):.3e}", flush=True)
    nu, q = p.choose_nu_hat(cfg)
    nur, qr = ref.tr_choose_nu_hat(c, U0r, cfg)
    print("nu_hat", rel(nu, nur), q, qr)
    G = rng.standard_normal(p.shape)
    t = time.perf_counter()
    Ug = p.periodic_solve(G, cfg)
    tg = time.perf_counter() - t
    Ur = ref.tr_periodic_solve(c, nu, G, cfg)
    print(f"periodic_solve rel {rel(Ug, Ur):.3e} ({tg:.3f}s incl. factorisation)", flush=True)
    log = []
    t = time.perf_counter()
    U, rep = p.solve_m1_fixed_point(U0r, cfg, iterate_log=log)
    tg = time.perf_counter() - t
    r = ref.tr_solve_m1(c, nur, qr, U0r, cfg, keep_iterates=True)
    errs = [rel(log[k], r.iterates[k]) for k in range(min(len(log), len(r.iterates)))]
    hist = np.array(rep.residual_history)
    hrel = float(np.max(np.abs(hist[:len(r.history)] - r.history[:len(hist)]) / r.history[:len(hist)]))
    print(f"m1 gpu {rep.iterations} sweeps {rep.status} ({tg:.3f}s: setup {rep.setup_time:.3f}, sweeps "
          f"{rep.sweep_time:.3f}) ref {r.iterations} ({r.wall_time:.3f}s); max iterate rel {max(errs):.3e}; "
          f"history rel {hrel:.3e}; final rel {rel(U, r.U):.3e}")
    print("launches", p.launches)


if __name__ == "__main__":
    main()
