"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs the reference's own solver templates (tpfem static_init,
solve_m1_fixed_point, PeriodicSolver; compiled by oracle/Makefile into
oracle/_ref/libtpref.so with the shim SparseSolver) on the BASELINE physics.
Must run where /root/reference was available to build libtpref.so:

    make -C oracle && python tests/golden/make_golden.py [--cfg1]
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_2502_21013_b200.abi import default_cfg  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def checksum(a):
    """Order-sensitive, size-independent fingerprint of a slice-major array."""
    a = np.asarray(a, dtype=np.float64).reshape(-1)
    w = np.cos(0.001 * np.arange(a.size))
    return np.array([np.linalg.norm(a), a.sum(), (w * a).sum(), np.abs(a).max()])


def cfg0():
    d = ref.baseline_desc(0)
    cfg = default_cfg(tol=1e-8)
    F = ref.loads(d)
    m = ref.mass(d)
    U0, counts = ref.static_init(d, cfg)
    nu, q = ref.choose_nu_hat(d, U0, cfg)
    r = ref.solve_m1(d, nu, q, U0, cfg, keep_iterates=True)
    its = r.iterates
    np.savez_compressed(os.path.join(OUT, "cfg0_reference.npz"),
                        loads=F, mass=m, U0=U0, newton_counts=counts, nu_hat=nu, q=q,
                        history=r.history, iterations=r.iterations, status=r.status, U=r.U,
                        iterate_norms=np.array([np.linalg.norm(u) for u in its]),
                        step_norms=np.array([np.linalg.norm(its[k] - its[k - 1]) for k in range(1, len(its))]),
                        U1=its[1], U2=its[2])
    print("cfg0: iterations", r.iterations, "history", r.history[0], r.history[-1])


def cfg1(sweeps=2):
    d = ref.baseline_desc(1)
    cfg = default_cfg(tol=1e-8)
    t = time.time()
    U0, counts = ref.static_init(d, cfg)
    nu, q = ref.choose_nu_hat(d, U0, cfg)
    c2 = default_cfg(tol=1e-12, m1_max_outer=sweeps)
    r = ref.solve_m1(d, nu, q, U0, c2, keep_iterates=True, cache=2)
    np.savez_compressed(os.path.join(OUT, "cfg1_reference.npz"),
                        loads_checksum=checksum(ref.loads(d)), mass=ref.mass(d),
                        U0_checksum=checksum(U0), newton_counts=counts, nu_hat=nu, q=q,
                        history=r.history, iterate_checksums=np.array([checksum(u) for u in r.iterates]),
                        U0_sample=U0.reshape(-1)[::997], U_last_sample=r.U.reshape(-1)[::997])
    print("cfg1:", time.time() - t, "s; history", r.history)


def transformer():
    """The reference's own transformer problem (mesh.hpp / materials.hpp
    physics, transformer_saturated.json windings) through tpfem's setup and
    solve_m1_fixed_point: full vectors on a 12 x 10 mesh (N = 8), counts,
    histories, checksums and samples on the 40 x 40 mesh (N = 64)."""
    cfg = default_cfg(tol=1e-8)
    out = {}
    for tag, c in (("small", ref.tr_cfg(nx=12, ny=10, steps=8, j_amp=9.5e5)), ("sat", ref.tr_cfg(j_amp=9.5e5))):
        U0, counts = ref.tr_static_init(c, cfg)
        nu, q = ref.tr_choose_nu_hat(c, U0, cfg)
        r = ref.tr_solve_m1(c, nu, q, U0, cfg)
        out.update({f"{tag}_newton_counts": counts, f"{tag}_nu_hat": nu, f"{tag}_q": q,
                    f"{tag}_history": r.history, f"{tag}_iterations": r.iterations,
                    f"{tag}_U_checksum": checksum(r.U), f"{tag}_U0_checksum": checksum(U0),
                    f"{tag}_U_sample": r.U.reshape(-1)[::97], f"{tag}_U0_sample": U0.reshape(-1)[::97]})
        if tag == "small":
            out.update({"small_U0": U0, "small_U": r.U})
        print("transformer", tag, "iterations", r.iterations)
    np.savez_compressed(os.path.join(OUT, "transformer_reference.npz"), **out)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg1", action="store_true")
    ap.add_argument("--transformer", action="store_true")
    a = ap.parse_args()
    if a.transformer:
        transformer()
        sys.exit(0)
    cfg0()
    if a.cfg1:
        cfg1()
