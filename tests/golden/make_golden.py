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


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg1", action="store_true")
    a = ap.parse_args()
    cfg0()
    if a.cfg1:
        cfg1()
