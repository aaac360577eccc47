"""Oracle pinning (CPU-only).

* the numpy restatement (oracle/tp_oracle.py) against the golden fixtures
  produced by the compiled reference (tests/golden/make_golden.py),
* the numpy restatement against the reference's own known-answer tests,
  restated (test_periodic.cpp, test_fft.cpp, test_solvers.cpp),
* the reference's own GoogleTest binaries compiled against the shim
  (oracle/_ref/test_*), when built.
"""
import math
import os
import subprocess

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import tp_oracle as O
from paper_2502_21013_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def golden(name):
    path = os.path.join(GOLD, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not generated")
    return np.load(path)


def desc(config):
    from paper_2502_21013_b200 import api
    return api.baseline_desc(config)


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


# ---- reference KATs restated (test_periodic.cpp:84-145) ----------------

def test_symbol_special_cases():
    tau = 0.25
    assert O.symbol(0, 8, tau) == 0
    assert O.symbol(4, 8, tau) == 2.0 / tau
    s = O.symbol(2, 8, tau)
    assert abs(s.real - 1 / tau) < 1e-14 and abs(s.imag - 1 / tau) < 1e-14


def random_spd_tridiagonal(n, diag, off, rng):
    d = diag + rng.uniform(0, 0.5, n)
    return sp.diags([np.full(n - 1, off), d, np.full(n - 1, off)], [-1, 0, 1]).tocsr()


def all_at_once(M, K, G, tau):
    N, n = G.shape
    blocks = [[None] * N for _ in range(N)]
    for i in range(N):
        blocks[i][i] = M / tau + K
        j = (i + N - 1) % N
        blocks[i][j] = (blocks[i][j] if blocks[i][j] is not None else 0) - M / tau if N > 1 else blocks[i][i]
    if N == 1:
        A = K.tocsc()
    else:
        A = sp.bmat(blocks).tocsc()
    return sp.linalg.spsolve(A, G.reshape(-1)).reshape(N, n)


@pytest.mark.parametrize("steps", [1, 2, 5, 8, 16])
@pytest.mark.parametrize("n", [1, 5, 20])
def test_dft_solve_matches_all_at_once(steps, n):
    rng = np.random.default_rng(10 * steps + n)
    M = random_spd_tridiagonal(n, 2.0, -0.4, rng)
    K = random_spd_tridiagonal(n, 3.0, -1.0, rng)
    G = rng.uniform(-1, 1, (steps, n))
    tau = 0.02 / steps
    U = O.PeriodicSolver(M, K, tau, steps).solve(G)
    assert rel(U, all_at_once(M, K, G, tau)) <= 1e-9


def test_degenerate_mass_matches_all_at_once():
    """acceptance.cpp:108-172: diagonal mass with zero rows."""
    rng = np.random.default_rng(3)
    n, steps = 12, 8
    mdiag = np.where(np.arange(n) % 3 == 0, 0.0, 1.0 + rng.uniform(0, 1, n))
    M = sp.diags(mdiag).tocsr()
    K = random_spd_tridiagonal(n, 3.0, -1.0, rng)
    G = rng.uniform(-1, 1, (steps, n))
    tau = 0.01
    assert rel(O.PeriodicSolver(M, K, tau, steps).solve(G), all_at_once(M, K, G, tau)) <= 1e-9


def test_imaginary_residue_guard():
    """periodic.hpp:192-196 (test_periodic.cpp:197-206).  numpy's inverse of
    an exactly Hermitian spectrum can be exactly real, so the guard is driven
    with a negative tolerance, which must always fire."""
    rng = np.random.default_rng(82)
    M = random_spd_tridiagonal(3, 2.0, -0.4, rng)
    K = random_spd_tridiagonal(3, 3.0, -1.0, rng)
    G = rng.uniform(-1, 1, (4, 3))
    O.PeriodicSolver(M, K, 0.005, 4, imag_tol=1e-9).solve(G)
    with pytest.raises(O.SolveError):
        O.PeriodicSolver(M, K, 0.005, 4, imag_tol=-1.0).solve(G)


def test_fft_kats():
    """test_fft.cpp: delta <-> constant, single mode, round trip (numpy FFT
    used by the restatement has the reference's sign and normalisation)."""
    N = 16
    d = np.zeros(N, complex)
    d[0] = 1
    assert np.allclose(np.fft.fft(d), np.ones(N))
    k = 3
    x = np.exp(2j * math.pi * k * np.arange(N) / N)
    X = np.fft.fft(x)
    assert abs(X[k] - N) < 1e-12 and np.abs(np.delete(X, k)).max() < 1e-12
    y = np.random.default_rng(0).standard_normal(N)
    assert np.allclose(np.fft.ifft(np.fft.fft(y)).real, y, atol=1e-15)


def test_stopping_rule():
    assert O.stopping_check([10.0, 1.0, 1e-3], 1e-4)
    assert not O.stopping_check([10.0, 1.0, 2e-3], 1e-4)
    assert O.stopping_check([10.0, 1e-3], 1e-4)
    assert O.stopping_check([0.0], 1e-4)
    with pytest.raises(ValueError):
        O.stopping_check([], 1e-4)


# ---- physics restatement vs the compiled reference (golden) -------------

def test_setup_against_golden():
    g = golden("cfg0_reference.npz")
    s = O.GridSetup(desc(0))
    assert rel(s.loads(), g["loads"]) <= 1e-14
    assert rel(s.mass_diag(), g["mass"]) <= 1e-14


def test_static_init_against_golden():
    g = golden("cfg0_reference.npz")
    s = O.GridSetup(desc(0))
    U0, counts = O.static_init(s, s.loads())
    assert np.array_equal(counts, g["newton_counts"])
    assert rel(U0, g["U0"]) <= 1e-12
    nu, q = s.choose_nu_hat(U0)
    assert np.allclose(nu, g["nu_hat"], rtol=1e-12)
    assert abs(q - float(g["q"])) <= 1e-12


@pytest.mark.slow
def test_m1_against_golden():
    g = golden("cfg0_reference.npz")
    s = O.GridSetup(desc(0))
    K = s.stiffness_frozen(g["nu_hat"])
    r = O.solve_m1_fixed_point(s, K, s.loads(), g["U0"], tol=1e-8, keep_iterates=True)
    assert r.iterations == int(g["iterations"])
    assert rel(r.iterates[1], g["U1"]) <= 1e-12
    assert rel(r.iterates[2], g["U2"]) <= 1e-12
    assert rel(r.U, g["U"]) <= 1e-10
    h = np.array(r.history)
    assert np.all(np.abs(h - g["history"]) <= 1e-10 * g["history"][0] + 1e-6 * g["history"])


def test_cfg1_setup_against_golden():
    g = golden("cfg1_reference.npz")
    s = O.GridSetup(desc(1))
    assert rel(s.mass_diag(), g["mass"]) <= 1e-14
    from tests.golden.make_golden import checksum
    c, ref_c = checksum(s.loads()), g["loads_checksum"]
    assert np.all(np.abs(c - ref_c) <= 1e-12 * ref_c[0])


# ---- the reference's own unit tests, compiled against the shim ----------

REFTESTS = ["test_sparse", "test_solve", "test_fft", "test_periodic", "test_solvers", "test_oracle",
            "test_assembly", "test_materials", "test_mesh"]


@pytest.mark.parametrize("name", REFTESTS)
def test_reference_unit_tests_pass_with_shim(name):
    exe = os.path.join(ROOT, "oracle", "_ref", name)
    if not os.path.exists(exe):
        pytest.skip("reference tests not built (make -C oracle reftests)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "0 failed" in out.stdout
