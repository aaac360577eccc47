"""GPU parity on the BASELINE configs the product reports numbers on, against
fixtures written by the REFERENCE itself (tests/golden/make_golden_large.py:
tpfem's static_init, solve_m1_fixed_point and PeriodicSolver block solves,
compiled in oracle/_ref).  Whole iterates at these sizes cannot be
committed, so every iterate is compared through its checksum (norm, sum,
cos-weighted sum, max |.|), ||U^k - U^{k-1}|| and a strided sample
(SURVEY.md §8(d)).

Tolerances: iteration and Newton counts identical; iterate norms and samples
within 1e-10 relative (north_star); residual histories within the measured
agreement written next to each assertion.
"""
import os

import numpy as np
import pytest

from paper_2502_21013_b200 import Problem, baseline_desc, default_cfg
from paper_2502_21013_b200.abi import TP_NU_HAT_THEORY

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
ITERATE_TOL = 1e-10


def golden(name):
    path = os.path.join(GOLD, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not generated (tests/golden/make_golden_large.py)")
    return np.load(path)


def checksum(a):
    a = np.asarray(a, dtype=np.float64).reshape(-1)
    w = np.cos(0.001 * np.arange(a.size))
    return np.array([np.linalg.norm(a), a.sum(), (w * a).sum(), np.abs(a).max()])


def assert_checksum_close(got, want, tol=ITERATE_TOL, what="", size=None):
    """norm relative; the two signed sums relative to norm * sqrt(size) (a
    bound on the l1 scale, so cancellation inside a sum cannot turn
    rounding into a failure); max |.| relative at 10x the tolerance (a
    single entry)."""
    nrm = max(want[0], 1e-300)
    assert abs(got[0] - want[0]) <= tol * nrm, (what, "norm", got[0], want[0])
    if size:
        for i, name in ((1, "sum"), (2, "weighted sum")):
            assert abs(got[i] - want[i]) <= tol * nrm * np.sqrt(size), (what, name, got[i], want[i])
    assert abs(got[3] - want[3]) <= tol * max(want[3], 1e-300) * 10, (what, "max", got[3], want[3])


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


class Digests:
    """Per-iterate digests of the device M1 iterates (iterate callback)."""

    def __init__(self, stride):
        self.stride = stride
        self.rows, self.samples = [], []
        self.prev = None

    def __call__(self, k, U, res):
        flat = U.reshape(-1)
        self.size = flat.size
        d = checksum(flat)
        step = 0.0 if self.prev is None else float(np.linalg.norm(flat - self.prev))
        self.rows.append(np.r_[d, step])
        self.samples.append(flat[::self.stride].copy())
        self.prev = flat.copy()
        return False


def _compare_iterates(dig, g, tol=ITERATE_TOL):
    gd, gs = g["digests"], g["samples"]
    assert len(dig.rows) == gd.shape[0], (len(dig.rows), gd.shape[0])
    worst = 0.0
    for k, (row, smp) in enumerate(zip(dig.rows, dig.samples)):
        assert_checksum_close(row[:4], gd[k, :4], tol, what=f"iterate {k}", size=dig.size)
        # ||U^k - U^{k-1}|| relative to the iterate (the step itself shrinks to
        # the contraction floor)
        assert abs(row[4] - gd[k, 4]) <= tol * gd[k, 0], (k, row[4], gd[k, 4])
        e = rel(smp, gs[k])
        worst = max(worst, e)
        assert e <= tol, (k, e)
    return worst


def test_cfg1_full_m1_matches_reference():
    """BASELINE config 1 (256^2 cells, N = 256) end to end: static_init ->
    frozen-field nu_hat -> M1 to 1e-8.  Same Newton counts, same number of
    sweeps and status, every iterate within 1e-10."""
    g = golden("cfg1_full_reference.npz")
    cfg = default_cfg(tol=1e-8)
    with Problem(baseline_desc(1)) as p:
        U0, counts = p.static_init(cfg)
        assert np.array_equal(counts, g["newton_counts"])
        assert_checksum_close(checksum(U0), g["U0_checksum"], what="U0")
        nu, q = p.choose_nu_hat(cfg)
        assert np.allclose(nu, g["nu_hat"], rtol=1e-12, atol=0)
        dig = Digests(int(g["stride"]))
        U, rep = p.solve_m1_fixed_point(None, cfg, callback=dig)
    assert rep.iterations == int(g["iterations"]), (rep.iterations, int(g["iterations"]))
    assert rep.status == ("converged" if int(g["status"]) == 0 else rep.status)
    h, hr = np.asarray(rep.residual_history), g["history"]
    assert h.shape == hr.shape
    # residual history: within 1e-10 of the first residual everywhere
    # (measured 6e-12: late entries sit 1e-8 below the first, where the
    # two solvers' 1e-12-accurate block solves and fp64 rounding of the
    # residual set them apart by ~1e-14 absolute) and within 1e-7 relative
    # wherever the residual is above 1e-4 of the first
    assert np.max(np.abs(h - hr)) <= 1e-10 * hr[0], np.max(np.abs(h - hr)) / hr[0]
    big = hr > 1e-4 * hr[0]
    assert np.max(np.abs(h - hr)[big] / hr[big]) <= 1e-7
    _compare_iterates(dig, g)
    assert_checksum_close(checksum(U), g["U_checksum"], what="final U")


@pytest.mark.parametrize("config", [2, 3])
def test_sampled_slices_and_frequency_blocks(config):
    """Configs 2 and 3 at full size, per stage: static_init's per-slice
    damped Newton on sampled slices (solvers.hpp:282-294) and the frequency
    block solves (periodic.hpp:252-289) at k in {0, 1, N/4, N/2}, the latter
    through the production tp_periodic_solve on a right-hand side whose
    spectrum lives on exactly those frequencies: G_i = sum_k Re(b_k e^{2 pi i
    k i / N}) gives U_i = sum_k Re(x_k e^{2 pi i k i / N}) with x_k the block
    solutions.  The checker ran with its SparseSolver throw threshold at 1e-8
    (fixture `relaxed`): the reference's 1e-10 contract is below the fp64
    floor of ||b - A x|| on these grids."""
    g = golden(f"cfg{config}_sampled_reference.npz")
    d = baseline_desc(config)
    cfg = default_cfg(tol=1e-8)
    stride = int(g["stride"])
    slices = g["slices"]
    with Problem(d) as p:
        U0, counts = p.static_init(cfg)
        assert np.array_equal(counts[slices], g["newton_counts"]), (counts[slices], g["newton_counts"])
        for j, i in enumerate(slices):
            assert rel(U0[i, ::stride], g["U_slice_samples"][j]) <= ITERATE_TOL
            assert_checksum_close(checksum(U0[i]), g["U_slice_checksums"][j], what=f"slice {i}")
        del U0
        N, n = p.steps, p.n_dof
        ks = g["ks"]
        rng = np.random.default_rng(int(g["rhs_seed"]))
        B = np.empty((ks.size, n), dtype=np.complex128)
        for j, k in enumerate(ks):
            B[j] = rng.standard_normal(n) + (1j * rng.standard_normal(n) if 0 < 2 * k < N else 0)
        G = np.zeros((N, n))
        t = np.arange(N)
        for j, k in enumerate(ks):
            c, s = np.cos(2 * np.pi * k * t / N), np.sin(2 * np.pi * k * t / N)
            for i0 in range(0, N, 64):  # Re(b e^{i theta}) = Re b cos - Im b sin, in slice chunks
                G[i0:i0 + 64] += np.outer(c[i0:i0 + 64], B[j].real) - np.outer(s[i0:i0 + 64], B[j].imag)
        p.set_nu_hat(g["nu_hat"], 0.5)
        U = p.periodic_solve(G, cfg)
        del G
        X = g["X_samples"]
        for i in np.unique(np.linspace(0, N - 1, 6).round().astype(int)):
            want = sum((X[j] * np.exp(2j * np.pi * k * i / N)).real for j, k in enumerate(ks))
            assert rel(U[i, ::stride], want) <= ITERATE_TOL, (i, rel(U[i, ::stride], want))


@pytest.mark.parametrize("config,name", [(5, "cfg5_sweeps_reference.npz"), (4, "cfg4_sweeps_reference.npz"),
                                         (2, "cfg2_sweeps_reference.npz")])
def test_sweeps_from_zero_match_reference(config, name):
    """Full-size sweeps from U^0 = 0 (SURVEY.md §8(d) secondary parity case)
    with theory-mode nu_hat (assembly.hpp:280-283), then the reference's
    first sweeps.  Config 5 is config 4's linear control (nu == nu0): one
    sweep converges."""
    g = golden(name)
    count = int(g["iterations"])
    cfg = default_cfg(tol=1e-12, m1_max_outer=count, nu_hat_mode=TP_NU_HAT_THEORY)
    with Problem(baseline_desc(config)) as p:
        U0 = np.zeros(p.shape)
        p.set_state(U0)
        nu, q = p.choose_nu_hat(cfg)
        assert np.allclose(nu, g["nu_hat"], rtol=1e-12, atol=0)
        dig = Digests(int(g["stride"]))
        U, rep = p.solve_m1_fixed_point(U0, cfg, callback=dig)
    assert rep.iterations == count
    h, hr = np.asarray(rep.residual_history), g["history"]
    assert h.shape == hr.shape
    # ||R(0)|| = ||F|| summed over 5e8 entries in two different orders:
    # measured 1.2e-12 apart at cfg 5, 1.1e-11 at cfg 2 (whose later
    # residuals agree to 1.7e-13 and iterates to 7e-14: the difference is
    # the summation of a norm dominated by few coil entries,
    # profiles/r2o_cfg2_diag.txt)
    assert abs(h[0] - hr[0]) <= (3e-11 if config == 2 else 1e-11) * hr[0]
    # within 1e-10 of the first residual everywhere (config 4: 1e-9), 1e-6
    # relative where the residual is above 1e-6 of the first (config 5 lands
    # at the rounding floor after its one sweep: 1.5e-11 vs 5.0e-12 against a
    # first 2.6).  Config 4 (J0 = 200, Bs = 0.5, nu_inf = 50) evaluates
    # R = F - K(U) with terms far above their sum: its history agrees to
    # 2.0e-10 of the first residual while the iterates agree to 3e-14, for
    # any block tolerance 1e-12..1e-14 (tools/zero_sweeps_diag.py,
    # profiles/r2o_cfg4_diag.txt) -- the residual's own rounding
    hist_tol = 1e-9 if config == 4 else 1e-10
    assert np.max(np.abs(h - hr)) <= hist_tol * hr[0], (h, hr)
    big = hr > 1e-6 * hr[0]
    assert np.max(np.abs(h - hr)[big] / hr[big]) <= 1e-6, (h, hr)
    if config == 5:  # the linear control converges in one sweep (BASELINE.json configs[4])
        assert h[1] <= 1e-10 * h[0] and hr[1] <= 1e-10 * hr[0]
    _compare_iterates(dig, g)


def test_cfg4_sweeps_from_static_init_match_reference():
    """Config 4 from the production start: the reference's static_init over
    all 2048 slices, frozen-field nu_hat, then its first three M1 sweeps --
    Newton counts, U^0, nu_hat, the residual history (which rises over the
    first sweeps from static_init, on both sides) and every iterate."""
    g = golden("cfg4_static_sweeps_reference.npz")
    count = int(g["iterations"])
    cfg = default_cfg(tol=1e-12, m1_max_outer=count)
    with Problem(baseline_desc(4)) as p:
        U0, counts = p.static_init(cfg)
        assert np.array_equal(counts, g["newton_counts"])
        assert_checksum_close(checksum(U0), g["U0_checksum"], what="U0", size=U0.size)
        assert rel(U0.reshape(-1)[::int(g["stride"])], g["U0_sample"]) <= ITERATE_TOL
        nu, q = p.choose_nu_hat(cfg)
        assert np.allclose(nu, g["nu_hat"], rtol=1e-12, atol=0)
        dig = Digests(int(g["stride"]))
        U, rep = p.solve_m1_fixed_point(None, cfg, callback=dig)
    assert rep.iterations == count
    h, hr = np.asarray(rep.residual_history), g["history"]
    assert h.shape == hr.shape
    assert np.max(np.abs(h - hr) / hr) <= 1e-8, (h, hr)
    _compare_iterates(dig, g)
