"""TEST INFRASTRUCTURE ONLY -- ctypes front end of oracle/_ref/libtpref.so.

libtpref.so is the reference's own solver templates (tpfem, compiled from
/root/reference/proj/include by oracle/Makefile with the shim SparseSolver)
driving the BASELINE grid physics (oracle/grid_problem.hpp).  Only tests/,
__graft_entry__.smoke() and bench.py's CPU legs may use this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from paper_2502_21013_b200.abi import (TP_OK, TpProblemDesc, TpSolverCfg, default_cfg)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libtpref.so")
_lib = None


class RefError(RuntimeError):
    def __init__(self, code, msg, residual):
        super().__init__(f"[{code}] {msg}")
        self.code, self.residual = code, residual


def available() -> bool:
    return os.path.exists(LIB_PATH)


def select(variant: str = "") -> None:
    """Switch to another build of the checker: "" = libtpref.so (the
    reference's 1e-10 SparseSolver contract), "relaxed" = libtpref_relaxed.so
    (same build, shim throw threshold 1e-8: BASELINE grids >= 1024^2 where
    1e-10 is below the fp64 residual floor)."""
    global LIB_PATH, _lib
    LIB_PATH = os.path.join(_HERE, "_ref", "libtpref_relaxed.so" if variant == "relaxed" else "libtpref.so")
    _lib = None


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} missing: run `make -C oracle` where /root/reference exists")
        L = C.CDLL(LIB_PATH)
        dp = C.POINTER(C.c_double)
        ip = C.POINTER(C.c_int32)
        D = C.POINTER(TpProblemDesc)
        G = C.POINTER(TpSolverCfg)
        L.tpref_last_error.argtypes = [C.c_char_p, C.c_size_t, dp]
        L.tpref_desc_baseline.argtypes = [C.c_int32, D]
        L.tpref_hardware_threads.argtypes = []
        L.tpref_sizes.argtypes = [D, ip, ip, dp]
        L.tpref_loads.argtypes = [D, dp]
        L.tpref_mass.argtypes = [D, dp]
        L.tpref_sigma.argtypes = [D, dp]
        L.tpref_apply_k.argtypes = [D, dp, dp, C.c_int32]
        L.tpref_jacobian_apply.argtypes = [D, dp, dp, dp]
        L.tpref_static_init.argtypes = [D, G, dp, ip]
        L.tpref_choose_nu_hat.argtypes = [D, G, dp, dp, dp]
        L.tpref_residual.argtypes = [D, dp, dp, dp, C.c_int32]
        L.tpref_periodic_solve.argtypes = [D, G, dp, dp, dp]
        L.tpref_solve_m1.argtypes = [D, G, dp, C.c_double, dp, dp, dp, dp, C.c_int32, ip, ip, dp,
                                     C.c_int32, dp]
        L.tpref_solve_m2.argtypes = [D, G, dp, dp, dp, C.c_int32, ip, ip, dp]
        L.tpref_solve_m3.argtypes = [D, G, dp, dp, dp, C.c_int32, ip, ip, dp]
        _lib = L
    return _lib


def _ptr(a):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(C.c_double if a.dtype == np.float64 else C.c_int32))


def _check(code):
    if code != TP_OK:
        buf = C.create_string_buffer(1024)
        res = C.c_double()
        lib().tpref_last_error(buf, 1024, C.byref(res))
        raise RefError(code, buf.value.decode(), res.value)


def baseline_desc(config: int) -> TpProblemDesc:
    d = TpProblemDesc()
    _check(lib().tpref_desc_baseline(config, C.byref(d)))
    return d


def hardware_threads() -> int:
    return int(lib().tpref_hardware_threads())


def sizes(desc):
    n, N, tau = C.c_int32(), C.c_int32(), C.c_double()
    _check(lib().tpref_sizes(C.byref(desc), C.byref(n), C.byref(N), C.byref(tau)))
    return n.value, N.value, tau.value


def loads(desc):
    n, N, _ = sizes(desc)
    F = np.zeros((N, n))
    _check(lib().tpref_loads(C.byref(desc), _ptr(F)))
    return F


def mass(desc):
    n, _, _ = sizes(desc)
    m = np.zeros(n)
    _check(lib().tpref_mass(C.byref(desc), _ptr(m)))
    return m


def sigma(desc):
    c = desc.cells
    s = np.zeros(2 * c * c)
    _check(lib().tpref_sigma(C.byref(desc), _ptr(s)))
    return s


def apply_k(desc, U):
    U = np.ascontiguousarray(U, dtype=np.float64)
    out = np.zeros_like(U)
    cnt = 1 if U.ndim == 1 else U.shape[0]
    _check(lib().tpref_apply_k(C.byref(desc), _ptr(U), _ptr(out), cnt))
    return out


def jacobian_apply(desc, u, v):
    u = np.ascontiguousarray(u, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    y = np.zeros_like(v)
    _check(lib().tpref_jacobian_apply(C.byref(desc), _ptr(u), _ptr(v), _ptr(y)))
    return y


def static_init(desc, cfg: TpSolverCfg | None = None):
    cfg = cfg or default_cfg()
    n, N, _ = sizes(desc)
    U0 = np.zeros((N, n))
    counts = np.zeros(N, dtype=np.int32)
    _check(lib().tpref_static_init(C.byref(desc), C.byref(cfg), _ptr(U0), _ptr(counts)))
    return U0, counts


def choose_nu_hat(desc, U0, cfg: TpSolverCfg | None = None):
    cfg = cfg or default_cfg()
    U0 = np.ascontiguousarray(U0, dtype=np.float64)
    nu = np.zeros(5)
    q = C.c_double()
    _check(lib().tpref_choose_nu_hat(C.byref(desc), C.byref(cfg), _ptr(U0), _ptr(nu), C.byref(q)))
    return nu, q.value


def residual(desc, U, threads=0):
    U = np.ascontiguousarray(U, dtype=np.float64)
    R = np.zeros_like(U)
    nrm = C.c_double()
    _check(lib().tpref_residual(C.byref(desc), _ptr(U), _ptr(R), C.byref(nrm),
                                threads or hardware_threads()))
    return R, nrm.value


def periodic_solve(desc, nu_hat, G, cfg: TpSolverCfg | None = None):
    cfg = cfg or default_cfg()
    G = np.ascontiguousarray(G, dtype=np.float64)
    U = np.zeros_like(G)
    nu = np.ascontiguousarray(nu_hat, dtype=np.float64)
    _check(lib().tpref_periodic_solve(C.byref(desc), C.byref(cfg), _ptr(nu), _ptr(G), _ptr(U)))
    return U


@dataclass
class RefM1Result:
    U: np.ndarray
    history: np.ndarray
    contraction: np.ndarray
    iterations: int
    status: int
    iterates: np.ndarray | None = None
    wall_time: float = 0.0
    setup_time: float = 0.0


def solve_m1(desc, nu_hat, q, U0, cfg: TpSolverCfg | None = None, keep_iterates=False,
             cache=0) -> RefM1Result:
    """tpfem::solve_m1_fixed_point on the grid problem (solvers.hpp:301-369)."""
    cfg = cfg or default_cfg()
    U0 = np.ascontiguousarray(U0, dtype=np.float64)
    cap = cfg.m1_max_outer + 1
    hist = np.zeros(cap)
    contr = np.zeros(cap)
    it = C.c_int32()
    st = C.c_int32()
    U = np.zeros_like(U0)
    its = np.zeros((cap,) + U0.shape) if keep_iterates else None
    times = np.zeros(2)
    nu = np.ascontiguousarray(nu_hat, dtype=np.float64)
    _check(lib().tpref_solve_m1(C.byref(desc), C.byref(cfg), _ptr(nu), q, _ptr(U0), _ptr(U),
                                _ptr(hist), _ptr(contr), cap, C.byref(it), C.byref(st),
                                _ptr(its), cache, _ptr(times)))
    k = it.value
    return RefM1Result(U=U, history=hist[:k + 1].copy(), contraction=contr[:k].copy(),
                       iterations=k, status=st.value,
                       iterates=None if its is None else its[:k + 1].copy(),
                       wall_time=float(times[0]), setup_time=float(times[1]))


def solve_m2(desc, U0, cfg: TpSolverCfg | None = None):
    """tpfem::solve_m2_newton on the grid problem (solvers.hpp:375-484).
    Returns (U, history, iterations, status, wall seconds)."""
    cfg = cfg or default_cfg()
    U0 = np.ascontiguousarray(U0, dtype=np.float64)
    cap = cfg.m2_max_outer + 1
    hist = np.zeros(cap)
    it = C.c_int32()
    st = C.c_int32()
    wall = np.zeros(1)
    U = np.zeros_like(U0)
    _check(lib().tpref_solve_m2(C.byref(desc), C.byref(cfg), _ptr(U0), _ptr(U), _ptr(hist), cap, C.byref(it),
                                C.byref(st), _ptr(wall)))
    k = it.value
    return U, hist[:k + 1].copy(), k, st.value, float(wall[0])


def solve_m3(desc, U0, cfg: TpSolverCfg | None = None):
    """tpfem::solve_m3_timestepping on the grid problem (solvers.hpp:489-542).
    Returns (U, history, iterations, status, wall seconds)."""
    cfg = cfg or default_cfg()
    U0 = np.ascontiguousarray(U0, dtype=np.float64)
    cap = cfg.m3_max_cycles + 1
    hist = np.zeros(cap)
    it = C.c_int32()
    st = C.c_int32()
    wall = np.zeros(1)
    U = np.zeros_like(U0)
    _check(lib().tpref_solve_m3(C.byref(desc), C.byref(cfg), _ptr(U0), _ptr(U), _ptr(hist), cap, C.byref(it),
                                C.byref(st), _ptr(wall)))
    k = it.value
    return U, hist[:k + 1].copy(), k, st.value, float(wall[0])


# ---------------------------------------------------------------- transformer (reference physics)
class TrCfg(C.Structure):
    """tpref_mesh_cfg: configs/transformer.json fields (RunConfig, config.hpp:39-53)."""
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("refinements", C.c_int32), ("steps", C.c_int32),
                ("period", C.c_double), ("s_max", C.c_double), ("flux_samples", C.c_int32),
                ("pad_", C.c_int32), ("j_amp", C.c_double)]


def tr_cfg(nx=40, ny=40, refinements=0, steps=64, period=0.02, s_max=3.0, flux_samples=10001,
           j_amp=0.0) -> TrCfg:
    """j_amp: winding amplitude override (0: MaterialTable::transformer's 1.9e4;
    configs/transformer_saturated.json uses 9.5e5)."""
    return TrCfg(nx, ny, refinements, steps, period, s_max, flux_samples, 0, j_amp)


def _trlib():
    L = lib()
    if not getattr(L, "_tr_ready", False):
        dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int32)
        T, G = C.POINTER(TrCfg), C.POINTER(TpSolverCfg)
        L.tpref_tr_mesh.argtypes = [C.c_int32, C.c_int32, C.c_int32, ip, ip, ip, dp, ip, ip]
        L.tpref_tr_loads.argtypes = [T, dp]
        L.tpref_tr_mass.argtypes = [T, ip, ip, ip, ip, dp]
        L.tpref_tr_apply_k.argtypes = [T, dp, dp, C.c_int32]
        L.tpref_tr_residual.argtypes = [T, dp, dp, dp]
        L.tpref_tr_static_init.argtypes = [T, G, dp, ip]
        L.tpref_tr_choose_nu_hat.argtypes = [T, G, dp, dp, dp]
        L.tpref_tr_periodic_solve.argtypes = [T, G, dp, dp, dp]
        L.tpref_tr_solve_m1.argtypes = [T, G, dp, C.c_double, dp, dp, dp, C.c_int32, ip, ip, dp, dp]
        L.tpref_tr_solve_m23.argtypes = [T, G, C.c_int32, dp, dp, dp, C.c_int32, ip, ip, dp]
        L._tr_ready = True
    return L


def tr_mesh(nx, ny, refinements=0):
    """build_rectilinear_mesh(transformer_regions()) + refine_uniform (mesh.hpp:139-246):
    (vertices (nv, 2), triangles (nt, 3), region (nt,), n_dof)."""
    L = _trlib()
    nv, nt, nd = C.c_int32(), C.c_int32(), C.c_int32()
    _check(L.tpref_tr_mesh(nx, ny, refinements, C.byref(nv), C.byref(nt), C.byref(nd), None, None, None))
    V = np.zeros((nv.value, 2))
    Tr = np.zeros((nt.value, 3), dtype=np.int32)
    R = np.zeros(nt.value, dtype=np.int32)
    _check(L.tpref_tr_mesh(nx, ny, refinements, None, None, None, _ptr(V), _ptr(Tr), _ptr(R)))
    return V, Tr, R, nd.value


def tr_sizes(c: TrCfg):
    return tr_mesh(c.nx, c.ny, c.refinements)[3], c.steps


def tr_loads(c: TrCfg):
    n, N = tr_sizes(c)
    F = np.zeros((N, n))
    _check(_trlib().tpref_tr_loads(C.byref(c), _ptr(F)))
    return F


def tr_apply_k(c: TrCfg, U):
    U = np.ascontiguousarray(U, dtype=np.float64)
    out = np.zeros_like(U)
    _check(_trlib().tpref_tr_apply_k(C.byref(c), _ptr(U), _ptr(out), 1 if U.ndim == 1 else U.shape[0]))
    return out


def tr_residual(c: TrCfg, U):
    U = np.ascontiguousarray(U, dtype=np.float64)
    R = np.zeros_like(U)
    nrm = C.c_double()
    _check(_trlib().tpref_tr_residual(C.byref(c), _ptr(U), _ptr(R), C.byref(nrm)))
    return R, nrm.value


def tr_static_init(c: TrCfg, cfg: TpSolverCfg | None = None):
    cfg = cfg or default_cfg()
    n, N = tr_sizes(c)
    U0 = np.zeros((N, n))
    counts = np.zeros(N, dtype=np.int32)
    _check(_trlib().tpref_tr_static_init(C.byref(c), C.byref(cfg), _ptr(U0), _ptr(counts)))
    return U0, counts


def tr_choose_nu_hat(c: TrCfg, U0, cfg: TpSolverCfg | None = None):
    cfg = cfg or default_cfg()
    U0 = np.ascontiguousarray(U0, dtype=np.float64)
    nu = np.zeros(5)
    q = C.c_double()
    _check(_trlib().tpref_tr_choose_nu_hat(C.byref(c), C.byref(cfg), _ptr(U0), _ptr(nu), C.byref(q)))
    return nu, q.value


def tr_periodic_solve(c: TrCfg, nu_hat, G, cfg: TpSolverCfg | None = None):
    cfg = cfg or default_cfg()
    G = np.ascontiguousarray(G, dtype=np.float64)
    U = np.zeros_like(G)
    nu = np.ascontiguousarray(nu_hat, dtype=np.float64)
    _check(_trlib().tpref_tr_periodic_solve(C.byref(c), C.byref(cfg), _ptr(nu), _ptr(G), _ptr(U)))
    return U


def tr_solve_m1(c: TrCfg, nu_hat, q, U0, cfg: TpSolverCfg | None = None, keep_iterates=False) -> RefM1Result:
    """solve_m1_fixed_point on the reference's own transformer problem."""
    cfg = cfg or default_cfg()
    U0 = np.ascontiguousarray(U0, dtype=np.float64)
    cap = cfg.m1_max_outer + 1
    hist = np.zeros(cap)
    it, st = C.c_int32(), C.c_int32()
    U = np.zeros_like(U0)
    its = np.zeros((cap,) + U0.shape) if keep_iterates else None
    wall = np.zeros(1)
    nu = np.ascontiguousarray(nu_hat, dtype=np.float64)
    _check(_trlib().tpref_tr_solve_m1(C.byref(c), C.byref(cfg), _ptr(nu), q, _ptr(U0), _ptr(U), _ptr(hist), cap,
                                      C.byref(it), C.byref(st), _ptr(its), _ptr(wall)))
    k = it.value
    return RefM1Result(U=U, history=hist[:k + 1].copy(), contraction=np.zeros(0), iterations=k, status=st.value,
                       iterates=None if its is None else its[:k + 1].copy(), wall_time=float(wall[0]))


def tr_solve_m23(c: TrCfg, method: int, U0, cfg: TpSolverCfg | None = None):
    """solve_m2_newton (method 2) / solve_m3_timestepping (3) on the reference
    transformer: (U, history, iterations, status, wall seconds)."""
    cfg = cfg or default_cfg()
    U0 = np.ascontiguousarray(U0, dtype=np.float64)
    cap = (cfg.m2_max_outer if method == 2 else cfg.m3_max_cycles) + 1
    hist = np.zeros(cap)
    it, st = C.c_int32(), C.c_int32()
    wall = np.zeros(1)
    U = np.zeros_like(U0)
    _check(_trlib().tpref_tr_solve_m23(C.byref(c), C.byref(cfg), method, _ptr(U0), _ptr(U), _ptr(hist), cap,
                                       C.byref(it), C.byref(st), _ptr(wall)))
    k = it.value
    return U, hist[:k + 1].copy(), k, st.value, float(wall[0])


# ---------------------------------------------------------------- large-config parity support
def _biglib():
    L = lib()
    if not getattr(L, "_big_ready", False):
        dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int32)
        D, G = C.POINTER(TpProblemDesc), C.POINTER(TpSolverCfg)
        L.tpref_solve_m1_digest.argtypes = [D, G, dp, C.c_double, dp, dp, dp, dp, C.c_int32, ip, ip, dp,
                                            C.c_int64, dp, C.c_int32, dp]
        L.tpref_static_init_slices.argtypes = [D, G, ip, C.c_int32, dp, ip]
        L.tpref_frequency_blocks.argtypes = [D, G, dp, ip, C.c_int32, dp, dp]
        L._big_ready = True
    return L


@dataclass
class RefM1Digest:
    U: np.ndarray
    history: np.ndarray
    contraction: np.ndarray
    iterations: int
    status: int
    digests: np.ndarray      # (iterations+1) x 5: norm, sum, cos-weighted sum, max|.|, ||U^k - U^{k-1}||
    samples: np.ndarray      # (iterations+1) x ceil(N n / stride): U^k[::stride]
    wall_time: float = 0.0


def solve_m1_digest(desc, nu_hat, q, U0, cfg: TpSolverCfg | None = None, stride=997, cache=0) -> RefM1Digest:
    """solve_m1_fixed_point (solvers.hpp:301-369) keeping per-iterate digests
    and strided samples instead of whole iterates."""
    cfg = cfg or default_cfg()
    U0 = np.ascontiguousarray(U0, dtype=np.float64)
    cap = cfg.m1_max_outer + 1
    hist, contr = np.zeros(cap), np.zeros(cap)
    it, st = C.c_int32(), C.c_int32()
    U = np.zeros_like(U0)
    dig = np.zeros((cap, 5))
    ns = -(-U0.size // stride)
    smp = np.zeros((cap, ns))
    wall = np.zeros(1)
    nu = np.ascontiguousarray(nu_hat, dtype=np.float64)
    _check(_biglib().tpref_solve_m1_digest(C.byref(desc), C.byref(cfg), _ptr(nu), q, _ptr(U0), _ptr(U),
                                           _ptr(hist), _ptr(contr), cap, C.byref(it), C.byref(st), _ptr(dig),
                                           stride, _ptr(smp), cache, _ptr(wall)))
    k = it.value
    return RefM1Digest(U=U, history=hist[:k + 1].copy(), contraction=contr[:k].copy(), iterations=k,
                       status=st.value, digests=dig[:k + 1].copy(), samples=smp[:k + 1].copy(),
                       wall_time=float(wall[0]))


def static_init_slices(desc, slices, cfg: TpSolverCfg | None = None):
    """static_init's per-slice Newton (solvers.hpp:282-294) on the listed slices:
    (U (len x n), newton counts)."""
    cfg = cfg or default_cfg()
    n, _, _ = sizes(desc)
    sl = np.ascontiguousarray(slices, dtype=np.int32)
    U = np.zeros((sl.size, n))
    counts = np.zeros(sl.size, dtype=np.int32)
    _check(_biglib().tpref_static_init_slices(C.byref(desc), C.byref(cfg), _ptr(sl), sl.size, _ptr(U),
                                              _ptr(counts)))
    return U, counts


def frequency_blocks(desc, nu_hat, ks, B, cfg: TpSolverCfg | None = None):
    """(lambda_k M + K_hat) x_k = b_k for the listed k (solve_frequency,
    periodic.hpp:252-289); B: len(ks) x n complex."""
    cfg = cfg or default_cfg()
    ks = np.ascontiguousarray(ks, dtype=np.int32)
    B = np.ascontiguousarray(B, dtype=np.complex128)
    X = np.zeros_like(B)
    nu = np.ascontiguousarray(nu_hat, dtype=np.float64)
    _check(_biglib().tpref_frequency_blocks(C.byref(desc), C.byref(cfg), _ptr(nu), _ptr(ks), ks.size,
                                            B.ctypes.data_as(C.POINTER(C.c_double)),
                                            X.ctypes.data_as(C.POINTER(C.c_double))))
    return X


STAGES = ("A_rhs", "B_forward_dft", "D_inverse_dft", "E_residual", "C_blocks")


def sweep_sample(desc, nu_hat, slices, cols, blocks=0, threads=0, reps=1):
    """Stage-by-stage timing of one reference sweep on a bounded sample
    (tpref_sweep_sample), `reps` times after one setup: (list of dicts of
    seconds for A (RHS on `slices` slices), B / D (forward / inverse
    transforms on `cols` columns), E (residual on the slices), C (`blocks`
    frequency-block solves), setup seconds)."""
    L = lib()
    if not getattr(L, "_ss_ready", False):
        dp = C.POINTER(C.c_double)
        L.tpref_sweep_sample.argtypes = [C.POINTER(TpProblemDesc), C.POINTER(TpSolverCfg), dp, C.c_int32,
                                         C.c_int32, C.c_int32, C.c_int32, dp, dp]
        L._ss_ready = True
    cfg = default_cfg(threads=threads or hardware_threads())
    t = np.zeros((max(1, reps), 5))
    setup = C.c_double()
    nu = np.ascontiguousarray(nu_hat, dtype=np.float64)
    _check(L.tpref_sweep_sample(C.byref(desc), C.byref(cfg), _ptr(nu), slices, cols, blocks, reps, _ptr(t),
                                C.byref(setup)))
    return [dict(zip(STAGES, row.tolist())) for row in t], setup.value
