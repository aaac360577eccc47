"""General-mesh path: the reference's own P1 meshes and transformer physics
over the C ABI of include/tpgpu_mesh.h.

Names follow tpfem (/root/reference/proj/include/tpfem):
  transformer_mesh            build_rectilinear_mesh(transformer_regions())
                              + refine_uniform          mesh.hpp:139-246, runner.hpp:27-31
  transformer_materials       MaterialTable::transformer  materials.hpp:67-79
  MeshProblem.transformer     setup_transformer up to static_init  runner.hpp:46-73
  MeshProblem.static_init     static_init               solvers.hpp:276-296
  MeshProblem.choose_nu_hat   choose_nu_hat + flux_bounds  assembly.hpp:236-303
  MeshProblem.solve_m1_fixed_point  solve_m1_fixed_point  solvers.hpp:301-369
  MeshProblem.periodic_solve  PeriodicSolver::solve     periodic.hpp:154-198
  MeshProblem.solve_m2_newton solve_m2_newton           solvers.hpp:375-484
  MeshProblem.solve_m3_timestepping solve_m3_timestepping solvers.hpp:489-542
  MeshProblem.residual        residual + block_l2       periodic.hpp:35-67
  MeshProblem.apply_k         NonlinearOperator::apply  assembly.hpp:126-140
Errors as in api.py (ValueError / SolveError / RuntimeError); no CPU fallback.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from .abi import STATUS_NAMES, TP_ITERATE_CB, TpReport, TpSolverCfg, default_cfg
from .api import SolveReport, _check, _dp, _ip, lib

REGIONS = ("steel", "iron", "air", "winding_plus", "winding_minus")  # mesh.hpp:17-23

MESH_EXPORTS = [
    "tp_material_table_transformer", "tp_transformer_mesh", "tp_mesh_problem_create", "tp_mesh_problem_destroy",
    "tp_mesh_problem_sizes", "tp_mesh_loads", "tp_mesh_apply_k", "tp_mesh_residual", "tp_mesh_static_init",
    "tp_mesh_set_state", "tp_mesh_get_state", "tp_mesh_choose_nu_hat", "tp_mesh_set_nu_hat",
    "tp_mesh_periodic_solve", "tp_mesh_solve_m1", "tp_mesh_m1_begin", "tp_mesh_m1_sweep", "tp_mesh_problem_stream",
    "tp_mesh_problem_launches", "tp_mesh_solve_m2", "tp_mesh_solve_m3",
]


class TpExpMaterial(C.Structure):
    """MaterialCoefficients (materials.hpp:17-24)."""
    _fields_ = [("sigma", C.c_double), ("a", C.c_double), ("b", C.c_double), ("c", C.c_double),
                ("d", C.c_double), ("j_amp", C.c_double)]


class TpMeshDesc(C.Structure):
    _fields_ = [("n_vertices", C.c_int32), ("n_triangles", C.c_int32),
                ("vertices", C.POINTER(C.c_double)), ("triangles", C.POINTER(C.c_int32)),
                ("region", C.POINTER(C.c_int32)), ("material", TpExpMaterial * 5),
                ("steps", C.c_int32), ("flux_samples", C.c_int32), ("period", C.c_double),
                ("s_max", C.c_double)]


def _mlib():
    L = lib()
    if not getattr(L, "_mesh_ready", False):
        vp, dp, ip = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int32)
        G = C.POINTER(TpSolverCfg)
        L.tp_material_table_transformer.argtypes = [C.POINTER(TpExpMaterial)]
        L.tp_material_table_transformer.restype = None
        L.tp_transformer_mesh.argtypes = [C.c_int32, C.c_int32, C.c_int32, ip, ip, ip, dp, ip, ip]
        L.tp_mesh_problem_create.argtypes = [C.POINTER(TpMeshDesc), C.c_int32, C.POINTER(vp)]
        L.tp_mesh_problem_destroy.argtypes = [vp]
        L.tp_mesh_problem_destroy.restype = None
        L.tp_mesh_problem_sizes.argtypes = [vp, ip, ip, dp, ip]
        L.tp_mesh_loads.argtypes = [vp, dp]
        L.tp_mesh_apply_k.argtypes = [vp, dp, dp, C.c_int32]
        L.tp_mesh_residual.argtypes = [vp, dp, dp, dp]
        L.tp_mesh_static_init.argtypes = [vp, G, dp, ip]
        L.tp_mesh_set_state.argtypes = [vp, dp]
        L.tp_mesh_get_state.argtypes = [vp, dp]
        L.tp_mesh_choose_nu_hat.argtypes = [vp, G, dp, dp]
        L.tp_mesh_set_nu_hat.argtypes = [vp, dp, C.c_double]
        L.tp_mesh_periodic_solve.argtypes = [vp, G, dp, dp]
        L.tp_mesh_solve_m1.argtypes = [vp, G, dp, dp, C.POINTER(TpReport), dp, dp, C.c_int32, TP_ITERATE_CB, vp]
        for fn in ("tp_mesh_solve_m2", "tp_mesh_solve_m3"):
            getattr(L, fn).argtypes = [vp, G, dp, dp, C.POINTER(TpReport), dp, dp, C.c_int32]
        L.tp_mesh_m1_begin.argtypes = [vp, G, dp]
        L.tp_mesh_m1_sweep.argtypes = [vp, dp]
        L.tp_mesh_problem_stream.argtypes = [vp]
        L.tp_mesh_problem_stream.restype = vp
        L.tp_mesh_problem_launches.argtypes = [vp]
        L.tp_mesh_problem_launches.restype = C.c_int64
        L._mesh_ready = True
    return L


def transformer_materials(j_amp: float | None = None):
    """MaterialTable::transformer(); j_amp overrides the winding amplitude
    (+j_amp / -j_amp, as configs/transformer_saturated.json does with 9.5e5)."""
    m = (TpExpMaterial * 5)()
    _mlib().tp_material_table_transformer(m)
    if j_amp is not None:
        m[3].j_amp = j_amp
        m[4].j_amp = -j_amp
    return m


def transformer_mesh(nx: int = 40, ny: int = 40, refinements: int = 0):
    """(vertices (nv, 2), triangles (nt, 3), region (nt,), n_dof) of the
    reference's transformer mesh (host C++ in libtpgpu, no device needed)."""
    L = _mlib()
    nv, nt, nd = C.c_int32(), C.c_int32(), C.c_int32()
    _check(L.tp_transformer_mesh(nx, ny, refinements, C.byref(nv), C.byref(nt), C.byref(nd), None, None, None))
    V = np.zeros((nv.value, 2))
    T = np.zeros((nt.value, 3), dtype=np.int32)
    R = np.zeros(nt.value, dtype=np.int32)
    _check(L.tp_transformer_mesh(nx, ny, refinements, None, None, None, _dp(V), _ip(T), _ip(R)))
    return V, T, R, nd.value


class MeshProblem:
    """A P1 problem on a device (tp_mesh_problem)."""

    def __init__(self, vertices, triangles, region, materials, steps: int, period: float, s_max: float = 3.0,
                 flux_samples: int = 10001, device: int = 0):
        self._V = np.ascontiguousarray(vertices, dtype=np.float64)
        self._T = np.ascontiguousarray(triangles, dtype=np.int32)
        self._R = np.ascontiguousarray(region, dtype=np.int32)
        d = TpMeshDesc()
        d.n_vertices, d.n_triangles = self._V.shape[0], self._T.shape[0]
        d.vertices, d.triangles, d.region = _dp(self._V), _ip(self._T), _ip(self._R)
        for r in range(5):
            d.material[r] = materials[r]
        d.steps, d.period, d.s_max, d.flux_samples = steps, period, s_max, flux_samples
        self._h = C.c_void_p()
        _check(_mlib().tp_mesh_problem_create(C.byref(d), device, C.byref(self._h)))
        n, N, bw, tau = C.c_int32(), C.c_int32(), C.c_int32(), C.c_double()
        _check(_mlib().tp_mesh_problem_sizes(self._h, C.byref(n), C.byref(N), C.byref(tau), C.byref(bw)))
        self.n_dof, self.steps, self.tau, self.bandwidth = n.value, N.value, tau.value, bw.value

    @classmethod
    def transformer(cls, nx=40, ny=40, refinements=0, steps=64, period=0.02, j_amp=None, device=0):
        """configs/transformer.json (j_amp=9.5e5: transformer_saturated.json)."""
        V, T, R, _ = transformer_mesh(nx, ny, refinements)
        return cls(V, T, R, transformer_materials(j_amp), steps, period, device=device)

    def close(self):
        if self._h:
            _mlib().tp_mesh_problem_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def shape(self):
        return (self.steps, self.n_dof)

    def _state(self, U):
        U = np.ascontiguousarray(U, dtype=np.float64)
        if U.shape != self.shape:
            raise ValueError(f"state shape {U.shape} != {self.shape}")
        return U

    def loads(self):
        F = np.zeros(self.shape)
        _check(_mlib().tp_mesh_loads(self._h, _dp(F)))
        return F

    def apply_k(self, U):
        U = np.ascontiguousarray(U, dtype=np.float64)
        cnt = 1 if U.ndim == 1 else U.shape[0]
        out = np.zeros_like(U)
        _check(_mlib().tp_mesh_apply_k(self._h, _dp(U), _dp(out), cnt))
        return out

    def residual(self, U):
        U = self._state(U)
        R = np.zeros_like(U)
        nrm = C.c_double()
        _check(_mlib().tp_mesh_residual(self._h, _dp(U), _dp(R), C.byref(nrm)))
        return R, nrm.value

    def static_init(self, cfg: TpSolverCfg | None = None):
        cfg = cfg or default_cfg()
        U0 = np.zeros(self.shape)
        counts = np.zeros(self.steps, dtype=np.int32)
        _check(_mlib().tp_mesh_static_init(self._h, C.byref(cfg), _dp(U0), _ip(counts)))
        return U0, counts

    def set_state(self, U):
        _check(_mlib().tp_mesh_set_state(self._h, _dp(self._state(U))))

    def get_state(self):
        U = np.zeros(self.shape)
        _check(_mlib().tp_mesh_get_state(self._h, _dp(U)))
        return U

    def choose_nu_hat(self, cfg: TpSolverCfg | None = None):
        cfg = cfg or default_cfg()
        nu = np.zeros(5)
        q = C.c_double()
        _check(_mlib().tp_mesh_choose_nu_hat(self._h, C.byref(cfg), _dp(nu), C.byref(q)))
        return nu, q.value

    def set_nu_hat(self, nu_hat, q=float("nan")):
        nu = np.ascontiguousarray(nu_hat, dtype=np.float64)
        _check(_mlib().tp_mesh_set_nu_hat(self._h, _dp(nu), q))

    def periodic_solve(self, G, cfg: TpSolverCfg | None = None):
        cfg = cfg or default_cfg()
        G = self._state(G)
        U = np.zeros_like(G)
        _check(_mlib().tp_mesh_periodic_solve(self._h, C.byref(cfg), _dp(G), _dp(U)))
        return U

    def solve_m1_fixed_point(self, U0=None, cfg: TpSolverCfg | None = None, iterate_log=None):
        """Returns (U, SolveReport); iterate_log receives every iterate (solvers.hpp:306)."""
        cfg = cfg or default_cfg()
        U0a = None if U0 is None else self._state(U0)
        cap = cfg.m1_max_outer + 1
        hist, contr = np.zeros(cap), np.zeros(cap)
        U = np.zeros(self.shape)
        rep = TpReport()

        def _cb(k, ptr, res, user):
            arr = np.ctypeslib.as_array(ptr, shape=(self.steps * self.n_dof,))
            iterate_log.append(arr.reshape(self.shape).copy())
            return 0

        cb = TP_ITERATE_CB(_cb) if iterate_log is not None else TP_ITERATE_CB()
        _check(_mlib().tp_mesh_solve_m1(self._h, C.byref(cfg), _dp(U0a), _dp(U), C.byref(rep), _dp(hist),
                                        _dp(contr), cap, cb, None))
        k = rep.history_len
        return U, SolveReport(iterations=rep.iterations, residual_history=hist[:k].tolist(),
                              contraction_history=contr[:rep.contraction_len].tolist(), q_estimate=rep.q_estimate,
                              wall_time=rep.wall_time, status=STATUS_NAMES[rep.status],
                              setup_time=rep.setup_time, sweep_time=rep.sweep_time)

    def _m23(self, fn, method, cap, U0, cfg):
        U0a = None if U0 is None else self._state(U0)
        hist, contr = np.zeros(cap), np.zeros(cap)
        U = np.zeros(self.shape)
        rep = TpReport()
        _check(getattr(_mlib(), fn)(self._h, C.byref(cfg), _dp(U0a), _dp(U), C.byref(rep), _dp(hist), _dp(contr),
                                    cap))
        k = rep.history_len
        return U, SolveReport(method=method, iterations=rep.iterations, residual_history=hist[:k].tolist(),
                              contraction_history=contr[:rep.contraction_len].tolist(), q_estimate=rep.q_estimate,
                              wall_time=rep.wall_time, status=STATUS_NAMES[rep.status],
                              inner_iterations=rep.inner_iterations)

    def solve_m2_newton(self, U0=None, cfg: TpSolverCfg | None = None):
        """solve_m2_newton (solvers.hpp:375-484) -> (U, SolveReport)."""
        cfg = cfg or default_cfg()
        return self._m23("tp_mesh_solve_m2", "m2", cfg.m2_max_outer + 1, U0, cfg)

    def solve_m3_timestepping(self, U0=None, cfg: TpSolverCfg | None = None):
        """solve_m3_timestepping (solvers.hpp:489-542) -> (U, SolveReport)."""
        cfg = cfg or default_cfg()
        return self._m23("tp_mesh_solve_m3", "m3", cfg.m3_max_cycles + 1, U0, cfg)

    def m1_begin(self, cfg: TpSolverCfg | None = None) -> float:
        cfg = cfg or default_cfg()
        r = C.c_double()
        _check(_mlib().tp_mesh_m1_begin(self._h, C.byref(cfg), C.byref(r)))
        return r.value

    def m1_sweep(self) -> float:
        r = C.c_double()
        _check(_mlib().tp_mesh_m1_sweep(self._h, C.byref(r)))
        return r.value

    @property
    def stream(self) -> int:
        return int(_mlib().tp_mesh_problem_stream(self._h) or 0)

    @property
    def launches(self) -> int:
        return int(_mlib().tp_mesh_problem_launches(self._h))
