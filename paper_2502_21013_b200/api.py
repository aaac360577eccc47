"""Python mirror of the reference interface over the C ABI (include/tpgpu.h).

Names and semantics follow tpfem (/root/reference/proj/include/tpfem):
  Problem.static_init          static_init            solvers.hpp:276-296
  Problem.choose_nu_hat        choose_nu_hat          assembly.hpp:254-303
  Problem.solve_m1_fixed_point solve_m1_fixed_point   solvers.hpp:301-369
  Problem.periodic_solve       PeriodicSolver::solve  periodic.hpp:154-198
  Problem.residual / block_l2  residual, block_l2     periodic.hpp:35-67
  Problem.apply_k              NonlinearOperator::apply assembly.hpp:126-140
  stopping_check               stopping_check         solvers.hpp:100-103
  SolveError                   SolveError             solve.hpp:17-26
Errors raise like the reference: ValueError for invalid arguments
(std::invalid_argument), SolveError for numerical failure, and RuntimeError
for CUDA failures.  There is no CPU fallback: without the built library or a
GPU every call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from .abi import (TP_CONVERGED, TP_EINVAL, TP_ESOLVE, TP_ITERATE_CB, TP_OK, STATUS_NAMES,
                  TpProblemDesc, TpReport, TpShardPlan, TpSolverCfg, default_cfg)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtpgpu.so")
_lib = None

EXPORTS = [
    "tp_version", "tp_last_error", "tp_solver_cfg_default", "tp_problem_desc_baseline",
    "tp_problem_create", "tp_problem_destroy", "tp_problem_sizes", "tp_problem_loads",
    "tp_problem_mass", "tp_apply_k", "tp_residual", "tp_static_init", "tp_set_state",
    "tp_get_state", "tp_choose_nu_hat", "tp_set_nu_hat", "tp_periodic_solve", "tp_solve_m1", "tp_solve_m2", "tp_solve_m3",
    "tp_m1_begin", "tp_m1_sweep", "tp_sweep_stats", "tp_problem_stream", "tp_problem_launches",
    "tp_shard_plan_make", "tp_nccl_unique_id", "tp_comm_create", "tp_comm_destroy", "tp_comm_nccl",
    "tp_comm_rank", "tp_comm_size", "tp_comm_device", "tp_problem_create_sharded", "tp_problem_shard",
    "tp_kernel_timer", "tp_kernel_timer_select", "tp_comm_create_host", "tp_solve_residuals", "tp_shard_freq_order",
]

# tp_host_exchange_fn (tpgpu.h)
HOST_EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_void_p),
                               C.POINTER(C.c_size_t), C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_void_p),
                               C.POINTER(C.c_size_t))


class SolveError(RuntimeError):
    """Numerical failure with the achieved relative residual (solve.hpp:17-26)."""

    def __init__(self, msg, residual=-1.0):
        super().__init__(msg)
        self.residual = residual


def lib():
    """Load libtpgpu.so (raises if it has not been built -- no fallback)."""
    global _lib
    if _lib is None:
        # TPGPU_LIB: an in-tree experiment build (build.py --variant) instead
        path = os.path.join(_HERE, os.environ["TPGPU_LIB"]) if os.environ.get("TPGPU_LIB") else LIB_PATH
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `python -m paper_2502_21013_b200.build`")
        L = C.CDLL(path)
        dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int32)
        vp = C.c_void_p
        D, G = C.POINTER(TpProblemDesc), C.POINTER(TpSolverCfg)
        L.tp_version.restype = C.c_int
        L.tp_last_error.argtypes = [C.c_char_p, C.c_size_t, dp]
        L.tp_solver_cfg_default.argtypes = [G]
        L.tp_solver_cfg_default.restype = None
        L.tp_problem_desc_baseline.argtypes = [C.c_int32, D]
        L.tp_problem_create.argtypes = [D, C.c_int32, C.POINTER(vp)]
        L.tp_problem_destroy.argtypes = [vp]
        L.tp_problem_destroy.restype = None
        L.tp_problem_sizes.argtypes = [vp, ip, ip, dp]
        L.tp_problem_loads.argtypes = [vp, dp]
        L.tp_problem_mass.argtypes = [vp, dp]
        L.tp_apply_k.argtypes = [vp, dp, dp, C.c_int32]
        L.tp_residual.argtypes = [vp, dp, dp, dp]
        L.tp_static_init.argtypes = [vp, G, dp, ip]
        L.tp_set_state.argtypes = [vp, dp]
        L.tp_get_state.argtypes = [vp, dp]
        L.tp_choose_nu_hat.argtypes = [vp, G, dp, dp]
        L.tp_set_nu_hat.argtypes = [vp, dp, C.c_double]
        L.tp_periodic_solve.argtypes = [vp, G, dp, dp]
        L.tp_solve_m2.argtypes = [vp, G, dp, dp, C.POINTER(TpReport), dp, dp, C.c_int32]
        L.tp_solve_m3.argtypes = [vp, G, dp, dp, C.POINTER(TpReport), dp, dp, C.c_int32]
        L.tp_solve_m1.argtypes = [vp, G, dp, dp, C.POINTER(TpReport), dp, dp, C.c_int32,
                                  TP_ITERATE_CB, vp]
        L.tp_m1_begin.argtypes = [vp, G, dp]
        L.tp_m1_sweep.argtypes = [vp, dp, ip]
        L.tp_sweep_stats.argtypes = [vp, ip, C.POINTER(C.c_int64)]
        L.tp_solve_residuals.argtypes = [vp, dp, dp]
        L.tp_problem_stream.argtypes = [vp]
        L.tp_problem_stream.restype = vp
        L.tp_problem_launches.argtypes = [vp]
        L.tp_problem_launches.restype = C.c_int64
        SP = C.POINTER(TpShardPlan)
        L.tp_shard_plan_make.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32, SP]
        L.tp_shard_freq_order.argtypes = [C.c_int32, C.c_int32, C.c_int32, ip]
        L.tp_nccl_unique_id.argtypes = [C.c_char_p]
        L.tp_comm_create.argtypes = [C.c_char_p, C.c_int32, C.c_int32, C.c_int32, C.POINTER(vp)]
        L.tp_comm_create_host.argtypes = [C.c_int32, C.c_int32, C.c_int32, HOST_EXCHANGE_FN, vp, C.POINTER(vp)]
        L.tp_comm_destroy.argtypes = [vp]
        L.tp_comm_destroy.restype = None
        L.tp_comm_nccl.argtypes = [vp]
        L.tp_comm_nccl.restype = vp
        for f in ("tp_comm_rank", "tp_comm_size", "tp_comm_device"):
            getattr(L, f).argtypes = [vp]
            getattr(L, f).restype = C.c_int32
        L.tp_problem_create_sharded.argtypes = [D, vp, C.POINTER(vp)]
        L.tp_problem_shard.argtypes = [vp, SP]
        L.tp_kernel_timer.argtypes = [vp, C.c_int32, C.POINTER(C.c_int64), dp, dp]
        L.tp_kernel_timer_select.argtypes = [vp, C.c_int32]
        _lib = L
    return _lib


def _check(code):
    if code == TP_OK:
        return
    buf = C.create_string_buffer(2048)
    res = C.c_double()
    lib().tp_last_error(buf, 2048, C.byref(res))
    msg = buf.value.decode()
    if code == TP_EINVAL:
        raise ValueError(msg)
    if code == TP_ESOLVE:
        raise SolveError(msg, res.value)
    raise RuntimeError(msg)


def _dp(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_int32))


def baseline_desc(config: int) -> TpProblemDesc:
    d = TpProblemDesc()
    _check(lib().tp_problem_desc_baseline(config, C.byref(d)))
    return d


def stopping_check(history, tol) -> bool:
    """last <= tol * first, boundary inclusive (solvers.hpp:100-103)."""
    if len(history) == 0:
        raise ValueError("stopping check: empty history")
    return history[-1] <= tol * history[0]


def block_l2(R) -> float:
    return float(np.sqrt(np.sum(np.square(R))))


@dataclass
class SolveReport:
    """SolveReport (solvers.hpp:88-96) plus device counters."""
    method: str = "m1"
    iterations: int = 0
    residual_history: list = field(default_factory=list)
    contraction_history: list = field(default_factory=list)
    q_estimate: float = float("nan")
    wall_time: float = 0.0
    status: str = "converged"
    setup_time: float = 0.0
    sweep_time: float = 0.0
    inner_iterations: int = 0


def shard_plan(cells: int, steps: int, nranks: int, rank: int) -> TpShardPlan:
    """The partition every rank of a sharded problem uses (no GPU needed)."""
    p = TpShardPlan()
    _check(lib().tp_shard_plan_make(cells, steps, nranks, rank, C.byref(p)))
    return p


def shard_freq_order(cells: int, steps: int, nranks: int) -> np.ndarray:
    """Frequency held by every slot of the sharded half spectrum (snake order,
    DESIGN.md §6; the identity for one rank).  No GPU needed."""
    out = np.zeros(steps // 2 + 1, dtype=np.int32)
    _check(lib().tp_shard_freq_order(cells, steps, nranks, _ip(out)))
    return out


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().tp_nccl_unique_id(buf))
    return buf.raw


class Comm:
    """NCCL communicator of one rank (one process per GPU)."""

    def __init__(self, uid: bytes, nranks: int, rank: int, device: int):
        self._h = C.c_void_p()
        _check(lib().tp_comm_create(C.c_char_p(uid), nranks, rank, device, C.byref(self._h)))
        self.nranks, self.rank, self.device = nranks, rank, device

    @classmethod
    def from_torch(cls, device: int, group=None) -> "Comm":
        """Bootstrap over an initialised torch.distributed process group
        (gloo is enough: it only broadcasts the 128-byte NCCL id)."""
        import torch
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        uid = nccl_unique_id() if rank == 0 else bytes(128)
        t = torch.tensor(list(uid), dtype=torch.uint8)
        dist.broadcast(t, src=0, group=group)
        return cls(bytes(t.tolist()), world, rank, device)

    @classmethod
    def host_staged(cls, device: int, group=None) -> "Comm":
        """Host-staged transport over an initialised torch.distributed
        process group (gloo): every exchange of the sharded sweep goes
        through pinned host memory and point-to-point gloo messages
        (tp_comm_create_host).  For several ranks sharing one GPU (tests)."""
        import torch
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)

        def exchange(_user, ns, sp, sb, sz, nr, rp, rb, rz):
            try:
                reqs = []
                for i in range(ns):
                    a = np.ctypeslib.as_array(C.cast(sb[i], C.POINTER(C.c_uint8)), shape=(sz[i],))
                    reqs.append(dist.isend(torch.from_numpy(a.copy()), int(sp[i]), group=group))
                for i in range(nr):
                    a = np.ctypeslib.as_array(C.cast(rb[i], C.POINTER(C.c_uint8)), shape=(rz[i],))
                    reqs.append(dist.irecv(torch.from_numpy(a), int(rp[i]), group=group))
                for q in reqs:
                    q.wait()
                return 0
            except Exception:  # surfaces as TP_ECUDA "host transport callback failed"
                import traceback
                traceback.print_exc()
                return 1

        self = cls.__new__(cls)
        self._fn = HOST_EXCHANGE_FN(exchange)  # keep alive with the communicator
        self._h = C.c_void_p()
        _check(lib().tp_comm_create_host(world, rank, device, self._fn, None, C.byref(self._h)))
        self.nranks, self.rank, self.device = world, rank, device
        return self

    def close(self):
        if self._h:
            lib().tp_comm_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Problem:
    """One BASELINE-style grid problem resident on one CUDA device (or one
    rank's shard of it, see Problem.sharded)."""

    def __init__(self, desc: TpProblemDesc, device: int = 0, comm: "Comm | None" = None):
        self._h = C.c_void_p()
        self.desc = desc
        self.comm = comm
        if comm is None:
            _check(lib().tp_problem_create(C.byref(desc), device, C.byref(self._h)))
        else:
            _check(lib().tp_problem_create_sharded(C.byref(desc), comm._h, C.byref(self._h)))
        n, N, tau = C.c_int32(), C.c_int32(), C.c_double()
        _check(lib().tp_problem_sizes(self._h, C.byref(n), C.byref(N), C.byref(tau)))
        self.n_dof, self.steps, self.tau = n.value, N.value, tau.value

    @classmethod
    def baseline(cls, config: int, device: int = 0) -> "Problem":
        return cls(baseline_desc(config), device)

    @classmethod
    def sharded(cls, desc: TpProblemDesc, comm: Comm) -> "Problem":
        return cls(desc, comm.device, comm)

    def shard(self) -> TpShardPlan:
        p = TpShardPlan()
        _check(lib().tp_problem_shard(self._h, C.byref(p)))
        return p

    def close(self):
        if self._h:
            lib().tp_problem_destroy(self._h)
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

    # ---- setup products
    def loads(self) -> np.ndarray:
        F = np.zeros(self.shape)
        _check(lib().tp_problem_loads(self._h, _dp(F)))
        return F

    def mass(self) -> np.ndarray:
        m = np.zeros(self.n_dof)
        _check(lib().tp_problem_mass(self._h, _dp(m)))
        return m

    # ---- Problem concept
    def apply_k(self, U) -> np.ndarray:
        U = np.ascontiguousarray(U, dtype=np.float64)
        cnt = 1 if U.ndim == 1 else U.shape[0]
        if U.size != cnt * self.n_dof:
            raise ValueError("apply_k: size mismatch")
        out = np.zeros_like(U)
        _check(lib().tp_apply_k(self._h, _dp(U), _dp(out), cnt))
        return out

    def residual(self, U):
        U = self._state(U)
        R = np.zeros_like(U)
        nrm = C.c_double()
        _check(lib().tp_residual(self._h, _dp(U), _dp(R), C.byref(nrm)))
        return R, nrm.value

    # ---- methods
    def static_init(self, cfg: TpSolverCfg | None = None, want_state=True, out=None):
        """static_init (solvers.hpp:276-296).  out: caller buffer for U0
        (C-contiguous float64 of the state shape, e.g. pinned host memory)."""
        cfg = cfg or default_cfg()
        if out is not None:
            if out.shape != self.shape or out.dtype != np.float64 or not out.flags.c_contiguous:
                raise ValueError("out must be a C-contiguous float64 array of the state shape")
            U0 = out
        else:
            U0 = np.zeros(self.shape) if want_state else None
        counts = np.zeros(self.steps, dtype=np.int32)
        _check(lib().tp_static_init(self._h, C.byref(cfg), _dp(U0), _ip(counts)))
        return U0, counts

    def set_state(self, U):
        U = self._state(U)
        _check(lib().tp_set_state(self._h, _dp(U)))

    def get_state(self):
        U = np.zeros(self.shape)
        _check(lib().tp_get_state(self._h, _dp(U)))
        return U

    def choose_nu_hat(self, cfg: TpSolverCfg | None = None):
        cfg = cfg or default_cfg()
        nu = np.zeros(5)
        q = C.c_double()
        _check(lib().tp_choose_nu_hat(self._h, C.byref(cfg), _dp(nu), C.byref(q)))
        return nu, q.value

    def set_nu_hat(self, nu_hat, q=float("nan")):
        nu = np.ascontiguousarray(nu_hat, dtype=np.float64)
        if nu.shape != (5,):
            raise ValueError("nu_hat must have 5 entries")
        _check(lib().tp_set_nu_hat(self._h, _dp(nu), q))

    def periodic_solve(self, G, cfg: TpSolverCfg | None = None) -> np.ndarray:
        cfg = cfg or default_cfg()
        G = self._state(G)
        U = np.zeros_like(G)
        _check(lib().tp_periodic_solve(self._h, C.byref(cfg), _dp(G), _dp(U)))
        return U

    def solve_m1_fixed_point(self, U0=None, cfg: TpSolverCfg | None = None, iterate_log=None,
                             callback=None, out=None):
        """Returns (U, SolveReport).  iterate_log: list to receive every iterate
        (solvers.hpp:306); callback(k, U, residual) -> truthy aborts."""
        cfg = cfg or default_cfg()
        U0a = None if U0 is None else self._state(U0)
        cap = cfg.m1_max_outer + 1
        hist = np.zeros(cap)
        contr = np.zeros(cap)
        U = out if out is not None else np.zeros(self.shape)
        if U.shape != self.shape or U.dtype != np.float64 or not U.flags.c_contiguous:
            raise ValueError("out must be a C-contiguous float64 array of the state shape")
        rep = TpReport()

        want = iterate_log is not None or callback is not None

        def _cb(k, ptr, res, user):
            if iterate_log is not None:
                arr = np.ctypeslib.as_array(ptr, shape=(self.steps * self.n_dof,))
                iterate_log.append(arr.reshape(self.shape).copy())
            if callback is not None:
                arr = np.ctypeslib.as_array(ptr, shape=(self.steps * self.n_dof,))
                return 1 if callback(k, arr.reshape(self.shape), res) else 0
            return 0

        cb = TP_ITERATE_CB(_cb) if want else TP_ITERATE_CB()
        _check(lib().tp_solve_m1(self._h, C.byref(cfg), _dp(U0a), _dp(U), C.byref(rep), _dp(hist),
                                 _dp(contr), cap, cb, None))
        k = rep.history_len
        report = SolveReport(iterations=rep.iterations, residual_history=hist[:k].tolist(),
                             contraction_history=contr[:rep.contraction_len].tolist(),
                             q_estimate=rep.q_estimate, wall_time=rep.wall_time,
                             status=STATUS_NAMES[rep.status], setup_time=rep.setup_time,
                             sweep_time=rep.sweep_time, inner_iterations=rep.inner_iterations)
        return U, report

    def _solve_m23(self, fn, method, cap, U0, cfg, out):
        U0a = None if U0 is None else self._state(U0)
        hist = np.zeros(cap)
        contr = np.zeros(cap)
        U = out if out is not None else np.zeros(self.shape)
        rep = TpReport()
        _check(fn(self._h, C.byref(cfg), _dp(U0a), _dp(U), C.byref(rep), _dp(hist), _dp(contr), cap))
        k = rep.history_len
        report = SolveReport(method=method, iterations=rep.iterations, residual_history=hist[:k].tolist(),
                             contraction_history=contr[:rep.contraction_len].tolist(), q_estimate=rep.q_estimate,
                             wall_time=rep.wall_time, status=STATUS_NAMES[rep.status],
                             inner_iterations=rep.inner_iterations)
        return U, report

    def solve_m2_newton(self, U0=None, cfg: TpSolverCfg | None = None, out=None):
        """M2 all-at-once Newton (solve_m2_newton, solvers.hpp:375-484):
        FGMRES right-preconditioned by the periodic solver on the time-averaged
        Jacobian, Armijo line search.  Returns (U, SolveReport(method="m2"))."""
        cfg = cfg or default_cfg()
        return self._solve_m23(lib().tp_solve_m2, "m2", cfg.m2_max_outer + 1, U0, cfg, out)

    def solve_m3_timestepping(self, U0=None, cfg: TpSolverCfg | None = None, out=None):
        """M3 sequential time stepping toward the limit cycle
        (solve_m3_timestepping, solvers.hpp:489-542).  Returns
        (U, SolveReport(method="m3")); iterations = completed periods."""
        cfg = cfg or default_cfg()
        return self._solve_m23(lib().tp_solve_m3, "m3", cfg.m3_max_cycles + 1, U0, cfg, out)

    # ---- device-resident sweeps
    def m1_begin(self, cfg: TpSolverCfg | None = None) -> float:
        cfg = cfg or default_cfg()
        r0 = C.c_double()
        _check(lib().tp_m1_begin(self._h, C.byref(cfg), C.byref(r0)))
        return r0.value

    def m1_sweep(self):
        r = C.c_double()
        it = C.c_int32()
        _check(lib().tp_m1_sweep(self._h, C.byref(r), C.byref(it)))
        return r.value, it.value

    def sweep_stats(self):
        """(largest per-frequency iteration count, sum over frequency blocks of
        their iteration counts) of the last periodic solve."""
        mx, tot = C.c_int32(), C.c_int64()
        _check(lib().tp_sweep_stats(self._h, C.byref(mx), C.byref(tot)))
        return mx.value, tot.value

    def solve_residuals(self):
        """(largest ||r_k|| / max(||g_k||, ||g||/sqrt(K)), largest ||r_k|| / ||g_k||)
        over the frequency blocks of the last periodic solve (tp_solve_residuals)."""
        a, b = C.c_double(), C.c_double()
        _check(lib().tp_solve_residuals(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def kernel_timer_select(self, which: int):
        """0: fine up pass, 1: fine down pass, 2: fine apply (tp_kernel_timer_select)."""
        _check(lib().tp_kernel_timer_select(self._h, which))

    def kernel_timer(self, enable: bool):
        """(launches, ms, algorithmic bytes) of the dominant kernel since the
        last call; then enable/disable the CUDA-event timer."""
        n, ms, b = C.c_int64(), C.c_double(), C.c_double()
        _check(lib().tp_kernel_timer(self._h, 1 if enable else 0, C.byref(n), C.byref(ms), C.byref(b)))
        return n.value, ms.value, b.value

    @property
    def stream(self) -> int:
        return lib().tp_problem_stream(self._h) or 0

    @property
    def launches(self) -> int:
        return int(lib().tp_problem_launches(self._h))
