"""ctypes mirror of the C ABI data types in include/tpgpu.h.

Plain data only (structs, enums, status codes); no library is loaded here.
"""
from __future__ import annotations

import ctypes as C

TP_OK, TP_EINVAL, TP_ESOLVE, TP_ECUDA = 0, 1, 2, 3
TP_CONVERGED, TP_MAX_ITER, TP_STALLED = 0, 1, 2
TP_NU_HAT_THEORY, TP_NU_HAT_FROZEN_FIELD = 0, 1
TP_MAX_MATERIALS, TP_MAX_RECTS, TP_MAX_HARMONICS = 5, 8, 4

STATUS_NAMES = {TP_CONVERGED: "converged", TP_MAX_ITER: "max_iter", TP_STALLED: "stalled"}


class TpRect(C.Structure):
    _fields_ = [("x0", C.c_double), ("y0", C.c_double), ("x1", C.c_double), ("y1", C.c_double),
                ("material", C.c_int32), ("pad_", C.c_int32)]


class TpMaterial(C.Structure):
    _fields_ = [("sigma", C.c_double), ("sigma_noise", C.c_int32), ("n_harmonics", C.c_int32),
                ("nu0", C.c_double), ("nu_inf", C.c_double), ("bs", C.c_double),
                ("amp", C.c_double * TP_MAX_HARMONICS), ("phase", C.c_double * TP_MAX_HARMONICS),
                ("harmonic", C.c_int32 * TP_MAX_HARMONICS)]


class TpProblemDesc(C.Structure):
    _fields_ = [("cells", C.c_int32), ("steps", C.c_int32), ("period", C.c_double),
                ("n_rects", C.c_int32), ("n_materials", C.c_int32),
                ("rect", TpRect * TP_MAX_RECTS), ("material", TpMaterial * TP_MAX_MATERIALS),
                ("noise_seed", C.c_uint64), ("noise_lattice", C.c_int32),
                ("flux_samples", C.c_int32), ("noise_lo", C.c_double), ("noise_hi", C.c_double),
                ("noise_box", C.c_double * 4), ("s_max", C.c_double)]


class TpSolverCfg(C.Structure):
    _fields_ = [("tol", C.c_double), ("m1_max_outer", C.c_int32),
                ("armijo_max_halvings", C.c_int32), ("armijo_slope", C.c_double),
                ("armijo_backtrack", C.c_double), ("nu_hat_mode", C.c_int32),
                ("nu_hat_samples", C.c_int32), ("imag_tol", C.c_double),
                ("static_tol", C.c_double), ("static_max_newton", C.c_int32),
                ("threads", C.c_int32), ("inner_rtol", C.c_double),
                ("inner_max_iter", C.c_int32), ("warm_start", C.c_int32),
                ("freq_chunk", C.c_int32), ("slice_chunk", C.c_int32),
                ("freq_groups", C.c_int32), ("m2_max_outer", C.c_int32),
                ("m2_inner_tol", C.c_double), ("m2_inner_max", C.c_int32), ("m2_restart", C.c_int32),
                ("m3_max_cycles", C.c_int32), ("track_error_contraction", C.c_int32)]


class TpShardPlan(C.Structure):
    _fields_ = [("nranks", C.c_int32), ("rank", C.c_int32), ("row0", C.c_int32), ("row1", C.c_int32),
                ("freq0", C.c_int32), ("freq1", C.c_int32), ("slice0", C.c_int32),
                ("slice1", C.c_int32), ("n_local", C.c_int32)]


class TpReport(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("status", C.c_int32), ("history_len", C.c_int32),
                ("inner_iterations", C.c_int32), ("q_estimate", C.c_double),
                ("wall_time", C.c_double), ("setup_time", C.c_double),
                ("sweep_time", C.c_double), ("contraction_len", C.c_int32), ("pad_", C.c_int32)]


TP_ITERATE_CB = C.CFUNCTYPE(C.c_int, C.c_int32, C.POINTER(C.c_double), C.c_double, C.c_void_p)


def default_cfg(**overrides) -> TpSolverCfg:
    """SolverConfig defaults (solvers.hpp:49-69) + device inner-solver defaults."""
    c = TpSolverCfg()
    c.tol = 1e-4
    c.m1_max_outer = 200
    c.armijo_max_halvings = 30
    c.armijo_slope = 1e-4
    c.armijo_backtrack = 0.5
    c.nu_hat_mode = TP_NU_HAT_FROZEN_FIELD
    c.nu_hat_samples = 2000
    c.imag_tol = 1e-9
    c.static_tol = 1e-8
    c.static_max_newton = 50
    c.threads = 0
    c.inner_rtol = 1e-12
    c.inner_max_iter = 200
    c.warm_start = 1
    c.freq_chunk = 0
    c.slice_chunk = 0
    c.freq_groups = 0
    c.m2_max_outer = 50
    c.m2_inner_tol = 1e-8
    c.m2_inner_max = 300
    c.m2_restart = 60
    c.m3_max_cycles = 10
    c.track_error_contraction = 0
    for k, v in overrides.items():
        setattr(c, k, v)
    return c
