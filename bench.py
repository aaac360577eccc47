#!/usr/bin/env python3
"""Benchmark: space-time DoF/s per fixed-point sweep (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config 3] [--no-cpu-baseline] [--no-cfg1-leg] [--no-mesh]

One step = one fixed-point sweep over all N time slices of the workload
(solvers.hpp:326-342: RHS f + K_hat u - K(u), DFT along time, the N/2+1
frequency-block solves, inverse DFT, residual + norm).  Default workload:
BASELINE.json configs[3], the largest configuration that fits one GPU
(2048x2048 cells, 4,190,209 dofs, N = 1024: 4.29e9 space-time DoF, fp64,
~169 GB of HBM in use).

Timing: W untimed warm-up sweeps, then exactly K sweeps bracketed by a
barrier + cudaDeviceSynchronize and CUDA events on the library's stream,
max over ranks.  Every sweep streams U, G, Ghat, Uhat (34 GB each, >> L2).
`e2e` goes through the C ABI with pinned HOST buffers: each step uploads U,
runs one sweep (tp_solve_m1 with m1_max_outer = 1) and downloads U.
`full_solve` is the time-to-residual leg: static_init + nu_hat + solver
setup + sweeps until the residual reaches 1e-8 of the first, or stops
improving (the fp64 floor of the fixed point on configs 2 / 3),
with the time to every decade reached.  `cfg1_leg` repeats the sweep and
the full solve on configs[1] (the configuration the CPU reference can solve
to 1e-8), beside one reference sweep on the host.

Multi-GPU (torchrun, one process per GPU): the workload is SHARDED across
the ranks (strong scaling): node-row strips for K(u) /
residual / RHS / DFTs, frequency blocks for the solves, NCCL all-to-alls
between them, halo rows and rank-ordered scalar sums.  torch.distributed
(gloo) only bootstraps the NCCL communicator; `--replicas` runs independent
copies instead (weak scaling).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "space-time DoF/s per fixed-point sweep"
UNIT = "DoF/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if len(r) > 5 + k and r[5 + k].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo", rank=rank, world_size=world)
        pg = dist
    return world, rank, local, pg


def allreduce_max(pg, x: float) -> float:
    if pg is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64)
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


def barrier(pg):
    if pg is not None:
        pg.barrier()


def cudart():
    import torch  # noqa: F401  (loads the CUDA runtime for event timing)
    return torch


WORKLOAD_NAMES = {
    0: "BASELINE configs[0]: small 2D model problem",
    1: "BASELINE configs[1]: unit square, seeded sigma noise",
    2: "BASELINE configs[2]: transformer-like cross-section",
    3: "BASELINE configs[3]: scaling config (configs[2] geometry)",
    4: "BASELINE configs[4]: harmonic-rich strongly saturating",
    5: "BASELINE configs[4] linear control (nu == nu0)",
}


def workload_config(desc, config, world, replicas=False):
    n = (desc.cells - 1) ** 2
    D = n * desc.steps
    par = "single GPU" if world == 1 else (f"replicas x{world}" if replicas else
                                           f"sharded x{world}: row strips + frequency blocks, NCCL all-to-all")
    vec = 8.0 * D
    return D, {
        "workload": f"{WORKLOAD_NAMES.get(config, f'config {config}')}: {desc.cells}x{desc.cells} cells "
                    f"({n} dofs) x N={desc.steps} slices, fp64, U0 = static_init, frozen-field nu_hat",
        "baseline_config": config, "cells": desc.cells, "steps": desc.steps, "space_time_dof": D,
        "l2": f"inputs larger than L2 (U, G, Ghat, Uhat {vec / 1e9:.3g} GB each, streamed every sweep)",
        "parallelism": par,
    }


def warm_modules(device):
    """Pay CUDA module loading / first-launch costs on a tiny problem so the
    init timing of the workload is a warm process's (one untimed call)."""
    from paper_2502_21013_b200 import Problem, baseline_desc, default_cfg
    cfg = default_cfg(tol=1e-8, m1_max_outer=2)
    with Problem(baseline_desc(0), device=device) as w:
        w.static_init(cfg, want_state=False)
        w.choose_nu_hat(cfg)
        w.m1_begin(cfg)
        w.m1_sweep()


_PINNED = []


def pinned(shape, torch):
    """A page-locked host array of exactly `shape` (cudaHostRegister on a
    numpy buffer: torch's pinned allocator rounds a 34 GB request up to the
    next power of two)."""
    a = np.empty(shape, dtype=np.float64)
    a.fill(0.0)  # fault the pages in before locking them
    err = torch.cuda.cudart().cudaHostRegister(a.ctypes.data, a.nbytes, 0)
    if int(err) != 0:
        raise RuntimeError(f"cudaHostRegister failed ({err})")
    _PINNED.append(a)
    return a


def unpin(a, torch):
    for i, b in enumerate(_PINNED):
        if b is a:
            torch.cuda.cudart().cudaHostUnregister(a.ctypes.data)
            del _PINNED[i]
            return


def full_solve_leg(p, U0, cfg, init_s, D, jobs, pg, torch, stream, stall_window=20):
    """Time to residual: sweeps from U0 until history[-1] <= tol * history[0]
    (stopping_check, solvers.hpp:100-103), m1_max_outer, or no 5 % gain on
    the best residual for `stall_window` sweeps (the fp64 floor of the fixed
    point on configs 2 / 3: rounding of G = f + K_hat u - K(u) amplified by
    1 / (1 - q), q ~ 0.97 -- DESIGN.md §8).  Reports the time to every decade."""
    p.set_state(U0)
    t0 = time.perf_counter()
    r0 = p.m1_begin(cfg)
    t_setup = time.perf_counter() - t0
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(cfg.m1_max_outer + 1)]
    ev[0].record(stream)
    hist, its, fits = [r0], [], []
    best, since = r0, 0
    while len(its) < cfg.m1_max_outer and not hist[-1] <= cfg.tol * hist[0]:
        r, it = p.m1_sweep()
        hist.append(r)
        its.append(it)
        fits.append(p.sweep_stats()[1])
        ev[len(its)].record(stream)
        if r < 0.95 * best:
            best, since = r, 0
        else:
            since += 1
            if since >= stall_window:
                break
    torch.cuda.synchronize()
    sw = [ev[k].elapsed_time(ev[k + 1]) for k in range(len(its))]
    cum = np.cumsum(sw) / 1e3
    conv = bool(hist[-1] <= cfg.tol * hist[0])
    decades = {}
    for e in range(1, 9):
        k = next((i for i, x in enumerate(hist) if x <= 10.0 ** -e * hist[0]), None)
        if k is not None:
            decades[f"1e-{e}"] = {"sweeps": k, "time_to_residual_s": init_s + t_setup + (cum[k - 1] if k else 0.0)}
    best_ratio = min(hist) / hist[0]
    return {"tol": cfg.tol, "sweeps": len(its), "converged": conv,
            "stopped": "converged" if conv else ("max_iter" if len(its) >= cfg.m1_max_outer else "stalled"),
            "time_to_residual_s": init_s + t_setup + float(cum[-1]) if conv else None,
            "best_residual_ratio": best_ratio, "decades": decades,
            "init_s": init_s, "setup_s": t_setup, "sweeps_s": float(cum[-1]) if len(cum) else 0.0,
            "median_sweep_ms": float(np.median(sw)) if sw else None,
            "median_dof_per_s": D * jobs / (allreduce_max(pg, float(np.median(sw))) / 1e3) if sw else None,
            "inner_iterations_median": float(np.median(its)) if its else 0.0,
            "inner_iterations_max": int(max(its)) if its else 0,
            "frequency_iterations_mean": float(np.mean(fits)) if fits else 0.0,
            "history_first_last": [hist[0], hist[-1]]}


# ----------------------------------------------------------------- b200 arm
def run_b200(args):
    world, rank, local, pg = dist_setup()
    torch = cudart()
    torch.cuda.set_device(local)
    from paper_2502_21013_b200 import Problem, baseline_desc, default_cfg

    desc = baseline_desc(args.config)
    D, config = workload_config(desc, args.config, world, args.replicas)
    cfg = default_cfg(tol=1e-8)
    sharded = world > 1 and not args.replicas
    comm = None
    warm_modules(local)
    if sharded:
        from paper_2502_21013_b200 import Comm
        comm = Comm.from_torch(local)
        p = Problem.sharded(desc, comm)
    else:
        p = Problem(desc, device=local)
    Uh = pinned(p.shape, torch)  # U0, pinned: the e2e leg uploads it every step
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, counts = p.static_init(cfg, out=Uh)
    nu, q = p.choose_nu_hat(cfg)
    init_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    r0 = p.m1_begin(cfg)
    setup_s = time.perf_counter() - t0
    history = [r0]
    clk = ClockSampler(local).__enter__()  # sampled from the warm-up on, through the timed region
    for _ in range(args.warmup):
        history.append(p.m1_sweep()[0])
    stream = torch.cuda.ExternalStream(p.stream, device=local)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    inner = []
    launches0 = p.launches
    p.kernel_timer_select(DOMINANT[0])
    p.kernel_timer(True)  # CUDA events around the dominant kernel, over the timed region
    barrier(pg)
    torch.cuda.synchronize()
    evs[0].record(stream)
    fiters = []
    for k in range(args.steps):
        r, it = p.m1_sweep()
        history.append(r)
        inner.append(it)
        fiters.append(p.sweep_stats()[1])
        evs[k + 1].record(stream)
    torch.cuda.synchronize()
    clk.__exit__(None, None, None)
    barrier(pg)
    launches = p.launches - launches0
    k_launches, k_ms, k_bytes = p.kernel_timer(False)
    per = [evs[k].elapsed_time(evs[k + 1]) for k in range(args.steps)]
    total_ms = evs[0].elapsed_time(evs[-1])
    total_ms = allreduce_max(pg, total_ms)
    jobs = 1 if sharded else world  # sharded: one job over all GPUs; replicas: world jobs
    value = D * args.steps * jobs / (total_ms / 1e3)

    # Isolated calibration of the dominant kernel: the timed region runs the
    # frequency solves as concurrent groups (their kernels overlap, so a
    # launch's event-to-event time includes other groups' kernels).  More
    # sweeps with the groups serialized (freq_groups=1) time the kernel alone,
    # same events, same stream discipline.
    iso = None
    if args.calib_sweeps > 0:
        c_iso = default_cfg(tol=cfg.tol)
        c_iso.freq_groups = 1
        p.m1_begin(c_iso)
        p.m1_sweep()  # warm the rebuilt solver
        torch.cuda.synchronize()
        p.kernel_timer(True)
        for _ in range(args.calib_sweeps):
            p.m1_sweep()
        torch.cuda.synchronize()
        iso = p.kernel_timer(False)

    # Time to residual from the same U0 (setup excluded from the sweeps).
    full = full_solve_leg(p, Uh, cfg, init_s, D, jobs, pg, torch, stream) if args.full_solve else None

    # e2e through the C ABI with pinned host buffers (one sweep per call)
    e2e = None
    if args.e2e_steps > 0:
        Uo = pinned(p.shape, torch)
        c1 = default_cfg(tol=1e-12, m1_max_outer=1)
        p.solve_m1_fixed_point(Uh, c1, out=Uo)  # warm (hierarchy cached)
        times = []
        for _ in range(args.e2e_steps):
            barrier(pg)
            t = time.perf_counter()
            p.solve_m1_fixed_point(Uh, c1, out=Uo)
            times.append(time.perf_counter() - t)
        e2e_s = allreduce_max(pg, float(np.median(times)))
        e2e = {"value": D * jobs / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(Uh.nbytes),
               "d2h_bytes_per_step": int(Uo.nbytes), "step_s": e2e_s,
               "note": "tp_solve_m1 per step (m1_max_outer = 1): H2D of U0 from pinned host memory, initial "
                       "residual, one sweep warm-started from the spectrum of U0, D2H of U"}
        unpin(Uo, torch)
        del Uo

    hbm, src = peaks()
    n = (desc.cells - 1) ** 2
    roofline = dominant_kernel_roofline(args, k_launches, k_ms, k_bytes, iso, hbm, src, n)
    # Whole-sweep algorithmic bytes per GPU:
    # B = 72 D / P + 16 n (3 K / P + S sum_k it_k) over this rank's frequency
    # blocks (sum_k it_k counted exactly by the solver, tp_sweep_stats), with S
    # the complex streams per inner iteration and frequency as implemented
    # (streams_per_iteration: 15.0 at cfg 1, 15.46 at cfg 3) and 3 streams for
    # every block's initial residual.
    STREAMS = streams_per_iteration(desc.cells - 1)
    mean_inner = float(np.mean(inner)) if inner else 0.0
    mean_fit = float(np.mean(fiters)) if fiters else 0.0
    K = desc.steps // 2 + 1
    # + the initial residual of every block (r = g - A x0: read g, x0, write r)
    b_alg = 72.0 * D / (world if sharded else 1) + 16.0 * n * (3.0 * K / (world if sharded else 1)
                                                              + STREAMS * mean_fit)
    t_sweep = total_ms / 1e3 / args.steps
    sweep_roofline = {"bound": "hbm", "achieved": b_alg / t_sweep / 1e9, "peak": hbm, "unit": "GB/s",
                      "frac": b_alg / t_sweep / 1e9 / hbm, "bytes_per_sweep": b_alg,
                      "fixed_bytes_per_sweep": 72.0 * D, "streams_per_inner_iteration": STREAMS,
                      "inner_iterations_mean": mean_inner, "frequency_iterations_per_sweep": mean_fit}
    sweep_roofline.update(sweep_dram_crosscheck(args.config, b_alg, t_sweep, hbm))

    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
           "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f64",
           "data": f"synthetic (BASELINE.json configs[{args.config}] physics, seeded inputs)",
           "config": config, "impl": "b200", "clocks": clk.summary(),
           "e2e": e2e, "gpu_launches": launches, "roofline": roofline, "sweep_roofline": sweep_roofline,
           "sweep_ms": {"median": float(np.median(per)), "min": float(np.min(per)),
                        "max": float(np.max(per))},
           "inner_iterations": inner, "frequency_iterations": fiters, "newton_max": int(counts.max()),
           "init_s": init_s, "setup_s": setup_s, "full_solve": full,
           "residual_last": history[-1], "residual_first": history[0]}
    p.close()
    unpin(Uh, torch)
    del Uh
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(desc, nu, args.config)
    if rank == 0 and world == 1 and args.cfg1_leg and args.config != 1:
        out["cfg1_leg"] = cfg1_leg(args, torch)
    if rank == 0 and world == 1 and args.mesh:
        out["reference_mesh"] = mesh_leg(args)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if comm is not None:
        comm.close()


# The dominant kernel at the bench configs: the fine-level down pass
# (k_stream_down<Five>, fused with the Krylov update): 25 % of a cfg-3 sweep and
# 24 % of a cfg-1 sweep in the ncu launch lists (profiles/r2*_launches_cfg3_sweep.txt,
# r2c_launches_cfg1_sweep.txt; at cfg 1 the fused small-level cycle is level with
# it, and it has no HBM roofline: it keeps its levels in shared memory).
DOMINANT = (1, "k_stream_down<Five> (fine-level V-cycle down pass, fused Krylov update)")


def dominant_kernel_roofline(args, k_launches, k_ms, k_bytes, iso, hbm, src, n):
    """The kernel the library brackets with CUDA events (tp_kernel_timer,
    tp_kernel_timer_select): algorithmic bytes per launch = 4.25 complex values
    (read r, q; write r, z2 and the 1/4-size coarse right-hand side) x 16 B per
    fine node per active frequency (2.25 on the plain first pass), over its
    event-measured launch time."""
    def kstats(nl, ms, by):
        avg_ms = ms / max(nl, 1)
        b_launch = by / max(nl, 1)
        ach = b_launch / (avg_ms / 1e3) / 1e9 if nl else None
        return {"achieved": ach, "frac": (ach / hbm) if ach else None, "bytes_per_launch": b_launch,
                "avg_launch_ms": avg_ms, "launches": nl}

    timed = kstats(k_launches, k_ms, k_bytes)
    roofline = {"bound": "hbm", "kernel": DOMINANT[1], "peak": hbm,
                "unit": "GB/s", "traffic": None, "peak_source": src}
    if iso is not None and iso[0]:
        roofline.update(kstats(*iso))
        roofline["measured"] = ("live in bench.py: CUDA events around every launch on its stream, over "
                                f"{args.calib_sweeps} sweeps run right after the timed region with the frequency "
                                "groups serialized (freq_groups=1), so launches do not overlap other kernels")
        roofline["in_timed_region"] = dict(timed, note="concurrent frequency groups: a launch's event span "
                                           "includes the other groups' kernels")
    else:
        roofline.update(timed)
    # ncu DRAM bytes of this kernel per algorithmic byte, from the committed
    # launch list of the same config (profiles/kernel_traffic.json)
    try:
        with open(os.path.join(ROOT, "profiles", "kernel_traffic.json")) as f:
            kt = json.load(f).get(f"cfg{args.config}", {})
        ratio = kt.get("dominant_kernel_dram_over_algorithmic")
        if ratio and roofline.get("bytes_per_launch"):
            roofline["traffic"] = ratio * roofline["bytes_per_launch"]
            roofline["traffic_note"] = ("ncu dram__bytes_read+write per launch: the kernel's DRAM / algorithmic byte "
                                        "ratio from the committed launch list of this config "
                                        f"({kt.get('source')}) times this launch's algorithmic bytes")
    except Exception:
        pass
    return roofline


def streams_per_iteration(m):
    """Complex fine-level streams per inner COCG iteration and frequency, for
    the level sizes of this grid (m interior nodes per side): fine apply 6 +
    fused down 4.25 + up 3.25; every streamed Galerkin level (m_l > 63) 5.5
    of its own size; the fused small-level cycle reads b and writes z at its
    first level."""
    S = 13.5
    ml = (m - 1) // 2
    while ml > 63:
        S += 5.5 * (ml * ml) / (m * m)
        ml = (ml - 1) // 2
    S += 2.0 * (ml * ml) / (m * m)
    return S


def sweep_dram_crosscheck(config, b_alg, t_sweep, hbm):
    """SURVEY.md §8(d) cross-check: ncu DRAM bytes of one production sweep of
    this config over its algorithmic bytes (profiles/kernel_traffic.json, from
    the committed launch list and the solver's own counts of that sweep),
    applied to this run's algorithmic bytes; the roofline fraction on the
    smaller of the two."""
    try:
        with open(os.path.join(ROOT, "profiles", "kernel_traffic.json")) as f:
            kt = json.load(f).get(f"cfg{config}")
        if not kt or not kt.get("sweep_dram_over_algorithmic"):
            return {}
        dram = kt["sweep_dram_over_algorithmic"] * b_alg
        return {"dram_bytes_per_sweep": dram, "dram_source": kt.get("source"),
                "dram_over_algorithmic": kt["sweep_dram_over_algorithmic"],
                "frac_on_smaller": min(dram, b_alg) / t_sweep / 1e9 / hbm}
    except Exception:
        return {}


def cfg1_leg(args, torch):
    """configs[1] (256^2 cells, N = 256): the configuration the CPU reference
    solves to 1e-8 (tests/golden/cfg1_full_reference.npz: 8 host threads),
    device sweeps + time to 1e-8 here, one reference sweep on the host."""
    from paper_2502_21013_b200 import Problem, baseline_desc, default_cfg
    desc = baseline_desc(1)
    D = (desc.cells - 1) ** 2 * desc.steps
    cfg = default_cfg(tol=1e-8)
    with Problem(desc) as p:
        t0 = time.perf_counter()
        U0, _ = p.static_init(cfg)
        nu, q = p.choose_nu_hat(cfg)
        init_s = time.perf_counter() - t0
        p.m1_begin(cfg)
        for _ in range(3):
            p.m1_sweep()
        stream = torch.cuda.ExternalStream(p.stream, device=torch.cuda.current_device())
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        K = 20
        torch.cuda.synchronize()
        ev[0].record(stream)
        for _ in range(K):
            p.m1_sweep()
        ev[1].record(stream)
        ev[1].synchronize()
        sweep_ms = ev[0].elapsed_time(ev[1]) / K
        full = full_solve_leg(p, U0, cfg, init_s, D, 1, None, torch, stream)
    leg = {"workload": f"BASELINE configs[1]: {desc.cells}x{desc.cells} cells x N={desc.steps}",
           "sweep_ms": sweep_ms, "dof_per_s": D / (sweep_ms / 1e3), "full_solve": full}
    try:
        g = np.load(os.path.join(ROOT, "tests", "golden", "cfg1_full_reference.npz"))
        leg["reference_full_solve"] = {"sweeps": int(g["iterations"]), "m1_wall_s": float(g["m1_wall_s"]),
                                       "init_s": float(g["init_s"]), "threads": int(g["threads"]),
                                       "where": "the fixture run (tests/golden/make_golden_large.py cfg1), "
                                                "not this box"}
    except Exception:
        pass
    if not args.no_cpu_baseline:
        leg["cpu_baseline"] = cpu_baseline(desc, nu, 1, U0=U0, q=q)
    return leg


def mesh_leg(args):
    """General-mesh path on the reference's own config
    configs/transformer_saturated.json (40x40 snapped transformer mesh, 2142
    dofs, N=64, windings +-9.5e5 A/m^2) at tol 1e-8: device sweeps timed with
    CUDA events on the problem's stream; M1 to 1e-8 through the C ABI (host
    U0 in, U out) beside the reference's solve_m1_fixed_point on the same U0
    (oracle/_ref, all host threads)."""
    from paper_2502_21013_b200.mesh import MeshProblem
    from paper_2502_21013_b200 import default_cfg
    cfg = default_cfg(tol=1e-8)
    with MeshProblem.transformer(j_amp=9.5e5) as mp:
        U0, _ = mp.static_init(cfg)
        mp.choose_nu_hat(cfg)
        _, rep = mp.solve_m1_fixed_point(U0, cfg)          # warm
        t0 = time.perf_counter()
        U, rep = mp.solve_m1_fixed_point(U0, cfg)
        t_solve = time.perf_counter() - t0
        mp.set_state(U0)
        mp.m1_begin(cfg)
        for _ in range(3):
            mp.m1_sweep()
        import torch
        stream = torch.cuda.ExternalStream(mp.stream, device=0)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        K = 20
        torch.cuda.synchronize()
        ev[0].record(stream)
        for _ in range(K):
            mp.m1_sweep()
        ev[1].record(stream)
        ev[1].synchronize()
        sweep_ms = ev[0].elapsed_time(ev[1]) / K
        D = mp.n_dof * mp.steps
        leg = {"workload": "reference configs/transformer_saturated.json: 40x40 snapped transformer mesh "
                           f"({mp.n_dof} dofs, band {mp.bandwidth}) x N={mp.steps}, tol 1e-8",
               "sweep_ms": sweep_ms, "dof_per_s": D / (sweep_ms / 1e3), "m1_sweeps": rep.iterations,
               "m1_wall_s": t_solve}
    try:
        from oracle import ref
        if ref.available():
            c = ref.tr_cfg(j_amp=9.5e5)
            r = ref.tr_solve_m1(c, *ref.tr_choose_nu_hat(c, U0, cfg), U0, cfg)
            leg["reference_m1_wall_s"] = r.wall_time
            leg["reference_m1_sweeps"] = r.iterations
            leg["reference_threads"] = ref.hardware_threads()
    except Exception as e:  # the checker is optional on the box
        leg["reference_error"] = str(e)
    return leg


def stage_block_measurement(config):
    """Committed measurement of the reference's frequency-block stage on the
    GPU box's host (profiles/r2_ref_blocks.json, tools/ref_blocks.py): T
    concurrent complex blocks (lambda_k M + K_hat assembled, factorised,
    solved, residual-checked) on T threads take `round_wall_s`."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2_ref_blocks.json")) as f:
            return json.load(f).get(f"cfg{config}")
    except Exception:
        return None


def sampled_reference_sweep(desc, nu, config, cores, reps):
    """The reference sweep at sizes where one takes hours (configs >= 2,
    cache = never: every sweep factorises all N/2+1 blocks), stage by stage
    on a bounded sample (tpref_sweep_sample, the reference's own code per
    stage, cores threads): A / E on `cores` slices scaled by N / cores, B / D
    on 2048 * cores columns scaled by n / columns, C = ceil((N/2+1) / T)
    rounds of T concurrent block solves from the committed box measurement.
    Returns (per-rep sweep seconds, stages of the last rep, note)."""
    from oracle import ref
    N = desc.steps
    n = (desc.cells - 1) ** 2
    S = cores
    Cc = min(n, 2048 * cores)
    samples, setup = ref.sweep_sample(desc, nu, S, Cc, 0, threads=cores, reps=reps)
    blk = stage_block_measurement(config)
    K = N // 2 + 1
    t_c = None
    if blk:
        T = int(blk["concurrent_blocks"])
        t_c = -(-K // T) * float(blk["round_wall_s"])
    sweeps, stages = [], None
    for smp in samples:
        st = {"A_rhs": smp["A_rhs"] * N / S, "B_forward_dft": smp["B_forward_dft"] * n / Cc,
              "D_inverse_dft": smp["D_inverse_dft"] * n / Cc, "E_residual": smp["E_residual"] * N / S,
              "C_blocks": t_c}
        sweeps.append(sum(v for v in st.values() if v is not None))
        stages = st
    note = (f"stages A (RHS) and E (residual) timed live on {S} slices and scaled by N/{S}; B / D (time DFTs) "
            f"on {Cc} dof columns scaled by n/{Cc}; " +
            (f"C (the {K} frequency-block factorisations + solves, one per worker thread) = ceil({K}/"
             f"{blk['concurrent_blocks']}) rounds x {float(blk['round_wall_s']):.1f} s, the wall time of "
             f"{blk.get('concurrent_blocks_measured', blk['concurrent_blocks'])} concurrent blocks measured once on "
             f"the GPU box's host (tools/ref_blocks.py -> profiles/r2_ref_blocks.json; a full-host round is taken "
             f"to cost the same, which favours the reference)" if blk else
             "C (frequency blocks) NOT included: value is an upper bound on the reference's DoF/s"))
    return sweeps, stages, note, setup


def cpu_baseline(desc, nu, config, U0=None, q=None):
    """The reference's own sweep (oracle/_ref/libtpref.so) on the host cores:
    one full sweep where that takes seconds (configs 0 / 1, from the device's
    U0), a stage-by-stage sample otherwise (sampled_reference_sweep)."""
    from oracle import ref
    from paper_2502_21013_b200.abi import default_cfg
    if not ref.available():
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                "sample": "oracle/_ref/libtpref.so not built"}
    cores = ref.hardware_threads()
    D = (desc.cells - 1) ** 2 * desc.steps
    if U0 is not None:
        cfg = default_cfg(tol=1e-12, m1_max_outer=1, threads=cores)
        r = ref.solve_m1(desc, nu, q, U0, cfg, cache=0)
        sweep_s = max(r.wall_time - r.setup_time, 1e-9)
        samples, _ = ref.sweep_sample(desc, nu, cores, min(2048 * cores, (desc.cells - 1) ** 2), 0,
                                      threads=cores, reps=1)
        return {"value": D / sweep_s, "unit": UNIT, "cores": cores, "kind": "reference",
                "sample": f"one full sweep of the same workload (tpfem solve_m1_fixed_point, m1_max_outer=1, "
                          f"cache=automatic, {cores} threads, shim sparse LDL^T) from the device's U0; "
                          f"{sweep_s:.2f} s per sweep",
                "stage_sample_s": samples[0], "setup_and_initial_residual_s": r.setup_time}
    sweeps, stages, note, setup = sampled_reference_sweep(desc, nu, config, cores, reps=1)
    return {"value": D / sweeps[0], "unit": UNIT, "cores": cores, "kind": "reference",
            "sample": "one reference sweep estimated stage by stage: " + note, "stages_s": stages,
            "sweep_s": sweeps[0], "setup_s": setup}


# ------------------------------------------------------------ reference arm
def run_reference(args):
    world, rank, local, pg = dist_setup()
    if rank != 0:
        return
    from oracle import ref
    from paper_2502_21013_b200.abi import default_cfg
    desc = ref.baseline_desc(args.config)
    D, config = workload_config(desc, args.config, world)
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libtpref.so not built"}))
        return
    cores = ref.hardware_threads()
    cfg = default_cfg(tol=1e-8, threads=cores)
    out = {"metric": METRIC, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "f64", "data": "synthetic", "config": config, "impl": "reference"}
    if args.config <= 1:
        # Setup (not timed): the reference's own static_init and frozen-field
        # nu_hat.  A sweep's CPU cost does not depend on the state (every sweep
        # factorises all N/2+1 frequency blocks), so static_init runs at a loose
        # Newton tolerance to keep the arm within minutes.
        t0 = time.perf_counter()
        U0 = ref.static_init(desc, default_cfg(static_tol=1e-2, threads=cores))[0]
        nu, q = ref.choose_nu_hat(desc, U0, cfg)
        setup_s = time.perf_counter() - t0
        one = default_cfg(tol=1e-12, m1_max_outer=1, threads=cores)
        times = []
        U = U0
        for k in range(args.warmup + args.steps):
            r = ref.solve_m1(desc, nu, q, U, one, cache=0)
            if k >= args.warmup:
                times.append(max(r.wall_time - r.setup_time, 1e-9))
            U = r.U
        sample = ("full sweeps of the workload (tpfem solve_m1_fixed_point, m1_max_outer=1), tpfem compiled "
                  "from /root/reference with the shim sparse LDL^T; U0 = the reference's static_init at "
                  "static_tol 1e-2 (a sweep's cost does not depend on the state)")
        stages = None
    else:
        # nu_hat: the midpoint of each material law (a stage's cost does not
        # depend on it; the reference's own static_init at this size runs for hours)
        nu = np.ones(5)
        for m in range(desc.n_materials):
            nu[m] = 0.5 * (desc.material[m].nu0 + desc.material[m].nu_inf)
        sweeps, stages, note, setup_s = sampled_reference_sweep(desc, nu, args.config, cores,
                                                                args.warmup + args.steps)
        times = sweeps[args.warmup:]
        sample = "per step, one reference sweep estimated stage by stage: " + note
    tot = float(np.sum(times))
    value = D * len(times) / tot
    out.update({"value": value, "ms_per_step": tot / len(times) * 1e3,
                "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                                 "sample": sample},
                "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                "setup_s": setup_s, "sweep_s": times})
    if stages:
        out["stages_s"] = stages
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--calib-sweeps", type=int, default=3,
                    help="isolated dominant-kernel calibration sweeps after the timed region (0: off)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-mesh", dest="mesh", action="store_false",
                    help="skip the general-mesh leg (reference transformer config)")
    ap.add_argument("--no-full-solve", dest="full_solve", action="store_false")
    ap.add_argument("--no-cfg1-leg", dest="cfg1_leg", action="store_false",
                    help="skip the configs[1] leg (device sweeps + time to 1e-8 + one reference sweep)")
    ap.add_argument("--replicas", action="store_true", help="N>1: independent copies instead of sharding")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
