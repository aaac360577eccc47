"""A/B of static_init under environment settings read per call (TPGPU_NEWTON_*):
one static_init with the reference settings (exact Newton solves,
TPGPU_NEWTON_FORCING=0), then one per setting "NAME=VAL[,NAME=VAL...]";
prints time, Newton counts against the reference run and the U0 difference.
Usage: python tools/init_env_ab.py --config 2 --settings "" TPGPU_NEWTON_WARM=1
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2502_21013_b200 import Problem, baseline_desc, default_cfg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--settings", nargs="+", default=[""])
a = ap.parse_args()
cfg = default_cfg(tol=1e-8)
KEYS = ("TPGPU_NEWTON_FORCING", "TPGPU_NEWTON_WARM", "TPGPU_NEWTON_F32")


def apply(setting):
    for k in KEYS:
        os.environ.pop(k, None)
    for kv in filter(None, setting.split(",")):
        k, v = kv.split("=", 1)
        os.environ[k] = v


with Problem(baseline_desc(a.config)) as p:
    p.static_init(cfg, want_state=False)
    apply("TPGPU_NEWTON_FORCING=0")
    t = time.perf_counter()
    U_ref, c_ref = p.static_init(cfg)
    print(f"cfg {a.config} exact: {time.perf_counter() - t:.3f} s newton sum {c_ref.sum()}", flush=True)
    nrm = np.linalg.norm(U_ref)
    for st in a.settings:
        apply(st)
        t = time.perf_counter()
        U, c = p.static_init(cfg)
        dt = time.perf_counter() - t
        per = np.linalg.norm(U - U_ref, axis=1) / np.maximum(np.linalg.norm(U_ref, axis=1), 1e-300)
        print(f"cfg {a.config} [{st or 'default'}]: {dt:.3f} s counts_equal {bool(np.array_equal(c, c_ref))} "
              f"relU {np.linalg.norm(U - U_ref) / nrm:.2e} max_slice {per.max():.2e}", flush=True)
