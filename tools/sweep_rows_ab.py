"""A/B of the sweep kernel: the row-walking k_sweep_rows (default) against
the 32x8-tile k_sweep_slices (TPGPU_SWEEP_TILE=1), each in its own process.

Per config: static_init, frozen-field nu_hat, m1_begin (the initial residual:
one residual_and_rhs), two sweeps; prints r0, the sweep residuals and a
digest of U, then compares the two variants (r0 and the residuals to 1e-13 / 1e-12 of r0,
U to 1e-13 relative).  --time: also times residual_and_rhs alone (the
initial-residual call, CUDA events around m1_begin's kernel are not exposed,
so wall time of m1_begin over --reps calls after a sync).
Usage: python tools/sweep_rows_ab.py --configs 0 1 2
"""
import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys, time
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2502_21013_b200 import Problem, baseline_desc, default_cfg
cfg = default_cfg(tol=1e-8)
cfgi, reps = int(sys.argv[2]), int(sys.argv[3])
with Problem(baseline_desc(cfgi)) as p:
    p.static_init(cfg, want_state=False)
    p.choose_nu_hat(cfg)
    r0 = p.m1_begin(cfg)
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        p.m1_begin(cfg)
        t.append(time.perf_counter() - t0)
    res = [p.m1_sweep()[0] for _ in range(2)]
    U = p.get_state() if cfgi <= 2 else None
out = {"r0": r0, "res": res, "begin_s": sorted(t)[len(t) // 2] if t else None}
if U is not None:
    np.save(sys.argv[4], U)
print(json.dumps(out))
"""


def run(cfgi, env_extra, reps, path):
    env = dict(os.environ)
    env.pop("TPGPU_SWEEP_TILE", None)
    env.update(env_extra)
    r = subprocess.run([sys.executable, "-c", CHILD, ROOT, str(cfgi), str(reps), path], env=env,
                       capture_output=True, text=True, timeout=1800)
    if r.returncode != 0:
        raise SystemExit(r.stderr[-3000:])
    return json.loads(r.stdout.strip().splitlines()[-1])


def main():
    import numpy as np
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[0, 1, 2])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--rows-env", nargs="*", default=[], help="KEY=VAL for the rows run (e.g. TPGPU_LIB=libtpgpu_ra8.so)")
    a = ap.parse_args()
    ok = True
    for cfgi in a.configs:
        pr, pt = f"/tmp/U_rows_{cfgi}.npy", f"/tmp/U_tile_{cfgi}.npy"
        rows = run(cfgi, dict(e.split("=", 1) for e in a.rows_env), a.reps, pr)
        tile = run(cfgi, {"TPGPU_SWEEP_TILE": "1"}, a.reps, pt)
        d_r0 = abs(rows["r0"] - tile["r0"]) / tile["r0"]
        # sweep residuals against the first (near the fp64 floor of cfg >= 2 the
        # residual itself carries the summation-order noise of the partials)
        d_res = max(abs(x - y) / tile["r0"] for x, y in zip(rows["res"], tile["res"]))
        line = {"config": cfgi, "rows": rows, "tile": tile, "r0_rel": d_r0, "res_rel": d_res}
        good = d_r0 <= 1e-13 and d_res <= 1e-12
        if cfgi <= 2:
            Ur, Ut = np.load(pr), np.load(pt)
            line["U_rel"] = float(np.linalg.norm(Ur - Ut) / np.linalg.norm(Ut))
            line["U_bitwise"] = bool(np.array_equal(Ur, Ut))
            good = good and line["U_rel"] <= 1e-13
            os.remove(pr)
            os.remove(pt)
        line["ok"] = good
        ok = ok and good
        print(json.dumps(line), flush=True)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
