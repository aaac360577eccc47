import numpy as np, sys, os
sys.path.insert(0, '/root/repo')
from paper_2502_21013_b200 import Problem, baseline_desc, default_cfg
d = baseline_desc(0)
cfg = default_cfg(tol=1e-8)
hs = []
for rep in range(3):
    with Problem(d) as p:
        p.static_init(cfg, want_state=False)
        p.choose_nu_hat(cfg)
        U, r = p.solve_m1_fixed_point(None, cfg)
        hs.append(np.array(r.residual_history))
print("iters", [len(h) for h in hs], "max diff", max(np.max(np.abs(h - hs[0]) / hs[0]) for h in hs[1:]))
