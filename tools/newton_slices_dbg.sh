mkdir -p gpurun_out
cat > /tmp/one.py <<'PY'
import os,sys
sys.path.insert(0,'.')
from paper_2502_21013_b200 import Problem, baseline_desc, default_cfg
cfg=default_cfg(tol=1e-8)
with Problem(baseline_desc(1)) as p:
    U,c=p.static_init(cfg)
PY
TPGPU_DEBUG_NEWTON=2 python /tmp/one.py 2> gpurun_out/r2o_nslice_default.txt
TPGPU_DEBUG_NEWTON=2 TPGPU_NEWTON_FORCING=1e-2,1,1e-2 python /tmp/one.py 2> gpurun_out/r2o_nslice_forcing.txt
TPGPU_DEBUG_NEWTON=2 TPGPU_NEWTON_FORCING=1e-12,0,1e-10 TPGPU_NEWTON_RTOL=1e-12 python /tmp/one.py 2> gpurun_out/r2o_nslice_tight.txt
wc -l gpurun_out/r2o_nslice_*
