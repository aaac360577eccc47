#!/bin/bash
# usage: tools/ab_cfg.sh TAG CONFIG SWEEPS "name1:ENV=.. ENV2=.." "name2:..." ...
# device sweep times of BASELINE config CONFIG for each variant (environment
# settings, e.g. TPGPU_LIB=libtpgpu_x.so TPGPU_FFT_P=8), two passes
TAG=$1; C=$2; S=$3; shift 3
for pass in 1 2; do
  for spec in "$@"; do
    name=${spec%%:*}; envs=${spec#*:}
    env $envs python tools/run_config.py --config $C --max-sweeps $S --tol 1e-300 > gpurun_out/ab_${TAG}_${name}_$pass.json 2> gpurun_out/ab_${TAG}_${name}_$pass.err
    python -c "
import json; d=json.load(open('gpurun_out/ab_${TAG}_${name}_$pass.json'))
print('$name', 'pass $pass', 'median sweep ms', round(d['median_sweep_s']*1e3,2), 'init_s', round(d['init_s'],2), 'fi', d['frequency_iterations'][-3:])" || tail -3 gpurun_out/ab_${TAG}_${name}_$pass.err
  done
done
