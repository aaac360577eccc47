#!/bin/bash
# usage: tools/ab_cfg.sh TAG CONFIG SWEEPS lib1 lib2 ...   (lib "" = libtpgpu.so)
# device sweep times of BASELINE config CONFIG for each library variant, twice
TAG=$1; C=$2; S=$3; shift 3
for pass in 1 2; do
  for lib in "$@"; do
    TPGPU_LIB=$lib python tools/run_config.py --config $C --max-sweeps $S --tol 0 > gpurun_out/ab_${TAG}_${lib:-base}_$pass.json 2>&1
    python -c "
import json,sys; d=json.load(open('gpurun_out/ab_${TAG}_${lib:-base}_$pass.json'))
print('${lib:-base}', 'pass $pass', 'median sweep ms', round(d['median_sweep_s']*1e3,2), 'fi', d['frequency_iterations'][-3:])"
  done
done
