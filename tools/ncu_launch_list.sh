#!/bin/bash
# usage: tools/ncu_launch_list.sh TAG CONFIG [SWEEPS]
# per-launch time and DRAM bytes of the kernels of SWEEPS production sweeps
# (after warm-up) of BASELINE config CONFIG -> gpurun_out/launches_TAG_cfgC.csv
TAG=$1; C=$2; S=${3:-1}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --profile-from-start off --csv --log-file gpurun_out/launches_${TAG}_cfg${C}.csv \
    python tools/profile_sweep.py --config $C --sweeps $S --timer 1 > gpurun_out/ncu_${TAG}_cfg${C}.log 2>&1
python tools/launch_summary.py gpurun_out/launches_${TAG}_cfg${C}.csv > gpurun_out/launches_${TAG}_cfg${C}.txt
