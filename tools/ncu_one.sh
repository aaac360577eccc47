#!/bin/bash
# usage: tools/ncu_one.sh TAG CONFIG KERNEL_REGEX [SKIP]
# one `ncu --set full` capture of the first (or SKIP-th) matching launch in a
# production sweep of BASELINE config CONFIG -> gpurun_out/{details,raw,source}_TAG.csv
TAG=$1; C=$2; K=$3; S=${4:-0}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on --profile-from-start off --kernel-name-base demangled -k regex:"$K" -s $S -c 1 \
    -o /tmp/p_$TAG python tools/profile_sweep.py --config $C --sweeps 1 > gpurun_out/ncu_$TAG.log 2>&1
ncu -i /tmp/p_$TAG.ncu-rep --page details --csv > gpurun_out/details_$TAG.csv
ncu -i /tmp/p_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_$TAG.csv
ncu -i /tmp/p_$TAG.ncu-rep --page source --csv > gpurun_out/source_$TAG.csv 2>/dev/null
