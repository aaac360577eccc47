# usage: ncu_kernels.sh TAG "name1:skip1 name2:skip2 ..."  -- full ncu sets for selected launches
# (env such as TPGPU_LIB passes through to the profiled process)
TAG=$1; shift
python tools/profile_sweep.py --sweeps 1 > gpurun_out/prof_plain_$TAG.log 2>&1 || exit 1
for spec in $1; do
  k=${spec%%:*}; s=${spec##*:}
  ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"$k" -s $s -c 1 \
      -o /tmp/p_${TAG}_${k}_$s python tools/profile_sweep.py --sweeps 1 > gpurun_out/ncu_${TAG}_${k}_$s.log 2>&1
  ncu -i /tmp/p_${TAG}_${k}_$s.ncu-rep --page raw --csv > gpurun_out/raw_${TAG}_${k}_$s.csv
  ncu -i /tmp/p_${TAG}_${k}_$s.ncu-rep --page details --csv > gpurun_out/details_${TAG}_${k}_$s.csv
  ncu -i /tmp/p_${TAG}_${k}_$s.ncu-rep --page source --csv > gpurun_out/source_${TAG}_${k}_$s.csv 2>/dev/null
  ncu -i /tmp/p_${TAG}_${k}_$s.ncu-rep --page source --csv --print-source cuda > gpurun_out/srccuda_${TAG}_${k}_$s.csv 2>/dev/null
done
ls -la gpurun_out | tail -20
