# A/B of k_sweep_rows build variants (libtpgpu_<v>.so; "base" = libtpgpu.so): parity against the tile kernel, then ncu time at cfg 3
TAG=$1; shift
mkdir -p gpurun_out
for v in base "$@"; do
  case $v in base) E="";; *) E="--rows-env TPGPU_LIB=libtpgpu_$v.so";; esac
  timeout 600 python tools/sweep_rows_ab.py --configs 0 1 --reps 0 $E > gpurun_out/${TAG}_ab_$v.txt 2>&1; echo ab $v rc=$?
done
for v in base "$@"; do
  case $v in base) E="";; *) E="TPGPU_LIB=libtpgpu_$v.so";; esac
  env $E timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:k_sweep --profile-from-start off --csv --log-file gpurun_out/${TAG}_sweepk_$v.csv \
    python tools/profile_sweep.py --config 3 --warmup 1 --sweeps 1 > gpurun_out/${TAG}_prof_$v.log 2>&1; echo $v rc=$?
  python tools/launch_summary.py gpurun_out/${TAG}_sweepk_$v.csv | sed -n 2p
done
