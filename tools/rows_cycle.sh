set -x
timeout 900 python tools/sweep_rows_ab.py --configs 0 1 2 --reps 0 > gpurun_out/r2zf_rows_ab.txt 2>&1; echo ab rc=$?
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -x -q 2>&1 | tail -3
for v in rows tile sg2 sg8; do
  case $v in rows) E="";; tile) E="TPGPU_SWEEP_TILE=1";; sg2) E="TPGPU_LIB=libtpgpu_sg2.so";; sg8) E="TPGPU_LIB=libtpgpu_sg8.so";; esac
  env $E timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:k_sweep --profile-from-start off --csv --log-file gpurun_out/r2zf_sweepk_$v.csv \
    python tools/profile_sweep.py --config 3 --warmup 1 --sweeps 1 > gpurun_out/r2zf_prof_$v.log 2>&1; echo $v rc=$?
done
