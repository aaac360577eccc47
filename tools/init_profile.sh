# static_init profile: phase trace at cfg 3 (TPGPU_TRACE) and the kernel launch list at cfg 2
TAG=${1:-r2zg}
TPGPU_TRACE=1 TPGPU_DEBUG_NEWTON=1 timeout 600 python tools/profile_init.py --config 3 > gpurun_out/${TAG}_init_trace_cfg3.txt 2>&1; echo trace rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file gpurun_out/${TAG}_init_launches_cfg2.csv \
  python tools/profile_init.py --config 2 > gpurun_out/${TAG}_init_ncu_cfg2.log 2>&1; echo ncu rc=$?
python tools/launch_summary.py gpurun_out/${TAG}_init_launches_cfg2.csv > gpurun_out/${TAG}_init_launches_cfg2.txt 2>&1
