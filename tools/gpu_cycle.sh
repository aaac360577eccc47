# usage: gpu_cycle.sh TAG [bench-args] -- parity tests, bench, launch lists, dominant-kernel capture
TAG=$1; shift
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 900 python bench.py --steps 10 --warmup 3 "$@" > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?
# one sweep: per-launch durations and DRAM bytes
python tools/profile_sweep.py --sweeps 1 > gpurun_out/prof_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --profile-from-start off --csv --log-file gpurun_out/launches_$TAG.csv \
      python tools/profile_sweep.py --sweeps 1 > gpurun_out/ncu_$TAG.log 2>&1; echo sweep-list rc=$?
# the bench command itself (launch list; its printed numbers are not bench values)
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/launches_bench_$TAG.csv python bench.py --steps 2 --warmup 3 "$@" \
  > gpurun_out/ncu_bench_$TAG.log 2>&1; echo bench-list rc=$?
# full capture of the dominant kernel (fine-level up pass of the 2nd iteration)
bash tools/ncu_kernels.sh $TAG "k_stream_up:9" > /dev/null 2>&1; echo full rc=$?
