# usage: gpu_cycle.sh TAG [bench-args] -- parity tests, bench, launch list
TAG=$1; shift
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 600 python bench.py --steps 10 --warmup 3 "$@" > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python tools/profile_sweep.py --sweeps 1 > gpurun_out/prof_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_$TAG.csv python tools/profile_sweep.py --sweeps 1 > gpurun_out/ncu_$TAG.log 2>&1; echo rc=$?
