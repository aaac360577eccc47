# usage: cycle_r2zg.sh TAG -- full GPU suite, default bench (cfg 3), cfg-3 launch list, k_sweep_rows full capture
TAG=$1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/${TAG}_gputests.txt 2>&1; tail -3 gpurun_out/${TAG}_gputests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1; tail -2 gpurun_out/${TAG}_smoke.txt
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_cfg3.json 2> gpurun_out/${TAG}_bench.err; echo bench rc=$?
bash tools/ncu_launch_list.sh $TAG 3 1; echo list rc=$?
bash tools/ncu_one.sh ${TAG}_sweep_rows 3 k_sweep_rows 0; echo full rc=$?
