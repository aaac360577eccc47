b() { env "$@" timeout 300 python bench.py --steps 20 --warmup 3 --no-mesh --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['ms_per_step'],3), round(d['full_solve']['time_to_residual_s'],4), round(d['full_solve']['sweeps_s'],4))"; }
for i in 1 2; do
b TPGPU_FREQ_GROUPS=3
b TPGPU_FREQ_GROUPS=4
b TPGPU_FREQ_GROUPS=5
done
