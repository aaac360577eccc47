# A/B of frequency-group settings on cfg1 through bench.py (run on the GPU box)
b() { env "$@" timeout 300 python bench.py --steps 20 --warmup 3 --no-mesh --no-cpu-baseline --no-full-solve 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['ms_per_step'],3))"; }
for i in 1 2; do
b TPGPU_FREQ_GROUPS=3
b TPGPU_FREQ_GROUPS=4
b TPGPU_FREQ_GROUPS=5
b TPGPU_FREQ_GROUPS=8
b TPGPU_FREQ_GROUPS=4 TPGPU_GROUP_PRIO=2
b TPGPU_FREQ_GROUPS=6 TPGPU_GROUP_PRIO=2
b TPGPU_FREQ_GROUPS=8 TPGPU_GROUP_PRIO=2
done
