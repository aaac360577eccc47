# default lib (k_sweep_rows without the ns guard): parity vs tile + ncu time; static_init A/B of TPGPU_SLICE_STREAM_APPLY at cfg 2 / 3
mkdir -p gpurun_out
bash tools/ring_cycle.sh r2zl 2>&1
for c in 2 3; do
  for e in "" "TPGPU_SLICE_STREAM_APPLY=1"; do
    echo "== cfg $c [$e]"; env $e timeout 900 python tools/profile_init.py --config $c 2>&1 | tail -1
  done
done
