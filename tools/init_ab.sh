for t in 1e-12 1e-10 1e-8 1e-6; do
  echo "== NEWTON_RTOL $t"
  TPGPU_NEWTON_RTOL=$t timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "static_init or cfg1_against or m1_matches or cfg0" 2>&1 | tail -1
  TPGPU_NEWTON_RTOL=$t python tools/profile_init.py 2>&1 | tail -1
done
