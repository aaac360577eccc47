# new ragged-size sweep tests; A/B of the chunk height on the first Galerkin level (1000 <= m < 2000) at cfg 3
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "ragged" 2>&1 | tail -3
bash tools/ab_cfg.sh r2zn 3 12 "rh128:TPGPU_X=0" "rhmid64:TPGPU_RHMID=64" "rhmid32:TPGPU_RHMID=32"
