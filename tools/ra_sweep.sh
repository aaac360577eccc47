timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
run() { echo "== $*"; env "$@" timeout 300 python tools/mg_experiments.py 1e-12 2>&1 | grep rtol | sed 's/.*cfg1/cfg1/'; }
run X=1
run TPGPU_TILE_COARSE=1
run TPGPU_RA5=4
run TPGPU_RA5=8
run TPGPU_RA5U=4
run TPGPU_RA7=2
run TPGPU_RA7=6
run TPGPU_RA7U=4
run TPGPU_RH=32
