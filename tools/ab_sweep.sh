# A/B timing of library variants / env settings on cfg1 (run on the GPU box)
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
run() { echo "== $*"; env "$@" timeout 300 python tools/mg_experiments.py 1e-12 2>&1 | grep rtol; }
for v in "$@"; do run $v; done
