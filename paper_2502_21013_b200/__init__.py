"""B200-native fixed-point sweep of the time-periodic nonlinear eddy-current
solver of arXiv 2502.21013 (reference: tpfem).  CUDA kernels + C ABI in
csrc/ (libtpgpu.so, include/tpgpu.h); this package is the Python mirror of the
reference interface over that ABI."""
from .abi import TpProblemDesc, TpSolverCfg, default_cfg  # noqa: F401
from .api import (Comm, Problem, SolveError, SolveReport, baseline_desc, block_l2,  # noqa: F401
                  nccl_unique_id, shard_freq_order, shard_plan, stopping_check)
