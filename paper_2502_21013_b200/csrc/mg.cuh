// Batched geometric-multigrid-preconditioned conjugate-gradient solver on the
// structured P1 grid.  Replaces the reference's per-frequency sparse direct
// solves (PeriodicSolver::solve_frequency, periodic.hpp:252-289, through
// SparseSolver, solve.hpp:51-126) and the static-initialisation Newton solves
// (newton_elliptic, solvers.hpp:156-157).
//
//   MODE 0 (frequency): T = cplx, operator lambda_b M + K with shared real
//     7-point stencils per level, COCG in the bilinear form x^T y -- the
//     blocks are complex symmetric, not Hermitian (periodic.hpp:124).
//   MODE 1 (slice): T = double, per-batch real SPD stencils (Jacobians), PCG.
//
// Preconditioner: symmetric V(nu,nu) cycle, damped-Jacobi smoothing, P1
// interpolation on the nested triangulation, Galerkin coarse operators
// (R = P^T), exact dense solve on the coarsest grid (<= 7x7 nodes).  Batches
// converge independently (per-batch masks); all reductions are fixed-order.
#pragma once

#include "tp_internal.cuh"

namespace tpgpu {

// Slice-mode (Newton Jacobian) smoother: l1-Jacobi diagonal sum_j |J_ij| with
// the degree-2 Chebyshev weights for D_l1^-1 J on [1/15, 1] (1: on; 0: plain
// damped Jacobi, omega = 0.6 on the true diagonal).  Interval measured on cfg 2
// static_init (tools/init_omega_sweep.py, profiles/r2o_omega_sweep.txt,
// r2t_omega.txt): [1/6, 1] 3.98-4.00 s, [1/10, 1] 3.77, [1/15, 1] 3.69-3.70,
// [1/20, 1] 3.69, [1/25, 1] 4.05, [1/4, 1] 4.28; Newton counts equal
#ifndef TPGPU_SLICE_L1
#define TPGPU_SLICE_L1 1
#endif
constexpr double kL1Omega1 = 1.1583, kL1Omega2 = 4.9169;

struct MGConfig {
  int pre = 2, post = 2;    // smoothing sweeps
  // Damped-Jacobi steps with a degree-2 Chebyshev pair of weights for D^-1 A
  // on [1/3, 2] (pre: omega then omega2; post: omega2 then omega -- adjoint)
  double omega = 0.57;
  double omega2 = 1.7;
  double rtol = 1e-13;      // ||r_b|| <= rtol ||b_b||
  int max_iter = 200;
  bool rb_fine = true;      // red-black Gauss-Seidel on the 5-point fine level
};

// Operator data for the streaming kernels (mg_fine.cu).  Fine level: K_hat
// regenerated from cell materials + nu_hat (edge weights), lumped mass
// diagonal.  Galerkin levels: the shared 7-point K and M planes (stride n).
struct FineOp {
  const double* we = nullptr;     // (cells+1)^2 vertex grid: K_hat edge weight (X,Y)-(X+1,Y)
  const double* wn = nullptr;     // (cells+1)^2 vertex grid: K_hat edge weight (X,Y)-(X,Y+1)
  const double* mass = nullptr;   // n
  const double* K = nullptr;      // Galerkin levels: 7n (slice mode: per-slice Jacobians, stride kstride)
  const double* M = nullptr;      // Galerkin levels: 7n
  size_t kstride = 0;             // slice mode: coefficients per batch (7n)
  const float* Kf = nullptr;      // slice mode: fp32 C/E/N/NE planes for the V-cycle passes (optional)
  size_t kfstride = 0;            // floats per batch (4n)
  const cplx* lam = nullptr;      // per batch symbol
  int m = 0, c = 0, n = 0;
  int rha = 32;                   // rows per warp item of the apply pass (set at launch, rha_for)
};

// Krylov scalars reduced inside the fine passes (frequency mode, fused path):
// the consumer of a pass's per-warp partial sums sums them itself (every warp
// of a batch, fixed order) instead of a separate scalar kernel.  apply:
// rho_it = sum of the up pass's r^T z partials, beta = rho_it / rho_{it-1};
// down: mu = sum of the apply's p^T q partials, alpha = rho_it / mu.
struct ScalFuse {
  const double* part = nullptr;  // producer's partials, per (re, im) pairs per batch; nullptr: off
  int per = 0;
  const cplx* rho_r = nullptr;   // apply: rho of the previous iteration; down: this iteration's
  cplx* rho_w = nullptr;         // apply: this iteration's rho (written by one warp per batch)
  cplx* alpha = nullptr;         // down: alpha, the deferred x coefficient, mu (one warp per batch)
  cplx* xa = nullptr;
  cplx* mu = nullptr;
};

// The bottom levels of the frequency-mode V-cycle, run as one kernel
// (mg_small.cu): level 0 of this list is the first level whose work vectors
// fit in shared memory, the last is the coarsest (dense solve).
constexpr int kMaxSmall = 6;
struct SmallLevels {
  int levels = 0;
  int m[kMaxSmall] = {};
  const double* K[kMaxSmall] = {};
  const double* M[kMaxSmall] = {};
  // packed copies (pack_small_levels): per level 4 planes (C, E, N, NE) of
  // (m+2)^2 zero-padded {K, M} pairs
  const double2* KM[kMaxSmall] = {};
};
size_t small_cycle_smem(const int* m, int levels);
size_t small_pack_size(const int* m, int levels);  // doubles
void pack_small_levels(Problem& p, SmallLevels& sl, double* buf);
void launch_small_cycle(Problem& p, const SmallLevels& sl, const cplx* lam, const cplx* inv, const cplx* b,
                        cplx* z, const int* active, double om1, double om2, int nb, int n_active);

// Stencils of one level for the whole batch (slice mode) or shared (freq mode).
struct LevelOp {
  int m = 0, n = 0;
  const double* K = nullptr;  // freq: 7n shared ; slice: 7n per batch (stride 7n)
  const double* M = nullptr;  // freq only
  bool five = false;          // freq mode: K 5-point and M diagonal (fine level)
  FineOp fine;                // freq mode level 0: streaming kernels (we != nullptr)
  const float* Kf = nullptr;  // slice mode: fp32 copies of the C/E/N/NE planes (4n per batch) for the V-cycle
  bool drop_m = false;        // freq mode Galerkin level: the V-cycle's level operator is K alone
                              // (max |lambda| M negligible against K, Problem::build_freq_work)
};

template <int MODE>
struct BatchSolver {
  using T = typename std::conditional<MODE == 0, cplx, double>::type;
  Problem* p = nullptr;
  MGConfig cfg;
  int B = 0;                      // batch capacity
  std::vector<LevelOp> ops;       // per level
  const T* coarse_inv = nullptr;  // n_L^2 per batch
  const cplx* lam = nullptr;      // freq mode: per batch symbol (device)
  const int* ext_mask = nullptr;  // optional: batches with mask 0 are skipped
  // optional stopping floor: batch b stops at ||r_b||^2 <= rtol^2 max(||b_b||^2,
  // bfloor_scale * *bfloor) (device scalar: ||b||^2 of the whole right-hand side)
  const double* bfloor = nullptr;
  double bfloor_scale = 0.0;
  // optional per-batch tolerance: batch b stops at rtol^2 * bscale[b] times
  // its reference (inexact Newton forcing terms, newton.cu)
  const double* bscale = nullptr;
  // work
  std::vector<DevBuf<T>> lb, lz0, lz1;  // per level (level 0: b is external)
  DevBuf<T> r, r2, p0, p1, q;
  DevBuf<T> xa;  // deferred solution-update coefficient per batch (fused Krylov update)
  DevBuf<double> part;
  DevBuf<T> rho, mu, alpha, beta;
  DevBuf<T> rho2;               // fused scalars: rho of the two most recent iterations (2B)
  DevBuf<double> partA, partD;  // fused scalars: apply / down partials (kept apart from the up pass's)
  DevBuf<double> bn2, rn2, bown;
  DevBuf<int> active;
  DevBuf<int> count;
  DevBuf<unsigned> done_ctr;  // blocks of the stopping-test kernel that finished (last one publishes)
  int* h_count = nullptr;      // mapped pinned [2]
  int* h_count_dev = nullptr;  // its device address
  int cur_active = 0;      // active batches as last seen by the host (kernel-timer byte accounting)
  int small_from = -1;     // frequency mode: first level handled by the fused small-level cycle
  SmallLevels small;        // its levels (stencils packed into small_pack)
  DevBuf<double> small_pack;
  cudaEvent_t ev[2] = {nullptr, nullptr};

  void init(Problem* prob, const std::vector<LevelOp>& levels, int batches, const MGConfig& c);
  ~BatchSolver();
  // Solve A_b x_b = b_b for b < nb (<= B).  x holds the initial guess when
  // `warm`, else is overwritten from zero.  Returns iterations.
  int solve(const T* b, T* x, int nb, bool warm, SolveStats* st);
  void set_ops(const std::vector<LevelOp>& levels) { ops = levels; }

 private:
  void vcycle(int lvl, int nb, T* z_out_level0, bool dot);
  T* vcycle_level(int lvl, int nb, const T* bl, T* z_first, bool first_done, bool dot);
  T* vcycle_generic(int lvl, int nb, const T* bl, bool dot);
  bool stream_level(int l) const;  // slice mode: this level's passes run streamed
  FineOp stream_op(int l) const;   // the streaming kernels' view of level l
  // fine streaming level: down pass (optionally fusing r_out = r_in - alpha q),
  // and the rest of the cycle (coarse levels + up pass)
  void fine_down0(int nb, const T* r_in, const T* qv = nullptr, T* r_out = nullptr, const ScalFuse* sf = nullptr,
                  double* part_out = nullptr);
  T* fine_rest0(int nb, const T* bl, bool dot);
};

// fp32 copies of the C/E/N/NE planes of `batches` 7-point stencils (stride 7n
// -> 4n floats per batch)
void launch_planes_f32(Problem& p, const double* K, int m, float* Kf, int batches);
// Galerkin coarse stencil Ac = P^T Af P for `batches` stencils (stride 7n).
void launch_rap(Problem& p, const double* Af, int mf, double* Ac, int mc, int batches);
// Dense inverse of the coarsest operator per batch.
void launch_coarse_inverse_freq(Problem& p, const double* K, const double* M, int m,
                                const cplx* lam, cplx* inv, int batches);
void launch_coarse_inverse_slice(Problem& p, const double* J, int m, double* inv, int batches);
// Streaming kernels (mg_fine.cu).  kind: 0 apply, 1 down, 2 up.
int fine_partials(int m, int kind);
// (xa != nullptr: also x += xa p_in, the deferred update of the fused Krylov step)
void launch_fine_apply(Problem& p, const FineOp& op, const cplx* z, const cplx* pin, cplx* pout, cplx* q,
                       const cplx* beta, const int* active, int first, int nb, double* part, bool init,
                       cplx* x = nullptr, const cplx* xa = nullptr, const ScalFuse* sf = nullptr);
// V-cycle down / up passes of one level (fine: op.we set; Galerkin: op.K set)
// (q != nullptr: fine level with the fused Krylov update r_out = r - alpha q,
// partial ||r_out||^2 per warp item into part)
void launch_stream_down(Problem& p, const FineOp& op, const cplx* r, cplx* z2, cplx* bc, int mc,
                        const int* active, double om1, double om2, int nb, const cplx* q = nullptr,
                        const cplx* alpha = nullptr, cplx* rout = nullptr, double* part = nullptr,
                        const ScalFuse* sf = nullptr);
void launch_stream_up(Problem& p, const FineOp& op, const cplx* r, const cplx* z2, const cplx* xc, int mc,
                      cplx* z, const int* active, double om1, double om2, int nb, int dot, double* part);
// slice mode: real vectors, per-slice Jacobian stencils
void launch_stream_down(Problem& p, const FineOp& op, const double* r, double* z2, double* bc, int mc,
                        const int* active, double om1, double om2, int nb, const double* q = nullptr,
                        const double* alpha = nullptr, double* rout = nullptr, double* part = nullptr);
void launch_fine_apply(Problem& p, const FineOp& op, const double* z, const double* pin, double* pout, double* q,
                       const double* beta, const int* active, int first, int nb, double* part, bool init,
                       double* x = nullptr, const double* xa = nullptr);
void launch_stream_up(Problem& p, const FineOp& op, const double* r, const double* z2, const double* xc, int mc,
                      double* z, const int* active, double om1, double om2, int nb, int dot, double* part);
// Build fine-grid element stencils (K_hat or Jacobians at U, per batch).
void launch_element_stencil(Problem& p, bool jacobian, const double* U, double* st, int batches);

}  // namespace tpgpu
