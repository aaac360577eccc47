/*
 * tpgpu.h -- C ABI of the B200-native fixed-point sweep for the time-periodic
 * nonlinear eddy-current solver of arXiv 2502.21013 (reference: tpfem,
 * /root/reference/proj).
 *
 * The reference has no C ABI: it is header-only C++ templates whose plugin
 * seam is the `Problem` concept plus three generic entry points
 * (SURVEY.md §8(b)).  Every function below names the reference interface it
 * replaces.  Conventions:
 *   - all host arrays are caller-owned fp64, slice-major: X[i*n + j] is dof j
 *     of time slice i, slice i <-> time (i+1)*tau (state.hpp:9-33);
 *   - every function returns TP_OK or an error code; reference exceptions map
 *     to codes: std::invalid_argument -> TP_EINVAL, SolveError -> TP_ESOLVE
 *     (tp_last_error() returns the message and the achieved relative
 *     residual, like SolveError::residual(), solve.hpp:17-26), CUDA/NCCL
 *     failures -> TP_ECUDA;
 *   - non-convergence is not an error: it is tp_report.status (solvers.hpp:32);
 *   - one tp_problem is bound to one CUDA device and used from one host
 *     thread at a time; there is no global mutable state besides the
 *     thread-local last error.
 */
#ifndef TPGPU_H
#define TPGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TPGPU_VERSION 1

enum tp_status_code { TP_OK = 0, TP_EINVAL = 1, TP_ESOLVE = 2, TP_ECUDA = 3 };

/* SolveStatus, solvers.hpp:32 */
enum tp_solve_status { TP_CONVERGED = 0, TP_MAX_ITER = 1, TP_STALLED = 2 };

/* NuHatMode, assembly.hpp:207-210 */
enum tp_nu_hat_mode { TP_NU_HAT_THEORY = 0, TP_NU_HAT_FROZEN_FIELD = 1 };

/* kNumRegions, mesh.hpp:25: material labels 0..4 */
#define TP_MAX_MATERIALS 5
#define TP_MAX_RECTS 8
#define TP_MAX_HARMONICS 4

/* Painter's-order rectangle carrying a material label (RectRegion, mesh.hpp:46-51;
 * containment is inclusive, the last rectangle containing a cell centroid wins,
 * cells covered by none get material 0). */
typedef struct tp_rect {
  double x0, y0, x1, y1;
  int32_t material;
  int32_t pad_;
} tp_rect;

/* Per-material coefficients (replaces MaterialCoefficients, materials.hpp:17-24,
 * with the BASELINE.json law):
 *   nu(s)  = nu0 + (nu_inf - nu0) s^2 / (s^2 + bs^2)      (nu0 == nu_inf: linear)
 *   j(t)   = sum_h amp[h] * sin(2 pi harmonic[h] t / T + phase[h])
 *   sigma  = sigma * noise(centroid) when sigma_noise != 0, else sigma          */
typedef struct tp_material {
  double sigma;
  int32_t sigma_noise;
  int32_t n_harmonics;
  double nu0, nu_inf, bs;
  double amp[TP_MAX_HARMONICS];
  double phase[TP_MAX_HARMONICS];
  int32_t harmonic[TP_MAX_HARMONICS];
} tp_material;

/* Mesh/material/source setup (replaces build_rectilinear_mesh + MaterialTable +
 * assemble_mass/assemble_loads, mesh.hpp:141-190, assembly.hpp:50-106):
 * cells x cells uniform P1 grid on the unit square, each cell split along its
 * lower-left/upper-right diagonal, homogeneous Dirichlet boundary, free dofs
 * numbered row-major, lumped sigma-mass. */
typedef struct tp_problem_desc {
  int32_t cells;
  int32_t steps;           /* N implicit-Euler steps per period */
  double period;           /* T; tau = T/N */
  int32_t n_rects;
  int32_t n_materials;
  tp_rect rect[TP_MAX_RECTS];
  tp_material material[TP_MAX_MATERIALS];
  /* seeded sigma noise: L x L lattice over noise_box, values in [lo, hi],
   * splitmix64(seed) stream, bilinear at triangle centroids */
  uint64_t noise_seed;
  int32_t noise_lattice;
  int32_t flux_samples;    /* theory-mode sampling count (config.hpp:52, default 10001) */
  double noise_lo, noise_hi;
  double noise_box[4];
  double s_max;            /* theory-mode sampling range (config.hpp:51, default 3.0) */
} tp_problem_desc;

/* Mirrors SolverConfig (solvers.hpp:49-69) for the fields on this path, plus
 * the device linear-solver controls (no reference counterpart: the reference
 * solves every frequency block exactly with a sparse direct method). */
typedef struct tp_solver_cfg {
  double tol;                 /* relative block-residual tolerance, default 1e-4 */
  int32_t m1_max_outer;       /* default 200 */
  int32_t armijo_max_halvings;/* default 30 */
  double armijo_slope;        /* default 1e-4 */
  double armijo_backtrack;    /* default 0.5 */
  int32_t nu_hat_mode;        /* default TP_NU_HAT_FROZEN_FIELD */
  int32_t nu_hat_samples;     /* choose_nu_hat samples, default 2000 (assembly.hpp:270) */
  double imag_tol;            /* default 1e-9 */
  double static_tol;          /* default 1e-8 */
  int32_t static_max_newton;  /* default 50 */
  int32_t threads;            /* accepted for interface parity; unused on device */
  /* device frequency / Newton inner solver */
  double inner_rtol;          /* relative residual per block, default 1e-12 */
  int32_t inner_max_iter;     /* default 200 */
  int32_t warm_start;         /* start frequency solves from the previous sweep (default 1) */
  int32_t freq_chunk;         /* frequencies per batched solve (0 = automatic) */
  int32_t slice_chunk;        /* slices per batched Newton solve (0 = automatic) */
  int32_t freq_groups;        /* frequency groups solved concurrently on their own
                                 streams (0 = automatic: 5) */
  /* M2 all-at-once Newton (SolverConfig m2_*, solvers.hpp:52,63-65) */
  int32_t m2_max_outer;       /* default 50 */
  double m2_inner_tol;        /* FGMRES relative tolerance, default 1e-8 */
  int32_t m2_inner_max;       /* FGMRES iteration cap, default 300 */
  int32_t m2_restart;         /* FGMRES restart length, default 60 */
  int32_t m3_max_cycles;      /* M3 time-stepping periods (SolverConfig::m3_max_cycles), default 10 */
  int32_t track_error_contraction; /* SolverConfig::track_error_contraction (solvers.hpp:66-68, 347-360):
                                 M1 archives its iterates (host memory) and reports K_hat-norm
                                 error ratios against the final iterate as contraction_history */
} tp_solver_cfg;

/* Mirrors SolveReport (solvers.hpp:88-96); residual/contraction histories are
 * written to caller buffers passed to tp_solve_m1. */
typedef struct tp_report {
  int32_t iterations;
  int32_t status;             /* tp_solve_status */
  int32_t history_len;        /* entries written (min(iterations+1, cap)) */
  int32_t inner_iterations;   /* total inner (frequency-block) iterations */
  double q_estimate;
  double wall_time;           /* seconds, like SolveReport::wall_time (incl. setup) */
  double setup_time;          /* solver-hierarchy build, seconds */
  double sweep_time;          /* sum of sweep times, seconds */
  int32_t contraction_len;    /* contraction_history entries written */
  int32_t pad_;
} tp_report;

/* Per-iterate callback (the iterate_log of solve_m1_fixed_point,
 * solvers.hpp:306,317-319,366).  U is a HOST copy (N x n) valid during the call,
 * or NULL when the caller asked for norms only. Return nonzero to abort. */
typedef int (*tp_iterate_cb)(int32_t iterate, const double* U, double residual, void* user);

typedef struct tp_problem tp_problem;

/* ---- library ---------------------------------------------------------- */
int tp_version(void);
/* Message of the last error on this thread; *achieved = SolveError::residual(). */
int tp_last_error(char* buf, size_t cap, double* achieved);
void tp_solver_cfg_default(tp_solver_cfg* cfg);
/* BASELINE.json configs 0..4; 5 = config 4's linear control (nu == nu0). */
int tp_problem_desc_baseline(int32_t config, tp_problem_desc* desc);

/* ---- setup (mesh, materials, sources; runner.hpp:46-73 up to static_init) */
/* Grid sizes: K(u), the residual and the time transforms take any cells >= 2
 * and any N >= 1; the solvers (tp_static_init, tp_periodic_solve, tp_solve_*)
 * build a geometric hierarchy and need cells = 2^k * q with q <= 8
 * (TP_EINVAL otherwise; every BASELINE configuration is a power of two). */
int tp_problem_create(const tp_problem_desc* desc, int32_t device, tp_problem** out);
void tp_problem_destroy(tp_problem* p);
/* n_dof: dofs held by this problem (all free dofs; a sharded rank: its strip). */
int tp_problem_sizes(const tp_problem* p, int32_t* n_dof, int32_t* steps, double* tau);
/* assemble_loads (assembly.hpp:88-106): F, N x n */
int tp_problem_loads(tp_problem* p, double* F);
/* lumped mass diagonal, n */
int tp_problem_mass(tp_problem* p, double* m_diag);

/* ---- Problem concept (periodic.hpp:23-31) ------------------------------ */
/* NonlinearOperator::apply (assembly.hpp:126-140) on `count` slices. */
int tp_apply_k(tp_problem* p, const double* U, double* KU, int32_t count);
/* residual (periodic.hpp:35-58): R = F - A(U), N x n; returns ||R|| (block_l2). */
int tp_residual(tp_problem* p, const double* U, double* R, double* norm);

/* ---- methods ----------------------------------------------------------- */
/* static_init (solvers.hpp:276-296): U0 (N x n, may be NULL: kept on device as
 * the current state), newton_counts (N, may be NULL). */
int tp_static_init(tp_problem* p, const tp_solver_cfg* cfg, double* U0, int32_t* newton_counts);
/* current device state <-> host */
int tp_set_state(tp_problem* p, const double* U);
int tp_get_state(tp_problem* p, double* U);
/* choose_nu_hat + flux_bounds (assembly.hpp:254-303, materials.hpp:112-155)
 * over the current device state; installs K_hat.  nu_hat[TP_MAX_MATERIALS]. */
int tp_choose_nu_hat(tp_problem* p, const tp_solver_cfg* cfg, double* nu_hat, double* q);
/* install an explicit per-material nu_hat (assemble_stiffness_frozen, assembly.hpp:68-84) */
int tp_set_nu_hat(tp_problem* p, const double* nu_hat, double q);
/* PeriodicSolver::solve (periodic.hpp:154-198) with the installed M, K_hat:
 * G -> U, both N x n host. */
int tp_periodic_solve(tp_problem* p, const tp_solver_cfg* cfg, const double* G, double* U);
/* solve_m1_fixed_point (solvers.hpp:301-369).  U0 == NULL: start from the
 * current device state.  U_out may be NULL.  history/cap: residual_history;
 * contraction (may be NULL, cap entries): contraction_history. */
int tp_solve_m1(tp_problem* p, const tp_solver_cfg* cfg, const double* U0, double* U_out,
                tp_report* report, double* history, double* contraction, int32_t cap,
                tp_iterate_cb cb, void* user);

/* M2 all-at-once Newton: FGMRES right-preconditioned by the periodic solver on
 * the time-averaged Jacobian, Armijo line search (solve_m2_newton,
 * solvers.hpp:375-484).  Single-GPU problems.  Same outputs as tp_solve_m1
 * (q_estimate is NaN; inner_iterations = total FGMRES iterations). */
int tp_solve_m2(tp_problem* p, const tp_solver_cfg* cfg, const double* U0, double* U_out, tp_report* rep,
                double* history, double* contraction, int32_t cap);

/* M3 sequential time stepping toward the limit cycle: implicit Euler period
 * after period from U0, per-step damped Newton (solve_m3_timestepping,
 * solvers.hpp:489-542; newton_elliptic with mass_scale 1/tau).  Single GPU.
 * iterations = completed periods. */
int tp_solve_m3(tp_problem* p, const tp_solver_cfg* cfg, const double* U0, double* U_out, tp_report* rep,
                double* history, double* contraction, int32_t cap);

/* ---- device-resident sweep (benchmark / driver building blocks) -------- */
/* Builds the frequency solver (PeriodicSolver ctor, periodic.hpp:128-139) and
 * evaluates the initial residual of the current state (solvers.hpp:320-321). */
int tp_m1_begin(tp_problem* p, const tp_solver_cfg* cfg, double* residual0);
/* One fixed-point sweep (solvers.hpp:326-341) on the device state; returns
 * ||R|| of the new iterate and the inner iteration count of the sweep. */
int tp_m1_sweep(tp_problem* p, double* residual, int32_t* inner_iterations);
/* Inner-solve work of the last periodic solve (sweep): the largest iteration
 * count of any frequency block and the sum over blocks of their iteration
 * counts (the bench's algorithmic-byte count). */
int tp_sweep_stats(const tp_problem* p, int32_t* max_iterations, int64_t* frequency_iterations);
/* Achieved frequency-block residuals of the last periodic solve (the
 * reference's SparseSolver residual contract, solve.hpp:54,79-89): the
 * largest ||r_k|| / max(||g_k||, ||g|| / sqrt(K)) -- the stopping reference
 * the device enforces (<= inner_rtol; a batch that ends above 1e-10 of it
 * raises TP_ESOLVE) -- and the largest ||r_k|| / ||g_k|| against the block's
 * own right-hand side, the reference's per-solve measure.  The two differ
 * only for blocks whose right-hand side is below their equal share of the
 * spectrum (round-off-sized even harmonics), which stop at the share
 * (DESIGN.md §5). */
int tp_solve_residuals(const tp_problem* p, double* max_rel_floored, double* max_rel_own);
/* ---- multi-GPU (one process per GPU, NCCL over NVLink) ---------------
 * Partition of a sharded problem: node-row strip [row0,row1)
 * for K(u)/residual/RHS/DFT (all N slices local), frequency block
 * [freq0,freq1) for the block solves (full grid), slice block [slice0,slice1)
 * for the static initialisation.  Host state arrays of a sharded problem
 * (tp_set_state, tp_get_state, tp_static_init, tp_solve_m1, tp_periodic_solve)
 * are the rank's strip: N x n_local, slice-major. */
typedef struct tp_shard_plan {
  int32_t nranks, rank;
  int32_t row0, row1;
  int32_t freq0, freq1;
  int32_t slice0, slice1;
  int32_t n_local;
} tp_shard_plan;

typedef struct tp_comm tp_comm;

/* Pure host function (no GPU): the partition every rank computes.  freq0/freq1
 * are SLOTS of the half spectrum: frequencies are dealt to the ranks in snake
 * order and stored so that each rank's are contiguous;
 * tp_shard_freq_order gives the frequency held by every slot (N/2+1 entries;
 * the identity for one rank). */
int tp_shard_plan_make(int32_t cells, int32_t steps, int32_t nranks, int32_t rank, tp_shard_plan* out);
int tp_shard_freq_order(int32_t cells, int32_t steps, int32_t nranks, int32_t* slot_to_freq);
/* ncclGetUniqueId on one rank; the caller broadcasts the 128 bytes. */
int tp_nccl_unique_id(unsigned char id[128]);
int tp_comm_create(const unsigned char id[128], int32_t nranks, int32_t rank, int32_t device, tp_comm** out);
/* Host-staged transport (no NCCL): every exchange of the sharded sweep is
 * staged through pinned host memory and handed to `fn`, which must deliver
 * send_buf[i] (send_bytes[i]) to rank send_peer[i] and fill recv_buf[i]
 * (recv_bytes[i]) with what rank recv_peer[i] sent this rank in the same
 * call (peers never equal this rank; transfers to self stay on the device).
 * Returns 0 on success.  For ranks sharing one GPU (tests) or hosts without
 * NVLink; the stream is drained before each call, so no kernel ever waits on
 * another process. */
typedef int (*tp_host_exchange_fn)(void* user, int32_t nsend, const int32_t* send_peer,
                                   const void* const* send_buf, const size_t* send_bytes, int32_t nrecv,
                                   const int32_t* recv_peer, void* const* recv_buf, const size_t* recv_bytes);
int tp_comm_create_host(int32_t nranks, int32_t rank, int32_t device, tp_host_exchange_fn fn, void* user,
                        tp_comm** out);
void tp_comm_destroy(tp_comm* c);
void* tp_comm_nccl(tp_comm* c);
int32_t tp_comm_rank(const tp_comm* c);
int32_t tp_comm_size(const tp_comm* c);
int32_t tp_comm_device(const tp_comm* c);
int tp_problem_create_sharded(const tp_problem_desc* desc, tp_comm* comm, tp_problem** out);
int tp_problem_shard(const tp_problem* p, tp_shard_plan* out);

/* Live timing of one fine-level kernel (tp_kernel_timer_select) with CUDA
 * events: returns the launches / event time / algorithmic bytes accumulated
 * since the previous call, then enables (1) or disables (0) the timer. */
int tp_kernel_timer(tp_problem* p, int32_t enable, int64_t* launches, double* ms, double* bytes);
/* Which fine-level pass tp_kernel_timer brackets: 0 the up pass (default),
 * 1 the down pass (with the fused Krylov update), 2 the COCG apply. */
int tp_kernel_timer_select(tp_problem* p, int32_t which);
/* CUDA stream the problem launches on (cudaStream_t), for event timing. */
void* tp_problem_stream(tp_problem* p);
/* Kernel launches issued so far by this problem (for the bench's gpu_launches). */
int64_t tp_problem_launches(const tp_problem* p);

#ifdef __cplusplus
}
#endif

#endif /* TPGPU_H */
