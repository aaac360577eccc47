// Internal declarations of the B200 fixed-point-sweep library (libtpgpu.so).
// See DESIGN.md for the data layout and the kernel inventory.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <thread>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/tpgpu.h"

// One rank's transport for the sharded sweep (shard.cu): an NCCL
// communicator, or the host-staged exchange of tp_comm_create_host.
struct tp_comm {
  enum class Kind { Nccl, Host } kind = Kind::Nccl;
  void* comm = nullptr;  // ncclComm_t
  int nranks = 1, rank = 0, device = 0;
  tp_host_exchange_fn host_fn = nullptr;
  void* host_user = nullptr;
  void* host_buf = nullptr;  // pinned staging
  size_t host_cap = 0;
};

namespace tpgpu {

// ---------------------------------------------------------------- errors
struct Error : std::runtime_error {
  int code;
  double residual;
  Error(int c, const std::string& m, double r = -1.0) : std::runtime_error(m), code(c), residual(r) {}
};

[[noreturn]] void throw_cuda(cudaError_t e, const char* what, const char* file, int line);
#define TP_CUDA(x)                                                   \
  do {                                                               \
    cudaError_t tp_e_ = (x);                                         \
    if (tp_e_ != cudaSuccess) ::tpgpu::throw_cuda(tp_e_, #x, __FILE__, __LINE__); \
  } while (0)
#define TP_LAUNCHED(p)                                               \
  do {                                                               \
    ++(p)->launches;                                                 \
    cudaError_t tp_e_ = cudaGetLastError();                          \
    if (tp_e_ != cudaSuccess) ::tpgpu::throw_cuda(tp_e_, "kernel launch", __FILE__, __LINE__); \
  } while (0)

void set_last_error(const std::string& msg, double residual);
void validate_cfg(const tp_solver_cfg& c);  // validate(), solvers.hpp:71-86

// contraction_history from residual norms (solvers.hpp:361-365): the ratio
// r_{k+1} / r_k for every k with r_k > 0 (zero residuals are skipped, not
// zero-filled); returns the entries written (at most cap).
inline int residual_contraction(const std::vector<double>& hist, double* out, int cap) {
  int w = 0;
  for (size_t k = 0; k + 1 < hist.size() && w < cap; ++k)
    if (hist[k] > 0) {
      if (out) out[w] = hist[k + 1] / hist[k];
      ++w;
    }
  return w;
}

// ---------------------------------------------------------------- PDL
// Programmatic dependent launch for the kernel chains of the frequency solves
// (one stream per frequency group, ~9 dependent kernels per inner iteration):
// a kernel launched by launch_pdl may be scheduled while its predecessor
// drains; it waits in TP_PDL_ENTRY (griddepcontrol.wait: every prerequisite
// grid complete and its memory visible) before touching memory, and at once
// allows its own dependents to launch.  Every kernel launched through
// launch_pdl must start with TP_PDL_ENTRY (a no-op under a normal launch).
// TPGPU_PDL=0 launches normally.
#ifndef TPGPU_PDL_TRIGGER
#define TPGPU_PDL_TRIGGER 0
#endif
#define TP_PDL_ENTRY()                                               \
  do {                                                               \
    asm volatile("griddepcontrol.wait;\n" ::: "memory");            \
    if (TPGPU_PDL_TRIGGER) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); \
  } while (0)
bool pdl_enabled();

// Experiment: stream-event trace of one host thread's launches (TPGPU_TRACE=1;
// problem.cu prints the live time between consecutive marks per group)
struct StreamTrace {
  std::vector<std::pair<const char*, cudaEvent_t>> ev;
};
extern thread_local StreamTrace* tl_trace;
void trace_report(StreamTrace& trace, const std::string& label, cudaStream_t s);
inline void trace_mark(const char* name, cudaStream_t s) {
  if (!tl_trace) return;
  cudaEvent_t e;
  TP_CUDA(cudaEventCreate(&e));
  TP_CUDA(cudaEventRecord(e, s));
  tl_trace->ev.emplace_back(name, e);
}
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cudaLaunchConfig_t c = {};
  c.gridDim = grid;
  c.blockDim = block;
  c.dynamicSmemBytes = smem;
  c.stream = s;
  c.attrs = at;
  c.numAttrs = 1;
  TP_CUDA(cudaLaunchKernelEx(&c, kern, static_cast<KArgs>(args)...));
}

inline void require(bool ok, const std::string& msg) {
  if (!ok) throw Error(TP_EINVAL, msg);
}

// ---------------------------------------------------------------- complex
struct __align__(16) cplx {
  double re, im;
};
__host__ __device__ inline cplx mk(double r, double i) { return cplx{r, i}; }
__host__ __device__ inline cplx operator+(cplx a, cplx b) { return {a.re + b.re, a.im + b.im}; }
__host__ __device__ inline cplx operator-(cplx a, cplx b) { return {a.re - b.re, a.im - b.im}; }
__host__ __device__ inline cplx operator*(cplx a, cplx b) {
  return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}
__host__ __device__ inline cplx operator*(double s, cplx a) { return {s * a.re, s * a.im}; }
__host__ __device__ inline cplx conj(cplx a) { return {a.re, -a.im}; }
__host__ __device__ inline double norm2(cplx a) { return a.re * a.re + a.im * a.im; }
__host__ __device__ inline double norm2(double a) { return a * a; }
__host__ __device__ inline cplx cdiv(cplx a, cplx b) {
  const double d = b.re * b.re + b.im * b.im;
  return {(a.re * b.re + a.im * b.im) / d, (a.im * b.re - a.re * b.im) / d};
}
__host__ __device__ inline double cdiv(double a, double b) { return a / b; }

// ---------------------------------------------------------------- device buffers
template <class T>
struct DevBuf {
  T* ptr = nullptr;
  size_t count = 0;
  bool owned = true;  // false: a view into another buffer (alias)
  DevBuf() = default;
  explicit DevBuf(size_t n) { alloc(n); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : ptr(o.ptr), count(o.count), owned(o.owned) { o.ptr = nullptr; o.count = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); ptr = o.ptr; count = o.count; owned = o.owned; o.ptr = nullptr; o.count = 0; }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t n) {
    release();
    if (n) TP_CUDA(cudaMalloc(reinterpret_cast<void**>(&ptr), n * sizeof(T)));
    count = n;
    owned = true;
  }
  void alias(T* p, size_t n) {
    release();
    ptr = p;
    count = n;
    owned = false;
  }
  void ensure(size_t n) { if (count < n) alloc(n); }
  void release() {
    if (ptr && owned) cudaFree(ptr);
    ptr = nullptr;
    count = 0;
    owned = true;
  }
  T* get() const { return ptr; }
  size_t bytes() const { return count * sizeof(T); }
};

// ---------------------------------------------------------------- grid
// Interior node (x, y), 0 <= x, y < m = cells-1, index y*m + x; it is vertex
// (x+1, y+1) of the (cells+1)^2 vertex lattice.  Cell (i, j) has triangles
// T1 = {v(i,j), v(i+1,j), v(i+1,j+1)} and T2 = {v(i,j), v(i+1,j+1), v(i,j+1)}.
// 7-point stencils are stored SoA: st[d*n + i], d in the order below.
enum StencilDir { SC = 0, SW_ = 1, SE_ = 2, SS_ = 3, SN_ = 4, SSW = 5, SNE = 6 };
constexpr int kDirs = 7;
__host__ __device__ constexpr int dir_dx(int d) { return d == 1 ? -1 : d == 2 ? 1 : d == 5 ? -1 : d == 6 ? 1 : 0; }
__host__ __device__ constexpr int dir_dy(int d) { return d == 3 ? -1 : d == 4 ? 1 : d == 5 ? -1 : d == 6 ? 1 : 0; }

struct MaterialDev {
  double nu0, nu_inf, bs2;  // bs2 = Bs^2
  int linear;
};

// ---------------------------------------------------------------- multigrid
// One level of the geometric hierarchy (P1 interpolation on the nested
// triangulation, Galerkin coarse operators).
struct Level {
  int m = 0;          // interior nodes per side
  int n = 0;          // m*m
  DevBuf<double> K;   // 7*n real stencil (frequency mode: shared)
  DevBuf<double> M;   // 7*n real stencil (frequency mode: shared)
};

class Problem;

// Batched multigrid-preconditioned conjugate-gradient solver.  Frequency mode
// (T = cplx): operator lambda_b M + K with shared real stencils, COCG (complex
// symmetric, bilinear form).  Slice mode (T = double): per-batch real SPD
// stencils (Newton Jacobians), PCG.
struct SolveStats {
  int iterations = 0;
  int64_t batch_iterations = 0;
  double max_rel_residual = 0;      // ||r_k|| / max(||g_k||, ||g|| / sqrt(K)): the enforced stopping reference
  double max_rel_residual_own = 0;  // ||r_k|| / ||g_k||: the reference SparseSolver's per-solve measure
};

// ---------------------------------------------------------------- host workers
// Persistent helper threads that drive concurrent frequency groups (each
// group's kernels go to its own stream; the host thread of a group waits on
// its own convergence counters).  run(f) calls f(0) on the caller and f(g),
// g = 1..n, on the helpers, and returns when all have finished: no thread is
// created per sweep.
class WorkerPool {
 public:
  explicit WorkerPool(int helpers) {
    for (int g = 1; g <= helpers; ++g) th_.emplace_back([this, g] { loop(g); });
  }
  ~WorkerPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int helpers() const { return (int)th_.size(); }
  void run(const std::function<void(int)>& f) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = &f;
      pending_ = (int)th_.size();
      ++gen_;
    }
    cv_.notify_all();
    f(0);
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [this] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  void loop(int g) {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int)>* job;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
        job = job_;
      }
      (*job)(g);  // f catches its own exceptions (problem.cu)
      {
        std::lock_guard<std::mutex> lk(mu_);
        --pending_;
      }
      done_cv_.notify_one();
    }
  }
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* job_ = nullptr;
  int pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// ---------------------------------------------------------------- sharding
// One rank of a multi-GPU problem: node-row strip [y0, y1)
// for the operator / residual / DFT stages (all N slices local), frequency
// block [k0, k1) for the solves (full grid), slice block [s0, s1) for the
// static initialisation (full grid).  P == 1 is the single-GPU problem.
struct ShardInfo {
  int P = 1, r = 0;
  int y0 = 0, y1 = 0;
  int k0 = 0, k1 = 0;
  int s0 = 0, s1 = 0;
  int nr = 0;  // local dofs (y1-y0)*m
  std::vector<int> ys, ks, ss;  // partition points, P+1 each (ks: frequency slots)
  std::vector<int> kperm;       // slot -> frequency (empty: identity, P == 1)
  tp_comm* comm = nullptr;      // NCCL or host-staged transport (shard.cu)
};
void make_partition(int m, int K, int N, int P, int r, ShardInfo& sh);

// ---------------------------------------------------------------- problem
class Problem {
 public:
  Problem(const tp_problem_desc& d, int device, const ShardInfo* shard = nullptr);
  ~Problem();

  // host setup products
  tp_problem_desc desc;
  int device = 0;
  int c = 0, m = 0, n = 0, N = 0, K = 0;  // cells, nodes/side, dofs, steps, frequencies N/2+1
  double tau = 0, T = 0;
  std::vector<uint8_t> cell_mat;      // c*c
  std::vector<double> tri_sigma;      // 2*c*c
  std::vector<double> mass;           // n (lumped)
  std::vector<int> src_mats;          // materials with sources
  std::vector<double> src_prof;       // nsrc * n  (int j(t)=1 phi_i over the material)
  std::vector<double> src_time;       // N * nsrc  (j_r(t_n))
  std::vector<double> nu_hat;         // TP_MAX_MATERIALS
  double q_estimate = 0;
  bool nu_hat_set = false;

  // device constants
  cudaStream_t stream = nullptr;
  // stream the calling host thread launches on: the problem's stream, or the
  // per-thread override of a concurrently driven frequency half (problem.cu)
  static thread_local cudaStream_t tl_stream;
  cudaStream_t cur_stream() const { return tl_stream ? tl_stream : stream; }
  std::atomic<int64_t> launches{0};
  tp_solver_cfg sweep_cfg{};  // the configuration tp_m1_begin set up the sweeps with
  int num_sms = 148;
  DevBuf<uint8_t> d_cell_mat;
  DevBuf<double> d_mass;
  DevBuf<double> d_src_prof;
  DevBuf<double> d_src_time;
  DevBuf<MaterialDev> d_mat;
  DevBuf<double> d_nu_hat;
  DevBuf<uint8_t> d_rflags;  // region flags of the row-walking sweep kernel (op_kernels.cu)
  int rflags_key = -1;       // the row-chunk height they were built for
  DevBuf<double> d_coef;      // [we | wn | mass] of the fine streaming kernels (one L2-persisting block)
  DevBuf<double> d_we, d_wn;  // K_hat edge weights on the (c+1)^2 vertex grid (views into d_coef)
  void l2_persist(const void* base, size_t bytes, const std::vector<cudaStream_t>& ss);
  // device state
  DevBuf<double> U;     // N*n current iterate (slice-major)
  DevBuf<double> G;     // N*n right-hand side of the next sweep
  DevBuf<cplx> Ghat;    // K*n  (frequency-major)
  DevBuf<cplx> Uhat;    // K*n  (frequency-major)
  DevBuf<double> part;  // reduction partials
  DevBuf<double> red;   // reduced scalars
  bool state_valid = false;
  bool uhat_valid = false;

  // frequency-solver hierarchy
  std::vector<Level> levels;
  bool freq_ready = false;
  int freq_chunk = 0;
  struct FreqWork;
  std::unique_ptr<FreqWork> fw;

  std::shared_ptr<void> fft_plan;

  // multi-GPU (P > 1): partition, halo rows, frequency-block spectra
  ShardInfo sh;
  bool sharded() const { return sh.comm != nullptr; }
  DevBuf<double> halo_lo, halo_hi, halo_send;  // N*m each
  DevBuf<cplx> Ghat_f, Uhat_f, xstage;         // (k1-k0)*n frequency blocks, staging
  DevBuf<double> red_all;                      // P doubles (allgather)
  DevBuf<int> d_kslot;                         // frequency -> spectrum slot (sharded; else none)
  int freq_of_slot(int s) const { return sh.kperm.empty() ? s : sh.kperm[s]; }
  DevBuf<cplx> uhat_prev;  // warm-start extrapolation: the spectrum of the sweep before
  bool uhat_prev_valid = false;
  double extrap_theta = 0.0;  // > 0: the next periodic_solve_with extrapolates its warm start
  double resid_prev = -1.0, resid_last = -1.0;  // the last two M1 residual norms
  DevBuf<double> spec_sq;  // forward-DFT |X|^2 partials, then [last] the total (frequency stopping floor)
  void exchange_halo();
  double global_sum(double local);
  void global_sum_dev(const double* d_in, int count, double* d_out);  // no host round trip
  void global_minmax(double* lo, double* hi, int count);
  double global_max(double v) {
    double lo = v, hi = v;
    global_minmax(&lo, &hi, 1);
    return hi;
  }
  void global_sum_ints(std::vector<int>& v);
  void alltoall_to_freq(const cplx* src = nullptr, cplx* dst = nullptr);  // Ghat (K x nr) -> Ghat_f ((k1-k0) x n)
  // warm start of the first sweep's frequency solves: the spectrum of the
  // current state U (its frequency blocks) as the initial guess
  void seed_spectrum();
  void alltoall_from_freq();  // Uhat_f -> Uhat (K x nr)
  void slices_to_strips(const double* Us);  // static-init slices (full grid) -> U strips
  cplx* spec_in() { return sharded() ? Ghat_f.get() : Ghat.get(); }
  cplx* spec_out() { return sharded() ? Uhat_f.get() : Uhat.get(); }

  // live kernel timing for bench.py's roofline (enabled on request): the
  // dominant kernel (fine-level V-cycle up pass) is bracketed by CUDA events
  struct KernelTimer {
    std::mutex mu;
    bool on = false;
    int which = 0;  // tp_kernel_timer_select: 0 fine up pass, 1 fine down pass, 2 fine apply
    int64_t launches = 0;
    double bytes = 0, ms = 0;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;
    void drain();
    // bracket one launch of kernel `kind` on stream s (alg_bytes: its algorithmic bytes)
    template <class F>
    void time(int kind, cudaStream_t s, double alg_bytes, F&& launch) {
      if (!on || kind != which) {
        launch();
        return;
      }
      cudaEvent_t e0 = nullptr, e1 = nullptr;
      TP_CUDA(cudaEventCreate(&e0));
      TP_CUDA(cudaEventCreate(&e1));
      TP_CUDA(cudaEventRecord(e0, s));
      launch();
      TP_CUDA(cudaEventRecord(e1, s));
      std::lock_guard<std::mutex> lk(mu);
      pending.emplace_back(e0, e1);
      bytes += alg_bytes;
      ++launches;
    }
  } ktimer;

  // pinned host scratch
  double* h_scalars = nullptr;  // pinned, 4096 doubles

  // ---- operations (defined across the .cu files)
  void upload_constants();
  void install_nu_hat(const double* nu, double q);
  void build_frequency_solver(const tp_solver_cfg& cfg);
  void build_freq_work(std::vector<Level>& lv, std::unique_ptr<FreqWork>& out, const double* K0,
                       const tp_solver_cfg& cfg, int want_groups);
  void periodic_solve_with(FreqWork& w, const double* in, double* out, bool warm, const tp_solver_cfg& cfg,
                           SolveStats* st);
  // a periodic solver for lambda_k M + K0 (K0: fine 7-point stencil, device)
  // as an opaque handle, and its application in -> out (cold start)
  std::shared_ptr<void> make_periodic_precond(const double* K0, const tp_solver_cfg& cfg);
  void precond_solve(void* handle, const double* in, double* out, const tp_solver_cfg& cfg);
  // K(u) for `count` slices of `u` into `out` (device pointers)
  void apply_k_dev(const double* u, double* out, int count);
  // fused residual + next RHS over the device state: returns ||R||
  double residual_and_rhs(bool want_rhs);
  // residual only (host-facing)
  void residual_dev(const double* u, double* r, int count_slices);
  // periodic linear solve of the device G into the device U
  void periodic_solve_dev(const tp_solver_cfg& cfg, SolveStats* st);
  void static_init_dev(const tp_solver_cfg& cfg, int32_t* newton_counts);
  // M2 all-at-once Newton (m2.cu) from the device state U
  struct M2Result {
    int iterations = 0, status = 0;
    int64_t inner_total = 0;
    std::vector<double> history;
  };
  void solve_m2_dev(const tp_solver_cfg& cfg, M2Result& res);
  void solve_m3_dev(const tp_solver_cfg& cfg, M2Result& res);  // M3 time stepping (m3.cu)
  void field_ranges(double* lo, double* hi, int* any);
  // block_norm_khat(a - b) (periodic.hpp:70-75) over the N slices, device arrays
  double khat_norm_diff(const double* a, const double* b);
  int last_inner = 0;
  int64_t last_freq_iters = 0;  // sum over frequency blocks of the last periodic solve
  double last_rel_floored = 0, last_rel_own = 0;  // achieved block residuals of the last periodic solve
};

// kernels / helpers implemented in the .cu files
// sq (optional): per-block partial sums of |X|^2 over the half spectrum written
// (rdft_forward_blocks(p) of them)
void launch_rdft_forward(Problem& p, const double* G, cplx* Ghat, double* sq = nullptr);
int rdft_forward_blocks(Problem& p);
// returns imaginary-residue norm^2 partial sum and real norm^2 (host)
void launch_rdft_inverse(Problem& p, const cplx* Uhat, double* U, double* re2, double* im2);
double reduce_sum(Problem& p, const double* partials, int count);
// The same real time-DFTs over any slice-major N x n array (general-mesh
// problems, mesh.cu): plan slot, reduction scratch and pinned scalars of the owner
struct DftCtx {
  int N;
  size_t n;
  cudaStream_t stream;
  std::shared_ptr<void>* plan;
  DevBuf<double>* part;
  DevBuf<double>* red;
  double* h_scalars;
  std::atomic<int64_t>* launches;
  const int* kslot = nullptr;  // frequency k -> row of the half spectrum (nullptr: k)
};
int dft_forward_blocks(const DftCtx& c);
void dft_forward(const DftCtx& c, const double* G, cplx* Ghat, double* sq = nullptr);
void dft_inverse(const DftCtx& c, const cplx* Uhat, double* U, double* re2, double* im2);
void reduce_sum_dev(Problem& p, const double* partials, int count, double* out);  // no host sync

}  // namespace tpgpu
