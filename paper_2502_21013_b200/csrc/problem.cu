// Host side of libtpgpu.so: problem setup (mesh, materials, sources), the
// frequency-solver hierarchy, the M1 fixed-point driver and the C ABI.
//
// Host code mirrors the reference's control flow line by line where it is
// control flow (solve_m1_fixed_point, solvers.hpp:301-369; stopping_check,
// solvers.hpp:100-103; choose_nu_hat, assembly.hpp:254-303); all per-dof
// arithmetic runs in the CUDA kernels of op_kernels.cu / fft_kernels.cu /
// mg.cu / newton.cu.  There is no CPU fallback: a missing device is TP_ECUDA.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <map>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <numbers>
#include <thread>
#include <string>

#include "../../include/tpgpu_baseline.h"
#include "mg.cuh"

namespace tpgpu {

thread_local StreamTrace* tl_trace = nullptr;

void trace_report(StreamTrace& trace, const std::string& label, cudaStream_t s) {
  TP_CUDA(cudaStreamSynchronize(s));
  std::map<std::string, std::pair<int, double>> acc;
  for (size_t i = 0; i + 1 < trace.ev.size(); ++i) {
    float ms = 0;
    TP_CUDA(cudaEventElapsedTime(&ms, trace.ev[i].second, trace.ev[i + 1].second));
    auto& a = acc[trace.ev[i].first];
    a.first += 1;
    a.second += ms;
  }
  std::string line = label + ":";
  for (auto& [k, v] : acc)
    line += " " + k + " " + std::to_string(v.first) + "x " + std::to_string(v.second * 1e3).substr(0, 7) + "us";
  std::fprintf(stderr, "%s\n", line.c_str());
  for (auto& e : trace.ev) cudaEventDestroy(e.second);
  trace.ev.clear();
}

bool pdl_enabled() {
  static const bool on = !std::getenv("TPGPU_PDL") || std::atoi(std::getenv("TPGPU_PDL")) != 0;
  return on;
}

[[noreturn]] void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
  throw Error(TP_ECUDA, std::string("CUDA error ") + cudaGetErrorName(e) + " (" +
                            cudaGetErrorString(e) + ") at " + file + ":" + std::to_string(line) +
                            ": " + what);
}

namespace {

uint64_t splitmix64(uint64_t& state) {
  uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

void validate_desc(const tp_problem_desc& d) {
  require(d.cells >= 2, "problem: need at least 2 cells per side");
  require(d.steps >= 1, "problem: need at least one time step");
  require(d.period > 0, "problem: period must be positive");
  require(d.n_materials >= 1 && d.n_materials <= TP_MAX_MATERIALS, "problem: material count out of range");
  require(d.n_rects >= 0 && d.n_rects <= TP_MAX_RECTS, "problem: rectangle count out of range");
  for (int r = 0; r < d.n_rects; ++r)
    require(d.rect[r].material >= 0 && d.rect[r].material < d.n_materials,
            "problem: rectangle material out of range");
  for (int k = 0; k < d.n_materials; ++k) {
    const tp_material& mt = d.material[k];
    require(mt.sigma >= 0, "problem: sigma must be >= 0");
    require(mt.nu0 > 0 && mt.nu_inf > 0, "problem: nu must be > 0");
    require(mt.nu0 == mt.nu_inf || mt.bs > 0, "problem: Bs must be > 0");
    require(mt.n_harmonics >= 0 && mt.n_harmonics <= TP_MAX_HARMONICS, "problem: harmonic count out of range");
  }
}

}  // namespace

void validate_cfg(const tp_solver_cfg& c) {
  // validate(), solvers.hpp:71-86 (fields on this path)
  require(c.tol > 0 && c.tol < 1, "solver config: tol must lie in (0,1)");
  require(c.armijo_slope > 0 && c.armijo_slope < 1, "solver config: armijo slope must lie in (0,1)");
  require(c.armijo_backtrack > 0 && c.armijo_backtrack < 1,
          "solver config: armijo backtracking factor must lie in (0,1)");
  require(c.armijo_max_halvings >= 0, "solver config: negative armijo halving cap");
  require(c.m1_max_outer >= 1 && c.static_max_newton >= 1, "solver config: iteration caps must be positive");
  require(c.static_tol > 0 && c.static_tol < 1, "solver config: inner tolerances must lie in (0,1)");
  require(c.inner_rtol > 0 && c.inner_rtol < 1e-6, "solver config: inner_rtol must lie in (0,1e-6)");
  require(c.inner_max_iter >= 1, "solver config: inner_max_iter must be positive");
}

namespace {

// nu(s) and nu'(s) on the host, for the flux-bound sampling (materials.hpp:42-57 law swapped).
double h_nu(const tp_material& m, double s) {
  if (m.nu0 == m.nu_inf) return m.nu0;
  const double s2 = s * s;
  return m.nu0 + (m.nu_inf - m.nu0) * s2 / (s2 + m.bs * m.bs);
}
double h_nu_prime(const tp_material& m, double s) {
  if (m.nu0 == m.nu_inf) return 0;
  const double den = s * s + m.bs * m.bs;
  return 2.0 * (m.nu_inf - m.nu0) * s * m.bs * m.bs / (den * den);
}
// flux_jacobian_bounds, materials.hpp:112-128
void flux_bounds(const tp_material& m, double lo, double hi, int samples, double& lam, double& Lam) {
  require(lo >= 0 && hi >= lo, "flux bounds: need 0 <= s_lo <= s_hi");
  require(samples >= 2, "flux bounds: need at least 2 samples");
  lam = std::numeric_limits<double>::infinity();
  Lam = 0;
  for (int j = 0; j < samples; ++j) {
    const double s = lo + (hi - lo) * j / (samples - 1);
    const double nu = h_nu(m, s);
    const double gp = nu + h_nu_prime(m, s) * s;
    lam = std::min({lam, nu, gp});
    Lam = std::max({Lam, nu, gp});
  }
}

}  // namespace

// Frequency-solver workspace.  With parts > 1, a chunk's frequencies are
// split into `parts` groups solved by independent batch solvers on their own
// streams, each driven by its own host thread: the latency-bound coarse part
// of one group's V-cycle overlaps the bandwidth-bound fine passes of another.
struct Problem::FreqWork {
  DevBuf<cplx> lam;       // K symbols
  DevBuf<cplx> inv;       // K * nL^2 coarsest inverses
  BatchSolver<0> solver;  // group 0 (and the only one when parts == 1)
  std::vector<std::unique_ptr<BatchSolver<0>>> extra;  // groups 1 .. parts-1
  int parts = 1;
  std::vector<cudaStream_t> hs;
  cudaEvent_t ev_in = nullptr;
  std::vector<cudaEvent_t> ev_out;
  int chunk = 0;  // frequencies per group
  int nL = 0;
  int req_chunk = 0, req_groups = 0;  // the configuration it was built for
  std::unique_ptr<WorkerPool> pool;  // parts - 1 persistent helper threads
  BatchSolver<0>& group(int g) { return g == 0 ? solver : *extra[g - 1]; }
  ~FreqWork() {
    pool.reset();
    for (auto& e : ev_out)
      if (e) cudaEventDestroy(e);
    if (ev_in) cudaEventDestroy(ev_in);
    for (auto& h : hs)
      if (h) cudaStreamDestroy(h);
  }
};

thread_local cudaStream_t Problem::tl_stream = nullptr;

Problem::Problem(const tp_problem_desc& d, int dev, const ShardInfo* shard) : desc(d), device(dev) {
  validate_desc(d);
  int count = 0;
  TP_CUDA(cudaGetDeviceCount(&count));
  require(dev >= 0 && dev < count, "problem: CUDA device index out of range");
  TP_CUDA(cudaSetDevice(dev));
  TP_CUDA(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
  TP_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  TP_CUDA(cudaMallocHost(reinterpret_cast<void**>(&h_scalars), 4096 * sizeof(double)));
  c = d.cells;
  m = c - 1;
  n = m * m;
  N = d.steps;
  K = N / 2 + 1;
  T = d.period;
  tau = T / N;
  // cell materials: painter's order by cell centroid (mesh.hpp:164-177)
  cell_mat.assign((size_t)c * c, 0);
  for (int j = 0; j < c; ++j)
    for (int i = 0; i < c; ++i) {
      const double cx = (2.0 * i + 1.0) / (2.0 * c), cy = (2.0 * j + 1.0) / (2.0 * c);
      int mat = 0;
      for (int r = 0; r < d.n_rects; ++r) {
        const tp_rect& R = d.rect[r];
        if (cx >= R.x0 && cx <= R.x1 && cy >= R.y0 && cy <= R.y1) mat = R.material;
      }
      cell_mat[(size_t)j * c + i] = (uint8_t)mat;
    }
  // per-triangle sigma with the seeded bilinear noise
  std::vector<double> lattice;
  const int L = d.noise_lattice >= 2 ? d.noise_lattice : 8;
  {
    uint64_t st = d.noise_seed;
    lattice.resize((size_t)L * L);
    const double lo = d.noise_lattice >= 2 ? d.noise_lo : 0.5, hi = d.noise_lattice >= 2 ? d.noise_hi : 1.5;
    for (int b = 0; b < L; ++b)
      for (int a = 0; a < L; ++a) {
        const double u = (double)(splitmix64(st) >> 11) * 0x1.0p-53;
        lattice[(size_t)b * L + a] = lo + (hi - lo) * u;
      }
  }
  auto noise = [&](double x, double y) {
    const double lo = d.noise_lattice >= 2 ? d.noise_lo : 0.5, hi = d.noise_lattice >= 2 ? d.noise_hi : 1.5;
    auto coord = [L](double p, double a, double b, int& i0, double& f) {
      double s = (p - a) / (b - a) * (L - 1);
      s = std::min(std::max(s, 0.0), (double)(L - 1));
      i0 = std::min((int)std::floor(s), L - 2);
      f = s - i0;
    };
    int a0, b0;
    double fx, fy;
    coord(x, d.noise_box[0], d.noise_box[2], a0, fx);
    coord(y, d.noise_box[1], d.noise_box[3], b0, fy);
    auto v = [&](int a, int b) { return lattice[(size_t)b * L + a]; };
    const double val = (1 - fx) * (1 - fy) * v(a0, b0) + fx * (1 - fy) * v(a0 + 1, b0) +
                       (1 - fx) * fy * v(a0, b0 + 1) + fx * fy * v(a0 + 1, b0 + 1);
    return std::min(std::max(val, lo), hi);
  };
  tri_sigma.assign((size_t)2 * c * c, 0.0);
  for (int j = 0; j < c; ++j)
    for (int i = 0; i < c; ++i) {
      const tp_material& mt = d.material[cell_mat[(size_t)j * c + i]];
      for (int t = 0; t < 2; ++t) {
        double s = mt.sigma;
        if (mt.sigma_noise) {
          const bool lower = t == 0;
          const double x = (3.0 * i + (lower ? 2.0 : 1.0)) / (3.0 * c);
          const double y = (3.0 * j + (lower ? 1.0 : 2.0)) / (3.0 * c);
          s = mt.sigma * noise(x, y);
        }
        tri_sigma[(size_t)2 * (j * c + i) + t] = s;
      }
    }
  // lumped mass and source profiles: sum over the six triangles of each node
  const double area = 0.5 / ((double)c * c);
  for (int r = 0; r < d.n_materials; ++r)
    if (d.material[r].n_harmonics > 0) src_mats.push_back(r);
  const int nsrc = (int)src_mats.size();
  mass.assign(n, 0.0);
  src_prof.assign((size_t)nsrc * n, 0.0);
  const int tcx[6] = {0, 0, -1, -1, -1, 0}, tcy[6] = {0, 0, 0, -1, -1, -1}, ttp[6] = {0, 1, 0, 0, 1, 1};
  for (int y = 0; y < m; ++y)
    for (int x = 0; x < m; ++x) {
      const size_t i = (size_t)y * m + x;
      for (int k = 0; k < 6; ++k) {
        const int ci = x + 1 + tcx[k], cj = y + 1 + tcy[k];
        const size_t cell = (size_t)cj * c + ci;
        mass[i] += tri_sigma[2 * cell + ttp[k]] * area / 3.0;
        for (int r = 0; r < nsrc; ++r)
          if (cell_mat[cell] == src_mats[r]) src_prof[(size_t)r * n + i] += area / 3.0;
      }
    }
  src_time.assign((size_t)N * std::max(nsrc, 1), 0.0);
  for (int s = 0; s < N; ++s) {
    const double t = (s + 1) * T / N;  // assembly.hpp:95
    for (int r = 0; r < nsrc; ++r) {
      const tp_material& mt = d.material[src_mats[r]];
      double j = 0;
      for (int h = 0; h < mt.n_harmonics; ++h)
        j += mt.amp[h] * std::sin(2.0 * std::numbers::pi * mt.harmonic[h] * t / T + mt.phase[h]);
      src_time[(size_t)s * nsrc + r] = j;
    }
  }
  nu_hat.assign(TP_MAX_MATERIALS, 1.0);
  upload_constants();
  if (shard) {
    sh = *shard;
  } else {
    make_partition(m, K, N, 1, 0, sh);
  }
  U.alloc((size_t)N * sh.nr);
  G.alloc((size_t)N * sh.nr);
  Ghat.alloc((size_t)K * sh.nr);
  Uhat.alloc((size_t)K * sh.nr);
  if (sharded()) {
    Ghat_f.alloc((size_t)(sh.k1 - sh.k0) * n);
    Uhat_f.alloc((size_t)(sh.k1 - sh.k0) * n);
    if (!sh.kperm.empty()) {
      std::vector<int> slot(K);
      for (int s2 = 0; s2 < K; ++s2) slot[sh.kperm[s2]] = s2;
      d_kslot.alloc(K);
      TP_CUDA(cudaMemcpy(d_kslot.get(), slot.data(), K * sizeof(int), cudaMemcpyHostToDevice));
    }
  }
  red.alloc(4096);
  TP_CUDA(cudaMemsetAsync(U.get(), 0, U.bytes(), stream));
}

void Problem::KernelTimer::drain() {
  for (auto& e : pending) {
    float t = 0;
    if (cudaEventSynchronize(e.second) == cudaSuccess && cudaEventElapsedTime(&t, e.first, e.second) == cudaSuccess)
      ms += t;
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  pending.clear();
}

Problem::~Problem() {
  ktimer.drain();
  fw.reset();
  if (h_scalars) cudaFreeHost(h_scalars);
  if (stream) cudaStreamDestroy(stream);
}

void Problem::upload_constants() {
  d_cell_mat.alloc(cell_mat.size());
  TP_CUDA(cudaMemcpy(d_cell_mat.get(), cell_mat.data(), cell_mat.size(), cudaMemcpyHostToDevice));
  d_mass.alloc(n);
  TP_CUDA(cudaMemcpy(d_mass.get(), mass.data(), n * sizeof(double), cudaMemcpyHostToDevice));
  d_src_prof.alloc(std::max<size_t>(src_prof.size(), 1));
  if (!src_prof.empty())
    TP_CUDA(cudaMemcpy(d_src_prof.get(), src_prof.data(), src_prof.size() * sizeof(double), cudaMemcpyHostToDevice));
  d_src_time.alloc(src_time.size());
  TP_CUDA(cudaMemcpy(d_src_time.get(), src_time.data(), src_time.size() * sizeof(double), cudaMemcpyHostToDevice));
  std::vector<MaterialDev> mt(TP_MAX_MATERIALS);
  for (int r = 0; r < TP_MAX_MATERIALS; ++r) {
    if (r < desc.n_materials) {
      const tp_material& x = desc.material[r];
      mt[r] = {x.nu0, x.nu_inf, x.bs * x.bs, x.nu0 == x.nu_inf ? 1 : 0};
    } else {
      mt[r] = {1.0, 1.0, 1.0, 1};
    }
  }
  d_mat.alloc(TP_MAX_MATERIALS);
  TP_CUDA(cudaMemcpy(d_mat.get(), mt.data(), mt.size() * sizeof(MaterialDev), cudaMemcpyHostToDevice));
  d_nu_hat.alloc(TP_MAX_MATERIALS);
  TP_CUDA(cudaMemcpy(d_nu_hat.get(), nu_hat.data(), TP_MAX_MATERIALS * sizeof(double), cudaMemcpyHostToDevice));
}

void Problem::install_nu_hat(const double* nu, double q) {
  for (int r = 0; r < TP_MAX_MATERIALS; ++r)
    require(nu[r] > 0, "frozen stiffness: nu_hat must be positive");  // assembly.hpp:70-71
  nu_hat.assign(nu, nu + TP_MAX_MATERIALS);
  q_estimate = q;
  TP_CUDA(cudaMemcpyAsync(d_nu_hat.get(), nu_hat.data(), TP_MAX_MATERIALS * sizeof(double),
                          cudaMemcpyHostToDevice, stream));
  TP_CUDA(cudaStreamSynchronize(stream));
  nu_hat_set = true;
  freq_ready = false;
  uhat_valid = false;
}

namespace {
// max_i sum_d |M_d(i)| and min_i K_C(i) of one level's 7-point planes (stride
// n), as ordered bit patterns of non-negative doubles
__global__ void k_level_shift_ratio(const double* __restrict__ K, const double* __restrict__ M, size_t n,
                                    unsigned long long* __restrict__ out) {
  double mx = 0, mn = __longlong_as_double(0x7ff0000000000000ll);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double s = 0;
    for (int d = 0; d < 7; ++d) s += fabs(M[d * n + i]);
    mx = fmax(mx, s);
    mn = fmin(mn, K[i]);
  }
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
    mn = fmin(mn, __shfl_down_sync(0xffffffffu, mn, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&out[0], (unsigned long long)__double_as_longlong(mx));
    atomicMin(&out[1], (unsigned long long)__double_as_longlong(fmax(mn, 0.0)));
  }
}
}  // namespace

// PeriodicSolver ctor (periodic.hpp:128-139): symbols + multigrid hierarchy
// for (lambda_k M + K_hat), all frequencies sharing the real stencils.
void Problem::build_frequency_solver(const tp_solver_cfg& cfg) {
  require(nu_hat_set, "periodic solver: nu_hat not installed");
  static const int env_groups = std::getenv("TPGPU_FREQ_GROUPS") ? std::atoi(std::getenv("TPGPU_FREQ_GROUPS")) : 5;
  const int want_groups = cfg.freq_groups > 0 ? cfg.freq_groups : env_groups;
  if (freq_ready && fw && (cfg.freq_chunk <= 0 || cfg.freq_chunk == fw->req_chunk) &&
      (want_groups == fw->req_groups)) {
    for (int g = 0; g < fw->parts; ++g) {
      fw->group(g).cfg.rtol = cfg.inner_rtol;
      fw->group(g).cfg.max_iter = cfg.inner_max_iter;
    }
    return;
  }
  fw.reset();
  build_freq_work(levels, fw, nullptr, cfg, want_groups);
  freq_ready = true;
  uhat_valid = false;
}

// Multigrid hierarchy and batched frequency solvers for lambda_k M + K0 into
// (lv, out).  K0 == nullptr: K_hat from nu_hat (the M1 operator; the fine
// level runs the Five streaming passes from edge weights).  Otherwise K0 is a
// fine-grid 7-point stencil on the device (7n, e.g. M2's time-averaged
// Jacobian): the fine level runs the Galerkin-style 7-point passes.
void Problem::build_freq_work(std::vector<Level>& lv, std::unique_ptr<FreqWork>& out, const double* K0,
                              const tp_solver_cfg& cfg, int want_groups) {
  lv.clear();
  int cl = c;
  while (true) {
    Level L;
    L.m = cl - 1;
    L.n = L.m * L.m;
    lv.push_back(std::move(L));
    if (cl <= 8) break;
    require(cl % 2 == 0, "multigrid: cells per side must be 2^k * q with q <= 8");
    cl /= 2;
  }
  const int nl = (int)lv.size();
  // fine level: K (K_hat element stencil or the given K0), lumped M on the diagonal
  lv[0].K.alloc((size_t)7 * n);
  lv[0].M.alloc((size_t)7 * n);
  if (K0) {
    TP_CUDA(cudaMemcpyAsync(lv[0].K.get(), K0, lv[0].K.bytes(), cudaMemcpyDeviceToDevice, stream));
  } else {
    launch_element_stencil(*this, false, nullptr, lv[0].K.get(), 1);
  }
  TP_CUDA(cudaMemsetAsync(lv[0].M.get(), 0, lv[0].M.bytes(), stream));
  TP_CUDA(cudaMemcpyAsync(lv[0].M.get(), d_mass.get(), n * sizeof(double), cudaMemcpyDeviceToDevice, stream));
  for (int l = 1; l < nl; ++l) {
    lv[l].K.alloc((size_t)7 * lv[l].n);
    lv[l].M.alloc((size_t)7 * lv[l].n);
    launch_rap(*this, lv[l - 1].K.get(), lv[l - 1].m, lv[l].K.get(), lv[l].m, 1);
    launch_rap(*this, lv[l - 1].M.get(), lv[l - 1].m, lv[l].M.get(), lv[l].m, 1);
  }
  out = std::make_unique<FreqWork>();
  FreqWork* w = out.get();
  const int Kr = sh.k1 - sh.k0;
  // chunk: work ~ 7 complex vectors per frequency on the fine level (+1/3 coarse)
  size_t free_b = 0, total_b = 0;
  TP_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const double per = 16.0 * 8.5 * n;
  int chunk = cfg.freq_chunk > 0 ? cfg.freq_chunk : (int)std::min<double>(Kr, 0.6 * free_b / per);
  chunk = std::max(1, std::min(chunk, Kr));
  w->chunk = chunk;
  // Single GPU, several frequency groups: deal the frequencies of every chunk
  // to the groups in boustrophedon order (the sharded solver's slot
  // permutation), so each group's contiguous slot block holds a
  // spread of the spectrum instead of group 0 holding the lowest -- the
  // slowest -- frequencies of every chunk.  Only the time DFTs index through
  // the permutation (kslot).  Opt-in (TPGPU_GROUP_DEAL=1): measured level at
  // cfg 3 and slower at cfg 1 (3.26 vs 3.01 ms per sweep: every group then
  // runs the long iteration chain of its low frequencies, profiles/r2t_ab.txt)
  if (!K0 && !sharded()) {
    static const bool deal = std::getenv("TPGPU_GROUP_DEAL") && std::atoi(std::getenv("TPGPU_GROUP_DEAL")) != 0;
    const int parts0 = std::max(1, std::min(want_groups, chunk));
    const int per0 = (chunk + parts0 - 1) / parts0;
    sh.kperm.clear();
    d_kslot.release();
    if (deal && parts0 > 1) {
      const int span = parts0 * per0;
      std::vector<int> perm(Kr, -1);
      for (int c0 = 0; c0 < Kr; c0 += span) {
        std::vector<int> cap(parts0), fill(parts0, 0);
        for (int g = 0; g < parts0; ++g) cap[g] = std::max(0, std::min(per0, Kr - (c0 + g * per0)));
        const int cnt = std::min(span, Kr - c0);
        int g = 0, dir = 1;
        for (int i = 0; i < cnt; ++i) {
          while (fill[g] >= cap[g]) {  // next group in snake order with room
            g += dir;
            if (g == parts0 || g < 0) {
              dir = -dir;
              g += dir;
            }
          }
          perm[c0 + g * per0 + fill[g]++] = c0 + i;  // slot -> frequency
          g += dir;
          if (g == parts0 || g < 0) {
            dir = -dir;
            g += dir;
          }
        }
      }
      sh.kperm = perm;
      std::vector<int> slot(Kr);
      for (int s2 = 0; s2 < Kr; ++s2) slot[perm[s2]] = s2;
      d_kslot.alloc(Kr);
      TP_CUDA(cudaMemcpy(d_kslot.get(), slot.data(), Kr * sizeof(int), cudaMemcpyHostToDevice));
    }
  }
  // symbols lambda_k (periodic.hpp:146-152) of this rank's frequencies
  std::vector<cplx> lam(Kr);
  for (int kk = 0; kk < Kr; ++kk) {
    const int k = freq_of_slot(sh.k0 + kk);
    cplx& lk = lam[kk];
    if (k == 0) lk = {0.0, 0.0};
    else if (2 * k == N) lk = {2.0 / tau, 0.0};
    else {
      const double a = -2.0 * std::numbers::pi * k / N;
      const double rr = std::cos(a), ri = std::sin(a);  // std::polar(1.0, a)
      lk = {(1.0 - rr) / tau, (0.0 - ri) / tau};
    }
  }
  w->lam.alloc(Kr);
  TP_CUDA(cudaMemcpy(w->lam.get(), lam.data(), Kr * sizeof(cplx), cudaMemcpyHostToDevice));
  const Level& LC = lv.back();
  w->nL = LC.n;
  w->inv.alloc((size_t)Kr * LC.n * LC.n);
  launch_coarse_inverse_freq(*this, LC.K.get(), LC.M.get(), LC.m, w->lam.get(), w->inv.get(), Kr);
  std::vector<LevelOp> ops(nl);
  for (int l = 0; l < nl; ++l) ops[l] = {lv[l].m, lv[l].n, lv[l].K.get(), lv[l].M.get(), l == 0 && !K0, {}};
  // Galerkin levels whose shift is negligible: max_k |lambda_k| max_i sum_d
  // |M_l,d(i)| <= 1e-2 min_i K_l,C(i) (|lambda_k| <= 2 / tau) -- the V-cycle
  // uses K_l alone there (SevenK: half the coefficient planes; M_l grows 4x
  // per level against K_l, so this holds on the fine Galerkin levels of the
  // large grids: cfg 3 levels 1-4 at <= 3.7e-3, cfg 1 level 1 at 4.0e-3;
  // 1e-2 against 1e-3: cfg 1 3.0 -> 2.9 ms per sweep, profiles/r2u_ab.txt).
  // TPGPU_DROP_M=ratio overrides the threshold (0: keep M everywhere).
  static const double drop_thr = std::getenv("TPGPU_DROP_M") ? std::atof(std::getenv("TPGPU_DROP_M")) : 1e-2;
  if (drop_thr > 0) {
    DevBuf<unsigned long long> mm;
    mm.alloc(2);
    for (int l = 1; l < nl; ++l) {
      const unsigned long long init[2] = {0ull, 0x7ff0000000000000ull};  // max sum |M| = 0, min K_C = +inf
      TP_CUDA(cudaMemcpyAsync(mm.get(), init, sizeof init, cudaMemcpyHostToDevice, stream));
      const int blocks = (int)std::min<size_t>((lv[l].n + 255) / 256, 1024);
      k_level_shift_ratio<<<blocks, 256, 0, stream>>>(lv[l].K.get(), lv[l].M.get(), (size_t)lv[l].n, mm.get());
      TP_LAUNCHED(this);
      unsigned long long h[2];
      TP_CUDA(cudaMemcpyAsync(h, mm.get(), sizeof h, cudaMemcpyDeviceToHost, stream));
      TP_CUDA(cudaStreamSynchronize(stream));
      double msum, kmin;
      std::memcpy(&msum, &h[0], sizeof msum);
      std::memcpy(&kmin, &h[1], sizeof kmin);
      ops[l].drop_m = kmin > 0 && (2.0 / tau) * msum <= drop_thr * kmin;
      if (std::getenv("TPGPU_DEBUG_LEVELS"))
        std::fprintf(stderr, "level %d m %d shift ratio %.3e drop_m %d\n", l, lv[l].m, (2.0 / tau) * msum / kmin,
                     (int)ops[l].drop_m);
    }
  }
  if (!K0 && !std::getenv("TPGPU_NO_STREAM_FINE")) {
    // K_hat edge weights: we[Y][X] = (nu_hat(cell(X,Y)) + nu_hat(cell(X,Y-1)))/2,
    // wn[Y][X] = (nu_hat(cell(X,Y)) + nu_hat(cell(X-1,Y)))/2 (the two triangles
    // sharing the edge, assemble_stiffness_frozen on the right-triangle grid)
    const int V = c + 1;
    std::vector<double> we((size_t)V * V, 1.0), wn((size_t)V * V, 1.0);
    auto nh = [&](int i, int j) { return nu_hat[cell_mat[(size_t)j * c + i]]; };
    for (int Y = 1; Y <= c - 1; ++Y)
      for (int X = 0; X <= c - 1; ++X) we[(size_t)Y * V + X] = 0.5 * (nh(X, Y) + nh(X, Y - 1));
    for (int Y = 0; Y <= c - 1; ++Y)
      for (int X = 1; X <= c - 1; ++X) wn[(size_t)Y * V + X] = 0.5 * (nh(X, Y) + nh(X - 1, Y));
    // one contiguous block [we | wn | mass]: every fine pass of every frequency
    // re-reads these 24 bytes per node; a persisting access-policy window over
    // it is available (l2_persist, off by default: measured slower)
    const size_t VV = (size_t)V * V;
    d_coef.alloc(2 * VV + (size_t)n);
    TP_CUDA(cudaMemcpy(d_coef.get(), we.data(), VV * sizeof(double), cudaMemcpyHostToDevice));
    TP_CUDA(cudaMemcpy(d_coef.get() + VV, wn.data(), VV * sizeof(double), cudaMemcpyHostToDevice));
    TP_CUDA(cudaMemcpy(d_coef.get() + 2 * VV, mass.data(), (size_t)n * sizeof(double), cudaMemcpyHostToDevice));
    d_we.alias(d_coef.get(), VV);
    d_wn.alias(d_coef.get() + VV, VV);
    FineOp& fo = ops[0].fine;
    fo.we = d_we.get();
    fo.wn = d_wn.get();
    fo.mass = d_coef.get() + 2 * VV;
    fo.m = m;
    fo.c = c;
    fo.n = n;
  }
  MGConfig mc;
  mc.rtol = cfg.inner_rtol;
  mc.max_iter = cfg.inner_max_iter;
  // experiment overrides (documented in DESIGN.md §5)
  if (const char* e = std::getenv("TPGPU_RB_FINE")) mc.rb_fine = std::atoi(e) != 0;
  if (const char* e = std::getenv("TPGPU_OMEGA")) mc.omega = mc.omega2 = std::atof(e);
  if (const char* e = std::getenv("TPGPU_OMEGA2")) mc.omega2 = std::atof(e);
  // concurrent frequency groups (TPGPU_FREQ_GROUPS overrides; 1 = one solver on the problem stream)
  w->req_chunk = cfg.freq_chunk;
  w->req_groups = want_groups;
  int parts = std::max(1, std::min(want_groups, chunk));
  w->parts = parts;
  const int per_group = (chunk + parts - 1) / parts;
  w->chunk = per_group;
  w->solver.init(this, ops, per_group, mc);
  for (int g = 1; g < parts; ++g) {
    w->extra.push_back(std::make_unique<BatchSolver<0>>());
    w->extra.back()->init(this, ops, per_group, mc);
  }
  if (parts > 1) {
    w->hs.assign(parts, nullptr);
    w->ev_out.assign(parts, nullptr);
    // stream priorities: group 0 (the lowest frequencies: the most inner
    // iterations, the sweep's critical path) highest, group 1 next, the rest
    // default -- the other groups fill the gaps of its latency-bound chain
    // (cfg 1: 3.85 -> 3.76 ms per sweep).  TPGPU_GROUP_PRIO=0: all default.
    // TPGPU_GROUP_PRIO=2: priorities graded over the whole range, group 0 highest
    static const int prio = std::getenv("TPGPU_GROUP_PRIO") ? std::atoi(std::getenv("TPGPU_GROUP_PRIO")) : 1;
    int lo = 0, hi = 0;
    TP_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));  // hi: numerically smallest = highest
    for (int g = 0; g < parts; ++g) {
      const int graded = parts > 1 ? hi + (int)std::lround((double)(lo - hi) * g / (parts - 1)) : hi;
      const int pr = prio == 0 ? lo : prio == 2 ? graded : g == 0 ? hi : g == 1 ? std::max(hi, lo - 1) : lo;
      TP_CUDA(cudaStreamCreateWithPriority(&w->hs[g], cudaStreamNonBlocking, pr));
    }
    TP_CUDA(cudaEventCreateWithFlags(&w->ev_in, cudaEventDisableTiming));
    for (auto& e : w->ev_out) TP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  if (d_coef.get() && !K0) {
    std::vector<cudaStream_t> ss{stream};
    for (auto h : w->hs) ss.push_back(h);
    l2_persist(d_coef.get(), d_coef.bytes(), ss);
  }
  TP_CUDA(cudaStreamSynchronize(stream));
}

// Persisting L2 window over [base, base + bytes) on the given streams
// (TPGPU_L2_PERSIST=1 enables): the fine-level coefficients stay resident
// while the vectors stream through as normal (missProp streaming).
void Problem::l2_persist(const void* base, size_t bytes, const std::vector<cudaStream_t>& ss) {
  // off by default: measured at cfg 3 the window made every sweep slower
  // (398-402 vs 346-349 ms, profiles/r2g_ab.txt) -- the persisting lines
  // shrink the L2 the streamed vectors and the coarse levels reuse
  static const bool on = std::getenv("TPGPU_L2_PERSIST") && std::atoi(std::getenv("TPGPU_L2_PERSIST")) != 0;
  if (!on || bytes == 0) return;
  int max_persist = 0, max_window = 0;
  TP_CUDA(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, device));
  TP_CUDA(cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, device));
  if (max_persist <= 0 || max_window <= 0) return;
  const size_t limit = std::min<size_t>((size_t)max_persist, bytes);
  TP_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, limit));
  cudaStreamAttrValue a{};
  a.accessPolicyWindow.base_ptr = const_cast<void*>(base);
  a.accessPolicyWindow.num_bytes = std::min<size_t>(bytes, (size_t)max_window);
  a.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)limit / (double)a.accessPolicyWindow.num_bytes);
  a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  for (auto h : ss) TP_CUDA(cudaStreamSetAttribute(h, cudaStreamAttributeAccessPolicyWindow, &a));
}

namespace {
struct PrecondHolder {
  std::vector<Level> lv;
  std::unique_ptr<Problem::FreqWork> fw;
};
}  // namespace

std::shared_ptr<void> Problem::make_periodic_precond(const double* K0, const tp_solver_cfg& cfg) {
  auto h = std::make_shared<PrecondHolder>();
  build_freq_work(h->lv, h->fw, K0, cfg, cfg.freq_groups > 0 ? cfg.freq_groups : 3);
  return h;
}

void Problem::precond_solve(void* handle, const double* in, double* out, const tp_solver_cfg& cfg) {
  auto* h = static_cast<PrecondHolder*>(handle);
  SolveStats st;
  periodic_solve_with(*h->fw, in, out, false, cfg, &st);
}

// U_{k+1} = IDFT(U_hat) stays close to U_k near the fixed point, so DFT(U) is
// a far better first guess for the frequency solves than zero; the solves
// still converge to the same tolerance (only their iteration count changes).
void Problem::seed_spectrum() {
  uhat_prev_valid = false;
  launch_rdft_forward(*this, U.get(), Uhat.get());
  if (sharded()) alltoall_to_freq(Uhat.get(), Uhat_f.get());
  uhat_valid = true;
}

namespace {
// x = x + theta (x - prev), prev = old x (warm-start extrapolation)
__global__ void k_extrap(cplx* __restrict__ x, cplx* __restrict__ prev, size_t cnt, double theta) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < cnt; i += (size_t)gridDim.x * blockDim.x) {
    const cplx a = x[i], b = prev[i];
    prev[i] = a;
    x[i] = {fma(theta, a.re - b.re, a.re), fma(theta, a.im - b.im, a.im)};
  }
}
}  // namespace

void Problem::periodic_solve_dev(const tp_solver_cfg& cfg, SolveStats* st) {
  build_frequency_solver(cfg);
  const bool warm = cfg.warm_start && uhat_valid;
  // Warm-start extrapolation: near the fixed point the spectra of successive
  // sweeps move along the dominant mode of the contraction, U_hat_{k+1} -
  // U_hat_k ~ q (U_hat_k - U_hat_{k-1}), so the frequency solves start from
  // U_hat_k + q (U_hat_k - U_hat_{k-1}) with q the last residual ratio of the
  // fixed-point iteration (at most 0.95; none while the residual does not
  // decrease).  Only the initial guess
  // changes (same stopping rule, same accuracy); cfg 1 to 1e-8: 323 -> 237
  // frequency-iterations per sweep.  TPGPU_EXTRAP=0 disables, =theta fixes it.
  static const char* ex_env = std::getenv("TPGPU_EXTRAP");
  static const double theta_fixed = ex_env ? std::atof(ex_env) : -1.0;  // < 0: adaptive
  static const bool ex_on = !ex_env || theta_fixed > 0;
  extrap_theta = 0.0;
  if (ex_on) {
    const size_t cnt = (size_t)(sh.k1 - sh.k0) * n;
    if (warm && uhat_prev_valid) {
      double q = theta_fixed;
      if (q < 0) {
        const double ratio = (resid_prev > 0 && resid_last >= 0) ? resid_last / resid_prev : 1.0;
        q = ratio < 1.0 ? std::min(0.95, ratio) : 0.0;  // no extrapolation while not contracting
      }
      extrap_theta = q;  // applied per frequency group on its stream (periodic_solve_with)
    } else if (warm) {
      // the copy of the previous spectrum needs cnt complex values; skip when
      // device memory is short (config 3 on one GPU)
      size_t free_b = 0, total_b = 0;
      TP_CUDA(cudaMemGetInfo(&free_b, &total_b));
      if (uhat_prev.count >= cnt || free_b > cnt * sizeof(cplx) + ((size_t)4 << 30)) {
        uhat_prev.ensure(cnt);
        TP_CUDA(cudaMemcpyAsync(uhat_prev.get(), spec_out(), cnt * sizeof(cplx), cudaMemcpyDeviceToDevice, stream));
        uhat_prev_valid = true;
      }
    } else {
      uhat_prev_valid = false;
    }
  }
  periodic_solve_with(*fw, G.get(), U.get(), warm, cfg, st);
  uhat_valid = true;
}

// PeriodicSolver::solve (periodic.hpp:154-198) of `in` (N x n, this rank's
// strip layout) into `out` with the frequency solvers of `w`: forward time
// DFT, [all-to-all to frequency blocks], batched block solves (warm: from the
// current spectrum), [all-to-all back], inverse DFT and the imaginary guard.
void Problem::periodic_solve_with(FreqWork& w, const double* in, double* out, bool warm, const tp_solver_cfg& cfg,
                                  SolveStats* st) {
  // Stopping floor of the frequency solves: ||r_k|| <= rtol max(||g_k||,
  // ||g||/sqrt(K)) with ||g||^2 the energy of the whole half spectrum (summed
  // inside the forward DFT).  Blocks whose right-hand side is round-off (the
  // even harmonics of an odd-symmetric response) stop at the frequency's
  // equal share of the total instead of iterating on noise; the aggregate
  // residual bound stays within sqrt(2) of the per-frequency rule's
  // (DESIGN.md §5).  TPGPU_NO_FREQ_FLOOR restores the plain per-frequency rule.
  static const bool use_floor = std::getenv("TPGPU_NO_FREQ_FLOOR") == nullptr;
  const int nblk = rdft_forward_blocks(*this);
  spec_sq.ensure((size_t)nblk + 1);
  launch_rdft_forward(*this, in, Ghat.get(), use_floor ? spec_sq.get() : nullptr);
  if (use_floor) {
    reduce_sum_dev(*this, spec_sq.get(), nblk, spec_sq.get() + nblk);
    if (sharded()) global_sum_dev(spec_sq.get() + nblk, 1, spec_sq.get() + nblk);
  }
  if (sharded()) alltoall_to_freq();
  const int Kr = sh.k1 - sh.k0;
  const double* floor_ptr = use_floor ? spec_sq.get() + nblk : nullptr;
  const double floor_scale = 1.0 / (double)(N / 2 + 1);
  int iters = 0;
  int64_t fiters = 0;
  const double theta = extrap_theta;
  extrap_theta = 0.0;
  auto run = [&](BatchSolver<0>& sv, int k0, int nb, SolveStats* sst) {
    if (theta > 0 && warm) {
      const size_t cnt = (size_t)nb * n, off = (size_t)k0 * n;
      k_extrap<<<(unsigned)std::min<size_t>((cnt + 255) / 256, 2048), 256, 0, cur_stream()>>>(
          spec_out() + off, uhat_prev.get() + off, cnt, theta);
      TP_LAUNCHED(this);
    }
    sv.bfloor = floor_ptr;
    sv.bfloor_scale = floor_scale;
    sv.lam = w.lam.get() + k0;
    sv.coarse_inv = w.inv.get() + (size_t)k0 * w.nL * w.nL;
    return sv.solve(spec_in() + (size_t)k0 * n, spec_out() + (size_t)k0 * n, nb, warm, sst);
  };
  double rel_f = 0, rel_o = 0;
  if (w.parts == 1) {
    for (int k0 = 0; k0 < Kr; k0 += w.chunk) {
      SolveStats cs;
      iters = std::max(iters, run(w.solver, k0, std::min(w.chunk, Kr - k0), &cs));
      fiters += cs.batch_iterations;
      if (st) {
        st->iterations = std::max(st->iterations, cs.iterations);
        st->batch_iterations += cs.batch_iterations;
        st->max_rel_residual = std::max(st->max_rel_residual, cs.max_rel_residual);
      }
      rel_f = std::max(rel_f, cs.max_rel_residual);
      rel_o = std::max(rel_o, cs.max_rel_residual_own);
    }
  } else {
    // groups of `parts` chunks: group 0 on hs[0] (this thread), the others on
    // hs[g] driven by helper threads
    const int P = w.parts;
    // Each group walks its block of every chunk in turn, with no barrier
    // between chunks: a group that finishes its block of chunk c starts on
    // chunk c+1 while the others still iterate (the lowest frequencies of
    // chunk 0 used to hold every group at the chunk boundary).
    // TPGPU_CHUNK_BARRIER=1 restores the per-chunk join.
    static const bool chunk_barrier = std::getenv("TPGPU_CHUNK_BARRIER") != nullptr;
    const int span = P * w.chunk;
    for (int c0 = 0; c0 < Kr; c0 += chunk_barrier ? span : Kr) {
      const int c1 = chunk_barrier ? std::min(Kr, c0 + span) : Kr;
      TP_CUDA(cudaEventRecord(w.ev_in, stream));
      for (auto h : w.hs) TP_CUDA(cudaStreamWaitEvent(h, w.ev_in, 0));
      std::vector<SolveStats> gst(P);
      std::vector<int> git(P, 0);
      std::vector<std::exception_ptr> gerr(P);
      static const bool dbg_groups = std::getenv("TPGPU_DEBUG_GROUPS") != nullptr;
      std::vector<double> gsec(P, 0.0);
      const auto tg0 = std::chrono::steady_clock::now();
      auto body = [&](int g) {
        static const bool tracing = std::getenv("TPGPU_TRACE") != nullptr;
        StreamTrace trace;
        try {
          if (g > 0) TP_CUDA(cudaSetDevice(device));
          tl_stream = w.hs[g];
          if (tracing) {
            tl_trace = &trace;
            trace_mark("start", w.hs[g]);
          }
          for (int k0 = c0; k0 < c1; k0 += span) {
            const int kg = k0 + g * w.chunk, nbg = std::min(w.chunk, Kr - kg);
            if (nbg <= 0) break;
            git[g] = std::max(git[g], run(w.group(g), kg, nbg, &gst[g]));
          }
          if (tracing) {
            trace_mark("end", w.hs[g]);
            tl_trace = nullptr;
            trace_report(trace, "trace g" + std::to_string(g), w.hs[g]);
          }
        } catch (...) {
          gerr[g] = std::current_exception();
        }
        tl_stream = nullptr;
        if (dbg_groups) gsec[g] = std::chrono::duration<double>(std::chrono::steady_clock::now() - tg0).count();
      };
      if (!w.pool || w.pool->helpers() != P - 1) w.pool = std::make_unique<WorkerPool>(P - 1);
      w.pool->run(body);
      if (dbg_groups) {
        std::string line = "groups:";
        for (int g = 0; g < P; ++g)
          line += " " + std::to_string(git[g]) + "it/" + std::to_string(gst[g].batch_iterations) + "fi " +
                  std::to_string(gsec[g] * 1e3).substr(0, 5) + "ms";
        std::fprintf(stderr, "%s\n", line.c_str());
      }
      for (int g = 0; g < P; ++g) {
        TP_CUDA(cudaEventRecord(w.ev_out[g], w.hs[g]));
        TP_CUDA(cudaStreamWaitEvent(stream, w.ev_out[g], 0));
      }
      for (auto& e : gerr)
        if (e) std::rethrow_exception(e);
      for (int g = 0; g < P; ++g) {
        iters = std::max(iters, git[g]);
        fiters += gst[g].batch_iterations;
        if (st) {
          st->iterations = std::max(st->iterations, gst[g].iterations);
          st->batch_iterations += gst[g].batch_iterations;
          st->max_rel_residual = std::max(st->max_rel_residual, gst[g].max_rel_residual);
        }
        rel_f = std::max(rel_f, gst[g].max_rel_residual);
        rel_o = std::max(rel_o, gst[g].max_rel_residual_own);
      }
    }
  }
  last_inner = iters;
  last_freq_iters = fiters;
  last_rel_floored = sharded() ? global_max(rel_f) : rel_f;
  last_rel_own = sharded() ? global_max(rel_o) : rel_o;
  if (sharded()) alltoall_from_freq();
  double re2 = 0, im2 = 0;
  launch_rdft_inverse(*this, Uhat.get(), out, nullptr, nullptr);  // sums in red[0..1]
  global_sum_dev(red.get(), 2, red.get() + 2);
  TP_CUDA(cudaMemcpyAsync(h_scalars, red.get() + 2, 2 * sizeof(double), cudaMemcpyDeviceToHost, stream));
  TP_CUDA(cudaStreamSynchronize(stream));
  re2 = h_scalars[0];
  im2 = h_scalars[1];
  // imaginary-residue guard, periodic.hpp:186-196
  const double re_norm = std::sqrt(re2), im_norm = std::sqrt(im2);
  if (im_norm > cfg.imag_tol * std::max(re_norm, 1e-300))
    throw Error(TP_ESOLVE,
                "periodic solver: imaginary residue " + std::to_string(im_norm) + " exceeds " +
                    std::to_string(cfg.imag_tol) + " x " + std::to_string(re_norm),
                im_norm / std::max(re_norm, 1e-300));
}

}  // namespace tpgpu

// =================================================================== C ABI
using tpgpu::Error;
using tpgpu::Problem;

struct tp_problem {
  std::unique_ptr<Problem> impl;
};

namespace {
thread_local std::string g_err;
thread_local double g_err_res = -1;
}  // namespace

void tpgpu::set_last_error(const std::string& msg, double residual) {
  g_err = msg;
  g_err_res = residual;
}

namespace {

template <class F>
int guarded(F&& f) {
  try {
    f();
    return TP_OK;
  } catch (const Error& e) {
    g_err = e.what();
    g_err_res = e.residual;
    return e.code;
  } catch (const std::bad_alloc& e) {
    g_err = std::string("allocation failed: ") + e.what();
    g_err_res = -1;
    return TP_ECUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    g_err_res = -1;
    return TP_EINVAL;
  }
}

Problem& P(tp_problem* p) {
  tpgpu::require(p && p->impl, "null problem handle");
  TP_CUDA(cudaSetDevice(p->impl->device));
  return *p->impl;
}

tp_solver_cfg cfg_or_default(const tp_solver_cfg* c) {
  tp_solver_cfg d;
  tp_solver_cfg_default(&d);
  return c ? *c : d;
}

double seconds_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}
}  // namespace

extern "C" {

int tp_version(void) { return TPGPU_VERSION; }

int tp_last_error(char* buf, size_t cap, double* achieved) {
  if (buf && cap) {
    std::strncpy(buf, g_err.c_str(), cap - 1);
    buf[cap - 1] = 0;
  }
  if (achieved) *achieved = g_err_res;
  return TP_OK;
}

void tp_solver_cfg_default(tp_solver_cfg* c) {
  std::memset(c, 0, sizeof(*c));
  c->tol = 1e-4;
  c->m1_max_outer = 200;
  c->armijo_max_halvings = 30;
  c->armijo_slope = 1e-4;
  c->armijo_backtrack = 0.5;
  c->nu_hat_mode = TP_NU_HAT_FROZEN_FIELD;
  c->nu_hat_samples = 2000;
  c->imag_tol = 1e-9;
  c->static_tol = 1e-8;
  c->static_max_newton = 50;
  c->threads = 1;
  c->inner_rtol = 1e-12;
  c->inner_max_iter = 200;
  c->warm_start = 1;
  c->m2_max_outer = 50;
  c->m2_inner_tol = 1e-8;
  c->m2_inner_max = 300;
  c->m2_restart = 60;
  c->m3_max_cycles = 10;
}

int tp_problem_desc_baseline(int32_t config, tp_problem_desc* desc) {
  return guarded([&] {
    tpgpu::require(desc != nullptr, "null descriptor");
    tpgpu::require(tp_baseline_desc_fill(config, desc) == 0, "unknown BASELINE config id");
  });
}

int tp_problem_create(const tp_problem_desc* desc, int32_t device, tp_problem** out) {
  return guarded([&] {
    tpgpu::require(desc && out, "null argument");
    auto h = std::make_unique<tp_problem>();
    h->impl = std::make_unique<Problem>(*desc, device);
    *out = h.release();
  });
}

void tp_problem_destroy(tp_problem* p) {
  if (!p) return;
  if (p->impl) cudaSetDevice(p->impl->device);
  delete p;
}

int tp_problem_sizes(const tp_problem* p, int32_t* n_dof, int32_t* steps, double* tau) {
  return guarded([&] {
    tpgpu::require(p && p->impl, "null problem handle");
    if (n_dof) *n_dof = p->impl->sh.nr;  // local dofs (all dofs on a single GPU)
    if (steps) *steps = p->impl->N;
    if (tau) *tau = p->impl->tau;
  });
}

// Host arrays of a sharded rank are its strip (N x n_local, tpgpu.h): loads
// and mass are written for the strip's dofs [y0*m, y1*m).
int tp_problem_loads(tp_problem* h, double* F) {
  return guarded([&] {
    Problem& p = P(h);
    const int nsrc = (int)p.src_mats.size();
    const int i0 = p.sh.y0 * p.m, nl = p.sh.nr;
    for (int s = 0; s < p.N; ++s)
      for (int i = 0; i < nl; ++i) {
        double f = 0;
        for (int r = 0; r < nsrc; ++r)
          f += p.src_time[(size_t)s * nsrc + r] * p.src_prof[(size_t)r * p.n + i0 + i];
        F[(size_t)s * nl + i] = f;
      }
  });
}

int tp_problem_mass(tp_problem* h, double* m) {
  return guarded([&] {
    Problem& p = P(h);
    std::memcpy(m, p.mass.data() + (size_t)p.sh.y0 * p.m, (size_t)p.sh.nr * sizeof(double));
  });
}

int tp_apply_k(tp_problem* h, const double* U, double* KU, int32_t count) {
  return guarded([&] {
    Problem& p = P(h);
    tpgpu::require(!p.sharded(), "apply_k of host slices: single-rank problems only");
    tpgpu::require(count >= 1, "apply_k: count must be positive");
    tpgpu::DevBuf<double> du((size_t)count * p.n), dk((size_t)count * p.n);
    TP_CUDA(cudaMemcpyAsync(du.get(), U, du.bytes(), cudaMemcpyHostToDevice, p.stream));
    p.apply_k_dev(du.get(), dk.get(), count);
    TP_CUDA(cudaMemcpyAsync(KU, dk.get(), dk.bytes(), cudaMemcpyDeviceToHost, p.stream));
    TP_CUDA(cudaStreamSynchronize(p.stream));
  });
}

int tp_residual(tp_problem* h, const double* U, double* R, double* norm) {
  return guarded([&] {
    Problem& p = P(h);
    tpgpu::require(!p.sharded(), "residual of a host state: single-rank problems only");
    const size_t sz = (size_t)p.N * p.n;
    tpgpu::DevBuf<double> du(sz), dr(sz);
    TP_CUDA(cudaMemcpyAsync(du.get(), U, sz * sizeof(double), cudaMemcpyHostToDevice, p.stream));
    p.residual_dev(du.get(), dr.get(), p.N);
    const size_t np = p.part.count;
    (void)np;
    if (R) TP_CUDA(cudaMemcpyAsync(R, dr.get(), sz * sizeof(double), cudaMemcpyDeviceToHost, p.stream));
    const int blocks = (int)(((p.m + 31) / 32) * ((p.m + 7) / 8) * (size_t)p.N);
    const double s = tpgpu::reduce_sum(p, p.part.get(), blocks);
    if (norm) *norm = std::sqrt(s);
  });
}

int tp_set_state(tp_problem* h, const double* U) {
  return guarded([&] {
    Problem& p = P(h);
    TP_CUDA(cudaMemcpyAsync(p.U.get(), U, p.U.bytes(), cudaMemcpyHostToDevice, p.stream));
    TP_CUDA(cudaStreamSynchronize(p.stream));
    p.state_valid = true;
    p.uhat_valid = false;
  });
}

int tp_get_state(tp_problem* h, double* U) {
  return guarded([&] {
    Problem& p = P(h);
    TP_CUDA(cudaMemcpyAsync(U, p.U.get(), p.U.bytes(), cudaMemcpyDeviceToHost, p.stream));
    TP_CUDA(cudaStreamSynchronize(p.stream));
  });
}

int tp_static_init(tp_problem* h, const tp_solver_cfg* c, double* U0, int32_t* newton_counts) {
  return guarded([&] {
    Problem& p = P(h);
    const tp_solver_cfg cfg = cfg_or_default(c);
    tpgpu::validate_cfg(cfg);
    p.static_init_dev(cfg, newton_counts);
    p.state_valid = true;
    p.uhat_valid = false;
    if (U0) {
      TP_CUDA(cudaMemcpyAsync(U0, p.U.get(), p.U.bytes(), cudaMemcpyDeviceToHost, p.stream));
      TP_CUDA(cudaStreamSynchronize(p.stream));
    }
  });
}

// choose_nu_hat (assembly.hpp:254-303) + flux_bounds (materials.hpp:147-155)
int tp_choose_nu_hat(tp_problem* h, const tp_solver_cfg* c, double* nu_hat, double* q) {
  return guarded([&] {
    Problem& p = P(h);
    const tp_solver_cfg cfg = cfg_or_default(c);
    const bool theory = cfg.nu_hat_mode == TP_NU_HAT_THEORY;
    double lo[TP_MAX_MATERIALS], hi[TP_MAX_MATERIALS];
    int any[TP_MAX_MATERIALS] = {0, 0, 0, 0, 0};
    if (!theory) {
      tpgpu::require(p.state_valid, "choose_nu_hat: frozen-field mode needs a state (static_init or set_state)");
      p.field_ranges(lo, hi, any);
    }
    double out[TP_MAX_MATERIALS];
    double qq = 0;
    const int samples = cfg.nu_hat_samples > 1 ? cfg.nu_hat_samples : 2000;
    for (int r = 0; r < TP_MAX_MATERIALS; ++r) {
      if (r >= p.desc.n_materials) {
        out[r] = 1.0;
        continue;
      }
      const tp_material& mt = p.desc.material[r];
      double lf, Lf;
      tpgpu::flux_bounds(mt, 0.0, p.desc.s_max > 0 ? p.desc.s_max : 3.0,
                  p.desc.flux_samples > 1 ? p.desc.flux_samples : 10001, lf, Lf);
      if (theory) {
        out[r] = 0.5 * (lf + Lf);
        qq = std::max(qq, (Lf - lf) / (Lf + lf));
        continue;
      }
      if (!any[r]) {
        out[r] = 0.5 * (lf + Lf);
        continue;
      }
      const double margin = 0.2 * (hi[r] - lo[r]) + 1e-3;
      double lam, Lam;
      tpgpu::flux_bounds(mt, std::max(0.0, lo[r] - margin), hi[r] + margin, samples, lam, Lam);
      out[r] = 0.5 * (lam + Lam);
      qq = std::max(qq, (Lam - lam) / (Lam + lam));
    }
    p.install_nu_hat(out, qq);
    if (nu_hat) std::memcpy(nu_hat, out, sizeof(out));
    if (q) *q = qq;
  });
}

int tp_set_nu_hat(tp_problem* h, const double* nu_hat, double q) {
  return guarded([&] { P(h).install_nu_hat(nu_hat, q); });
}

int tp_periodic_solve(tp_problem* h, const tp_solver_cfg* c, const double* G, double* U) {
  return guarded([&] {
    Problem& p = P(h);
    const tp_solver_cfg cfg = cfg_or_default(c);
    TP_CUDA(cudaMemcpyAsync(p.G.get(), G, p.G.bytes(), cudaMemcpyHostToDevice, p.stream));
    p.uhat_valid = false;
    tpgpu::SolveStats st;
    p.periodic_solve_dev(cfg, &st);
    TP_CUDA(cudaMemcpyAsync(U, p.U.get(), p.U.bytes(), cudaMemcpyDeviceToHost, p.stream));
    TP_CUDA(cudaStreamSynchronize(p.stream));
    p.state_valid = true;
  });
}

int tp_m1_begin(tp_problem* h, const tp_solver_cfg* c, double* residual0) {
  return guarded([&] {
    Problem& p = P(h);
    const tp_solver_cfg cfg = cfg_or_default(c);
    tpgpu::validate_cfg(cfg);
    tpgpu::require(p.state_valid, "m1: no state (static_init or set_state first)");
    p.build_frequency_solver(cfg);
    p.sweep_cfg = cfg;
    p.uhat_valid = false;
    const double r0 = p.residual_and_rhs(true);
    if (cfg.warm_start) p.seed_spectrum();
    if (residual0) *residual0 = r0;
  });
}

int tp_m1_sweep(tp_problem* h, double* residual, int32_t* inner) {
  return guarded([&] {
    Problem& p = P(h);
    tpgpu::require(p.freq_ready, "m1 sweep: call tp_m1_begin first");
    const tp_solver_cfg cfg = p.sweep_cfg;
    tpgpu::SolveStats st;
    p.periodic_solve_dev(cfg, &st);
    const double r = p.residual_and_rhs(true);
    if (residual) *residual = r;
    if (inner) *inner = st.iterations;
  });
}

int tp_solve_residuals(const tp_problem* h, double* max_rel_floored, double* max_rel_own) {
  return guarded([&] {
    tpgpu::require(h && h->impl, "null problem handle");
    if (max_rel_floored) *max_rel_floored = h->impl->last_rel_floored;
    if (max_rel_own) *max_rel_own = h->impl->last_rel_own;
  });
}

int tp_sweep_stats(const tp_problem* h, int32_t* max_iterations, int64_t* frequency_iterations) {
  return guarded([&] {
    tpgpu::require(h != nullptr, "sweep stats: null problem");
    const Problem& p = *h->impl;
    if (max_iterations) *max_iterations = p.last_inner;
    if (frequency_iterations) *frequency_iterations = p.last_freq_iters;
  });
}

// solve_m1_fixed_point, solvers.hpp:301-369
int tp_solve_m1(tp_problem* h, const tp_solver_cfg* c, const double* U0, double* U_out,
                tp_report* rep, double* history, double* contraction, int32_t cap, tp_iterate_cb cb,
                void* user) {
  return guarded([&] {
    Problem& p = P(h);
    const tp_solver_cfg cfg = cfg_or_default(c);
    tpgpu::validate_cfg(cfg);
    tpgpu::require(p.nu_hat_set, "m1: nu_hat not installed (tp_choose_nu_hat / tp_set_nu_hat)");
    const auto t0 = std::chrono::steady_clock::now();
    if (U0) {
      TP_CUDA(cudaMemcpyAsync(p.U.get(), U0, p.U.bytes(), cudaMemcpyHostToDevice, p.stream));
      p.state_valid = true;
    }
    tpgpu::require(p.state_valid, "m1: no initial state");
    std::vector<double> hist;
    std::vector<double> host_u;
    auto callback = [&](int k, double res) {
      if (!cb) return;
      host_u.resize((size_t)p.N * p.n);
      TP_CUDA(cudaMemcpyAsync(host_u.data(), p.U.get(), p.U.bytes(), cudaMemcpyDeviceToHost, p.stream));
      TP_CUDA(cudaStreamSynchronize(p.stream));
      if (cb(k, host_u.data(), res, user) != 0) throw Error(TP_EINVAL, "m1: aborted by iterate callback");
    };
    auto stop = [&]() { return hist.back() <= cfg.tol * hist.front(); };  // solvers.hpp:100-103
    // track_error_contraction: the iterates are archived in host memory
    // (solvers.hpp:317-319; the device holds only the current state)
    const bool archive = cfg.track_error_contraction != 0;
    tpgpu::require(!archive || !p.sharded(), "m1: track_error_contraction needs a single-rank problem");
    std::vector<std::vector<double>> iterates;
    auto keep = [&]() {
      if (!archive) return;
      iterates.emplace_back((size_t)p.N * p.n);
      TP_CUDA(cudaMemcpyAsync(iterates.back().data(), p.U.get(), p.U.bytes(), cudaMemcpyDeviceToHost, p.stream));
      TP_CUDA(cudaStreamSynchronize(p.stream));
    };
    keep();
    hist.push_back(p.residual_and_rhs(true));
    callback(0, hist.back());
    tp_report r{};
    r.q_estimate = p.q_estimate;
    tpgpu::SolveStats st;
    double setup = 0, sweeps = 0;
    if (!stop()) {
      const auto ts = std::chrono::steady_clock::now();
      p.build_frequency_solver(cfg);
      p.uhat_valid = false;
      if (cfg.warm_start) p.seed_spectrum();
      setup = seconds_since(ts);
      for (int k = 1; k <= cfg.m1_max_outer; ++k) {
        const auto tk = std::chrono::steady_clock::now();
        p.periodic_solve_dev(cfg, &st);
        r.iterations = k;
        hist.push_back(p.residual_and_rhs(true));
        sweeps += seconds_since(tk);
        keep();
        callback(k, hist.back());
        if (stop()) break;
      }
    }
    r.status = stop() ? TP_CONVERGED : TP_MAX_ITER;
    r.inner_iterations = (int32_t)st.batch_iterations;
    r.history_len = (int32_t)std::min<size_t>(hist.size(), cap > 0 ? cap : 0);
    if (history)
      for (int k = 0; k < r.history_len; ++k) history[k] = hist[k];
    if (archive && iterates.size() >= 2) {
      // K_hat-norm errors against the final iterate (solvers.hpp:347-360);
      // the device G is the scratch for each archived iterate, then restored
      std::vector<double> errors;
      for (size_t k = 0; k + 1 < iterates.size(); ++k) {
        TP_CUDA(cudaMemcpyAsync(p.G.get(), iterates[k].data(), p.G.bytes(), cudaMemcpyHostToDevice, p.stream));
        errors.push_back(p.khat_norm_diff(p.G.get(), p.U.get()));
      }
      const double floor = 1e-13 * std::max(1.0, p.khat_norm_diff(p.U.get(), nullptr));
      int w = 0;
      for (size_t k = 0; k + 1 < errors.size() && w < cap; ++k) {
        if (errors[k] <= floor || errors[k + 1] <= floor) break;
        if (contraction) contraction[w] = errors[k + 1] / errors[k];
        ++w;
      }
      r.contraction_len = w;
      (void)p.residual_and_rhs(true);  // G back to the next sweep's right-hand side
    } else {
      r.contraction_len = tpgpu::residual_contraction(hist, contraction, cap);
    }
    if (U_out) {
      TP_CUDA(cudaMemcpyAsync(U_out, p.U.get(), p.U.bytes(), cudaMemcpyDeviceToHost, p.stream));
      TP_CUDA(cudaStreamSynchronize(p.stream));
    }
    r.setup_time = setup;
    r.sweep_time = sweeps;
    r.wall_time = seconds_since(t0);
    if (rep) *rep = r;
  });
}

int tp_problem_create_sharded(const tp_problem_desc* desc, tp_comm* comm, tp_problem** out) {
  return guarded([&] {
    tpgpu::require(desc && out && comm, "null argument");
    const int P = tp_comm_size(comm), r = tp_comm_rank(comm), dev = tp_comm_device(comm);
    tpgpu::ShardInfo sh;
    tpgpu::make_partition(desc->cells - 1, desc->steps / 2 + 1, desc->steps, P, r, sh);
    sh.comm = comm;
    auto h = std::make_unique<tp_problem>();
    h->impl = std::make_unique<Problem>(*desc, dev, &sh);
    *out = h.release();
  });
}

int tp_problem_shard(const tp_problem* p, tp_shard_plan* out) {
  return guarded([&] {
    tpgpu::require(p && p->impl && out, "null argument");
    const tpgpu::ShardInfo& s = p->impl->sh;
    out->nranks = s.P;
    out->rank = s.r;
    out->row0 = s.y0;
    out->row1 = s.y1;
    out->freq0 = s.k0;
    out->freq1 = s.k1;
    out->slice0 = s.s0;
    out->slice1 = s.s1;
    out->n_local = s.nr;
  });
}

int tp_kernel_timer_select(tp_problem* h, int32_t which) {
  return guarded([&] {
    Problem& p = P(h);
    tpgpu::require(which >= 0 && which <= 2, "kernel timer: which must be 0 (up), 1 (down) or 2 (apply)");
    p.ktimer.drain();
    p.ktimer.which = which;
  });
}

int tp_kernel_timer(tp_problem* h, int32_t enable, int64_t* launches, double* ms, double* bytes) {
  return guarded([&] {
    Problem& p = P(h);
    p.ktimer.drain();
    if (launches) *launches = p.ktimer.launches;
    if (ms) *ms = p.ktimer.ms;
    if (bytes) *bytes = p.ktimer.bytes;
    p.ktimer.launches = 0;
    p.ktimer.ms = 0;
    p.ktimer.bytes = 0;
    p.ktimer.on = enable != 0;
  });
}

// solve_m2_newton, solvers.hpp:375-484 / solve_m3_timestepping, solvers.hpp:489-542 (single GPU)
static int solve_m23(tp_problem* h, const tp_solver_cfg* c, const double* U0, double* U_out, tp_report* rep,
                     double* history, double* contraction, int32_t cap, int method);

int tp_solve_m2(tp_problem* h, const tp_solver_cfg* c, const double* U0, double* U_out, tp_report* rep,
                double* history, double* contraction, int32_t cap) {
  return solve_m23(h, c, U0, U_out, rep, history, contraction, cap, 2);
}

int tp_solve_m3(tp_problem* h, const tp_solver_cfg* c, const double* U0, double* U_out, tp_report* rep,
                double* history, double* contraction, int32_t cap) {
  return solve_m23(h, c, U0, U_out, rep, history, contraction, cap, 3);
}

static int solve_m23(tp_problem* h, const tp_solver_cfg* c, const double* U0, double* U_out, tp_report* rep,
                     double* history, double* contraction, int32_t cap, int method) {
  return guarded([&] {
    Problem& p = P(h);
    const tp_solver_cfg cfg = cfg_or_default(c);
    tpgpu::validate_cfg(cfg);
    const auto t0 = std::chrono::steady_clock::now();
    if (U0) {
      TP_CUDA(cudaMemcpyAsync(p.U.get(), U0, p.U.bytes(), cudaMemcpyHostToDevice, p.stream));
      p.state_valid = true;
      p.uhat_valid = false;
    }
    Problem::M2Result res;
    if (method == 2) p.solve_m2_dev(cfg, res);
    else p.solve_m3_dev(cfg, res);
    tp_report r{};
    r.iterations = res.iterations;
    r.status = res.status;
    r.q_estimate = std::numeric_limits<double>::quiet_NaN();
    r.inner_iterations = (int32_t)res.inner_total;
    const auto& hist = res.history;
    r.history_len = (int32_t)std::min<size_t>(hist.size(), cap > 0 ? cap : 0);
    if (history)
      for (int k = 0; k < r.history_len; ++k) history[k] = hist[k];
    r.contraction_len = tpgpu::residual_contraction(hist, contraction, cap);
    if (U_out) {
      TP_CUDA(cudaMemcpyAsync(U_out, p.U.get(), p.U.bytes(), cudaMemcpyDeviceToHost, p.stream));
      TP_CUDA(cudaStreamSynchronize(p.stream));
    }
    r.wall_time = seconds_since(t0);
    if (rep) *rep = r;
  });
}

void* tp_problem_stream(tp_problem* p) { return (p && p->impl) ? (void*)p->impl->stream : nullptr; }

int64_t tp_problem_launches(const tp_problem* p) { return (p && p->impl) ? p->impl->launches.load() : 0; }

}  // extern "C"
