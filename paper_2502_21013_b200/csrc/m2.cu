// M2: all-at-once Newton for the periodic system (solve_m2_newton,
// solvers.hpp:375-484) on the device -- SURVEY.md §8(f) f2.
//
// Per outer step: the per-slice Jacobians J_i(U) (k_element_stencil, the
// reference's jacobian_k), their time average (solvers.hpp:401-422) as the
// stiffness of a time-invariant periodic preconditioner P = (M d_t + J_avg)^-1
// (this package's frequency solver built on the averaged stencil), restarted
// FGMRES (detail::fgmres, solvers.hpp:187-270) on A delta = R with
// A v = M (v_i - v_{i-1})/tau + J_i v_i, then the Armijo line search on the
// block residual.  Vectors stay on the device; the Arnoldi scalars (modified
// Gram-Schmidt dots, Givens rotations, the small triangular solve) are made on
// the host from deterministic device reductions, in the reference's order.
#include <cmath>
#include <memory>
#include <string>
#include <vector>

#include "mg.cuh"

namespace tpgpu {

double residual_norm_dev(Problem& p, const double* u, double* r);

namespace {

constexpr int BT = 256;

// J_avg = (J_0 + J_1 + ... + J_{N-1}) / N, summed in slice order (solvers.hpp:410-415)
__global__ void k_average(const double* __restrict__ J, size_t per, int N, double* __restrict__ out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < per; i += (size_t)gridDim.x * blockDim.x) {
    double s = J[i];
    for (int k = 1; k < N; ++k) s += J[(size_t)k * per + i];
    out[i] = s / N;
  }
}

// out_i = M (v_i - v_{i-1}) / tau + J_i v_i for every slice i (solvers.hpp:426-440;
// lumped M; J_i applied in CSR column order SW, S, W, C, E, N, NE)
__global__ void k_m2_apply(const double* __restrict__ J, const double* __restrict__ mass,
                           const double* __restrict__ v, double* __restrict__ out, int m, int N, double tau) {
  const size_t n = (size_t)m * m;
  const int s = blockIdx.y;
  const double* vs = v + (size_t)s * n;
  const double* vp = v + (size_t)((s + N - 1) % N) * n;
  const double* Js = J + (size_t)s * 7 * n;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int x = (int)(i % m), y = (int)(i / m);
    double jv = 0;
    if (x > 0 && y > 0) jv += Js[SSW * n + i] * vs[i - m - 1];
    if (y > 0) jv += Js[SS_ * n + i] * vs[i - m];
    if (x > 0) jv += Js[SW_ * n + i] * vs[i - 1];
    jv += Js[SC * n + i] * vs[i];
    if (x + 1 < m) jv += Js[SE_ * n + i] * vs[i + 1];
    if (y + 1 < m) jv += Js[SN_ * n + i] * vs[i + m];
    if (x + 1 < m && y + 1 < m) jv += Js[SNE * n + i] * vs[i + m + 1];
    const double dv = (vs[i] - vp[i]) / tau;
    out[(size_t)s * n + i] = mass[i] * dv + jv;
  }
}

__global__ void k_dot_part(const double* __restrict__ a, const double* __restrict__ b, size_t n,
                           double* __restrict__ part) {
  __shared__ double sh[BT / 32];
  double v = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    v = fma(a[i], b[i], v);
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0;
    for (int w = 0; w < BT / 32; ++w) s += sh[w];
    part[blockIdx.x] = s;
  }
}

// y = a x + y ; or y = a x (overwrite)
__global__ void k_axpy(double a, const double* __restrict__ x, double* __restrict__ y, size_t n, int overwrite) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    y[i] = overwrite ? a * x[i] : fma(a, x[i], y[i]);
}

}  // namespace

// Device vectors of the flat space-time size with deterministic dots.
struct M2Blas {
  Problem& p;
  size_t n;
  int blocks;
  DevBuf<double> part;
  M2Blas(Problem& pp, size_t nn) : p(pp), n(nn) {
    blocks = std::min<int>(4 * p.num_sms, (int)((n + BT - 1) / BT));
    part.alloc(blocks);
  }
  double dot(const double* a, const double* b) {
    k_dot_part<<<blocks, BT, 0, p.cur_stream()>>>(a, b, n, part.get());
    TP_LAUNCHED(&p);
    return reduce_sum(p, part.get(), blocks);
  }
  double norm2(const double* a) { return std::sqrt(dot(a, a)); }
  void axpy(double a, const double* x, double* y) {
    k_axpy<<<blocks, BT, 0, p.cur_stream()>>>(a, x, y, n, 0);
    TP_LAUNCHED(&p);
  }
  void scale_into(double a, const double* x, double* y) {
    k_axpy<<<blocks, BT, 0, p.cur_stream()>>>(a, x, y, n, 1);
    TP_LAUNCHED(&p);
  }
  void copy(const double* x, double* y) {
    TP_CUDA(cudaMemcpyAsync(y, x, n * sizeof(double), cudaMemcpyDeviceToDevice, p.cur_stream()));
  }
};

void Problem::solve_m2_dev(const tp_solver_cfg& cfg, M2Result& res) {
  require(!sharded(), "m2: single-rank problems only");
  require(state_valid, "m2: no initial state");
  const size_t flat = (size_t)N * n;
  M2Blas bl(*this, flat);
  const int restart = cfg.m2_restart, max_total = cfg.m2_inner_max;
  require(restart >= 1 && max_total >= 1 && cfg.m2_max_outer >= 1, "m2: iteration caps must be positive");
  require(cfg.m2_inner_tol > 0 && cfg.m2_inner_tol < 1, "m2: inner tolerance must lie in (0,1)");
  DevBuf<double> R(flat), Rt(flat), trial(flat), delta(flat), w(flat), Jall((size_t)N * 7 * n), Javg((size_t)7 * n);
  std::vector<DevBuf<double>> V(restart + 1), Z(restart);
  for (auto& v : V) v.alloc(flat);
  for (auto& z : Z) z.alloc(flat);
  std::shared_ptr<void> pw;  // the periodic preconditioner of this outer step
  tp_solver_cfg pcfg = cfg;  // preconditioner: the periodic solver's own controls

  double rnorm = residual_norm_dev(*this, U.get(), R.get());
  res.history.assign(1, rnorm);
  res.status = TP_CONVERGED;
  res.iterations = 0;
  res.inner_total = 0;
  auto stop = [&] { return res.history.back() <= cfg.tol * res.history.front(); };
  while (!stop()) {
    if (res.iterations >= cfg.m2_max_outer) {
      res.status = TP_MAX_ITER;
      break;
    }
    // per-slice Jacobians at U and their time average
    launch_element_stencil(*this, true, U.get(), Jall.get(), N);
    k_average<<<4 * num_sms, BT, 0, stream>>>(Jall.get(), (size_t)7 * n, N, Javg.get());
    TP_LAUNCHED(this);
    pw.reset();
    pw = make_periodic_precond(Javg.get(), pcfg);
    // FGMRES(restart) for A delta = R from delta = 0 (solvers.hpp:187-270)
    auto apply_a = [&](const double* v, double* out) {
      dim3 g((unsigned)std::min<size_t>((n + BT - 1) / BT, 256), N);
      k_m2_apply<<<g, BT, 0, stream>>>(Jall.get(), d_mass.get(), v, out, m, N, tau);
      TP_LAUNCHED(this);
    };
    auto apply_p = [&](const double* v, double* out) { precond_solve(pw.get(), v, out, pcfg); };
    const double bnorm = rnorm;  // ||R||
    TP_CUDA(cudaMemsetAsync(delta.get(), 0, delta.bytes(), stream));
    int total = 0;
    bool inner_ok = bnorm == 0;
    if (!inner_ok) {
      const double target = cfg.m2_inner_tol * bnorm;
      bl.copy(R.get(), w.get());  // r = b - A*0
      while (true) {
        const double beta = bl.norm2(w.get());
        if (beta <= target) {
          inner_ok = true;
          break;
        }
        const int mm = restart;
        bl.scale_into(1.0 / beta, w.get(), V[0].get());
        std::vector<double> H((size_t)(mm + 1) * mm, 0.0), cs(mm), sn(mm), g(mm + 1, 0.0);
        auto h = [&](int i, int j) -> double& { return H[(size_t)i * mm + j]; };
        g[0] = beta;
        int cols = 0;
        for (int j = 0; j < mm && total < max_total; ++j, ++total) {
          apply_p(V[j].get(), Z[j].get());
          apply_a(Z[j].get(), w.get());
          for (int i = 0; i <= j; ++i) {
            const double d = bl.dot(w.get(), V[i].get());
            h(i, j) = d;
            bl.axpy(-d, V[i].get(), w.get());
          }
          const double wnorm = bl.norm2(w.get());
          h(j + 1, j) = wnorm;
          for (int i = 0; i < j; ++i) {
            const double t = cs[i] * h(i, j) + sn[i] * h(i + 1, j);
            h(i + 1, j) = -sn[i] * h(i, j) + cs[i] * h(i + 1, j);
            h(i, j) = t;
          }
          const double denom = std::hypot(h(j, j), h(j + 1, j));
          if (denom == 0) {
            cols = j;
            ++total;
            break;
          }
          cs[j] = h(j, j) / denom;
          sn[j] = h(j + 1, j) / denom;
          h(j, j) = denom;
          h(j + 1, j) = 0;
          g[j + 1] = -sn[j] * g[j];
          g[j] = cs[j] * g[j];
          cols = j + 1;
          if (wnorm == 0 || std::abs(g[j + 1]) <= target) {
            ++total;
            break;
          }
          if (j + 1 < mm) bl.scale_into(1.0 / wnorm, w.get(), V[j + 1].get());
        }
        // y from the triangular H, delta += Z y
        std::vector<double> y(cols, 0.0);
        for (int i = cols - 1; i >= 0; --i) {
          double acc = g[i];
          for (int j = i + 1; j < cols; ++j) acc -= h(i, j) * y[j];
          y[i] = acc / h(i, i);
        }
        for (int j = 0; j < cols; ++j) bl.axpy(y[j], Z[j].get(), delta.get());
        // true residual r = b - A delta
        apply_a(delta.get(), w.get());
        k_axpy<<<bl.blocks, BT, 0, stream>>>(-1.0, R.get(), w.get(), flat, 0);  // w = A delta - b
        TP_LAUNCHED(this);
        bl.scale_into(-1.0, w.get(), w.get());  // w = b - A delta
        if (bl.norm2(w.get()) <= target) {
          inner_ok = true;
          break;
        }
        if (total >= max_total) break;
      }
    }
    res.inner_total += total;
    if (!inner_ok)
      throw Error(TP_ESOLVE, "newton solver: inner linear solve missed its tolerance within " +
                                 std::to_string(max_total) + " iterations",
                  -1.0);
    // Armijo backtracking on the block residual (solvers.hpp:456-470)
    double alpha = 1.0;
    bool accepted = false;
    for (int hv = 0; hv <= cfg.armijo_max_halvings; ++hv) {
      bl.copy(U.get(), trial.get());
      bl.axpy(alpha, delta.get(), trial.get());
      const double tnorm = residual_norm_dev(*this, trial.get(), Rt.get());
      if (tnorm < rnorm && tnorm <= (1.0 - cfg.armijo_slope * alpha) * rnorm) {
        bl.copy(trial.get(), U.get());
        bl.copy(Rt.get(), R.get());
        rnorm = tnorm;
        accepted = true;
        break;
      }
      alpha *= cfg.armijo_backtrack;
    }
    if (!accepted) {
      res.status = TP_STALLED;
      break;
    }
    res.iterations += 1;
    res.history.push_back(rnorm);
    if (stop()) {
      res.status = TP_CONVERGED;
      break;
    }
  }
  if (stop()) res.status = TP_CONVERGED;
  TP_CUDA(cudaStreamSynchronize(stream));
  uhat_valid = false;  // the preconditioner solves overwrote the M1 warm-start spectrum
}

}  // namespace tpgpu
