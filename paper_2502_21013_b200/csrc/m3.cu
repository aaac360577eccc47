// M3: sequential implicit-Euler time stepping toward the limit cycle
// (solve_m3_timestepping, solvers.hpp:489-542) -- SURVEY.md §8(f) f4, the
// comparator the paper's periodic methods are measured against.
//
// Period after period from U0: step i solves M (u - u_{i-1})/tau + K(u) = f_i
// by the reference's damped Newton (newton_elliptic, solvers.hpp:131-182,
// mass_scale = 1/tau, started from u_{i-1}): Jacobian J(u) + M/tau (element
// stencil + lumped mass on the diagonal), its Galerkin hierarchy and a
// single-slice MG-PCG solve (the slice-mode batch solver with one batch),
// Armijo backtracking on the step residual.  Inherently sequential in time:
// every kernel works on one slice, so the path is launch/latency-bound -- it
// is here for completeness of the reference's method set, not for speed.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <memory>
#include <string>
#include <vector>

#include "mg.cuh"

namespace tpgpu {

double residual_norm_dev(Problem& p, const double* u, double* r);
void newton_residual(Problem& p, const double* Ub, const double* Db, const double* d_alpha, double* Ut,
                     double* Rt, const int* d_slice_of, const int* d_active, int batches, double* norms2_host,
                     DevBuf<double>& part, DevBuf<double>& red, const double* rhs, double ms);

namespace {

// rhs = f_i + (1/tau) M u_prev   (solvers.hpp:516-518; lumped M)
__global__ void k_m3_rhs(double* __restrict__ rhs, const double* __restrict__ uprev,
                         const double* __restrict__ mass, const double* __restrict__ src_prof,
                         const double* __restrict__ src_time, int nsrc, int slice, size_t n, double inv_tau) {
  for (size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x; j < n; j += (size_t)gridDim.x * blockDim.x) {
    double f = 0;
    for (int r = 0; r < nsrc; ++r) f += src_time[slice * nsrc + r] * src_prof[r * n + j];
    rhs[j] = f + inv_tau * (mass[j] * uprev[j]);
  }
}

// J_C += ms * M  (add_scaled(mass_scale, M, 1.0, J), lumped M on the diagonal)
__global__ void k_add_mass(double* __restrict__ Jc, const double* __restrict__ mass, double ms, size_t n) {
  for (size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x; j < n; j += (size_t)gridDim.x * blockDim.x)
    Jc[j] = ms * mass[j] + Jc[j];
}

__global__ void k_sq_part(const double* __restrict__ a, size_t n, double* __restrict__ part) {
  __shared__ double sh[8];
  double v = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    v = fma(a[i], a[i], v);
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0;
    for (int w = 0; w < 8; ++w) s += sh[w];
    part[blockIdx.x] = s;
  }
}

__global__ void k_accept1(double* __restrict__ u, double* __restrict__ r, const double* __restrict__ ut,
                          const double* __restrict__ rt, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    u[i] = ut[i];
    r[i] = rt[i];
  }
}

}  // namespace

void Problem::solve_m3_dev(const tp_solver_cfg& cfg, M2Result& res) {
  require(!sharded(), "m3: single-rank problems only");
  require(state_valid, "m3: no initial state");
  require(cfg.m3_max_cycles >= 1, "m3: iteration caps must be positive");
  // hierarchy of the single-slice Newton systems (as static_init)
  std::vector<int> ms;
  for (int cl = c;; cl /= 2) {
    ms.push_back(cl - 1);
    if (cl <= 8) break;
    require(cl % 2 == 0, "multigrid: cells per side must be 2^k * q with q <= 8");
  }
  const int nl = (int)ms.size();
  const int nL = ms.back() * ms.back();
  DevBuf<double> ub(n), rb(n), db(n), ut(n), rt(n), rhs(n), inv((size_t)nL * nL), part, red, sq(256);
  std::vector<DevBuf<double>> J(nl);
  for (int l = 0; l < nl; ++l) J[l].alloc((size_t)7 * ms[l] * ms[l]);
  DevBuf<int> d_slice(1), d_active(1), d_acc(1);
  DevBuf<double> d_alpha(1);
  const int one = 1;
  TP_CUDA(cudaMemcpyAsync(d_slice.get(), &one, sizeof(int), cudaMemcpyHostToDevice, stream));  // (unused: rhs given)
  TP_CUDA(cudaMemcpyAsync(d_active.get(), &one, sizeof(int), cudaMemcpyHostToDevice, stream));
  std::vector<LevelOp> ops(nl);
  for (int l = 0; l < nl; ++l) ops[l] = {ms[l], ms[l] * ms[l], J[l].get(), nullptr, false, {}};
  MGConfig mc;
  mc.rtol = std::max(cfg.inner_rtol, 1e-10);  // the reference SparseSolver's contract (solve.hpp:79-89)
  mc.max_iter = cfg.inner_max_iter;
  mc.omega = mc.omega2 = 0.6;
  if (TPGPU_SLICE_L1 && !std::getenv("TPGPU_TILE_SLICE")) {  // l1-Jacobi + Chebyshev (mg.cuh)
    mc.omega = kL1Omega1;
    mc.omega2 = kL1Omega2;
  }
  BatchSolver<1> solver;
  solver.init(this, ops, 1, mc);
  solver.coarse_inv = inv.get();
  const double inv_tau = 1.0 / tau;
  const int nsrc = (int)src_mats.size();
  const unsigned gb = (unsigned)std::min<size_t>((n + 255) / 256, 256);
  auto norm2 = [&](const double* a) {
    k_sq_part<<<gb, 256, 0, stream>>>(a, n, sq.get());
    TP_LAUNCHED(this);
    return std::sqrt(reduce_sum(*this, sq.get(), (int)gb));
  };
  double nrm2 = 0;
  auto residual_at = [&](const double* u, const double* d, double* ures, double* rres) {
    newton_residual(*this, u, d, d ? d_alpha.get() : nullptr, ures, rres, d_slice.get(), d_active.get(), 1, &nrm2,
                    part, red, rhs.get(), inv_tau);
    return std::sqrt(nrm2);
  };
  // newton_elliptic (solvers.hpp:131-182) on the slice in ub
  auto newton = [&](int cycle, int step_i) {
    const auto fail = [&](const std::string& what, double resid) {
      throw Error(TP_ESOLVE,
                  "time stepping, cycle " + std::to_string(cycle) + ", step " + std::to_string(step_i + 1) + ": " +
                      what,
                  resid);
    };
    double rnorm = residual_at(ub.get(), nullptr, nullptr, rb.get());
    const double scale = std::max(norm2(rhs.get()), rnorm);
    if (scale == 0 || rnorm <= cfg.static_tol * scale) return;
    for (int step = 1; step <= cfg.static_max_newton; ++step) {
      launch_element_stencil(*this, true, ub.get(), J[0].get(), 1);
      k_add_mass<<<gb, 256, 0, stream>>>(J[0].get() + (size_t)SC * n, d_mass.get(), inv_tau, n);
      TP_LAUNCHED(this);
      for (int l = 1; l < nl; ++l) launch_rap(*this, J[l - 1].get(), ms[l - 1], J[l].get(), ms[l], 1);
      launch_coarse_inverse_slice(*this, J[nl - 1].get(), ms[nl - 1], inv.get(), 1);
      SolveStats st;
      solver.solve(rb.get(), db.get(), 1, false, &st);
      double alpha = 1.0;
      bool accepted = false;
      for (int h = 0; h <= cfg.armijo_max_halvings; ++h) {
        TP_CUDA(cudaMemcpyAsync(d_alpha.get(), &alpha, sizeof(double), cudaMemcpyHostToDevice, stream));
        const double tnorm = residual_at(ub.get(), db.get(), ut.get(), rt.get());
        if (tnorm <= (1.0 - cfg.armijo_slope * alpha) * rnorm) {
          k_accept1<<<gb, 256, 0, stream>>>(ub.get(), rb.get(), ut.get(), rt.get(), n);
          TP_LAUNCHED(this);
          rnorm = tnorm;
          accepted = true;
          break;
        }
        alpha *= cfg.armijo_backtrack;
      }
      if (!accepted) fail("newton: line search exhausted at residual " + std::to_string(rnorm), rnorm / scale);
      if (rnorm <= cfg.static_tol * scale) return;
    }
    fail("newton: no convergence within " + std::to_string(cfg.static_max_newton) + " steps", rnorm / scale);
  };

  DevBuf<double> R((size_t)N * n);
  res.history.assign(1, residual_norm_dev(*this, U.get(), R.get()));
  res.status = TP_CONVERGED;
  res.iterations = 0;
  res.inner_total = 0;
  auto stop = [&] { return res.history.back() <= cfg.tol * res.history.front(); };
  // u_prev = U[N-1]
  TP_CUDA(cudaMemcpyAsync(ub.get(), U.get() + (size_t)(N - 1) * n, n * sizeof(double), cudaMemcpyDeviceToDevice,
                          stream));
  while (!stop()) {
    if (res.iterations >= cfg.m3_max_cycles) {
      res.status = TP_MAX_ITER;
      break;
    }
    for (int i = 0; i < N; ++i) {
      k_m3_rhs<<<gb, 256, 0, stream>>>(rhs.get(), ub.get(), d_mass.get(), d_src_prof.get(), d_src_time.get(), nsrc,
                                       i, n, inv_tau);
      TP_LAUNCHED(this);
      newton(res.iterations + 1, i);
      TP_CUDA(cudaMemcpyAsync(U.get() + (size_t)i * n, ub.get(), n * sizeof(double), cudaMemcpyDeviceToDevice,
                              stream));
    }
    res.iterations += 1;
    res.history.push_back(residual_norm_dev(*this, U.get(), R.get()));
    if (stop()) {
      res.status = TP_CONVERGED;
      break;
    }
  }
  if (stop()) res.status = TP_CONVERGED;
  TP_CUDA(cudaStreamSynchronize(stream));
  uhat_valid = false;
}

}  // namespace tpgpu
