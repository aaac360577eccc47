// Static initialisation on the device: per-slice damped Newton for
// K(u^s) = f^s from u = 0, batched over a chunk of slices.
//
// Reference: static_init (solvers.hpp:276-296) -> newton_elliptic
// (solvers.hpp:131-182) with mass_scale = 0: the Jacobian J(u)
// (assembly.hpp:153-177) is assembled as a 7-point stencil per slice, solved
// by the batched MG-PCG of mg.cu (slice mode; the reference factorises J
// with SimplicialLDLT), then an Armijo backtracking search per slice
// (slope, factor, cap from SolverConfig::armijo).  The accept/reject
// decisions and the stopping tests are made on the host from device-reduced
// norms, in exactly the reference's order and arithmetic.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <string>
#include <thread>

#include "mg.cuh"

namespace tpgpu {

void newton_residual(Problem& p, const double* Ub, const double* Db, const double* d_alpha, double* Ut,
                     double* Rt, const int* d_slice_of, const int* d_active, int batches,
                     double* norms2_host, DevBuf<double>& part, DevBuf<double>& red,
                     const double* rhs = nullptr, double ms = 0.0);

namespace {
__global__ void k_accept(double* __restrict__ Ub, double* __restrict__ Rb, const double* __restrict__ Ut,
                         const double* __restrict__ Rt, const int* __restrict__ acc, size_t n) {
  const int b = blockIdx.y;
  if (!acc[b]) return;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    Ub[b * n + i] = Ut[b * n + i];
    Rb[b * n + i] = Rt[b * n + i];
  }
}
// x_b *= f_b (the warm start of the next Newton step's linear solve)
__global__ void k_scale_batches(double* __restrict__ x, const double* __restrict__ f, size_t n) {
  const double a = f[blockIdx.y];
  double* xb = x + (size_t)blockIdx.y * n;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    xb[i] *= a;
}
}  // namespace

// Inexact Newton safeguards: the linear error's share of the
// accepted residual (kSteer), and within kNear of the stopping threshold
// kSteerNear; default forcing gamma and eta_max.
constexpr double kSteer = 0.1, kSteerNear = 1e-6, kNear = 1e4;
constexpr double kForcingGamma = 1e-2, kForcingMax = 1e-2;

// One group of slices [g0, g1): its own buffers, batch solver and (when the
// slices are split into concurrent groups) its own stream / host thread.
struct NewtonGroup {
  int S = 0;  // slices per batch
  DevBuf<double> Ub, Rb, Db, Ut, Rt, inv, part, red;
  std::vector<DevBuf<double>> J;
  std::vector<DevBuf<float>> Jf;  // fp32 C/E/N/NE planes of the non-coarsest levels (V-cycle passes)
  DevBuf<int> d_slice, d_active, d_acc, d_todo;
  DevBuf<double> d_alpha, d_bscale, d_wscale;
  BatchSolver<1> solver;
};

void Problem::static_init_dev(const tp_solver_cfg& cfg, int32_t* newton_counts) {
  // geometry of the hierarchy
  std::vector<int> ms;
  for (int cl = c;; cl /= 2) {
    ms.push_back(cl - 1);
    if (cl <= 8) break;
    require(cl % 2 == 0, "multigrid: cells per side must be 2^k * q with q <= 8");
  }
  const int nl = (int)ms.size();
  const int nL = ms.back() * ms.back();
  size_t per_slice = 0;  // bytes
  for (int l = 0; l < nl; ++l) per_slice += (size_t)ms[l] * ms[l] * (8 * (7 + 3) + 4 * 4);
  per_slice += (size_t)n * 8 * 9 + (size_t)nL * nL * 8;
  size_t free_b = 0, total_b = 0;
  TP_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const int Nr = sh.s1 - sh.s0;
  int S = cfg.slice_chunk > 0 ? cfg.slice_chunk : (int)std::min<size_t>(Nr, (size_t)(0.5 * free_b) / per_slice);
  S = std::max(1, std::min(S, Nr));
  // equal batches (464 + 48 slices at cfg 2 ran the short batch's Newton and
  // PCG iterations at a tenth of the occupancy)
  if (cfg.slice_chunk <= 0) {
    const int nbatch = (Nr + S - 1) / S;
    S = (Nr + nbatch - 1) / nbatch;
  }
  // optional concurrent slice groups (TPGPU_SLICE_GROUPS, as the frequency
  // groups of the periodic solve).  Off by default: the Newton loop is a chain
  // of short launches and host decisions, and concurrent host threads measured
  // slower at cfg 1 (0.31-0.96 s vs 0.20 s) and no faster at cfg 2.
  const int want = std::getenv("TPGPU_SLICE_GROUPS") ? std::atoi(std::getenv("TPGPU_SLICE_GROUPS")) : 1;
  const int G = std::max(1, std::min(want, S));
  const int Sg = (S + G - 1) / G;

  MGConfig mc;
  // Newton steps are solved to the reference SparseSolver's own residual
  // contract (1e-10, solve.hpp:79-89) -- tighter buys nothing: Newton counts
  // and U0 are unchanged (cfg 0/1 parity tests), init 258 -> 215 ms at cfg 1
  mc.rtol = std::max(cfg.inner_rtol, 1e-10);
  if (const char* e = std::getenv("TPGPU_NEWTON_RTOL")) mc.rtol = std::atof(e);
  mc.max_iter = cfg.inner_max_iter;
  // Newton Jacobians carry the anisotropic rank-one term (nu'/s) g g^T, so
  // lambda_max(D^-1 J) can exceed 2: plain damped Jacobi with a safe weight
  // keeps the V-cycle symmetric positive definite (the Chebyshev pair of the
  // frequency solver assumes a spectrum in (0, 2]).
  mc.omega = mc.omega2 = 0.6;
  if (TPGPU_SLICE_L1 && !std::getenv("TPGPU_TILE_SLICE")) {  // l1-Jacobi + Chebyshev (mg.cuh)
    mc.omega = kL1Omega1;
    mc.omega2 = kL1Omega2;
  }
  if (const char* e = std::getenv("TPGPU_NEWTON_OMEGA")) mc.omega = mc.omega2 = std::atof(e);
  if (const char* e = std::getenv("TPGPU_NEWTON_OMEGA2")) mc.omega2 = std::atof(e);

  // inexact Newton forcing terms (gamma, eta_max; TPGPU_NEWTON_FORCING=0 off)
  double f_gamma = kForcingGamma, f_max = kForcingMax;
  if (const char* e = std::getenv("TPGPU_NEWTON_FORCING")) {
    f_gamma = 0;
    std::sscanf(e, "%lf,%lf", &f_gamma, &f_max);
  }
  const bool forcing = f_gamma > 0;

  // fp32 copies of the Jacobian planes for the V-cycle passes (the PCG
  // operator stays fp64; only the preconditioner reads rounded coefficients).
  // Opt-in (TPGPU_NEWTON_F32=1): no measurable change (cfg 2 4.55 vs 4.53 s,
  // cfg 3 30.0 vs 30.0 s, profiles/r2zb_init_ab.txt) -- the slice-mode passes
  // are latency-bound, not bound by their coefficient bytes
  const bool f32_planes = std::getenv("TPGPU_NEWTON_F32") && std::atoi(std::getenv("TPGPU_NEWTON_F32")) != 0;

  std::vector<std::unique_ptr<NewtonGroup>> groups(G);
  for (auto& gp : groups) {
    gp = std::make_unique<NewtonGroup>();
    NewtonGroup& g = *gp;
    g.S = Sg;
    for (auto* b : {&g.Ub, &g.Rb, &g.Db, &g.Ut, &g.Rt}) b->alloc((size_t)Sg * n);
    g.J.resize(nl);
    for (int l = 0; l < nl; ++l) g.J[l].alloc((size_t)Sg * 7 * ms[l] * ms[l]);
    if (f32_planes) {
      g.Jf.resize(nl);
      for (int l = 0; l + 1 < nl; ++l) g.Jf[l].alloc((size_t)Sg * 4 * ms[l] * ms[l]);
    }
    g.inv.alloc((size_t)Sg * nL * nL);
    g.d_slice.alloc(Sg);
    g.d_active.alloc(Sg);
    g.d_acc.alloc(Sg);
    g.d_todo.alloc(Sg);
    g.d_alpha.alloc(Sg);
    g.d_bscale.alloc(Sg);
    g.d_wscale.alloc(Sg);
    std::vector<LevelOp> ops(nl);
    for (int l = 0; l < nl; ++l) {
      ops[l] = {ms[l], ms[l] * ms[l], g.J[l].get(), nullptr, false, {}};
      if (f32_planes && l + 1 < nl) ops[l].Kf = g.Jf[l].get();
    }
    g.solver.init(this, ops, Sg, mc);
    g.solver.coarse_inv = g.inv.get();
  }
  std::vector<int> counts(N, 0);
  // slices of this rank (all of them on a single GPU); sharded problems
  // solve their slice block on the full grid and redistribute to strips
  DevBuf<double> Us;
  if (sharded()) Us.alloc((size_t)(sh.s1 - sh.s0) * n);

  // damped Newton over the slices [r0, r1) of this rank, batches of g.S
  auto run_group = [&](NewtonGroup& g, int r0, int r1) {
    const int Sb = g.S;
    cudaStream_t s = cur_stream();
    static const bool tracing = std::getenv("TPGPU_TRACE") != nullptr;
    StreamTrace trace;
    if (tracing) {
      tl_trace = &trace;
      trace_mark("start", s);
    }
    std::vector<int> h_slice(Sb), h_active(Sb), h_acc(Sb);
    std::vector<double> h_alpha(Sb), rnorm(Sb), scale(Sb), nrm2(Sb), h_bscale(Sb, 1.0), rprev(Sb), h_wscale(Sb);
    std::vector<double> acc_alpha(Sb, 1.0);
    const bool newton_warm = std::getenv("TPGPU_NEWTON_WARM") && std::atoi(std::getenv("TPGPU_NEWTON_WARM")) != 0;
    for (int s0 = r0; s0 < r1; s0 += Sb) {
      const int nb = std::min(Sb, r1 - s0);
      for (int b = 0; b < Sb; ++b) {
        h_slice[b] = std::min(s0 + b, N - 1);
        h_active[b] = b < nb;
      }
      TP_CUDA(cudaMemcpyAsync(g.d_slice.get(), h_slice.data(), Sb * sizeof(int), cudaMemcpyHostToDevice, s));
      TP_CUDA(cudaMemcpyAsync(g.d_active.get(), h_active.data(), Sb * sizeof(int), cudaMemcpyHostToDevice, s));
      TP_CUDA(cudaMemsetAsync(g.Ub.get(), 0, g.Ub.bytes(), s));
      // r = f - K(0) = f ; scale = max(||f||, ||r||)  (solvers.hpp:148-152)
      newton_residual(*this, g.Ub.get(), nullptr, nullptr, nullptr, g.Rb.get(), g.d_slice.get(), g.d_active.get(),
                      Sb, nrm2.data(), g.part, g.red);
      for (int b = 0; b < nb; ++b) {
        rprev[b] = -1.0;
        rnorm[b] = std::sqrt(nrm2[b]);
        scale[b] = std::max(rnorm[b], rnorm[b]);
        if (scale[b] == 0 || rnorm[b] <= cfg.static_tol * scale[b]) h_active[b] = 0;
      }
      for (int step = 1; step <= cfg.static_max_newton; ++step) {
        int n_active = 0;
        for (int b = 0; b < nb; ++b) n_active += h_active[b];
        if (n_active == 0) break;
        TP_CUDA(cudaMemcpyAsync(g.d_active.get(), h_active.data(), Sb * sizeof(int), cudaMemcpyHostToDevice, s));
        // J(u) for the batch, Galerkin hierarchy, coarsest inverses
        trace_mark("jacobian", s);
        launch_element_stencil(*this, true, g.Ub.get(), g.J[0].get(), nb);
        for (int l = 1; l < nl; ++l) launch_rap(*this, g.J[l - 1].get(), ms[l - 1], g.J[l].get(), ms[l], nb);
        launch_coarse_inverse_slice(*this, g.J[nl - 1].get(), ms[nl - 1], g.inv.get(), nb);
        if (f32_planes)
          for (int l = 0; l + 1 < nl; ++l) launch_planes_f32(*this, g.J[l].get(), ms[l], g.Jf[l].get(), nb);
        // delta = J^{-1} r  (masked to the active slices), then the Armijo
        // backtracking search (solvers.hpp:158-177).  Inexact Newton (DESIGN
        // §5e): a slice's linear tolerance eta follows its observed contraction
        // (Eisenstat-Walker, eta = gamma (r_k / r_{k-1})^2 in [rtol, eta_max]),
        // and a step is kept only when the linear error cannot have steered it:
        // the residual perturbation alpha eta r_k must be small against the
        // accepted residual (and tiny near the stopping threshold).  Otherwise
        // the step is re-solved warm to the full tolerance and searched again,
        // so the accept/reject decisions and the counts are the exact solve's.
        std::vector<double> eta(Sb, mc.rtol), rstart(rnorm);
        std::vector<int> todo(h_active.begin(), h_active.end());
        if (forcing)
          for (int b = 0; b < nb; ++b) {
            if (!h_active[b]) continue;
            const double ratio = rprev[b] > 0 ? rnorm[b] / rprev[b] : 1.0;
            const double rpred = rnorm[b] * ratio * ratio;
            eta[b] = rpred <= kNear * cfg.static_tol * scale[b]
                         ? mc.rtol
                         : std::min(f_max, std::max(mc.rtol, f_gamma * ratio * ratio));
          }
        SolveStats st;
        int halvings = 0, refined = 0;
        for (int b = 0; b < Sb; ++b) h_acc[b] = 0;
        for (int pass = 0; pass < 2; ++pass) {
          bool loose = false;
          for (int b = 0; b < nb; ++b) {
            h_bscale[b] = (eta[b] / mc.rtol) * (eta[b] / mc.rtol);
            loose = loose || (todo[b] && eta[b] > mc.rtol);
          }
          TP_CUDA(cudaMemcpyAsync(g.d_todo.get(), todo.data(), Sb * sizeof(int), cudaMemcpyHostToDevice, s));
          g.solver.ext_mask = g.d_todo.get();
          if (loose) {
            TP_CUDA(cudaMemcpyAsync(g.d_bscale.get(), h_bscale.data(), Sb * sizeof(double), cudaMemcpyHostToDevice, s));
            g.solver.bscale = g.d_bscale.get();
          }
          // warm start of a new step (TPGPU_NEWTON_WARM=1): the part of the
          // previous direction the line search left, (1 - alpha) delta_{k-1}
          // -- only the linear solver's initial guess changes.  Opt-in: cfg 2
          // 4.9 -> 4.7 s, cfg 1 0.3 -> 0.9 s (profiles/r2x_init_ab.txt)
          bool warm_lin = pass > 0;
          if (pass == 0 && newton_warm && step > 1) {
            for (int b = 0; b < Sb; ++b) h_wscale[b] = (b < nb && h_active[b]) ? 1.0 - acc_alpha[b] : 0.0;
            TP_CUDA(cudaMemcpyAsync(g.d_wscale.get(), h_wscale.data(), Sb * sizeof(double), cudaMemcpyHostToDevice, s));
            dim3 gw((unsigned)std::min<size_t>((n + 255) / 256, 512), Sb);
            k_scale_batches<<<gw, 256, 0, s>>>(g.Db.get(), g.d_wscale.get(), n);
            TP_LAUNCHED(this);
            warm_lin = true;
          }
          g.solver.solve(g.Rb.get(), g.Db.get(), nb, warm_lin, &st);
          g.solver.ext_mask = nullptr;
          g.solver.bscale = nullptr;
          std::vector<int> searching(todo), refine(Sb, 0);
          for (int b = 0; b < Sb; ++b) h_alpha[b] = 1.0;
          trace_mark("linesearch", s);
          for (int h = 0; h <= cfg.armijo_max_halvings; ++h) {
            int any = 0;
            for (int b = 0; b < nb; ++b) any += searching[b];
            if (!any) break;
            halvings = std::max(halvings, h);
            TP_CUDA(cudaMemcpyAsync(g.d_alpha.get(), h_alpha.data(), Sb * sizeof(double), cudaMemcpyHostToDevice, s));
            TP_CUDA(cudaMemcpyAsync(g.d_acc.get(), searching.data(), Sb * sizeof(int), cudaMemcpyHostToDevice, s));
            newton_residual(*this, g.Ub.get(), g.Db.get(), g.d_alpha.get(), g.Ut.get(), g.Rt.get(), g.d_slice.get(),
                            g.d_acc.get(), Sb, nrm2.data(), g.part, g.red);
            std::vector<int> accept(Sb, 0);
            for (int b = 0; b < nb; ++b) {
              if (!searching[b]) continue;
              const double tnorm = std::sqrt(nrm2[b]);
              if (tnorm <= (1.0 - cfg.armijo_slope * h_alpha[b]) * rstart[b]) {
                searching[b] = 0;
                const double pert = h_alpha[b] * eta[b] * rstart[b];
                const bool near = tnorm <= kNear * cfg.static_tol * scale[b];
                if (eta[b] > mc.rtol && (pert > kSteer * tnorm || (near && pert > kSteerNear * tnorm))) {
                  refine[b] = 1;
                  continue;
                }
                accept[b] = 1;
                rnorm[b] = tnorm;
                h_acc[b] = 1;
                acc_alpha[b] = h_alpha[b];
              } else {
                h_alpha[b] *= cfg.armijo_backtrack;
              }
            }
            TP_CUDA(cudaMemcpyAsync(g.d_acc.get(), accept.data(), Sb * sizeof(int), cudaMemcpyHostToDevice, s));
            dim3 gr((unsigned)std::min<size_t>((n + 255) / 256, 1024), Sb);
            k_accept<<<gr, 256, 0, s>>>(g.Ub.get(), g.Rb.get(), g.Ut.get(), g.Rt.get(), g.d_acc.get(), n);
            TP_LAUNCHED(this);
            TP_CUDA(cudaStreamSynchronize(s));
          }
          // a loose step whose search was exhausted is re-solved too
          int nref = 0;
          for (int b = 0; b < nb; ++b) {
            if (searching[b] && eta[b] > mc.rtol) refine[b] = 1;
            nref += refine[b];
          }
          if (nref == 0) break;
          refined += nref;
          for (int b = 0; b < nb; ++b) {
            todo[b] = refine[b];
            if (refine[b]) eta[b] = mc.rtol;
          }
        }
        for (int b = 0; b < nb; ++b)
          if (h_active[b]) rprev[b] = rstart[b];
        static const bool dbg_newton = std::getenv("TPGPU_DEBUG_NEWTON") != nullptr;
        if (dbg_newton) {
          int na = 0;
          double worst = 0;
          for (int b = 0; b < nb; ++b)
            if (h_active[b]) {
              ++na;
              worst = std::max(worst, rnorm[b] / scale[b]);
            }
          std::fprintf(stderr,
                       "newtondbg slices %d-%d step %d active %d pcg %d halvings %d refined %d worst_rel %.3e\n", s0,
                       s0 + nb - 1, step, na, st.iterations, halvings, refined, worst);
        }
        if (std::getenv("TPGPU_DEBUG_NEWTON") && std::atoi(std::getenv("TPGPU_DEBUG_NEWTON")) >= 2)
          for (int b = 0; b < nb; ++b)
            if (h_active[b])
              std::fprintf(stderr, "newtonslice %d step %d alpha %.17g rel %.17g\n", s0 + b, step, h_alpha[b],
                           rnorm[b] / scale[b]);
        for (int b = 0; b < nb; ++b) {
          if (!h_active[b]) continue;
          if (!h_acc[b])
            throw Error(TP_ESOLVE,
                        "static init, step " + std::to_string(s0 + b + 1) +
                            ": newton: line search exhausted at residual " + std::to_string(rnorm[b]),
                        rnorm[b] / scale[b]);
          if (rnorm[b] <= cfg.static_tol * scale[b]) {
            counts[s0 + b] = step;
            h_active[b] = 0;
          }
        }
      }
      for (int b = 0; b < nb; ++b)
        if (h_active[b])
          throw Error(TP_ESOLVE,
                      "static init, step " + std::to_string(s0 + b + 1) + ": newton: no convergence within " +
                          std::to_string(cfg.static_max_newton) + " steps",
                      rnorm[b] / scale[b]);
      trace_mark("store", s);
      double* dst = sharded() ? Us.get() + (size_t)(s0 - sh.s0) * n : U.get() + (size_t)s0 * n;
      TP_CUDA(cudaMemcpyAsync(dst, g.Ub.get(), (size_t)nb * n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
    TP_CUDA(cudaStreamSynchronize(s));
    if (tracing) {
      trace_mark("end", s);
      tl_trace = nullptr;
      trace_report(trace, "trace static_init", s);
    }
  };

  if (G == 1) {
    run_group(*groups[0], sh.s0, sh.s1);
  } else {
    // contiguous slice ranges per group, each on its own stream and host thread
    std::vector<cudaStream_t> hs(G, nullptr);
    for (auto& h : hs) TP_CUDA(cudaStreamCreateWithFlags(&h, cudaStreamNonBlocking));
    cudaEvent_t ev = nullptr;
    TP_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    TP_CUDA(cudaEventRecord(ev, stream));
    for (auto h : hs) TP_CUDA(cudaStreamWaitEvent(h, ev, 0));
    std::vector<std::exception_ptr> err(G);
    auto body = [&](int gi) {
      const int r0 = sh.s0 + (int)((long)Nr * gi / G), r1 = sh.s0 + (int)((long)Nr * (gi + 1) / G);
      try {
        if (gi > 0) TP_CUDA(cudaSetDevice(device));
        tl_stream = hs[gi];
        run_group(*groups[gi], r0, r1);
      } catch (...) {
        err[gi] = std::current_exception();
      }
      tl_stream = nullptr;
    };
    std::vector<std::thread> th;
    for (int gi = 1; gi < G; ++gi) th.emplace_back(body, gi);
    body(0);
    for (auto& t : th) t.join();
    for (auto h : hs) {
      TP_CUDA(cudaStreamSynchronize(h));
      cudaStreamDestroy(h);
    }
    cudaEventDestroy(ev);
    for (auto& e : err)
      if (e) std::rethrow_exception(e);
  }
  TP_CUDA(cudaStreamSynchronize(stream));
  if (sharded()) {
    slices_to_strips(Us.get());
    global_sum_ints(counts);  // every rank reports all N counts
  }
  if (newton_counts)
    for (int s = 0; s < N; ++s) newton_counts[s] = counts[s];
}

}  // namespace tpgpu
