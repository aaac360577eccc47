// tpgpu_tpfem.hpp -- reference-side binding: lets tpfem code (runner.hpp-style
// drivers, tests) call the B200 sweep through include/tpgpu.h with the
// reference's own types and signatures.
//
//   tpfem::PeriodicState U0 = tpgpu::static_init(prob, cfg);          // solvers.hpp:276-278
//   auto [U, rep] = tpgpu::solve_m1_fixed_point(prob, U0, cfg);       // solvers.hpp:301-306
//
// prob is a GpuProblem (BASELINE uniform grids, tpgpu.h) or a GpuMeshProblem
// built from the reference's own tpfem::Mesh + tpfem::MaterialTable
// (tpgpu_mesh.h: build_transformer_mesh / refine_uniform meshes, the
// reference's transformer physics).
//
// Requires the tpfem headers (tpfem/solvers.hpp) on the include path and
// libtpgpu.so at link time.  Header-only; the mapping of types is:
//   tpfem::SolverConfig   -> tp_solver_cfg      (solvers.hpp:49-69)
//   tpfem::SolveReport    <- tp_report + history (solvers.hpp:88-96)
//   tpfem::SolveError     <- TP_ESOLVE          (solve.hpp:17-26)
//   std::invalid_argument <- TP_EINVAL
#pragma once

#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "tpfem/assembly.hpp"
#include "tpfem/mesh.hpp"
#include "tpfem/solvers.hpp"
#include "tpgpu.h"
#include "tpgpu_mesh.h"

namespace tpgpu {

inline void check(int code) {
  if (code == TP_OK) return;
  char msg[1024];
  double res = -1;
  tp_last_error(msg, sizeof msg, &res);
  if (code == TP_EINVAL) throw std::invalid_argument(msg);
  if (code == TP_ESOLVE) throw tpfem::SolveError(msg, res);
  throw std::runtime_error(msg);
}

/// SolverConfig -> tp_solver_cfg.  Every field of the reference's config is
/// mapped or has no device meaning: `transform` (radix-2 vs direct DFT) only
/// selects the algorithm of the same transform (the device picks Stockham for
/// powers of two and a direct DFT otherwise); `cache` / `cache_budget_bytes`
/// govern the reference's per-frequency factor cache, and the device has no
/// factorisations to cache (matrix-free MG-COCG per block); `threads` is the
/// CPU worker count.  Those are accepted and validated, not silently dropped.
inline tp_solver_cfg to_c(const tpfem::SolverConfig& s) {
  tp_solver_cfg c;
  tp_solver_cfg_default(&c);
  c.tol = s.tol;
  c.m1_max_outer = s.m1_max_outer;
  c.armijo_slope = s.armijo.slope;
  c.armijo_backtrack = s.armijo.backtrack;
  c.armijo_max_halvings = s.armijo.max_halvings;
  c.nu_hat_mode = s.nu_hat_mode == tpfem::NuHatMode::theory ? TP_NU_HAT_THEORY : TP_NU_HAT_FROZEN_FIELD;
  c.imag_tol = s.imag_tol;
  c.static_tol = s.static_tol;
  c.static_max_newton = s.static_max_newton;
  c.threads = s.threads;
  c.m2_max_outer = s.m2_max_outer;
  c.m2_inner_tol = s.m2_inner_tol;
  c.m2_inner_max = s.m2_inner_max;
  c.m2_restart = s.m2_restart;
  c.m3_max_cycles = s.m3_max_cycles;
  c.track_error_contraction = s.track_error_contraction ? 1 : 0;
  return c;
}

/// Owning handle of a device-resident grid problem.
class GpuProblem {
 public:
  explicit GpuProblem(const tp_problem_desc& d, int device = 0) {
    tp_problem* p = nullptr;
    check(tp_problem_create(&d, device, &p));
    h_.reset(p);
    check(tp_problem_sizes(p, &n_, &steps_, &tau_));
  }
  tpfem::Index n_dof() const { return n_; }
  int steps() const { return steps_; }
  double tau() const { return tau_; }
  tp_problem* get() const { return h_.get(); }
  /// Problem::apply_k (periodic.hpp:29) on one slice.
  void apply_k(const double* u, double* out) const { check(tp_apply_k(h_.get(), u, out, 1)); }

 private:
  struct Del {
    void operator()(tp_problem* p) const { tp_problem_destroy(p); }
  };
  std::unique_ptr<tp_problem, Del> h_;
  int32_t n_ = 0, steps_ = 0;
  double tau_ = 0;
};

/// Owning handle of a device-resident problem on a reference mesh: the
/// setup_transformer pipeline (runner.hpp:46-73) up to static_init, from the
/// reference's own Mesh and MaterialTable (vertices, triangles, labels and
/// coefficients are passed through unchanged; dofs are numbered by the same
/// finalize_mesh rule, so states are interchangeable with tpfem's).
class GpuMeshProblem {
 public:
  GpuMeshProblem(const tpfem::Mesh& mesh, const tpfem::MaterialTable& mat, int steps, double period,
                 double s_max = 3.0, int flux_samples = 10001, int device = 0) {
    std::vector<double> xy;
    std::vector<int32_t> tri, reg;
    for (const auto& v : mesh.vertices) xy.insert(xy.end(), {v[0], v[1]});
    for (const auto& t : mesh.triangles) tri.insert(tri.end(), {(int32_t)t[0], (int32_t)t[1], (int32_t)t[2]});
    for (const auto r : mesh.region) reg.push_back(static_cast<int32_t>(r));
    tp_mesh_desc d{};
    d.n_vertices = static_cast<int32_t>(mesh.vertices.size());
    d.n_triangles = static_cast<int32_t>(mesh.triangles.size());
    d.vertices = xy.data();
    d.triangles = tri.data();
    d.region = reg.data();
    for (int r = 0; r < tpfem::kNumRegions; ++r) {
      const auto& m = mat.at(static_cast<tpfem::Region>(r));
      d.material[r] = tp_exp_material{m.sigma, m.a, m.b, m.c, m.d, m.j_amp};
    }
    d.steps = steps;
    d.period = period;
    d.s_max = s_max;
    d.flux_samples = flux_samples;
    tp_mesh_problem* p = nullptr;
    check(tp_mesh_problem_create(&d, device, &p));
    h_.reset(p);
    check(tp_mesh_problem_sizes(p, &n_, &steps_, &tau_, &bw_));
  }
  tpfem::Index n_dof() const { return n_; }
  int steps() const { return steps_; }
  double tau() const { return tau_; }
  tp_mesh_problem* get() const { return h_.get(); }
  void apply_k(const double* u, double* out) const { check(tp_mesh_apply_k(h_.get(), u, out, 1)); }

 private:
  struct Del {
    void operator()(tp_mesh_problem* p) const { tp_mesh_problem_destroy(p); }
  };
  std::unique_ptr<tp_mesh_problem, Del> h_;
  int32_t n_ = 0, steps_ = 0, bw_ = 0;
  double tau_ = 0;
};

namespace detail {
// the C entry points of each problem kind
inline int c_static_init(GpuProblem& p, const tp_solver_cfg* c, double* U, int32_t* n) {
  return tp_static_init(p.get(), c, U, n);
}
inline int c_static_init(GpuMeshProblem& p, const tp_solver_cfg* c, double* U, int32_t* n) {
  return tp_mesh_static_init(p.get(), c, U, n);
}
inline int c_choose(GpuProblem& p, const tp_solver_cfg* c, double* nu, double* q) {
  return tp_choose_nu_hat(p.get(), c, nu, q);
}
inline int c_choose(GpuMeshProblem& p, const tp_solver_cfg* c, double* nu, double* q) {
  return tp_mesh_choose_nu_hat(p.get(), c, nu, q);
}
inline int c_loads(GpuProblem& p, double* F) { return tp_problem_loads(p.get(), F); }
inline int c_loads(GpuMeshProblem& p, double* F) { return tp_mesh_loads(p.get(), F); }
inline int c_m1(GpuProblem& p, const tp_solver_cfg* c, const double* U0, double* U, tp_report* r, double* h,
                double* ct, int32_t cap, tp_iterate_cb cb, void* u) {
  return tp_solve_m1(p.get(), c, U0, U, r, h, ct, cap, cb, u);
}
inline int c_m1(GpuMeshProblem& p, const tp_solver_cfg* c, const double* U0, double* U, tp_report* r, double* h,
                double* ct, int32_t cap, tp_iterate_cb cb, void* u) {
  return tp_mesh_solve_m1(p.get(), c, U0, U, r, h, ct, cap, cb, u);
}
}  // namespace detail

template <class P>
inline tpfem::PeriodicState static_init(P& p, const tpfem::SolverConfig& cfg,
                                        std::vector<int>* newton_counts = nullptr) {
  tpfem::validate(cfg);
  tpfem::PeriodicState U(p.steps(), p.n_dof(), p.tau());
  std::vector<int32_t> counts(static_cast<std::size_t>(p.steps()));
  const tp_solver_cfg c = to_c(cfg);
  check(detail::c_static_init(p, &c, U.data.data(), counts.data()));
  if (newton_counts) newton_counts->assign(counts.begin(), counts.end());
  return U;
}

/// choose_nu_hat (assembly.hpp:254-303) from the device state; returns q.
template <class P>
inline double choose_nu_hat(P& p, const tpfem::SolverConfig& cfg,
                            std::array<double, tpfem::kNumRegions>* nu_hat = nullptr) {
  const tp_solver_cfg c = to_c(cfg);
  double nu[TP_MAX_MATERIALS], q = 0;
  check(detail::c_choose(p, &c, nu, &q));
  if (nu_hat)
    for (int r = 0; r < tpfem::kNumRegions; ++r) (*nu_hat)[static_cast<std::size_t>(r)] = nu[r];
  return q;
}

/// solve_m1_fixed_point (solvers.hpp:301-369) with K_hat = the installed
/// frozen stiffness; iterate_log as in the reference.
template <class P>
inline std::pair<tpfem::PeriodicState, tpfem::SolveReport> solve_m1_fixed_point(
    P& p, const tpfem::PeriodicState& U0, const tpfem::SolverConfig& cfg,
    std::vector<tpfem::PeriodicState>* iterate_log = nullptr) {
  tpfem::validate(cfg);
  const tp_solver_cfg c = to_c(cfg);
  const int cap = cfg.m1_max_outer + 1;
  std::vector<double> hist(static_cast<std::size_t>(cap)), contr(static_cast<std::size_t>(cap));
  tpfem::PeriodicState U(p.steps(), p.n_dof(), p.tau());
  tp_report rep{};
  struct Log {
    std::vector<tpfem::PeriodicState>* log;
    const tpfem::PeriodicState* shape;
  } ctx{iterate_log, &U0};
  auto cb = [](int32_t, const double* u, double, void* user) -> int {
    auto* c2 = static_cast<Log*>(user);
    tpfem::PeriodicState s(c2->shape->steps, c2->shape->n_dof, c2->shape->tau);
    std::copy(u, u + s.data.size(), s.data.begin());
    c2->log->push_back(std::move(s));
    return 0;
  };
  check(detail::c_m1(p, &c, U0.data.data(), U.data.data(), &rep, hist.data(), contr.data(), cap,
                    iterate_log ? +cb : nullptr, &ctx));
  tpfem::SolveReport r;
  r.method = tpfem::Method::m1;
  r.iterations = rep.iterations;
  r.residual_history.assign(hist.begin(), hist.begin() + rep.history_len);
  r.contraction_history.assign(contr.begin(), contr.begin() + rep.contraction_len);
  r.q_estimate = rep.q_estimate;
  r.wall_time = rep.wall_time;
  r.status = rep.status == TP_CONVERGED ? tpfem::SolveStatus::converged : tpfem::SolveStatus::max_iter;
  return {std::move(U), std::move(r)};
}

/// The reference's full signature (solvers.hpp:301-306): K_hat and F are
/// the problem's own frozen stiffness and loads (runner.hpp:68,
/// assembly.hpp:68-106), which the device problem assembles itself from the
/// installed nu_hat and the source description; their shapes are checked and
/// F is compared against the device loads, so a caller passing different
/// operators gets std::invalid_argument instead of a silently different
/// solve.  q_estimate is reported back as SolveReport::q_estimate.
template <class P>
inline std::pair<tpfem::PeriodicState, tpfem::SolveReport> solve_m1_fixed_point(
    P& p, const tpfem::SparseMatrix<double>& K_hat, const tpfem::BlockRhs& F, const tpfem::PeriodicState& U0,
    const tpfem::SolverConfig& cfg, double q_estimate = std::numeric_limits<double>::quiet_NaN(),
    std::vector<tpfem::PeriodicState>* iterate_log = nullptr) {
  if (K_hat.rows() != p.n_dof() || K_hat.cols() != p.n_dof() || F.steps != p.steps() || F.n_dof != p.n_dof() ||
      U0.steps != p.steps() || U0.n_dof != p.n_dof())
    throw std::invalid_argument("fixed-point solver: shape mismatch");
  std::vector<double> Fd(F.data.size());
  check(detail::c_loads(p, Fd.data()));
  double num = 0, den = 0;
  for (std::size_t i = 0; i < Fd.size(); ++i) {
    num += (Fd[i] - F.data[i]) * (Fd[i] - F.data[i]);
    den += F.data[i] * F.data[i];
  }
  if (num > 1e-24 * std::max(den, 1e-300))
    throw std::invalid_argument("fixed-point solver: F differs from the device problem's loads");
  auto out = solve_m1_fixed_point(p, U0, cfg, iterate_log);
  out.second.q_estimate = q_estimate;
  return out;
}

}  // namespace tpgpu
