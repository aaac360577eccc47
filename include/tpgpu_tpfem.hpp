// tpgpu_tpfem.hpp -- reference-side binding: lets tpfem code (runner.hpp-style
// drivers, tests) call the B200 sweep through include/tpgpu.h with the
// reference's own types and signatures.
//
//   tpfem::PeriodicState U0 = tpgpu::static_init(prob, cfg);          // solvers.hpp:276-278
//   auto [U, rep] = tpgpu::solve_m1_fixed_point(prob, U0, cfg);       // solvers.hpp:301-306
//
// Requires the tpfem headers (tpfem/solvers.hpp) on the include path and
// libtpgpu.so at link time.  Header-only; the mapping of types is:
//   tpfem::SolverConfig   -> tp_solver_cfg      (solvers.hpp:49-69)
//   tpfem::SolveReport    <- tp_report + history (solvers.hpp:88-96)
//   tpfem::SolveError     <- TP_ESOLVE          (solve.hpp:17-26)
//   std::invalid_argument <- TP_EINVAL
#pragma once

#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "tpfem/solvers.hpp"
#include "tpgpu.h"

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

inline tpfem::PeriodicState static_init(GpuProblem& p, const tpfem::SolverConfig& cfg,
                                        std::vector<int>* newton_counts = nullptr) {
  tpfem::validate(cfg);
  tpfem::PeriodicState U(p.steps(), p.n_dof(), p.tau());
  std::vector<int32_t> counts(static_cast<std::size_t>(p.steps()));
  const tp_solver_cfg c = to_c(cfg);
  check(tp_static_init(p.get(), &c, U.data.data(), counts.data()));
  if (newton_counts) newton_counts->assign(counts.begin(), counts.end());
  return U;
}

/// choose_nu_hat (assembly.hpp:254-303) from the device state; returns q.
inline double choose_nu_hat(GpuProblem& p, const tpfem::SolverConfig& cfg,
                            std::array<double, tpfem::kNumRegions>* nu_hat = nullptr) {
  const tp_solver_cfg c = to_c(cfg);
  double nu[TP_MAX_MATERIALS], q = 0;
  check(tp_choose_nu_hat(p.get(), &c, nu, &q));
  if (nu_hat)
    for (int r = 0; r < tpfem::kNumRegions; ++r) (*nu_hat)[static_cast<std::size_t>(r)] = nu[r];
  return q;
}

/// solve_m1_fixed_point (solvers.hpp:301-369) with K_hat = the installed
/// frozen stiffness; iterate_log as in the reference.
inline std::pair<tpfem::PeriodicState, tpfem::SolveReport> solve_m1_fixed_point(
    GpuProblem& p, const tpfem::PeriodicState& U0, const tpfem::SolverConfig& cfg,
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
  check(tp_solve_m1(p.get(), &c, U0.data.data(), U.data.data(), &rep, hist.data(), contr.data(), cap,
                    iterate_log ? +cb : nullptr, &ctx));
  tpfem::SolveReport r;
  r.method = tpfem::Method::m1;
  r.iterations = rep.iterations;
  r.residual_history.assign(hist.begin(), hist.begin() + rep.history_len);
  r.contraction_history.assign(contr.begin(), contr.begin() + std::max(0, rep.history_len - 1));
  r.q_estimate = rep.q_estimate;
  r.wall_time = rep.wall_time;
  r.status = rep.status == TP_CONVERGED ? tpfem::SolveStatus::converged : tpfem::SolveStatus::max_iter;
  return {std::move(U), std::move(r)};
}

}  // namespace tpgpu
