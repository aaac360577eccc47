// TEST INFRASTRUCTURE ONLY -- C ABI over the reference's own solver templates
// (built by oracle/Makefile into oracle/_ref/libtpref.so; never linked into
// the product).  Used by tests/ as the parity checker, by bench.py's
// cpu_baseline leg and by `bench.py --impl reference`.
//
// Every entry point drives reference code unchanged:
//   tpref_static_init   -> tpfem::static_init            (solvers.hpp:276-296)
//   tpref_solve_m1      -> tpfem::solve_m1_fixed_point   (solvers.hpp:301-369)
//   tpref_solve_m2      -> tpfem::solve_m2_newton        (solvers.hpp:375-484)
//   tpref_solve_m3      -> tpfem::solve_m3_timestepping  (solvers.hpp:489-542)
//   tpref_periodic_solve-> tpfem::PeriodicSolver::solve  (periodic.hpp:154-198)
//   tpref_residual      -> tpfem::residual + block_l2    (periodic.hpp:35-67)
// with tporacle::GridProblem (grid_problem.hpp) supplying the BASELINE physics,
// and (tpref_tr_*) the reference's own transformer problem end to end
// (build_rectilinear_mesh + refine_uniform, MaterialTable::transformer,
// NonlinearOperator, assemble_mass / assemble_loads, FemProblem: the
// setup_transformer pipeline, runner.hpp:27-73) for the general-mesh path.
#include <chrono>
#include <cstring>
#include <string>
#include <thread>

#include "grid_problem.hpp"
#include "tpfem/assembly.hpp"
#include "tpfem/mesh.hpp"
#include "tpfem/periodic.hpp"
#include "tpfem/solvers.hpp"
#include "../include/tpgpu_baseline.h"
#include "../include/tpgpu_mesh.h"

namespace {

thread_local std::string g_err;
thread_local double g_err_res = -1;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return TP_OK;
  } catch (const tpfem::SolveError& e) {
    g_err = e.what();
    g_err_res = e.residual();
    return TP_ESOLVE;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    g_err_res = -1;
    return TP_EINVAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    g_err_res = -1;
    return TP_EINVAL;
  }
}

tpfem::SolverConfig to_ref(const tp_solver_cfg* c) {
  tpfem::SolverConfig s;
  if (!c) return s;
  s.tol = c->tol;
  s.m1_max_outer = c->m1_max_outer;
  s.armijo.slope = c->armijo_slope;
  s.armijo.backtrack = c->armijo_backtrack;
  s.armijo.max_halvings = c->armijo_max_halvings;
  s.nu_hat_mode = c->nu_hat_mode == TP_NU_HAT_THEORY ? tpfem::NuHatMode::theory
                                                     : tpfem::NuHatMode::frozen_field;
  s.imag_tol = c->imag_tol;
  s.static_tol = c->static_tol;
  s.static_max_newton = c->static_max_newton;
  if (c->m2_max_outer > 0) s.m2_max_outer = c->m2_max_outer;
  if (c->m2_inner_tol > 0) s.m2_inner_tol = c->m2_inner_tol;
  if (c->m2_inner_max > 0) s.m2_inner_max = c->m2_inner_max;
  if (c->m2_restart > 0) s.m2_restart = c->m2_restart;
  if (c->m3_max_cycles > 0) s.m3_max_cycles = c->m3_max_cycles;
  s.track_error_contraction = c->track_error_contraction != 0;
  s.threads = c->threads > 0 ? c->threads
                             : static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  return s;
}

tpfem::PeriodicState state_from(const tporacle::GridProblem& p, const double* U) {
  tpfem::PeriodicState s(p.steps(), p.n_dof(), p.tau());
  std::memcpy(s.data.data(), U, s.data.size() * sizeof(double));
  return s;
}

std::array<double, tpfem::kNumRegions> nu_array(const double* nu_hat) {
  std::array<double, tpfem::kNumRegions> a{};
  for (int r = 0; r < tpfem::kNumRegions; ++r) a[static_cast<std::size_t>(r)] = nu_hat[r];
  return a;
}

}  // namespace

extern "C" {

int tpref_last_error(char* buf, size_t cap, double* achieved) {
  if (buf && cap) {
    std::strncpy(buf, g_err.c_str(), cap - 1);
    buf[cap - 1] = 0;
  }
  if (achieved) *achieved = g_err_res;
  return TP_OK;
}

int tpref_desc_baseline(int32_t config, tp_problem_desc* d) {
  return tp_baseline_desc_fill(config, d) == 0 ? TP_OK : TP_EINVAL;
}

int tpref_hardware_threads(void) { return static_cast<int>(std::thread::hardware_concurrency()); }

int tpref_sizes(const tp_problem_desc* d, int32_t* n, int32_t* N, double* tau) {
  return guarded([&] {
    tporacle::validate_desc(*d);
    if (n) *n = (d->cells - 1) * (d->cells - 1);
    if (N) *N = d->steps;
    if (tau) *tau = d->period / d->steps;
  });
}

int tpref_loads(const tp_problem_desc* d, double* F) {
  return guarded([&] {
    const tporacle::GridProblem p(*d);
    const tpfem::BlockRhs f = p.loads();
    std::memcpy(F, f.data.data(), f.data.size() * sizeof(double));
  });
}

int tpref_mass(const tp_problem_desc* d, double* m) {
  return guarded([&] {
    const tporacle::GridProblem p(*d);
    std::vector<double> ones(static_cast<std::size_t>(p.n_dof()), 1.0);
    p.mass().multiply(ones.data(), m);
  });
}

int tpref_sigma(const tp_problem_desc* d, double* sigma) {
  return guarded([&] {
    const tporacle::GridProblem p(*d);
    std::memcpy(sigma, p.sigma().data(), p.sigma().size() * sizeof(double));
  });
}

int tpref_apply_k(const tp_problem_desc* d, const double* U, double* out, int32_t count) {
  return guarded([&] {
    const tporacle::GridProblem p(*d);
    const std::size_t n = static_cast<std::size_t>(p.n_dof());
    for (int i = 0; i < count; ++i) p.apply_k(U + i * n, out + i * n);
  });
}

/// y = J(u) v for one slice (Jacobian KAT support).
int tpref_jacobian_apply(const tp_problem_desc* d, const double* u, const double* v, double* y) {
  return guarded([&] {
    const tporacle::GridProblem p(*d);
    p.jacobian_k(u).multiply(v, y);
  });
}

int tpref_static_init(const tp_problem_desc* d, const tp_solver_cfg* c, double* U0,
                      int32_t* newton_counts) {
  return guarded([&] {
    const tporacle::GridProblem p(*d);
    const tpfem::BlockRhs F = p.loads();
    std::vector<int> counts;
    const tpfem::PeriodicState U = tpfem::static_init(p, F, p.tau(), to_ref(c), &counts);
    std::memcpy(U0, U.data.data(), U.data.size() * sizeof(double));
    if (newton_counts)
      for (std::size_t i = 0; i < counts.size(); ++i) newton_counts[i] = counts[i];
  });
}

int tpref_choose_nu_hat(const tp_problem_desc* d, const tp_solver_cfg* c, const double* U0,
                        double* nu_hat, double* q) {
  return guarded([&] {
    const tporacle::GridProblem p(*d);
    const tpfem::SolverConfig cfg = to_ref(c);
    const int samples = (c && c->nu_hat_samples > 1) ? c->nu_hat_samples : 2000;
    const tpfem::NuHatChoice ch = p.choose_nu_hat(cfg.nu_hat_mode, state_from(p, U0), samples);
    for (int r = 0; r < tpfem::kNumRegions; ++r) nu_hat[r] = ch.nu_hat[static_cast<std::size_t>(r)];
    if (q) *q = ch.q;
  });
}

int tpref_residual(const tp_problem_desc* d, const double* U, double* R, double* norm,
                   int32_t threads) {
  return guarded([&] {
    const tporacle::GridProblem p(*d);
    const tpfem::BlockRhs F = p.loads();
    const tpfem::BlockRhs res = tpfem::residual(p, state_from(p, U), F, std::max(1, threads));
    if (R) std::memcpy(R, res.data.data(), res.data.size() * sizeof(double));
    if (norm) *norm = tpfem::block_l2(res);
  });
}

int tpref_periodic_solve(const tp_problem_desc* d, const tp_solver_cfg* c, const double* nu_hat,
                         const double* G, double* U) {
  return guarded([&] {
    const tporacle::GridProblem p(*d);
    const tpfem::SolverConfig cfg = to_ref(c);
    const tpfem::SparseMatrix<double> K = p.stiffness_frozen(nu_array(nu_hat));
    tpfem::PeriodicSolverOptions opts = tpfem::make_periodic_options(cfg);
    opts.cache = tpfem::CachePolicy::never;
    const tpfem::PeriodicSolver solver(p.mass(), K, p.tau(), p.steps(), opts);
    tpfem::BlockRhs g(p.steps(), p.n_dof());
    std::memcpy(g.data.data(), G, g.data.size() * sizeof(double));
    const tpfem::PeriodicState u = solver.solve(g);
    std::memcpy(U, u.data.data(), u.data.size() * sizeof(double));
  });
}

/// solve_m1_fixed_point on the grid problem.  cache: 0 automatic, 1 always,
/// 2 never.  iterates (may be NULL): (cap) x N x n, iterate k at offset k*N*n.
/// times[0] = wall seconds of the call, times[1] = PeriodicSolver setup +
/// initial residual seconds (measured separately on the same inputs).
int tpref_solve_m1(const tp_problem_desc* d, const tp_solver_cfg* c, const double* nu_hat,
                   double q, const double* U0, double* U_out, double* history,
                   double* contraction, int32_t cap, int32_t* iterations, int32_t* status,
                   double* iterates, int32_t cache, double* times) {
  return guarded([&] {
    const tporacle::GridProblem p(*d);
    tpfem::SolverConfig cfg = to_ref(c);
    cfg.cache = cache == 1 ? tpfem::CachePolicy::always
                           : cache == 2 ? tpfem::CachePolicy::never : tpfem::CachePolicy::automatic;
    const tpfem::BlockRhs F = p.loads();
    const tpfem::SparseMatrix<double> K = p.stiffness_frozen(nu_array(nu_hat));
    const tpfem::PeriodicState U0s = state_from(p, U0);
    std::vector<tpfem::PeriodicState> log;
    const auto t0 = std::chrono::steady_clock::now();
    auto [U, rep] = tpfem::solve_m1_fixed_point(p, K, F, U0s, cfg, q, iterates ? &log : nullptr);
    const auto t1 = std::chrono::steady_clock::now();
    if (times) {
      times[0] = std::chrono::duration<double>(t1 - t0).count();
      const auto s0 = std::chrono::steady_clock::now();
      const tpfem::PeriodicSolver setup(p.mass(), K, p.tau(), p.steps(), tpfem::make_periodic_options(cfg));
      const tpfem::BlockRhs R0 = tpfem::residual(p, U0s, F, cfg.threads);
      (void)tpfem::block_l2(R0);
      times[1] = std::chrono::duration<double>(std::chrono::steady_clock::now() - s0).count();
    }
    if (U_out) std::memcpy(U_out, U.data.data(), U.data.size() * sizeof(double));
    for (std::size_t k = 0; k < rep.residual_history.size() && static_cast<int>(k) < cap; ++k)
      history[k] = rep.residual_history[k];
    if (contraction)
      for (std::size_t k = 0; k < rep.contraction_history.size() && static_cast<int>(k) < cap; ++k)
        contraction[k] = rep.contraction_history[k];
    if (iterations) *iterations = rep.iterations;
    if (status) *status = static_cast<int32_t>(rep.status);
    if (iterates) {
      const std::size_t sz = U.data.size();
      for (std::size_t k = 0; k < log.size() && static_cast<int>(k) < cap; ++k)
        std::memcpy(iterates + k * sz, log[k].data.data(), sz * sizeof(double));
    }
  });
}

// tpfem::solve_m2_newton (solvers.hpp:375-484) on the grid problem
int tpref_solve_m2(const tp_problem_desc* d, const tp_solver_cfg* c, const double* U0, double* U_out,
                   double* history, int32_t cap, int32_t* iterations, int32_t* status, double* wall) {
  return guarded([&] {
    const tporacle::GridProblem p(*d);
    const tpfem::SolverConfig cfg = to_ref(c);
    const tpfem::BlockRhs F = p.loads();
    const tpfem::PeriodicState U0s = state_from(p, U0);
    const auto t0 = std::chrono::steady_clock::now();
    auto [U, rep] = tpfem::solve_m2_newton(p, F, U0s, cfg);
    if (wall) *wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (U_out) std::memcpy(U_out, U.data.data(), U.data.size() * sizeof(double));
    for (std::size_t k = 0; k < rep.residual_history.size() && static_cast<int>(k) < cap; ++k)
      history[k] = rep.residual_history[k];
    if (iterations) *iterations = rep.iterations;
    if (status) *status = static_cast<int32_t>(rep.status);
  });
}

// tpfem::solve_m3_timestepping (solvers.hpp:489-542) on the grid problem
int tpref_solve_m3(const tp_problem_desc* d, const tp_solver_cfg* c, const double* U0, double* U_out,
                   double* history, int32_t cap, int32_t* iterations, int32_t* status, double* wall) {
  return guarded([&] {
    const tporacle::GridProblem p(*d);
    const tpfem::SolverConfig cfg = to_ref(c);
    const tpfem::BlockRhs F = p.loads();
    const tpfem::PeriodicState U0s = state_from(p, U0);
    const auto t0 = std::chrono::steady_clock::now();
    auto [U, rep] = tpfem::solve_m3_timestepping(p, F, U0s, cfg);
    if (wall) *wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (U_out) std::memcpy(U_out, U.data.data(), U.data.size() * sizeof(double));
    for (std::size_t k = 0; k < rep.residual_history.size() && static_cast<int>(k) < cap; ++k)
      history[k] = rep.residual_history[k];
    if (iterations) *iterations = rep.iterations;
    if (status) *status = static_cast<int32_t>(rep.status);
  });
}

}  // extern "C"

// ---------------------------------------------------------------- transformer (reference physics)
extern "C" {
// configs/transformer.json fields (RunConfig, config.hpp:39-53)
typedef struct tpref_mesh_cfg {
  int32_t nx, ny, refinements, steps;
  double period, s_max;
  int32_t flux_samples, pad_;
  double j_amp;  // winding current amplitude override (configs/transformer_saturated.json); 0: table value
} tpref_mesh_cfg;
}

namespace {

// runner.hpp:27-31 + 46-73 (up to static_init), on the reference's own types
struct TrSetup {
  std::shared_ptr<const tpfem::Mesh> mesh;
  tpfem::MaterialTable mat = tpfem::MaterialTable::transformer();
  std::unique_ptr<tpfem::NonlinearOperator> op;
  tpfem::SparseMatrix<double> M;
  tpfem::BlockRhs F;
  double tau = 0;
  int N = 0;
  explicit TrSetup(const tpref_mesh_cfg& c) {
    if (c.j_amp != 0) {  // parse_materials override (config.hpp:146-170)
      auto wp = mat.at(tpfem::Region::winding_plus), wm = mat.at(tpfem::Region::winding_minus);
      wp.j_amp = c.j_amp;
      wm.j_amp = -c.j_amp;
      mat.set(tpfem::Region::winding_plus, wp);
      mat.set(tpfem::Region::winding_minus, wm);
    }
    tpfem::Mesh m = tpfem::build_rectilinear_mesh(tpfem::transformer_regions(), c.nx, c.ny);
    for (int r = 0; r < c.refinements; ++r) m = tpfem::refine_uniform(m);
    mesh = std::make_shared<const tpfem::Mesh>(std::move(m));
    op = std::make_unique<tpfem::NonlinearOperator>(mesh, mat);
    N = c.steps;
    tau = c.period / c.steps;
    F = tpfem::assemble_loads(*mesh, mat, c.steps, c.period);
    M = tpfem::assemble_mass(*mesh, mat);
  }
  tpfem::FemProblem problem() const { return tpfem::FemProblem{&M, op.get()}; }
  tpfem::PeriodicState state(const double* U) const {
    tpfem::PeriodicState s(N, op->n_dof(), tau);
    std::memcpy(s.data.data(), U, s.data.size() * sizeof(double));
    return s;
  }
};

}  // namespace

extern "C" {

int tpref_tr_mesh(int32_t nx, int32_t ny, int32_t refinements, int32_t* nv, int32_t* nt, int32_t* ndof,
                  double* verts, int32_t* tris, int32_t* region) {
  return guarded([&] {
    tpfem::Mesh m = tpfem::build_rectilinear_mesh(tpfem::transformer_regions(), nx, ny);
    for (int r = 0; r < refinements; ++r) m = tpfem::refine_uniform(m);
    if (nv) *nv = m.n_vertices();
    if (nt) *nt = m.n_triangles();
    if (ndof) *ndof = m.n_dof();
    if (verts)
      for (int v = 0; v < m.n_vertices(); ++v) {
        verts[2 * v] = m.vertices[v][0];
        verts[2 * v + 1] = m.vertices[v][1];
      }
    if (tris)
      for (int t = 0; t < m.n_triangles(); ++t)
        for (int k = 0; k < 3; ++k) tris[3 * t + k] = m.triangles[t][k];
    if (region)
      for (int t = 0; t < m.n_triangles(); ++t) region[t] = static_cast<int32_t>(m.region[t]);
  });
}

int tpref_tr_material(tp_exp_material* out) {
  return guarded([&] {
    const auto t = tpfem::MaterialTable::transformer();
    for (int r = 0; r < tpfem::kNumRegions; ++r) {
      const auto& m = t.at(static_cast<tpfem::Region>(r));
      out[r] = tp_exp_material{m.sigma, m.a, m.b, m.c, m.d, m.j_amp};
    }
  });
}

int tpref_tr_loads(const tpref_mesh_cfg* c, double* F) {
  return guarded([&] {
    const TrSetup s(*c);
    std::memcpy(F, s.F.data.data(), s.F.data.size() * sizeof(double));
  });
}

// consistent mass as CSR (rowptr n+1, col nnz, val nnz); call with NULL
// arrays first for n / nnz
int tpref_tr_mass(const tpref_mesh_cfg* c, int32_t* n, int32_t* nnz, int32_t* rowptr, int32_t* col,
                  double* val) {
  return guarded([&] {
    const TrSetup s(*c);
    const auto& M = s.M;
    if (n) *n = static_cast<int32_t>(M.rows());
    if (nnz) *nnz = static_cast<int32_t>(M.nnz());
    if (rowptr)
      for (std::size_t i = 0; i <= static_cast<std::size_t>(M.rows()); ++i) rowptr[i] = M.row_offsets()[i];
    if (col)
      for (std::size_t k = 0; k < static_cast<std::size_t>(M.nnz()); ++k) col[k] = M.col_indices()[k];
    if (val)
      for (std::size_t k = 0; k < static_cast<std::size_t>(M.nnz()); ++k) val[k] = M.values()[k];
  });
}

int tpref_tr_apply_k(const tpref_mesh_cfg* c, const double* U, double* out, int32_t count) {
  return guarded([&] {
    const TrSetup s(*c);
    const std::size_t n = static_cast<std::size_t>(s.op->n_dof());
    for (int i = 0; i < count; ++i) s.op->apply(U + i * n, out + i * n);
  });
}

int tpref_tr_residual(const tpref_mesh_cfg* c, const double* U, double* R, double* norm) {
  return guarded([&] {
    const TrSetup s(*c);
    const tpfem::BlockRhs Rb = tpfem::residual(s.problem(), s.state(U), s.F, 1);
    if (R) std::memcpy(R, Rb.data.data(), Rb.data.size() * sizeof(double));
    if (norm) *norm = tpfem::block_l2(Rb);
  });
}

int tpref_tr_static_init(const tpref_mesh_cfg* c, const tp_solver_cfg* sc, double* U0, int32_t* counts) {
  return guarded([&] {
    const TrSetup s(*c);
    std::vector<int> nc;
    const tpfem::PeriodicState U = tpfem::static_init(s.problem(), s.F, s.tau, to_ref(sc), &nc);
    std::memcpy(U0, U.data.data(), U.data.size() * sizeof(double));
    if (counts)
      for (std::size_t i = 0; i < nc.size(); ++i) counts[i] = nc[i];
  });
}

// runner.hpp:62-66: ranges over every slice of U0, flux_bounds(s_max,
// flux_samples), choose_nu_hat(mode, bounds, table, &ranges, samples)
int tpref_tr_choose_nu_hat(const tpref_mesh_cfg* c, const tp_solver_cfg* sc, const double* U0, double* nu_hat,
                           double* q) {
  return guarded([&] {
    const TrSetup s(*c);
    const tpfem::SolverConfig cfg = to_ref(sc);
    const tpfem::FluxBounds bounds = tpfem::flux_bounds(s.mat, c->s_max, c->flux_samples);
    tpfem::RegionFieldRanges ranges;
    const std::size_t n = static_cast<std::size_t>(s.op->n_dof());
    for (int i = 0; i < s.N; ++i) tpfem::absorb_field_ranges(*s.op, U0 + i * n, ranges);
    const int samples = sc && sc->nu_hat_samples > 0 ? sc->nu_hat_samples : 2000;
    const tpfem::NuHatChoice ch = tpfem::choose_nu_hat(cfg.nu_hat_mode, bounds, s.mat, &ranges, samples);
    for (int r = 0; r < tpfem::kNumRegions; ++r) nu_hat[r] = ch.nu_hat[static_cast<std::size_t>(r)];
    if (q) *q = ch.q;
  });
}

int tpref_tr_periodic_solve(const tpref_mesh_cfg* c, const tp_solver_cfg* sc, const double* nu_hat,
                            const double* G, double* U) {
  return guarded([&] {
    const TrSetup s(*c);
    const tpfem::SolverConfig cfg = to_ref(sc);
    const auto K = tpfem::assemble_stiffness_frozen(*s.mesh, nu_array(nu_hat));
    const tpfem::PeriodicSolver ps(s.M, K, s.tau, s.N, tpfem::make_periodic_options(cfg));
    tpfem::BlockRhs Gb(s.N, s.op->n_dof());
    std::memcpy(Gb.data.data(), G, Gb.data.size() * sizeof(double));
    const tpfem::PeriodicState X = ps.solve(Gb);
    std::memcpy(U, X.data.data(), X.data.size() * sizeof(double));
  });
}

// solve_m1_fixed_point(FemSystem, op, F, U0, cfg) as run_transformer_method
// (runner.hpp:84) calls it; iterates (may be NULL): (cap) x N x n
int tpref_tr_solve_m1(const tpref_mesh_cfg* c, const tp_solver_cfg* sc, const double* nu_hat, double q,
                      const double* U0, double* U_out, double* history, int32_t cap, int32_t* iterations,
                      int32_t* status, double* iterates, double* wall) {
  return guarded([&] {
    const TrSetup s(*c);
    const tpfem::SolverConfig cfg = to_ref(sc);
    const auto K = tpfem::assemble_stiffness_frozen(*s.mesh, nu_array(nu_hat));
    std::vector<tpfem::PeriodicState> log;
    const auto t0 = std::chrono::steady_clock::now();
    auto [U, rep] = tpfem::solve_m1_fixed_point(s.problem(), K, s.F, s.state(U0), cfg, q,
                                                iterates ? &log : nullptr);
    if (wall) *wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (U_out) std::memcpy(U_out, U.data.data(), U.data.size() * sizeof(double));
    for (std::size_t k = 0; k < rep.residual_history.size() && static_cast<int>(k) < cap; ++k)
      history[k] = rep.residual_history[k];
    if (iterations) *iterations = rep.iterations;
    if (status) *status = static_cast<int32_t>(rep.status);
    if (iterates) {
      const std::size_t sz = U.data.size();
      for (std::size_t k = 0; k < log.size() && static_cast<int>(k) < cap; ++k)
        std::memcpy(iterates + k * sz, log[k].data.data(), sz * sizeof(double));
    }
  });
}

}  // extern "C"

// solve_m2_newton / solve_m3_timestepping on the reference transformer
// problem (run_transformer_method, runner.hpp:85-86)
extern "C" int tpref_tr_solve_m23(const tpref_mesh_cfg* c, const tp_solver_cfg* sc, int32_t method, const double* U0,
                                  double* U_out, double* history, int32_t cap, int32_t* iterations, int32_t* status,
                                  double* wall) {
  return guarded([&] {
    const TrSetup s(*c);
    const tpfem::SolverConfig cfg = to_ref(sc);
    const auto t0 = std::chrono::steady_clock::now();
    auto [U, rep] = method == 2 ? tpfem::solve_m2_newton(s.problem(), s.F, s.state(U0), cfg)
                                : tpfem::solve_m3_timestepping(s.problem(), s.F, s.state(U0), cfg);
    if (wall) *wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (U_out) std::memcpy(U_out, U.data.data(), U.data.size() * sizeof(double));
    for (std::size_t k = 0; k < rep.residual_history.size() && static_cast<int>(k) < cap; ++k)
      history[k] = rep.residual_history[k];
    if (iterations) *iterations = rep.iterations;
    if (status) *status = static_cast<int32_t>(rep.status);
  });
}

// ---------------------------------------------------------------- large-config parity support
// Entry points for parity at BASELINE configs too large to archive whole
// iterates of ("per-iterate ||U^k|| and ||U^k - U^{k-1}||,
// plus full vectors at the iterates the oracle can afford").
namespace {

// Order-sensitive fingerprint of one iterate; must match
// tests/golden/make_golden.py:checksum (norm, sum, cos-weighted sum, max |.|).
void digest_of(const double* a, std::size_t n, double* out) {
  long double ss = 0, s = 0, ws = 0;
  double mx = 0;
  for (std::size_t i = 0; i < n; ++i) {
    const double v = a[i];
    ss += static_cast<long double>(v) * v;
    s += v;
    ws += static_cast<long double>(std::cos(0.001 * static_cast<double>(i))) * v;
    mx = std::max(mx, std::abs(v));
  }
  out[0] = std::sqrt(static_cast<double>(ss));
  out[1] = static_cast<double>(s);
  out[2] = static_cast<double>(ws);
  out[3] = mx;
}

}  // namespace

extern "C" {

/// solve_m1_fixed_point (solvers.hpp:301-369) with the iterate log reduced
/// on the fly: digests (cap x 5: checksum of U^k, then ||U^k - U^{k-1}||,
/// 0 for k = 0), samples (cap x ceil(N n / stride): U^k[::stride]).
int tpref_solve_m1_digest(const tp_problem_desc* d, const tp_solver_cfg* c, const double* nu_hat, double q,
                          const double* U0, double* U_out, double* history, double* contraction, int32_t cap,
                          int32_t* iterations, int32_t* status, double* digests, int64_t stride,
                          double* samples, int32_t cache, double* wall) {
  return guarded([&] {
    const tporacle::GridProblem p(*d);
    tpfem::SolverConfig cfg = to_ref(c);
    cfg.cache = cache == 1 ? tpfem::CachePolicy::always
                           : cache == 2 ? tpfem::CachePolicy::never : tpfem::CachePolicy::automatic;
    const tpfem::BlockRhs F = p.loads();
    const tpfem::SparseMatrix<double> K = p.stiffness_frozen(nu_array(nu_hat));
    std::vector<tpfem::PeriodicState> log;
    const auto t0 = std::chrono::steady_clock::now();
    auto [U, rep] = tpfem::solve_m1_fixed_point(p, K, F, state_from(p, U0), cfg, q, &log);
    if (wall) *wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (U_out) std::memcpy(U_out, U.data.data(), U.data.size() * sizeof(double));
    for (std::size_t k = 0; k < rep.residual_history.size() && static_cast<int>(k) < cap; ++k)
      history[k] = rep.residual_history[k];
    if (contraction)
      for (std::size_t k = 0; k < rep.contraction_history.size() && static_cast<int>(k) < cap; ++k)
        contraction[k] = rep.contraction_history[k];
    if (iterations) *iterations = rep.iterations;
    if (status) *status = static_cast<int32_t>(rep.status);
    const std::size_t sz = U.data.size();
    const std::size_t ns = stride > 0 ? (sz + static_cast<std::size_t>(stride) - 1) / static_cast<std::size_t>(stride) : 0;
    for (std::size_t k = 0; k < log.size() && static_cast<int>(k) < cap; ++k) {
      const double* a = log[k].data.data();
      digest_of(a, sz, digests + 5 * k);
      long double dd = 0;
      if (k > 0) {
        const double* b = log[k - 1].data.data();
        for (std::size_t i = 0; i < sz; ++i) dd += static_cast<long double>(a[i] - b[i]) * (a[i] - b[i]);
      }
      digests[5 * k + 4] = std::sqrt(static_cast<double>(dd));
      if (samples)
        for (std::size_t s = 0; s < ns; ++s) samples[k * ns + s] = a[s * static_cast<std::size_t>(stride)];
    }
  });
}

/// The body of static_init's slice loop (solvers.hpp:282-294) for the listed
/// slices only: newton_elliptic(p, 0, f^i, u = 0, static_tol, static_max_newton).
/// U_out: count x n; counts: count.
int tpref_static_init_slices(const tp_problem_desc* d, const tp_solver_cfg* c, const int32_t* slices,
                             int32_t count, double* U_out, int32_t* counts) {
  return guarded([&] {
    const tporacle::GridProblem p(*d);
    const tpfem::SolverConfig cfg = to_ref(c);
    const std::size_t n = static_cast<std::size_t>(p.n_dof());
    tpfem::parallel_for(0, count, cfg.threads, [&](int s) {
      const int i = slices[s];
      if (i < 0 || i >= p.steps()) throw std::invalid_argument("static_init_slices: slice out of range");
      std::vector<double> rhs(n, 0.0);
      p.load_slice(i, rhs.data());
      std::vector<double> u(n, 0.0);
      counts[s] = tpfem::detail::newton_elliptic(p, 0.0, rhs, u, cfg.static_tol, cfg.static_max_newton,
                                                  cfg.armijo);
      std::copy(u.begin(), u.end(), U_out + static_cast<std::size_t>(s) * n);
    });
  });
}

/// The frequency-block solves of PeriodicSolver::solve_frequency
/// (periodic.hpp:252-289) for the listed frequencies, on caller right-hand
/// sides: (lambda_k M + K_hat) x = b with lambda_k = PeriodicSolver::symbol(k)
/// (periodic.hpp:146-152); real blocks (k = 0, N/2) as two real solves of
/// real_block(k), complex ones through complex_block(k) = add_scaled(lambda_k,
/// to_complex(M), 1, to_complex(K_hat)).  B, X: count x n complex (re, im
/// interleaved).  Every solve carries the SparseSolver residual contract.
int tpref_frequency_blocks(const tp_problem_desc* d, const tp_solver_cfg* c, const double* nu_hat,
                           const int32_t* ks, int32_t count, const double* B, double* X) {
  return guarded([&] {
    const tporacle::GridProblem p(*d);
    const tpfem::SolverConfig cfg = to_ref(c);
    const tpfem::SparseMatrix<double> K = p.stiffness_frozen(nu_array(nu_hat));
    tpfem::PeriodicSolverOptions opts = tpfem::make_periodic_options(cfg);
    opts.cache = tpfem::CachePolicy::never;
    const tpfem::PeriodicSolver ps(p.mass(), K, p.tau(), p.steps(), opts);
    const std::size_t n = static_cast<std::size_t>(p.n_dof());
    const int N = p.steps();
    const auto Mc = tpfem::to_complex(p.mass());
    const auto Kc = tpfem::to_complex(K);
    tpfem::parallel_for(0, count, cfg.threads, [&](int s) {
      const int k = ks[s];
      if (k < 0 || 2 * k > N) throw std::invalid_argument("frequency_blocks: k outside 0..N/2");
      const double* b = B + 2 * n * static_cast<std::size_t>(s);
      double* x = X + 2 * n * static_cast<std::size_t>(s);
      const std::complex<double> lam = ps.symbol(k);
      if (k == 0 || 2 * k == N) {
        const tpfem::SparseSolver<double> solver(tpfem::add_scaled(lam.real(), p.mass(), 1.0, K));
        std::vector<double> bre(n), bim(n);
        for (std::size_t j = 0; j < n; ++j) {
          bre[j] = b[2 * j];
          bim[j] = b[2 * j + 1];
        }
        const std::vector<double> xre = solver.solve(bre), xim = solver.solve(bim);
        for (std::size_t j = 0; j < n; ++j) {
          x[2 * j] = xre[j];
          x[2 * j + 1] = xim[j];
        }
      } else {
        const tpfem::SparseSolver<std::complex<double>> solver(
            tpfem::add_scaled(lam, Mc, std::complex<double>{1.0, 0.0}, Kc));
        std::vector<std::complex<double>> bc(n);
        for (std::size_t j = 0; j < n; ++j) bc[j] = {b[2 * j], b[2 * j + 1]};
        const std::vector<std::complex<double>> xc = solver.solve(bc);
        for (std::size_t j = 0; j < n; ++j) {
          x[2 * j] = xc[j].real();
          x[2 * j + 1] = xc[j].imag();
        }
      }
    });
  });
}

}  // extern "C"

extern "C" {

/// Bounded sample of one reference sweep for bench.py's reference arm at
/// sizes where a whole sweep takes hours: each stage of the sweep timed on a
/// sample with the reference's own code, each a parallel_for over
/// cfg.threads like the reference's:
///   times[0] A  the RHS lambda (solvers.hpp:326-336) on `slices` slices:
///               apply_k, K_hat.multiply, g = f + K_hat u - K(u)
///   times[1] B  the forward transform (periodic.hpp:163-167) on `cols` dof
///               columns: gather a column of length N, DftPlan::forward
///   times[2] D  the inverse transform + Re / Im sums (periodic.hpp:174-185)
///               on the same columns
///   times[3] E  the residual lambda (periodic.hpp:43-52) on the slices:
///               apply_k, M (u - u_prev) / tau, r = f - M du - K(u)
///   times[4] C  `blocks` frequency-block solves (solve_frequency,
///               periodic.hpp:252-289: assemble lambda_k M + K_hat, factorise,
///               solve, residual contract), k = 1 .. blocks; 0 skips
/// The state is a seeded smooth field (the stages' cost does not depend on
/// it).  setup_s: GridProblem + K_hat construction (not part of a sweep),
/// done once; the stages then run `reps` times (times: reps x 5).
int tpref_sweep_sample(const tp_problem_desc* d, const tp_solver_cfg* c, const double* nu_hat, int32_t slices,
                       int32_t cols, int32_t blocks, int32_t reps, double* times, double* setup_s) {
  return guarded([&] {
    using clk = std::chrono::steady_clock;
    const auto secs = [](clk::time_point a) { return std::chrono::duration<double>(clk::now() - a).count(); };
    auto t0 = clk::now();
    const tporacle::GridProblem p(*d);
    const tpfem::SolverConfig cfg = to_ref(c);
    const tpfem::SparseMatrix<double> K = p.stiffness_frozen(nu_array(nu_hat));
    const std::size_t n = static_cast<std::size_t>(p.n_dof());
    const int N = p.steps();
    const double tau = p.tau();
    const int S = std::max(1, std::min<int>(slices, N));
    // state: S+1 consecutive slices of a smooth seeded field
    std::vector<double> U((static_cast<std::size_t>(S) + 1) * n), F(static_cast<std::size_t>(S) * n, 0.0);
    for (std::size_t s = 0; s <= static_cast<std::size_t>(S); ++s)
      for (std::size_t j = 0; j < n; ++j)
        U[s * n + j] = 1e-3 * std::sin(0.001 * static_cast<double>(j) + 0.1 * static_cast<double>(s));
    for (int s = 0; s < S; ++s) p.load_slice(s, F.data() + static_cast<std::size_t>(s) * n);
    if (setup_s) *setup_s = secs(t0);
    std::vector<double> G(static_cast<std::size_t>(S) * n), R(static_cast<std::size_t>(S) * n);
    const tpfem::DftPlan plan(N, cfg.transform);
    const int C = std::max(1, std::min<int>(cols, static_cast<int>(n)));
    std::vector<std::complex<double>> work(static_cast<std::size_t>(C) * N);
    std::vector<double> src(static_cast<std::size_t>(N) * C);
    std::vector<double> re2(C), im2(C);
    const tpfem::SparseMatrix<double>& M = p.mass();
    for (int rep = 0; rep < std::max(1, reps); ++rep, times += 5) {
    // A: RHS
    t0 = clk::now();
    tpfem::parallel_for(0, S, cfg.threads, [&](int i) {
      const double* u = U.data() + (static_cast<std::size_t>(i) + 1) * n;
      double* g = G.data() + static_cast<std::size_t>(i) * n;
      std::vector<double> ku(n), khu(n);
      p.apply_k(u, ku.data());
      K.multiply(u, khu.data());
      const double* f = F.data() + static_cast<std::size_t>(i) * n;
      for (std::size_t j = 0; j < n; ++j) g[j] = f[j] + khu[j] - ku[j];
    });
    times[0] = secs(t0);
    // B, D: transforms over `cols` columns (gather stride n like periodic.hpp:165)
    for (std::size_t k = 0; k < src.size(); ++k) src[k] = std::cos(0.37 * static_cast<double>(k));
    t0 = clk::now();
    tpfem::parallel_for(0, C, cfg.threads, [&](int j) {
      std::complex<double>* col = work.data() + static_cast<std::size_t>(j) * N;
      for (int i = 0; i < N; ++i) col[i] = src[static_cast<std::size_t>(i) * C + j];
      plan.forward(col);
    });
    times[1] = secs(t0);
    t0 = clk::now();
    tpfem::parallel_for(0, C, cfg.threads, [&](int j) {
      std::complex<double>* col = work.data() + static_cast<std::size_t>(j) * N;
      plan.inverse(col);
      double r = 0, m = 0;
      for (int i = 0; i < N; ++i) {
        src[static_cast<std::size_t>(i) * C + j] = col[i].real();
        r += col[i].real() * col[i].real();
        m += col[i].imag() * col[i].imag();
      }
      re2[j] = r;
      im2[j] = m;
    });
    times[2] = secs(t0);
    // E: residual
    t0 = clk::now();
    tpfem::parallel_for(0, S, cfg.threads, [&](int i) {
      const double* u = U.data() + (static_cast<std::size_t>(i) + 1) * n;
      const double* uprev = U.data() + static_cast<std::size_t>(i) * n;
      double* r = R.data() + static_cast<std::size_t>(i) * n;
      std::vector<double> ku(n), du(n), mdu(n);
      p.apply_k(u, ku.data());
      for (std::size_t j = 0; j < n; ++j) du[j] = (u[j] - uprev[j]) / tau;
      M.multiply(du.data(), mdu.data());
      const double* f = F.data() + static_cast<std::size_t>(i) * n;
      for (std::size_t j = 0; j < n; ++j) r[j] = f[j] - mdu[j] - ku[j];
    });
    times[3] = secs(t0);
    // C: frequency blocks k = 1..blocks
    times[4] = 0;
    if (blocks > 0) {
      tpfem::PeriodicSolverOptions opts = tpfem::make_periodic_options(cfg);
      opts.cache = tpfem::CachePolicy::never;
      const tpfem::PeriodicSolver ps(M, K, tau, N, opts);
      const auto Mc = tpfem::to_complex(M);
      const auto Kc = tpfem::to_complex(K);
      t0 = clk::now();
      tpfem::parallel_for(1, blocks + 1, cfg.threads, [&](int k) {
        const tpfem::SparseSolver<std::complex<double>> solver(
            tpfem::add_scaled(ps.symbol(k), Mc, std::complex<double>{1.0, 0.0}, Kc));
        std::vector<std::complex<double>> b(n);
        for (std::size_t j = 0; j < n; ++j) b[j] = {G[j], 0.5 * G[j]};
        (void)solver.solve(b);
      });
      times[4] = secs(t0);
    }
    }  // reps
  });
}

}  // extern "C"
