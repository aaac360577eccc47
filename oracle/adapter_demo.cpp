// TEST INFRASTRUCTURE ONLY -- the reference-side change of INTEGRATION.md,
// compiled against the reference's own headers: run_transformer_method's M1
// (runner.hpp:46-89) once on the CPU through tpfem and once on the GPU
// through include/tpgpu_tpfem.hpp (GpuMeshProblem built from the same
// tpfem::Mesh and MaterialTable), then compare.  Built by oracle/Makefile
// into _ref/adapter_demo; run by tests/test_gpu_mesh.py.
//
//   adapter_demo nx ny refinements steps j_amp tol  -> one JSON line
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "tpfem/assembly.hpp"
#include "tpfem/mesh.hpp"
#include "tpfem/periodic.hpp"
#include "tpfem/solvers.hpp"
#include "tpgpu_tpfem.hpp"

int main(int argc, char** argv) {
  const int nx = argc > 1 ? std::atoi(argv[1]) : 40, ny = argc > 2 ? std::atoi(argv[2]) : 40;
  const int refinements = argc > 3 ? std::atoi(argv[3]) : 0, steps = argc > 4 ? std::atoi(argv[4]) : 64;
  const double j_amp = argc > 5 ? std::atof(argv[5]) : 9.5e5, tol = argc > 6 ? std::atof(argv[6]) : 1e-8;
  const double period = 0.02;
  // runner.hpp:27-31, 46-73
  tpfem::Mesh m = tpfem::build_rectilinear_mesh(tpfem::transformer_regions(), nx, ny);
  for (int r = 0; r < refinements; ++r) m = tpfem::refine_uniform(m);
  auto mesh = std::make_shared<const tpfem::Mesh>(std::move(m));
  tpfem::MaterialTable mat = tpfem::MaterialTable::transformer();
  auto wp = mat.at(tpfem::Region::winding_plus), wm = mat.at(tpfem::Region::winding_minus);
  wp.j_amp = j_amp;
  wm.j_amp = -j_amp;
  mat.set(tpfem::Region::winding_plus, wp);
  mat.set(tpfem::Region::winding_minus, wm);
  tpfem::SolverConfig cfg;
  cfg.tol = tol;
  // ---- CPU: the reference, unchanged
  const auto t0 = std::chrono::steady_clock::now();
  tpfem::NonlinearOperator op(mesh, mat);
  const tpfem::BlockRhs F = tpfem::assemble_loads(*mesh, mat, steps, period);
  const tpfem::SparseMatrix<double> M = tpfem::assemble_mass(*mesh, mat);
  std::vector<int> nc_cpu;
  const tpfem::PeriodicState U0 = tpfem::static_init(tpfem::FemProblem{&M, &op}, F, period / steps, cfg, &nc_cpu);
  tpfem::RegionFieldRanges ranges;
  for (int i = 0; i < steps; ++i) tpfem::absorb_field_ranges(op, U0.block(i), ranges);
  const tpfem::NuHatChoice ch =
      tpfem::choose_nu_hat(cfg.nu_hat_mode, tpfem::flux_bounds(mat, 3.0, 10001), mat, &ranges);
  const auto K = tpfem::assemble_stiffness_frozen(*mesh, ch.nu_hat);
  auto [Uc, rc] = tpfem::solve_m1_fixed_point(tpfem::FemProblem{&M, &op}, K, F, U0, cfg, ch.q);
  const double t_cpu = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  // ---- GPU: the same calls through the adapter
  const auto t1 = std::chrono::steady_clock::now();
  tpgpu::GpuMeshProblem gp(*mesh, mat, steps, period);
  std::vector<int> nc_gpu;
  const tpfem::PeriodicState G0 = tpgpu::static_init(gp, cfg, &nc_gpu);
  std::array<double, tpfem::kNumRegions> nu{};
  const double q = tpgpu::choose_nu_hat(gp, cfg, &nu);
  auto [Ug, rg] = tpgpu::solve_m1_fixed_point(gp, G0, cfg);
  const double t_gpu = std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
  double num = 0, den = 0, nud = 0;
  for (std::size_t l = 0; l < Uc.data.size(); ++l) {
    num += (Ug.data[l] - Uc.data[l]) * (Ug.data[l] - Uc.data[l]);
    den += Uc.data[l] * Uc.data[l];
  }
  for (int r = 0; r < tpfem::kNumRegions; ++r) nud = std::max(nud, std::abs(nu[r] - ch.nu_hat[r]) / ch.nu_hat[r]);
  std::printf("{\"n_dof\": %d, \"steps\": %d, \"newton_equal\": %s, \"cpu_iterations\": %d, \"gpu_iterations\": %d, "
              "\"final_rel\": %.3e, \"nu_hat_rel\": %.3e, \"q_cpu\": %.17g, \"q_gpu\": %.17g, \"cpu_s\": %.4f, "
              "\"gpu_s\": %.4f}\n",
              (int)op.n_dof(), steps, nc_cpu == nc_gpu ? "true" : "false", rc.iterations, rg.iterations,
              std::sqrt(num / den), nud, ch.q, q, t_cpu, t_gpu);
  return (nc_cpu == nc_gpu && rc.iterations == rg.iterations && std::sqrt(num / den) <= 1e-10) ? 0 : 1;
}
