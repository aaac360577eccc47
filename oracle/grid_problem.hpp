// TEST INFRASTRUCTURE ONLY -- the BASELINE.json physics expressed as a
// `Problem` for the reference's own templates.
//
// The reference's solver layer (static_init, solve_m1_fixed_point, residual,
// PeriodicSolver, DftPlan, SparseMatrix; solvers.hpp / periodic.hpp / fft.hpp
// / sparse.hpp) is used unchanged.  What BASELINE.json asks for that the
// reference API cannot express is restated here, each piece next to the
// reference code it follows:
//   * uniform P1 grid (no edge snapping), painted by cell centroid
//       -- build_rectilinear_mesh, mesh.hpp:141-190; numbering by the
//          reference's own detail::finalize_mesh, mesh.hpp:87-103
//   * nu(s) = nu0 + (nu_inf-nu0) s^2/(s^2+Bs^2), nu'(s)
//       -- MaterialTable::nu / nu_prime, materials.hpp:42-57
//   * lumped sigma-mass with per-triangle sigma (seeded bilinear noise)
//       -- assemble_mass, assembly.hpp:50-65
//   * loads with sum-of-sines sources per material
//       -- assemble_loads, assembly.hpp:88-106; source_current, materials.hpp:60-65
//   * K(u) and its Jacobian with the new law
//       -- NonlinearOperator::apply / jacobian, assembly.hpp:126-177
//   * flux-Jacobian bounds and frozen-field nu_hat with the new law
//       -- flux_jacobian_bounds, materials.hpp:112-128; choose_nu_hat,
//          assembly.hpp:254-291
// The frozen stiffness itself is the reference's assemble_stiffness_frozen
// (assembly.hpp:68-84) and field ranges come from its absorb_field_ranges
// (assembly.hpp:236-242).
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <limits>
#include <memory>
#include <numbers>
#include <stdexcept>
#include <vector>

#include "tpfem/assembly.hpp"
#include "tpfem/mesh.hpp"
#include "tpfem/sparse.hpp"
#include "tpfem/state.hpp"
#include "../include/tpgpu.h"

namespace tporacle {

using tpfem::Index;

inline std::uint64_t splitmix64(std::uint64_t& state) {
  std::uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/// Seeded L x L lattice over desc.noise_box, bilinear, clamped to [lo, hi].
class SigmaNoise {
 public:
  explicit SigmaNoise(const tp_problem_desc& d) : d_(d) {
    const int L = d.noise_lattice;
    if (L < 2) throw std::invalid_argument("noise: lattice must be >= 2");
    v_.resize(static_cast<std::size_t>(L) * L);
    std::uint64_t state = d.noise_seed;
    for (int b = 0; b < L; ++b)
      for (int a = 0; a < L; ++a) {
        const double u = static_cast<double>(splitmix64(state) >> 11) * 0x1.0p-53;
        v_[static_cast<std::size_t>(b) * L + a] = d.noise_lo + (d.noise_hi - d.noise_lo) * u;
      }
  }
  double at(double x, double y) const {
    const int L = d_.noise_lattice;
    const auto coord = [L](double p, double lo, double hi, int& i0, double& f) {
      double s = (p - lo) / (hi - lo) * (L - 1);
      s = std::min(std::max(s, 0.0), static_cast<double>(L - 1));
      i0 = std::min(static_cast<int>(std::floor(s)), L - 2);
      f = s - i0;
    };
    int a0, b0;
    double fx, fy;
    coord(x, d_.noise_box[0], d_.noise_box[2], a0, fx);
    coord(y, d_.noise_box[1], d_.noise_box[3], b0, fy);
    const auto v = [&](int a, int b) { return v_[static_cast<std::size_t>(b) * L + a]; };
    double val = (1 - fx) * (1 - fy) * v(a0, b0) + fx * (1 - fy) * v(a0 + 1, b0) +
                 (1 - fx) * fy * v(a0, b0 + 1) + fx * fy * v(a0 + 1, b0 + 1);
    return std::min(std::max(val, d_.noise_lo), d_.noise_hi);
  }

 private:
  tp_problem_desc d_;
  std::vector<double> v_;
};

/// nu(s) and nu'(s) of one material (BASELINE law).
struct Law {
  double nu0 = 1, nu_inf = 1, bs = 1;
  double nu(double s) const {
    if (!(s >= 0)) throw std::invalid_argument("nu: field magnitude must be >= 0");
    if (nu0 == nu_inf) return nu0;
    const double s2 = s * s;
    return nu0 + (nu_inf - nu0) * s2 / (s2 + bs * bs);
  }
  double nu_prime(double s) const {
    if (!(s >= 0)) throw std::invalid_argument("nu_prime: field magnitude must be >= 0");
    if (nu0 == nu_inf) return 0;
    const double den = s * s + bs * bs;
    return 2.0 * (nu_inf - nu0) * s * bs * bs / (den * den);
  }
};

inline void validate_desc(const tp_problem_desc& d) {
  if (d.cells < 2) throw std::invalid_argument("problem: need at least 2 cells per side");
  if (d.steps < 1) throw std::invalid_argument("problem: need at least one time step");
  if (!(d.period > 0)) throw std::invalid_argument("problem: period must be positive");
  if (d.n_materials < 1 || d.n_materials > TP_MAX_MATERIALS)
    throw std::invalid_argument("problem: material count out of range");
  if (d.n_rects < 0 || d.n_rects > TP_MAX_RECTS)
    throw std::invalid_argument("problem: rectangle count out of range");
  for (int r = 0; r < d.n_rects; ++r)
    if (d.rect[r].material < 0 || d.rect[r].material >= d.n_materials)
      throw std::invalid_argument("problem: rectangle material out of range");
  for (int m = 0; m < d.n_materials; ++m) {
    const tp_material& mt = d.material[m];
    if (!(mt.sigma >= 0)) throw std::invalid_argument("problem: sigma must be >= 0");
    if (!(mt.nu0 > 0) || !(mt.nu_inf > 0)) throw std::invalid_argument("problem: nu must be > 0");
    if (mt.nu0 != mt.nu_inf && !(mt.bs > 0)) throw std::invalid_argument("problem: Bs must be > 0");
    if (mt.n_harmonics < 0 || mt.n_harmonics > TP_MAX_HARMONICS)
      throw std::invalid_argument("problem: harmonic count out of range");
  }
}

/// The grid problem: satisfies the reference's Problem concept
/// (periodic.hpp:23-31: n_dof, mass, apply_k, jacobian_k).
class GridProblem {
 public:
  explicit GridProblem(const tp_problem_desc& d) : d_(d) {
    validate_desc(d);
    const int c = d.cells;
    auto mesh = std::make_shared<tpfem::Mesh>();
    mesh->xmin = mesh->ymin = 0.0;
    mesh->xmax = mesh->ymax = 1.0;
    for (int j = 0; j <= c; ++j)
      for (int i = 0; i <= c; ++i)
        mesh->vertices.push_back({static_cast<double>(i) / c, static_cast<double>(j) / c});
    const Index cols = c + 1;
    for (int j = 0; j < c; ++j)
      for (int i = 0; i < c; ++i) {
        const double cx = (2.0 * i + 1.0) / (2.0 * c), cy = (2.0 * j + 1.0) / (2.0 * c);
        int mat = 0;
        for (int r = 0; r < d.n_rects; ++r) {
          const tp_rect& R = d.rect[r];
          if (cx >= R.x0 && cx <= R.x1 && cy >= R.y0 && cy <= R.y1) mat = R.material;
        }
        const Index v00 = j * cols + i, v10 = v00 + 1, v01 = v00 + cols, v11 = v01 + 1;
        mesh->triangles.push_back({v00, v10, v11});
        mesh->triangles.push_back({v00, v11, v01});
        mesh->region.push_back(static_cast<tpfem::Region>(mat));
        mesh->region.push_back(static_cast<tpfem::Region>(mat));
      }
    tpfem::detail::finalize_mesh(*mesh);
    mesh_ = mesh;
    op_ = std::make_unique<tpfem::NonlinearOperator>(mesh_, tpfem::MaterialTable{});
    const auto& elems = op_->elements();
    for (int m = 0; m < TP_MAX_MATERIALS; ++m) {
      if (m < d.n_materials) law_[m] = {d.material[m].nu0, d.material[m].nu_inf, d.material[m].bs};
    }
    // Per-triangle sigma (triangle t of cell (i,j): t = 2*(j*c+i) + {0: lower-right, 1: upper-left}).
    const SigmaNoise noise(d.noise_lattice >= 2 ? d : with_default_lattice(d));
    sigma_.resize(elems.size());
    for (std::size_t t = 0; t < elems.size(); ++t) {
      const tp_material& mt = d.material[static_cast<int>(elems[t].region)];
      double s = mt.sigma;
      if (mt.sigma_noise) {
        const long cell = static_cast<long>(t / 2);
        const long i = cell % c, j = cell / c;
        const bool lower = (t % 2) == 0;
        const double x = (3.0 * i + (lower ? 2.0 : 1.0)) / (3.0 * c);
        const double y = (3.0 * j + (lower ? 1.0 : 2.0)) / (3.0 * c);
        s = mt.sigma * noise.at(x, y);
      }
      sigma_[t] = s;
    }
    // Lumped mass: m_i = sum_T sigma_T |T| / 3.
    std::vector<tpfem::Triplet<double>> trips;
    for (std::size_t t = 0; t < elems.size(); ++t) {
      if (sigma_[t] == 0) continue;
      const double w = sigma_[t] * elems[t].area / 3.0;
      for (int k = 0; k < 3; ++k)
        if (elems[t].dof[k] >= 0) trips.push_back({elems[t].dof[k], elems[t].dof[k], w});
    }
    M_ = tpfem::SparseMatrix<double>::from_triplets(n_dof(), n_dof(), std::move(trips), true);
  }

  Index n_dof() const { return mesh_->n_dof(); }
  int steps() const { return d_.steps; }
  double tau() const { return d_.period / d_.steps; }
  const tpfem::SparseMatrix<double>& mass() const { return M_; }
  const tpfem::Mesh& mesh() const { return *mesh_; }
  const tpfem::NonlinearOperator& geometry() const { return *op_; }
  const Law& law(int m) const { return law_[m]; }
  const std::vector<double>& sigma() const { return sigma_; }

  /// out_i = integral nu(|grad u|) grad u . grad phi_i  (assembly.hpp:126-140).
  void apply_k(const double* u, double* out) const {
    for (Index i = 0; i < n_dof(); ++i) out[i] = 0;
    for (const tpfem::ElementData& e : op_->elements()) {
      double gx = 0, gy = 0;
      for (int k = 0; k < 3; ++k) {
        if (e.dof[k] < 0) continue;
        gx += u[e.dof[k]] * e.gx[k];
        gy += u[e.dof[k]] * e.gy[k];
      }
      const double s = std::hypot(gx, gy);
      const double nu = law_[static_cast<int>(e.region)].nu(s);
      for (int k = 0; k < 3; ++k)
        if (e.dof[k] >= 0) out[e.dof[k]] += nu * e.area * (gx * e.gx[k] + gy * e.gy[k]);
    }
  }

  /// Jacobian [nu I + (nu'/s) g g^T] per element (assembly.hpp:153-177).
  tpfem::SparseMatrix<double> jacobian_k(const double* u) const {
    std::vector<tpfem::Triplet<double>> trips;
    for (const tpfem::ElementData& e : op_->elements()) {
      double gx = 0, gy = 0;
      for (int k = 0; k < 3; ++k) {
        if (e.dof[k] < 0) continue;
        gx += u[e.dof[k]] * e.gx[k];
        gy += u[e.dof[k]] * e.gy[k];
      }
      const double s = std::hypot(gx, gy);
      const Law& law = law_[static_cast<int>(e.region)];
      const double nu = law.nu(s);
      double rank1 = 0;
      if (s > 0) rank1 = law.nu_prime(s) / s;
      for (int i = 0; i < 3; ++i) {
        if (e.dof[i] < 0) continue;
        for (int j = 0; j < 3; ++j) {
          if (e.dof[j] < 0) continue;
          const double iso = nu * (e.gx[i] * e.gx[j] + e.gy[i] * e.gy[j]);
          const double dir = rank1 * (gx * e.gx[i] + gy * e.gy[i]) * (gx * e.gx[j] + gy * e.gy[j]);
          trips.push_back({e.dof[i], e.dof[j], e.area * (iso + dir)});
        }
      }
    }
    return tpfem::SparseMatrix<double>::from_triplets(n_dof(), n_dof(), std::move(trips), true);
  }

  /// Source current of material m at time t (materials.hpp:60-65 with sines).
  double source_current(int m, double t) const {
    const tp_material& mt = d_.material[m];
    double j = 0;
    for (int h = 0; h < mt.n_harmonics; ++h)
      j += mt.amp[h] * std::sin(2.0 * std::numbers::pi * mt.harmonic[h] * t / d_.period + mt.phase[h]);
    return j;
  }

  /// f^n_i = integral j(t^n) phi_i, t^n = (n+1) T/N, one-third rule (assembly.hpp:88-106).
  tpfem::BlockRhs loads() const {
    const int N = d_.steps;
    tpfem::BlockRhs f(N, n_dof());
    for (int n = 0; n < N; ++n) load_slice(n, f.block(n));
    return f;
  }

  /// f^n alone (fn zero-initialised by the caller), for samples of configs
  /// whose whole F does not fit in host memory.
  void load_slice(int n, double* fn) const {
    const double t = (n + 1) * d_.period / d_.steps;
    for (const tpfem::ElementData& e : op_->elements()) {
      const double j = source_current(static_cast<int>(e.region), t);
      if (j == 0) continue;
      const double contrib = j * e.area / 3.0;
      for (int k = 0; k < 3; ++k)
        if (e.dof[k] >= 0) fn[e.dof[k]] += contrib;
    }
  }

  /// Sampled eigenvalue range of the flux-map Jacobian (materials.hpp:112-128).
  tpfem::RegionBounds flux_jacobian_bounds(int m, double s_lo, double s_hi, int samples) const {
    if (!(s_lo >= 0) || !(s_hi >= s_lo))
      throw std::invalid_argument("flux bounds: need 0 <= s_lo <= s_hi");
    if (samples < 2) throw std::invalid_argument("flux bounds: need at least 2 samples");
    tpfem::RegionBounds b;
    b.lambda = std::numeric_limits<double>::infinity();
    b.Lambda = 0;
    for (int j = 0; j < samples; ++j) {
      const double s = s_lo + (s_hi - s_lo) * j / (samples - 1);
      const double nu = law_[m].nu(s);
      const double gp = nu + law_[m].nu_prime(s) * s;
      b.lambda = std::min({b.lambda, nu, gp});
      b.Lambda = std::max({b.Lambda, nu, gp});
    }
    return b;
  }

  /// Frozen-field / theory nu_hat (assembly.hpp:254-291); materials beyond
  /// n_materials get nu_hat = 1 so the reference's positivity check passes.
  tpfem::NuHatChoice choose_nu_hat(tpfem::NuHatMode mode, const tpfem::PeriodicState& U0,
                                   int samples) const {
    tpfem::RegionFieldRanges ranges;
    if (mode == tpfem::NuHatMode::frozen_field)
      for (int i = 0; i < U0.steps; ++i) tpfem::absorb_field_ranges(*op_, U0.block(i), ranges);
    tpfem::NuHatChoice out;
    for (int r = 0; r < tpfem::kNumRegions; ++r) {
      if (r >= d_.n_materials) {
        out.nu_hat[static_cast<std::size_t>(r)] = 1.0;
        continue;
      }
      const tpfem::RegionBounds full = flux_jacobian_bounds(r, 0.0, d_.s_max, d_.flux_samples);
      const tpfem::FieldRange& range = ranges[static_cast<std::size_t>(r)];
      if (mode == tpfem::NuHatMode::theory) {
        out.nu_hat[static_cast<std::size_t>(r)] = 0.5 * (full.lambda + full.Lambda);
        out.q = std::max(out.q, (full.Lambda - full.lambda) / (full.Lambda + full.lambda));
        continue;
      }
      if (!range.any) {
        out.nu_hat[static_cast<std::size_t>(r)] = 0.5 * (full.lambda + full.Lambda);
        continue;
      }
      const double margin = 0.2 * (range.hi - range.lo) + 1e-3;
      const double lo = std::max(0.0, range.lo - margin);
      const double hi = range.hi + margin;
      const tpfem::RegionBounds b = flux_jacobian_bounds(r, lo, hi, samples);
      out.nu_hat[static_cast<std::size_t>(r)] = 0.5 * (b.lambda + b.Lambda);
      out.q = std::max(out.q, (b.Lambda - b.lambda) / (b.Lambda + b.lambda));
    }
    return out;
  }

  tpfem::SparseMatrix<double> stiffness_frozen(const std::array<double, tpfem::kNumRegions>& nu_hat) const {
    return tpfem::assemble_stiffness_frozen(*mesh_, nu_hat);
  }

 private:
  static tp_problem_desc with_default_lattice(tp_problem_desc d) {
    d.noise_lattice = 8;
    d.noise_lo = 0.5;
    d.noise_hi = 1.5;
    return d;
  }

  tp_problem_desc d_;
  std::shared_ptr<const tpfem::Mesh> mesh_;
  std::unique_ptr<tpfem::NonlinearOperator> op_;
  std::array<Law, TP_MAX_MATERIALS> law_{};
  std::vector<double> sigma_;
  tpfem::SparseMatrix<double> M_;
};

}  // namespace tporacle
