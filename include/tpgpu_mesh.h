/*
 * tpgpu_mesh.h -- general-mesh path of libtpgpu: the
 * reference's own P1 meshes and transformer physics on the device, so the
 * reference's configs (configs/transformer.json, table.json, speedup.json:
 * build_transformer_mesh + MaterialTable::transformer) run through the same
 * fixed-point sweep as the BASELINE grids.
 *
 * What differs from the uniform-grid problem of tpgpu.h:
 *   - any conforming P1 triangulation of a rectangle (vertices, positively
 *     oriented triangles, a region label per triangle); boundary vertices and
 *     dof numbers follow the reference's finalize_mesh (mesh.hpp:86-103);
 *   - the reference's material law nu(s) = a min{exp(b s^2), c} + d with
 *     sigma and a cos source per region (MaterialCoefficients,
 *     materials.hpp:17-24, 42-65);
 *   - the consistent sigma-mass (assemble_mass, assembly.hpp:48-65) and the
 *     element-wise loads F (assemble_loads, assembly.hpp:86-106);
 *   - M1, M2 and M3 (configs/transformer.json's "method": "all");
 *   - every frequency block (and every static-init Newton Jacobian) is
 *     factorised once with a banded complex-symmetric LDL^T in a
 *     reverse-Cuthill-McKee order and solved directly, as the reference's
 *     PeriodicSolver caches one factorisation per block (periodic.hpp:211-248).
 *
 * Conventions are those of tpgpu.h: caller-owned fp64 host arrays in
 * slice-major order X[i*n + j] (dof j of slice i, slice i <-> time (i+1) tau),
 * TP_OK / TP_EINVAL / TP_ESOLVE / TP_ECUDA, tp_last_error() for messages.
 */
#ifndef TPGPU_MESH_H
#define TPGPU_MESH_H

#include "tpgpu.h"

#ifdef __cplusplus
extern "C" {
#endif

/* MaterialCoefficients (materials.hpp:17-24): nu(s) = a*min{exp(b s^2), c} + d,
 * source j(t) = j_amp * cos(2 pi t / T). Region codes (mesh.hpp:17-23):
 * 0 steel, 1 iron, 2 air, 3 winding_plus, 4 winding_minus. */
typedef struct tp_exp_material {
  double sigma, a, b, c, d, j_amp;
} tp_exp_material;

/* A P1 problem: mesh + material table + time discretisation. */
typedef struct tp_mesh_desc {
  int32_t n_vertices;
  int32_t n_triangles;
  const double* vertices;    /* 2 * n_vertices: x, y */
  const int32_t* triangles;  /* 3 * n_triangles, positively oriented */
  const int32_t* region;     /* n_triangles, codes 0..TP_MAX_MATERIALS-1 */
  tp_exp_material material[TP_MAX_MATERIALS];
  int32_t steps;             /* N */
  int32_t flux_samples;      /* theory-mode samples (RunConfig::flux_samples, config.hpp:52; 0 = 10001) */
  double period;             /* T */
  double s_max;              /* theory-mode range (RunConfig::s_max, config.hpp:51; 0 = 3.0) */
} tp_mesh_desc;

typedef struct tp_mesh_problem tp_mesh_problem;

/* MaterialTable::transformer() (materials.hpp:67-79). */
void tp_material_table_transformer(tp_exp_material out[TP_MAX_MATERIALS]);

/* build_rectilinear_mesh(transformer_regions(), nx, ny) followed by
 * `refinements` x refine_uniform (runner.hpp:27-31, mesh.hpp:105-246).
 * Two-call pattern: pass NULL arrays to get the sizes; then arrays of
 * 2*nv doubles, 3*nt and nt int32.  n_dof may be NULL. */
int tp_transformer_mesh(int32_t nx, int32_t ny, int32_t refinements, int32_t* nv, int32_t* nt,
                        int32_t* n_dof, double* vertices, int32_t* triangles, int32_t* region);

/* Setup: element data, consistent mass, loads, banded ordering. */
int tp_mesh_problem_create(const tp_mesh_desc* desc, int32_t device, tp_mesh_problem** out);
void tp_mesh_problem_destroy(tp_mesh_problem* p);
/* n_dof, N, tau and the half-bandwidth of the RCM-ordered operators. */
int tp_mesh_problem_sizes(const tp_mesh_problem* p, int32_t* n_dof, int32_t* steps, double* tau,
                          int32_t* bandwidth);
/* assemble_loads (assembly.hpp:86-106): F, N x n. */
int tp_mesh_loads(tp_mesh_problem* p, double* F);
/* NonlinearOperator::apply (assembly.hpp:126-140) on `count` slices. */
int tp_mesh_apply_k(tp_mesh_problem* p, const double* U, double* KU, int32_t count);
/* residual + block_l2 (periodic.hpp:35-67): R (N x n, may be NULL), ||R||. */
int tp_mesh_residual(tp_mesh_problem* p, const double* U, double* R, double* norm);
/* static_init (solvers.hpp:276-296): Newton per slice from u = 0; U0 (may be
 * NULL: kept as the device state), newton_counts (N, may be NULL). */
int tp_mesh_static_init(tp_mesh_problem* p, const tp_solver_cfg* cfg, double* U0, int32_t* newton_counts);
int tp_mesh_set_state(tp_mesh_problem* p, const double* U);
int tp_mesh_get_state(tp_mesh_problem* p, double* U);
/* choose_nu_hat (assembly.hpp:236-303) over the current state with the
 * flux bounds of the desc's s_max / flux_samples; installs K_hat. */
int tp_mesh_choose_nu_hat(tp_mesh_problem* p, const tp_solver_cfg* cfg, double* nu_hat, double* q);
int tp_mesh_set_nu_hat(tp_mesh_problem* p, const double* nu_hat, double q);
/* PeriodicSolver::solve (periodic.hpp:154-198): G -> U (N x n host). */
int tp_mesh_periodic_solve(tp_mesh_problem* p, const tp_solver_cfg* cfg, const double* G, double* U);
/* solve_m1_fixed_point (solvers.hpp:301-369), outputs as tp_solve_m1. */
int tp_mesh_solve_m1(tp_mesh_problem* p, const tp_solver_cfg* cfg, const double* U0, double* U_out,
                     tp_report* report, double* history, double* contraction, int32_t cap,
                     tp_iterate_cb cb, void* user);
/* solve_m2_newton (solvers.hpp:375-484) and solve_m3_timestepping
 * (solvers.hpp:489-542) on the mesh problem; outputs as tp_solve_m2 / _m3. */
int tp_mesh_solve_m2(tp_mesh_problem* p, const tp_solver_cfg* cfg, const double* U0, double* U_out,
                     tp_report* report, double* history, double* contraction, int32_t cap);
int tp_mesh_solve_m3(tp_mesh_problem* p, const tp_solver_cfg* cfg, const double* U0, double* U_out,
                     tp_report* report, double* history, double* contraction, int32_t cap);
/* device-resident sweeps (benchmarks): factorise the blocks + initial
 * residual; one sweep returning ||R||. */
int tp_mesh_m1_begin(tp_mesh_problem* p, const tp_solver_cfg* cfg, double* residual0);
int tp_mesh_m1_sweep(tp_mesh_problem* p, double* residual);
void* tp_mesh_problem_stream(tp_mesh_problem* p);
int64_t tp_mesh_problem_launches(const tp_mesh_problem* p);

#ifdef __cplusplus
}
#endif

#endif /* TPGPU_MESH_H */
