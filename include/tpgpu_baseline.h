/*
 * tpgpu_baseline.h -- the BASELINE.json workload descriptions as plain data
 * (header-only, C99/C++).  Shared by the product (tp_problem_desc_baseline)
 * and the test-side reference driver so both build the same inputs.
 *
 * Geometry not fixed by BASELINE.json (configs 2/3 "transformer-like") and
 * the source amplitude J0 of configs 2/3 are choices of this repo,
 * documented in DESIGN.md §2.
 */
#ifndef TPGPU_BASELINE_H
#define TPGPU_BASELINE_H

#include <string.h>

#include "tpgpu.h"

#define TP_NOISE_SEED 0x5eed2024ULL

static inline void tp_material_set(tp_material* m, double sigma, double nu0, double nu_inf,
                                   double bs) {
  memset(m, 0, sizeof(*m));
  m->sigma = sigma;
  m->nu0 = nu0;
  m->nu_inf = nu_inf;
  m->bs = bs;
}

static inline void tp_material_add_source(tp_material* m, double amp, int32_t harmonic,
                                          double phase) {
  const int32_t h = m->n_harmonics++;
  m->amp[h] = amp;
  m->harmonic[h] = harmonic;
  m->phase[h] = phase;
}

static inline void tp_desc_add_rect(tp_problem_desc* d, double x0, double y0, double x1,
                                    double y1, int32_t material) {
  tp_rect* r = &d->rect[d->n_rects++];
  r->x0 = x0;
  r->y0 = y0;
  r->x1 = x1;
  r->y1 = y1;
  r->material = material;
  r->pad_ = 0;
}

/* Returns 0 on success, 1 for an unknown config id. */
static inline int tp_baseline_desc_fill(int32_t config, tp_problem_desc* d) {
  memset(d, 0, sizeof(*d));
  d->period = 1.0;
  d->noise_seed = TP_NOISE_SEED;
  d->noise_lattice = 8;
  d->noise_lo = 0.5;
  d->noise_hi = 1.5;
  d->s_max = 3.0;
  d->flux_samples = 10001;
  if (config == 0 || config == 1 || config == 4 || config == 5) {
    /* Unit square; conductor [0.25,0.75]^2 (sigma=1); coil [0.1,0.2]x[0.3,0.7];
     * nu(s) = nu0 + (nu_inf-nu0) s^2/(s^2+Bs^2) everywhere. */
    const double bs = (config >= 4) ? 0.5 : 1.0;
    const double j0 = (config >= 4) ? 200.0 : 20.0;
    const double nu_inf = (config == 5) ? 1.0 : 50.0;
    d->cells = (config == 0) ? 32 : (config == 1) ? 256 : 512;
    d->steps = (config == 0) ? 64 : (config == 1) ? 256 : 2048;
    d->n_materials = 3;
    tp_material_set(&d->material[0], 0.0, 1.0, nu_inf, bs); /* background */
    tp_material_set(&d->material[1], 1.0, 1.0, nu_inf, bs); /* conductor */
    tp_material_set(&d->material[2], 0.0, 1.0, nu_inf, bs); /* coil */
    if (config == 1) d->material[1].sigma_noise = 1;
    tp_material_add_source(&d->material[2], j0, 1, 0.0);
    if (config >= 4) {
      tp_material_add_source(&d->material[2], 0.3 * j0, 3, 0.0);
      tp_material_add_source(&d->material[2], 0.1 * j0, 5, 0.0);
    }
    tp_desc_add_rect(d, 0.25, 0.25, 0.75, 0.75, 1);
    tp_desc_add_rect(d, 0.1, 0.3, 0.2, 0.7, 2);
    d->noise_box[0] = 0.25;
    d->noise_box[1] = 0.25;
    d->noise_box[2] = 0.75;
    d->noise_box[3] = 0.75;
    return 0;
  }
  if (config == 2 || config == 3) {
    /* Transformer-like cross-section: iron core (rectangle with a window),
     * two coils in the window, conductive tank strip, air elsewhere. */
    const double nu_inf = 1000.0, j0 = 20.0;
    d->cells = (config == 2) ? 1024 : 2048;
    d->steps = (config == 2) ? 512 : 1024;
    d->n_materials = 5;
    tp_material_set(&d->material[0], 0.0, nu_inf, nu_inf, 1.5); /* air (linear) */
    tp_material_set(&d->material[1], 0.0, 1.0, nu_inf, 1.5);    /* iron */
    tp_material_set(&d->material[2], 0.0, nu_inf, nu_inf, 1.5); /* coil A */
    tp_material_set(&d->material[3], 0.0, nu_inf, nu_inf, 1.5); /* coil B */
    tp_material_set(&d->material[4], 5.0, nu_inf, nu_inf, 1.5); /* tank strip */
    tp_material_add_source(&d->material[2], j0, 1, 0.0);
    tp_material_add_source(&d->material[3], -0.5 * j0, 1, 0.3);
    tp_desc_add_rect(d, 0.15, 0.15, 0.75, 0.85, 1); /* core */
    tp_desc_add_rect(d, 0.30, 0.30, 0.60, 0.70, 0); /* window */
    tp_desc_add_rect(d, 0.33, 0.35, 0.42, 0.65, 2); /* coil A */
    tp_desc_add_rect(d, 0.48, 0.35, 0.57, 0.65, 3); /* coil B */
    tp_desc_add_rect(d, 0.85, 0.10, 0.90, 0.90, 4); /* tank strip */
    return 0;
  }
  return 1;
}

#endif /* TPGPU_BASELINE_H */
