// Fine-level (level 0, frequency mode) kernels of the MG-COCG solver,
// written as warp-streaming stencils.
//
// On the fine grid lambda_k M + K_hat is a 5-point operator whose
// coefficients are cheap to regenerate: K_hat's edge weights come from the
// cell materials (1 byte per cell) and nu_hat (K_hat(V,E) = -(nu_hat(T1) +
// nu_hat(T2'))/2 for the two triangles on the edge -- assemble_stiffness_frozen,
// assembly.hpp:68-84, on the uniform right-triangle grid) and M is the lumped
// diagonal.  So the kernels stream only the complex vectors: a warp owns a
// strip of columns (one column per lane, halo lanes on both sides) and
// walks a chunk of rows, keeping the rows it needs in registers; east/west
// neighbours come from warp shuffles, north/south from the register window.
// No shared memory, no block barriers, one 512-byte coalesced row load per
// vector per step, the next row's loads issued before the current row's math.
//
//   k_fine_apply   p = z + beta p ; q = A p ; partial p^T q          (COCG)
//                  or r = b - A x, partials ||b||^2, ||r||^2         (init)
//   k_fine_down    z1 = w r/d ; z2 = z1 + w (r - A z1)/d ; res = r - A z2 ;
//                  b_c = P^T res ; writes z2 and b_c                  (V-cycle down)
//   k_fine_up      zc = z2 + P x_c ; z3, z4 = two Jacobi steps ;
//                  writes z4, partial r^T z4                          (V-cycle up)
#include "mg.cuh"

namespace tpgpu {

namespace {

constexpr int WL = 32;     // lanes per warp
constexpr int WPB = 4;     // warps per block
constexpr int RH = 64;     // rows per warp work item

__device__ __forceinline__ cplx cm(cplx a, cplx b) {
  return {fma(a.re, b.re, -a.im * b.im), fma(a.re, b.im, a.im * b.re)};
}
__device__ __forceinline__ cplx cinv(cplx a) {
  const double d = 1.0 / fma(a.re, a.re, a.im * a.im);
  return {a.re * d, -a.im * d};
}
__device__ __forceinline__ cplx cs(double s, cplx a) { return {s * a.re, s * a.im}; }
__device__ __forceinline__ cplx shf_up(cplx v) {
  return {__shfl_up_sync(0xffffffffu, v.re, 1), __shfl_up_sync(0xffffffffu, v.im, 1)};
}
__device__ __forceinline__ cplx shf_dn(cplx v) {
  return {__shfl_down_sync(0xffffffffu, v.re, 1), __shfl_down_sync(0xffffffffu, v.im, 1)};
}

// Per-lane coefficient rows.  Cell row j: A = nu_hat(mat(x+1, j)), B = nu_hat(mat(x, j)).
struct CellRow {
  double A, B;
};

__device__ __forceinline__ CellRow cell_row(const FineOp& op, int x, int j) {
  // lanes outside the domain (x < 0 or x >= m) read clamped cells; their
  // values never reach an owned output (vectors are zero there)
  const int c = op.c;
  const int jj = min(max(j, 0), c - 1);
  const int i1 = min(max(x + 1, 0), c - 1), i0 = min(max(x, 0), c - 1);
  const uint8_t* row = op.cmat + (size_t)jj * c;
  return {__ldg(op.nuh + row[i1]), __ldg(op.nuh + row[i0])};
}

struct Coef {
  double kc, we, ww, wn, ws, mm;
};

// node row y uses cell rows y (lower) and y+1 (upper)
__device__ __forceinline__ Coef coef_of(const CellRow& lo, const CellRow& up, double mass) {
  Coef k;
  k.we = 0.5 * (up.A + lo.A);
  k.ww = 0.5 * (up.B + lo.B);
  k.wn = 0.5 * (up.A + up.B);
  k.ws = 0.5 * (lo.A + lo.B);
  k.kc = (up.A + lo.A) + (up.B + lo.B);
  k.mm = mass;
  return k;
}

__device__ __forceinline__ cplx diag(const Coef& k, cplx l) { return {fma(l.re, k.mm, k.kc), l.im * k.mm}; }

// (A v) at a node: d v - wE vE - wW vW - wN vN - wS vS (neighbours of
// Dirichlet vertices are zero vectors, their edge weights stay on the diagonal)
__device__ __forceinline__ cplx apply_at(const Coef& k, cplx l, cplx v, cplx vw, cplx ve, cplx vs, cplx vn) {
  cplx acc = cm(diag(k, l), v);
  acc.re -= k.we * ve.re + k.ww * vw.re + k.wn * vn.re + k.ws * vs.re;
  acc.im -= k.we * ve.im + k.ww * vw.im + k.wn * vn.im + k.ws * vs.im;
  return acc;
}

__device__ __forceinline__ void warp_pair(double& a, double& b) {
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_down_sync(0xffffffffu, a, o);
    b += __shfl_down_sync(0xffffffffu, b, o);
  }
}

struct Item {
  int b, strip, chunk, ys, ye, xs;
  bool ok;
};

// warp work item: ((b * nch) + chunk) * ns + strip
__device__ __forceinline__ Item item_of(int m, int own, int nb, const int* __restrict__ active) {
  Item it;
  const int w = blockIdx.x * WPB + (threadIdx.x >> 5);
  const int ns = (m + own - 1) / own, nch = (m + RH - 1) / RH;
  it.strip = w % ns;
  it.chunk = (w / ns) % nch;
  it.b = w / (ns * nch);
  it.ok = it.b < nb && (!active || active[it.b]);
  it.ys = it.chunk * RH;
  it.ye = min(it.ys + RH, m);
  it.xs = it.strip * own;
  return it;
}

__device__ __forceinline__ cplx ld(const cplx* __restrict__ v, int x, int y, int m, bool colok) {
  return (colok && y >= 0 && y < m) ? v[(size_t)y * m + x] : cplx{0, 0};
}

// ---------------------------------------------------------------- apply
// INIT = 0: p = first ? z : z + beta p_in -> p_out ; q = A p ; part += p^T q
// INIT = 1: r = b - A x (b in z, x in pin, r to q) ; part += (|b|^2, |r|^2)
template <int INIT>
__global__ void __launch_bounds__(WL * WPB) k_fine_apply(FineOp op, const cplx* __restrict__ z,
                                                         const cplx* __restrict__ pin, cplx* __restrict__ pout,
                                                         cplx* __restrict__ q, const cplx* __restrict__ beta,
                                                         const int* __restrict__ active, int first, int nb,
                                                         double* __restrict__ part) {
  constexpr int H = 1, OWN = WL - 2 * H;
  const int m = op.m;
  const Item it = item_of(m, OWN, nb, INIT ? nullptr : active);
  if (!it.ok) return;
  const int lane = threadIdx.x & 31;
  const int x = it.xs - H + lane;
  const bool colok = x >= 0 && x < m;
  const bool own = lane >= H && lane < WL - H && colok;
  const size_t o = (size_t)it.b * op.n;
  const cplx* zb = z + o;
  const cplx* pb = pin + o;
  const cplx l = op.lam[it.b];
  const cplx bt = (INIT || first) ? cplx{0, 0} : beta[it.b];
  // rows: p at y-1, y, y+1 around the output row y
  auto pval = [&](int y) -> cplx {
    if (INIT) return ld(pb, x, y, m, colok);  // x (solution) for the residual
    cplx v = ld(zb, x, y, m, colok);
    if (!first) {
      const cplx pp = ld(pb, x, y, m, colok);
      v = {fma(bt.re, pp.re, fma(-bt.im, pp.im, v.re)), fma(bt.re, pp.im, fma(bt.im, pp.re, v.im))};
    }
    return v;
  };
  CellRow clo = cell_row(op, x, it.ys), cup = cell_row(op, x, it.ys + 1);
  cplx pm = pval(it.ys - 1), p0 = pval(it.ys), pn = pval(it.ys + 1);
  double s0 = 0, s1 = 0;
  for (int y = it.ys; y < it.ye; ++y) {
    // prefetch row y+2 and the next upper cell row
    const cplx pnn = pval(y + 2);
    const CellRow cnext = cell_row(op, x, y + 2);
    const double mass = colok ? __ldg(op.mass + (size_t)y * m + x) : 0.0;
    const Coef k = coef_of(clo, cup, mass);
    const cplx pw = shf_up(p0), pe = shf_dn(p0);
    const cplx Ap = apply_at(k, l, p0, pw, pe, pm, pn);
    if (own) {
      const size_t i = o + (size_t)y * m + x;
      if (INIT) {
        const cplx bi = zb[(size_t)y * m + x];
        const cplx r = {bi.re - Ap.re, bi.im - Ap.im};
        q[i] = r;
        s0 += bi.re * bi.re + bi.im * bi.im;
        s1 += r.re * r.re + r.im * r.im;
      } else {
        pout[i] = p0;
        q[i] = Ap;
        const cplx t = cm(p0, Ap);
        s0 += t.re;
        s1 += t.im;
      }
    }
    pm = p0;
    p0 = pn;
    pn = pnn;
    clo = cup;
    cup = cnext;
  }
  warp_pair(s0, s1);
  if (lane == 0) {
    const int ns = (m + OWN - 1) / OWN, nch = (m + RH - 1) / RH;
    const size_t per = (size_t)ns * nch;
    const size_t k = (size_t)it.b * per + (size_t)it.chunk * ns + it.strip;
    part[2 * k] = s0;
    part[2 * k + 1] = s1;
  }
}

// ---------------------------------------------------------------- down
__global__ void __launch_bounds__(WL * WPB, 5) k_fine_down(FineOp op, const cplx* __restrict__ rv,
                                                        cplx* __restrict__ z2out, cplx* __restrict__ bc,
                                                        int mc, const int* __restrict__ active, double omega,
                                                        int nb) {
  constexpr int H = 3, OWN = 26;  // lanes 3..28 own fine columns; even strip start
  const int m = op.m;
  const Item it = item_of(m, OWN, nb, active);
  if (!it.ok) return;
  const int lane = threadIdx.x & 31;
  const int x = it.xs - H + lane;
  const bool colok = x >= 0 && x < m;
  const bool own = lane >= H && lane < H + OWN && colok;
  const size_t o = (size_t)it.b * op.n;
  const cplx* rb = rv + o;
  const cplx l = op.lam[it.b];
  const int ys = it.ys, ye = it.ye;
  // pipeline over input rows yi = ys-2 .. ye+2 (z1 rows), z2 rows yi-1, residual rows yi-2
  // windows
  cplx r0 = {0, 0}, r1 = {0, 0}, r2 = {0, 0};      // r at yi, yi-1, yi-2
  cplx a0 = {0, 0}, a1 = {0, 0}, a2 = {0, 0};      // z1 at yi, yi-1, yi-2
  cplx b1 = {0, 0}, b2 = {0, 0}, b3 = {0, 0};      // z2 at yi-1, yi-2, yi-3
  cplx q2 = {0, 0}, q3 = {0, 0}, q4 = {0, 0};      // res at yi-2, yi-3, yi-4
  // cell rows yi+1, yi, yi-1, yi-2 and masses of node rows yi, yi-1, yi-2
  CellRow cr0 = cell_row(op, x, ys - 1), cr1 = cell_row(op, x, ys - 2), cr2{0, 0}, cr3{0, 0};
  double ms0 = 0, ms1 = 0, ms2 = 0;
  cplx rnext = ld(rb, x, ys - 2, m, colok);
  for (int yi = ys - 2; yi <= ye + 2; ++yi) {
    const cplx rcur = rnext;
    if (yi + 1 <= ye + 2) rnext = ld(rb, x, yi + 1, m, colok);
    const bool rowok = yi >= 0 && yi < m;
    // shift windows
    if (yi > ys - 2) {
      cr3 = cr2; cr2 = cr1; cr1 = cr0;
      cr0 = cell_row(op, x, yi + 1);
    }
    ms2 = ms1; ms1 = ms0;
    ms0 = (colok && rowok) ? __ldg(op.mass + (size_t)yi * m + x) : 0.0;
    r2 = r1; r1 = r0; r0 = rcur;
    a2 = a1; a1 = a0;
    a0 = (colok && rowok) ? cs(omega, cm(r0, cinv(diag(coef_of(cr1, cr0, ms0), l)))) : cplx{0, 0};
    // z2 at row yi-1
    b3 = b2; b2 = b1;
    {
      const int y = yi - 1;
      const cplx aw = shf_up(a1), ae = shf_dn(a1);
      if (colok && y >= 0 && y < m) {
        const Coef k1 = coef_of(cr2, cr1, ms1);
        const cplx Aa = apply_at(k1, l, a1, aw, ae, a2, a0);
        const cplx d = diag(k1, l);
        const cplx t = cm({r1.re - Aa.re, r1.im - Aa.im}, cinv(d));
        b1 = {fma(omega, t.re, a1.re), fma(omega, t.im, a1.im)};
      } else {
        b1 = {0, 0};
      }
      if (own && y >= ys && y < ye) z2out[o + (size_t)y * m + x] = b1;
    }
    // residual at row yi-2
    q4 = q3; q3 = q2;
    {
      const int y = yi - 2;
      const cplx bw = shf_up(b2), be = shf_dn(b2);
      if (colok && y >= 0 && y < m) {
        const cplx Ab = apply_at(coef_of(cr3, cr2, ms2), l, b2, bw, be, b3, b1);
        q2 = {r2.re - Ab.re, r2.im - Ab.im};
      } else {
        q2 = {0, 0};
      }
    }
    // restriction: centre row yc = yi-3 (odd fine row 2Y+1 inside the owned rows)
    {
      const int yc = yi - 3;
      const cplx qw = shf_up(q3), qe = shf_dn(q3);
      const cplx q4w = shf_up(q4), q2e = shf_dn(q2);
      if (yc >= ys && yc < ye && (yc & 1) && own && (x & 1)) {
        const int X = x >> 1, Y = yc >> 1;
        if (X < mc && Y < mc) {
          cplx acc = q3;
          acc.re += 0.5 * (qw.re + qe.re + q4.re + q2.re + q4w.re + q2e.re);
          acc.im += 0.5 * (qw.im + qe.im + q4.im + q2.im + q4w.im + q2e.im);
          bc[(size_t)it.b * mc * mc + (size_t)Y * mc + X] = acc;
        }
      }
    }
  }
}

// ---------------------------------------------------------------- up
__global__ void __launch_bounds__(WL * WPB, 5) k_fine_up(FineOp op, const cplx* __restrict__ rv,
                                                      const cplx* __restrict__ z2in, const cplx* __restrict__ xc,
                                                      int mc, cplx* __restrict__ zout,
                                                      const int* __restrict__ active, double omega, int nb,
                                                      int dot, double* __restrict__ part) {
  constexpr int H = 2, OWN = WL - 2 * H;  // 28
  const int m = op.m;
  const Item it = item_of(m, OWN, nb, active);
  if (!it.ok) return;
  const int lane = threadIdx.x & 31;
  const int x = it.xs - H + lane;
  const bool colok = x >= 0 && x < m;
  const bool own = lane >= H && lane < WL - H && colok;
  const size_t o = (size_t)it.b * op.n;
  const size_t oc = (size_t)it.b * mc * mc;
  const cplx* rb = rv + o;
  const cplx* zb = z2in + o;
  const cplx* xb = xc + oc;
  const cplx l = op.lam[it.b];
  const int ys = it.ys, ye = it.ye;
  // P1 prolongation of the coarse correction at fine node (x, y)
  auto zc_at = [&](int y) -> cplx {
    if (!colok || y < 0 || y >= m) return {0, 0};
    cplx v = zb[(size_t)y * m + x];
    const int a = x + 1, bb = y + 1, ah = a >> 1, bh = bb >> 1;
    auto add = [&](int A, int B, double w) {
      if (A >= 1 && A <= mc && B >= 1 && B <= mc) {
        const cplx c = xb[(size_t)(B - 1) * mc + (A - 1)];
        v.re = fma(w, c.re, v.re);
        v.im = fma(w, c.im, v.im);
      }
    };
    const bool ao = a & 1, bo = bb & 1;
    if (!ao && !bo) add(ah, bh, 1.0);
    else if (ao && !bo) { add(ah, bh, 0.5); add(ah + 1, bh, 0.5); }
    else if (!ao && bo) { add(ah, bh, 0.5); add(ah, bh + 1, 0.5); }
    else { add(ah, bh, 0.5); add(ah + 1, bh + 1, 0.5); }
    return v;
  };
  // pipeline over input rows yi = ys-2 .. ye+1: zc at yi, z3 at yi-1, z4 at yi-2
  cplx c0 = {0, 0}, c1 = {0, 0}, c2 = {0, 0};  // zc at yi, yi-1, yi-2
  cplx r0 = {0, 0}, r1 = {0, 0}, r2 = {0, 0};  // r at yi, yi-1, yi-2
  cplx e1 = {0, 0}, e2 = {0, 0}, e3 = {0, 0};  // z3 at yi-1, yi-2, yi-3
  CellRow cr0 = cell_row(op, x, ys - 1), cr1 = cell_row(op, x, ys - 2), cr2{0, 0}, cr3{0, 0};
  double ms0 = 0, ms1 = 0, ms2 = 0;
  cplx cnext = zc_at(ys - 2), rnext = ld(rb, x, ys - 2, m, colok);
  double s0 = 0, s1 = 0;
  for (int yi = ys - 2; yi <= ye + 1; ++yi) {
    const cplx ccur = cnext, rcur = rnext;
    if (yi + 1 <= ye + 1) {
      cnext = zc_at(yi + 1);
      rnext = ld(rb, x, yi + 1, m, colok);
    }
    const bool rowok = yi >= 0 && yi < m;
    if (yi > ys - 2) {
      cr3 = cr2; cr2 = cr1; cr1 = cr0;
      cr0 = cell_row(op, x, yi + 1);
    }
    ms2 = ms1; ms1 = ms0;
    ms0 = (colok && rowok) ? __ldg(op.mass + (size_t)yi * m + x) : 0.0;
    c2 = c1; c1 = c0; c0 = ccur;
    r2 = r1; r1 = r0; r0 = rcur;
    // z3 at row yi-1
    e3 = e2; e2 = e1;
    {
      const int y = yi - 1;
      const cplx cw = shf_up(c1), ce = shf_dn(c1);
      if (colok && y >= 0 && y < m) {
        const Coef k1 = coef_of(cr2, cr1, ms1);
        const cplx Ac = apply_at(k1, l, c1, cw, ce, c2, c0);
        const cplx t = cm({r1.re - Ac.re, r1.im - Ac.im}, cinv(diag(k1, l)));
        e1 = {fma(omega, t.re, c1.re), fma(omega, t.im, c1.im)};
      } else {
        e1 = {0, 0};
      }
    }
    // z4 at row yi-2
    {
      const int y = yi - 2;
      const cplx ew = shf_up(e2), ee = shf_dn(e2);
      if (own && y >= ys && y < ye) {
        const Coef k2 = coef_of(cr3, cr2, ms2);
        const cplx Ae = apply_at(k2, l, e2, ew, ee, e3, e1);
        const cplx t = cm({r2.re - Ae.re, r2.im - Ae.im}, cinv(diag(k2, l)));
        const cplx z4 = {fma(omega, t.re, e2.re), fma(omega, t.im, e2.im)};
        zout[o + (size_t)y * m + x] = z4;
        if (dot) {
          const cplx pr = cm(r2, z4);
          s0 += pr.re;
          s1 += pr.im;
        }
      }
    }
  }
  if (dot) {
    warp_pair(s0, s1);
    if (lane == 0) {
      const int ns = (m + OWN - 1) / OWN, nch = (m + RH - 1) / RH;
      const size_t per = (size_t)ns * nch;
      const size_t k = (size_t)it.b * per + (size_t)it.chunk * ns + it.strip;
      part[2 * k] = s0;
      part[2 * k + 1] = s1;
    }
  }
}

int items_per_batch(int m, int own) { return ((m + own - 1) / own) * ((m + RH - 1) / RH); }

dim3 grid_for(int m, int own, int nb) {
  const long warps = (long)items_per_batch(m, own) * nb;
  return dim3((unsigned)((warps + WPB - 1) / WPB));
}

}  // namespace

int fine_partials(int m, int kind) { return items_per_batch(m, kind == 0 ? 30 : kind == 1 ? 26 : 28); }

void launch_fine_apply(Problem& p, const FineOp& op, const cplx* z, const cplx* pin, cplx* pout, cplx* q,
                       const cplx* beta, const int* active, int first, int nb, double* part, bool init) {
  const dim3 g = grid_for(op.m, 30, nb);
  if (init)
    k_fine_apply<1><<<g, WL * WPB, 0, p.stream>>>(op, z, pin, pout, q, beta, active, first, nb, part);
  else
    k_fine_apply<0><<<g, WL * WPB, 0, p.stream>>>(op, z, pin, pout, q, beta, active, first, nb, part);
  TP_LAUNCHED(&p);
}

void launch_fine_down(Problem& p, const FineOp& op, const cplx* r, cplx* z2, cplx* bc, int mc,
                      const int* active, double omega, int nb) {
  k_fine_down<<<grid_for(op.m, 26, nb), WL * WPB, 0, p.stream>>>(op, r, z2, bc, mc, active, omega, nb);
  TP_LAUNCHED(&p);
}

void launch_fine_up(Problem& p, const FineOp& op, const cplx* r, const cplx* z2, const cplx* xc, int mc,
                    cplx* z, const int* active, double omega, int nb, int dot, double* part) {
  k_fine_up<<<grid_for(op.m, 28, nb), WL * WPB, 0, p.stream>>>(op, r, z2, xc, mc, z, active, omega, nb, dot,
                                                              part);
  TP_LAUNCHED(&p);
}

}  // namespace tpgpu
