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
__device__ __forceinline__ cplx cs(double s, cplx a) { return {s * a.re, s * a.im}; }
__device__ __forceinline__ cplx shf_up(cplx v) {
  return {__shfl_up_sync(0xffffffffu, v.re, 1), __shfl_up_sync(0xffffffffu, v.im, 1)};
}
__device__ __forceinline__ cplx shf_dn(cplx v) {
  return {__shfl_down_sync(0xffffffffu, v.re, 1), __shfl_down_sync(0xffffffffu, v.im, 1)};
}

// Per-row coefficients of the lane's node: K_hat edge weights to E/W/N/S
// (the diagonal is their sum) and the lumped mass.  op.we / op.wn are
// (c+1)^2 vertex grids: we[Y][X] = weight of the edge (X,Y)-(X+1,Y),
// wn[Y][X] = weight of the edge (X,Y)-(X,Y+1); node (x,y) is vertex (x+1,y+1).
struct RowK {
  double we, ww, wn, ws, mm;
};

// Load the lane's row-y coefficients; ws comes from the previous row's wn,
// ww from the west lane's we (warp shuffle, all lanes participate).
__device__ __forceinline__ RowK row_k(const FineOp& op, int x, int y, double wn_prev) {
  const int c = op.c, m = op.m;
  const int X = min(max(x + 1, 0), c), Y = min(max(y + 1, 0), c);
  const size_t v = (size_t)Y * (c + 1) + X;
  RowK k;
  k.we = __ldg(op.we + v);
  k.wn = __ldg(op.wn + v);
  k.ww = __shfl_up_sync(0xffffffffu, k.we, 1);
  k.ws = wn_prev;
  k.mm = (x >= 0 && x < m && y >= 0 && y < m) ? __ldg(op.mass + (size_t)y * m + x) : 0.0;
  return k;
}
// Compact per-row window entry: the lane's own we, wn and mass.
struct RowW {
  double we, wn, mm;
};
__device__ __forceinline__ RowW row_w(const FineOp& op, int x, int y) {
  const int c = op.c, m = op.m;
  const int X = min(max(x + 1, 0), c), Y = min(max(y + 1, 0), c);
  const size_t v = (size_t)Y * (c + 1) + X;
  RowW w;
  w.we = __ldg(op.we + v);
  w.wn = __ldg(op.wn + v);
  w.mm = (x >= 0 && x < m && y >= 0 && y < m) ? __ldg(op.mass + (size_t)y * m + x) : 0.0;
  return w;
}
// full coefficients of a row from its window entry and the row below (all lanes call)
__device__ __forceinline__ RowK expand(const RowW& w, const RowW& below) {
  return {w.we, __shfl_up_sync(0xffffffffu, w.we, 1), w.wn, below.wn, w.mm};
}
// wn of row y-1 for the first row of a chunk
__device__ __forceinline__ double wn_of(const FineOp& op, int x, int y) {
  const int c = op.c;
  const int X = min(max(x + 1, 0), c), Y = min(max(y + 1, 0), c);
  return __ldg(op.wn + (size_t)Y * (c + 1) + X);
}

__device__ __forceinline__ cplx diag(const RowK& k, cplx l) {
  const double kc = (k.we + k.ww) + (k.wn + k.ws);
  return {fma(l.re, k.mm, kc), l.im * k.mm};
}
__device__ __forceinline__ cplx rcp(cplx a) {
  const double d = __drcp_rn(fma(a.re, a.re, a.im * a.im));
  return {a.re * d, -a.im * d};
}

// (A v) at a node: d v - wE vE - wW vW - wN vN - wS vS (neighbours of
// Dirichlet vertices are zero vectors, their edge weights stay on the diagonal)
__device__ __forceinline__ cplx apply_at(const RowK& k, cplx l, cplx v, cplx vw, cplx ve, cplx vs, cplx vn) {
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


// Row-streamed vector access: pointer to (row y, lane column), zero outside.
struct RowPtr {
  const cplx* p;  // element (y, x) of the current row (clamped column)
  int m;
  bool colok;
  __device__ __forceinline__ cplx at(int y) const {
    return (colok && y >= 0 && y < m) ? p[(long)y * m] : cplx{0, 0};
  }
};

// ---------------------------------------------------------------- apply
// INIT = 0: p = first ? z : z + beta p_in -> p_out ; q = A p ; part += p^T q
// INIT = 1: r = b - A x (b in z, x in pin, r to q) ; part += (|b|^2, |r|^2)
template <int INIT>
__global__ void __launch_bounds__(WL * WPB, 6) k_fine_apply(FineOp op, const cplx* __restrict__ z,
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
  const int xc = min(max(x, 0), m - 1);
  const size_t o = (size_t)it.b * op.n;
  const RowPtr Z{z + o + xc, m, colok}, P{pin + o + xc, m, colok};
  cplx* const po = pout + o + xc;
  cplx* const qo = q + o + xc;
  const cplx l = op.lam[it.b];
  const cplx bt = (INIT || first) ? cplx{0, 0} : beta[it.b];
  auto pval = [&](int y) -> cplx {
    if (INIT) return P.at(y);  // x (solution) for the residual
    cplx v = Z.at(y);
    if (!first) {
      const cplx pp = P.at(y);
      v = {fma(bt.re, pp.re, fma(-bt.im, pp.im, v.re)), fma(bt.re, pp.im, fma(bt.im, pp.re, v.im))};
    }
    return v;
  };
  double wnp = wn_of(op, x, it.ys - 1);
  cplx pm = pval(it.ys - 1), p0 = pval(it.ys), pn = pval(it.ys + 1);
  double s0 = 0, s1 = 0;
  for (int y = it.ys; y < it.ye; ++y) {
    const cplx pnn = pval(y + 2);  // next row in flight during this row's math
    const RowK k = row_k(op, x, y, wnp);
    wnp = k.wn;
    const cplx pw = shf_up(p0), pe = shf_dn(p0);
    const cplx Ap = apply_at(k, l, p0, pw, pe, pm, pn);
    if (own) {
      const long i = (long)y * m;
      if (INIT) {
        const cplx bi = Z.p[i];
        const cplx r = {bi.re - Ap.re, bi.im - Ap.im};
        qo[i] = r;
        s0 += bi.re * bi.re + bi.im * bi.im;
        s1 += r.re * r.re + r.im * r.im;
      } else {
        po[i] = p0;
        qo[i] = Ap;
        const cplx t = cm(p0, Ap);
        s0 += t.re;
        s1 += t.im;
      }
    }
    pm = p0;
    p0 = pn;
    pn = pnn;
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
// With q != nullptr the Krylov residual update is fused in: the right-hand
// side is r_new = r - alpha q (read r and q, write r_new to rout for the
// owned block, partial ||r_new||^2 per warp item), replacing the separate
// x/r update pass (x is updated in the next apply, k_apply_dot).
__global__ void __launch_bounds__(WL * WPB, 4) k_fine_down(FineOp op, const cplx* __restrict__ rv,
                                                           cplx* __restrict__ z2out, cplx* __restrict__ bc,
                                                           int mc, const int* __restrict__ active, double om1,
                                                           double om2, int nb, const cplx* __restrict__ qv,
                                                           const cplx* __restrict__ alpha, cplx* __restrict__ rout,
                                                           double* __restrict__ part) {
  constexpr int H = 3, OWN = 26;  // lanes 3..28 own fine columns; even strip start
  const int m = op.m;
  const Item it = item_of(m, OWN, nb, active);
  if (!it.ok) return;
  const int lane = threadIdx.x & 31;
  const int x = it.xs - H + lane;
  const bool colok = x >= 0 && x < m;
  const bool own = lane >= H && lane < H + OWN && colok;
  const int xc = min(max(x, 0), m - 1);
  const size_t o = (size_t)it.b * op.n;
  const RowPtr R{rv + o + xc, m, colok};
  const RowPtr Q{qv ? qv + o + xc : rv + o + xc, m, colok};
  cplx* const ro = rout ? rout + o + xc : nullptr;
  const cplx al = qv ? alpha[it.b] : cplx{0, 0};
  cplx* const zo = z2out + o + xc;
  const cplx l = op.lam[it.b];
  const int ys = it.ys, ye = it.ye;
  const bool cown = own && (x & 1) && (x >> 1) < mc;  // coarse centre column
  double rn2 = 0;
  auto rhs = [&](int y) -> cplx {
    cplx v = R.at(y);
    if (qv) {
      const cplx qq = Q.at(y);
      v.re -= al.re * qq.re - al.im * qq.im;
      v.im -= al.re * qq.im + al.im * qq.re;
    }
    return v;
  };
  cplx* const bco = bc + (size_t)it.b * mc * mc + (x >> 1);
  // pipeline over input rows yi = ys-2 .. ye+2: z1 at yi, z2 at yi-1,
  // residual at yi-2, restriction centred on yi-3
  cplx r0{0, 0}, r1{0, 0}, r2{0, 0};  // r at yi, yi-1, yi-2
  cplx a0{0, 0}, a1{0, 0}, a2{0, 0};  // z1 at yi, yi-1, yi-2
  cplx b1{0, 0}, b2{0, 0}, b3{0, 0};  // z2 at yi-1, yi-2, yi-3
  cplx q2{0, 0}, q3{0, 0}, q4{0, 0};  // res at yi-2, yi-3, yi-4
  RowW w0 = row_w(op, x, ys - 3), w1{}, w2{}, w3{};  // rows yi, yi-1, yi-2, yi-3
  RowW wnx = row_w(op, x, ys - 2);                   // row yi+1 in flight
  cplx rnext = rhs(ys - 2);
  cplx id0{0, 0}, id1{0, 0};  // 1/d of rows yi, yi-1
  for (int yi = ys - 2; yi <= ye + 2; ++yi) {
    const cplx rcur = rnext;
    rnext = rhs(yi + 1);
    if (qv && own && yi >= ys && yi < ye) {
      ro[(long)yi * m] = rcur;
      rn2 += rcur.re * rcur.re + rcur.im * rcur.im;
    }
    r2 = r1; r1 = r0; r0 = rcur;
    w3 = w2; w2 = w1; w1 = w0;
    w0 = wnx;
    wnx = row_w(op, x, yi + 1);
    // z1 = omega r / d at row yi (zero outside the domain: r = 0 there)
    a2 = a1; a1 = a0;
    id1 = id0;
    id0 = rcp(diag(expand(w0, w1), l));
    a0 = cs(om1, cm(r0, id0));
    // z2 at row yi-1
    b3 = b2; b2 = b1;
    {
      const cplx aw = shf_up(a1), ae = shf_dn(a1);
      const RowK k1 = expand(w1, w2);
      const cplx Aa = apply_at(k1, l, a1, aw, ae, a2, a0);
      const cplx t = cm({r1.re - Aa.re, r1.im - Aa.im}, id1);
      const int y = yi - 1;
      const bool in = colok && y >= 0 && y < m;
      b1 = in ? cplx{fma(om2, t.re, a1.re), fma(om2, t.im, a1.im)} : cplx{0, 0};
      if (own && y >= ys && y < ye) zo[(long)y * m] = b1;
    }
    // residual at row yi-2
    q4 = q3; q3 = q2;
    {
      const cplx bw = shf_up(b2), be = shf_dn(b2);
      const cplx Ab = apply_at(expand(w2, w3), l, b2, bw, be, b3, b1);
      const int y = yi - 2;
      q2 = (colok && y >= 0 && y < m) ? cplx{r2.re - Ab.re, r2.im - Ab.im} : cplx{0, 0};
    }
    // restriction centred on row yc = yi-3 (odd fine row 2Y+1 of the chunk)
    {
      const int yc = yi - 3;
      const cplx qw = shf_up(q3), qe = shf_dn(q3);
      const cplx q4w = shf_up(q4), q2e = shf_dn(q2);
      if (cown && (yc & 1) && yc >= ys && yc < ye && (yc >> 1) < mc) {
        cplx acc = q3;
        acc.re += 0.5 * (qw.re + qe.re + q4.re + q2.re + q4w.re + q2e.re);
        acc.im += 0.5 * (qw.im + qe.im + q4.im + q2.im + q4w.im + q2e.im);
        bco[(size_t)(yc >> 1) * mc] = acc;
      }
    }
  }
  if (qv) {
    double z = 0;
    warp_pair(rn2, z);
    if ((threadIdx.x & 31) == 0) {
      const int ns = (m + OWN - 1) / OWN, nch = (m + RH - 1) / RH;
      const size_t k = (size_t)it.b * ((size_t)ns * nch) + (size_t)it.chunk * ns + it.strip;
      part[2 * k] = rn2;
      part[2 * k + 1] = 0.0;
    }
  }
}

// ---------------------------------------------------------------- up
__global__ void __launch_bounds__(WL * WPB, 4) k_fine_up(FineOp op, const cplx* __restrict__ rv,
                                                         const cplx* __restrict__ z2in, const cplx* __restrict__ xcv,
                                                         int mc, cplx* __restrict__ zout,
                                                         const int* __restrict__ active, double om1, double om2, int nb,
                                                         int dot, double* __restrict__ part) {
  constexpr int H = 2, OWN = WL - 2 * H;  // 28
  const int m = op.m;
  const Item it = item_of(m, OWN, nb, active);
  if (!it.ok) return;
  const int lane = threadIdx.x & 31;
  const int x = it.xs - H + lane;
  const bool colok = x >= 0 && x < m;
  const bool own = lane >= H && lane < WL - H && colok;
  const int xc = min(max(x, 0), m - 1);
  const size_t o = (size_t)it.b * op.n;
  const RowPtr R{rv + o + xc, m, colok}, Z2{z2in + o + xc, m, colok};
  cplx* const zo = zout + o + xc;
  const cplx* xb = xcv + (size_t)it.b * mc * mc;
  const cplx l = op.lam[it.b];
  const int ys = it.ys, ye = it.ye;
  // P1 prolongation: fine vertex a = x+1 (column parity fixed per lane)
  const int a = x + 1, ah = a >> 1;
  const bool ao = a & 1;
  auto coarse = [&](int A, int B) -> cplx {
    return (A >= 1 && A <= mc && B >= 1 && B <= mc) ? xb[(size_t)(B - 1) * mc + (A - 1)] : cplx{0, 0};
  };
  auto zc_at = [&](int y) -> cplx {
    cplx v = Z2.at(y);
    if (!colok || y < 0 || y >= m) return v;
    const int bb = y + 1, bh = bb >> 1;
    cplx c1, c2{0, 0};
    double w1 = 0.5;
    if (!ao && !(bb & 1)) { c1 = coarse(ah, bh); w1 = 1.0; }
    else if (ao && !(bb & 1)) { c1 = coarse(ah, bh); c2 = coarse(ah + 1, bh); }
    else if (!ao) { c1 = coarse(ah, bh); c2 = coarse(ah, bh + 1); }
    else { c1 = coarse(ah, bh); c2 = coarse(ah + 1, bh + 1); }
    v.re = fma(w1, c1.re, fma(0.5, c2.re, v.re));
    v.im = fma(w1, c1.im, fma(0.5, c2.im, v.im));
    return v;
  };
  // pipeline over input rows yi = ys-2 .. ye+1: zc at yi, z3 at yi-1, z4 at yi-2
  cplx c0{0, 0}, c1{0, 0}, c2{0, 0};  // zc at yi, yi-1, yi-2
  cplx r0{0, 0}, r1{0, 0}, r2{0, 0};  // r at yi, yi-1, yi-2
  cplx e1{0, 0}, e2{0, 0}, e3{0, 0};  // z3 at yi-1, yi-2, yi-3
  RowW w0 = row_w(op, x, ys - 3), w1{}, w2{}, w3{};  // rows yi, yi-1, yi-2, yi-3
  RowW wnx = row_w(op, x, ys - 2);                   // row yi+1 in flight
  cplx cnext = zc_at(ys - 2), rnext = R.at(ys - 2);
  double s0 = 0, s1 = 0;
  cplx jd1{0, 0}, jd2{0, 0};  // 1/d of rows yi-1, yi-2
  for (int yi = ys - 2; yi <= ye + 1; ++yi) {
    const cplx ccur = cnext, rcur = rnext;
    cnext = zc_at(yi + 1);
    rnext = R.at(yi + 1);
    c2 = c1; c1 = c0; c0 = ccur;
    r2 = r1; r1 = r0; r0 = rcur;
    w3 = w2; w2 = w1; w1 = w0;
    w0 = wnx;
    wnx = row_w(op, x, yi + 1);
    // z3 at row yi-1
    e3 = e2; e2 = e1;
    {
      const cplx cw = shf_up(c1), ce = shf_dn(c1);
      const RowK k1 = expand(w1, w2);
      const cplx Ac = apply_at(k1, l, c1, cw, ce, c2, c0);
      jd2 = jd1;
      jd1 = rcp(diag(k1, l));
      const cplx t = cm({r1.re - Ac.re, r1.im - Ac.im}, jd1);
      const int y = yi - 1;
      e1 = (colok && y >= 0 && y < m) ? cplx{fma(om2, t.re, c1.re), fma(om2, t.im, c1.im)} : cplx{0, 0};
    }
    // z4 at row yi-2
    {
      const cplx ew = shf_up(e2), ee = shf_dn(e2);
      const RowK k2 = expand(w2, w3);
      const int y = yi - 2;
      if (own && y >= ys && y < ye) {
        const cplx Ae = apply_at(k2, l, e2, ew, ee, e3, e1);
        const cplx t = cm({r2.re - Ae.re, r2.im - Ae.im}, jd2);
        const cplx z4 = {fma(om1, t.re, e2.re), fma(om1, t.im, e2.im)};
        zo[(long)y * m] = z4;
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
                      const int* active, double om1, double om2, int nb, const cplx* q, const cplx* alpha,
                      cplx* rout, double* part) {
  k_fine_down<<<grid_for(op.m, 26, nb), WL * WPB, 0, p.stream>>>(op, r, z2, bc, mc, active, om1, om2, nb, q,
                                                               alpha, rout, part);
  TP_LAUNCHED(&p);
}

void launch_fine_up(Problem& p, const FineOp& op, const cplx* r, const cplx* z2, const cplx* xc, int mc,
                    cplx* z, const int* active, double om1, double om2, int nb, int dot, double* part) {
  k_fine_up<<<grid_for(op.m, 28, nb), WL * WPB, 0, p.stream>>>(op, r, z2, xc, mc, z, active, om1, om2, nb, dot,
                                                              part);
  TP_LAUNCHED(&p);
}

}  // namespace tpgpu
