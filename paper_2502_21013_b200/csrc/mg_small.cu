// The bottom of the frequency-mode V-cycle in one kernel: every level from
// the first one that fits in shared memory (m <= 63 on the baseline grids)
// down to the dense coarsest solve, one thread block per frequency.
//
// Below the fine grid and its first Galerkin level the V-cycle is a chain of
// small passes (a few thousand nodes per frequency and level), each bounded
// by launch latency and by its pipeline fill rather than by bandwidth: seven
// launches per V-cycle for ~40 KB of work per frequency.  Here a block keeps
// every vector of those levels in shared memory (two work vectors on the top
// small level, right-hand side + two on the others), reads the shared
// Galerkin stencils through L1/L2 and the top level's right-hand side from
// global memory, and walks the same V(2,2) sweep as the streaming passes:
//   down  z1 = w1 b/d ; z2 = z1 + w2 (b - A z1)/d ; b_c = P^T (b - A z2)
//   coarsest  x = inv b (dense, per frequency)
//   up    zc = z2 + P x_c ; z3 = zc + w2 (b - A zc)/d ; z4 = z3 + w1 (b - A z3)/d
// with __syncthreads between the half-steps.  The same operator, weights and
// transfer operators as mg.cu / mg_fine.cu, so the preconditioner (and COCG's
// iterates) do not depend on which path ran.
#include "mg.cuh"

namespace tpgpu {

namespace {

constexpr int SNT = 1024;  // threads per block (one block per frequency)

__device__ __forceinline__ cplx cmul(cplx a, cplx b) {
  return {fma(a.re, b.re, -a.im * b.im), fma(a.re, b.im, a.im * b.re)};
}
// 1/a from the hardware reciprocal estimate + one Newton step (as mg_fine.cu's
// smoothers: the V-cycle only needs a fixed D^-1, not a correctly rounded one)
__device__ __forceinline__ cplx crcp(cplx a) {
  const double x = fma(a.re, a.re, a.im * a.im);
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double d = fma(r, fma(-x, r, 1.0), r);
  return {a.re * d, -a.im * d};
}

struct Lvl {
  const double* K;
  const double* M;
  int m, n;
};

__device__ __forceinline__ cplx coefc(const Lvl& L, int dir, int i, cplx l) {
  const double k = __ldg(L.K + (size_t)dir * L.n + i), mm = __ldg(L.M + (size_t)dir * L.n + i);
  return {fma(l.re, mm, k), l.im * mm};
}

// diagonal and off-diagonal part of (lambda M + K) v at node (x, y); v in
// shared memory.  Off-diagonal part in split form sum K_d v_d + l sum M_d v_d.
__device__ __forceinline__ void stencil(const Lvl& L, int x, int y, cplx l, const cplx* v, cplx& d, cplx& off) {
  const int m = L.m, i = y * m + x;
  d = coefc(L, SC, i, l);
  cplx sk{0, 0}, sm{0, 0};
  auto add = [&](int dir, int at, cplx vv) {
    const double k = __ldg(L.K + (size_t)dir * L.n + at), mm = __ldg(L.M + (size_t)dir * L.n + at);
    sk.re = fma(k, vv.re, sk.re);
    sk.im = fma(k, vv.im, sk.im);
    sm.re = fma(mm, vv.re, sm.re);
    sm.im = fma(mm, vv.im, sm.im);
  };
  if (x + 1 < m) add(SE_, i, v[i + 1]);
  if (x > 0) add(SE_, i - 1, v[i - 1]);
  if (y + 1 < m) add(SN_, i, v[i + m]);
  if (y > 0) add(SN_, i - m, v[i - m]);
  if (x + 1 < m && y + 1 < m) add(SNE, i, v[i + m + 1]);
  if (x > 0 && y > 0) add(SNE, i - m - 1, v[i - m - 1]);
  off = sk + cmul(l, sm);
}

// z_out = z_in + w (b - A z_in) / d  (z_in == nullptr: z_out = w b / d)
__device__ __forceinline__ void jacobi(const Lvl& L, cplx l, const cplx* b_g, const cplx* b_s, const cplx* zin,
                                       cplx* zout, double w) {
  for (int i = threadIdx.x; i < L.n; i += SNT) {
    const int y = i / L.m, x = i - y * L.m;
    const cplx bi = b_g ? b_g[i] : b_s[i];
    if (!zin) {
      const cplx d = coefc(L, SC, i, l);
      zout[i] = w * cmul(bi, crcp(d));
    } else {
      cplx d, off;
      stencil(L, x, y, l, zin, d, off);
      const cplx r = bi - off - cmul(d, zin[i]);
      zout[i] = zin[i] + w * cmul(r, crcp(d));
    }
  }
}

__device__ __forceinline__ void residual(const Lvl& L, cplx l, const cplx* b_g, const cplx* b_s, const cplx* z,
                                         cplx* res) {
  for (int i = threadIdx.x; i < L.n; i += SNT) {
    const int y = i / L.m, x = i - y * L.m;
    cplx d, off;
    stencil(L, x, y, l, z, d, off);
    res[i] = (b_g ? b_g[i] : b_s[i]) - off - cmul(d, z[i]);
  }
}

// b_c = P^T res (interior fine centre (2X+1, 2Y+1) and its six neighbours)
__device__ __forceinline__ void restrict_to(int m, int mc, const cplx* res, cplx* bc) {
  for (int I = threadIdx.x; I < mc * mc; I += SNT) {
    const int Y = I / mc, X = I - Y * mc;
    const int f = (2 * Y + 1) * m + 2 * X + 1;
    const cplx side = res[f - 1] + res[f + 1] + res[f - m] + res[f + m] + res[f - m - 1] + res[f + m + 1];
    bc[I] = res[f] + 0.5 * side;
  }
}

// z += P x_c (P1 interpolation on the nested triangulation)
__device__ __forceinline__ void prolong_add(int m, int mc, const cplx* xc, cplx* z) {
  for (int i = threadIdx.x; i < m * m; i += SNT) {
    const int y = i / m, x = i - y * m;
    const int a = x + 1, b = y + 1, ah = a >> 1, bh = b >> 1;
    auto at = [&](int A, int B) -> cplx {
      return (A >= 1 && A <= mc && B >= 1 && B <= mc) ? xc[(B - 1) * mc + (A - 1)] : cplx{0, 0};
    };
    cplx v;
    if (!(a & 1) && !(b & 1)) v = at(ah, bh);
    else if (a & 1 && !(b & 1)) v = 0.5 * (at(ah, bh) + at(ah + 1, bh));
    else if (!(a & 1)) v = 0.5 * (at(ah, bh) + at(ah, bh + 1));
    else v = 0.5 * (at(ah, bh) + at(ah + 1, bh + 1));
    z[i] = z[i] + v;
  }
}

__global__ void __launch_bounds__(SNT, 1) k_small_cycle(SmallLevels sl, const cplx* __restrict__ lam,
                                                        const cplx* __restrict__ inv, const cplx* __restrict__ b0,
                                                        cplx* __restrict__ z0, const int* __restrict__ active,
                                                        double om1, double om2) {
  TP_PDL_ENTRY();
  const int bt = blockIdx.x;
  if (active && !active[bt]) return;
  extern __shared__ __align__(16) unsigned char small_smem[];
  cplx* sm = reinterpret_cast<cplx*>(small_smem);
  const int nl = sl.levels;  // levels handled, the last is the coarsest
  // shared layout: level 0: zA, zB; levels 1..nl-2: b, zA, zB; coarsest: b, x
  // sl.m[j] for a runtime j without a dynamically indexed parameter array
  auto mof = [&](int j) -> int {
    int v = 0;
#pragma unroll
    for (int k = 0; k < kMaxSmall; ++k)
      if (k == j) v = sl.m[k];
    return v;
  };
  auto lvl = [&](int j) -> Lvl { return {sl.K[j], sl.M[j], sl.m[j], sl.m[j] * sl.m[j]}; };
  auto base = [&](int j) -> cplx* {
    cplx* q = sm;
#pragma unroll
    for (int k = 0; k < kMaxSmall; ++k)
      if (k < j) q += (size_t)sl.m[k] * sl.m[k] * ((k == 0 || k == nl - 1) ? 2 : 3);
    return q;
  };
  auto bs = [&](int j) -> cplx* { return j == 0 ? nullptr : base(j); };
  auto za = [&](int j) -> cplx* { return base(j) + (j == 0 ? 0 : mof(j) * mof(j)); };
  auto zb = [&](int j) -> cplx* { return za(j) + mof(j) * mof(j); };
  const cplx l = lam[bt];
  const int n0 = sl.m[0] * sl.m[0];
  const cplx* bg = b0 + (size_t)bt * n0;
  // down (loops unrolled over the level bound: static indices into sl)
#pragma unroll
  for (int j = 0; j < kMaxSmall - 1; ++j) {
    if (j >= nl - 1) break;
    const Lvl L = lvl(j);
    const cplx* b_g = j == 0 ? bg : nullptr;
    cplx *b = bs(j), *a = za(j), *c = zb(j);
    jacobi(L, l, b_g, b, nullptr, a, om1);  // z1
    __syncthreads();
    jacobi(L, l, b_g, b, a, c, om2);  // z2
    __syncthreads();
    residual(L, l, b_g, b, c, a);
    __syncthreads();
    restrict_to(L.m, sl.m[j + 1], a, bs(j + 1));
    __syncthreads();
  }
  // coarsest: x = inv b (inv transposed: A[j * nc + i] = inv(i, j)), spread
  // over the whole block: G groups of nc threads each sum a strided share of
  // the columns (coalesced rows of A), then a fixed-order sum of the G partials
  // (scratch: level 0's first work vector, free until the up pass).  One
  // thread per row walking all nc columns left the other warps at the barrier
  // for a quarter of the kernel (ncu stall sampling).
  {
    const int nc = mof(nl - 1) * mof(nl - 1);
    const cplx* A = inv + (size_t)bt * nc * nc;
    const cplx* bc = bs(nl - 1);
    cplx* x = za(nl - 1);
    cplx* scratch = za(0);
    const int G = max(1, min(SNT / nc, n0 / nc));
    const int t = threadIdx.x, g = t / nc, i = t - g * nc;
    if (g < G) {
      cplx acc{0, 0};
      for (int k = g; k < nc; k += G) acc = acc + cmul(A[(size_t)k * nc + i], bc[k]);
      scratch[g * nc + i] = acc;
    }
    __syncthreads();
    for (int r = t; r < nc; r += SNT) {
      cplx acc = scratch[r];
      for (int q = 1; q < G; ++q) acc = acc + scratch[q * nc + r];
      x[r] = acc;
    }
    __syncthreads();
  }
  // up
#pragma unroll
  for (int j = kMaxSmall - 2; j >= 0; --j) {
    if (j > nl - 2) continue;
    const Lvl L = lvl(j);
    const cplx* b_g = j == 0 ? bg : nullptr;
    cplx *b = bs(j), *a = za(j), *c = zb(j);
    const cplx* xc = (j == nl - 2) ? za(nl - 1) : zb(j + 1);
    prolong_add(L.m, sl.m[j + 1], xc, c);  // zc = z2 + P x_c
    __syncthreads();
    jacobi(L, l, b_g, b, c, a, om2);  // z3
    __syncthreads();
    jacobi(L, l, b_g, b, a, c, om1);  // z4
    __syncthreads();
  }
  cplx* zo = z0 + (size_t)bt * n0;
  const cplx* z4 = zb(0);
  for (int i = threadIdx.x; i < n0; i += SNT) zo[i] = z4[i];
}

}  // namespace

size_t small_cycle_smem(const int* m, int levels) {
  size_t c = 0;
  for (int j = 0; j < levels; ++j) {
    const size_t n = (size_t)m[j] * m[j];
    c += (j == 0 || j == levels - 1) ? 2 * n : 3 * n;
  }
  return c * sizeof(cplx);
}

void launch_small_cycle(Problem& p, const SmallLevels& sl, const cplx* lam, const cplx* inv, const cplx* b,
                        cplx* z, const int* active, double om1, double om2, int nb) {
  const size_t sm = small_cycle_smem(sl.m, sl.levels);
  static const bool attr = [] {  // (thread-safe one-time init: the largest opt-in size)
    return cudaFuncSetAttribute(k_small_cycle, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) ==
           cudaSuccess;
  }();
  require(attr && sm <= 227 * 1024, "small-level cycle: shared memory");
  launch_pdl(k_small_cycle, dim3(nb), dim3(SNT), sm, p.cur_stream(), sl, lam, inv, b, z, active, om1, om2);
  TP_LAUNCHED(&p);
}

}  // namespace tpgpu
