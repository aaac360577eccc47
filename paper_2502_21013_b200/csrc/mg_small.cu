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
//
// Layout: every level's vectors are stored zero-padded, (m+2)^2 with the node
// (x, y) at (y+1)(m+2) + x+1, and the level's stencil is a packed copy
// (pack_small_levels) of its C, E, N, NE planes as {K, M} pairs on the same
// padded grid -- so a node's 7-point row is 7 16-byte coefficient loads and
// 7 neighbour reads with no boundary tests, and threads map to (x, y) by
// shifts (a power-of-two row pitch) instead of divisions.
#include <cooperative_groups.h>
#include <cstdlib>

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
  const double2* C;  // 4 planes of np padded {K, M}
  int m, w, np;      // nodes per side, padded pitch m+2, padded size
  int sh;            // log2 of the power-of-two thread pitch >= m
};

#ifndef TPGPU_SMALL_UNROLL
#define TPGPU_SMALL_UNROLL 1
#endif
#define TP_SMALL_PRAGMA(x) _Pragma(#x)
#define TP_SMALL_UNROLL_N(n) TP_SMALL_PRAGMA(unroll n)
#define TP_SMALL_UNROLL TP_SMALL_UNROLL_N(TPGPU_SMALL_UNROLL)
// threads of the block over the level's nodes: x = tid & (2^sh - 1), rows
// stepping by SNT >> sh
#define FOR_ROWS(L, YLO, YHI, ...)                                                  \
  {                                                                                 \
    const int x_ = threadIdx.x & ((1 << (L).sh) - 1);                               \
    if (x_ < (L).m)                                                                 \
      TP_SMALL_UNROLL                                                               \
      for (int y_ = (YLO) + (threadIdx.x >> (L).sh); y_ < (YHI); y_ += SNT >> (L).sh) { \
        const int x = x_, y = y_;                                                   \
        const int P = (y + 1) * (L).w + x + 1;                                      \
        __VA_ARGS__                                                                 \
      }                                                                             \
  }
#define FOR_NODES(L, ...) FOR_ROWS(L, 0, (L).m, __VA_ARGS__)

__device__ __forceinline__ cplx diag_of(double2 c, cplx l) { return {fma(l.re, c.y, c.x), l.im * c.y}; }

// diagonal and off-diagonal part of (lambda M + K) v at padded node P; v in
// shared memory (zero border).  Off-diagonal in split form sum K_d v_d + l sum M_d v_d.
__device__ __forceinline__ void stencil(const Lvl& L, int P, cplx l, const cplx* v, cplx& d, cplx& off) {
  const double2* C = L.C;
  const int w = L.w, np = L.np;
  const double2 cc = __ldg(C + P);
  const double2 kE = __ldg(C + np + P), kW = __ldg(C + np + P - 1);
  const double2 kN = __ldg(C + 2 * np + P), kS = __ldg(C + 2 * np + P - w);
  const double2 kNE = __ldg(C + 3 * np + P), kSW = __ldg(C + 3 * np + P - w - 1);
  const cplx vE = v[P + 1], vW = v[P - 1], vN = v[P + w], vS = v[P - w], vNE = v[P + w + 1], vSW = v[P - w - 1];
  cplx sk, sm;
  sk.re = kE.x * vE.re + kW.x * vW.re + kN.x * vN.re + kS.x * vS.re + kNE.x * vNE.re + kSW.x * vSW.re;
  sk.im = kE.x * vE.im + kW.x * vW.im + kN.x * vN.im + kS.x * vS.im + kNE.x * vNE.im + kSW.x * vSW.im;
  sm.re = kE.y * vE.re + kW.y * vW.re + kN.y * vN.re + kS.y * vS.re + kNE.y * vNE.re + kSW.y * vSW.re;
  sm.im = kE.y * vE.im + kW.y * vW.im + kN.y * vN.im + kS.y * vS.im + kNE.y * vNE.im + kSW.y * vSW.im;
  d = diag_of(cc, l);
  off = sk + cmul(l, sm);
}

// z_out = z_in + w (b - A z_in) / d  (z_in == nullptr: z_out = w b / d);
// b from global (unpadded, b_g) on the top level, else from shared (padded)
__device__ __forceinline__ void jacobi(const Lvl& L, cplx l, const cplx* b_g, const cplx* b_s, const cplx* zin,
                                       cplx* zout, double w, int ylo = 0, int yhi = 1 << 30) {
  FOR_ROWS(L, ylo, min(yhi, L.m), {
    const cplx bi = b_g ? b_g[y * L.m + x] : b_s[P];
    if (!zin) {
      const cplx d = diag_of(__ldg(L.C + P), l);
      zout[P] = w * cmul(bi, crcp(d));
    } else {
      cplx d, off;
      stencil(L, P, l, zin, d, off);
      const cplx r = bi - off - cmul(d, zin[P]);
      zout[P] = zin[P] + w * cmul(r, crcp(d));
    }
  })
}

__device__ __forceinline__ void residual(const Lvl& L, cplx l, const cplx* b_g, const cplx* b_s, const cplx* z,
                                         cplx* res, int ylo = 0, int yhi = 1 << 30) {
  FOR_ROWS(L, ylo, min(yhi, L.m), {
    cplx d, off;
    stencil(L, P, l, z, d, off);
    res[P] = (b_g ? b_g[y * L.m + x] : b_s[P]) - off - cmul(d, z[P]);
  })
}

// b_c = P^T res (interior fine centre (2X+1, 2Y+1) and its six neighbours)
__device__ __forceinline__ void restrict_to(const Lvl& F, const Lvl& Cc, const cplx* res, cplx* bc, int ylo = 0,
                                            int yhi = 1 << 30, cplx* bc2 = nullptr) {
  const int w = F.w;
  FOR_ROWS(Cc, ylo, min(yhi, Cc.m), {
    const int f = (2 * y + 2) * w + 2 * x + 2;
    const cplx side = res[f - 1] + res[f + 1] + res[f - w] + res[f + w] + res[f - w - 1] + res[f + w + 1];
    const cplx v = res[f] + 0.5 * side;
    bc[P] = v;
    if (bc2) bc2[P] = v;  // the cluster partner's copy
  })
}

// z += P x_c (P1 interpolation on the nested triangulation); coarse vertex
// (A, B), A, B in [0, mc+1], sits at padded index B (mc+2) + A (zero border)
__device__ __forceinline__ void prolong_add(const Lvl& F, const Lvl& Cc, const cplx* xc, cplx* z, int ylo = 0,
                                            int yhi = 1 << 30) {
  const int wc = Cc.w;
  FOR_ROWS(F, ylo, min(yhi, F.m), {
    const int a = x + 1, b = y + 1, ah = a >> 1, bh = b >> 1;
    const int c0 = bh * wc + ah;
    cplx v;
    if (!(a & 1) && !(b & 1)) v = xc[c0];
    else if (a & 1 && !(b & 1)) v = 0.5 * (xc[c0] + xc[c0 + 1]);
    else if (!(a & 1)) v = 0.5 * (xc[c0] + xc[c0 + wc]);
    else v = 0.5 * (xc[c0] + xc[c0 + wc + 1]);
    z[P] = z[P] + v;
  })
}

__device__ __forceinline__ int pitch_shift(int m) { return m <= 1 ? 0 : 32 - __clz(m - 1); }

// CL = 2: a cluster of two blocks per frequency splits the top small level's
// rows between them (the level carries ~60 % of the kernel's time): after each
// half-step a block stores its boundary row into its partner's copy of the
// vector (distributed shared memory) and the pair meets at a cluster barrier;
// the restriction's coarse rows go to both blocks, which then run the lower
// levels and the coarsest solve redundantly (identical arithmetic).
template <int CL>
__global__ void __launch_bounds__(SNT, 1) k_small_cycle(SmallLevels sl, const cplx* __restrict__ lam,
                                                        const cplx* __restrict__ inv, const cplx* __restrict__ b0,
                                                        cplx* __restrict__ z0, const int* __restrict__ active,
                                                        double om1, double om2, int smem_c16) {
  TP_PDL_ENTRY();
  const int bt = blockIdx.x / CL;
  if (active && !active[bt]) return;
  extern __shared__ __align__(16) unsigned char small_smem[];
  cplx* sm = reinterpret_cast<cplx*>(small_smem);
  // zero borders: clear the whole work area once
  for (int k = threadIdx.x; k < smem_c16; k += SNT) sm[k] = cplx{0, 0};
  const int nl = sl.levels;  // levels handled, the last is the coarsest
  // shared layout (padded): level 0: zA, zB; levels 1..nl-2: b, zA, zB; coarsest: b, x
  auto mof = [&](int j) -> int {  // sl.m[j] for a runtime j (no dynamically indexed parameter array)
    int v = 0;
#pragma unroll
    for (int k = 0; k < kMaxSmall; ++k)
      if (k == j) v = sl.m[k];
    return v;
  };
  auto npad = [&](int j) -> int { return (mof(j) + 2) * (mof(j) + 2); };
  auto lvl = [&](int j) -> Lvl {
    const int m = sl.m[j];
    return {sl.KM[j], m, m + 2, (m + 2) * (m + 2), pitch_shift(m)};
  };
  auto base = [&](int j) -> cplx* {
    cplx* q = sm;
#pragma unroll
    for (int k = 0; k < kMaxSmall; ++k)
      if (k < j) q += (size_t)(sl.m[k] + 2) * (sl.m[k] + 2) * ((k == 0 || k == nl - 1) ? 2 : 3);
    return q;
  };
  auto bs = [&](int j) -> cplx* { return j == 0 ? nullptr : base(j); };
  auto za = [&](int j) -> cplx* { return base(j) + (j == 0 ? 0 : npad(j)); };
  auto zb = [&](int j) -> cplx* { return za(j) + npad(j); };
  const cplx l = lam[bt];
  const int m0 = sl.m[0], n0 = m0 * m0;
  const cplx* bg = b0 + (size_t)bt * n0;
  // top-level rows of this block: [ya, yb); coarse rows of its restriction [Ya, Yb)
  int rank = 0, ya = 0, yb = m0, Ya = 0, Yb = 1 << 30;
  const int ymid = (m0 + 1) / 2;
  if constexpr (CL == 2) {
    rank = (int)cooperative_groups::this_cluster().block_rank();
    ya = rank == 0 ? 0 : ymid;
    yb = rank == 0 ? ymid : m0;
    Ya = rank == 0 ? 0 : ymid / 2;
    Yb = rank == 0 ? ymid / 2 : (1 << 30);
  }
  // the partner's copy of a vector of this block's shared memory
  auto remote = [&](cplx* v) -> cplx* {
    if constexpr (CL == 2) return cooperative_groups::this_cluster().map_shared_rank(v, rank ^ 1);
    else return nullptr;
  };
  // after a top-level half-step: boundary row to the partner, then both meet
  auto exchange = [&](cplx* v) {
    if constexpr (CL == 2) {
      const int row = rank == 0 ? yb - 1 : ya, w = m0 + 2;
      __syncthreads();  // the row was written by other threads of this block
      cplx* r = remote(v);
      for (int x = threadIdx.x; x < m0; x += SNT) r[(row + 1) * w + x + 1] = v[(row + 1) * w + x + 1];
      cooperative_groups::this_cluster().sync();
    } else {
      __syncthreads();
    }
  };
  if constexpr (CL == 2) cooperative_groups::this_cluster().sync();  // both cleared before remote stores
  else __syncthreads();
  // down (loops unrolled over the level bound: static indices into sl)
#pragma unroll
  for (int j = 0; j < kMaxSmall - 1; ++j) {
    if (j >= nl - 1) break;
    const Lvl L = lvl(j);
    const cplx* b_g = j == 0 ? bg : nullptr;
    cplx *b = bs(j), *a = za(j), *c = zb(j);
    if (j == 0 && CL == 2) {
      jacobi(L, l, b_g, b, nullptr, a, om1, ya, yb);  // z1
      exchange(a);
      jacobi(L, l, b_g, b, a, c, om2, ya, yb);  // z2
      exchange(c);
      residual(L, l, b_g, b, c, a, ya, yb);
      exchange(a);
      restrict_to(L, lvl(1), a, bs(1), Ya, Yb, remote(bs(1)));
      if constexpr (CL == 2) cooperative_groups::this_cluster().sync();
    } else {
      jacobi(L, l, b_g, b, nullptr, a, om1);  // z1
      __syncthreads();
      jacobi(L, l, b_g, b, a, c, om2);  // z2
      __syncthreads();
      residual(L, l, b_g, b, c, a);
      __syncthreads();
      restrict_to(L, lvl(j + 1), a, bs(j + 1));
      __syncthreads();
    }
  }
  // coarsest: x = inv b (inv transposed: A[j * nc + i] = inv(i, j)), spread
  // over the whole block: G groups of nc threads each sum a strided share of
  // the columns (coalesced rows of A), then a fixed-order sum of the G partials
  // (scratch: level 0's first work vector, free until the up pass).  One
  // thread per row walking all nc columns left the other warps at the barrier
  // for a quarter of the kernel (ncu stall sampling).
  {
    const int mc = mof(nl - 1), nc = mc * mc, wc = mc + 2;
    const cplx* A = inv + (size_t)bt * nc * nc;
    const cplx* bc = bs(nl - 1);
    cplx* x = za(nl - 1);
    cplx* scratch = za(0);
    const int G = max(1, min(SNT / nc, npad(0) / nc));
    const int t = threadIdx.x, g = t / nc, i = t - g * nc;
    if (g < G) {
      cplx acc{0, 0};
      for (int k = g; k < nc; k += G) {
        const int ky = k / mc, kx = k - ky * mc;
        acc = acc + cmul(A[(size_t)k * nc + i], bc[(ky + 1) * wc + kx + 1]);
      }
      scratch[g * nc + i] = acc;
    }
    __syncthreads();
    for (int r = t; r < nc; r += SNT) {
      cplx acc = scratch[r];
      for (int q = 1; q < G; ++q) acc = acc + scratch[q * nc + r];
      const int ry = r / mc, rx = r - ry * mc;
      x[(ry + 1) * wc + rx + 1] = acc;
    }
    __syncthreads();
    // level 0's first work vector is zero-bordered again before its next use
    // as a padded vector (the up pass writes its interior only)
    for (int k = t; k < G * nc; k += SNT) scratch[k] = cplx{0, 0};
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
    if (j == 0 && CL == 2) {
      prolong_add(L, lvl(1), xc, c, ya, yb);  // zc = z2 + P x_c
      exchange(c);
      jacobi(L, l, b_g, b, c, a, om2, ya, yb);  // z3
      exchange(a);
      jacobi(L, l, b_g, b, a, c, om1, ya, yb);  // z4
      __syncthreads();
    } else {
      prolong_add(L, lvl(j + 1), xc, c);  // zc = z2 + P x_c
      __syncthreads();
      jacobi(L, l, b_g, b, c, a, om2);  // z3
      __syncthreads();
      jacobi(L, l, b_g, b, a, c, om1);  // z4
      __syncthreads();
    }
  }
  cplx* zo = z0 + (size_t)bt * n0;
  const cplx* z4 = zb(0);
  const Lvl L0 = lvl(0);
  FOR_ROWS(L0, ya, yb, { zo[y * L0.m + x] = z4[P]; })
  // the partner may still read this block's shared memory (remote stores are
  // done, but keep both alive until the pair is through)
  if constexpr (CL == 2) cooperative_groups::this_cluster().sync();
}

// packed, zero-padded {K, M} planes C, E, N, NE of one level
__global__ void k_pack_small(const double* __restrict__ K, const double* __restrict__ M, int m,
                             double2* __restrict__ out) {
  const int w = m + 2, np = w * w, n = m * m;
  const int dirs[4] = {SC, SE_, SN_, SNE};
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < 4 * np; k += gridDim.x * blockDim.x) {
    const int q = k / np, P = k - q * np;
    const int py = P / w, px = P - py * w;
    const int x = px - 1, y = py - 1;
    double2 v{0.0, 0.0};
    if (x >= 0 && x < m && y >= 0 && y < m) {
      const size_t i = (size_t)dirs[q] * n + (size_t)y * m + x;
      v = {K[i], M[i]};
    }
    out[k] = v;
  }
}

}  // namespace

size_t small_cycle_smem(const int* m, int levels) {
  size_t c = 0;
  for (int j = 0; j < levels; ++j) {
    const size_t n = (size_t)(m[j] + 2) * (m[j] + 2);
    c += (j == 0 || j == levels - 1) ? 2 * n : 3 * n;
  }
  return c * sizeof(cplx);
}

size_t small_pack_size(const int* m, int levels) {
  size_t c = 0;
  for (int j = 0; j < levels; ++j) c += (size_t)8 * (m[j] + 2) * (m[j] + 2);
  return c;
}

void pack_small_levels(Problem& p, SmallLevels& sl, double* buf) {
  for (int j = 0; j < sl.levels; ++j) {
    const int m = sl.m[j], np = (m + 2) * (m + 2);
    double2* out = reinterpret_cast<double2*>(buf);
    k_pack_small<<<(4 * np + 255) / 256, 256, 0, p.cur_stream()>>>(sl.K[j], sl.M[j], m, out);
    TP_LAUNCHED(&p);
    sl.KM[j] = out;
    buf += (size_t)8 * np;
  }
}

void launch_small_cycle(Problem& p, const SmallLevels& sl, const cplx* lam, const cplx* inv, const cplx* b,
                        cplx* z, const int* active, double om1, double om2, int nb, int n_active) {
  const size_t sm = small_cycle_smem(sl.m, sl.levels);
  static const bool attr = [] {  // (thread-safe one-time init: the largest opt-in size)
    return cudaFuncSetAttribute(k_small_cycle<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) ==
               cudaSuccess &&
           cudaFuncSetAttribute(k_small_cycle<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) ==
               cudaSuccess;
  }();
  require(attr && sm <= 227 * 1024, "small-level cycle: shared memory");
  require(sl.KM[0] != nullptr, "small-level cycle: stencils not packed");
  // two-block clusters when few frequencies are active (the tail of a solve:
  // half the latency; with many active frequencies the second SM per frequency
  // costs the concurrent groups more than it saves -- cfg 1 3.38 vs 3.33 ms
  // always-on).  TPGPU_SMALL_CLUSTER = the largest active count that uses them.
  static const int cl_max = std::getenv("TPGPU_SMALL_CLUSTER") ? std::atoi(std::getenv("TPGPU_SMALL_CLUSTER")) : 0;
  if (n_active <= cl_max && sl.levels >= 2 && sl.m[0] >= 15) {
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cudaLaunchConfig_t c = {};
    c.gridDim = dim3(2 * nb);
    c.blockDim = dim3(SNT);
    c.dynamicSmemBytes = sm;
    c.stream = p.cur_stream();
    c.attrs = at;
    c.numAttrs = 2;
    TP_CUDA(cudaLaunchKernelEx(&c, k_small_cycle<2>, sl, lam, inv, b, z, active, om1, om2, (int)(sm / sizeof(cplx))));
  } else {
    launch_pdl(k_small_cycle<1>, dim3(nb), dim3(SNT), sm, p.cur_stream(), sl, lam, inv, b, z, active, om1, om2,
               (int)(sm / sizeof(cplx)));
  }
  TP_LAUNCHED(&p);
}

}  // namespace tpgpu
