// Batched multigrid-preconditioned CG/COCG -- see mg.cuh.
//
// Kernel layout: a block owns a 32x8 tile of nodes of one level and walks the
// active batches (frequencies or slices) of its batch group.  Vector tiles
// (+1 halo) are staged in shared memory (16-byte complex accesses) and the
// next batch's tile is prefetched into registers while the current one is
// computed.  Stencil families:
//   FAM 1  fine level, frequency mode: K_hat is 5-point and M is the lumped
//          diagonal, so a thread keeps its 5 + 1 real coefficients in
//          registers and the off-diagonal products are real x complex;
//   FAM 0  coarse levels, frequency mode: Galerkin 7-point K and M shared by
//          all frequencies, staged once per block in shared memory;
//   FAM 2  slice mode (Newton): per-batch 7-point J from global memory.
// Restriction forms the fine residual tile in shared memory and gathers P^T
// from it; prolongation interpolates the coarse correction while staging the
// tile.  32-bit node indices within a level, 64-bit batch offsets.
//
// Per fine node and batch (16 B complex) one Krylov iteration streams:
// apply+dot (read z, p; write p, q), update (read x, p, r, q; write x, r, z),
// pre-smooth (read z, r; write z), residual+restrict (read z, r), prolong +
// smooth (read z, r; write z), smooth+dot (read z, r; write z) = 22 vector
// streams on the fine level, ~1/3 of that again on the coarse levels.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "mg.cuh"

namespace tpgpu {

namespace {

constexpr int TX = 32, TY = 8, NT = TX * TY;
constexpr int HX = TX + 2, HY = TY + 2, HN = HX * HY;  // halo tile: 340 values
constexpr int RX = TX + 3, RY = TY + 3, RN = RX * RY;  // restriction tile: 385 values

template <int MODE>
using TT = typename std::conditional<MODE == 0, cplx, double>::type;

__device__ __forceinline__ cplx mul(cplx a, cplx b) {
  return {fma(a.re, b.re, -a.im * b.im), fma(a.re, b.im, a.im * b.re)};
}
__device__ __forceinline__ double mul(double a, double b) { return a * b; }
__device__ __forceinline__ cplx zero_of(cplx) { return {0, 0}; }
__device__ __forceinline__ double zero_of(double) { return 0; }
__device__ __forceinline__ void add_dot(double (&v)[2], cplx a, cplx b) {
  const cplx t = mul(a, b);
  v[0] += t.re;
  v[1] += t.im;
}
__device__ __forceinline__ void add_dot(double (&v)[2], double a, double b) { v[0] += a * b; }
__device__ __forceinline__ cplx inv_of(cplx a) {
  const double d = 1.0 / fma(a.re, a.re, a.im * a.im);
  return {a.re * d, -a.im * d};
}
__device__ __forceinline__ double inv_of(double a) { return 1.0 / a; }
// smoother D^-1: hardware reciprocal estimate + one Newton step (~46 bits, no
// special-case path; the V-cycle only needs a fixed diagonal scaling)
__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return fma(r, fma(-x, r, 1.0), r);
}
__device__ __forceinline__ cplx sinv(cplx a) {
  const double d = fast_rcp(fma(a.re, a.re, a.im * a.im));
  return {a.re * d, -a.im * d};
}
__device__ __forceinline__ double sinv(double a) { return fast_rcp(a); }
__device__ __forceinline__ cplx axpy_r(double k, cplx v, cplx acc) { return {fma(k, v.re, acc.re), fma(k, v.im, acc.im)}; }

// Level operator.  MODE 0: lambda_b M + K with shared stencils; MODE 1:
// per-batch stencil J_b.
template <int MODE>
struct Op;
template <>
struct Op<0> {
  const double* K;
  const double* M;
  const cplx* lam;
  int n, m;
};
template <>
struct Op<1> {
  const double* J;
  int n, m;
};

// ---- stencil coefficient families
struct StageF {
  double v[14][NT];
};

struct CoefStaged {  // FAM 0
  const StageF* s;
  cplx l;
  int tid;
  __device__ __forceinline__ cplx c(int d) const {
    const double mm = s->v[7 + d][tid];
    return {fma(l.re, mm, s->v[d][tid]), l.im * mm};
  }
  __device__ __forceinline__ cplx diag() const { return c(0); }
};

struct FineRegs {  // FAM 1 per-thread data
  double k0, kw, ke, ks, kn, m0;
};

struct CoefFine {
  FineRegs r;
  cplx l;
  __device__ __forceinline__ cplx diag() const { return {fma(l.re, r.m0, r.k0), l.im * r.m0}; }
};

struct CoefSlice {  // FAM 2
  const double* J;
  int n, i, m;
  __device__ __forceinline__ double c(int d) const { return __ldg(J + (size_t)d * n + i); }
  // plane d at node j (clamped into the grid: off-grid neighbours multiply zero halo values)
  __device__ __forceinline__ double c_at(int d, int j) const { return __ldg(J + (size_t)d * n + max(j, 0)); }
  __device__ __forceinline__ double diag() const { return c(0); }
};

template <class T, int W>
__device__ __forceinline__ T apply_tile(const CoefStaged& a, const T (*s)[W], int lx, int ly) {
  T acc = mul(a.c(0), s[ly][lx]);
  acc = acc + mul(a.c(1), s[ly][lx - 1]);
  acc = acc + mul(a.c(2), s[ly][lx + 1]);
  acc = acc + mul(a.c(3), s[ly - 1][lx]);
  acc = acc + mul(a.c(4), s[ly + 1][lx]);
  acc = acc + mul(a.c(5), s[ly - 1][lx - 1]);
  acc = acc + mul(a.c(6), s[ly + 1][lx + 1]);
  return acc;
}
template <int W>
__device__ __forceinline__ cplx apply_tile(const CoefFine& a, const cplx (*s)[W], int lx, int ly) {
  cplx acc = mul(a.diag(), s[ly][lx]);
  acc = axpy_r(a.r.kw, s[ly][lx - 1], acc);
  acc = axpy_r(a.r.ke, s[ly][lx + 1], acc);
  acc = axpy_r(a.r.ks, s[ly - 1][lx], acc);
  acc = axpy_r(a.r.kn, s[ly + 1][lx], acc);
  return acc;
}
// The element-assembled Jacobian is symmetric: W(i) = E(i-1), S(i) = N(i-m),
// SW(i) = NE(i-m-1), so four of its seven planes are read (32 instead of 56
// bytes per node and slice; neighbouring threads share the sectors)
template <class T, int W>
__device__ __forceinline__ T apply_tile(const CoefSlice& a, const T (*s)[W], int lx, int ly) {
  T acc = a.c(SC) * s[ly][lx];
  acc = acc + a.c_at(SE_, a.i - 1) * s[ly][lx - 1];
  acc = acc + a.c(SE_) * s[ly][lx + 1];
  acc = acc + a.c_at(SN_, a.i - a.m) * s[ly - 1][lx];
  acc = acc + a.c(SN_) * s[ly + 1][lx];
  acc = acc + a.c_at(SNE, a.i - a.m - 1) * s[ly - 1][lx - 1];
  acc = acc + a.c(SNE) * s[ly + 1][lx + 1];
  return acc;
}

// Per-kernel coefficient context
template <int MODE, int FAM>
struct Ctx;
template <>
struct Ctx<0, 0> {
  StageF* st;
  __device__ void init(const Op<0>& op, int i, bool in, int tid) {
#pragma unroll
    for (int d = 0; d < 7; ++d) {
      st->v[d][tid] = in ? __ldg(op.K + (size_t)d * op.n + i) : 0.0;
      st->v[7 + d][tid] = in ? __ldg(op.M + (size_t)d * op.n + i) : 0.0;
    }
  }
  __device__ CoefStaged at(const Op<0>& op, int b, int, int tid) const { return {st, op.lam[b], tid}; }
};
template <>
struct Ctx<0, 1> {
  FineRegs r;
  __device__ void init(const Op<0>& op, int i, bool in, int) {
    if (in) {
      const size_t n = op.n;
      r = {__ldg(op.K + i), __ldg(op.K + n + i), __ldg(op.K + 2 * n + i), __ldg(op.K + 3 * n + i),
           __ldg(op.K + 4 * n + i), __ldg(op.M + i)};
    } else {
      r = {1, 0, 0, 0, 0, 0};
    }
  }
  __device__ CoefFine at(const Op<0>& op, int b, int, int) const { return {r, op.lam[b]}; }
};
template <>
struct Ctx<1, 2> {
  __device__ void init(const Op<1>&, int, bool, int) {}
  __device__ CoefSlice at(const Op<1>& op, int b, int i, int) const {
    return {op.J + (size_t)b * 7 * op.n, op.n, i, op.m};
  }
};

// coefficients of an arbitrary node (restriction extras): full 7-point
template <int MODE>
__device__ __forceinline__ void coef_global(const Op<MODE>& op, int b, int i, TT<MODE> a[7]);
template <>
__device__ __forceinline__ void coef_global<0>(const Op<0>& op, int b, int i, cplx a[7]) {
  const cplx l = op.lam[b];
  for (int d = 0; d < 7; ++d) {
    const double mm = __ldg(op.M + (size_t)d * op.n + i);
    a[d] = cplx{fma(l.re, mm, __ldg(op.K + (size_t)d * op.n + i)), l.im * mm};
  }
}
template <>
__device__ __forceinline__ void coef_global<1>(const Op<1>& op, int b, int i, double a[7]) {
  for (int d = 0; d < 7; ++d) a[d] = __ldg(op.J + (size_t)b * 7 * op.n + (size_t)d * op.n + i);
}

template <int MODE>
__device__ __forceinline__ TT<MODE> diag_global(const Op<MODE>& op, int b, int i);
template <>
__device__ __forceinline__ cplx diag_global<0>(const Op<0>& op, int b, int i) {
  const cplx l = op.lam[b];
  const double mm = __ldg(op.M + i);
  return {fma(l.re, mm, __ldg(op.K + i)), l.im * mm};
}
template <>
__device__ __forceinline__ double diag_global<1>(const Op<1>& op, int b, int i) {
  return __ldg(op.J + (size_t)b * 7 * op.n + i);
}

// Block-wide reduction of one batch's pair into part[(b*tiles + tile)*2 + c].
__device__ __forceinline__ void block_pair(double v0, double v1, double* __restrict__ part, int b) {
  __shared__ double sh[2][NT / 32];
  const int tid = threadIdx.y * TX + threadIdx.x;
  for (int o = 16; o > 0; o >>= 1) {
    v0 += __shfl_down_sync(0xffffffffu, v0, o);
    v1 += __shfl_down_sync(0xffffffffu, v1, o);
  }
  if ((tid & 31) == 0) {
    sh[0][tid >> 5] = v0;
    sh[1][tid >> 5] = v1;
  }
  __syncthreads();
  if (tid == 0) {
    double a = 0, c = 0;
    for (int w = 0; w < NT / 32; ++w) {
      a += sh[0][w];
      c += sh[1][w];
    }
    const size_t tiles = (size_t)gridDim.x * gridDim.y;
    const size_t tile = (size_t)blockIdx.y * gridDim.x + blockIdx.x;
    part[((size_t)b * tiles + tile) * 2] = a;
    part[((size_t)b * tiles + tile) * 2 + 1] = c;
  }
}

// fine node (fx, fy) -> coarse parents (mc per side), P1 weights.
__device__ __forceinline__ int parents(int fx, int fy, int mc, int* cx, int* cy, double* w) {
  const int a = fx + 1, b = fy + 1;  // vertex coords on the fine lattice
  int np = 0;
  auto add = [&](int A, int B, double ww) {
    if (A >= 1 && A <= mc && B >= 1 && B <= mc) {
      cx[np] = A - 1;
      cy[np] = B - 1;
      w[np] = ww;
      ++np;
    }
  };
  const int ah = a >> 1, bh = b >> 1;
  const bool ao = a & 1, bo = b & 1;
  if (!ao && !bo) add(ah, bh, 1.0);
  else if (ao && !bo) { add(ah, bh, 0.5); add(ah + 1, bh, 0.5); }
  else if (!ao && bo) { add(ah, bh, 0.5); add(ah, bh + 1, 0.5); }
  else { add(ah, bh, 0.5); add(ah + 1, bh + 1, 0.5); }
  return np;
}

// next active batch of this block's group after `b` (uniform), or -1
__device__ __forceinline__ int next_active(const int* __restrict__ active, int b, int nb, int BB) {
  const int end = min(nb, (int)(blockIdx.z + 1) * BB);
  for (int c = b + 1; c < end; ++c)
    if (!active || active[c]) return c;
  return -1;
}

#define TILE_PROLOGUE                                                 \
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;   \
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;               \
  const int x = x0 + tx, y = y0 + ty;                                 \
  const int m = op.m, n = op.n;                                       \
  const bool in = (x < m) && (y < m);                                 \
  const int i = in ? y * m + x : 0;                                   \
  (void)tid;

// Two halo elements per thread (k = tid, tid + NT) of a tile of width W and
// count HNW, origin (x0-1, y0-1).
template <int W, int HNW>
struct Halo {
  int ia, ib;  // linear node index, -1 outside the domain or tile
  __device__ __forceinline__ void init(int tid, int x0, int y0, int m) {
    ia = idx(tid, x0, y0, m);
    ib = (tid + NT < HNW) ? idx(tid + NT, x0, y0, m) : -1;
  }
  __device__ __forceinline__ static int idx(int k, int x0, int y0, int m) {
    const int ly = k / W, lx = k - ly * W;
    const int xx = x0 - 1 + lx, yy = y0 - 1 + ly;
    return (xx >= 0 && xx < m && yy >= 0 && yy < m) ? yy * m + xx : -1;
  }
  template <class T>
  __device__ __forceinline__ static void store(T (*s)[W], int k, T v) {
    const int ly = k / W;
    s[ly][k - ly * W] = v;
  }
};

// r = b - A x (warm) or r = b, x = 0 (cold); partials (||b||^2, ||r||^2).
template <int MODE, int FAM>
__global__ void __launch_bounds__(NT, 4) k_init(Op<MODE> op, const TT<MODE>* __restrict__ bv,
                                                TT<MODE>* __restrict__ x_, TT<MODE>* __restrict__ r,
                                                int nb, int BB, int warm, double* __restrict__ part) {
  using T = TT<MODE>;
  __shared__ T s[HY][HX];
  __shared__ StageF st_[FAM == 0 ? 1 : 0 + 1];
  TILE_PROLOGUE
  Ctx<MODE, FAM> cx;
  if constexpr (FAM == 0) cx.st = st_;
  if (warm) cx.init(op, i, in, tid);
  Halo<HX, HN> h;
  h.init(tid, x0, y0, m);
  for (int b = next_active(nullptr, blockIdx.z * BB - 1, nb, BB); b >= 0; b = next_active(nullptr, b, nb, BB)) {
    const size_t o = (size_t)b * n;
    if (warm) {
      Halo<HX, HN>::store(s, tid, h.ia >= 0 ? x_[o + h.ia] : zero_of(T{}));
      if (tid + NT < HN) Halo<HX, HN>::store(s, tid + NT, h.ib >= 0 ? x_[o + h.ib] : zero_of(T{}));
    }
    __syncthreads();
    double v0 = 0, v1 = 0;
    if (in) {
      const T bi = bv[o + i];
      T ri = bi;
      if (warm) ri = bi - apply_tile(cx.at(op, b, i, tid), s, tx + 1, ty + 1);
      else x_[o + i] = zero_of(bi);
      r[o + i] = ri;
      v0 = norm2(bi);
      v1 = norm2(ri);
    }
    block_pair(v0, v1, part, b);
    __syncthreads();
  }
}

template <int MODE>
__global__ void __launch_bounds__(NT, 4) k_zero_flagged(Op<MODE> op, TT<MODE>* __restrict__ x_, int nb,
                                                        int BB, const int* __restrict__ zero) {
  TILE_PROLOGUE
  if (!in) return;
  for (int k = 0; k < BB; ++k) {
    const int b = blockIdx.z * BB + k;
    if (b >= nb) break;
    if (zero[b]) x_[(size_t)b * n + i] = zero_of(x_[0]);
  }
}

// p_out = first ? z : z + beta p_in ;  q = A p_out ; partial p^T q
template <int MODE, int FAM>
__global__ void __launch_bounds__(NT, 4) k_apply_dot(Op<MODE> op, const TT<MODE>* __restrict__ z,
                                                     const TT<MODE>* __restrict__ pin,
                                                     TT<MODE>* __restrict__ pout, TT<MODE>* __restrict__ q,
                                                     const TT<MODE>* __restrict__ beta,
                                                     const int* __restrict__ active, int first, int nb,
                                                     int BB, double* __restrict__ part,
                                                     TT<MODE>* __restrict__ xs, const TT<MODE>* __restrict__ xa) {
  using T = TT<MODE>;
  __shared__ T s[HY][HX];
  __shared__ StageF st_[FAM == 0 ? 1 : 0 + 1];
  TILE_PROLOGUE
  // fused solution update of the previous iteration: x += alpha_prev p_prev
  // (every batch with a pending coefficient, active or just converged)
  if (xa && in && !first)
    for (int k = 0; k < BB; ++k) {
      const int b = blockIdx.z * BB + k;
      if (b >= nb) break;
      const T al = xa[b];
      if (norm2(al) == 0.0) continue;
      const size_t j = (size_t)b * n + i;
      xs[j] = xs[j] + mul(al, pin[j]);
    }
  Ctx<MODE, FAM> cx;
  if constexpr (FAM == 0) cx.st = st_;
  cx.init(op, i, in, tid);
  Halo<HX, HN> h;
  h.init(tid, x0, y0, m);
  const bool has1 = tid + NT < HN;
  T z0 = zero_of(T{}), p0 = zero_of(T{}), z1 = zero_of(T{}), p1 = zero_of(T{});
  auto fetch = [&](int b) {
    const size_t o = (size_t)b * n;
    if (h.ia >= 0) { z0 = z[o + h.ia]; if (!first) p0 = pin[o + h.ia]; }
    if (h.ib >= 0) { z1 = z[o + h.ib]; if (!first) p1 = pin[o + h.ib]; }
  };
  int b = next_active(active, blockIdx.z * BB - 1, nb, BB);
  if (b >= 0) fetch(b);
  while (b >= 0) {
    const int bn = next_active(active, b, nb, BB);
    const T bt = first ? zero_of(T{}) : beta[b];
    Halo<HX, HN>::store(s, tid, h.ia >= 0 ? (first ? z0 : z0 + mul(bt, p0)) : zero_of(T{}));
    if (has1) Halo<HX, HN>::store(s, tid + NT, h.ib >= 0 ? (first ? z1 : z1 + mul(bt, p1)) : zero_of(T{}));
    __syncthreads();
    if (bn >= 0) fetch(bn);
    double v[2] = {0, 0};
    if (in) {
      const size_t o = (size_t)b * n;
      const T pi = s[ty + 1][tx + 1];
      const T qi = apply_tile(cx.at(op, b, i, tid), s, tx + 1, ty + 1);
      pout[o + i] = pi;
      q[o + i] = qi;
      add_dot(v, pi, qi);
    }
    block_pair(v[0], v[1], part, b);
    __syncthreads();
    b = bn;
  }
}

// x += alpha p ; r -= alpha q ; partial ||r||^2 ; z = omega r / a_C
template <int MODE>
__global__ void __launch_bounds__(NT, 4) k_update(Op<MODE> op, TT<MODE>* __restrict__ x_,
                                                  TT<MODE>* __restrict__ r, const TT<MODE>* __restrict__ p,
                                                  const TT<MODE>* __restrict__ q,
                                                  const TT<MODE>* __restrict__ alpha,
                                                  const int* __restrict__ active, double omega,
                                                  TT<MODE>* __restrict__ z, int nb, int BB,
                                                  double* __restrict__ part) {
  using T = TT<MODE>;
  TILE_PROLOGUE
  for (int b = next_active(active, blockIdx.z * BB - 1, nb, BB); b >= 0; b = next_active(active, b, nb, BB)) {
    double v0 = 0;
    if (in) {
      const size_t j = (size_t)b * n + i;
      const T al = alpha[b];
      x_[j] = x_[j] + mul(al, p[j]);
      const T rj = r[j] - mul(al, q[j]);
      r[j] = rj;
      v0 = norm2(rj);
      if (z) z[j] = omega * mul(rj, sinv(diag_global<MODE>(op, b, i)));
    }
    block_pair(v0, 0.0, part, b);
    __syncthreads();
  }
}

// ===================================================================
// Fused V-cycle passes with halo-2 temporal blocking.
//
// k_down (level l): from the level's right-hand side r, two smoothing
// half-steps from zero (damped Jacobi x2, or one forward red-black
// Gauss-Seidel sweep on the 5-point fine level), the residual r - A z2 and
// its restriction P^T to level l+1, in one pass: reads r once (tile + halo 2),
// writes z2 (tile) and the coarse right-hand side.
// k_up (level l): z2 + P x_{l+1} on the halo-2 tile, two post-smoothing
// half-steps (Jacobi x2, or one backward black-red Gauss-Seidel sweep), in
// one pass: reads z2, r, x_{l+1}; writes z4 (and the partial r^T z4 on the
// fine level).  Pre and post smoothers are adjoint, restriction is P^T and
// the coarsest solve is exact, so the V-cycle is a symmetric (in x^T y)
// preconditioner and COCG's short recurrence holds.
// Regions in tile-local coordinates (origin x0-2, y0-2): staged grid
// H2 = 37x13; down pass: z1 on H2, z2 on D = [1,36)x[1,12), residual on
// Q = [2,35)x[2,11) (tile + the extra column/row the restriction gathers);
// up pass: z3 on H1 = [1,35)x[1,11), z4 on the tile [2,34)x[2,10).
constexpr int H2X = TX + 5, H2Y = TY + 5, H2N = H2X * H2Y;  // 481
constexpr int DX = TX + 3, DY = TY + 3, DN = DX * DY;       // 385
constexpr int H1X = TX + 2, H1Y = TY + 2, H1N = H1X * H1Y;  // 340
constexpr int QX = TX + 1, QY = TY + 1, QN = QX * QY;       // 297
enum { SM_JAC = 0, SM_RB = 1, SM_J1 = 2 };  // J1: one Jacobi step pre and post

template <int FAM>
struct CoefPlanes;
template <>
struct CoefPlanes<1> {  // fine: diag K, diag M, 4 real off-diagonals (W, E, S, N)
  static constexpr int planes = 6;
};
template <>
struct CoefPlanes<0> {  // coarse frequency mode, symmetric: K and M at C, E, N, NE
  static constexpr int planes = 8;
};
template <>
struct CoefPlanes<2> {  // slice mode, symmetric J (per batch): C, E, N, NE
  static constexpr int planes = 4;
};

template <int MODE, int FAM>
__device__ __forceinline__ void stage_coefs(const Op<MODE>& op, double* cf, int b, int x0, int y0) {
  const int tid = threadIdx.y * TX + threadIdx.x;
  const int m = op.m;
  const size_t n = op.n;
  for (int k = tid; k < H2N; k += NT) {
    const int ly = k / H2X, lx = k - ly * H2X;
    const int gx = x0 - 2 + lx, gy = y0 - 2 + ly;
    const bool in = gx >= 0 && gx < m && gy >= 0 && gy < m;
    const size_t i = in ? (size_t)gy * m + gx : 0;
    if constexpr (FAM == 1) {
      const Op<0>& o = op;
      cf[0 * H2N + k] = in ? __ldg(o.K + i) : 1.0;
      cf[1 * H2N + k] = in ? __ldg(o.M + i) : 0.0;
      for (int d = 1; d <= 4; ++d) cf[(1 + d) * H2N + k] = in ? __ldg(o.K + d * n + i) : 0.0;
    } else if constexpr (FAM == 0) {
      // Galerkin operators are symmetric: W(i) = E(i-1), S(i) = N(i-m),
      // SW(i) = NE(i-m-1), so four planes per matrix describe them
      const Op<0>& o = op;
      const int dirs[4] = {SC, SE_, SN_, SNE};
      for (int q = 0; q < 4; ++q) {
        cf[q * H2N + k] = in ? __ldg(o.K + dirs[q] * n + i) : (q == 0 ? 1.0 : 0.0);
        cf[(4 + q) * H2N + k] = in ? __ldg(o.M + dirs[q] * n + i) : 0.0;
      }
    } else {
      // the element-assembled Jacobian is symmetric: W(i) = E(i-1), S(i) = N(i-m),
      // SW(i) = NE(i-m-1) -- the smoothers read four planes (the PCG operator
      // itself, k_apply_dot, still applies all seven)
      const Op<1>& o = op;
      const double* J = o.J + (size_t)b * 7 * n;
      const int dirs[4] = {SC, SE_, SN_, SNE};
      for (int q = 0; q < 4; ++q) cf[q * H2N + k] = in ? __ldg(J + dirs[q] * n + i) : (q == 0 ? 1.0 : 0.0);
    }
  }
}

// diagonal coefficient at H2 index h
template <int MODE, int FAM>
__device__ __forceinline__ TT<MODE> cdiag(const double* cf, int h, cplx l) {
  if constexpr (FAM == 2) {
    return cf[h];
  } else if constexpr (FAM == 1) {
    return cplx{fma(l.re, cf[H2N + h], cf[h]), l.im * cf[H2N + h]};
  } else {
    return cplx{fma(l.re, cf[4 * H2N + h], cf[h]), l.im * cf[4 * H2N + h]};
  }
}

// off-diagonal part sum_{d>0} a_d v[nbr_d] at H2 position (lx, ly)
template <int MODE, int FAM>
__device__ __forceinline__ TT<MODE> coff(const double* cf, const TT<MODE>* v, int lx, int ly, cplx l) {
  using T = TT<MODE>;
  const int h = ly * H2X + lx;
  const T vw = v[h - 1], ve = v[h + 1], vs = v[h - H2X], vn = v[h + H2X];
  if constexpr (FAM == 1) {
    cplx acc = axpy_r(cf[2 * H2N + h], vw, cplx{0, 0});
    acc = axpy_r(cf[3 * H2N + h], ve, acc);
    acc = axpy_r(cf[4 * H2N + h], vs, acc);
    acc = axpy_r(cf[5 * H2N + h], vn, acc);
    return acc;
  } else if constexpr (FAM == 2) {
    const T vsw = v[h - H2X - 1], vne = v[h + H2X + 1];
    return cf[1 * H2N + h - 1] * vw + cf[1 * H2N + h] * ve + cf[2 * H2N + h - H2X] * vs + cf[2 * H2N + h] * vn +
           cf[3 * H2N + h - H2X - 1] * vsw + cf[3 * H2N + h] * vne;
  } else {
    const T vsw = v[h - H2X - 1], vne = v[h + H2X + 1];
    // (plane, node) of each neighbour's coefficient: W = E(h-1), E = E(h),
    // S = N(h-row), N = N(h), SW = NE(h-row-1), NE = NE(h)
    const int pl[6] = {1, 1, 2, 2, 3, 3};
    const int at[6] = {h - 1, h, h - H2X, h, h - H2X - 1, h};
    const T vv[6] = {vw, ve, vs, vn, vsw, vne};
    T acc = zero_of(T{});
#pragma unroll
    for (int d = 0; d < 6; ++d) {
      const double kk = cf[pl[d] * H2N + at[d]], mm = cf[(4 + pl[d]) * H2N + at[d]];
      acc = acc + mul(cplx{fma(l.re, mm, kk), l.im * mm}, vv[d]);
    }
    return acc;
  }
}

template <int MODE, int FAM>
static constexpr size_t fused_smem(bool down) {
  (void)down;
  return (size_t)CoefPlanes<FAM>::planes * H2N * sizeof(double) + (size_t)3 * H2N * sizeof(TT<MODE>);
}

template <int MODE>
__device__ __forceinline__ cplx lam_of(const Op<MODE>& op, int b) {
  if constexpr (MODE == 0) return op.lam[b];
  else return cplx{0, 0};
}

template <int MODE, int FAM, int SM>
__global__ void __launch_bounds__(NT, 4) k_down(Op<MODE> op, Op<MODE> opc, const TT<MODE>* __restrict__ rv,
                                                TT<MODE>* __restrict__ z2out, TT<MODE>* __restrict__ bc,
                                                const int* __restrict__ active, double omega, double omega2,
                                                int nb, int BB) {
  using T = TT<MODE>;
  extern __shared__ __align__(16) unsigned char dsm[];
  double* cf = reinterpret_cast<double*>(dsm);
  T* sR = reinterpret_cast<T*>(dsm + (size_t)CoefPlanes<FAM>::planes * H2N * sizeof(double));
  T* sZ = sR + H2N;
  T* sW = sZ + H2N;
  T* sQ = sZ;  // residual tile reuses z1's storage (z1 is dead once z2 is formed)
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int m = op.m, n = op.n;
  if constexpr (FAM != 2) stage_coefs<MODE, FAM>(op, cf, 0, x0, y0);
  // my two H2 elements
  auto h2idx = [&](int k) {
    const int ly = k / H2X, lx = k - ly * H2X;
    const int gx = x0 - 2 + lx, gy = y0 - 2 + ly;
    return (k < H2N && gx >= 0 && gx < m && gy >= 0 && gy < m) ? gy * m + gx : -1;
  };
  const int ia = h2idx(tid), ib = h2idx(tid + NT);
  const bool hasb = tid + NT < H2N;
  // coarse node of this thread (first 64 threads)
  const int mcs = opc.m, nc = opc.n;
  const int cxl = tid & 15, cyl = tid >> 4;
  const int X = (x0 >> 1) + cxl, Y = (y0 >> 1) + cyl;
  const bool cin = tid < 64 && X < mcs && Y < mcs;
  const int ci = cin ? Y * mcs + X : 0;
  T ra = zero_of(T{}), rb = zero_of(T{});
  auto fetch = [&](int b) {
    const size_t o = (size_t)b * n;
    ra = ia >= 0 ? rv[o + ia] : zero_of(T{});
    rb = ib >= 0 ? rv[o + ib] : zero_of(T{});
  };
  int b = next_active(active, blockIdx.z * BB - 1, nb, BB);
  if (b >= 0) fetch(b);
  while (b >= 0) {
    const int bn = next_active(active, b, nb, BB);
    if constexpr (FAM == 2) stage_coefs<MODE, FAM>(op, cf, b, x0, y0);
    sR[tid] = ra;
    if (hasb) sR[tid + NT] = rb;
    __syncthreads();
    if (bn >= 0) fetch(bn);
    const cplx l = lam_of(op, b);
    // half-step 1 on H2 (from zero)
    for (int k = tid; k < H2N; k += NT) {
      const int ly = k / H2X, lx = k - ly * H2X;
      const T d = cdiag<MODE, FAM>(cf, k, l);
      T v;
      if constexpr (SM == SM_RB) {
        const int red = ((x0 - 2 + lx + y0 - 2 + ly) & 1) == 0;
        v = red ? mul(sR[k], sinv(d)) : zero_of(T{});
      } else {
        v = omega * mul(sR[k], sinv(d));
      }
      sZ[k] = v;
    }
    __syncthreads();
    // half-step 2 on D
    for (int k = tid; k < DN; k += NT) {
      const int ly = 1 + k / DX, lx = 1 + (k - (ly - 1) * DX);
      const int h = ly * H2X + lx;
      const T d = cdiag<MODE, FAM>(cf, h, l);
      const T off = coff<MODE, FAM>(cf, sZ, lx, ly, l);
      T v;
      if constexpr (SM == SM_RB) {
        const int red = ((x0 - 2 + lx + y0 - 2 + ly) & 1) == 0;
        v = red ? sZ[h] : mul(sR[h] - off, sinv(d));
      } else if constexpr (SM == SM_J1) {
        (void)d;
        (void)off;
        v = sZ[h];
      } else {
        v = sZ[h] + omega2 * mul(sR[h] - off - mul(d, sZ[h]), sinv(d));
      }
      sW[h] = v;
    }
    __syncthreads();
    // residual r - A z2 on [2,35)x[2,11); z2 of the tile to global
    for (int k = tid; k < QN; k += NT) {
      const int qy = k / QX, qx = k - qy * QX;
      const int lx = 2 + qx, ly = 2 + qy, h = ly * H2X + lx;
      const T z = sW[h];
      sQ[k] = sR[h] - coff<MODE, FAM>(cf, sW, lx, ly, l) - mul(cdiag<MODE, FAM>(cf, h, l), z);
      const int gx = x0 + qx, gy = y0 + qy;
      if (qx < TX && qy < TY && gx < m && gy < m) z2out[(size_t)b * n + gy * m + gx] = z;
    }
    __syncthreads();
    if (cin) {
      const int fx = 2 * cxl + 1, fy = 2 * cyl + 1;  // local fine centre in sQ
      const T side = sQ[fy * QX + fx - 1] + sQ[fy * QX + fx + 1] + sQ[(fy - 1) * QX + fx] +
                     sQ[(fy + 1) * QX + fx] + sQ[(fy - 1) * QX + fx - 1] + sQ[(fy + 1) * QX + fx + 1];
      bc[(size_t)b * nc + ci] = sQ[fy * QX + fx] + 0.5 * side;
    }
    __syncthreads();
    b = bn;
  }
}

template <int MODE, int FAM, int SM>
__global__ void __launch_bounds__(NT, 4) k_up(Op<MODE> op, const TT<MODE>* __restrict__ rv,
                                              const TT<MODE>* __restrict__ z2in,
                                              const TT<MODE>* __restrict__ xc, int mc,
                                              TT<MODE>* __restrict__ zout, const int* __restrict__ active,
                                              double omega, double omega2, int nb, int BB, int dot,
                                              double* __restrict__ part) {
  using T = TT<MODE>;
  extern __shared__ __align__(16) unsigned char dsm[];
  double* cf = reinterpret_cast<double*>(dsm);
  T* sR = reinterpret_cast<T*>(dsm + (size_t)CoefPlanes<FAM>::planes * H2N * sizeof(double));
  T* sZ = sR + H2N;
  T* sW = sZ + H2N;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int m = op.m, n = op.n;
  const int nc = mc * mc;
  if constexpr (FAM != 2) stage_coefs<MODE, FAM>(op, cf, 0, x0, y0);
  int ia = -1, ib = -1, pa0 = -1, pa1 = -1, pb0 = -1, pb1 = -1;
  double wa = 0, wb = 0;
  {
    auto setup = [&](int k, int& idx, int& p0, int& p1, double& w0) {
      if (k >= H2N) return;
      const int ly = k / H2X, lx = k - ly * H2X;
      const int gx = x0 - 2 + lx, gy = y0 - 2 + ly;
      if (gx < 0 || gx >= m || gy < 0 || gy >= m) return;
      idx = gy * m + gx;
      int cxp[2], cyp[2];
      double w[2];
      const int np = parents(gx, gy, mc, cxp, cyp, w);
      if (np > 0) { p0 = cyp[0] * mc + cxp[0]; w0 = w[0]; }
      if (np > 1) p1 = cyp[1] * mc + cxp[1];
    };
    setup(tid, ia, pa0, pa1, wa);
    setup(tid + NT, ib, pb0, pb1, wb);
  }
  const bool hasb = tid + NT < H2N;
  T za = zero_of(T{}), zb = zero_of(T{}), ra = zero_of(T{}), rb = zero_of(T{});
  auto fetch = [&](int b) {
    const size_t o = (size_t)b * n, oc = (size_t)b * nc;
    za = zero_of(T{});
    ra = zero_of(T{});
    if (ia >= 0) {
      za = z2in[o + ia];
      if (pa0 >= 0) za = za + wa * xc[oc + pa0];
      if (pa1 >= 0) za = za + 0.5 * xc[oc + pa1];
      ra = rv[o + ia];
    }
    zb = zero_of(T{});
    rb = zero_of(T{});
    if (ib >= 0) {
      zb = z2in[o + ib];
      if (pb0 >= 0) zb = zb + wb * xc[oc + pb0];
      if (pb1 >= 0) zb = zb + 0.5 * xc[oc + pb1];
      rb = rv[o + ib];
    }
  };
  int b = next_active(active, blockIdx.z * BB - 1, nb, BB);
  if (b >= 0) fetch(b);
  while (b >= 0) {
    const int bn = next_active(active, b, nb, BB);
    if constexpr (FAM == 2) stage_coefs<MODE, FAM>(op, cf, b, x0, y0);
    sZ[tid] = za;
    sR[tid] = ra;
    if (hasb) {
      sZ[tid + NT] = zb;
      sR[tid + NT] = rb;
    }
    __syncthreads();
    if (bn >= 0) fetch(bn);
    const cplx l = lam_of(op, b);
    // post half-step 1 on H1 (Jacobi, or the black points of a backward sweep)
    for (int k = tid; k < H1N; k += NT) {
      const int ly = 1 + k / H1X, lx = 1 + (k - (ly - 1) * H1X);
      const int h = ly * H2X + lx;
      const T d = cdiag<MODE, FAM>(cf, h, l);
      const T off = coff<MODE, FAM>(cf, sZ, lx, ly, l);
      T v;
      if constexpr (SM == SM_RB) {
        const int red = ((x0 - 2 + lx + y0 - 2 + ly) & 1) == 0;
        v = red ? sZ[h] : mul(sR[h] - off, sinv(d));
      } else if constexpr (SM == SM_J1) {
        (void)d;
        (void)off;
        v = sZ[h];
      } else {
        v = sZ[h] + omega2 * mul(sR[h] - off - mul(d, sZ[h]), sinv(d));
      }
      sW[h] = v;
    }
    __syncthreads();
    // post half-step 2 on the tile (Jacobi, or the red points)
    double vd[2] = {0, 0};
    {
      const int lx = tx + 2, ly = ty + 2, h = ly * H2X + lx;
      const int gx = x0 + tx, gy = y0 + ty;
      if (gx < m && gy < m) {
        const T d = cdiag<MODE, FAM>(cf, h, l);
        const T off = coff<MODE, FAM>(cf, sW, lx, ly, l);
        T v;
        if constexpr (SM == SM_RB) {
          const int red = ((gx + gy) & 1) == 0;
          v = red ? mul(sR[h] - off, sinv(d)) : sW[h];
        } else {
          v = sW[h] + omega * mul(sR[h] - off - mul(d, sW[h]), sinv(d));
        }
        zout[(size_t)b * n + gy * m + gx] = v;
        if (dot) add_dot(vd, sR[h], v);
      }
    }
    if (dot) block_pair(vd[0], vd[1], part, b);
    __syncthreads();
    b = bn;
  }
}

// x += xa p for the frequencies with a deferred update (fused Krylov step)
template <class T>
__global__ void k_xfix(T* __restrict__ x, const T* __restrict__ p, const T* __restrict__ xa, size_t n, int nb) {
  TP_PDL_ENTRY();
  const int b = blockIdx.y;
  if (b >= nb) return;
  const T a = xa[b];
  if (norm2(a) == 0.0) return;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const size_t j = (size_t)b * n + i;
    x[j] = x[j] + mul(a, p[j]);
  }
}

// partial b^T z
template <int MODE>
__global__ void __launch_bounds__(NT, 4) k_dot(Op<MODE> op, const TT<MODE>* __restrict__ a_,
                                               const TT<MODE>* __restrict__ z, const int* __restrict__ active,
                                               int nb, int BB, double* __restrict__ part) {
  TILE_PROLOGUE
  for (int b = next_active(active, blockIdx.z * BB - 1, nb, BB); b >= 0; b = next_active(active, b, nb, BB)) {
    double v[2] = {0, 0};
    if (in) add_dot(v, a_[(size_t)b * n + i], z[(size_t)b * n + i]);
    block_pair(v[0], v[1], part, b);
    __syncthreads();
  }
}

// dense coarsest solve x = inv b, one block per batch
template <class T>
__global__ void k_coarse_solve(const T* __restrict__ inv, const T* __restrict__ bc, T* __restrict__ xc,
                               int nL, const int* __restrict__ active) {
  const int b = blockIdx.x;
  if (!active[b]) return;
  const T* A = inv + (size_t)b * nL * nL;  // transposed: A[j*nL + i] = inv(i, j)
  for (int i = threadIdx.x; i < nL; i += blockDim.x) {
    T acc = zero_of(bc[0]);
    for (int j = 0; j < nL; ++j) acc = acc + mul(A[(size_t)j * nL + i], bc[(size_t)b * nL + j]);
    xc[(size_t)b * nL + i] = acc;
  }
}

// ---- per-batch scalar updates (one block per batch, fixed-order sums)
__device__ __forceinline__ void batch_sum(const double* __restrict__ part, int per, int b, double& s0,
                                          double& s1) {
  __shared__ double sh[2][32];
  double a = 0, c = 0;
  for (int k = threadIdx.x; k < per; k += blockDim.x) {
    a += part[((size_t)b * per + k) * 2];
    c += part[((size_t)b * per + k) * 2 + 1];
  }
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_down_sync(0xffffffffu, a, o);
    c += __shfl_down_sync(0xffffffffu, c, o);
  }
  if ((threadIdx.x & 31) == 0) {
    sh[0][threadIdx.x >> 5] = a;
    sh[1][threadIdx.x >> 5] = c;
  }
  __syncthreads();
  s0 = 0;
  s1 = 0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) {
      s0 += sh[0][w];
      s1 += sh[1][w];
    }
}

template <class T>
__device__ __forceinline__ T from2(double a, double b);
template <>
__device__ __forceinline__ cplx from2<cplx>(double a, double b) { return {a, b}; }
template <>
__device__ __forceinline__ double from2<double>(double a, double) { return a; }

enum Stage { ST_INIT = 0, ST_RHO0 = 1, ST_ALPHA = 2, ST_RN = 3, ST_BETA = 4 };

template <class T>
__global__ void k_scalars(int stage, const double* __restrict__ part, int per, int nb, double rtol2,
                          T* __restrict__ rho, T* __restrict__ mu, T* __restrict__ alpha,
                          T* __restrict__ beta, double* __restrict__ bn2, double* __restrict__ rn2,
                          int* __restrict__ active, int* __restrict__ zero, const int* __restrict__ mask,
                          T* __restrict__ xa, int* __restrict__ count = nullptr,
                          const double* __restrict__ bfloor = nullptr, double fscale = 0.0,
                          int* __restrict__ count_clear = nullptr, volatile int* __restrict__ pub = nullptr,
                          unsigned* __restrict__ done = nullptr, double* __restrict__ bown = nullptr,
                          const double* __restrict__ bscale = nullptr) {
  TP_PDL_ENTRY();
  const int b = blockIdx.x;
  if (b >= nb) return;
  // ST_RN with pub: the last block to finish publishes the active count to
  // mapped host memory (the host reads it after an event)
  auto arrive = [&]() {
    if (!pub || stage != ST_RN || threadIdx.x != 0) return;
    __threadfence();
    if (atomicAdd(done, 1u) == (unsigned)nb - 1u) {
      __threadfence();
      *pub = atomicAdd(count, 0);
      *done = 0u;
      __threadfence_system();
    }
  };
  // fused-scalar path (no ST_ALPHA stage): ST_RN clears the other counter slot
  // for the next iteration and retires the deferred x coefficient of batches
  // that converged an iteration ago (their last update was applied by this
  // iteration's apply)
  if (count_clear && b == 0 && threadIdx.x == 0) *count_clear = 0;
  if (count_clear && xa && threadIdx.x == 0 && stage == ST_RN && !active[b]) xa[b] = from2<T>(0.0, 0.0);
  // active-batch counter of this iteration: cleared by ST_ALPHA, summed by ST_RN
  // (integer atomics: the count is exact whatever the block order)
  if (count && stage == ST_ALPHA && b == 0 && threadIdx.x == 0) *count = 0;
  if (xa && threadIdx.x == 0 && (stage == ST_INIT || (stage == ST_ALPHA && !active[b]))) xa[b] = from2<T>(0.0, 0.0);
  if (stage != ST_INIT && !active[b]) {
    arrive();
    return;
  }
  double s0, s1;
  batch_sum(part, per, b, s0, s1);
  if (threadIdx.x != 0) return;
  switch (stage) {
    case ST_INIT: {
      // stopping reference: ||g_k||^2, floored at the frequency's equal share
      // of the whole right-hand side (BatchSolver::bfloor)
      const double bref = (bfloor ? fmax(s0, fscale * *bfloor) : s0) * (bscale ? bscale[b] : 1.0);
      bn2[b] = bref;
      if (bown) bown[b] = s0;  // the block's own ||g_k||^2 (SparseSolver contract, solve.hpp:79-89)
      rn2[b] = s1;
      zero[b] = (s0 == 0.0);
      active[b] = (!mask || mask[b]) && (s0 > 0.0) && (s1 > rtol2 * bref);
      break;
    }
    case ST_RHO0:
      rho[b] = from2<T>(s0, s1);
      break;
    case ST_ALPHA: {
      const T m = from2<T>(s0, s1);
      mu[b] = m;
      alpha[b] = cdiv(rho[b], m);
      if (xa) xa[b] = alpha[b];
      break;
    }
    case ST_RN:
      rn2[b] = s0;
      active[b] = s0 > rtol2 * bn2[b];
      if (count && active[b]) atomicAdd(count, 1);
      arrive();
      break;
    case ST_BETA: {
      const T rn = from2<T>(s0, s1);
      beta[b] = cdiv(rn, rho[b]);
      rho[b] = rn;
      break;
    }
  }
}

__global__ void k_count_active(const int* __restrict__ active, int nb, int* __restrict__ count) {
  __shared__ int sh[32];
  int c = 0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) c += active[b];
  for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) s += sh[w];
    count[0] = s;
    count[1] = 0;  // the first iteration's counter slot
  }
}

// ---- hierarchy construction kernels

// Galerkin product P^T A P for one coarse node per thread.  The coarse
// centre (X, Y) is fine node (2X+1, 2Y+1); its P^T row gathers the 7 fine
// nodes fx = 2X+1+ox_s (weights 1, 1/2 x 6), each fine stencil entry d
// reaches fine node g = f + dir_d, and P interpolates g from its one or two
// coarse parents -- all offsets relative to (X, Y) are compile-time constants
// (fully unrolled), only the grid-boundary tests are run time.
__device__ __forceinline__ constexpr int floordiv2(int v) { return v >= 0 ? v / 2 : -((1 - v) / 2); }
__device__ __forceinline__ constexpr int dir_of(int ex, int ey) {
  return (ex == 0 && ey == 0) ? SC
         : (ex == -1 && ey == 0) ? SW_
         : (ex == 1 && ey == 0) ? SE_
         : (ex == 0 && ey == -1) ? SS_
         : (ex == 0 && ey == 1) ? SN_
         : (ex == -1 && ey == -1) ? SSW
         : (ex == 1 && ey == 1) ? SNE
                                : -1;
}

__global__ void k_rap(const double* __restrict__ Af, int mf, double* __restrict__ Ac, int mc) {
  const size_t nf = (size_t)mf * mf, nc = (size_t)mc * mc;
  const int b = blockIdx.y;
  const size_t ic = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (ic >= nc) return;
  const double* A = Af + (size_t)b * 7 * nf;
  const int X = (int)(ic % mc), Y = (int)(ic / mc);
  constexpr int sox[7] = {0, -1, 1, 0, 0, -1, 1}, soy[7] = {0, 0, 0, -1, 1, -1, 1};
  double out[7] = {0, 0, 0, 0, 0, 0, 0};
#pragma unroll
  for (int s = 0; s < 7; ++s) {
    const double sw = s == 0 ? 1.0 : 0.5;
    const int fx = 2 * X + 1 + sox[s], fy = 2 * Y + 1 + soy[s];
    if (fx < 0 || fx >= mf || fy < 0 || fy >= mf) continue;
    const size_t fi = (size_t)fy * mf + fx;
#pragma unroll
    for (int d = 0; d < 7; ++d) {
      // fine neighbour g = f + dir_d, vertex (a, b) = g + 1 = 2 (X+1, Y+1) + (ox, oy)
      const int ox = sox[s] + dir_dx(d), oy = soy[s] + dir_dy(d);
      const int gx = fx + dir_dx(d), gy = fy + dir_dy(d);
      if (gx < 0 || gx >= mf || gy < 0 || gy >= mf) continue;
      const double a = __ldg(A + d * nf + fi) * sw;
      // parents relative to (X, Y): first (fx2, fy2); second +1 in x and/or y
      const int px = floordiv2(ox), py = floordiv2(oy);
      const bool aodd = (ox & 1) != 0, bodd = (oy & 1) != 0;
      const double w1 = (aodd || bodd) ? 0.5 : 1.0;
      {
        const int e = dir_of(px, py);
        const int CX = X + px, CY = Y + py;
        if (e >= 0 && CX >= 0 && CX < mc && CY >= 0 && CY < mc) out[e] += a * w1;
      }
      if (aodd || bodd) {
        const int qx = px + (aodd ? 1 : 0), qy = py + (bodd ? 1 : 0);
        const int e = dir_of(qx, qy);
        const int CX = X + qx, CY = Y + qy;
        if (e >= 0 && CX >= 0 && CX < mc && CY >= 0 && CY < mc) out[e] += a * 0.5;
      }
    }
  }
  double* C = Ac + (size_t)b * 7 * nc;
#pragma unroll
  for (int d = 0; d < 7; ++d) C[d * nc + ic] = out[d];
}

// Gauss-Jordan inverse of the dense coarsest operator (no pivoting: SPD or
// complex symmetric with SPD Hermitian part), one block per batch.
template <int MODE>
__global__ void k_dense_inverse(const double* __restrict__ K, const double* __restrict__ M,
                                const cplx* __restrict__ lam, int m, TT<MODE>* __restrict__ inv,
                                size_t batch_stride_K) {
  using T = TT<MODE>;
  extern __shared__ unsigned char raw[];
  T* A = reinterpret_cast<T*>(raw);
  const int n = m * m, w = 2 * n;
  const int b = blockIdx.x;
  const double* Kb = K + (size_t)b * batch_stride_K;
  for (int t = threadIdx.x; t < n * w; t += blockDim.x) A[t] = zero_of(A[0]);
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int x = i % m, y = i / m;
    for (int d = 0; d < 7; ++d) {
      const int nx = x + dir_dx(d), ny = y + dir_dy(d);
      if (nx < 0 || nx >= m || ny < 0 || ny >= m) continue;
      const int j = ny * m + nx;
      T a;
      if constexpr (MODE == 0) {
        const cplx l = lam[b];
        a = cplx{l.re * M[d * n + i] + Kb[d * n + i], l.im * M[d * n + i]};
      } else {
        a = Kb[d * n + i];
      }
      A[(size_t)i * w + j] = A[(size_t)i * w + j] + a;
    }
    A[(size_t)i * w + n + i] = from2<T>(1.0, 0.0);
  }
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    const T piv = inv_of(A[(size_t)k * w + k]);
    __syncthreads();
    for (int j = threadIdx.x; j < w; j += blockDim.x) A[(size_t)k * w + j] = mul(A[(size_t)k * w + j], piv);
    __syncthreads();
    for (int t = threadIdx.x; t < n * w; t += blockDim.x) {
      const int i = t / w, j = t % w;
      if (i == k) continue;
      const T f = A[(size_t)i * w + k];
      if (j == k) continue;
      A[t] = A[t] - mul(f, A[(size_t)k * w + j]);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x)
      if (i != k) A[(size_t)i * w + k] = zero_of(A[0]);
    __syncthreads();
  }
  // stored transposed (column j contiguous over rows i) so the coarse solve
  // reads it coalesced
  for (int t = threadIdx.x; t < n * n; t += blockDim.x) {
    const int j = t / n, i = t % n;
    inv[(size_t)b * n * n + t] = A[(size_t)i * w + n + j];
  }
}

}  // namespace

namespace {
__global__ void k_planes_f32(const double* __restrict__ K, float* __restrict__ Kf, size_t n) {
  const int b = blockIdx.y;
  const double* Kb = K + (size_t)b * 7 * n;
  float* Fb = Kf + (size_t)b * 4 * n;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    Fb[i] = (float)Kb[(size_t)SC * n + i];
    Fb[n + i] = (float)Kb[(size_t)SE_ * n + i];
    Fb[2 * n + i] = (float)Kb[(size_t)SN_ * n + i];
    Fb[3 * n + i] = (float)Kb[(size_t)SNE * n + i];
  }
}
}  // namespace

void launch_planes_f32(Problem& p, const double* K, int m, float* Kf, int batches) {
  const size_t n = (size_t)m * m;
  const dim3 g((unsigned)std::min<size_t>((n + 255) / 256, 1024), batches);
  k_planes_f32<<<g, 256, 0, p.cur_stream()>>>(K, Kf, n);
  TP_LAUNCHED(&p);
}

void launch_rap(Problem& p, const double* Af, int mf, double* Ac, int mc, int batches) {
  const size_t nc = (size_t)mc * mc;
  dim3 grid((unsigned)((nc + 127) / 128), batches);
  k_rap<<<grid, 128, 0, p.cur_stream()>>>(Af, mf, Ac, mc);
  TP_LAUNCHED(&p);
}

template <int MODE>
static void launch_dense_inverse(Problem& p, const double* K, const double* M, int m, const cplx* lam,
                                 TT<MODE>* inv, int batches, size_t strideK) {
  const int n = m * m;
  const size_t smem = (size_t)n * 2 * n * sizeof(TT<MODE>);
  require(smem <= 200 * 1024, "multigrid: coarsest grid too large for the dense solve");
  TP_CUDA(cudaFuncSetAttribute(k_dense_inverse<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_dense_inverse<MODE><<<batches, 256, smem, p.cur_stream()>>>(K, M, lam, m, inv, strideK);
  TP_LAUNCHED(&p);
}

void launch_coarse_inverse_freq(Problem& p, const double* K, const double* M, int m, const cplx* lam,
                                cplx* inv, int batches) {
  launch_dense_inverse<0>(p, K, M, m, lam, inv, batches, 0);
}

void launch_coarse_inverse_slice(Problem& p, const double* J, int m, double* inv, int batches) {
  launch_dense_inverse<1>(p, J, nullptr, m, nullptr, inv, batches, (size_t)7 * m * m);
}

// ---------------------------------------------------------------- solver

template <int MODE>
static Op<MODE> make_op(const LevelOp& L, const cplx* lam);
template <>
Op<0> make_op<0>(const LevelOp& L, const cplx* lam) {
  return Op<0>{L.K, L.M, lam, L.n, L.m};
}
template <>
Op<1> make_op<1>(const LevelOp& L, const cplx*) {
  return Op<1>{L.K, L.n, L.m};
}

// launch geometry for a level: 32x8 node tiles x batch groups of BB
struct Geo {
  dim3 grid;
  int BB;
  int tiles;
};

static Geo geo_for(int m, int nb, int num_sms, int max_bb) {
  Geo g;
  const int gx = (m + TX - 1) / TX, gy = (m + TY - 1) / TY;
  g.tiles = gx * gy;
  // enough blocks to fill the machine ~4x, then batch loop inside a block
  int bb = (int)std::max<long>(1, (long)g.tiles * nb / (4L * num_sms));
  bb = std::min(bb, max_bb);
  g.BB = bb;
  g.grid = dim3(gx, gy, (nb + bb - 1) / bb);
  return g;
}

template <int MODE>
void BatchSolver<MODE>::init(Problem* prob, const std::vector<LevelOp>& levels, int batches,
                             const MGConfig& c) {
  p = prob;
  cfg = c;
  B = batches;
  ops = levels;
  const int L = (int)levels.size();
  lb.resize(L);
  lz0.resize(L);
  lz1.resize(L);
  for (int l = 0; l < L; ++l) {
    const size_t sz = (size_t)B * levels[l].n;
    if (l > 0) lb[l].alloc(sz);
    lz0[l].alloc(sz);
    if (l < L - 1 || L == 1) lz1[l].alloc(sz);
  }
  // frequency mode: the first level from which the rest of the cycle fits
  // one block's shared memory runs as the fused small-level kernel
  small_from = -1;
  if (MODE == 0 && !std::getenv("TPGPU_NO_SMALL")) {
    for (int l = 1; l + 1 < L; ++l) {
      if (L - l > kMaxSmall || levels[l].five) continue;
      int ms[kMaxSmall];
      for (int j = l; j < L; ++j) ms[j - l] = levels[j].m;
      static const size_t cap_kb = std::getenv("TPGPU_SMALL_KB") ? std::atoi(std::getenv("TPGPU_SMALL_KB")) : 224;
      if (small_cycle_smem(ms, L - l) <= cap_kb * 1024) {
        small_from = l;
        break;
      }
    }
  }
  if (small_from >= 0) {
    small = SmallLevels{};
    small.levels = L - small_from;
    for (int j = small_from; j < L; ++j) {
      small.m[j - small_from] = levels[j].m;
      small.K[j - small_from] = levels[j].K;
      small.M[j - small_from] = levels[j].M;
    }
    small_pack.alloc(small_pack_size(small.m, small.levels));
    pack_small_levels(*p, small, small_pack.get());
  }
  const size_t n0 = (size_t)B * levels[0].n;
  r.alloc(n0);
  if (L > 1 && ((MODE == 0 && levels[0].fine.we) || MODE == 1)) r2.alloc(n0);
  xa.alloc(B);
  p0.alloc(n0);
  p1.alloc(n0);
  q.alloc(n0);
  const size_t tiles = (size_t)((levels[0].m + TX - 1) / TX) * ((levels[0].m + TY - 1) / TY);
  const size_t perf = (size_t)fine_partials(levels[0].m, 0) + fine_partials(levels[0].m, 2);
  part.alloc((size_t)B * (tiles + perf) * 2 + 64);
  rho.alloc(B);
  mu.alloc(B);
  alpha.alloc(B);
  beta.alloc(B);
  bn2.alloc(B);
  bown.alloc(B);
  rn2.alloc(B);
  active.alloc(2 * B);
  count.alloc(2);
  done_ctr.alloc(1);
  TP_CUDA(cudaMemset(done_ctr.get(), 0, sizeof(unsigned)));
  if (!h_count) {
    // mapped pinned memory: the per-iteration active count is published by
    // the last block of the stopping-test kernel instead of a D2H copy, so the
    // solver's kernel chain is not broken by a copy node every iteration
    TP_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h_count), 2 * sizeof(int), cudaHostAllocMapped));
    TP_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h_count_dev), h_count, 0));
  }
  for (auto& e : ev)
    if (!e) TP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
}

template <int MODE>
BatchSolver<MODE>::~BatchSolver() {
  if (h_count) cudaFreeHost(h_count);
  for (auto& e : ev)
    if (e) cudaEventDestroy(e);
}

template <int MODE, int FAM, int SM>
static void set_fused_attrs() {
  static bool done = false;
  if (done) return;
  TP_CUDA(cudaFuncSetAttribute(k_down<MODE, FAM, SM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)fused_smem<MODE, FAM>(true)));
  TP_CUDA(cudaFuncSetAttribute(k_up<MODE, FAM, SM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)fused_smem<MODE, FAM>(false)));
  done = true;
}

// slice mode: levels with at least 15 nodes per side run the streaming passes
// (TPGPU_TILE_SLICE: the 32x8-tile kernels everywhere)
template <int MODE>
bool BatchSolver<MODE>::stream_level(int l) const {
  if constexpr (MODE == 1) {
    // (the l1-Jacobi smoother exists in the streaming passes only: with it every
    // non-coarsest level streams)
    static const bool tile = std::getenv("TPGPU_TILE_SLICE") != nullptr;
    return !tile && l + 1 < (int)ops.size() && (TPGPU_SLICE_L1 || ops[l].m >= 15);
  } else {
    return false;
  }
}

template <int MODE>
typename BatchSolver<MODE>::T* BatchSolver<MODE>::vcycle_level(int l, int nb, const T* bl, T*, bool,
                                                              bool dot) {
  const int L = (int)ops.size();
  const Op<MODE> op = make_op<MODE>(ops[l], lam);
  // coarse levels: few batches per block -- their blocks are latency-bound
  // chains (stage, two smoothing steps, residual), so more blocks in flight win
  static const int coarse_bb = std::getenv("TPGPU_COARSE_BB") ? std::atoi(std::getenv("TPGPU_COARSE_BB")) : 4;
  const Geo g = geo_for(ops[l].m, nb, p->num_sms, l == 0 ? 8 : coarse_bb);
  int* act = active.get();
  cudaStream_t s = p->cur_stream();
  const dim3 blk(TX, TY);
#define DISPATCH_FAM(lv, CALL)          \
  if constexpr (MODE == 1) {            \
    constexpr int FAM = 2;              \
    CALL;                               \
  } else if (ops[lv].five) {            \
    constexpr int FAM = 1;              \
    CALL;                               \
  } else {                              \
    constexpr int FAM = 0;              \
    CALL;                               \
  }
  if (L == 1) {
    k_coarse_solve<T><<<nb, 64, 0, s>>>(coarse_inv, bl, lz0[0].get(), ops[0].n, act);
    TP_LAUNCHED(p);
    if (dot) {
      k_dot<MODE><<<g.grid, blk, 0, s>>>(op, bl, lz0[0].get(), act, nb, g.BB, part.get());
      TP_LAUNCHED(p);
    }
    return lz0[0].get();
  }
  const Op<MODE> opc = make_op<MODE>(ops[l + 1], lam);
  T* z2 = lz0[l].get();
  T* zo = lz1[l].get();
  if constexpr (MODE == 0) {
    if (l == small_from) {
      trace_mark("small", p->cur_stream());
      launch_small_cycle(*p, small, lam, coarse_inv, bl, zo, act, cfg.omega, cfg.omega2, nb, cur_active);
      return zo;
    }
    if (ops[l].fine.we) {
      fine_down0(nb, bl);
      return fine_rest0(nb, bl, dot);
    }
  }
  return vcycle_generic(l, nb, bl, dot);
}

// the streaming-kernel view of level l: the fine K_hat edge weights (frequency
// mode) or the per-slice Jacobian stencils (slice mode)
template <int MODE>
FineOp BatchSolver<MODE>::stream_op(int l) const {
  FineOp so;
  if constexpr (MODE == 0) {
    so = ops[l].fine;
    so.lam = lam;
  } else {
    so.K = ops[l].K;
    so.kstride = (size_t)7 * ops[l].n;
    so.m = ops[l].m;
    so.n = ops[l].n;
  }
  return so;
}

template <int MODE>
void BatchSolver<MODE>::fine_down0(int nb, const T* r_in, const T* qv, T* r_out, const ScalFuse* sf,
                                   double* part_out) {
  const FineOp fo = stream_op(0);
  if constexpr (MODE == 0)
    // algorithmic bytes per fine node and active frequency: fused (the Krylov
    // update rides along) read r, q, write r, z2 and the 1/4 coarse rhs = 4.25
    // values; plain read r, write z2 and the coarse rhs = 2.25
    p->ktimer.time(1, p->cur_stream(), (qv ? 4.25 : 2.25) * (double)sizeof(T) * (double)ops[0].n * (double)cur_active,
                   [&] {
                     launch_stream_down(*p, fo, r_in, lz0[0].get(), lb[1].get(), ops[1].m, active.get(), cfg.omega,
                                        cfg.omega2, nb, qv, qv ? alpha.get() : nullptr, r_out,
                                        qv ? (part_out ? part_out : part.get()) : nullptr, sf);
                   });
  else
    launch_stream_down(*p, fo, r_in, lz0[0].get(), lb[1].get(), ops[1].m, active.get(), cfg.omega, cfg.omega2, nb,
                       qv, qv ? alpha.get() : nullptr, r_out, qv ? part.get() : nullptr);
}

template <int MODE>
typename BatchSolver<MODE>::T* BatchSolver<MODE>::fine_rest0(int nb, const T* bl, bool dot) {
  const int l = 0;
  const int L = (int)ops.size();
  int* act = active.get();
  cudaStream_t s = p->cur_stream();
  T* z2 = lz0[l].get();
  T* zo = lz1[l].get();
  {
    {
      const FineOp fo = stream_op(l);
      T* xcf;
      if (l + 1 == L - 1) {
        k_coarse_solve<T><<<nb, 64, 0, s>>>(coarse_inv, lb[l + 1].get(), lz0[l + 1].get(), ops[l + 1].n, act);
        TP_LAUNCHED(p);
        xcf = lz0[l + 1].get();
      } else {
        xcf = vcycle_level(l + 1, nb, lb[l + 1].get(), nullptr, false, false);
      }
      trace_mark("up", s);
      // algorithmic bytes: read z2, r and the coarse correction (1/4), write z --
      // 3.25 values per fine node of every active frequency
      p->ktimer.time(0, s, 3.25 * (double)sizeof(T) * (double)ops[l].n * (double)cur_active, [&] {
        launch_stream_up(*p, fo, bl, z2, xcf, ops[l + 1].m, zo, act, cfg.omega, cfg.omega2, nb, dot ? 1 : 0,
                         part.get());
      });
      return zo;
    }
  }
  return zo;
}

template <int MODE>
typename BatchSolver<MODE>::T* BatchSolver<MODE>::vcycle_generic(int l, int nb, const T* bl, bool dot) {
  const int L = (int)ops.size();
  const Op<MODE> op = make_op<MODE>(ops[l], lam);
  static const int coarse_bb = std::getenv("TPGPU_COARSE_BB") ? std::atoi(std::getenv("TPGPU_COARSE_BB")) : 4;
  const Geo g = geo_for(ops[l].m, nb, p->num_sms, l == 0 ? 8 : coarse_bb);
  int* act = active.get();
  cudaStream_t s = p->cur_stream();
  const dim3 blk(TX, TY);
  const Op<MODE> opc = make_op<MODE>(ops[l + 1], lam);
  T* z2 = lz0[l].get();
  T* zo = lz1[l].get();
  const bool rb = cfg.rb_fine && ops[l].five;
  static const bool tile_coarse = std::getenv("TPGPU_TILE_COARSE") != nullptr;
  static const bool coarse_j1 = std::getenv("TPGPU_COARSE_J1") != nullptr;
  const bool j1 = coarse_j1 && l > 0;
  if constexpr (MODE == 1) {
    // slice mode: warp-streaming passes over the per-slice Jacobian stencils
    if (stream_level(l)) {
      FineOp so;
      so.K = ops[l].K;
      so.kstride = (size_t)7 * ops[l].n;
      so.Kf = ops[l].Kf;
      so.kfstride = (size_t)4 * ops[l].n;
      so.m = ops[l].m;
      so.n = ops[l].n;
      launch_stream_down(*p, so, bl, z2, lb[l + 1].get(), ops[l + 1].m, act, cfg.omega, cfg.omega2, nb);
      T* xs;
      if (l + 1 == L - 1) {
        k_coarse_solve<T><<<nb, 64, 0, s>>>(coarse_inv, lb[l + 1].get(), lz0[l + 1].get(), ops[l + 1].n, act);
        TP_LAUNCHED(p);
        xs = lz0[l + 1].get();
      } else {
        xs = vcycle_level(l + 1, nb, lb[l + 1].get(), nullptr, false, false);
      }
      launch_stream_up(*p, so, bl, z2, xs, ops[l + 1].m, zo, act, cfg.omega, cfg.omega2, nb, dot ? 1 : 0,
                       part.get());
      return zo;
    }
  }
  if constexpr (MODE == 0) {
    // Galerkin levels of the frequency solver: warp-streaming passes
    if (!ops[l].five && !j1 && !tile_coarse && ops[l].m >= 7) {
      FineOp so;
      so.K = ops[l].K;
      so.M = ops[l].drop_m ? nullptr : ops[l].M;
      so.lam = lam;
      so.m = ops[l].m;
      so.n = ops[l].n;
      trace_mark("g-down", s);
      launch_stream_down(*p, so, bl, z2, lb[l + 1].get(), ops[l + 1].m, act, cfg.omega, cfg.omega2, nb);
      T* xs;
      if (l + 1 == L - 1) {
        k_coarse_solve<T><<<nb, 64, 0, s>>>(coarse_inv, lb[l + 1].get(), lz0[l + 1].get(), ops[l + 1].n, act);
        TP_LAUNCHED(p);
        xs = lz0[l + 1].get();
      } else {
        xs = vcycle_level(l + 1, nb, lb[l + 1].get(), nullptr, false, false);
      }
      trace_mark("g-up", s);
      launch_stream_up(*p, so, bl, z2, xs, ops[l + 1].m, zo, act, cfg.omega, cfg.omega2, nb, dot ? 1 : 0,
                       part.get());
      return zo;
    }
  }
  // down: smoothing from zero, residual, restriction
#define LAUNCH_DOWN(SMV)                                                                        \
  DISPATCH_FAM(l, (set_fused_attrs<MODE, FAM, SMV>(),                                          \
                   k_down<MODE, FAM, SMV><<<g.grid, blk, fused_smem<MODE, FAM>(true), s>>>(     \
                       op, opc, bl, z2, lb[l + 1].get(), act, cfg.omega, cfg.omega2, nb, g.BB)))
  if (rb) { LAUNCH_DOWN(SM_RB); } else if (j1) { LAUNCH_DOWN(SM_J1); } else { LAUNCH_DOWN(SM_JAC); }
  TP_LAUNCHED(p);
  T* xc;
  if (l + 1 == L - 1) {
    k_coarse_solve<T><<<nb, 64, 0, s>>>(coarse_inv, lb[l + 1].get(), lz0[l + 1].get(), ops[l + 1].n, act);
    TP_LAUNCHED(p);
    xc = lz0[l + 1].get();
  } else {
    xc = vcycle_level(l + 1, nb, lb[l + 1].get(), nullptr, false, false);
  }
  const int mcl = ops[l + 1].m;
  const int d = dot ? 1 : 0;
#define LAUNCH_UP(SMV)                                                                          \
  DISPATCH_FAM(l, (set_fused_attrs<MODE, FAM, SMV>(),                                          \
                   k_up<MODE, FAM, SMV><<<g.grid, blk, fused_smem<MODE, FAM>(false), s>>>(      \
                       op, bl, z2, xc, mcl, zo, act, cfg.omega, cfg.omega2, nb, g.BB, d, part.get())))
  if (rb) { LAUNCH_UP(SM_RB); } else if (j1) { LAUNCH_UP(SM_J1); } else { LAUNCH_UP(SM_JAC); }
  TP_LAUNCHED(p);
  return zo;
}

template <int MODE>
int BatchSolver<MODE>::solve(const T* b, T* x, int nb, bool warm, SolveStats* st) {
  require(nb <= B, "batch solver: too many right-hand sides");
  const Op<MODE> op0 = make_op<MODE>(ops[0], lam);
  const Geo g0 = geo_for(ops[0].m, nb, p->num_sms, 8);
  const dim3 blk(TX, TY);
  const bool fine = MODE == 0 && ops[0].fine.we != nullptr;
  // level 0 streamed (frequency mode: K_hat edge weights; slice mode: the
  // per-slice Jacobian stencils) -- the streaming apply / fused update apply
  const bool stream0 = fine || (MODE == 1 && stream_level(0));
  // partials per batch of each producing kernel
  const int per_t = g0.tiles;
  const int per_a = stream0 ? fine_partials(ops[0].m, 0) : per_t;   // streaming init / apply
  // V-cycle dot (up pass of level 0): streaming layout when that pass is streamed
  static const bool tile_coarse0 = std::getenv("TPGPU_TILE_COARSE") != nullptr;
  const bool up0_streamed = fine || stream_level(0) ||
                            (MODE == 0 && ops.size() > 1 && !ops[0].five && !tile_coarse0 && ops[0].m >= 7 &&
                             small_from != 0);
  const int per_u = up0_streamed ? fine_partials(ops[0].m, 2) : per_t;
  // fine level: the ring-staged streaming apply (mg_fine.cu) -- measured 8.08
  // vs 8.39 ms per cfg-1 sweep against the smem-tile apply (TPGPU_TILE_APPLY)
  static const bool use_stream_apply = std::getenv("TPGPU_TILE_APPLY") == nullptr;
  // slice mode: the tile apply (reading the symmetric Jacobian's four planes)
  // and the separate update pass measured faster than the streaming apply with
  // the fused update (cfg 1 init, ncu: 97 vs 99 ms); TPGPU_SLICE_STREAM_APPLY opts in
  static const bool slice_sapply = std::getenv("TPGPU_SLICE_STREAM_APPLY") != nullptr;
  const bool sapply = stream0 && use_stream_apply && (MODE == 0 || slice_sapply);
  // fused Krylov update (fine streaming path): r -= alpha q inside the fine
  // down pass (partial ||r||^2 from there), x += alpha p deferred to the next
  // apply -- the separate update pass disappears (cfg 1: 8.10 -> 7.65 ms per
  // sweep; TPGPU_UNFUSED_UPDATE restores the update pass)
  static const bool want_fuse = std::getenv("TPGPU_UNFUSED_UPDATE") == nullptr;
  const bool fused = sapply && ops.size() > 1 && want_fuse;
  const int per_d = stream0 ? fine_partials(ops[0].m, 1) : per_t;  // fused down (||r||^2)
  const double rtol2 = cfg.rtol * cfg.rtol;
  int* act = active.get();
  int* zero = active.get() + B;
  T* const xa_ptr = fused ? xa.get() : nullptr;
  // fused scalars (frequency mode, fused fine path): the apply reduces rho and
  // beta from the up pass's partials, the down pass mu and alpha from the
  // apply's -- two scalar kernels per iteration fewer on the critical path
  // (TPGPU_SCALAR_KERNELS=1 keeps them)
  static const bool want_fscal = std::getenv("TPGPU_SCALAR_KERNELS") == nullptr;
  static const bool use_publish = std::getenv("TPGPU_COUNT_MEMCPY") == nullptr;
  const bool fscal = MODE == 0 && fused && want_fscal;
  if (fscal) {
    rho2.ensure((size_t)2 * B);
    partA.ensure((size_t)B * per_a * 2);
    partD.ensure((size_t)B * per_d * 2);
  }
  cudaStream_t s = p->cur_stream();
  const int l = 0;
  // one k_scalars stage over `per` partials per batch (launch + count)
  auto scalars = [&](int stage, const double* partials, int per, int* cnt, int* cnt_clear, const double* floor_ptr,
                     double floor_scale, volatile int* pub = nullptr) {
    launch_pdl(k_scalars<T>, dim3(nb), dim3(256), 0, s, stage, partials, per, nb, rtol2, rho.get(), mu.get(),
               alpha.get(), beta.get(), bn2.get(), rn2.get(), act, zero, ext_mask, xa_ptr, cnt, floor_ptr,
               floor_scale, cnt_clear, pub, pub ? done_ctr.get() : static_cast<unsigned*>(nullptr), bown.get(),
               bscale);
    TP_LAUNCHED(p);
  };
  trace_mark("pcg-init", s);
  if (warm && sapply) {
    launch_fine_apply(*p, stream_op(0), b, x, nullptr, r.get(), nullptr, nullptr, 1, nb, part.get(), true);
  } else {
    DISPATCH_FAM(l, (k_init<MODE, FAM><<<g0.grid, blk, 0, s>>>(op0, b, x, r.get(), nb, g0.BB, warm ? 1 : 0, part.get())));
    TP_LAUNCHED(p);
  }
  scalars(ST_INIT, part.get(), (warm && sapply) ? per_a : per_t, nullptr, nullptr, bfloor, bfloor_scale);
  if (warm) {
    k_zero_flagged<MODE><<<g0.grid, blk, 0, s>>>(op0, x, nb, g0.BB, zero);
    TP_LAUNCHED(p);
  }
  k_count_active<<<1, 256, 0, s>>>(act, nb, count.get());
  TP_LAUNCHED(p);
  TP_CUDA(cudaMemcpyAsync(h_count, count.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  TP_CUDA(cudaStreamSynchronize(s));
  static const bool dbg_freq = std::getenv("TPGPU_DEBUG_FREQ") != nullptr;
  std::vector<int> dbg_it(dbg_freq ? nb : 0, 1);
  int iters = 0;
  int64_t batch_iters = 0;
  int last_active = h_count[0];
  cur_active = last_active;
  T* rcur = r.get();
  T* rnext = r2.get();
  T* pin = p0.get();
  T* pout = p1.get();
  if (last_active > 0) {
    T* z = vcycle_level(0, nb, rcur, nullptr, false, true);
    if (!fscal) scalars(ST_RHO0, part.get(), ops.size() > 1 ? per_u : per_t, nullptr, nullptr, nullptr, 0.0);
    bool done = false;
    for (int it = 1; it <= cfg.max_iter; ++it) {
      const int first = it == 1 ? 1 : 0;
      trace_mark("apply", s);
      const int par = it & 1;
      if (fscal) {
        if constexpr (MODE == 0) {
          ScalFuse sf;
          sf.part = part.get();  // the up pass's r^T z partials
          sf.per = per_u;
          sf.rho_r = rho2.get() + (size_t)(par ^ 1) * B;
          sf.rho_w = rho2.get() + (size_t)par * B;
          // algorithmic bytes: read z, p (not on the first iteration), x; write p, q, x
          p->ktimer.time(2, s, (first ? 5.0 : 6.0) * (double)sizeof(T) * (double)ops[0].n * (double)cur_active, [&] {
            launch_fine_apply(*p, stream_op(0), z, pin, pout, q.get(), beta.get(), act, first, nb, partA.get(), false,
                              x, xa_ptr, &sf);
          });
        }
      } else if (sapply) {
        launch_fine_apply(*p, stream_op(0), z, pin, pout, q.get(), beta.get(), act, first, nb, part.get(), false,
                          fused ? x : nullptr, xa_ptr);
      } else {
        DISPATCH_FAM(l, (k_apply_dot<MODE, FAM><<<g0.grid, blk, 0, s>>>(op0, z, pin, pout, q.get(), beta.get(), act,
                                                                        first, nb, g0.BB, part.get(), x, xa_ptr)));
        TP_LAUNCHED(p);
      }
      const int slot = it & 1;
      trace_mark("scalars", s);
      if (!fscal) scalars(ST_ALPHA, part.get(), sapply ? per_a : per_t, count.get() + slot, nullptr, nullptr, 0.0);
      if (fscal) {
        trace_mark("down", s);
        if constexpr (MODE == 0) {
          ScalFuse sf;
          sf.part = partA.get();  // the apply's p^T q partials
          sf.per = per_a;
          sf.rho_r = rho2.get() + (size_t)par * B;
          sf.alpha = alpha.get();
          sf.xa = xa.get();
          sf.mu = mu.get();
          fine_down0(nb, rcur, q.get(), rnext, &sf, partD.get());
        }
      } else if (fused) {
        trace_mark("down", s);
        fine_down0(nb, rcur, q.get(), rnext);
      } else {
        trace_mark("update", s);
        k_update<MODE><<<g0.grid, blk, 0, s>>>(op0, x, rcur, pout, q.get(), alpha.get(), act, cfg.omega, nullptr,
                                               nb, g0.BB, part.get());
        TP_LAUNCHED(p);
      }
      trace_mark("scalars", s);
      scalars(ST_RN, fscal ? partD.get() : part.get(), fused ? per_d : per_t, count.get() + slot,
              fscal ? count.get() + (slot ^ 1) : nullptr, nullptr, 0.0,
              use_publish ? static_cast<volatile int*>(h_count_dev + slot) : nullptr);
      if (!use_publish)
        TP_CUDA(cudaMemcpyAsync(h_count + slot, count.get() + slot, sizeof(int), cudaMemcpyDeviceToHost, s));
      TP_CUDA(cudaEventRecord(ev[slot], s));
      if (dbg_freq) {  // experiment: per-frequency iteration counts (synchronizes every iteration)
        std::vector<int> ha(nb);
        TP_CUDA(cudaMemcpyAsync(ha.data(), act, nb * sizeof(int), cudaMemcpyDeviceToHost, s));
        TP_CUDA(cudaStreamSynchronize(s));
        for (int k = 0; k < nb; ++k) dbg_it[k] += ha[k] ? 1 : 0;
      }
      // frequency-iterations (exact): iteration 1 works on the initially
      // active batches, iteration it >= 2 on those still active after it - 1
      if (it == 1) batch_iters += last_active;
      if (it >= 2) {
        TP_CUDA(cudaEventSynchronize(ev[slot ^ 1]));
        last_active = h_count[slot ^ 1];
        cur_active = last_active;
        if (last_active == 0) {
          iters = it - 1;
          done = true;
          break;
        }
        batch_iters += last_active;
      }
      iters = it;
      if (fused) {
        std::swap(rcur, rnext);
        z = fine_rest0(nb, rcur, true);
      } else {
        trace_mark("vcycle", s);
        z = vcycle_level(0, nb, rcur, nullptr, false, true);
      }
      trace_mark("scalars", s);
      if (!fscal) scalars(ST_BETA, part.get(), ops.size() > 1 ? per_u : per_t, nullptr, nullptr, nullptr, 0.0);
      std::swap(pin, pout);
    }
    if (!done) {
      TP_CUDA(cudaStreamSynchronize(s));
      last_active = h_count[iters & 1];
    }
    if (fused) {
      // the deferred x += alpha p of the last iteration (nothing is pending
      // when the loop ended by convergence: its final apply consumed it)
      const dim3 gx((unsigned)std::min<size_t>((ops[0].n + 255) / 256, 64), nb);
      launch_pdl(k_xfix<T>, gx, dim3(256), 0, s, x, static_cast<const T*>(done ? pout : pin), static_cast<const T*>(xa.get()),
                 (size_t)ops[0].n, nb);
      TP_LAUNCHED(p);
    }
  }
  TP_CUDA(cudaStreamSynchronize(s));
  std::vector<double> hb(nb), hr(nb), ho(nb);
  TP_CUDA(cudaMemcpyAsync(hb.data(), bn2.get(), nb * sizeof(double), cudaMemcpyDeviceToHost, s));
  TP_CUDA(cudaMemcpyAsync(hr.data(), rn2.get(), nb * sizeof(double), cudaMemcpyDeviceToHost, s));
  TP_CUDA(cudaMemcpyAsync(ho.data(), bown.get(), nb * sizeof(double), cudaMemcpyDeviceToHost, s));
  TP_CUDA(cudaStreamSynchronize(s));
  // achieved relative residual per block: against the stopping reference
  // (the block's own ||g_k|| floored at its share of the whole spectrum) and
  // against the block's own right-hand side (the reference SparseSolver's
  // per-solve contract); both reported, the floored one is enforced
  double worst = 0, worst_own = 0;
  for (int k = 0; k < nb; ++k) {
    if (hb[k] > 0) worst = std::max(worst, std::sqrt(hr[k] / hb[k]));
    if (ho[k] > 0) worst_own = std::max(worst_own, std::sqrt(hr[k] / ho[k]));
  }
  if (dbg_freq) {
    std::string line = "freqdbg nb " + std::to_string(nb) + " iters " + std::to_string(iters) + " |";
    for (int k = 0; k < nb; ++k) {
      char buf[64];
      std::snprintf(buf, sizeof buf, " %d:%.2e", dbg_it[k], std::sqrt(hb[k]));
      line += buf;
    }
    std::fprintf(stderr, "%s\n", line.c_str());
  }
  if (st) {
    st->iterations = std::max(st->iterations, iters);
    st->batch_iterations += batch_iters;
    st->max_rel_residual = std::max(st->max_rel_residual, worst);
    st->max_rel_residual_own = std::max(st->max_rel_residual_own, worst_own);
  }
  if (last_active > 0 && !(worst <= 1e-10))
    throw Error(TP_ESOLVE,
                "multigrid solve: relative residual " + std::to_string(worst) +
                    " exceeds the 1e-10 contract after " + std::to_string(iters) + " iterations",
                worst);
  return iters;
}

template struct BatchSolver<0>;
template struct BatchSolver<1>;

}  // namespace tpgpu
