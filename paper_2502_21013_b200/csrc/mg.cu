// Batched multigrid-preconditioned CG/COCG -- see mg.cuh.
//
// Traffic notes (per fine node, per batch, per Krylov iteration; 16 B per
// complex value): apply+dot (read z, p; write p, q), update (read x, p, r, q;
// write x, r, z), one extra pre-smooth, residual+restrict, prolong+smooth,
// last smooth+dot: ~22 streams on the fine level, ~1/3 more on the coarse
// levels.  The kernels keep one thread per node and loop over BPT batches so
// the shared frequency-mode stencil is loaded once per node.
#include <algorithm>
#include <cmath>

#include "mg.cuh"

namespace tpgpu {

namespace {

constexpr int NT = 256;

template <int MODE>
struct Op;

template <>
struct Op<0> {
  const double* K;
  const double* M;
  const cplx* lam;
  size_t n;
  int m;
  struct Pre {
    double k[7], mm[7];
  };
  __device__ __forceinline__ void pre(size_t i, Pre& P) const {
#pragma unroll
    for (int d = 0; d < 7; ++d) {
      P.k[d] = K[d * n + i];
      P.mm[d] = M[d * n + i];
    }
  }
  __device__ __forceinline__ void coef(const Pre& P, int b, size_t, cplx a[7]) const {
    const cplx l = lam[b];
#pragma unroll
    for (int d = 0; d < 7; ++d) a[d] = {fma(l.re, P.mm[d], P.k[d]), l.im * P.mm[d]};
  }
};

template <>
struct Op<1> {
  const double* J;
  size_t n;
  int m;
  struct Pre {};
  __device__ __forceinline__ void pre(size_t, Pre&) const {}
  __device__ __forceinline__ void coef(const Pre&, int b, size_t i, double a[7]) const {
    const double* s = J + (size_t)b * 7 * n;
#pragma unroll
    for (int d = 0; d < 7; ++d) a[d] = s[d * n + i];
  }
};

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
__device__ __forceinline__ cplx inv_of(cplx a) { return cdiv(cplx{1, 0}, a); }
__device__ __forceinline__ double inv_of(double a) { return 1.0 / a; }

struct Nbr {
  long off[7];
  bool ok[7];
};

__device__ __forceinline__ void neighbours(size_t i, int m, Nbr& nb) {
  const int x = (int)(i % m), y = (int)(i / m);
  nb.off[0] = 0; nb.ok[0] = true;
  nb.off[1] = -1; nb.ok[1] = x > 0;
  nb.off[2] = 1; nb.ok[2] = x < m - 1;
  nb.off[3] = -m; nb.ok[3] = y > 0;
  nb.off[4] = m; nb.ok[4] = y < m - 1;
  nb.off[5] = -m - 1; nb.ok[5] = x > 0 && y > 0;
  nb.off[6] = m + 1; nb.ok[6] = x < m - 1 && y < m - 1;
}

template <class T>
__device__ __forceinline__ T apply7(const T a[7], const T* __restrict__ v, size_t i, const Nbr& nb) {
  T acc = mul(a[0], v[i]);
#pragma unroll
  for (int d = 1; d < 7; ++d)
    if (nb.ok[d]) acc = acc + mul(a[d], v[i + nb.off[d]]);
  return acc;
}

template <int BPT>
__device__ __forceinline__ void block_partials(double (&v)[BPT][2], double* __restrict__ part, int b0,
                                               int nb, int per) {
  __shared__ double sh[BPT][2][NT / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < BPT; ++k)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      double x = v[k][c];
      for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
      if (lane == 0) sh[k][c][w] = x;
    }
  __syncthreads();
  if ((int)threadIdx.x < BPT * 2) {
    const int k = threadIdx.x >> 1, c = threadIdx.x & 1;
    double s = 0;
    for (int ww = 0; ww < NT / 32; ++ww) s += sh[k][c][ww];
    const int b = b0 + k;
    if (b < nb) part[((size_t)b * gridDim.x + blockIdx.x) * 2 + c] = s;
  }
}

// r = b - A x (warm) or r = b, x = 0 (cold); partials (||b||^2, ||r||^2).
template <int MODE, int BPT>
__global__ void __launch_bounds__(NT) k_init(Op<MODE> op, const TT<MODE>* __restrict__ bv,
                                             TT<MODE>* __restrict__ x, TT<MODE>* __restrict__ r,
                                             int nb, int warm, double* __restrict__ part) {
  using T = TT<MODE>;
  const size_t n = op.n;
  const size_t i = (size_t)blockIdx.x * NT + threadIdx.x;
  const int b0 = blockIdx.y * BPT;
  double v[BPT][2] = {};
  if (i < n) {
    typename Op<MODE>::Pre P;
    Nbr nbr;
    if (warm) {
      op.pre(i, P);
      neighbours(i, op.m, nbr);
    }
#pragma unroll
    for (int k = 0; k < BPT; ++k) {
      const int b = b0 + k;
      if (b >= nb) break;
      const T bi = bv[(size_t)b * n + i];
      T ri = bi;
      if (warm) {
        T a[7];
        op.coef(P, b, i, a);
        ri = bi - apply7(a, x + (size_t)b * n, i, nbr);
      } else {
        x[(size_t)b * n + i] = zero_of(bi);
      }
      r[(size_t)b * n + i] = ri;
      v[k][0] += norm2(bi);
      v[k][1] += norm2(ri);
    }
  }
  block_partials<BPT>(v, part, b0, nb, gridDim.x);
}

template <int MODE, int BPT>
__global__ void __launch_bounds__(NT) k_zero_flagged(TT<MODE>* __restrict__ x, size_t n, int nb,
                                                     const int* __restrict__ zero) {
  const size_t i = (size_t)blockIdx.x * NT + threadIdx.x;
  if (i >= n) return;
  for (int k = 0; k < BPT; ++k) {
    const int b = blockIdx.y * BPT + k;
    if (b >= nb) break;
    if (zero[b]) x[(size_t)b * n + i] = zero_of(x[0]);
  }
}

// p_out = first ? z : z + beta p_in ;  q = A p_out ; partial p^T q
template <int MODE, int BPT>
__global__ void __launch_bounds__(NT) k_apply_dot(Op<MODE> op, const TT<MODE>* __restrict__ z,
                                                  const TT<MODE>* __restrict__ pin,
                                                  TT<MODE>* __restrict__ pout, TT<MODE>* __restrict__ q,
                                                  const TT<MODE>* __restrict__ beta,
                                                  const int* __restrict__ active, int first, int nb,
                                                  double* __restrict__ part) {
  using T = TT<MODE>;
  const size_t n = op.n;
  const size_t i = (size_t)blockIdx.x * NT + threadIdx.x;
  const int b0 = blockIdx.y * BPT;
  double v[BPT][2] = {};
  if (i < n) {
    typename Op<MODE>::Pre P;
    op.pre(i, P);
    Nbr nbr;
    neighbours(i, op.m, nbr);
#pragma unroll
    for (int k = 0; k < BPT; ++k) {
      const int b = b0 + k;
      if (b >= nb) break;
      if (!active[b]) continue;
      const size_t o = (size_t)b * n;
      T a[7];
      op.coef(P, b, i, a);
      const T bt = first ? zero_of(a[0]) : beta[b];
      T acc = zero_of(a[0]), pi = zero_of(a[0]);
#pragma unroll
      for (int d = 0; d < 7; ++d) {
        if (!nbr.ok[d]) continue;
        const size_t j = o + i + nbr.off[d];
        const T pj = first ? z[j] : z[j] + mul(bt, pin[j]);
        if (d == 0) pi = pj;
        acc = acc + mul(a[d], pj);
      }
      pout[o + i] = pi;
      q[o + i] = acc;
      add_dot(v[k], pi, acc);
    }
  }
  block_partials<BPT>(v, part, b0, nb, gridDim.x);
}

// x += alpha p ; r -= alpha q ; partial ||r||^2 ; z = omega r / a_C
template <int MODE, int BPT>
__global__ void __launch_bounds__(NT) k_update(Op<MODE> op, TT<MODE>* __restrict__ x,
                                               TT<MODE>* __restrict__ r, const TT<MODE>* __restrict__ p,
                                               const TT<MODE>* __restrict__ q,
                                               const TT<MODE>* __restrict__ alpha,
                                               const int* __restrict__ active, double omega,
                                               TT<MODE>* __restrict__ z, int nb,
                                               double* __restrict__ part) {
  using T = TT<MODE>;
  const size_t n = op.n;
  const size_t i = (size_t)blockIdx.x * NT + threadIdx.x;
  const int b0 = blockIdx.y * BPT;
  double v[BPT][2] = {};
  if (i < n) {
    typename Op<MODE>::Pre P;
    op.pre(i, P);
#pragma unroll
    for (int k = 0; k < BPT; ++k) {
      const int b = b0 + k;
      if (b >= nb) break;
      if (!active[b]) continue;
      const size_t j = (size_t)b * n + i;
      const T al = alpha[b];
      x[j] = x[j] + mul(al, p[j]);
      const T rj = r[j] - mul(al, q[j]);
      r[j] = rj;
      v[k][0] += norm2(rj);
      if (z) {
        T a[7];
        op.coef(P, b, i, a);
        z[j] = omega * mul(rj, inv_of(a[0]));
      }
    }
  }
  block_partials<BPT>(v, part, b0, nb, gridDim.x);
}

// z_out = z_in + omega (b - A z_in)/a_C ; optional partial b^T z_out
template <int MODE, int BPT>
__global__ void __launch_bounds__(NT) k_smooth(Op<MODE> op, const TT<MODE>* __restrict__ bv,
                                               const TT<MODE>* __restrict__ zin,
                                               TT<MODE>* __restrict__ zout,
                                               const int* __restrict__ active, double omega, int nb,
                                               int dot, double* __restrict__ part) {
  using T = TT<MODE>;
  const size_t n = op.n;
  const size_t i = (size_t)blockIdx.x * NT + threadIdx.x;
  const int b0 = blockIdx.y * BPT;
  double v[BPT][2] = {};
  if (i < n) {
    typename Op<MODE>::Pre P;
    op.pre(i, P);
    Nbr nbr;
    neighbours(i, op.m, nbr);
#pragma unroll
    for (int k = 0; k < BPT; ++k) {
      const int b = b0 + k;
      if (b >= nb) break;
      if (!active[b]) continue;
      const size_t o = (size_t)b * n;
      T a[7];
      op.coef(P, b, i, a);
      const T res = bv[o + i] - apply7(a, zin + o, i, nbr);
      const T zi = zin[o + i] + omega * mul(res, inv_of(a[0]));
      zout[o + i] = zi;
      if (dot) add_dot(v[k], bv[o + i], zi);
    }
  }
  if (dot) block_partials<BPT>(v, part, b0, nb, gridDim.x);
}

// fine node (fx, fy) -> parents in the coarse node grid (mc per side), P1 weights.
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
  const bool ao = a & 1, bo = b & 1;
  if (!ao && !bo) add(a / 2, b / 2, 1.0);
  else if (ao && !bo) { add(a / 2, b / 2, 0.5); add(a / 2 + 1, b / 2, 0.5); }
  else if (!ao && bo) { add(a / 2, b / 2, 0.5); add(a / 2, b / 2 + 1, 0.5); }
  else { add(a / 2, b / 2, 0.5); add(a / 2 + 1, b / 2 + 1, 0.5); }
  return np;
}

// bc = P^T (bf - Af zf) ; optionally zc = omega bc / ac_C (first coarse Jacobi sweep)
template <int MODE, int BPT>
__global__ void __launch_bounds__(NT) k_restrict(Op<MODE> opf, Op<MODE> opc,
                                                 const TT<MODE>* __restrict__ bf,
                                                 const TT<MODE>* __restrict__ zf,
                                                 TT<MODE>* __restrict__ bc, TT<MODE>* __restrict__ zc,
                                                 const int* __restrict__ active, double omega, int nb) {
  using T = TT<MODE>;
  const size_t nc = opc.n, nf = opf.n;
  const int mc = opc.m, mf = opf.m;
  const size_t ic = (size_t)blockIdx.x * NT + threadIdx.x;
  if (ic >= nc) return;
  const int X = (int)(ic % mc), Y = (int)(ic / mc);
  const int sox[7] = {0, -1, 1, 0, 0, -1, 1}, soy[7] = {0, 0, 0, -1, 1, -1, 1};
  const double sw[7] = {1.0, 0.5, 0.5, 0.5, 0.5, 0.5, 0.5};
  const int b0 = blockIdx.y * BPT;
  T acc[BPT];
#pragma unroll
  for (int k = 0; k < BPT; ++k) acc[k] = zero_of(acc[0]);
  for (int s = 0; s < 7; ++s) {
    const int fx = 2 * X + 1 + sox[s], fy = 2 * Y + 1 + soy[s];
    if (fx < 0 || fx >= mf || fy < 0 || fy >= mf) continue;
    const size_t fi = (size_t)fy * mf + fx;
    typename Op<MODE>::Pre P;
    opf.pre(fi, P);
    Nbr nbr;
    neighbours(fi, mf, nbr);
#pragma unroll
    for (int k = 0; k < BPT; ++k) {
      const int b = b0 + k;
      if (b >= nb) break;
      if (!active[b]) continue;
      T a[7];
      opf.coef(P, b, fi, a);
      const size_t o = (size_t)b * nf;
      const T res = bf[o + fi] - apply7(a, zf + o, fi, nbr);
      acc[k] = acc[k] + sw[s] * res;
    }
  }
  typename Op<MODE>::Pre Pc;
  if (zc) opc.pre(ic, Pc);
#pragma unroll
  for (int k = 0; k < BPT; ++k) {
    const int b = b0 + k;
    if (b >= nb) break;
    if (!active[b]) continue;
    bc[(size_t)b * nc + ic] = acc[k];
    if (zc) {
      T a[7];
      opc.coef(Pc, b, ic, a);
      zc[(size_t)b * nc + ic] = omega * mul(acc[k], inv_of(a[0]));
    }
  }
}

// zc = z_in + P xc (node and neighbours), z_out = zc + omega (b - A zc)/a_C
template <int MODE, int BPT>
__global__ void __launch_bounds__(NT) k_prolong_smooth(Op<MODE> op, const TT<MODE>* __restrict__ bv,
                                                       const TT<MODE>* __restrict__ zin,
                                                       const TT<MODE>* __restrict__ xc, int mc,
                                                       TT<MODE>* __restrict__ zout,
                                                       const int* __restrict__ active, double omega,
                                                       int nb, int dot, double* __restrict__ part) {
  using T = TT<MODE>;
  const size_t n = op.n;
  const size_t ncs = (size_t)mc * mc;
  const int m = op.m;
  const size_t i = (size_t)blockIdx.x * NT + threadIdx.x;
  const int b0 = blockIdx.y * BPT;
  double v[BPT][2] = {};
  if (i < n) {
    typename Op<MODE>::Pre P;
    op.pre(i, P);
    Nbr nbr;
    neighbours(i, m, nbr);
    const int x = (int)(i % m), y = (int)(i / m);
    // parents of the node and its neighbours
    int pcx[7][2], pcy[7][2], np[7];
    double pw[7][2];
    for (int d = 0; d < 7; ++d) {
      np[d] = 0;
      if (!nbr.ok[d]) continue;
      np[d] = parents(x + dir_dx(d), y + dir_dy(d), mc, pcx[d], pcy[d], pw[d]);
    }
#pragma unroll
    for (int k = 0; k < BPT; ++k) {
      const int b = b0 + k;
      if (b >= nb) break;
      if (!active[b]) continue;
      const size_t o = (size_t)b * n, oc = (size_t)b * ncs;
      T a[7];
      op.coef(P, b, i, a);
      T Az = zero_of(a[0]), zi = zero_of(a[0]);
#pragma unroll
      for (int d = 0; d < 7; ++d) {
        if (!nbr.ok[d]) continue;
        T zj = zin[o + i + nbr.off[d]];
        for (int t = 0; t < np[d]; ++t) zj = zj + pw[d][t] * xc[oc + (size_t)pcy[d][t] * mc + pcx[d][t]];
        if (d == 0) zi = zj;
        Az = Az + mul(a[d], zj);
      }
      const T bi = bv[o + i];
      const T zo = zi + omega * mul(bi - Az, inv_of(a[0]));
      zout[o + i] = zo;
      if (dot) add_dot(v[k], bi, zo);
    }
  }
  if (dot) block_partials<BPT>(v, part, b0, nb, gridDim.x);
}

// partial b^T z
template <int MODE, int BPT>
__global__ void __launch_bounds__(NT) k_dot(const TT<MODE>* __restrict__ a, const TT<MODE>* __restrict__ z,
                                            size_t n, const int* __restrict__ active, int nb,
                                            double* __restrict__ part) {
  const size_t i = (size_t)blockIdx.x * NT + threadIdx.x;
  const int b0 = blockIdx.y * BPT;
  double v[BPT][2] = {};
  if (i < n)
    for (int k = 0; k < BPT; ++k) {
      const int b = b0 + k;
      if (b >= nb) break;
      if (!active[b]) continue;
      add_dot(v[k], a[(size_t)b * n + i], z[(size_t)b * n + i]);
    }
  block_partials<BPT>(v, part, b0, nb, gridDim.x);
}

// dense coarsest solve x = inv b, one block per batch
template <class T>
__global__ void k_coarse_solve(const T* __restrict__ inv, const T* __restrict__ bc, T* __restrict__ xc,
                               int nL, const int* __restrict__ active) {
  const int b = blockIdx.x;
  if (!active[b]) return;
  const T* A = inv + (size_t)b * nL * nL;
  for (int i = threadIdx.x; i < nL; i += blockDim.x) {
    T acc = zero_of(bc[0]);
    for (int j = 0; j < nL; ++j) acc = acc + mul(A[(size_t)i * nL + j], bc[(size_t)b * nL + j]);
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
                          int* __restrict__ active, int* __restrict__ zero, const int* __restrict__ mask) {
  const int b = blockIdx.x;
  if (b >= nb) return;
  if (stage != ST_INIT && !active[b]) return;
  double s0, s1;
  batch_sum(part, per, b, s0, s1);
  if (threadIdx.x != 0) return;
  switch (stage) {
    case ST_INIT:
      bn2[b] = s0;
      rn2[b] = s1;
      zero[b] = (s0 == 0.0);
      active[b] = (!mask || mask[b]) && (s0 > 0.0) && (s1 > rtol2 * s0);
      break;
    case ST_RHO0:
      rho[b] = from2<T>(s0, s1);
      break;
    case ST_ALPHA: {
      const T m = from2<T>(s0, s1);
      mu[b] = m;
      alpha[b] = cdiv(rho[b], m);
      break;
    }
    case ST_RN:
      rn2[b] = s0;
      active[b] = s0 > rtol2 * bn2[b];
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
    *count = s;
  }
}

// ---- hierarchy construction kernels

__global__ void k_rap(const double* __restrict__ Af, int mf, double* __restrict__ Ac, int mc) {
  const size_t nf = (size_t)mf * mf, nc = (size_t)mc * mc;
  const int b = blockIdx.y;
  const size_t ic = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (ic >= nc) return;
  const double* A = Af + (size_t)b * 7 * nf;
  const int X = (int)(ic % mc), Y = (int)(ic / mc);
  const int sox[7] = {0, -1, 1, 0, 0, -1, 1}, soy[7] = {0, 0, 0, -1, 1, -1, 1};
  const double sw[7] = {1.0, 0.5, 0.5, 0.5, 0.5, 0.5, 0.5};
  double out[7] = {0, 0, 0, 0, 0, 0, 0};
  for (int s = 0; s < 7; ++s) {
    const int fx = 2 * X + 1 + sox[s], fy = 2 * Y + 1 + soy[s];
    if (fx < 0 || fx >= mf || fy < 0 || fy >= mf) continue;
    const size_t fi = (size_t)fy * mf + fx;
    for (int d = 0; d < 7; ++d) {
      const double a = A[d * nf + fi];
      if (a == 0.0) continue;
      const int gx = fx + dir_dx(d), gy = fy + dir_dy(d);
      if (gx < 0 || gx >= mf || gy < 0 || gy >= mf) continue;
      int cx[2], cy[2];
      double w[2];
      const int np = parents(gx, gy, mc, cx, cy, w);
      for (int t = 0; t < np; ++t) {
        const int ex = cx[t] - X, ey = cy[t] - Y;
        int e = -1;
        for (int dd = 0; dd < 7; ++dd)
          if (dir_dx(dd) == ex && dir_dy(dd) == ey) e = dd;
        if (e >= 0) out[e] += sw[s] * a * w[t];
      }
    }
  }
  double* C = Ac + (size_t)b * 7 * nc;
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
  for (int t = threadIdx.x; t < n * n; t += blockDim.x) {
    const int i = t / n, j = t % n;
    inv[(size_t)b * n * n + t] = A[(size_t)i * w + n + j];
  }
}

}  // namespace

void launch_rap(Problem& p, const double* Af, int mf, double* Ac, int mc, int batches) {
  const size_t nc = (size_t)mc * mc;
  dim3 grid((unsigned)((nc + 127) / 128), batches);
  k_rap<<<grid, 128, 0, p.stream>>>(Af, mf, Ac, mc);
  TP_LAUNCHED(&p);
}

template <int MODE>
static void launch_dense_inverse(Problem& p, const double* K, const double* M, int m, const cplx* lam,
                                 TT<MODE>* inv, int batches, size_t strideK) {
  const int n = m * m;
  const size_t smem = (size_t)n * 2 * n * sizeof(TT<MODE>);
  require(smem <= 200 * 1024, "multigrid: coarsest grid too large for the dense solve");
  TP_CUDA(cudaFuncSetAttribute(k_dense_inverse<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_dense_inverse<MODE><<<batches, 256, smem, p.stream>>>(K, M, lam, m, inv, strideK);
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
static constexpr int bpt() { return MODE == 0 ? 4 : 1; }

template <int MODE>
static Op<MODE> make_op(const LevelOp& L, const cplx* lam);
template <>
Op<0> make_op<0>(const LevelOp& L, const cplx* lam) {
  return Op<0>{L.K, L.M, lam, (size_t)L.n, L.m};
}
template <>
Op<1> make_op<1>(const LevelOp& L, const cplx*) {
  return Op<1>{L.K, (size_t)L.n, L.m};
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
  const size_t n0 = (size_t)B * levels[0].n;
  r.alloc(n0);
  p0.alloc(n0);
  p1.alloc(n0);
  q.alloc(n0);
  const size_t per = (levels[0].n + NT - 1) / NT;
  part.alloc((size_t)B * per * 2 + 64);
  rho.alloc(B);
  mu.alloc(B);
  alpha.alloc(B);
  beta.alloc(B);
  bn2.alloc(B);
  rn2.alloc(B);
  active.alloc(2 * B);
  count.alloc(2);
  if (!h_count) TP_CUDA(cudaMallocHost(reinterpret_cast<void**>(&h_count), 2 * sizeof(int)));
  for (auto& e : ev)
    if (!e) TP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
}

template <int MODE>
BatchSolver<MODE>::~BatchSolver() {
  if (h_count) cudaFreeHost(h_count);
  for (auto& e : ev)
    if (e) cudaEventDestroy(e);
}

namespace {
template <int MODE, int BPT>
__global__ void __launch_bounds__(NT) k_jacobi0(Op<MODE> op, const TT<MODE>* __restrict__ bv,
                                                TT<MODE>* __restrict__ z, const int* __restrict__ active,
                                                double omega, int nb) {
  using T = TT<MODE>;
  const size_t n = op.n;
  const size_t i = (size_t)blockIdx.x * NT + threadIdx.x;
  if (i >= n) return;
  typename Op<MODE>::Pre P;
  op.pre(i, P);
  for (int k = 0; k < BPT; ++k) {
    const int b = blockIdx.y * BPT + k;
    if (b >= nb) break;
    if (!active[b]) continue;
    T a[7];
    op.coef(P, b, i, a);
    z[(size_t)b * n + i] = omega * mul(bv[(size_t)b * n + i], inv_of(a[0]));
  }
}
}  // namespace

template <int MODE>
typename BatchSolver<MODE>::T* BatchSolver<MODE>::vcycle_level(int l, int nb, const T* bl, T* /*unused*/,
                                                              bool /*unused*/, bool dot) {
  constexpr int K = bpt<MODE>();
  const int L = (int)ops.size();
  const Op<MODE> op = make_op<MODE>(ops[l], lam);
  const size_t n = ops[l].n;
  dim3 g((unsigned)((n + NT - 1) / NT), (unsigned)((nb + K - 1) / K));
  int* act = active.get();
  if (L == 1) {
    k_coarse_solve<T><<<nb, 64, 0, p->stream>>>(coarse_inv, bl, lz0[0].get(), ops[0].n, act);
    TP_LAUNCHED(p);
    if (dot) {
      k_dot<MODE, K><<<g, NT, 0, p->stream>>>(bl, lz0[0].get(), n, act, nb, part.get());
      TP_LAUNCHED(p);
    }
    return lz0[0].get();
  }
  T* z = lz0[l].get();
  T* o = lz1[l].get();
  for (int s = 1; s < cfg.pre; ++s) {
    k_smooth<MODE, K><<<g, NT, 0, p->stream>>>(op, bl, z, o, act, cfg.omega, nb, 0, part.get());
    TP_LAUNCHED(p);
    std::swap(z, o);
  }
  const bool coarse_next = (l + 1 == L - 1);
  const Op<MODE> opc = make_op<MODE>(ops[l + 1], lam);
  const size_t nc = ops[l + 1].n;
  dim3 gc((unsigned)((nc + NT - 1) / NT), (unsigned)((nb + K - 1) / K));
  k_restrict<MODE, K><<<gc, NT, 0, p->stream>>>(op, opc, bl, z, lb[l + 1].get(),
                                                 coarse_next ? nullptr : lz0[l + 1].get(), act,
                                                 cfg.omega, nb);
  TP_LAUNCHED(p);
  T* xc;
  if (coarse_next) {
    k_coarse_solve<T><<<nb, 64, 0, p->stream>>>(coarse_inv, lb[l + 1].get(), lz0[l + 1].get(),
                                                ops[l + 1].n, act);
    TP_LAUNCHED(p);
    xc = lz0[l + 1].get();
  } else {
    xc = vcycle_level(l + 1, nb, lb[l + 1].get(), nullptr, false, false);
  }
  k_prolong_smooth<MODE, K><<<g, NT, 0, p->stream>>>(op, bl, z, xc, ops[l + 1].m, o, act, cfg.omega,
                                                     nb, (dot && cfg.post == 1) ? 1 : 0, part.get());
  TP_LAUNCHED(p);
  std::swap(z, o);
  for (int s = 1; s < cfg.post; ++s) {
    const int d = (dot && s == cfg.post - 1) ? 1 : 0;
    k_smooth<MODE, K><<<g, NT, 0, p->stream>>>(op, bl, z, o, act, cfg.omega, nb, d, part.get());
    TP_LAUNCHED(p);
    std::swap(z, o);
  }
  return z;
}

template <int MODE>
int BatchSolver<MODE>::solve(const T* b, T* x, int nb, bool warm, SolveStats* st) {
  constexpr int K = bpt<MODE>();
  require(nb <= B, "batch solver: too many right-hand sides");
  const Op<MODE> op0 = make_op<MODE>(ops[0], lam);
  const size_t n0 = ops[0].n;
  dim3 g0((unsigned)((n0 + NT - 1) / NT), (unsigned)((nb + K - 1) / K));
  const int per0 = (int)g0.x;
  const double rtol2 = cfg.rtol * cfg.rtol;
  int* act = active.get();
  int* zero = active.get() + B;
  cudaStream_t s = p->stream;
  k_init<MODE, K><<<g0, NT, 0, s>>>(op0, b, x, r.get(), nb, warm ? 1 : 0, part.get());
  TP_LAUNCHED(p);
  k_scalars<T><<<nb, 256, 0, s>>>(ST_INIT, part.get(), per0, nb, rtol2, rho.get(), mu.get(),
                                  alpha.get(), beta.get(), bn2.get(), rn2.get(), act, zero, ext_mask);
  TP_LAUNCHED(p);
  if (warm) {
    k_zero_flagged<MODE, K><<<g0, NT, 0, s>>>(x, n0, nb, zero);
    TP_LAUNCHED(p);
  }
  k_count_active<<<1, 256, 0, s>>>(act, nb, count.get());
  TP_LAUNCHED(p);
  TP_CUDA(cudaMemcpyAsync(h_count, count.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  TP_CUDA(cudaStreamSynchronize(s));
  int iters = 0;
  int64_t batch_iters = 0;
  int last_active = h_count[0];
  if (last_active > 0) {
    k_jacobi0<MODE, K><<<g0, NT, 0, s>>>(op0, r.get(), lz0[0].get(), act, cfg.omega, nb);
    TP_LAUNCHED(p);
    T* z = vcycle_level(0, nb, r.get(), nullptr, false, true);
    k_scalars<T><<<nb, 256, 0, s>>>(ST_RHO0, part.get(), per0, nb, rtol2, rho.get(), mu.get(),
                                    alpha.get(), beta.get(), bn2.get(), rn2.get(), act, zero, ext_mask);
    TP_LAUNCHED(p);
    T* pin = p0.get();
    T* pout = p1.get();
    bool done = false;
    for (int it = 1; it <= cfg.max_iter; ++it) {
      k_apply_dot<MODE, K><<<g0, NT, 0, s>>>(op0, z, pin, pout, q.get(), beta.get(), act,
                                             it == 1 ? 1 : 0, nb, part.get());
      TP_LAUNCHED(p);
      k_scalars<T><<<nb, 256, 0, s>>>(ST_ALPHA, part.get(), per0, nb, rtol2, rho.get(), mu.get(),
                                      alpha.get(), beta.get(), bn2.get(), rn2.get(), act, zero, ext_mask);
      TP_LAUNCHED(p);
      k_update<MODE, K><<<g0, NT, 0, s>>>(op0, x, r.get(), pout, q.get(), alpha.get(), act,
                                          cfg.omega, ops.size() > 1 ? lz0[0].get() : nullptr, nb,
                                          part.get());
      TP_LAUNCHED(p);
      k_scalars<T><<<nb, 256, 0, s>>>(ST_RN, part.get(), per0, nb, rtol2, rho.get(), mu.get(),
                                      alpha.get(), beta.get(), bn2.get(), rn2.get(), act, zero, ext_mask);
      TP_LAUNCHED(p);
      const int slot = it & 1;
      k_count_active<<<1, 256, 0, s>>>(act, nb, count.get() + slot);
      TP_LAUNCHED(p);
      TP_CUDA(cudaMemcpyAsync(h_count + slot, count.get() + slot, sizeof(int), cudaMemcpyDeviceToHost, s));
      TP_CUDA(cudaEventRecord(ev[slot], s));
      batch_iters += last_active;
      if (it >= 2) {
        TP_CUDA(cudaEventSynchronize(ev[slot ^ 1]));
        last_active = h_count[slot ^ 1];
        if (last_active == 0) {
          iters = it - 1;
          batch_iters -= 0;
          done = true;
          break;
        }
      }
      iters = it;
      z = vcycle_level(0, nb, r.get(), nullptr, false, true);
      k_scalars<T><<<nb, 256, 0, s>>>(ST_BETA, part.get(), per0, nb, rtol2, rho.get(), mu.get(),
                                      alpha.get(), beta.get(), bn2.get(), rn2.get(), act, zero, ext_mask);
      TP_LAUNCHED(p);
      std::swap(pin, pout);
    }
    if (!done) {
      TP_CUDA(cudaStreamSynchronize(s));
      last_active = h_count[iters & 1];
    }
  }
  TP_CUDA(cudaStreamSynchronize(s));
  std::vector<double> hb(nb), hr(nb);
  TP_CUDA(cudaMemcpy(hb.data(), bn2.get(), nb * sizeof(double), cudaMemcpyDeviceToHost));
  TP_CUDA(cudaMemcpy(hr.data(), rn2.get(), nb * sizeof(double), cudaMemcpyDeviceToHost));
  double worst = 0;
  for (int k = 0; k < nb; ++k)
    if (hb[k] > 0) worst = std::max(worst, std::sqrt(hr[k] / hb[k]));
  if (st) {
    st->iterations = std::max(st->iterations, iters);
    st->batch_iterations += batch_iters;
    st->max_rel_residual = std::max(st->max_rel_residual, worst);
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
