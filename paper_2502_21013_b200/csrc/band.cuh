// Banded LDL^T kernels of the general-mesh path (mesh.cu): the direct block
// solves that stand in for the reference's cached sparse factorisations
// (PeriodicSolver, periodic.hpp:211-248; newton_elliptic's SparseSolver,
// solvers.hpp:156).  Complex symmetric blocks are factorised without
// conjugation (periodic.hpp:124), like the reference's complex LDL^T.
//
// Band layout: row r of a block holds columns r-bw .. r at offsets 0 .. bw
// (diagonal at bw), W = bw+1 entries per row, blocks back to back.
#pragma once

#include "tp_internal.cuh"

namespace tpgpu {
namespace band {

__device__ __forceinline__ double mulv(double a, double b) { return a * b; }
__device__ __forceinline__ cplx mulv(cplx a, cplx b) { return a * b; }
__device__ __forceinline__ double divv(double a, double b) { return a / b; }
__device__ __forceinline__ cplx divv(cplx a, cplx b) { return cdiv(a, b); }
__device__ __forceinline__ bool is_zero(double a) { return a == 0.0; }
__device__ __forceinline__ bool is_zero(cplx a) { return a.re == 0.0 && a.im == 0.0; }
__device__ __forceinline__ double shfl(double v, int l) { return __shfl_sync(0xffffffffu, v, l); }
__device__ __forceinline__ cplx shfl(cplx v, int l) { return {shfl(v.re, l), shfl(v.im, l)}; }
// a - b c
__device__ __forceinline__ double fnma(double b, double c, double a) { return fma(-b, c, a); }
__device__ __forceinline__ cplx fnma(cplx b, cplx c, cplx a) {
  return {fma(-b.re, c.re, fma(b.im, c.im, a.re)), fma(-b.re, c.im, fma(-b.im, c.re, a.im))};
}

template <int BYTES>
__device__ __forceinline__ void cpa(void* sdst, const void* g, bool ok) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  if constexpr (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(g), "r"(ok ? 16 : 0));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(g), "r"(ok ? 8 : 0));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// ---------------------------------------------------------------- factorisation
// Right-looking band LDL^T, one block per CTA.  Step c: multipliers
// l_i = a_ic / d_c (i = c+1 .. c+bw), trailing triangle a_ik -= l_i a_kc.
// RING: the active rows c .. c+bw live in a shared-memory ring (slot r % W);
// row c is written back once final and row c+W loaded in its slot.  Without
// RING the window is updated in global memory (large bandwidths).
// A zero pivot sets *fail.
template <class T, bool RING>
__global__ void __launch_bounds__(512) k_factor(T* __restrict__ bandp, int n, int bw, const int* __restrict__ on,
                                                int* __restrict__ fail) {
  const int b = blockIdx.x;
  if (on && !on[b]) return;
  const int W = bw + 1;
  T* A = bandp + (size_t)b * n * W;
  extern __shared__ __align__(16) unsigned char fsm[];
  T* col = reinterpret_cast<T*>(fsm);  // bw: a_{c+1+a, c}
  T* lsc = col + bw;                   // bw: l_{c+1+a}
  T* ring = lsc + bw;                  // RING: W x W
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  if (RING)
    for (int idx = threadIdx.x; idx < min(W, n) * W; idx += blockDim.x) ring[idx] = A[idx];
  __syncthreads();
  auto at = [&](int r, int off) -> T& { return RING ? ring[(r % W) * W + off] : A[(size_t)r * W + off]; };
  for (int c = 0; c < n; ++c) {
    const T d = at(c, bw);
    const int len = min(bw, n - 1 - c);
    for (int a = threadIdx.x; a < len; a += blockDim.x) {
      const T v = at(c + 1 + a, bw - 1 - a);
      col[a] = v;
      lsc[a] = divv(v, d);
    }
    if (threadIdx.x == 0 && is_zero(d)) bad = 1;
    __syncthreads();
    if (bad) break;
    for (int idx = threadIdx.x; idx < len * len; idx += blockDim.x) {
      const int a = idx / len, q = idx - a * len;
      if (q > a) continue;
      T& x = at(c + 1 + a, bw - (a - q));
      x = x - mulv(lsc[a], col[q]);
    }
    for (int a = threadIdx.x; a < len; a += blockDim.x) at(c + 1 + a, bw - 1 - a) = lsc[a];
    __syncthreads();
    if (RING) {
      // row c is final: write it back, bring row c+W into its slot
      const int sl = (c % W) * W;
      for (int q = threadIdx.x; q < W; q += blockDim.x) {
        A[(size_t)c * W + q] = ring[sl + q];
        if (c + W < n) ring[sl + q] = A[(size_t)(c + W) * W + q];
      }
      __syncthreads();
    }
  }
  if (threadIdx.x == 0 && bad) atomicExch(fail, 1);
}

// ---------------------------------------------------------------- solve
// x = (L D L^T)^-1 b, one warp per block, S = 1 + ceil(bw / 32) register
// slots per lane.  Both triangular sweeps are column-oriented over 32-column
// chunks: the unknowns of the active window stay in registers (lane l, slot s
// holds row base + 32 s + l, resp. base - 32 s + l going up), the final value
// of column c is broadcast with one shuffle, and every lane applies its
// column coefficients -- staged per chunk in shared memory by cp.async
// (zero-filled outside the band, so no predicates), NB buffers deep -- so the
// dependency chain per row is one shuffle and one fused multiply-add.
// gather: b = src[perm[p]]; scatter: dst[perm[p]] = x_p.  The forward result
// y / D is kept in shared memory (ysm) or in gscratch.
template <class T, int S, int NB>
__global__ void __launch_bounds__(32) k_solve(const T* __restrict__ bandp, const T* __restrict__ src,
                                              T* __restrict__ dst, const int* __restrict__ perm, int n, int bw,
                                              const int* __restrict__ on, T* __restrict__ gscratch) {
  const int b = blockIdx.x;
  if (on && !on[b]) return;
  constexpr int CH = 32 * S * 33;  // staged coefficients per chunk (forward rows padded to 33)
  const int lane = threadIdx.x;
  const int W = bw + 1;
  extern __shared__ __align__(16) unsigned char ssm[];
  T* stage = reinterpret_cast<T*>(ssm);
  T* y = gscratch ? gscratch + (size_t)b * n : stage + NB * CH;
  const T* A = bandp + (size_t)b * n * W;
  const T* s_ = src + (size_t)b * n;
  const int nch = (n + 31) >> 5;
  // forward stage of chunk base c: entry (ro, u) = L[c+ro][c+u] at
  // A + c W + bw + u + ro bw, valid for 0 < ro-u <= bw and c+ro < n (rows
  // padded to 33 entries: the compute loop reads a column across lanes)
  auto fwd_copy = [&](T* st, int c, int ro) {
    const int hi = min(lane + bw, n - 1 - c);
    const bool ok = ro > lane && ro <= hi;
    cpa<sizeof(T)>(&st[ro * 33 + lane], ok ? A + (size_t)c * W + bw + lane + (size_t)ro * bw : A, ok);
  };
  auto stage_fwd = [&](int m, T* st) {
#pragma unroll 4
    for (int ro = 0; ro < 32 * S; ++ro) fwd_copy(st, m << 5, ro);
    cpa_commit();
  };
  // backward stage of chunk base c: entry (u, s, l) = L[c+u][c-32s+l] at
  // A + c W + bw + l + u bw - 32 s, valid for 0 < u+32s-l <= bw, c+u < n, c-32s+l >= 0
  auto bwd_copy = [&](T* st, int c, int u, int s) {
    const int d = u + 32 * s - lane;
    const bool ok = d > 0 && d <= bw && c + u < n && c - 32 * s + lane >= 0;
    cpa<sizeof(T)>(&st[(u * S + s) * 32 + lane],
                   ok ? A + (size_t)c * W + bw + lane + (size_t)u * bw - 32 * s : A, ok);
  };
  auto stage_bwd = [&](int m, T* st) {
#pragma unroll 4
    for (int us = 0; us < 32 * S; ++us) bwd_copy(st, m << 5, us / S, us % S);
    cpa_commit();
  };
  T win[S];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int r = 32 * s + lane;
    win[s] = r < n ? s_[perm[r]] : T{};
  }
  // ---- forward: L y = b, then y / D.  The next chunk's coefficients are
  // staged while this chunk computes: its cp.async copies are issued inside
  // the u loop (S per step), filling the shuffle latency of the chain; the
  // values needed at the chunk end (D, the next right-hand-side rows) are
  // loaded at the chunk start.
  stage_fwd(0, stage);
  int pn = 32 * S + lane < n ? perm[32 * S + lane] : 0;  // perm of the row entering after chunk 0
  for (int m = 0; m < nch; ++m) {
    T* st = stage + (NB > 1 ? (m & 1) * CH : 0);
    T* nx = stage + (NB > 1 ? ((m + 1) & 1) * CH : 0);
    const int c0 = m << 5, r = c0 + lane, rn = c0 + 32 * S + lane;
    const T dg = r < n ? A[(size_t)r * W + bw] : T{};
    const T bn = rn < n ? s_[pn] : T{};
    pn = rn + 32 < n ? perm[rn + 32] : 0;
    cpa_wait<0>();
    __syncwarp();
    const bool pre = NB > 1 && m + 1 < nch;
    const int c1 = c0 + 32;
    if (pre) {
#pragma unroll
      for (int u = 0; u < 32; ++u) {
        const T yc = shfl(win[0], u);
#pragma unroll
        for (int s = 0; s < S; ++s) win[s] = fnma(st[(32 * s + lane) * 33 + u], yc, win[s]);
#pragma unroll
        for (int s = 0; s < S; ++s) fwd_copy(nx, c1, 32 * s + u);
      }
      cpa_commit();
    } else {
#pragma unroll
      for (int u = 0; u < 32; ++u) {
        const T yc = shfl(win[0], u);
#pragma unroll
        for (int s = 0; s < S; ++s) win[s] = fnma(st[(32 * s + lane) * 33 + u], yc, win[s]);
      }
    }
    if (r < n) y[r] = divv(win[0], dg);
#pragma unroll
    for (int s = 0; s + 1 < S; ++s) win[s] = win[s + 1];
    win[S - 1] = bn;
    __syncwarp();
    if (NB == 1 && m + 1 < nch) stage_fwd(m + 1, st);
  }
  __syncwarp();
  // ---- backward: L^T x = y / D, chunks from the last down
  const int mt = nch - 1;
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int r = (mt << 5) - 32 * s + lane;
    win[s] = (r >= 0 && r < n) ? y[r] : T{};
  }
  cpa_wait<0>();
  __syncwarp();
  stage_bwd(mt, stage);
  T* d_ = dst + (size_t)b * n;
  for (int m = mt, i = 0; m >= 0; --m, ++i) {
    T* st = stage + (NB > 1 ? (i & 1) * CH : 0);
    T* nx = stage + (NB > 1 ? ((i + 1) & 1) * CH : 0);
    const int c0 = m << 5, r = c0 + lane, rn = c0 - 32 * S + lane;
    const int pr = r < n ? perm[r] : 0;
    const T yn = rn >= 0 ? y[rn] : T{};
    cpa_wait<0>();
    __syncwarp();
    const bool pre = NB > 1 && m > 0;
    const int c1 = c0 - 32;
    if (pre) {
#pragma unroll
      for (int u = 31; u >= 0; --u) {
        const T xc = shfl(win[0], u);
#pragma unroll
        for (int s = 0; s < S; ++s) win[s] = fnma(st[(u * S + s) * 32 + lane], xc, win[s]);
#pragma unroll
        for (int s = 0; s < S; ++s) bwd_copy(nx, c1, u, s);
      }
      cpa_commit();
    } else {
#pragma unroll
      for (int u = 31; u >= 0; --u) {
        const T xc = shfl(win[0], u);
#pragma unroll
        for (int s = 0; s < S; ++s) win[s] = fnma(st[(u * S + s) * 32 + lane], xc, win[s]);
      }
    }
    if (r < n) d_[pr] = win[0];
#pragma unroll
    for (int s = 0; s + 1 < S; ++s) win[s] = win[s + 1];
    win[S - 1] = yn;
    __syncwarp();
    if (NB == 1 && m - 1 >= 0) stage_bwd(m - 1, st);
  }
}

}  // namespace band
}  // namespace tpgpu
