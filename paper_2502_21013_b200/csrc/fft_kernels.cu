// Time-axis DFTs of the periodic solve (reference: PeriodicSolver::solve,
// periodic.hpp:159-198, and DftPlan, fft.hpp:19-99).
//
// Forward: G (N x n, slice-major, real) -> Ghat (K x n, frequency-major,
// K = N/2+1 half spectrum; X_k = sum_i g_i e^{-2 pi i ik/N}, unnormalised).
// Inverse: Uhat (K x n) -> U (N x n), x_i = (1/N) sum_k X_k e^{+2 pi i ik/N}
// over the Hermitian extension X_{N-k} = conj(X_k) -- the reference's
// conjugate mirroring (periodic.hpp:285-288) made implicit.
//
// A block owns C = 2P consecutive dof columns and all N slices: the slice
// rows are read/written as C contiguous doubles (coalesced), two real columns
// are packed into one complex column, and each column is transformed in
// shared memory by the reference's own iterative radix-2 DIT (bit-reversed
// load, len = 2..N butterflies, fft.hpp:61-79) or, for non-power-of-two N, the
// direct O(N^2) transform (fft.hpp:81-93).
//
// The inverse also returns the partial sums behind the reference's
// imaginary-residue guard (periodic.hpp:172-196): sum Re^2 and the imaginary
// energy (Im X_0^2 + Im X_{N/2}^2)/N that the full complex inverse would
// produce.
#include <cmath>
#include <cstdlib>
#include <numbers>

#include "tp_internal.cuh"

namespace tpgpu {

namespace {

__device__ __forceinline__ int bitrev(int i, int bits) { return __brev(i) >> (32 - bits); }

__device__ __forceinline__ cplx cmul(cplx a, cplx b) {
  return {fma(a.re, b.re, -a.im * b.im), fma(a.re, b.im, a.im * b.re)};
}

__device__ __forceinline__ void acp8(void* sdst, const void* g, bool ok) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(g), "r"(ok ? 8 : 0) : "memory");
}
__device__ __forceinline__ void acp16(void* sdst, const void* g, bool ok) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(g), "r"(ok ? 16 : 0) : "memory");
}
__device__ __forceinline__ void acp_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// block sum of v into *out (thread 0); blockDim.x a multiple of 32
__device__ __forceinline__ void block_sum_to(double v, double* out) {
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    *out = t;
  }
}

template <bool INVERSE>
__device__ void transform(cplx* z, cplx* tmp, const cplx* __restrict__ tw, int N, int P, bool pow2) {
  const int tid = threadIdx.x, nt = blockDim.x;
  if (pow2) {
    for (int len = 2; len <= N; len <<= 1) {
      const int half = len >> 1, stride = N / len;
      for (int t = tid; t < P * (N >> 1); t += nt) {
        const int p = t / (N >> 1), bi = t % (N >> 1);
        const int base = (bi / half) * len, k = bi % half;
        cplx w = tw[k * stride];
        if (INVERSE) w.im = -w.im;
        cplx* a = z + (size_t)p * N;
        const cplx odd = cmul(a[base + k + half], w);
        const cplx even = a[base + k];
        a[base + k] = even + odd;
        a[base + k + half] = even - odd;
      }
      __syncthreads();
    }
  } else {
    for (int t = tid; t < P * N; t += nt) {
      const int p = t / N, k = t % N;
      const cplx* a = z + (size_t)p * N;
      cplx acc{0, 0};
      for (int j = 0; j < N; ++j) {
        cplx w = tw[(int)(((long long)k * j) % N)];
        if (INVERSE) w.im = -w.im;
        acc = acc + cmul(a[j], w);
      }
      tmp[(size_t)p * N + k] = acc;
    }
    __syncthreads();
    for (int t = tid; t < P * N; t += nt) z[t] = tmp[t];
    __syncthreads();
  }
}

__global__ void k_rdft_forward(const double* __restrict__ G, cplx* __restrict__ Ghat, size_t n, int N,
                               int P, int bits, int pow2, const cplx* __restrict__ tw,
                               double* __restrict__ sq, const int* __restrict__ kslot) {
  extern __shared__ cplx smem[];
  cplx* z = smem;
  cplx* tmp = smem + (size_t)P * N;
  const int C = 2 * P;
  const size_t j0 = (size_t)blockIdx.x * C;
  for (int t = threadIdx.x; t < N * C; t += blockDim.x) {
    const int i = t / C, cc = t % C;
    const double v = (j0 + cc < n) ? G[(size_t)i * n + j0 + cc] : 0.0;
    const int pos = pow2 ? bitrev(i, bits) : i;
    double* zp = reinterpret_cast<double*>(&z[(size_t)(cc >> 1) * N + pos]);
    zp[cc & 1] = v;
  }
  __syncthreads();
  transform<false>(z, tmp, tw, N, P, pow2);
  const int K = N / 2 + 1;
  double e = 0;
  for (int t = threadIdx.x; t < K * C; t += blockDim.x) {
    const int k = t / C, cc = t % C;
    if (j0 + cc >= n) continue;
    const cplx* a = z + (size_t)(cc >> 1) * N;
    const cplx Zk = a[k], Zm = conj(a[(N - k) % N]);
    cplx X;
    if ((cc & 1) == 0) X = {0.5 * (Zk.re + Zm.re), 0.5 * (Zk.im + Zm.im)};
    else X = {0.5 * (Zk.im - Zm.im), -0.5 * (Zk.re - Zm.re)};
    Ghat[(size_t)(kslot ? kslot[k] : k) * n + j0 + cc] = X;
    e = fma(X.re, X.re, fma(X.im, X.im, e));
  }
  if (sq) block_sum_to(e, sq + blockIdx.x);
}

__global__ void k_rdft_inverse(const cplx* __restrict__ Uhat, double* __restrict__ U, size_t n, int N,
                               int P, int bits, int pow2, const cplx* __restrict__ tw,
                               double* __restrict__ part, const int* __restrict__ kslot) {
  extern __shared__ cplx smem[];
  __shared__ double red[2][32];
  cplx* z = smem;
  cplx* tmp = smem + (size_t)P * N;
  const int C = 2 * P;
  const size_t j0 = (size_t)blockIdx.x * C;
  const int half = N / 2;
  const bool even = (N % 2) == 0;
  double im2 = 0;
  for (int t = threadIdx.x; t < N * P; t += blockDim.x) {
    const int k = t / P, p = t % P;
    const size_t ja = j0 + 2 * p, jb = ja + 1;
    cplx Xa{0, 0}, Xb{0, 0};
    const int kk = (k <= half) ? k : N - k;
    const size_t row = (size_t)(kslot ? kslot[kk] : kk) * n;
    if (ja < n) Xa = Uhat[row + ja];
    if (jb < n) Xb = Uhat[row + jb];
    cplx Z;
    if (k == 0 || (even && k == half)) {
      // self-conjugate bins: the real parts form the Hermitian spectrum; the
      // imaginary parts are what the full inverse would leave as Im(u)
      Z = {Xa.re, Xb.re};
      im2 += (Xa.im * Xa.im + Xb.im * Xb.im) / N;
    } else if (k <= half) {
      Z = {Xa.re - Xb.im, Xa.im + Xb.re};
    } else {
      Z = {Xa.re + Xb.im, -Xa.im + Xb.re};
    }
    z[(size_t)p * N + (pow2 ? bitrev(k, bits) : k)] = Z;
  }
  __syncthreads();
  transform<true>(z, tmp, tw, N, P, pow2);
  const double invN = 1.0 / N;
  double re2 = 0;
  for (int t = threadIdx.x; t < N * C; t += blockDim.x) {
    const int i = t / C, cc = t % C;
    if (j0 + cc >= n) continue;
    const cplx v = z[(size_t)(cc >> 1) * N + i];
    const double x = ((cc & 1) == 0 ? v.re : v.im) * invN;
    U[(size_t)i * n + j0 + cc] = x;
    re2 += x * x;
  }
  for (int o = 16; o > 0; o >>= 1) {
    re2 += __shfl_down_sync(0xffffffffu, re2, o);
    im2 += __shfl_down_sync(0xffffffffu, im2, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = re2;
    red[1][threadIdx.x >> 5] = im2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0, b = 0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) {
      a += red[0][w];
      b += red[1][w];
    }
    part[2 * blockIdx.x] = a;
    part[2 * blockIdx.x + 1] = b;
  }
}

// ------------------------------------------------------------------ Stockham
// Power-of-two N >= 16: self-sorting Stockham passes of radix 16 (then one
// pass of radix 2, 4 or 8 for the rest of N), each an in-register R-point DFT
// between one shared-memory load and one store, instead of log2(N) radix-2
// passes through shared memory.  Columns are interleaved in shared memory
// (z[pos * P + p]) so a warp's accesses of one pass hit consecutive 16-byte
// words.  Every thread holds 16 values per pass (T = P N / 16 threads):
// load, barrier, twiddle + DFT + store, barrier -- in place.
// Same transform as the reference's DftPlan (unnormalised forward, 1/N
// inverse, fft.hpp:61-99) up to rounding.
__constant__ double kC16[16] = {1.0,
                                0.92387953251128673848,
                                0.70710678118654752440,
                                0.38268343236508977173,
                                0.0,
                                -0.38268343236508977173,
                                -0.70710678118654752440,
                                -0.92387953251128673848,
                                -1.0,
                                -0.92387953251128673848,
                                -0.70710678118654752440,
                                -0.38268343236508977173,
                                0.0,
                                0.38268343236508977173,
                                0.70710678118654752440,
                                0.92387953251128673848};

// Shared layout of the Stockham columns: complex entry e = pos * P + p lives
// at zx(e) = e + e / 64 -- one 16-byte pad per kilobyte, so the first pass's
// stores (stride R P entries between the lanes of a warp) spread over the
// banks instead of hitting the same 64 bytes eight times (ncu at cfg 3: 52 %
// of the forward's shared stores were bank conflicts without it).
#ifndef TPGPU_FFT_PAD
#define TPGPU_FFT_PAD 1
#endif
__device__ __forceinline__ int zx(int e) { return TPGPU_FFT_PAD ? e + (e >> 6) : e; }
__host__ __device__ constexpr int zx_size(int e) { return TPGPU_FFT_PAD ? e + (e >> 6) + 1 : e; }

template <int R>
__device__ __forceinline__ constexpr int rev_bits(int i) {
  int r = 0;
  for (int b = 1; b < R; b <<= 1) {
    r = (r << 1) | (i & 1);
    i >>= 1;
  }
  return r;
}

// in-register R-point DFT, natural order in and out (radix-2 DIT)
template <int R, bool INV>
__device__ __forceinline__ void dft_reg(cplx (&v)[R]) {
  cplx t[R];
#pragma unroll
  for (int i = 0; i < R; ++i) t[i] = v[rev_bits<R>(i)];
  constexpr int LOG = R == 2 ? 1 : R == 4 ? 2 : R == 8 ? 3 : 4;
#pragma unroll
  for (int st = 0; st < LOG; ++st) {
    const int len = 2 << st;
#pragma unroll
    for (int i = 0; i < R; i += len) {
#pragma unroll
      for (int k = 0; k < len / 2; ++k) {
        const cplx a = t[i + k];
        cplx b = t[i + k + len / 2];
        if (k != 0) {
          // exp(-+2 pi i k / len) = cos - +i sin, from the 16-entry table
          const int m = k * (16 / len);
          const double c = kC16[m], sn = kC16[(m + 12) & 15];  // sin(x) = cos(x - pi/2)
          const cplx w = {c, INV ? sn : -sn};
          b = cmul(b, w);
        }
        t[i + k] = a + b;
        t[i + k + len / 2] = a - b;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < R; ++i) v[i] = t[i];
}

template <int R, bool INV>
__device__ __forceinline__ void stockham_pass(cplx* z, const cplx* tw, int N, int P, int Ns, int T) {
  constexpr int B = 16 / R;  // butterflies per thread
  cplx v[B][R];
  const int NR = N / R;
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const int t = threadIdx.x + b * T, p = t % P, j = t / P;
#pragma unroll
    for (int r = 0; r < R; ++r) v[b][r] = z[zx((j + r * NR) * P + p)];
  }
  __syncthreads();
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const int t = threadIdx.x + b * T, p = t % P, j = t / P;
    const int k = j % Ns;
    if (Ns > 1) {
      const int step = k * (N / (Ns * R));
#pragma unroll
      for (int r = 1; r < R; ++r) {
        cplx w = tw[r * step];
        if (INV) w.im = -w.im;
        v[b][r] = cmul(v[b][r], w);
      }
    }
    dft_reg<R, INV>(v[b]);
    const int base = (j / Ns) * Ns * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) z[zx((base + r * Ns) * P + p)] = v[b][r];
  }
  __syncthreads();
}

template <bool INV>
__device__ void stockham(cplx* z, const cplx* tw, int N, int P) {
  const int T = blockDim.x;
  int Ns = 1;
  while (Ns * 16 <= N) {
    stockham_pass<16, INV>(z, tw, N, P, Ns, T);
    Ns *= 16;
  }
  const int rest = N / Ns;
  if (rest == 8) stockham_pass<8, INV>(z, tw, N, P, Ns, T);
  else if (rest == 4) stockham_pass<4, INV>(z, tw, N, P, Ns, T);
  else if (rest == 2) stockham_pass<2, INV>(z, tw, N, P, Ns, T);
}

// shared layout: twiddles W_N^m (N), then the P interleaved columns (P N)
__global__ void __launch_bounds__(512) k_sfft_forward(const double* __restrict__ G, cplx* __restrict__ Ghat, size_t n, int N, int P,
                               const cplx* __restrict__ tw, double* __restrict__ sq,
                               const int* __restrict__ kslot) {
  extern __shared__ cplx smem[];
  cplx* tws = smem;
  cplx* z = smem + N;
  const int C = 2 * P;
  const size_t j0 = (size_t)blockIdx.x * C;
  // all loads in flight at once (cp.async, zero-fill past the last column)
  for (int t = threadIdx.x; t < N; t += blockDim.x) acp16(&tws[t], &tw[t], true);
  double* zd = reinterpret_cast<double*>(z);
  for (int t = threadIdx.x; t < N * C; t += blockDim.x) {
    const int i = t / C, cc = t - i * C;
    const bool ok = j0 + cc < n;
    acp8(&zd[2 * zx(i * P + (cc >> 1)) + (cc & 1)], G + (ok ? (size_t)i * n + j0 + cc : 0), ok);  // z[i P + cc/2].{re,im}
  }
  acp_wait_all();
  __syncthreads();
  stockham<false>(z, tws, N, P);
  const int K = N / 2 + 1;
  double e = 0;
  for (int t = threadIdx.x; t < K * C; t += blockDim.x) {
    const int k = t / C, cc = t - k * C;
    if (j0 + cc >= n) continue;
    const int p = cc >> 1;
    const cplx Zk = z[zx(k * P + p)], Zm = conj(z[zx(((N - k) % N) * P + p)]);
    cplx X;
    if ((cc & 1) == 0) X = {0.5 * (Zk.re + Zm.re), 0.5 * (Zk.im + Zm.im)};
    else X = {0.5 * (Zk.im - Zm.im), -0.5 * (Zk.re - Zm.re)};
    Ghat[(size_t)(kslot ? kslot[k] : k) * n + j0 + cc] = X;
    e = fma(X.re, X.re, fma(X.im, X.im, e));
  }
  if (sq) block_sum_to(e, sq + blockIdx.x);
}

__global__ void __launch_bounds__(512) k_sfft_inverse(const cplx* __restrict__ Uhat, double* __restrict__ U, size_t n, int N, int P,
                               const cplx* __restrict__ tw, double* __restrict__ part,
                               const int* __restrict__ kslot) {
  extern __shared__ cplx smem[];
  __shared__ double red[2][32];
  cplx* tws = smem;
  cplx* z = smem + N;
  const int C = 2 * P;
  const size_t j0 = (size_t)blockIdx.x * C;
  const int half = N / 2;
  // the Hermitian extension of the two packed columns, built straight from
  // the half spectrum: every (k, pair) loads X_a, X_b (two adjacent complex
  // columns, one 32-byte read; a block reads C complex = 16 C bytes per
  // frequency row) into registers and writes Z_k and Z_{N-k}; UNR pairs in
  // flight per thread (no shared staging of the raw spectrum: half the
  // shared footprint, twice the resident blocks)
  for (int t = threadIdx.x; t < N; t += blockDim.x) acp16(&tws[t], &tw[t], true);
  const int K = half + 1;
  const int total = K * P;
  double im2 = 0;
  constexpr int UNR = 4;
  for (int t0 = threadIdx.x; t0 < total; t0 += UNR * blockDim.x) {
    cplx xa[UNR], xb[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int t = t0 + u * blockDim.x;
      xa[u] = xb[u] = cplx{0, 0};
      if (t < total) {
        const int k = t / P, p = t - k * P;
        const size_t col = j0 + 2 * p;
        const cplx* src = Uhat + (size_t)(kslot ? kslot[k] : k) * n + col;
        if (col < n) xa[u] = src[0];
        if (col + 1 < n) xb[u] = src[1];
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int t = t0 + u * blockDim.x;
      if (t >= total) break;
      const int k = t / P, p = t - k * P;
      const cplx Xa = xa[u], Xb = xb[u];
      if (k == 0 || k == half) {
        z[zx(k * P + p)] = {Xa.re, Xb.re};
        im2 += (Xa.im * Xa.im + Xb.im * Xb.im) / N;
      } else {
        z[zx(k * P + p)] = {Xa.re - Xb.im, Xa.im + Xb.re};
        z[zx((N - k) * P + p)] = {Xa.re + Xb.im, -Xa.im + Xb.re};
      }
    }
  }
  acp_wait_all();
  __syncthreads();
  stockham<true>(z, tws, N, P);
  const double invN = 1.0 / N;
  double re2 = 0;
  const double* zd = reinterpret_cast<const double*>(z);
  for (int t = threadIdx.x; t < N * C; t += blockDim.x) {
    const int i = t / C, cc = t - i * C;
    if (j0 + cc >= n) continue;
    const double x = zd[2 * zx(i * P + (cc >> 1)) + (cc & 1)] * invN;
    U[(size_t)i * n + j0 + cc] = x;
    re2 += x * x;
  }
  for (int o = 16; o > 0; o >>= 1) {
    re2 += __shfl_down_sync(0xffffffffu, re2, o);
    im2 += __shfl_down_sync(0xffffffffu, im2, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = re2;
    red[1][threadIdx.x >> 5] = im2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0, b = 0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) {
      a += red[0][w];
      b += red[1][w];
    }
    part[2 * blockIdx.x] = a;
    part[2 * blockIdx.x + 1] = b;
  }
}

// ---------------------------------------------------------------- compile-time shapes
// The same Stockham transforms with N and the column pairs P as template
// constants (the plan's shapes for N = 64 .. 4096).  With N, P and every
// pass's Ns known at compile time, the per-element index arithmetic (t / P,
// t % P, j % Ns, the row/column split of the staging loops) folds to shifts
// and masks, and every thread walks one column with a pointer increment
// instead of a 64-bit multiply per element: the runtime-shaped kernels spent
// ~75 % of their issued instructions on integer work (IMAD 30 %, ISETP 11 %,
// LEA 8 %, the emulated divisions' IABS / I2F / F2I) against 15 % fp64,
// issue-bound at 2.25 TB/s at cfg 3 (profiles/r2o_sass_mix_fwd.txt).
// Compact twiddle table of the compile-time-shaped kernels: W_N^m =
// hi[m / 32] * lo[m % 32] from N/32 + 32 entries (1 KB at N = 1024 instead of
// the 16 KB full table, so three blocks fit an SM; the product adds ~1 ulp)
template <int N>
constexpr int tw_count() { return N / 32 + 32; }
// resident 256-thread blocks per SM the registers of the compile-time-shaped
// kernels are bounded for (3: 80 registers with ~150 bytes of spills -- measured
// slower, 310-346 vs 295-297 ms per cfg-3 sweep, profiles/r2u_ab.txt; 2: none)
#ifndef TPGPU_FFT_MINB
#define TPGPU_FFT_MINB 2
#endif
template <int N>
__device__ __forceinline__ cplx tw_at(const cplx* tw, int m) {
  return cmul(tw[m >> 5], tw[N / 32 + (m & 31)]);
}

template <int R, bool INV, int N, int P, int Ns, int VPT>
__device__ __forceinline__ void stockham_pass_t(cplx* z, const cplx* tw) {
  constexpr int T = P * N / VPT;
  constexpr int B = VPT / R;
  constexpr int NR = N / R;
  cplx v[B][R];
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const int t = threadIdx.x + b * T, p = t % P, j = t / P;
#pragma unroll
    for (int r = 0; r < R; ++r) v[b][r] = z[zx((j + r * NR) * P + p)];
  }
  __syncthreads();
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const int t = threadIdx.x + b * T, p = t % P, j = t / P;
    const int k = j % Ns;
    if constexpr (Ns > 1) {
      const int step = k * (N / (Ns * R));
#pragma unroll
      for (int r = 1; r < R; ++r) {
        cplx w = tw_at<N>(tw, r * step);
        if (INV) w.im = -w.im;
        v[b][r] = cmul(v[b][r], w);
      }
    }
    dft_reg<R, INV>(v[b]);
    const int base = (j / Ns) * Ns * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) z[zx((base + r * Ns) * P + p)] = v[b][r];
  }
  __syncthreads();
}

// VPT values per thread: 16 (radix-16 passes, then one of 8, 4 or 2) or 8
// (radix-8 passes, twice the threads at half the registers each)
template <bool INV, int N, int P, int VPT, int Ns = 1>
__device__ __forceinline__ void stockham_t(cplx* z, const cplx* tw) {
  if constexpr (VPT == 16 && Ns * 16 <= N) {
    stockham_pass_t<16, INV, N, P, Ns, VPT>(z, tw);
    stockham_t<INV, N, P, VPT, Ns * 16>(z, tw);
  } else if constexpr (VPT == 8 && Ns * 8 <= N) {
    stockham_pass_t<8, INV, N, P, Ns, VPT>(z, tw);
    stockham_t<INV, N, P, VPT, Ns * 8>(z, tw);
  } else if constexpr (N / Ns == 8) {
    stockham_pass_t<8, INV, N, P, Ns, VPT>(z, tw);
  } else if constexpr (N / Ns == 4) {
    stockham_pass_t<4, INV, N, P, Ns, VPT>(z, tw);
  } else if constexpr (N / Ns == 2) {
    stockham_pass_t<2, INV, N, P, Ns, VPT>(z, tw);
  }
}

template <int N, int P, int VPT = 16>
__global__ void __launch_bounds__(P * N / VPT, P * N / VPT == 256 ? TPGPU_FFT_MINB : P * N / VPT == 512 ? 2 : 1) k_sfft_forward_t(const double* __restrict__ G, cplx* __restrict__ Ghat,
                                                             size_t n, const cplx* __restrict__ tw,
                                                             double* __restrict__ sq, const int* __restrict__ kslot) {
  constexpr int T = P * N / VPT, C = 2 * P, K = N / 2 + 1, RS = T / C;  // RS: rows per sweep of the block
  static_assert(T % C == 0 && T <= 512, "shape");
  extern __shared__ cplx smem[];
  cplx* tws = smem;
  cplx* z = smem + tw_count<N>();
  const size_t j0 = (size_t)blockIdx.x * C;
  for (int t = threadIdx.x; t < tw_count<N>(); t += T) acp16(&tws[t], &tw[t], true);
  // this thread's column cc and rows i0, i0 + RS, ... (cp.async, zero-fill past the last column)
  const int cc = threadIdx.x % C, i0 = threadIdx.x / C, p = cc >> 1;
  const bool ok = j0 + cc < n;
  double* zd = reinterpret_cast<double*>(z);
  {
    const double* src = ok ? G + (size_t)i0 * n + j0 + cc : G;
    const size_t step = ok ? (size_t)RS * n : 0;
#pragma unroll 8
    for (int i = i0; i < N; i += RS, src += step) acp8(&zd[2 * zx(i * P + p) + (cc & 1)], src, ok);
  }
  acp_wait_all();
  __syncthreads();
  stockham_t<false, N, P, VPT>(z, tws);
  // untangle the two packed real columns: X = (Z_k + conj Z_{N-k}) / 2 (even
  // column), (Z_k - conj Z_{N-k}) / 2i (odd column)
  double e = 0;
  if (ok) {
    const bool odd = cc & 1;
    cplx* dst = Ghat + (size_t)i0 * n + j0 + cc;
    const size_t step = (size_t)RS * n;
    for (int k = i0; k < K; k += RS, dst += step) {
      const cplx Zk = z[zx(k * P + p)], Zm = conj(z[zx(((N - k) & (N - 1)) * P + p)]);
      const cplx X = odd ? cplx{0.5 * (Zk.im - Zm.im), -0.5 * (Zk.re - Zm.re)}
                         : cplx{0.5 * (Zk.re + Zm.re), 0.5 * (Zk.im + Zm.im)};
      if (kslot) Ghat[(size_t)kslot[k] * n + j0 + cc] = X;
      else *dst = X;
      e = fma(X.re, X.re, fma(X.im, X.im, e));
    }
  }
  if (sq) block_sum_to(e, sq + blockIdx.x);
}

template <int N, int P, int VPT = 16>
__global__ void __launch_bounds__(P * N / VPT, P * N / VPT == 256 ? TPGPU_FFT_MINB : P * N / VPT == 512 ? 2 : 1) k_sfft_inverse_t(const cplx* __restrict__ Uhat, double* __restrict__ U,
                                                             size_t n, const cplx* __restrict__ tw,
                                                             double* __restrict__ part, const int* __restrict__ kslot) {
  constexpr int T = P * N / VPT, C = 2 * P, half = N / 2, K = half + 1, RS = T / C, KS = T / P;
  static_assert(T % C == 0 && T <= 512, "shape");
  extern __shared__ cplx smem[];
  __shared__ double red[2][32];
  cplx* tws = smem;
  cplx* z = smem + tw_count<N>();
  const size_t j0 = (size_t)blockIdx.x * C;
  for (int t = threadIdx.x; t < tw_count<N>(); t += T) acp16(&tws[t], &tw[t], true);
  // the Hermitian extension of the two packed columns 2p, 2p+1, straight
  // from the half spectrum: this thread's pair p, frequencies k0, k0 + KS, ...
  const int p = threadIdx.x % P, k0 = threadIdx.x / P;
  const size_t col = j0 + 2 * p;
  const bool oka = col < n, okb = col + 1 < n;
  double im2 = 0;
  {
    const cplx* src = Uhat + (size_t)k0 * n + col;
    const size_t step = (size_t)KS * n;
    constexpr int UNR = 4;
    for (int kb = k0; kb < K; kb += UNR * KS) {
      cplx xa[UNR], xb[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int k = kb + u * KS;
        xa[u] = xb[u] = cplx{0, 0};
        if (k < K) {
          const cplx* s = kslot ? Uhat + (size_t)kslot[k] * n + col : src + (size_t)u * step;
          if (oka) xa[u] = s[0];
          if (okb) xb[u] = s[1];
        }
      }
      src += (size_t)UNR * step;
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int k = kb + u * KS;
        if (k >= K) break;
        const cplx Xa = xa[u], Xb = xb[u];
        if (k == 0 || k == half) {
          z[zx(k * P + p)] = {Xa.re, Xb.re};
          im2 += (Xa.im * Xa.im + Xb.im * Xb.im) / N;
        } else {
          z[zx(k * P + p)] = {Xa.re - Xb.im, Xa.im + Xb.re};
          z[zx((N - k) * P + p)] = {Xa.re + Xb.im, -Xa.im + Xb.re};
        }
      }
    }
  }
  acp_wait_all();
  __syncthreads();
  stockham_t<true, N, P, VPT>(z, tws);
  constexpr double invN = 1.0 / N;
  double re2 = 0;
  const double* zd = reinterpret_cast<const double*>(z);
  {
    const int cc = threadIdx.x % C, i0 = threadIdx.x / C;
    if (j0 + cc < n) {
      double* dst = U + (size_t)i0 * n + j0 + cc;
      const size_t step = (size_t)RS * n;
#pragma unroll 4
      for (int i = i0; i < N; i += RS, dst += step) {
        const double x = zd[2 * zx(i * P + (cc >> 1)) + (cc & 1)] * invN;
        *dst = x;
        re2 = fma(x, x, re2);
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    re2 += __shfl_down_sync(0xffffffffu, re2, o);
    im2 += __shfl_down_sync(0xffffffffu, im2, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = re2;
    red[1][threadIdx.x >> 5] = im2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0, b = 0;
    for (int w = 0; w < T / 32; ++w) {
      a += red[0][w];
      b += red[1][w];
    }
    part[2 * blockIdx.x] = a;
    part[2 * blockIdx.x + 1] = b;
  }
}

// the compiled shapes: (N, P) -> kernel pointers (nullptr: runtime-shaped kernels)
using FwdFn = void (*)(const double*, cplx*, size_t, const cplx*, double*, const int*);
using InvFn = void (*)(const cplx*, double*, size_t, const cplx*, double*, const int*);
template <int N, int P, int VPT = 16>
bool pick_shape(int n_, int p_, FwdFn& f, InvFn& g, int vpt = 16) {
  if (n_ != N || p_ != P || vpt != VPT) return false;
  f = k_sfft_forward_t<N, P, VPT>;
  g = k_sfft_inverse_t<N, P, VPT>;
  return true;
}
bool compiled_shape(int N, int P, FwdFn& f, InvFn& g, int vpt) {
  if (vpt == 8) return pick_shape<1024, 4, 8>(N, P, f, g, vpt) || pick_shape<512, 4, 8>(N, P, f, g, vpt);
  return pick_shape<64, 32>(N, P, f, g) || pick_shape<128, 16>(N, P, f, g) || pick_shape<256, 8>(N, P, f, g) ||
         pick_shape<512, 4>(N, P, f, g) || pick_shape<1024, 4>(N, P, f, g) || pick_shape<1024, 2>(N, P, f, g) ||
         pick_shape<1024, 8>(N, P, f, g) || pick_shape<2048, 4>(N, P, f, g) ||
         pick_shape<4096, 2>(N, P, f, g);
}

// ---------------------------------------------------------------- pipelined transforms
// Persistent, software-pipelined forms of k_sfft_forward / k_sfft_inverse for
// long periods (N >= 512): a block walks tiles of C = 2P columns with a
// stride of the grid and keeps the NEXT tile's loads in flight (cp.async into
// the second of two shared buffers) while it transforms and stores the
// current one.  The one-shot kernels load, then compute, then store, so at
// one or two resident blocks per SM HBM idled through every transform:
// 2.2-2.3 TB/s at cfg 3 (profiles/r2i_launches_cfg3_sweep.txt).

// stage tile `tile` of the real input (N rows x C doubles) into z (padded layout)
__device__ __forceinline__ void fwd_issue(double* zd, const double* __restrict__ G, size_t n, int N, int P,
                                          size_t tile) {
  const int C = 2 * P;
  const size_t j0 = tile * C;
  for (int t = threadIdx.x; t < N * C; t += blockDim.x) {
    const int i = t / C, cc = t - i * C;
    const bool ok = j0 + cc < n;
    acp8(&zd[2 * zx(i * P + (cc >> 1)) + (cc & 1)], G + (ok ? (size_t)i * n + j0 + cc : 0), ok);
  }
}

__global__ void __launch_bounds__(256, 1) k_sfft_forward_pp(const double* __restrict__ G, cplx* __restrict__ Ghat,
                                                           size_t n, int N, int P, const cplx* __restrict__ tw,
                                                           double* __restrict__ sq, const int* __restrict__ kslot,
                                                           size_t ntiles) {
  extern __shared__ cplx smem[];
  cplx* tws = smem;
  const int zsz = zx_size(P * N);
  cplx* zb[2] = {smem + N, smem + N + zsz};
  for (int t = threadIdx.x; t < N; t += blockDim.x) acp16(&tws[t], &tw[t], true);
  size_t tile = blockIdx.x;
  if (tile < ntiles) fwd_issue(reinterpret_cast<double*>(zb[0]), G, n, N, P, tile);
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  const int C = 2 * P, K = N / 2 + 1;
  double e = 0;
  for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {
    cplx* z = zb[it & 1];
    const size_t next = tile + gridDim.x;
    if (next < ntiles) fwd_issue(reinterpret_cast<double*>(zb[(it + 1) & 1]), G, n, N, P, next);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");  // this tile (and the twiddles) landed
    __syncthreads();
    stockham<false>(z, tws, N, P);
    const size_t j0 = tile * C;
    for (int t = threadIdx.x; t < K * C; t += blockDim.x) {
      const int k = t / C, cc = t - k * C;
      if (j0 + cc >= n) continue;
      const int p = cc >> 1;
      const cplx Zk = z[zx(k * P + p)], Zm = conj(z[zx(((N - k) % N) * P + p)]);
      cplx X;
      if ((cc & 1) == 0) X = {0.5 * (Zk.re + Zm.re), 0.5 * (Zk.im + Zm.im)};
      else X = {0.5 * (Zk.im - Zm.im), -0.5 * (Zk.re - Zm.re)};
      Ghat[(size_t)(kslot ? kslot[k] : k) * n + j0 + cc] = X;
      e = fma(X.re, X.re, fma(X.im, X.im, e));
    }
    __syncthreads();  // z is refilled two tiles on
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  if (sq) block_sum_to(e, sq + blockIdx.x);
}

// stage tile `tile` of the half spectrum (K rows x C complex) into raw
__device__ __forceinline__ void inv_issue(cplx* raw, const cplx* __restrict__ Uhat, size_t n, int N, int P,
                                          size_t tile, const int* __restrict__ kslot) {
  const int C = 2 * P, K = N / 2 + 1;
  const size_t j0 = tile * C;
  for (int t = threadIdx.x; t < K * C; t += blockDim.x) {
    const int k = t / C, cc = t - k * C;
    const bool ok = j0 + cc < n;
    acp16(&raw[t], Uhat + (ok ? (size_t)(kslot ? kslot[k] : k) * n + j0 + cc : 0), ok);
  }
}

__global__ void __launch_bounds__(256, 1) k_sfft_inverse_pp(const cplx* __restrict__ Uhat, double* __restrict__ U,
                                                           size_t n, int N, int P, const cplx* __restrict__ tw,
                                                           double* __restrict__ part, const int* __restrict__ kslot,
                                                           size_t ntiles) {
  extern __shared__ cplx smem[];
  __shared__ double red[2][32];
  const int C = 2 * P, half = N / 2, K = half + 1;
  cplx* tws = smem;
  cplx* z = smem + N;
  const int zsz = zx_size(P * N);
  cplx* rb[2] = {z + zsz, z + zsz + K * C};
  for (int t = threadIdx.x; t < N; t += blockDim.x) acp16(&tws[t], &tw[t], true);
  size_t tile = blockIdx.x;
  if (tile < ntiles) inv_issue(rb[0], Uhat, n, N, P, tile, kslot);
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  double re2 = 0, im2 = 0;
  const double invN = 1.0 / N;
  for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {
    const cplx* raw = rb[it & 1];
    const size_t next = tile + gridDim.x;
    if (next < ntiles) inv_issue(rb[(it + 1) & 1], Uhat, n, N, P, next, kslot);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    __syncthreads();
    // Hermitian extension of the two packed columns (N even: self-conjugate 0, N/2)
    for (int t = threadIdx.x; t < K * P; t += blockDim.x) {
      const int k = t / P, p = t - k * P;
      const cplx Xa = raw[k * C + 2 * p], Xb = raw[k * C + 2 * p + 1];
      if (k == 0 || k == half) {
        z[zx(k * P + p)] = {Xa.re, Xb.re};
        im2 += (Xa.im * Xa.im + Xb.im * Xb.im) / N;
      } else {
        z[zx(k * P + p)] = {Xa.re - Xb.im, Xa.im + Xb.re};
        z[zx((N - k) * P + p)] = {Xa.re + Xb.im, -Xa.im + Xb.re};
      }
    }
    __syncthreads();
    stockham<true>(z, tws, N, P);
    const size_t j0 = tile * C;
    const double* zd = reinterpret_cast<const double*>(z);
    for (int t = threadIdx.x; t < N * C; t += blockDim.x) {
      const int i = t / C, cc = t - i * C;
      if (j0 + cc >= n) continue;
      const double x = zd[2 * zx(i * P + (cc >> 1)) + (cc & 1)] * invN;
      U[(size_t)i * n + j0 + cc] = x;
      re2 += x * x;
    }
    __syncthreads();  // z rebuilt and this raw buffer refilled next
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  for (int o = 16; o > 0; o >>= 1) {
    re2 += __shfl_down_sync(0xffffffffu, re2, o);
    im2 += __shfl_down_sync(0xffffffffu, im2, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = re2;
    red[1][threadIdx.x >> 5] = im2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0, b = 0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) {
      a += red[0][w];
      b += red[1][w];
    }
    part[2 * blockIdx.x] = a;
    part[2 * blockIdx.x + 1] = b;
  }
}

__global__ void k_reduce_pairs(const double* __restrict__ part, int count, double* __restrict__ out) {
  __shared__ double sh[2][32];
  double a = 0, b = 0;
  for (int k = threadIdx.x; k < count; k += blockDim.x) {
    a += part[2 * k];
    b += part[2 * k + 1];
  }
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_down_sync(0xffffffffu, a, o);
    b += __shfl_down_sync(0xffffffffu, b, o);
  }
  if ((threadIdx.x & 31) == 0) {
    sh[0][threadIdx.x >> 5] = a;
    sh[1][threadIdx.x >> 5] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0, t = 0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) {
      s += sh[0][w];
      t += sh[1][w];
    }
    out[0] = s;
    out[1] = t;
  }
}

struct FftPlan {
  int N = 0, P = 0, bits = 0;
  bool pow2 = false;
  size_t smem = 0;
  DevBuf<cplx> tw;
  // Stockham path (power-of-two N >= 16): columns pairs per block, threads, shared bytes
  bool stockham = false;
  int sP = 0, sT = 0;    // forward: column pairs per block, threads
  int siP = 0, siT = 0;  // inverse
  FwdFn tf = nullptr;    // compile-time-shaped kernels for (N, sP) when compiled (sP == siP)
  InvFn ti = nullptr;
  DevBuf<cplx> tw2;      // their compact twiddle table (hi: W^{32j}, j < N/32; lo: W^i, i < 32)
  size_t tsmem = 0;      // their shared bytes
  int tT = 0;            // their threads per block
  size_t ssmem = 0, fsmem = 0;  // inverse (+ staged half spectrum) / forward
  // pipelined persistent kernels (N >= 512): column pairs, threads, shared bytes, grid
  bool pp_fwd = false, pp_inv = false;
  int pP = 0, pT = 0, pgrid = 0;
  size_t pfsmem = 0, pismem = 0;
};

FftPlan& plan_for(std::shared_ptr<void>& slot, int N) {
  if (slot) return *static_cast<FftPlan*>(slot.get());
  auto pl = std::make_shared<FftPlan>();
  pl->N = N;
  pl->pow2 = (N & (N - 1)) == 0;
  while ((1 << pl->bits) < N) ++pl->bits;
  int P = 8192 / N;
  P = std::max(1, std::min(16, P));
  const size_t bufs = pl->pow2 ? 1 : 2;
  while (P > 1 && (size_t)P * N * sizeof(cplx) * bufs > 160 * 1024) P >>= 1;
  require((size_t)P * N * sizeof(cplx) * bufs <= 200 * 1024, "dft: N too large for the shared-memory transform");
  pl->P = P;
  pl->smem = (size_t)P * N * sizeof(cplx) * bufs;
  std::vector<cplx> h(N);
  for (int k = 0; k < N; ++k) {
    const double a = -2.0 * std::numbers::pi * k / N;  // std::polar(1, a), fft.hpp:27-28
    h[k] = {std::cos(a), std::sin(a)};
  }
  pl->tw.alloc(N);
  TP_CUDA(cudaMemcpy(pl->tw.get(), h.data(), N * sizeof(cplx), cudaMemcpyHostToDevice));
  TP_CUDA(cudaFuncSetAttribute(k_rdft_forward, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl->smem));
  TP_CUDA(cudaFuncSetAttribute(k_rdft_inverse, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl->smem));
  // Stockham: P N / 16 threads (16 values each per pass), P N ~ 2048 complex
  // (36 KB of shared memory with the twiddles: six blocks per SM)
  if (pl->pow2 && N >= 16 && !std::getenv("TPGPU_RADIX2_DFT")) {
    static const int fp_env = std::getenv("TPGPU_FFT_P") ? std::atoi(std::getenv("TPGPU_FFT_P")) : 0;
    // at least 4 column pairs (64-byte row segments) for long periods: with 2
    // pairs at N = 1024 the 32-byte row reads held both transforms near 1.8
    // TB/s (cfg 3 launch list, profiles/r2c_launches_cfg3_sweep.txt); 4 pairs
    // -> 2.3 / 1.5 TB/s; 8 pairs (512 threads, one block per SM) measured
    // level with 4 on the whole sweep (profiles/r2h_ab.txt)
    int sP = fp_env > 0 ? fp_env : std::max(N >= 512 ? 4 : 1, 2048 / N);
    while (sP > 1 && (size_t)(N + zx_size(sP * N)) * sizeof(cplx) > 200 * 1024) sP >>= 1;
    const int T = sP * N / 16;
    if (T <= 512 && (size_t)(N + zx_size(sP * N)) * sizeof(cplx) <= 200 * 1024) {  // __launch_bounds__(512)
      pl->stockham = true;
      pl->sP = sP;
      pl->sT = std::max(32, T);
      // inverse: the same column pairs per block (TPGPU_IFFT_P overrides)
      static const int ip_env = std::getenv("TPGPU_IFFT_P") ? std::atoi(std::getenv("TPGPU_IFFT_P")) : 0;
      const int siP = ip_env > 0 ? ip_env : sP;
      pl->siP = siP;
      pl->siT = std::max(32, siP * N / 16);
      pl->ssmem = (size_t)(N + zx_size(siP * N)) * sizeof(cplx);
      pl->fsmem = (size_t)(N + zx_size(sP * N)) * sizeof(cplx);
      TP_CUDA(cudaFuncSetAttribute(k_sfft_forward, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl->fsmem));
      TP_CUDA(cudaFuncSetAttribute(k_sfft_inverse, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl->ssmem));
      // compile-time shapes (TPGPU_FFT_TEMPLATE=0: the runtime-shaped kernels)
      static const bool want_t = !std::getenv("TPGPU_FFT_TEMPLATE") || std::atoi(std::getenv("TPGPU_FFT_TEMPLATE")) != 0;
      FwdFn f = nullptr;
      InvFn g = nullptr;
      // values per thread of the compiled shapes (TPGPU_FFT_VPT=8: radix-8
      // passes with twice the threads at 64 registers; measured slower at
      // cfg 3: forward / inverse 22.1 / 24.4 vs 20.9 / 23.1 ms, 281 vs 277 ms
      // per sweep, profiles/r2zc_ab.txt -- the fourth pass through shared
      // memory and its barrier cost more than the doubled occupancy gains)
      static const int vpt_env = std::getenv("TPGPU_FFT_VPT") ? std::atoi(std::getenv("TPGPU_FFT_VPT")) : 16;
      int vpt = vpt_env == 8 && compiled_shape(N, sP, f, g, 8) ? 8 : 16;
      if (want_t && siP == sP && compiled_shape(N, sP, f, g, vpt)) {
        pl->tf = f;
        pl->ti = g;
        pl->tT = sP * N / vpt;
        const int nt = N / 32 + 32;
        std::vector<cplx> t2(nt);
        for (int j = 0; j < N / 32; ++j) {
          const double a = -2.0 * std::numbers::pi * (32.0 * j) / N;
          t2[j] = {std::cos(a), std::sin(a)};
        }
        for (int i = 0; i < 32; ++i) {
          const double a = -2.0 * std::numbers::pi * i / N;
          t2[N / 32 + i] = {std::cos(a), std::sin(a)};
        }
        pl->tw2.alloc(nt);
        TP_CUDA(cudaMemcpy(pl->tw2.get(), t2.data(), nt * sizeof(cplx), cudaMemcpyHostToDevice));
        pl->tsmem = (size_t)(nt + zx_size(sP * N)) * sizeof(cplx);
        TP_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(f), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)pl->tsmem));
        TP_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(g), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)pl->tsmem));
      }
    }
  }
  // pipelined forms: two tiles of P column pairs (+ twiddles; the inverse also
  // stages two raw half-spectrum tiles), one block of P N / 16 threads per SM
  // opt-in (TPGPU_FFT_PIPELINE=1): measured slower than the one-shot kernels
  // at cfg 3 (378.6 vs 351.2 ms per sweep, profiles/r2j_ab.txt; the inverse
  // moved 108 GB of DRAM for its 68.8 GB of data)
  static const bool want_pp = std::getenv("TPGPU_FFT_PIPELINE") && std::atoi(std::getenv("TPGPU_FFT_PIPELINE")) != 0;
  if (pl->stockham && N >= 512 && want_pp) {
    int dev = 0, sms = 148, maxsm = 0;
    TP_CUDA(cudaGetDevice(&dev));
    TP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    TP_CUDA(cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    static const int pp_env = std::getenv("TPGPU_FFT_PP_P") ? std::atoi(std::getenv("TPGPU_FFT_PP_P")) : 4;
    for (int P = pp_env; P >= 2; P >>= 1) {
      const size_t fs = (size_t)(N + 2 * zx_size(P * N)) * sizeof(cplx);
      const size_t is = (size_t)(N + zx_size(P * N) + 2 * (N / 2 + 1) * 2 * P) * sizeof(cplx) + 2 * 32 * sizeof(double);
      const int T = P * N / 16;
      if (T > 256) continue;  // __launch_bounds__(256, 1)
      const bool f_ok = fs <= (size_t)maxsm, i_ok = is <= (size_t)maxsm;
      if (!f_ok) continue;
      pl->pp_fwd = true;
      pl->pp_inv = i_ok;
      pl->pP = P;
      pl->pT = T;
      pl->pgrid = sms;
      pl->pfsmem = fs;
      pl->pismem = is - 2 * 32 * sizeof(double);
      TP_CUDA(cudaFuncSetAttribute(k_sfft_forward_pp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fs));
      if (i_ok)
        TP_CUDA(cudaFuncSetAttribute(k_sfft_inverse_pp, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)pl->pismem));
      break;
    }
  }
  slot = pl;
  return *pl;
}

void launched(const DftCtx& c) {
  if (c.launches) ++*c.launches;
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw_cuda(e, "kernel launch", __FILE__, __LINE__);
}

}  // namespace

int dft_forward_blocks(const DftCtx& c) {
  FftPlan& pl = plan_for(*c.plan, c.N);
  if (pl.pp_fwd) return pl.pgrid;
  const int C = 2 * (pl.stockham ? pl.sP : pl.P);
  return (int)((c.n + C - 1) / C);
}

void dft_forward(const DftCtx& c, const double* G, cplx* Ghat, double* sq) {
  FftPlan& pl = plan_for(*c.plan, c.N);
  const int blocks = dft_forward_blocks(c);
  if (pl.pp_fwd) {
    const size_t ntiles = (c.n + 2 * pl.pP - 1) / (2 * pl.pP);
    k_sfft_forward_pp<<<pl.pgrid, pl.pT, pl.pfsmem, c.stream>>>(G, Ghat, c.n, pl.N, pl.pP, pl.tw.get(), sq, c.kslot,
                                                                 ntiles);
  } else if (pl.tf) {
    pl.tf<<<blocks, pl.tT, pl.tsmem, c.stream>>>(G, Ghat, c.n, pl.tw2.get(), sq, c.kslot);
  } else if (pl.stockham) {
    k_sfft_forward<<<blocks, pl.sT, pl.fsmem, c.stream>>>(G, Ghat, c.n, pl.N, pl.sP, pl.tw.get(), sq, c.kslot);
  } else {
    k_rdft_forward<<<blocks, 256, pl.smem, c.stream>>>(G, Ghat, c.n, pl.N, pl.P, pl.bits, pl.pow2, pl.tw.get(),
                                                       sq, c.kslot);
  }
  launched(c);
}

void dft_inverse(const DftCtx& c, const cplx* Uhat, double* U, double* re2, double* im2) {
  FftPlan& pl = plan_for(*c.plan, c.N);
  const int C = 2 * (pl.stockham ? pl.siP : pl.P);
  const int blocks = pl.pp_inv ? pl.pgrid : (int)((c.n + C - 1) / C);
  c.part->ensure((size_t)2 * blocks);
  c.red->ensure(16);
  if (pl.pp_inv) {
    const size_t ntiles = (c.n + 2 * pl.pP - 1) / (2 * pl.pP);
    k_sfft_inverse_pp<<<pl.pgrid, pl.pT, pl.pismem, c.stream>>>(Uhat, U, c.n, pl.N, pl.pP, pl.tw.get(),
                                                                 c.part->get(), c.kslot, ntiles);
  } else if (pl.ti) {
    pl.ti<<<blocks, pl.tT, pl.tsmem, c.stream>>>(Uhat, U, c.n, pl.tw2.get(), c.part->get(), c.kslot);
  } else if (pl.stockham) {
    k_sfft_inverse<<<blocks, pl.siT, pl.ssmem, c.stream>>>(Uhat, U, c.n, pl.N, pl.siP, pl.tw.get(),
                                                            c.part->get(), c.kslot);
  } else {
    k_rdft_inverse<<<blocks, 256, pl.smem, c.stream>>>(Uhat, U, c.n, pl.N, pl.P, pl.bits, pl.pow2, pl.tw.get(),
                                                       c.part->get(), c.kslot);
  }
  launched(c);
  k_reduce_pairs<<<1, 1024, 0, c.stream>>>(c.part->get(), blocks, c.red->get());
  launched(c);
  if (re2 || im2) {
    TP_CUDA(cudaMemcpyAsync(c.h_scalars, c.red->get(), 2 * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    TP_CUDA(cudaStreamSynchronize(c.stream));
    if (re2) *re2 = c.h_scalars[0];
    if (im2) *im2 = c.h_scalars[1];
  }
}

namespace {
DftCtx ctx_of(Problem& p) {
  // columns of this rank's strip
  return DftCtx{p.N, (size_t)p.sh.nr, p.stream, &p.fft_plan, &p.part, &p.red, p.h_scalars, &p.launches,
                p.d_kslot.get()};
}
}  // namespace

int rdft_forward_blocks(Problem& p) { return dft_forward_blocks(ctx_of(p)); }

void launch_rdft_forward(Problem& p, const double* G, cplx* Ghat, double* sq) {
  dft_forward(ctx_of(p), G, Ghat, sq);
}

void launch_rdft_inverse(Problem& p, const cplx* Uhat, double* U, double* re2, double* im2) {
  dft_inverse(ctx_of(p), Uhat, U, re2, im2);
}

}  // namespace tpgpu
