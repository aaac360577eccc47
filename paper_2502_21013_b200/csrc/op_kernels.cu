// Nonlinear operator kernels: K(u), the fused residual + fixed-point RHS, and
// the P1 element-stencil assembly (K_hat and Newton Jacobians).
//
// Reference: NonlinearOperator::apply (assembly.hpp:126-140), the M1 RHS
// lambda (solvers.hpp:326-336), residual (periodic.hpp:35-58),
// assemble_stiffness_frozen (assembly.hpp:68-84), jacobian (assembly.hpp:153-177).
//
// Structured-grid restatement: with h = 1/c, area = h^2/2 and basis gradients
// c*s_a (s_a in {-1,0,1}^2), the element term nu*area*grad u.grad phi_a is
// (nu/2) * (dx*sx_a + dy*sy_a) where (dx, dy) are vertex differences -- the
// h factors cancel.  Each 32x8 node tile stages u (+1 halo) in shared memory,
// evaluates nu(|grad u|) once per triangle, then every node gathers its six
// incident triangles (no atomics, deterministic).
#include "tp_internal.cuh"

namespace tpgpu {

// 1/x to full double precision without the special-case path of the correctly
// rounded reciprocal: hardware estimate + two Newton steps (x > 0 normal here:
// s^2 + Bs^2 with Bs > 0)
__device__ __forceinline__ double acc_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = fma(r, fma(-x, r, 1.0), r);
  return fma(r, fma(-x, r, 1.0), r);
}

namespace {

constexpr int TX = 32, TY = 8;

__device__ __forceinline__ double nu_of(const MaterialDev& mt, double s2) {
  if (mt.linear) return mt.nu0;
  // s2/(s2+Bs^2) with a correctly rounded reciprocal (one more rounding than
  // the reference's division: ~1 ulp, far below the 1e-13 K(u) parity bar)
  return fma(mt.nu_inf - mt.nu0, s2 * acc_rcp(s2 + mt.bs2), mt.nu0);
}

// Shared-memory tile: vertices [x0, x0+TX+1] x [y0, y0+TY+1] (vertex coords),
// cells [x0, x0+TX] x [y0, y0+TY].
struct Tile {
  double u[TY + 2][TX + 2];
  double w[2][TY + 1][TX + 1];   // nu_T / 2 (nonlinear)
  double wh[2][TY + 1][TX + 1];  // nu_hat_T / 2 (frozen)
};

// u at vertex (X, Y) of slice `us` (0 on the Dirichlet boundary).
__device__ __forceinline__ double vertex_u(const double* __restrict__ us, int m, int X, int Y) {
  return (X >= 1 && X <= m && Y >= 1 && Y <= m) ? us[(size_t)(Y - 1) * m + (X - 1)] : 0.0;
}

// A row strip of the node grid held by one rank: node rows [y0, y0+rows) of
// a slice at `us` (local row-major), plus the halo rows y0-1 (`lo`) and
// y0+rows (`hi`) from the neighbouring ranks (nullptr: none / boundary).
struct StripView {
  const double* lo;
  const double* hi;
  int y0, rows;
};

__device__ __forceinline__ double vertex_u(const double* __restrict__ us, const StripView& sv, int m, int X,
                                           int Y) {
  const int x = X - 1, y = Y - 1;
  if (x < 0 || x >= m || y < 0 || y >= m) return 0.0;
  const int ly = y - sv.y0;
  if (ly < 0) return (ly == -1 && sv.lo) ? sv.lo[x] : 0.0;
  if (ly >= sv.rows) return (ly == sv.rows && sv.hi) ? sv.hi[x] : 0.0;
  return us[(size_t)ly * m + x];
}

template <bool NEED_NU, bool NEED_HAT>
__device__ void tile_load(Tile& t, const double* __restrict__ us, const StripView& sv,
                          const double* __restrict__ ds, double alpha, int m, int c, int x0, int y0,
                          const uint8_t* __restrict__ cell_mat, const MaterialDev* __restrict__ mats,
                          const double* __restrict__ nu_hat) {
  const int tid = threadIdx.y * TX + threadIdx.x;
  for (int k = tid; k < (TY + 2) * (TX + 2); k += TX * TY) {
    const int ly = k / (TX + 2), lx = k % (TX + 2);
    double v = vertex_u(us, sv, m, x0 + lx, y0 + ly);
    if (ds) v += alpha * vertex_u(ds, m, x0 + lx, y0 + ly);
    t.u[ly][lx] = v;
  }
  __syncthreads();
  const double c2 = (double)c * (double)c;
  for (int k = tid; k < (TY + 1) * (TX + 1); k += TX * TY) {
    const int ly = k / (TX + 1), lx = k % (TX + 1);
    const int i = x0 + lx, j = y0 + ly;
    double w1 = 0, w2 = 0, h = 0;
    if (i < c && j < c) {
      const MaterialDev mt = mats[cell_mat[(size_t)j * c + i]];
      if (NEED_NU) {
        const double u00 = t.u[ly][lx], u10 = t.u[ly][lx + 1];
        const double u01 = t.u[ly + 1][lx], u11 = t.u[ly + 1][lx + 1];
        const double ax = u10 - u00, ay = u11 - u10;  // T1
        const double bx = u11 - u01, by = u01 - u00;  // T2
        w1 = 0.5 * nu_of(mt, c2 * (ax * ax + ay * ay));
        w2 = 0.5 * nu_of(mt, c2 * (bx * bx + by * by));
      }
      if (NEED_HAT) h = 0.5 * nu_hat[cell_mat[(size_t)j * c + i]];
    }
    t.w[0][ly][lx] = w1;
    t.w[1][ly][lx] = w2;
    t.wh[0][ly][lx] = h;
    t.wh[1][ly][lx] = h;
  }
  __syncthreads();
}

// Sum over the six triangles around node (tx, ty) of W_T * (dx*sx + dy*sy).
template <int WHICH>  // 0: w (nonlinear), 1: wh (frozen)
__device__ __forceinline__ double gather(const Tile& t, int tx, int ty) {
  const int lx = tx + 1, ly = ty + 1;  // vertex of the node inside the tile
  const double uC = t.u[ly][lx], uE = t.u[ly][lx + 1], uW = t.u[ly][lx - 1];
  const double uN = t.u[ly + 1][lx], uS = t.u[ly - 1][lx];
  const double uNE = t.u[ly + 1][lx + 1], uSW = t.u[ly - 1][lx - 1];
  const auto& W = WHICH == 0 ? t.w : t.wh;
  // cell (X,Y) -> tile cell (lx, ly); (X-1,Y) -> (lx-1, ly); (X-1,Y-1) -> (lx-1, ly-1); (X,Y-1) -> (lx, ly-1)
  double acc = 0;
  acc += W[0][ly][lx] * (-(uE - uC));                    // T1(X,Y), local 0
  acc += W[1][ly][lx] * (-(uN - uC));                    // T2(X,Y), local 0
  acc += W[0][ly][lx - 1] * ((uC - uW) - (uN - uC));     // T1(X-1,Y), local 1
  acc += W[0][ly - 1][lx - 1] * (uC - uS);               // T1(X-1,Y-1), local 2
  acc += W[1][ly - 1][lx - 1] * (uC - uW);               // T2(X-1,Y-1), local 1
  acc += W[1][ly - 1][lx] * (-(uE - uC) + (uC - uS));    // T2(X,Y-1), local 2
  (void)uNE;
  (void)uSW;
  return acc;
}

__device__ __forceinline__ double block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  const int nw = (blockDim.x * blockDim.y) / 32;
  __syncthreads();
  if ((tid & 31) == 0) sh[tid >> 5] = v;
  __syncthreads();
  double s = 0;
  if (tid == 0)
    for (int w = 0; w < nw; ++w) s += sh[w];
  return s;
}

// out = K(u) per slice.
__global__ void __launch_bounds__(TX * TY) k_apply_k(const double* __restrict__ U, double* __restrict__ out,
                                                     int m, int c, const uint8_t* __restrict__ cell_mat,
                                                     const MaterialDev* __restrict__ mats) {
  __shared__ Tile t;
  const size_t n = (size_t)m * m;
  const int s = blockIdx.z;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const StripView sv{nullptr, nullptr, 0, m};
  tile_load<true, false>(t, U + s * n, sv, nullptr, 0.0, m, c, x0, y0, cell_mat, mats, nullptr);
  const int x = x0 + threadIdx.x, y = y0 + threadIdx.y;
  if (x < m && y < m) out[s * n + (size_t)y * m + x] = gather<0>(t, threadIdx.x, threadIdx.y);
}

// One pass over the current iterate U (all N slices):
//   R^s = F^s - M (u^s - u^{s-1})/tau - K(u^s)           (periodic.hpp:35-58)
//   G^s = F^s + K_hat u^s - K(u^s)                        (solvers.hpp:326-336)
// K(u) is evaluated once and shared.  R is never written: per-block partial
// sums of R^2 go to `part` (block_l2 is reduced deterministically).
// Strip form: the grid covers the local node rows [sy0, sy0+rows) (global
// coordinates for materials, mass and sources; U, G, R local with slice
// stride rows*m; halo rows lo/hi with slice stride m).
template <bool WANT_G, bool WANT_R>
__global__ void __launch_bounds__(TX * TY) k_sweep_fused(
    const double* __restrict__ U, const double* __restrict__ halo_lo, const double* __restrict__ halo_hi,
    int sy0, int rows, double* __restrict__ G, double* __restrict__ R,
    double* __restrict__ part, int m, int c, int N, double inv_tau,
    const uint8_t* __restrict__ cell_mat, const MaterialDev* __restrict__ mats,
    const double* __restrict__ nu_hat, const double* __restrict__ mass,
    const double* __restrict__ src_prof, const double* __restrict__ src_time, int nsrc) {
  __shared__ Tile t;
  __shared__ double red[32];
  const size_t n = (size_t)m * m;
  const size_t nl = (size_t)rows * m;
  const int s = blockIdx.z;
  const int x0 = blockIdx.x * TX, y0 = sy0 + blockIdx.y * TY;
  const StripView sv{halo_lo ? halo_lo + (size_t)s * m : nullptr, halo_hi ? halo_hi + (size_t)s * m : nullptr,
                     sy0, rows};
  tile_load<true, WANT_G>(t, U + s * nl, sv, nullptr, 0.0, m, c, x0, y0, cell_mat, mats, nu_hat);
  const int x = x0 + threadIdx.x, y = y0 + threadIdx.y;
  double r2 = 0;
  if (x < m && y < sy0 + rows) {
    const size_t i = (size_t)y * m + x;               // global
    const size_t il = (size_t)(y - sy0) * m + x;      // local
    double f = 0;
    for (int r = 0; r < nsrc; ++r) f += src_time[s * nsrc + r] * src_prof[r * n + i];
    const double ku = gather<0>(t, threadIdx.x, threadIdx.y);
    if (WANT_G) {
      const double khu = gather<1>(t, threadIdx.x, threadIdx.y);
      G[s * nl + il] = f + khu - ku;
    }
    const double mi = mass[i];
    double mdu = 0;
    if (mi != 0) {
      const int sp = (s + N - 1) % N;
      mdu = mi * ((t.u[threadIdx.y + 1][threadIdx.x + 1] - U[sp * nl + il]) * inv_tau);
    }
    const double res = f - mdu - ku;
    if (WANT_R && R) R[s * nl + il] = res;
    r2 = res * res;
  }
  const double tot = block_sum(r2, red);
  if (threadIdx.x == 0 && threadIdx.y == 0)
    part[((size_t)s * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = tot;
}

// Slice-looped form of k_sweep_fused (the one used by the sweep): a block
// owns one 32x8 node tile and SB consecutive slices, so everything that
// does not depend on u -- per-cell material law and nu_hat, per-node mass
// and source profiles -- is loaded once and reused SB times, u^{s-1} comes
// from the previous slice's tile, and r^2 is reduced once per block.  The
// u tiles of the next SD-1 slices are in flight (cp.async ring of SD slots,
// zero-filled off the domain, one barrier per slice): with one slice of
// look-ahead the kernel was latency-bound at ~1.3 TB/s.
#ifndef TPGPU_SWEEP_SB
#define TPGPU_SWEEP_SB 16
#endif
constexpr int SB = TPGPU_SWEEP_SB;  // slices per block
#ifndef TPGPU_SWEEP_SD
#define TPGPU_SWEEP_SD 6
#endif
constexpr int SD = TPGPU_SWEEP_SD;
// thread rows per block: the 32 x 8 node tile has 33 x 9 = 297 cells, so
// with TY thread rows 41 threads (two warps) evaluate a second cell while the
// other six warps wait at the slice barrier; TYT = 10 rows (320 threads)
// evaluate every cell in one round and leave two warps idle in the node pass,
// but fit two blocks per SM instead of three: 45.4 vs 42.7 ms per cfg-3 sweep
// in the ncu launch lists (profiles/r2u_*, r2o_*), level in the sweep A/B
// (profiles/r2q_ab.txt) -- 8 rows kept
#ifndef TPGPU_SWEEP_TYT
#define TPGPU_SWEEP_TYT 8
#endif
constexpr int TYT = TPGPU_SWEEP_TYT;
constexpr int SNT = TX * TYT;  // threads per block
// resident blocks per SM the registers are bounded for
#ifndef TPGPU_SWEEP_MINB
#define TPGPU_SWEEP_MINB (TYT > TY ? 2 : 3)
#endif

__device__ __forceinline__ void cp_async8(void* sdst, const void* g, bool ok) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(g), "r"(ok ? 8 : 0) : "memory");
}

template <bool WANT_G>
__global__ void __launch_bounds__(SNT, TPGPU_SWEEP_MINB) k_sweep_slices(
    const double* __restrict__ U, const double* __restrict__ halo_lo, const double* __restrict__ halo_hi,
    int sy0, int rows, double* __restrict__ G, double* __restrict__ part, int m, int c, int N, double inv_tau,
    const uint8_t* __restrict__ cell_mat, const MaterialDev* __restrict__ mats,
    const double* __restrict__ nu_hat, const double* __restrict__ mass,
    const double* __restrict__ src_prof, const double* __restrict__ src_time, int nsrc) {
  __shared__ double su[SD][TY + 2][TX + 2];
  __shared__ double cnu0[TY + 1][TX + 1], cdnu[TY + 1][TX + 1], cbs2[TY + 1][TX + 1], chat[TY + 1][TX + 1];
  __shared__ double wnu[2][2][TY + 1][TX + 1];  // nu_T / 2 (T1, T2 per cell) of two slices
  __shared__ double red[32];
  __shared__ double stime[SB * TP_MAX_MATERIALS];  // source amplitudes of the block's slices
  const size_t n = (size_t)m * m;
  const size_t nl = (size_t)rows * m;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
  const int x0 = blockIdx.x * TX, y0 = sy0 + blockIdx.y * TY;
  const int sbeg = blockIdx.z * SB, send = min(N, sbeg + SB);
  // staged tile elements of this thread (<= 2): source of vertex (X, Y) =
  // (x0 + lx, y0 + ly) in slice s = base + s * stride (main strip, or the
  // neighbours' halo rows), or zero (Dirichlet boundary / outside)
  constexpr int TN = (TY + 2) * (TX + 2);
  const int k0 = tid, k1 = tid + SNT;
  const double* sb[2];
  size_t sstr[2];
  bool sok[2];
  int sly[2], slx[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int k = e == 0 ? k0 : k1;
    const int ly = k / (TX + 2), lx = k % (TX + 2);
    sly[e] = ly;
    slx[e] = lx;
    const int x = x0 + lx - 1, y = y0 + ly - 1;  // node of vertex (X, Y)
    sb[e] = U;
    sstr[e] = nl;
    sok[e] = false;
    if (k < TN && x >= 0 && x < m && y >= 0 && y < m) {
      const int yl = y - sy0;
      if (yl < 0) {
        if (yl == -1 && halo_lo) { sb[e] = halo_lo + x; sstr[e] = m; sok[e] = true; }
      } else if (yl >= rows) {
        if (yl == rows && halo_hi) { sb[e] = halo_hi + x; sstr[e] = m; sok[e] = true; }
      } else {
        sb[e] = U + (size_t)yl * m + x;
        sok[e] = true;
      }
    }
  }
  // staged element pointers at slice sbeg, advanced by one slice per issue
  // (issue is called for consecutive slices)
  const double* sp0 = sok[0] ? sb[0] + (size_t)sbeg * sstr[0] : U;
  const double* sp1 = sok[1] ? sb[1] + (size_t)sbeg * sstr[1] : U;
  const size_t sst0 = sok[0] ? sstr[0] : 0, sst1 = sok[1] ? sstr[1] : 0;
  auto issue = [&](int sl) {
    if (sl < send) {
      double(*t)[TX + 2] = su[sl % SD];
      cp_async8(&t[sly[0]][slx[0]], sp0, sok[0]);
      if (k1 < TN) cp_async8(&t[sly[1]][slx[1]], sp1, sok[1]);
      sp0 += sst0;
      sp1 += sst1;
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
#pragma unroll
  for (int j = 0; j < SD - 1; ++j) issue(sbeg + j);
  for (int k = tid; k < (send - sbeg) * nsrc; k += SNT) stime[k] = src_time[(size_t)sbeg * nsrc + k];
  // per-cell material constants of the tile (+ halo cells)
  for (int k = tid; k < (TY + 1) * (TX + 1); k += SNT) {
    const int ly = k / (TX + 1), lx = k % (TX + 1);
    const int i = x0 + lx, j = y0 + ly;
    double a = 0, b = 0, bs = 1, h = 0;
    if (i < c && j < c) {
      const int mt = cell_mat[(size_t)j * c + i];
      const MaterialDev md = mats[mt];
      a = md.nu0;
      b = md.linear ? 0.0 : md.nu_inf - md.nu0;
      bs = md.bs2;
      h = WANT_G ? 0.5 * nu_hat[mt] : 0.0;
    }
    cnu0[ly][lx] = a;
    cdnu[ly][lx] = b;
    cbs2[ly][lx] = bs;
    chat[ly][lx] = h;
  }
  const int x = x0 + tx, y = y0 + ty;
  const bool own = ty < TY && x < m && y < sy0 + rows;
  const size_t i = own ? (size_t)y * m + x : 0;           // global
  const size_t il = own ? (size_t)(y - sy0) * m + x : 0;  // local
  const double mi = own ? mass[i] : 0.0;
  double prof[TP_MAX_MATERIALS];
#pragma unroll
  for (int r = 0; r < TP_MAX_MATERIALS; ++r) prof[r] = (own && r < nsrc) ? src_prof[r * n + i] : 0.0;
  double uprev = 0;
  if (own && mi != 0) uprev = U[(size_t)((sbeg + N - 1) % N) * nl + il];
  double* gp = WANT_G ? G + (size_t)sbeg * nl + il : nullptr;
  const double inv_c2 = 1.0 / ((double)c * (double)c);
  // slice-invariant operands in registers: the material law of this thread's
  // cells (cell pass) and nu_hat / 2 of the node's six incident triangles
  constexpr int NCELL = (TY + 1) * (TX + 1);
  const int kc0 = tid, kc1 = tid + SNT;
  __syncthreads();  // per-cell material constants staged
  double cl[2][3];
#pragma unroll
  for (int e = 0; e < (SNT >= NCELL ? 1 : 2); ++e) {
    const int k = e == 0 ? kc0 : kc1;
    const int cy = k / (TX + 1), cx = k - cy * (TX + 1);
    const bool ok = k < NCELL;
    // folded: nu/2 = (dnu/2) q / (q + Bs^2/c^2) + nu0/2 with q = |grad u|^2 / c^2
    cl[e][0] = ok ? 0.5 * cdnu[cy][cx] : 0.0;
    cl[e][1] = ok ? cbs2[cy][cx] * inv_c2 : 1.0;
    cl[e][2] = ok ? 0.5 * cnu0[cy][cx] : 0.0;
  }
  const int cxs[6] = {0, 0, -1, -1, -1, 0}, cys[6] = {0, 0, 0, -1, -1, -1};
  double hat[6];
#pragma unroll
  for (int t6 = 0; t6 < 6; ++t6) hat[t6] = (WANT_G && ty < TY) ? chat[ty + 1 + cys[t6]][tx + 1 + cxs[t6]] : 0.0;
  double r2 = 0;
  // nu(|grad u|) / 2 once per triangle: the (TY+1) x (TX+1) cells under the
  // node tile, two triangles each (T1 lower-right: d = (u10-u00, u11-u10);
  // T2 upper-left: d = (u11-u01, u01-u00)) -- each triangle is shared by
  // three nodes, which used to evaluate its law three times.  Software
  // pipelined: iteration s evaluates the cells of slice s+1 and gathers the
  // nodes of slice s, one barrier per slice (wnu double-buffered)
  auto cell_pass = [&](int sl) {
    const double(*t)[TX + 2] = su[sl % SD];
    double(*w)[TY + 1][TX + 1] = wnu[sl & 1];
#pragma unroll
    for (int e = 0; e < (SNT >= NCELL ? 1 : 2); ++e) {
      const int k = e == 0 ? kc0 : kc1;
      if (k < NCELL) {
        const int cy = k / (TX + 1), cx = k - cy * (TX + 1);
        const double u00 = t[cy][cx], u10 = t[cy][cx + 1], u01 = t[cy + 1][cx], u11 = t[cy + 1][cx + 1];
        const double ax = u10 - u00, ay = u11 - u10, bx = u11 - u01, by = u01 - u00;
        const double qa = fma(ax, ax, ay * ay), qb = fma(bx, bx, by * by);
        w[0][cy][cx] = fma(cl[e][0], qa * acc_rcp(qa + cl[e][1]), cl[e][2]);
        w[1][cy][cx] = fma(cl[e][0], qb * acc_rcp(qb + cl[e][1]), cl[e][2]);
      }
    }
  };
  asm volatile("cp.async.wait_group %0;\n" ::"n"(SD - 2) : "memory");
  __syncthreads();  // slice sbeg staged
  cell_pass(sbeg);
  for (int s = sbeg; s < send; ++s) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(SD - 3) : "memory");
    __syncthreads();  // slice s+1 staged; the cells of slice s evaluated; slice s-1's slot and weights free
    issue(s + SD - 1);
    if (s + 1 < send) cell_pass(s + 1);
    if (own) {
      const double(*t)[TX + 2] = su[s % SD];
      const double(*w)[TY + 1][TX + 1] = wnu[s & 1];
      const int lx = tx + 1, ly = ty + 1;
      const double uC = t[ly][lx], uE = t[ly][lx + 1], uW = t[ly][lx - 1];
      const double uN = t[ly + 1][lx], uS = t[ly - 1][lx];
      // the six incident triangles (cell, type): contribution dx*sx + dy*sy
      // T1(X,Y) -(uE-uC); T2(X,Y) -(uN-uC); T1(X-1,Y) (uC-uW)-(uN-uC);
      // T1(X-1,Y-1) uC-uS; T2(X-1,Y-1) uC-uW; T2(X,Y-1) -(uE-uC)+(uC-uS)
      const double con[6] = {-(uE - uC), -(uN - uC), (uC - uW) - (uN - uC), uC - uS, uC - uW, -(uE - uC) + (uC - uS)};
      const int tt[6] = {0, 1, 0, 0, 1, 1};
      double ku = 0, kh = 0;
#pragma unroll
      for (int t6 = 0; t6 < 6; ++t6) {
        ku = fma(w[tt[t6]][ly + cys[t6]][lx + cxs[t6]], con[t6], ku);
        if (WANT_G) kh = fma(hat[t6], con[t6], kh);
      }
      double f = 0;
#pragma unroll
      for (int r = 0; r < TP_MAX_MATERIALS; ++r)
        if (r < nsrc) f = fma(stime[(s - sbeg) * nsrc + r], prof[r], f);
      if (WANT_G) {
        *gp = f + kh - ku;
        gp += nl;
      }
      const double mdu = mi != 0 ? mi * ((uC - uprev) * inv_tau) : 0.0;
      const double res = f - mdu - ku;
      r2 = fma(res, res, r2);
      uprev = uC;
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  const double tot = block_sum(r2, red);
  if (tid == 0) part[((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = tot;
}

// Row-walking form of the sweep kernel (the default; TPGPU_SWEEP_TILE=1 keeps
// k_sweep_slices): one warp owns a column strip of RW_LANES = 30 nodes (32
// lanes: the strip plus one halo column on each side), a chunk of node rows
// and SG consecutive slices, and walks its rows upward with u rows y-1, y,
// y+1 (and y+2 in flight) of its slices in registers.  East/west
// neighbours and the west triangles come by warp shuffles, the triangles of
// the cell row below are carried from the previous row: no shared-memory
// tile and no block barrier (k_sweep_slices is bound by its per-slice
// barrier and its shared-memory wavefronts).  nu(|grad u|) is
// evaluated once per triangle (the halo lanes' cells excepted) behind one
// warp vote per row, and skipped where no lane of the strip sits in a
// nonlinear cell: there the weight is nu0/2, exactly what the fma gives with
// dnu = 0.  The row body is branch-free otherwise (halo lanes and slices past
// N compute unused values; stores and the residual sum are predicated): the
// kernel is instruction-issue bound, and divergent branches cost a
// convergence check before every shuffle group (27.5 -> 24.8 -> 20.3 ms at
// cfg 3 with the u-row ring below, profiles/r2zi_ab.txt, r2zk_ab.txt).  Slice-invariant row data (cell materials, lumped
// mass, source profiles) is loaded once per row for the SG slices, and only
// in the strips/chunks where it is nonzero (host-built region flags);
// u^{s-1} is the previous slice's register row (the group's first slice
// reads slice s0-1 where there is mass).  Per node the formulas and the
// summation order are k_sweep_slices', so U-> G is bitwise the same; the
// residual partials are summed per block in another fixed order.
constexpr int RW_LANES = 30;
constexpr int RW_WARPS = 4;  // warps per block: consecutive slice groups of one region
#ifndef TPGPU_SWEEP_SG
#define TPGPU_SWEEP_SG 4
#endif
#ifndef TPGPU_SWEEP_H
#define TPGPU_SWEEP_H 64
#endif

// source row of node row y (global) for the lane's column: nullptr = zero
// (Dirichlet boundary, outside the strip and its halo rows); `st` = stride
// between consecutive slices
__device__ __forceinline__ const double* rw_row(const double* U, const double* lo, const double* hi, int sy0,
                                                int rows, int m, size_t nl, int y, int x, bool colok, size_t& st) {
  st = 0;
  if (!colok || y < 0 || y >= m) return nullptr;
  const int ly = y - sy0;
  if (ly >= 0 && ly < rows) {
    st = nl;
    return U + (size_t)ly * m + x;
  }
  if (ly == -1 && lo) {
    st = m;
    return lo + x;
  }
  if (ly == rows && hi) {
    st = m;
    return hi + x;
  }
  return nullptr;
}

#ifndef TPGPU_SWEEP_MINB_RW
#define TPGPU_SWEEP_MINB_RW 4
#endif
// rows of u staged ahead through a private per-warp shared-memory ring by
// per-lane cp.async copies (0: row y+2 is prefetched into registers instead).
// A lane reads back only what it copied itself, so cp.async.wait_group is
// the only synchronisation; RA + 2 slots, the overwritten slot was read two
// rows earlier.  Zero rows (boundary, outside the strip) are zero-filled by
// the copy (src-size 0).
#ifndef TPGPU_SWEEP_RA
#define TPGPU_SWEEP_RA 4
#endif
constexpr int RW_RA = TPGPU_SWEEP_RA;
constexpr int RW_SLOTS = RW_RA > 0 ? RW_RA + 2 : 1;
template <bool WANT_G, int SG, int NS>  // NS: source profiles held per node (>= nsrc)
__global__ void __launch_bounds__(32 * RW_WARPS, TPGPU_SWEEP_MINB_RW) k_sweep_rows(
    const double* __restrict__ U, const double* __restrict__ halo_lo, const double* __restrict__ halo_hi,
    int sy0, int rows, double* __restrict__ G, double* __restrict__ part, int m, int c, int N, double inv_tau,
    const uint8_t* __restrict__ cell_mat, const MaterialDev* __restrict__ mats,
    const double* __restrict__ nu_hat, const double* __restrict__ mass,
    const double* __restrict__ src_prof, const double* __restrict__ src_time, int nsrc,
    const uint8_t* __restrict__ rflags, int H, int nstrips, int nsgb) {
  __shared__ double tab[4][TP_MAX_MATERIALS];  // per material: dnu/2, Bs^2/c^2, nu0/2, nu_hat/2
  __shared__ double stime[RW_WARPS][SG][TP_MAX_MATERIALS];
  __shared__ double red[RW_WARPS];
  __shared__ double ring[RW_RA > 0 ? RW_WARPS : 1][RW_SLOTS][RW_RA > 0 ? SG : 1][RW_RA > 0 ? 32 : 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const size_t n = (size_t)m * m;
  const size_t nl = (size_t)rows * m;
  const double inv_c2 = 1.0 / ((double)c * (double)c);
  if (threadIdx.x < TP_MAX_MATERIALS) {
    const MaterialDev md = mats[threadIdx.x];
    tab[0][threadIdx.x] = md.linear ? 0.0 : 0.5 * (md.nu_inf - md.nu0);
    tab[1][threadIdx.x] = md.bs2 * inv_c2;
    tab[2][threadIdx.x] = 0.5 * md.nu0;
    tab[3][threadIdx.x] = WANT_G ? 0.5 * nu_hat[threadIdx.x] : 0.0;
  }
  const int region = blockIdx.x / nsgb, sgb = blockIdx.x - region * nsgb;
  const int strip = region % nstrips, chunk = region / nstrips;
  const int s0 = (sgb * RW_WARPS + w) * SG;
  const int ns = max(0, min(SG, N - s0));
  for (int k = lane; k < SG * TP_MAX_MATERIALS; k += 32) {
    const int sl = k / TP_MAX_MATERIALS, r = k - sl * TP_MAX_MATERIALS;
    stime[w][sl][r] = (sl < ns && r < nsrc) ? src_time[(size_t)(s0 + sl) * nsrc + r] : 0.0;
  }
  __syncthreads();
  const int flags = rflags[region];
  const bool hasm = flags & 1, hasf = flags & 2;
  const int X = strip * RW_LANES + lane;  // vertex column (node x = X - 1)
  const int x = X - 1;
  const bool colok = X >= 1 && X <= m;
  const bool own = lane >= 1 && lane <= RW_LANES && colok;
  const bool cellok = X <= c - 1;  // this lane's cell column exists
  const int ya = sy0 + chunk * H, yb = min(sy0 + rows, ya + H);
  double r2 = 0;
#ifdef TPGPU_SWEEP_NSGUARD
  if (ns > 0)
#endif
  {
    // (no `ns > 0` guard: every access below is predicated on k < ns, and a
    // branch on the warp index makes the compiler treat the whole row loop as
    // possibly divergent -- a convergence check before every shuffle group)
    // u of row y for the group's slices (zero-filled), material of cell (X, j)
    auto load_u = [&](int y, double (&v)[SG]) {
      size_t st;
      const double* p = rw_row(U, halo_lo, halo_hi, sy0, rows, m, nl, y, x, colok, st);
#pragma unroll
      for (int k = 0; k < SG; ++k) v[k] = (p && k < ns) ? __ldg(p + (size_t)(s0 + k) * st) : 0.0;
    };
    // the same row into the ring slot at byte offset `so` (asynchronous).
    // Rows ya+2 .. yb-1 are interior rows of this rank's strip: a running
    // pointer (`pint`, one row per call) and the slice stride nl; row yb can be
    // a halo or boundary row (rw_row, selected by predicates: measured faster
    // than a direct load of that row when it is due, 20.3 vs 21.6 ms at cfg 3);
    // rows past yb are never read
    const unsigned ring_lane = (unsigned)__cvta_generic_to_shared(&ring[w][0][0][RW_RA > 0 ? lane : 0]);
    constexpr unsigned SLOT_B = SG * 32 * 8;
    const double* pint = U + (size_t)s0 * nl + (size_t)(ya + 2 - sy0) * m + x;
    auto stage_u = [&](int y, unsigned so) {
      const double* q = pint;
      size_t st = nl;
      bool ok = colok && y < yb;
      if (y == yb) {
        q = rw_row(U, halo_lo, halo_hi, sy0, rows, m, nl, y, x, colok, st);
        ok = q != nullptr;
        if (ok) q += (size_t)s0 * st;
      }
      pint += m;
#pragma unroll
      for (int k = 0; k < SG; ++k) {
        const bool okk = ok && k < ns;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(ring_lane + so + k * 256), "l"(okk ? q : U),
                     "r"(okk ? 8 : 0)
                     : "memory");
        q += st;
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    auto load_mat = [&](int j) -> int { return (cellok && j >= 0 && j < c) ? (int)__ldg(cell_mat + (size_t)j * c + X) : -1; };
    // row-invariant per-node data for node row y (mass, source profiles, u^{s0-1})
    auto load_node = [&](int y, double& mi, double (&pr)[NS], double& up) {
      const bool ok = own && y < yb;
      const size_t i = (size_t)y * m + x;
      mi = 0.0;
      up = 0.0;
      if (hasm && ok) {
        mi = __ldg(mass + i);
        if (mi != 0.0) up = __ldg(U + (size_t)((s0 + N - 1) % N) * nl + (size_t)(y - sy0) * m + x);
      }
#pragma unroll
      for (int r = 0; r < NS; ++r) pr[r] = (hasf && ok && r < nsrc) ? __ldg(src_prof + r * n + i) : 0.0;
    };
    // the two triangles of cell (X, j) from u at its corners
    auto cell = [&](int mt, double u00, double u10, double u01, double u11, double& w1, double& w2) {
      if (mt < 0) {
        w1 = w2 = 0.0;
        return;
      }
      const double c0 = tab[0][mt], c1 = tab[1][mt], c2 = tab[2][mt];
      if (c0 == 0.0) {  // linear material: fma(0, finite, nu0/2) == nu0/2
        w1 = w2 = c2;
        return;
      }
      const double ax = u10 - u00, ay = u11 - u10, bx = u11 - u01, by = u01 - u00;
      const double qa = fma(ax, ax, ay * ay), qb = fma(bx, bx, by * by);
      w1 = fma(c0, qa * acc_rcp(qa + c1), c2);
      w2 = fma(c0, qb * acc_rcp(qb + c1), c2);
    };
    constexpr unsigned FULL = 0xffffffffu;
    double uS[SG], uC[SG], uN[SG], uQ[SG];
    double b2[SG], t3[SG], t4[SG];  // lower cell row: own T2, west T1, west T2
    load_u(ya - 1, uS);
    load_u(ya, uC);
    int matL = load_mat(ya);  // cell row below node row ya
    load_u(ya + 1, uN);
    int matU = load_mat(ya + 1);
    double mi, pr[NS], up;
    load_node(ya, mi, pr, up);
    {
#pragma unroll
      for (int k = 0; k < SG; ++k) {
        const double e0 = __shfl_down_sync(FULL, uS[k], 1), e1 = __shfl_down_sync(FULL, uC[k], 1);
        double w1, w2;
        cell(matL, uS[k], e0, uC[k], e1, w1, w2);
        b2[k] = w2;
        t3[k] = __shfl_up_sync(FULL, w1, 1);
        t4[k] = __shfl_up_sync(FULL, w2, 1);
      }
    }
    double hb = matL >= 0 ? tab[3][matL] : 0.0;
    double h3 = __shfl_up_sync(FULL, hb, 1);
    double* gp = WANT_G ? G + (size_t)(ya - sy0) * m + x : nullptr;
    unsigned slot_r = 0, slot_w = (RW_RA % RW_SLOTS) * SLOT_B;  // ring byte offset of row y+2 / of row y+2+RA
    if constexpr (RW_RA > 0) {
#pragma unroll
      for (int j = 0; j < RW_RA; ++j) stage_u(ya + 2 + j, j * SLOT_B);
    }
    if (WANT_G) gp += (size_t)s0 * nl;
    for (int y = ya; y < yb; ++y) {
      // in flight: row y+2 and its cell row, the next row's node data
      if constexpr (RW_RA > 0) {
        asm volatile("cp.async.wait_group %0;\n" ::"n"(RW_RA > 0 ? RW_RA - 1 : 0) : "memory");
        stage_u(y + 2 + RW_RA, slot_w);
        slot_w = slot_w + SLOT_B == RW_SLOTS * SLOT_B ? 0 : slot_w + SLOT_B;
      } else {
        load_u(y + 2, uQ);
      }
      const int matQ = load_mat(y + 2);
      double mi2, pr2[NS], up2;
      load_node(y + 1, mi2, pr2, up2);
      const double ha = matU >= 0 ? tab[3][matU] : 0.0;
      const double hau = __shfl_up_sync(FULL, ha, 1);
      // the row's cell material is the same for the SG slices: coefficients
      // once per row, and one warp-uniform branch around the material law
      // (no lane of the strip in a nonlinear cell: weights are nu0/2)
      const int mtc = max(matU, 0);
      const double c0 = tab[0][mtc], c1 = tab[1][mtc], c2 = matU >= 0 ? tab[2][mtc] : 0.0;
      const bool nlin = matU >= 0 && c0 != 0.0;
      const bool anynl = __any_sync(FULL, nlin);
      double* gk = gp;  // G of (slice s0 + k, row y)
#pragma unroll
      for (int k = 0; k < SG; ++k) {
        const double uc = uC[k];
        const double uE = __shfl_down_sync(FULL, uc, 1), uW = __shfl_up_sync(FULL, uc, 1);
        const double un = uN[k], us = uS[k];
        const double uNE = __shfl_down_sync(FULL, un, 1);
        double a1 = c2, a2 = c2;
        if (anynl) {
          const double ax = uE - uc, ay = uNE - uE, bx = uNE - un, by = un - uc;
          const double qa = fma(ax, ax, ay * ay), qb = fma(bx, bx, by * by);
          const double n1 = fma(c0, qa * acc_rcp(qa + c1), c2), n2 = fma(c0, qb * acc_rcp(qb + c1), c2);
          a1 = nlin ? n1 : c2;
          a2 = nlin ? n2 : c2;
        }
        const double a1u = __shfl_up_sync(FULL, a1, 1), a2u = __shfl_up_sync(FULL, a2, 1);
        {
          // every lane evaluates its node (halo lanes and slices past N: values unused)
          const bool act = own && k < ns;
          const double con[6] = {-(uE - uc), -(un - uc), (uc - uW) - (un - uc), uc - us, uc - uW,
                                 -(uE - uc) + (uc - us)};
          const double wt[6] = {a1, a2, a1u, t3[k], t4[k], b2[k]};
          const double hh[6] = {ha, ha, hau, h3, h3, hb};
          double ku = 0, kh = 0;
#pragma unroll
          for (int t6 = 0; t6 < 6; ++t6) {
            ku = fma(wt[t6], con[t6], ku);
            if (WANT_G) kh = fma(hh[t6], con[t6], kh);
          }
          double f = 0;
          if (hasf) {
#pragma unroll
            for (int r = 0; r < NS; ++r)
              if (r < nsrc) f = fma(stime[w][k][r], pr[r], f);
          }
          if (WANT_G && act) __stcs(gk, f + kh - ku);
          if (WANT_G) gk += nl;
          const double uprev = k == 0 ? up : uC[k > 0 ? k - 1 : 0];
          const double mdu = mi != 0 ? mi * ((uc - uprev) * inv_tau) : 0.0;
          const double res = f - mdu - ku;
          r2 = act ? fma(res, res, r2) : r2;
        }
        b2[k] = a2;
        t3[k] = a1u;
        t4[k] = a2u;
      }
#pragma unroll
      for (int k = 0; k < SG; ++k) {
        uS[k] = uC[k];
        uC[k] = uN[k];
        if constexpr (RW_RA > 0) {  // row y+2, landed (wait_group above)
          asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(uN[k]) : "r"(ring_lane + slot_r + k * 256) : "memory");
        } else {
          uN[k] = uQ[k];
        }
      }
      if constexpr (RW_RA > 0) slot_r = slot_r + SLOT_B == RW_SLOTS * SLOT_B ? 0 : slot_r + SLOT_B;
      matU = matQ;
      hb = ha;
      h3 = hau;
      mi = mi2;
      up = up2;
#pragma unroll
      for (int r = 0; r < NS; ++r) pr[r] = pr2[r];
      if (WANT_G) gp += m;
    }
  }
  if constexpr (RW_RA > 0) asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  // fixed-order block reduction: butterfly within the warp, warps in order
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) r2 += __shfl_xor_sync(0xffffffffu, r2, o);
  if (lane == 0) red[w] = r2;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0;
#pragma unroll
    for (int k = 0; k < RW_WARPS; ++k) s += red[k];
    part[blockIdx.x] = s;
  }
}

__global__ void k_reduce_sum(const double* __restrict__ in, int count, double* __restrict__ out) {
  __shared__ double sh[32];
  double v = 0;
  for (int k = threadIdx.x; k < count; k += blockDim.x) v += in[k];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) s += sh[w];
    *out = s;
  }
}

// Element-stencil assembly: per node, the 7-point row of
//   sum_T (1/2) s_a^T Q_T s_b,   Q_T = a_T I + b_T g g^T  (g = grad u on T).
// Frozen stiffness: a_T = nu_hat, b_T = 0.  Newton Jacobian: a_T = nu(s),
// b_T = nu'(s)/s (0 at s = 0), s = |g|  (assembly.hpp:153-177).
// Output st[d*n + i] for batch `blockIdx.z` (stride 7n).
template <bool JAC>
__global__ void __launch_bounds__(256) k_element_stencil(
    const double* __restrict__ U, double* __restrict__ st, int m, int c,
    const uint8_t* __restrict__ cell_mat, const MaterialDev* __restrict__ mats,
    const double* __restrict__ nu_hat) {
  const size_t n = (size_t)m * m;
  const int b = blockIdx.z;
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int x = (int)(i % m), y = (int)(i / m);
  const int X = x + 1, Y = y + 1;
  const double* us = JAC ? U + b * n : nullptr;
  const double cc = (double)c;
  // triangle list: (cell dx, cell dy, type, local a); sign vectors per type
  // T1: s0=(-1,0) s1=(1,-1) s2=(0,1);  T2: s0=(0,-1) s1=(1,0) s2=(-1,1)
  const int tcx[6] = {0, 0, -1, -1, -1, 0};
  const int tcy[6] = {0, 0, 0, -1, -1, -1};
  const int ttp[6] = {0, 1, 0, 0, 1, 1};
  const int tla[6] = {0, 0, 1, 2, 1, 2};
  double row[7] = {0, 0, 0, 0, 0, 0, 0};
  for (int k = 0; k < 6; ++k) {
    const int ci = X + tcx[k], cj = Y + tcy[k];
    const int tp = ttp[k], a = tla[k];
    const MaterialDev mt = mats[cell_mat[(size_t)cj * c + ci]];
    // vertices of the triangle (vertex coords) and their sign vectors
    int vx[3], vy[3];
    vx[0] = ci; vy[0] = cj;
    if (tp == 0) { vx[1] = ci + 1; vy[1] = cj; vx[2] = ci + 1; vy[2] = cj + 1; }
    else         { vx[1] = ci + 1; vy[1] = cj + 1; vx[2] = ci; vy[2] = cj + 1; }
    const int sxa[2][3] = {{-1, 1, 0}, {0, 1, -1}};
    const int sya[2][3] = {{0, -1, 1}, {-1, 0, 1}};
    double qa, qb = 0, gx = 0, gy = 0;
    if (JAC) {
      const double u0 = vertex_u(us, m, vx[0], vy[0]);
      const double u1 = vertex_u(us, m, vx[1], vy[1]);
      const double u2 = vertex_u(us, m, vx[2], vy[2]);
      gx = cc * (sxa[tp][0] * u0 + sxa[tp][1] * u1 + sxa[tp][2] * u2);
      gy = cc * (sya[tp][0] * u0 + sya[tp][1] * u1 + sya[tp][2] * u2);
      const double s2 = gx * gx + gy * gy;
      qa = nu_of(mt, s2);
      if (!mt.linear && s2 > 0) {
        // nu'(s)/s = 2 (nu_inf - nu0) Bs^2 / (s^2 + Bs^2)^2
        const double den = s2 + mt.bs2;
        qb = 2.0 * (mt.nu_inf - mt.nu0) * mt.bs2 / (den * den);
      }
    } else {
      qa = nu_hat[cell_mat[(size_t)cj * c + ci]];
    }
    const double sax = sxa[tp][a], say = sya[tp][a];
    // area * grad phi_a^T Q grad phi_b with grad phi = c s, area = 1/(2c^2):
    //   (1/2) [qa (s_a.s_b) + qb (g.s_a)(g.s_b)],  g the true gradient.
    const double gsa = gx * sax + gy * say;
    for (int bb = 0; bb < 3; ++bb) {
      const double sbx = sxa[tp][bb], sby = sya[tp][bb];
      double v = qa * (sax * sbx + say * sby);
      if (JAC) v += qb * gsa * (gx * sbx + gy * sby);
      v *= 0.5;
      const int ddx = vx[bb] - X, ddy = vy[bb] - Y;
      int d;
      if (ddx == 0 && ddy == 0) d = SC;
      else if (ddx == -1 && ddy == 0) d = SW_;
      else if (ddx == 1 && ddy == 0) d = SE_;
      else if (ddx == 0 && ddy == -1) d = SS_;
      else if (ddx == 0 && ddy == 1) d = SN_;
      else if (ddx == -1 && ddy == -1) d = SSW;
      else d = SNE;
      row[d] += v;
    }
  }
  // drop couplings to Dirichlet vertices
  for (int d = 1; d < 7; ++d) {
    const int nx = x + dir_dx(d), ny = y + dir_dy(d);
    if (nx < 0 || nx >= m || ny < 0 || ny >= m) row[d] = 0;
  }
  double* o = st + (size_t)b * 7 * n;
  for (int d = 0; d < 7; ++d) o[d * n + i] = row[d];
}

}  // namespace

void reduce_sum_dev(Problem& p, const double* partials, int count, double* out) {
  k_reduce_sum<<<1, 1024, 0, p.stream>>>(partials, count, out);
  TP_LAUNCHED(&p);
}

double reduce_sum(Problem& p, const double* partials, int count) {
  k_reduce_sum<<<1, 1024, 0, p.stream>>>(partials, count, p.red.get());
  TP_LAUNCHED(&p);
  TP_CUDA(cudaMemcpyAsync(p.h_scalars, p.red.get(), sizeof(double), cudaMemcpyDeviceToHost, p.stream));
  TP_CUDA(cudaStreamSynchronize(p.stream));
  return p.h_scalars[0];
}

// sum_n (a^n - b^n)^T K_hat (a^n - b^n) over `count` slices (block_norm_khat,
// periodic.hpp:70-75, of a difference of iterates): the frozen stiffness on
// the right-triangle grid is the graph Laplacian of its edge weights
// (we: vertex (X,Y)-(X+1,Y), wn: (X,Y)-(X,Y+1); Dirichlet vertices are zero),
// so x^T K_hat x = sum over edges of w (x_i - x_j)^2.  Each node owns its east
// and north edges, plus the west / south edge when that neighbour is on the
// boundary.  One partial per block, reduced in fixed order.
__global__ void __launch_bounds__(256) k_khat_quadform(const double* __restrict__ a, const double* __restrict__ b,
                                                       const double* __restrict__ we, const double* __restrict__ wn,
                                                       int m, int c, int count, double* __restrict__ part) {
  __shared__ double red[32];
  const size_t n = (size_t)m * m;
  const size_t total = n * count;
  const int V = c + 1;
  double acc = 0;
  for (size_t g = (size_t)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += (size_t)gridDim.x * blockDim.x) {
    const size_t sl = g / n, i = g - sl * n;
    const int x = (int)(i % m), y = (int)(i / m);  // vertex (X, Y) = (x + 1, y + 1)
    const double* A = a + sl * n;
    const double* B = b ? b + sl * n : nullptr;  // b == nullptr: the norm of a itself
    const double v = A[i] - (B ? B[i] : 0.0);
    const int X = x + 1, Y = y + 1;
    const double ve = x + 1 < m ? A[i + 1] - (B ? B[i + 1] : 0.0) : 0.0;
    const double vn = y + 1 < m ? A[i + m] - (B ? B[i + m] : 0.0) : 0.0;
    double t = we[(size_t)Y * V + X] * (ve - v) * (ve - v) + wn[(size_t)Y * V + X] * (vn - v) * (vn - v);
    if (x == 0) t += we[(size_t)Y * V + 0] * v * v;
    if (y == 0) t += wn[(size_t)0 * V + X] * v * v;
    acc += t;
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s2 = 0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) s2 += red[w];
    part[blockIdx.x] = s2;
  }
}

double Problem::khat_norm_diff(const double* a, const double* b) {
  require(d_we.get() != nullptr, "K_hat norm: frequency solver not built");
  require(!sharded(), "K_hat norm: single-rank problems only");
  const int blocks = 4 * num_sms;
  part.ensure((size_t)blocks);
  k_khat_quadform<<<blocks, 256, 0, stream>>>(a, b, d_we.get(), d_wn.get(), m, c, N, part.get());
  TP_LAUNCHED(this);
  return std::sqrt(std::max(0.0, reduce_sum(*this, part.get(), blocks)));
}

void Problem::apply_k_dev(const double* u, double* out, int count) {
  dim3 grid((m + TX - 1) / TX, (m + TY - 1) / TY, count);
  k_apply_k<<<grid, dim3(TX, TY), 0, stream>>>(u, out, m, c, d_cell_mat.get(), d_mat.get());
  TP_LAUNCHED(this);
}

static size_t sweep_partials(int m, int N) {
  return (size_t)((m + TX - 1) / TX) * ((m + TY - 1) / TY) * N;
}

// region flags of the row-walking sweep kernel: per (row chunk, column strip)
// of this rank's node rows, bit 0 = some node has mass, bit 1 = some node
// has a source profile
static std::vector<uint8_t> sweep_region_flags(const Problem& p, int H, int nstrips, int nchunks) {
  std::vector<uint8_t> f((size_t)nstrips * nchunks, 0);
  const int nsrc = (int)p.src_mats.size();
  for (int y = p.sh.y0; y < p.sh.y1; ++y)
    for (int x = 0; x < p.m; ++x) {
      const size_t i = (size_t)y * p.m + x;
      uint8_t b = p.mass[i] != 0.0 ? 1 : 0;
      for (int r = 0; r < nsrc; ++r)
        if (p.src_prof[(size_t)r * p.n + i] != 0.0) b |= 2;
      f[(size_t)((y - p.sh.y0) / H) * nstrips + x / RW_LANES] |= b;
    }
  return f;
}

double Problem::residual_and_rhs(bool want_rhs) {
  const int rows = sh.y1 - sh.y0;
  if (sharded()) exchange_halo();
  const int nsrc = (int)src_mats.size();
  require(nsrc <= TP_MAX_MATERIALS, "sweep: too many source materials");
  require(!want_rhs || nu_hat_set, "fixed-point sweep: nu_hat not installed");
  const double* lo = sharded() ? halo_lo.get() : nullptr;
  const double* hi = sharded() ? halo_hi.get() : nullptr;
  // k_sweep_slices (32x8 node tiles in shared memory) on request
  static const bool tile = std::getenv("TPGPU_SWEEP_TILE") != nullptr;
  size_t np;
  if (!tile) {
    constexpr int SG = TPGPU_SWEEP_SG, H = TPGPU_SWEEP_H;
    const int nstrips = (m + RW_LANES - 1) / RW_LANES, nchunks = (rows + H - 1) / H;
    const int nsgb = (N + SG * RW_WARPS - 1) / (SG * RW_WARPS);
    if (rflags_key != H) {
      const std::vector<uint8_t> f = sweep_region_flags(*this, H, nstrips, nchunks);
      d_rflags.alloc(f.size());
      TP_CUDA(cudaMemcpy(d_rflags.get(), f.data(), f.size(), cudaMemcpyHostToDevice));
      rflags_key = H;
    }
    const dim3 grid((unsigned)((size_t)nstrips * nchunks * nsgb));
    np = grid.x;
    part.ensure(np);
#define TP_SWEEP_ROWS(WG, NS)                                                                                   \
  k_sweep_rows<WG, SG, NS><<<grid, 32 * RW_WARPS, 0, stream>>>(                                                 \
      U.get(), lo, hi, sh.y0, rows, WG ? G.get() : nullptr, part.get(), m, c, N, 1.0 / tau, d_cell_mat.get(), \
      d_mat.get(), d_nu_hat.get(), d_mass.get(), d_src_prof.get(), d_src_time.get(), nsrc, d_rflags.get(), H,  \
      nstrips, nsgb)
    if (nsrc <= 2) {
      if (want_rhs) TP_SWEEP_ROWS(true, 2); else TP_SWEEP_ROWS(false, 2);
    } else {
      if (want_rhs) TP_SWEEP_ROWS(true, TP_MAX_MATERIALS); else TP_SWEEP_ROWS(false, TP_MAX_MATERIALS);
    }
#undef TP_SWEEP_ROWS
  } else {
    dim3 grid((m + TX - 1) / TX, (rows + TY - 1) / TY, (N + SB - 1) / SB);
    np = (size_t)grid.x * grid.y * grid.z;
    part.ensure(np);
    if (want_rhs) {
      k_sweep_slices<true><<<grid, dim3(TX, TYT), 0, stream>>>(
          U.get(), lo, hi, sh.y0, rows, G.get(), part.get(), m, c, N, 1.0 / tau, d_cell_mat.get(), d_mat.get(),
          d_nu_hat.get(), d_mass.get(), d_src_prof.get(), d_src_time.get(), nsrc);
    } else {
      k_sweep_slices<false><<<grid, dim3(TX, TYT), 0, stream>>>(
          U.get(), lo, hi, sh.y0, rows, nullptr, part.get(), m, c, N, 1.0 / tau, d_cell_mat.get(), d_mat.get(),
          d_nu_hat.get(), d_mass.get(), d_src_prof.get(), d_src_time.get(), nsrc);
    }
  }
  TP_LAUNCHED(this);
  reduce_sum_dev(*this, part.get(), (int)np, red.get());
  global_sum_dev(red.get(), 1, red.get() + 1);
  TP_CUDA(cudaMemcpyAsync(h_scalars, red.get() + 1, sizeof(double), cudaMemcpyDeviceToHost, stream));
  TP_CUDA(cudaStreamSynchronize(stream));
  const double r = std::sqrt(h_scalars[0]);
  if (want_rhs) {  // the fixed-point residual history (warm-start extrapolation, problem.cu)
    resid_prev = resid_last;
    resid_last = r;
  }
  return r;
}

// block residual of a device state u into r and its norm (block_l2)
double residual_norm_dev(Problem& p, const double* u, double* r) {
  p.residual_dev(u, r, p.N);
  return std::sqrt(reduce_sum(p, p.part.get(), (int)sweep_partials(p.m, p.N)));
}

void Problem::residual_dev(const double* u, double* r, int count_slices) {
  require(count_slices == N, "residual: needs all slices");
  require(!sharded(), "residual of a host state: single-rank problems only");
  dim3 grid((m + TX - 1) / TX, (m + TY - 1) / TY, N);
  part.ensure(sweep_partials(m, N));
  k_sweep_fused<false, true><<<grid, dim3(TX, TY), 0, stream>>>(
      u, nullptr, nullptr, 0, m, nullptr, r, part.get(), m, c, N, 1.0 / tau, d_cell_mat.get(), d_mat.get(),
      d_nu_hat.get(), d_mass.get(), d_src_prof.get(), d_src_time.get(), (int)src_mats.size());
  TP_LAUNCHED(this);
}

void launch_element_stencil(Problem& p, bool jacobian, const double* U, double* st, int batches) {
  dim3 grid((p.n + 255) / 256, 1, batches);
  if (jacobian)
    k_element_stencil<true><<<grid, 256, 0, p.cur_stream()>>>(U, st, p.m, p.c, p.d_cell_mat.get(),
                                                         p.d_mat.get(), nullptr);
  else
    k_element_stencil<false><<<grid, 256, 0, p.cur_stream()>>>(nullptr, st, p.m, p.c, p.d_cell_mat.get(),
                                                          p.d_mat.get(), p.d_nu_hat.get());
  TP_LAUNCHED(&p);
}

// ---- Newton helpers (static_init) -------------------------------------

namespace {

// r_s = f_s - K(u_s + alpha_s d_s) for the batch slices listed in `slices`;
// writes trial u and r, and per-block partial ||r||^2.
__global__ void __launch_bounds__(TX * TY) k_newton_residual(
    const double* __restrict__ Ub, const double* __restrict__ Db, const double* __restrict__ alpha,
    double* __restrict__ Ut, double* __restrict__ Rt, double* __restrict__ part,
    const int* __restrict__ slice_of, const int* __restrict__ active, int m, int c,
    const uint8_t* __restrict__ cell_mat, const MaterialDev* __restrict__ mats,
    const double* __restrict__ src_prof, const double* __restrict__ src_time, int nsrc,
    const double* __restrict__ rhs, double ms, const double* __restrict__ mass) {
  __shared__ Tile t;
  __shared__ double red[32];
  const size_t n = (size_t)m * m;
  const int b = blockIdx.z;
  const size_t pidx = ((size_t)b * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  if (!active[b]) {
    if (threadIdx.x == 0 && threadIdx.y == 0) part[pidx] = 0;
    return;
  }
  const int s = slice_of[b];
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const double a = alpha ? alpha[b] : 0.0;
  const StripView sv{nullptr, nullptr, 0, m};
  tile_load<true, false>(t, Ub + b * n, sv, Db ? Db + b * n : nullptr, a, m, c, x0, y0, cell_mat, mats,
                         nullptr);
  const int x = x0 + threadIdx.x, y = y0 + threadIdx.y;
  double r2 = 0;
  if (x < m && y < m) {
    const size_t i = (size_t)y * m + x;
    double res;
    if (rhs) {
      // time step (newton_elliptic with mass_scale, solvers.hpp:139-146): rhs - ms M u - K(u)
      res = rhs[b * n + i] - ms * (mass[i] * t.u[threadIdx.y + 1][threadIdx.x + 1]) -
            gather<0>(t, threadIdx.x, threadIdx.y);
    } else {
      double f = 0;
      for (int r = 0; r < nsrc; ++r) f += src_time[s * nsrc + r] * src_prof[r * n + i];
      res = f - gather<0>(t, threadIdx.x, threadIdx.y);
    }
    Rt[b * n + i] = res;
    if (Ut) Ut[b * n + i] = t.u[threadIdx.y + 1][threadIdx.x + 1];
    r2 = res * res;
  }
  const double tot = block_sum(r2, red);
  if (threadIdx.x == 0 && threadIdx.y == 0) part[pidx] = tot;
}

// per-batch sums of partials (fixed order)
__global__ void k_reduce_batches(const double* __restrict__ part, int per, double* __restrict__ out) {
  __shared__ double sh[32];
  const int b = blockIdx.x;
  double v = 0;
  for (int k = threadIdx.x; k < per; k += blockDim.x) v += part[(size_t)b * per + k];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) s += sh[w];
    out[b] = s;
  }
}

}  // namespace

// Evaluate r = f - K(u + alpha d) for a batch; returns per-batch ||r||^2 into
// host `norms2` (synchronising).
void newton_residual(Problem& p, const double* Ub, const double* Db, const double* d_alpha,
                     double* Ut, double* Rt, const int* d_slice_of, const int* d_active, int batches,
                     double* norms2_host, DevBuf<double>& part, DevBuf<double>& red, const double* rhs,
                     double ms) {
  dim3 grid((p.m + TX - 1) / TX, (p.m + TY - 1) / TY, batches);
  const int per = grid.x * grid.y;
  part.ensure((size_t)per * batches);
  red.ensure(batches + 16);
  cudaStream_t s = p.cur_stream();
  k_newton_residual<<<grid, dim3(TX, TY), 0, s>>>(
      Ub, Db, d_alpha, Ut, Rt, part.get(), d_slice_of, d_active, p.m, p.c, p.d_cell_mat.get(),
      p.d_mat.get(), p.d_src_prof.get(), p.d_src_time.get(), (int)p.src_mats.size(), rhs, ms, p.d_mass.get());
  TP_LAUNCHED(&p);
  k_reduce_batches<<<batches, 256, 0, s>>>(part.get(), per, red.get());
  TP_LAUNCHED(&p);
  TP_CUDA(cudaMemcpyAsync(norms2_host, red.get(), sizeof(double) * batches, cudaMemcpyDeviceToHost, s));
  TP_CUDA(cudaStreamSynchronize(s));
}

// per-material min/max of |grad u| over all slices of the device state
namespace {
// cells of cell rows [cy0, cy1) (vertex rows cy0 .. cy1), u from the strip view
__global__ void k_field_ranges(const double* __restrict__ U, const double* __restrict__ halo_lo,
                               const double* __restrict__ halo_hi, int sy0, int rows, int cy0, int cy1,
                               int m, int c, int N, const uint8_t* __restrict__ cell_mat,
                               double* __restrict__ lo, double* __restrict__ hi) {
  // one thread per cell per slice-group; partial min/max per block per material
  __shared__ double slo[TP_MAX_MATERIALS][256], shi[TP_MAX_MATERIALS][256];
  const size_t cells = (size_t)c * (cy1 - cy0);
  const size_t nl = (size_t)rows * m;
  double mlo[TP_MAX_MATERIALS], mhi[TP_MAX_MATERIALS];
  for (int r = 0; r < TP_MAX_MATERIALS; ++r) { mlo[r] = INFINITY; mhi[r] = -1.0; }
  const double cc = (double)c;
  for (size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x; k < cells * N;
       k += (size_t)gridDim.x * blockDim.x) {
    const int s = (int)(k / cells);
    const size_t cl = k % cells;
    const int i = (int)(cl % c), j = cy0 + (int)(cl / c);
    const size_t cell = (size_t)j * c + i;
    const double* us = U + s * nl;
    const StripView sv{halo_lo ? halo_lo + (size_t)s * m : nullptr, halo_hi ? halo_hi + (size_t)s * m : nullptr,
                       sy0, rows};
    const double u00 = vertex_u(us, sv, m, i, j), u10 = vertex_u(us, sv, m, i + 1, j);
    const double u01 = vertex_u(us, sv, m, i, j + 1), u11 = vertex_u(us, sv, m, i + 1, j + 1);
    const double s1 = hypot(cc * (u10 - u00), cc * (u11 - u10));
    const double s2 = hypot(cc * (u11 - u01), cc * (u01 - u00));
    const int r = cell_mat[cell];
    mlo[r] = fmin(mlo[r], fmin(s1, s2));
    mhi[r] = fmax(mhi[r], fmax(s1, s2));
  }
  for (int r = 0; r < TP_MAX_MATERIALS; ++r) { slo[r][threadIdx.x] = mlo[r]; shi[r][threadIdx.x] = mhi[r]; }
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w)
      for (int r = 0; r < TP_MAX_MATERIALS; ++r) {
        slo[r][threadIdx.x] = fmin(slo[r][threadIdx.x], slo[r][threadIdx.x + w]);
        shi[r][threadIdx.x] = fmax(shi[r][threadIdx.x], shi[r][threadIdx.x + w]);
      }
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int r = 0; r < TP_MAX_MATERIALS; ++r) {
      lo[blockIdx.x * TP_MAX_MATERIALS + r] = slo[r][0];
      hi[blockIdx.x * TP_MAX_MATERIALS + r] = shi[r][0];
    }
}
}  // namespace

void Problem::field_ranges(double* lo, double* hi, int* any) {
  const int blocks = 2 * num_sms;
  part.ensure((size_t)2 * blocks * TP_MAX_MATERIALS);
  // cell row j has vertex rows j, j+1 = node rows j-1, j: rank r owns cell
  // rows [y0, y1) (the last rank also the top row c-1)
  const int rows = sh.y1 - sh.y0;
  const int cy0 = sh.y0, cy1 = (sh.r == sh.P - 1) ? c : sh.y1;
  if (sharded()) exchange_halo();
  k_field_ranges<<<blocks, 256, 0, stream>>>(U.get(), sharded() ? halo_lo.get() : nullptr,
                                            sharded() ? halo_hi.get() : nullptr, sh.y0, rows, cy0, cy1, m, c, N,
                                            d_cell_mat.get(), part.get(), part.get() + blocks * TP_MAX_MATERIALS);
  TP_LAUNCHED(this);
  std::vector<double> h(2 * blocks * TP_MAX_MATERIALS);
  TP_CUDA(cudaMemcpyAsync(h.data(), part.get(), h.size() * sizeof(double), cudaMemcpyDeviceToHost, stream));
  TP_CUDA(cudaStreamSynchronize(stream));
  for (int r = 0; r < TP_MAX_MATERIALS; ++r) {
    lo[r] = INFINITY;
    hi[r] = -1.0;
    for (int b = 0; b < blocks; ++b) {
      lo[r] = std::fmin(lo[r], h[b * TP_MAX_MATERIALS + r]);
      hi[r] = std::fmax(hi[r], h[(blocks + b) * TP_MAX_MATERIALS + r]);
    }
  }
  global_minmax(lo, hi, TP_MAX_MATERIALS);
  for (int r = 0; r < TP_MAX_MATERIALS; ++r) any[r] = hi[r] >= 0.0;
}

}  // namespace tpgpu
