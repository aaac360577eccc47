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
#include <cstdlib>
#include <type_traits>

#include "mg.cuh"

namespace tpgpu {

namespace {

constexpr int WL = 32;     // lanes per warp
constexpr int WPB = 4;     // warps per block
constexpr int RH = 64;     // rows per warp work item
// rows per warp item of the apply pass
#ifndef TPGPU_RH_APPLY
#define TPGPU_RH_APPLY 32
#endif
constexpr int RHA = TPGPU_RH_APPLY;

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

// 1/a for the smoothers' D^-1.  TPGPU_FAST_RCP: hardware reciprocal estimate
// + one Newton step (~46 bits, no special-case path); the V-cycle stays one
// fixed symmetric operator (every pass uses this same function), only D^-1 is
// perturbed at the 1e-14 level.
#ifndef TPGPU_FAST_RCP
#define TPGPU_FAST_RCP 1
#endif
__device__ __forceinline__ double drcp(double x) {
#if TPGPU_FAST_RCP
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, e, r);
#else
  return __drcp_rn(x);
#endif
}
__device__ __forceinline__ cplx rcp(cplx a) {
  const double d = drcp(fma(a.re, a.re, a.im * a.im));
  return {a.re * d, -a.im * d};
}

// ---- the same operations on real values (slice mode: Newton Jacobians)
__device__ __forceinline__ double cm(double a, double b) { return a * b; }
__device__ __forceinline__ double cs(double s, double a) { return s * a; }
__device__ __forceinline__ double shf_up(double v) { return __shfl_up_sync(0xffffffffu, v, 1); }
__device__ __forceinline__ double shf_dn(double v) { return __shfl_down_sync(0xffffffffu, v, 1); }
__device__ __forceinline__ double rcp(double a) { return drcp(a); }
// a x + y, componentwise fma
__device__ __forceinline__ cplx fmav(double a, cplx x, cplx y) { return {fma(a, x.re, y.re), fma(a, x.im, y.im)}; }
__device__ __forceinline__ double fmav(double a, double x, double y) { return fma(a, x, y); }
// bilinear partial sums x^T y (the COCG dot: (re, im); real: (value, 0))
__device__ __forceinline__ void dot_acc(cplx x, cplx y, double& s0, double& s1) {
  const cplx t = cm(x, y);
  s0 += t.re;
  s1 += t.im;
}
__device__ __forceinline__ void dot_acc(double x, double y, double& s0, double&) { s0 += x * y; }
__device__ __forceinline__ double sq_acc(cplx v, double s) { return fma(v.re, v.re, fma(v.im, v.im, s)); }
__device__ __forceinline__ double sq_acc(double v, double s) { return fma(v, v, s); }

__device__ __forceinline__ void warp_pair(double& a, double& b) {
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_down_sync(0xffffffffu, a, o);
    b += __shfl_down_sync(0xffffffffu, b, o);
  }
}

// sum of batch b's `per` partial pairs, every lane the same fixed-order result
__device__ __forceinline__ cplx warp_batch_sum(const double* __restrict__ part, int per, int b) {
  double a = 0, c = 0;
  for (int k = threadIdx.x & 31; k < per; k += 32) {
    a += part[((size_t)b * per + k) * 2];
    c += part[((size_t)b * per + k) * 2 + 1];
  }
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
  }
  return {a, c};
}
__device__ __forceinline__ cplx cdivv(cplx a, cplx b) {
  const double d = 1.0 / fma(b.re, b.re, b.im * b.im);
  return {fma(a.re, b.re, a.im * b.im) * d, fma(a.im, b.re, -a.re * b.im) * d};
}

struct Item {
  int b, strip, chunk, ys, ye, xs;
  bool ok;
};

// ---------------------------------------------------------------- async row ring
// The down/up passes walk rows with a long dependent chain per row (two
// stencil applications, a complex reciprocal, shuffles), so a row load issued
// one row ahead does not cover HBM latency at the occupancy these register-
// heavy kernels reach.  Each warp therefore stages its input rows (vectors
// and coefficient rows) through private shared-memory rings with per-lane
// cp.async copies issued RA rows ahead: every lane reads back only the slots
// it wrote itself, so cp.async.wait_group is the only synchronisation (no
// barriers, no mbarriers).  Out-of-domain entries are zero-filled by the copy
// (src-size 0).  Vector rows are consumed at once (ring of RA + 2 slots, the
// overwritten slot was read two rows earlier); coefficient rows stay readable
// for the three rows below the current one (ring of RA + 4 slots).
__device__ __forceinline__ void cp16(void* sdst, const void* g, bool ok) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(g), "r"(ok ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp8(void* sdst, const void* g, bool ok) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(g), "r"(ok ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp4(void* sdst, const void* g, bool ok) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(g), "r"(ok ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// ---- bulk row staging (TMA engine, cp.async.bulk -> UBLKCP): one elected
// lane copies a warp's whole row segment of a vector (up to 32 x 16 bytes,
// complex rows are 16-byte aligned) into its ring slot and the slot's
// mbarrier counts the bytes in; the lanes wait on the barrier's phase.
// resident 128-thread blocks per SM the bulk-staged passes are bounded for
// (3: <= 168 registers, the cp.async passes' occupancy)
#ifndef TPGPU_BULK_MINB
#define TPGPU_BULK_MINB 3
#endif
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* g, unsigned bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(sdst)),
               "l"(g), "r"(bytes), "r"(smem_u32(b))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

template <class T, int NV>
struct VRowT {  // NV values per lane of one staged row
  T v[NV][WL];
};
template <int NV>
using VRow = VRowT<cplx, NV>;
// stage one vector element per lane (16 B complex, 8 B real)
__device__ __forceinline__ void cpv(cplx* sdst, const cplx* g, bool ok) { cp16(sdst, g, ok); }
__device__ __forceinline__ void cpv(double* sdst, const double* g, bool ok) { cp8(sdst, g, ok); }
template <int NW>
struct WRow {  // NW coefficient doubles per lane of one staged row
  double w[NW][WL];
};

// ---- stencil policies.  Src: per-lane cursor staging consecutive
// coefficient rows (row offsets advance by addition; rows and columns
// outside the stored grid are zero-filled).  diag / apply: the diagonal and
// the operator at row y from the staged rows y (sy) and y-1 (sb).
struct Five {  // fine level: K_hat from edge weights (we, wn), lumped mass
  using T = cplx;
  static constexpr int NW = 3;
  struct Src {
    const double *we, *wn, *mm;  // lane column bases (vertex column x+1 clamped to [0, c])
    int c, m;
    bool colw, colm;
  };
  static __device__ __forceinline__ Src src(const FineOp& op, int x, int xc, int, int) {
    Src s;
    s.c = op.c;
    s.m = op.m;
    s.colw = (unsigned)(x + 1) <= (unsigned)op.c;  // vertex column X = x+1
    s.colm = x >= 0 && x < op.m;
    const int X = min(max(x + 1, 0), op.c);
    s.we = op.we + X;
    s.wn = op.wn + X;
    s.mm = op.mass + xc;
    return s;
  }
  // stage row yr; moff = (row yr clamped to [0, m)) * m, shared with the vectors
  static __device__ __forceinline__ void stage(WRow<NW>& st, const Src& s, int lane, int yr, unsigned moff,
                                               bool rowok) {
    const bool wv = s.colw && (unsigned)(yr + 1) <= (unsigned)s.c;
    const unsigned woff = (unsigned)min(max(yr + 1, 0), s.c) * (unsigned)(s.c + 1);
    cp8(&st.w[0][lane], s.we + woff, wv);
    cp8(&st.w[1][lane], s.wn + woff, wv);
    cp8(&st.w[2][lane], s.mm + moff, s.colm && rowok);
  }
  // a row's coefficients in registers: own east/north weights, mass, the west
  // weight (the west lane's east weight, shuffled once per row) and the south
  // weight (the north weight of the row below)
  static constexpr int RETAIN = 0;  // staged rows are read once, in their own iteration
  static constexpr bool XLANE = false;
  struct Reg {
    double we, ww, wn, ws, mm;
  };
  static __device__ __forceinline__ Reg load(const WRow<NW>& st, int lane, const Reg& below) {
    Reg k;
    k.we = st.w[0][lane];
    k.wn = st.w[1][lane];
    k.mm = st.w[2][lane];
    k.ww = __shfl_up_sync(0xffffffffu, k.we, 1);
    k.ws = below.wn;
    return k;
  }
  static __device__ __forceinline__ Reg first(const WRow<NW>& st, int lane) {
    Reg z{0, 0, 0, 0, 0};
    return load(st, lane, z);
  }
  static __device__ __forceinline__ cplx diag(const Reg& y, cplx l) {
    const double kc = (y.we + y.ww) + (y.wn + y.ws);
    return {fma(l.re, y.mm, kc), l.im * y.mm};
  }
  // the smoother's diagonal: the operator's own
  static __device__ __forceinline__ cplx sdiag(const Reg&, cplx d) { return d; }
  // d v - wE vE - wW vW - wN vN - wS vS (neighbours of Dirichlet vertices are
  // zero vectors, their edge weights stay on the diagonal)
  // (l unused: the diagonal d from diag() carries the shift)
  static __device__ __forceinline__ cplx apply(const Reg& y, cplx, cplx d, cplx vs, cplx v, cplx vn) {
    const cplx vw = shf_up(v), ve = shf_dn(v);
    cplx acc = cm(d, v);
    acc.re -= y.we * ve.re + y.ww * vw.re + y.wn * vn.re + y.ws * vs.re;
    acc.im -= y.we * ve.im + y.ww * vw.im + y.wn * vn.im + y.ws * vs.im;
    return acc;
  }
};

struct Seven {  // coarse levels: Galerkin K and M, symmetric 7-point (C, E, N, NE planes)
  using T = cplx;
  static constexpr int NW = 8;  // K C E N NE, M C E N NE
  struct Src {
    const double *K, *M;  // lane column bases
    unsigned n;
    bool col;
  };
  static __device__ __forceinline__ Src src(const FineOp& op, int x, int xc, int, int) {
    Src s;
    s.K = op.K + xc;
    s.M = op.M + xc;
    s.n = (unsigned)op.n;
    s.col = x >= 0 && x < op.m;
    return s;
  }
  static __device__ __forceinline__ void stage(WRow<NW>& st, const Src& s, int lane, int, unsigned moff,
                                               bool rowok) {
    const bool v = s.col && rowok;
    const int dirs[4] = {SC, SE_, SN_, SNE};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      cp8(&st.w[q][lane], s.K + (dirs[q] * s.n + moff), v);
      cp8(&st.w[4 + q][lane], s.M + (dirs[q] * s.n + moff), v);
    }
  }
  // rows stay in the ring (8 planes are too many for register windows) and
  // are read on use: the ring retains the three rows below the current one
  static constexpr int RETAIN = 3;
  struct Reg {
    const WRow<NW>* p;   // this row
    const WRow<NW>* pb;  // the row below
    int lane;
  };
  static __device__ __forceinline__ Reg load(const WRow<NW>& st, int lane, const Reg& below) {
    return {&st, below.p, lane};
  }
  static __device__ __forceinline__ Reg first(const WRow<NW>& st, int lane) { return {&st, &st, lane}; }
  static __device__ __forceinline__ cplx coef(const WRow<NW>* r, int q, int lane, cplx l) {
    const double mm = r->w[4 + q][lane];
    return {fma(l.re, mm, r->w[q][lane]), l.im * mm};
  }
  static __device__ __forceinline__ cplx diag(const Reg& y, cplx l) { return coef(y.p, 0, y.lane, l); }
  static __device__ __forceinline__ cplx sdiag(const Reg&, cplx d) { return d; }
  // W = E(x-1), S = N(y-1), SW = NE(x-1, y-1).  Split form
  //   sum_d (K_d + l M_d) v_d = sum_d K_d v_d + l sum_d M_d v_d
  // (real x complex products, one complex multiply by l at the end); the
  // west lane's E / NE coefficients are read from its ring slot (XLANE: the
  // kernels __syncwarp after each ring wait, so every lane's copies are visible).
  static constexpr bool XLANE = true;
  static __device__ __forceinline__ cplx apply(const Reg& y, cplx l, cplx d, cplx vs, cplx v, cplx vn) {
    const int ln = y.lane, lw = ln > 0 ? ln - 1 : 0;
    const cplx vw = shf_up(v), ve = shf_dn(v), vne = shf_dn(vn), vsw = shf_up(vs);
    const WRow<NW>& a = *y.p;
    const WRow<NW>& b = *y.pb;
    // K and M coefficients of E, W, N, S, NE, SW
    const double kE = a.w[1][ln], kW = a.w[1][lw], kN = a.w[2][ln], kS = b.w[2][ln], kNE = a.w[3][ln],
                 kSW = b.w[3][lw];
    const double mE = a.w[5][ln], mW = a.w[5][lw], mN = a.w[6][ln], mS = b.w[6][ln], mNE = a.w[7][ln],
                 mSW = b.w[7][lw];
    cplx sk, sm;
    sk.re = kE * ve.re + kW * vw.re + kN * vn.re + kS * vs.re + kNE * vne.re + kSW * vsw.re;
    sk.im = kE * ve.im + kW * vw.im + kN * vn.im + kS * vs.im + kNE * vne.im + kSW * vsw.im;
    sm.re = mE * ve.re + mW * vw.re + mN * vn.re + mS * vs.re + mNE * vne.re + mSW * vsw.re;
    sm.im = mE * ve.im + mW * vw.im + mN * vn.im + mS * vs.im + mNE * vne.im + mSW * vsw.im;
    const cplx dv = cm(d, v), lm = cm(l, sm);
    return {dv.re + sk.re + lm.re, dv.im + sk.im + lm.im};
  }
};

// Galerkin levels of the frequency solver where the shift is negligible
// (max_k |lambda_k| M_l << K_l, measured per level when the hierarchy is
// built, Problem::build_freq_work): the level operator of the V-cycle is K_l
// alone -- four real planes instead of eight, a real diagonal.  Only the
// preconditioner changes (the COCG residual is the fine operator's own), and
// the V-cycle stays a fixed complex-symmetric operator.
struct SevenK {
  using T = cplx;
  static constexpr int NW = 4;  // K C E N NE
  struct Src {
    const double* K;
    unsigned n;
    bool col;
  };
  static __device__ __forceinline__ Src src(const FineOp& op, int x, int xc, int, int) {
    Src s;
    s.K = op.K + xc;
    s.n = (unsigned)op.n;
    s.col = x >= 0 && x < op.m;
    return s;
  }
  static __device__ __forceinline__ void stage(WRow<NW>& st, const Src& s, int lane, int, unsigned moff,
                                               bool rowok) {
    const bool v = s.col && rowok;
    const int dirs[4] = {SC, SE_, SN_, SNE};
#pragma unroll
    for (int q = 0; q < 4; ++q) cp8(&st.w[q][lane], s.K + (dirs[q] * s.n + moff), v);
  }
  static constexpr int RETAIN = 3;
  static constexpr bool XLANE = true;
  struct Reg {
    const WRow<NW>* p;
    const WRow<NW>* pb;
    int lane;
  };
  static __device__ __forceinline__ Reg load(const WRow<NW>& st, int lane, const Reg& below) {
    return {&st, below.p, lane};
  }
  static __device__ __forceinline__ Reg first(const WRow<NW>& st, int lane) { return {&st, &st, lane}; }
  static __device__ __forceinline__ cplx diag(const Reg& y, cplx) { return {y.p->w[0][y.lane], 0.0}; }
  static __device__ __forceinline__ cplx sdiag(const Reg&, cplx d) { return d; }
  static __device__ __forceinline__ cplx apply(const Reg& y, cplx, cplx d, cplx vs, cplx v, cplx vn) {
    const int ln = y.lane, lw = ln > 0 ? ln - 1 : 0;
    const cplx vw = shf_up(v), ve = shf_dn(v), vne = shf_dn(vn), vsw = shf_up(vs);
    const WRow<NW>& a = *y.p;
    const WRow<NW>& b = *y.pb;
    const double kE = a.w[1][ln], kW = a.w[1][lw], kN = a.w[2][ln], kS = b.w[2][ln], kNE = a.w[3][ln],
                 kSW = b.w[3][lw];
    const double re = kE * ve.re + kW * vw.re + kN * vn.re + kS * vs.re + kNE * vne.re + kSW * vsw.re;
    const double im = kE * ve.im + kW * vw.im + kN * vn.im + kS * vs.im + kNE * vne.im + kSW * vsw.im;
    return {fma(d.re, v.re, re), fma(d.re, v.im, im)};
  }
};

// slice mode (static_init Newton): per-slice symmetric 7-point Jacobians J_b
// (planes C, E, N, NE of the 7n-per-slice stencil), real vectors
// C = double: the Jacobian planes as assembled; C = float: single-precision
// copies of the four planes (FineOp::Kf, 4n floats per slice) for the V-cycle
// passes -- the preconditioner reads half the coefficient bytes, the PCG
// operator (the tile apply) keeps the fp64 Jacobian
template <class C>
struct SevenJT {
  using T = double;
  static constexpr int NW = 4;  // J C E N NE
  struct Src {
    const C* J;  // lane column base of this slice's stencil
    unsigned n;
    bool col;
  };
  static __device__ __forceinline__ Src src(const FineOp& op, int x, int xc, int, int b) {
    Src s;
    if constexpr (std::is_same_v<C, float>) s.J = op.Kf + (size_t)b * op.kfstride + xc;
    else s.J = op.K + (size_t)b * op.kstride + xc;
    s.n = (unsigned)op.n;
    s.col = x >= 0 && x < op.m;
    return s;
  }
  static __device__ __forceinline__ void stage(WRow<NW>& st, const Src& s, int lane, int, unsigned moff,
                                               bool rowok) {
    const bool v = s.col && rowok;
    if constexpr (std::is_same_v<C, float>) {
#pragma unroll
      for (int q = 0; q < 4; ++q) cp4(&st.w[q][lane], s.J + (q * s.n + moff), v);
    } else {
      const int dirs[4] = {SC, SE_, SN_, SNE};
#pragma unroll
      for (int q = 0; q < 4; ++q) cp8(&st.w[q][lane], s.J + (dirs[q] * s.n + moff), v);
    }
  }
  // coefficient q of lane ln from a staged row (floats sit in the first half of the slot)
  static __device__ __forceinline__ double cf(const WRow<NW>& r, int q, int ln) {
    if constexpr (std::is_same_v<C, float>) return (double)*reinterpret_cast<const float*>(&r.w[q][ln]);
    else return r.w[q][ln];
  }
  static constexpr int RETAIN = 3;
  static constexpr bool XLANE = true;
  struct Reg {
    const WRow<NW>* p;   // this row
    const WRow<NW>* pb;  // the row below
    int lane;
  };
  static __device__ __forceinline__ Reg load(const WRow<NW>& st, int lane, const Reg& below) {
    return {&st, below.p, lane};
  }
  static __device__ __forceinline__ Reg first(const WRow<NW>& st, int lane) { return {&st, &st, lane}; }
  static __device__ __forceinline__ double diag(const Reg& y, cplx) { return cf(*y.p, 0, y.lane); }
  // the smoother's diagonal: the l1 row sum sum_j |J_ij| (TPGPU_SLICE_L1, mg.cuh)
  // -- D_l1^-1 J has its spectrum in (0, 1] for any SPD J, so the Chebyshev
  // pair of weights is safe despite the anisotropic rank-one Jacobian term
  static __device__ __forceinline__ double sdiag(const Reg& y, double d) {
#if TPGPU_SLICE_L1
    const int ln = y.lane, lw = ln > 0 ? ln - 1 : 0;
    const WRow<NW>& a = *y.p;
    const WRow<NW>& b = *y.pb;
    return fabs(d) + fabs(cf(a, 1, ln)) + fabs(cf(a, 1, lw)) + fabs(cf(a, 2, ln)) + fabs(cf(b, 2, ln)) +
           fabs(cf(a, 3, ln)) + fabs(cf(b, 3, lw));
#else
    return d;
#endif
  }
  // W = E(x-1), S = N(y-1), SW = NE(x-1, y-1) (west lane's slots, XLANE)
  static __device__ __forceinline__ double apply(const Reg& y, cplx, double d, double vs, double v, double vn) {
    const int ln = y.lane, lw = ln > 0 ? ln - 1 : 0;
    const double vw = shf_up(v), ve = shf_dn(v), vne = shf_dn(vn), vsw = shf_up(vs);
    const WRow<NW>& a = *y.p;
    const WRow<NW>& b = *y.pb;
    const double off = cf(a, 1, ln) * ve + cf(a, 1, lw) * vw + cf(a, 2, ln) * vn + cf(b, 2, ln) * vs +
                       cf(a, 3, ln) * vne + cf(b, 3, lw) * vsw;
    return fma(d, v, off);
  }
};
using SevenJ = SevenJT<double>;
using SevenJF = SevenJT<float>;

template <class S, int NV, int RA, int WPBK>
constexpr size_t ring_smem() {
  return (size_t)WPBK *
         ((RA + 2) * sizeof(VRowT<typename S::T, NV>) + (RA + 2 + S::RETAIN) * sizeof(WRow<S::NW>));
}

__device__ __forceinline__ int wrap_inc(int s, int n) { return s + 1 == n ? 0 : s + 1; }

// warp work item with a runtime chunk height: ((b * nch) + chunk) * ns + strip
template <int WPBK>
__device__ __forceinline__ Item item_rh(int m, int own, int rh, int nb, const int* __restrict__ active) {
  Item it;
  const int w = blockIdx.x * WPBK + (threadIdx.x >> 5);
  const int ns = (m + own - 1) / own, nch = (m + rh - 1) / rh;
  it.strip = w % ns;
  it.chunk = (w / ns) % nch;
  it.b = w / (ns * nch);
  it.ok = it.b < nb && (!active || active[it.b]);
  it.ys = it.chunk * rh;
  it.ye = min(it.ys + rh, m);
  it.xs = it.strip * own;
  return it;
}

#ifndef TPGPU_STREAM_UNROLL
#define TPGPU_STREAM_UNROLL 3
#endif
// resident warps per SM the register allocation is bounded for (0: free)
#ifndef TPGPU_STREAM_MINW
#define TPGPU_STREAM_MINW 0
#endif
// stage rows past the chunk too (no branch in the row loop; the extra rows are
// loaded and never read)
#ifndef TPGPU_ISSUE_ALWAYS
#define TPGPU_ISSUE_ALWAYS 0
#endif
// restriction shuffles on every row (no divergent-shuffle fallback paths)
#ifndef TPGPU_RESTRICT_SHFL_ALWAYS
#define TPGPU_RESTRICT_SHFL_ALWAYS 0
#endif
#ifndef TPGPU_SEVEN_MINW
#define TPGPU_SEVEN_MINW 0
#endif
#define TP_MINB(W) (TPGPU_STREAM_MINW > 0 ? TPGPU_STREAM_MINW / (W) : 1)
// per stencil: resident warps per SM the registers are bounded for
#define TP_MINB_S(S, W) ((S::NW == 8 && TPGPU_SEVEN_MINW > 0) ? TPGPU_SEVEN_MINW / (W) : TP_MINB(W))
#ifndef TPGPU_SEVEN_UNROLL
#define TPGPU_SEVEN_UNROLL TPGPU_STREAM_UNROLL
#endif
#define TP_PRAGMA(x) _Pragma(#x)
#define TP_UNROLL(n) TP_PRAGMA(unroll n)

// warp work item over NB batches: ((g * nch) + chunk) * ns + strip, batches
// g*NB .. g*NB+NB-1 (inactive or missing ones are computed on a stand-in
// batch and never stored, so shuffles stay warp-uniform)
template <int WPBK, int NB>
struct ItemNB {
  int b[NB];
  bool on[NB];
  int strip, chunk, ys, ye, xs;
  bool ok;
};
template <int WPBK, int NB>
__device__ __forceinline__ ItemNB<WPBK, NB> item_nb(int m, int own, int rh, int nb, const int* __restrict__ active) {
  ItemNB<WPBK, NB> it;
  const int w = blockIdx.x * WPBK + (threadIdx.x >> 5);
  const int ns = (m + own - 1) / own, nch = (m + rh - 1) / rh;
  it.strip = w % ns;
  it.chunk = (w / ns) % nch;
  const int g = w / (ns * nch);
  int first = -1;
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    const int b = g * NB + j;
    it.on[j] = b < nb && (!active || active[b]);
    if (it.on[j] && first < 0) first = b;
  }
  it.ok = first >= 0;
#pragma unroll
  for (int j = 0; j < NB; ++j) it.b[j] = it.on[j] ? g * NB + j : first;
  it.ys = it.chunk * rh;
  it.ye = min(it.ys + rh, m);
  it.xs = it.strip * own;
  return it;
}

// ---------------------------------------------------------------- down
//   z1 = w1 r/d ; z2 = z1 + w2 (r - A z1)/d ; res = r - A z2 ; b_c = P^T res
// NB frequencies per warp share the coefficient rows, the addressing and the
// ring bookkeeping; their arithmetic chains are independent (ILP).
// FUSED (fine level, NB = 1): the Krylov residual update rides along -- the
// right-hand side is r_new = r - alpha q (read r and q, write r_new to rout
// for the owned rows, partial ||r_new||^2 per warp item), replacing the
// separate x/r update pass (x is updated in the next apply).
template <class S, int NB, int RA, int WPBK, bool FUSED = false, bool BULK = false>
__global__ void __launch_bounds__(WL * WPBK, BULK ? TPGPU_BULK_MINB : TP_MINB_S(S, WPBK)) k_stream_down(FineOp op, const typename S::T* __restrict__ rv,
                                                                         typename S::T* __restrict__ z2out,
                                                                         typename S::T* __restrict__ bc, int mc,
                                                                         int rh, const int* __restrict__ active,
                                                                         double om1, double om2, int nb,
                                                                         const typename S::T* __restrict__ qv = nullptr,
                                                                         const typename S::T* __restrict__ alpha = nullptr,
                                                                         typename S::T* __restrict__ rout = nullptr,
                                                                         double* __restrict__ part = nullptr,
                                                                         ScalFuse sf = ScalFuse{}) {
  using T = typename S::T;
  static_assert(!FUSED || NB == 1, "fused residual update: one frequency per warp");
  constexpr int H = 3, OWN = 26;  // lanes 3..28 own fine columns; even strip start
  constexpr int RV = RA + 2, RC = RA + 2 + S::RETAIN, NVV = FUSED ? 2 : NB;
  extern __shared__ __align__(16) unsigned char fine_smem[];
  const int m = op.m;
  TP_PDL_ENTRY();
  const ItemNB<WPBK, NB> it = item_nb<WPBK, NB>(m, OWN, rh, nb, active);
  if (!it.ok) return;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  VRowT<T, NVV>* const vring = reinterpret_cast<VRowT<T, NVV>*>(fine_smem) + wib * RV;
  WRow<S::NW>* const wring =
      reinterpret_cast<WRow<S::NW>*>(fine_smem + WPBK * RV * sizeof(VRowT<T, NVV>)) + wib * RC;
  // BULK: the warp's vector-row segments come in by cp.async.bulk, one
  // mbarrier per vector ring slot (after the coefficient rings)
  uint64_t* const bars = reinterpret_cast<uint64_t*>(fine_smem + WPBK * RV * sizeof(VRowT<T, NVV>) +
                                                     WPBK * RC * sizeof(WRow<S::NW>)) + wib * RV;
  const int blo = max(0, H - it.xs);                        // first lane with a column in [0, m)
  const int bhi = min(WL, m - (it.xs - H));                 // one past the last
  const unsigned bbytes = bhi > blo ? (unsigned)(bhi - blo) * (unsigned)sizeof(T) : 0u;
  unsigned bpar = 0, bpend = 0;  // per slot: parity of the last issued phase, issued-not-waited
  if constexpr (BULK) {
    if (lane == 0) {
      for (int q = 0; q < RV; ++q) mbar_init(&bars[q]);
      fence_proxy_async();
    }
    __syncwarp();
  }
  const T* const qp = FUSED ? qv + (size_t)it.b[0] * op.n + min(max(it.xs - H + lane, 0), op.m - 1) : nullptr;
  T* const ro = FUSED ? rout + (size_t)it.b[0] * op.n + min(max(it.xs - H + lane, 0), op.m - 1) : nullptr;
  T al{};
  if constexpr (FUSED) {
    if constexpr (std::is_same_v<T, cplx>) {
      if (sf.part) {
        // alpha = rho / (p^T q), reduced here from the apply's partials
        const int b0 = it.b[0];
        const cplx mu = warp_batch_sum(sf.part, sf.per, b0);
        al = cdivv(sf.rho_r[b0], mu);
        if (it.chunk == 0 && it.strip == 0 && (threadIdx.x & 31) == 0) {
          sf.alpha[b0] = al;
          sf.xa[b0] = al;
          sf.mu[b0] = mu;
        }
      } else {
        al = alpha[it.b[0]];
      }
    } else {
      al = alpha[it.b[0]];
    }
  }
  double rn2 = 0;
  const int x = it.xs - H + lane;
  const bool colok = x >= 0 && x < m;
  const bool own = lane >= H && lane < H + OWN && colok;
  const int xc = min(max(x, 0), m - 1);
  const T* rp[NB];
  T* zo[NB];
  T* bco[NB];
  cplx l[NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    const size_t o = (size_t)it.b[j] * op.n;
    rp[j] = rv + o + xc;
    zo[j] = z2out + o + xc;
    bco[j] = bc + (size_t)it.b[j] * mc * mc + (x >> 1);
    l[j] = op.lam ? op.lam[it.b[j]] : cplx{0, 0};
  }
  const int ys = it.ys, ye = it.ye;
  const int y0 = ys - 3, ylast = ye + 2;  // staged rows
  const bool cown = own && (x & 1) && (x >> 1) < mc;  // coarse centre column
  const typename S::Src src = S::src(op, x, xc, y0, it.b[0]);
  int vi = 0, wi = 0; // next ring slots to fill
  // stage row yr (rows outside [0, m) read row 0 / m-1 addresses and are zero-filled)
  auto issue = [&](int yr) {
    if (TPGPU_ISSUE_ALWAYS || yr <= ylast) {
      const bool rowok = (unsigned)yr < (unsigned)m, rin = colok && rowok;
      const unsigned off = (unsigned)min(max(yr, 0), m - 1) * (unsigned)m;
      if constexpr (BULK) {
        __syncwarp();  // every lane's reads of the slot (two rows ago) precede the refill
        if (lane == 0) {
          // the first staged row's vectors are never read: arrive without bytes
          const unsigned by = (rowok && yr != y0) ? bbytes : 0u;
          fence_proxy_async();  // the slot's earlier generic reads before the async writes
          mbar_expect(&bars[vi], by * NVV);
          if (by) {
            // lane blo's pointer is the segment start (rp / qp are per-lane column pointers)
            const size_t seg = (size_t)yr * m + (size_t)(it.xs - H + blo);
#pragma unroll
            for (int j = 0; j < NB; ++j)
              bulk_g2s(&vring[vi].v[j][blo], rv + (size_t)it.b[j] * op.n + seg, by, &bars[vi]);
            if (FUSED) bulk_g2s(&vring[vi].v[1][blo], qv + (size_t)it.b[0] * op.n + seg, by, &bars[vi]);
          }
        }
        bpar ^= 1u << vi;
        bpend |= 1u << vi;
      } else {
#pragma unroll
        for (int j = 0; j < NB; ++j) cpv(&vring[vi].v[j][lane], rp[j] + off, rin);
        if (FUSED) cpv(&vring[vi].v[1][lane], qp + off, rin);
      }
      S::stage(wring[wi], src, lane, yr, off, rowok);
      vi = wrap_inc(vi, RV);
      wi = wrap_inc(wi, RC);
    }
    cp_commit();
  };
  // pipeline over input rows yi = ys-2 .. ye+2: z1 at yi, z2 at yi-1,
  // residual at yi-2, restriction centred on yi-3
  T r0[NB], r1[NB], r2[NB];  // r at yi, yi-1, yi-2
  T a0[NB], a1[NB], a2[NB];  // z1 at yi, yi-1, yi-2
  T b1[NB], b2[NB], b3[NB];  // z2 at yi-1, yi-2, yi-3
  T q2[NB], q3[NB], q4[NB];  // res at yi-2, yi-3, yi-4
  T id0[NB], id1[NB];        // 1/d of rows yi, yi-1
  T d0[NB], d1[NB], d2[NB];  // d of rows yi, yi-1, yi-2
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    r0[j] = r1[j] = r2[j] = a0[j] = a1[j] = a2[j] = T{};
    b1[j] = b2[j] = b3[j] = q2[j] = q3[j] = q4[j] = id0[j] = id1[j] = T{};
    d0[j] = d1[j] = d2[j] = T{};
  }
#pragma unroll
  for (int j = 0; j <= RA; ++j) issue(y0 + j);
  // coefficient rows yi .. yi-3 (rows before y0 only feed halo values that
  // are never used: they repeat row y0)
  int vr = 0, sr = 0;  // ring slots of row yi
  cp_wait<RA>();
  if (S::XLANE) __syncwarp();
  typename S::Reg k0 = S::first(wring[0], lane), k1 = k0, k2 = k0;  // rows yi, yi-1, yi-2
  TP_UNROLL((S::NW == 8 ? TPGPU_SEVEN_UNROLL : TPGPU_STREAM_UNROLL))
  for (int yi = ys - 2; yi <= ylast; ++yi) {
    issue(yi + RA);
    vr = wrap_inc(vr, RV);
    sr = wrap_inc(sr, RC);
    cp_wait<RA>();
    if (S::XLANE) __syncwarp();
    if constexpr (BULK) {
      // the phase issued last for this slot: parity bit before that issue's flip
      mbar_wait(&bars[vr], ((bpar >> vr) & 1u) ^ 1u);
      bpend &= ~(1u << vr);
    }
    k2 = k1; k1 = k0;
    k0 = S::load(wring[sr], lane, k1);
    const bool in0 = colok && (unsigned)yi < (unsigned)m;
    const bool in1 = colok && (unsigned)(yi - 1) < (unsigned)m;
    const bool in2 = colok && (unsigned)(yi - 2) < (unsigned)m;
    const bool st1 = own && yi - 1 >= ys && yi - 1 < ye;
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      // (BULK: lanes off the grid and rows off the grid read zero, the bulk
      // copy fills only the segment inside it)
      r2[j] = r1[j]; r1[j] = r0[j]; r0[j] = (!BULK || in0) ? vring[vr].v[j][lane] : T{};
      if (FUSED) {
        const T qq = (!BULK || in0) ? vring[vr].v[1][lane] : T{};
        r0[j] = r0[j] - cm(al, qq);
        if (own && yi >= ys && yi < ye) {
          ro[(long)yi * m] = r0[j];
          rn2 = sq_acc(r0[j], rn2);
        }
      }
      // z1 = omega r / d at row yi (off-domain diagonals may vanish: z1 = 0 there)
      a2[j] = a1[j]; a1[j] = a0[j];
      id1[j] = id0[j];
      d2[j] = d1[j]; d1[j] = d0[j];
      d0[j] = S::diag(k0, l[j]);
      id0[j] = rcp(S::sdiag(k0, d0[j]));
      a0[j] = in0 ? cs(om1, cm(r0[j], id0[j])) : T{};
      // z2 at row yi-1
      b3[j] = b2[j]; b2[j] = b1[j];
      {
        const T Aa = S::apply(k1, l[j], d1[j], a2[j], a1[j], a0[j]);
        const T t = cm(r1[j] - Aa, id1[j]);
        b1[j] = in1 ? fmav(om2, t, a1[j]) : T{};
        if (st1 && it.on[j]) zo[j][(long)(yi - 1) * m] = b1[j];
      }
      // residual at row yi-2
      q4[j] = q3[j]; q3[j] = q2[j];
      {
        const T Ab = S::apply(k2, l[j], d2[j], b3[j], b2[j], b1[j]);
        q2[j] = in2 ? r2[j] - Ab : T{};
      }
    }
    // restriction centred on row yc = yi-3 (odd fine rows 2Y+1; warp-uniform branch)
    const int yc = yi - 3;
#if TPGPU_RESTRICT_SHFL_ALWAYS
    {
#else
    if ((yc & 1) && yc >= ys && yc < ye) {
#endif
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const T qw = shf_up(q3[j]), qe = shf_dn(q3[j]);
        const T q4w = shf_up(q4[j]), q2e = shf_dn(q2[j]);
        if ((yc & 1) && yc >= ys && yc < ye && cown && it.on[j] && (yc >> 1) < mc)
          bco[j][(size_t)(yc >> 1) * mc] = q3[j] + 0.5 * (qw + qe + q4[j] + q2[j] + q4w + q2e);
      }
    }
  }
  cp_wait<0>();
  if constexpr (BULK) {
    // copies issued but never consumed (the first staged row) land before exit
    for (int q = 0; q < RV; ++q)
      if ((bpend >> q) & 1u) mbar_wait(&bars[q], ((bpar >> q) & 1u) ^ 1u);
  }
  if (FUSED) {
    double zz = 0;
    warp_pair(rn2, zz);
    if (lane == 0) {
      const int ns = (m + OWN - 1) / OWN, nch = (m + rh - 1) / rh;
      const size_t k = (size_t)it.b[0] * ((size_t)ns * nch) + (size_t)it.chunk * ns + it.strip;
      part[2 * k] = rn2;
      part[2 * k + 1] = 0.0;
    }
  }
}

// ---------------------------------------------------------------- up
//   zc = z2 + P x_c ; z3, z4 = two Jacobi steps ; writes z4 (+ partial r^T z4)
// Staged per row and frequency: r, z2 and the (up to two) coarse values P x_c
// interpolates from at the lane's node; the coefficient row once.
template <class S, int NB, int RA, int WPBK, bool BULK = false>
__global__ void __launch_bounds__(WL * WPBK, BULK ? TPGPU_BULK_MINB : TP_MINB_S(S, WPBK)) k_stream_up(FineOp op, const typename S::T* __restrict__ rv,
                                                                       const typename S::T* __restrict__ z2in,
                                                                       const typename S::T* __restrict__ xcv, int mc,
                                                                       int rh, typename S::T* __restrict__ zout,
                                                                       const int* __restrict__ active, double om1,
                                                                       double om2, int nb, int dot,
                                                                       double* __restrict__ part) {
  using T = typename S::T;
  constexpr int H = 2, OWN = WL - 2 * H;  // 28
  constexpr int RV = RA + 2, RC = RA + 2 + S::RETAIN;
  extern __shared__ __align__(16) unsigned char fine_smem[];
  const int m = op.m;
  TP_PDL_ENTRY();
  const ItemNB<WPBK, NB> it = item_nb<WPBK, NB>(m, OWN, rh, nb, active);
  if (!it.ok) return;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  VRowT<T, 4 * NB>* const vring = reinterpret_cast<VRowT<T, 4 * NB>*>(fine_smem) + wib * RV;
  WRow<S::NW>* const wring =
      reinterpret_cast<WRow<S::NW>*>(fine_smem + WPBK * RV * sizeof(VRowT<T, 4 * NB>)) + wib * RC;
  // BULK: r and z2 rows by cp.async.bulk (the coarse values are gathered per lane)
  uint64_t* const bars = reinterpret_cast<uint64_t*>(fine_smem + WPBK * RV * sizeof(VRowT<T, 4 * NB>) +
                                                     WPBK * RC * sizeof(WRow<S::NW>)) + wib * RV;
  const int blo = max(0, H - it.xs);
  const int bhi = min(WL, m - (it.xs - H));
  const unsigned bbytes = bhi > blo ? (unsigned)(bhi - blo) * (unsigned)sizeof(T) : 0u;
  unsigned bpar = 0, bpend = 0;
  if constexpr (BULK) {
    if (lane == 0) {
      for (int q = 0; q < RV; ++q) mbar_init(&bars[q]);
      fence_proxy_async();
    }
    __syncwarp();
  }
  const int x = it.xs - H + lane;
  const bool colok = x >= 0 && x < m;
  const bool own = lane >= H && lane < WL - H && colok;
  const int xc = min(max(x, 0), m - 1);
  const T* rp[NB];
  const T* zp[NB];
  const T* xb[NB];
  T* zo[NB];
  cplx l[NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    const size_t o = (size_t)it.b[j] * op.n;
    rp[j] = rv + o + xc;
    zp[j] = z2in + o + xc;
    zo[j] = zout + o + xc;
    xb[j] = xcv + (size_t)it.b[j] * mc * mc;
    l[j] = op.lam ? op.lam[it.b[j]] : cplx{0, 0};
  }
  const int ys = it.ys, ye = it.ye;
  const int y0 = ys - 3, ylast = ye + 1;
  // P1 prolongation: fine vertex a = x+1 (column parity fixed per lane);
  // coarse columns A1 = ah and A2 (= ah+1 on odd vertex columns)
  const int a = x + 1, ah = a >> 1;
  const bool ao = a & 1;
  const int A2 = ao ? ah + 1 : ah;
  const bool cA1 = colok && ah >= 1 && ah <= mc, cA2 = colok && A2 >= 1 && A2 <= mc;
  const typename S::Src src = S::src(op, x, xc, y0, it.b[0]);
  int vi = 0, wi = 0;
  auto issue = [&](int yr) {
    if (TPGPU_ISSUE_ALWAYS || yr <= ylast) {
      const bool rowok = (unsigned)yr < (unsigned)m, rin = colok && rowok;
      const unsigned off = (unsigned)min(max(yr, 0), m - 1) * (unsigned)m;
      // coarse vertices of the node's P1 interpolation: (A1, B1) and (A2, B2);
      // the second is absent at coincident vertices
      const int bb = yr + 1, bh = bb >> 1;
      const int B2 = (bb & 1) ? bh + 1 : bh;
      const bool has2 = ao || (bb & 1);
      const bool ok1 = rin && cA1 && bh >= 1 && bh <= mc;
      const bool ok2 = rin && has2 && cA2 && B2 >= 1 && B2 <= mc;
      const unsigned c1 = ok1 ? (bh - 1) * mc + (ah - 1) : 0, c2 = ok2 ? (B2 - 1) * mc + (A2 - 1) : 0;
      VRowT<T, 4 * NB>& sv = vring[vi];
      if constexpr (BULK) {
        __syncwarp();
        if (lane == 0) {
          const unsigned by = (rowok && yr != y0) ? bbytes : 0u;
          fence_proxy_async();
          mbar_expect(&bars[vi], by * 2 * NB);
          if (by) {
            const size_t seg = (size_t)yr * m + (size_t)(it.xs - H + blo);
#pragma unroll
            for (int j = 0; j < NB; ++j) {
              bulk_g2s(&sv.v[4 * j][blo], rv + (size_t)it.b[j] * op.n + seg, by, &bars[vi]);
              bulk_g2s(&sv.v[4 * j + 1][blo], z2in + (size_t)it.b[j] * op.n + seg, by, &bars[vi]);
            }
          }
        }
        bpar ^= 1u << vi;
        bpend |= 1u << vi;
      }
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        if constexpr (!BULK) {
          cpv(&sv.v[4 * j][lane], rp[j] + off, rin);
          cpv(&sv.v[4 * j + 1][lane], zp[j] + off, rin);
        }
        cpv(&sv.v[4 * j + 2][lane], xb[j] + c1, ok1);
        cpv(&sv.v[4 * j + 3][lane], xb[j] + c2, ok2);
      }
      S::stage(wring[wi], src, lane, yr, off, rowok);
      vi = wrap_inc(vi, RV);
      wi = wrap_inc(wi, RC);
    }
    cp_commit();
  };
  // pipeline over input rows yi = ys-2 .. ye+1: zc at yi, z3 at yi-1, z4 at yi-2
  T c0[NB], c1[NB], c2[NB];  // zc at yi, yi-1, yi-2
  T r0[NB], r1[NB], r2[NB];  // r at yi, yi-1, yi-2
  T e1[NB], e2[NB], e3[NB];  // z3 at yi-1, yi-2, yi-3
  T jd1[NB], jd2[NB];        // 1/d of rows yi-1, yi-2
  T dd1[NB], dd2[NB];        // d of rows yi-1, yi-2
  double p0[NB], p1[NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    c0[j] = c1[j] = c2[j] = r0[j] = r1[j] = r2[j] = T{};
    e1[j] = e2[j] = e3[j] = jd1[j] = jd2[j] = dd1[j] = dd2[j] = T{};
    p0[j] = p1[j] = 0;
  }
#pragma unroll
  for (int j = 0; j <= RA; ++j) issue(y0 + j);
  int vr = 0, sr = 0;
  cp_wait<RA>();
  if (S::XLANE) __syncwarp();
  typename S::Reg k0 = S::first(wring[0], lane), k1 = k0, k2 = k0;  // rows yi, yi-1, yi-2
  TP_UNROLL((S::NW == 8 ? TPGPU_SEVEN_UNROLL : TPGPU_STREAM_UNROLL))
  for (int yi = ys - 2; yi <= ylast; ++yi) {
    issue(yi + RA);
    vr = wrap_inc(vr, RV);
    sr = wrap_inc(sr, RC);
    cp_wait<RA>();
    if (S::XLANE) __syncwarp();
    if constexpr (BULK) {
      mbar_wait(&bars[vr], ((bpar >> vr) & 1u) ^ 1u);
      bpend &= ~(1u << vr);
    }
    const VRowT<T, 4 * NB>& sv = vring[vr];
    const double wc1 = (!ao && !((yi + 1) & 1)) ? 1.0 : 0.5;
    k2 = k1; k1 = k0;
    k0 = S::load(wring[sr], lane, k1);
    const bool in1 = colok && (unsigned)(yi - 1) < (unsigned)m;
    const bool in0 = colok && (unsigned)yi < (unsigned)m;
    const bool st2 = own && yi - 2 >= ys && yi - 2 < ye;
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const T zz = (!BULK || in0) ? sv.v[4 * j + 1][lane] : T{}, x1 = sv.v[4 * j + 2][lane],
              x2 = sv.v[4 * j + 3][lane];
      const T ccur = fmav(wc1, x1, fmav(0.5, x2, zz));
      c2[j] = c1[j]; c1[j] = c0[j]; c0[j] = ccur;
      r2[j] = r1[j]; r1[j] = r0[j]; r0[j] = (!BULK || in0) ? sv.v[4 * j][lane] : T{};
      // z3 at row yi-1
      e3[j] = e2[j]; e2[j] = e1[j];
      {
        dd2[j] = dd1[j];
        dd1[j] = S::diag(k1, l[j]);
        const T Ac = S::apply(k1, l[j], dd1[j], c2[j], c1[j], c0[j]);
        jd2[j] = jd1[j];
        jd1[j] = rcp(S::sdiag(k1, dd1[j]));
        const T t = cm(r1[j] - Ac, jd1[j]);
        e1[j] = in1 ? fmav(om2, t, c1[j]) : T{};
      }
      // z4 at row yi-2
      {
        const T Ae = S::apply(k2, l[j], dd2[j], e3[j], e2[j], e1[j]);
        if (st2 && it.on[j]) {
          const T t = cm(r2[j] - Ae, jd2[j]);
          const T z4 = fmav(om1, t, e2[j]);
          zo[j][(long)(yi - 2) * m] = z4;
          if (dot) dot_acc(r2[j], z4, p0[j], p1[j]);
        }
      }
    }
  }
  cp_wait<0>();
  if constexpr (BULK) {
    for (int q = 0; q < RV; ++q)
      if ((bpend >> q) & 1u) mbar_wait(&bars[q], ((bpar >> q) & 1u) ^ 1u);
  }
  if (dot) {
    const int ns = (m + OWN - 1) / OWN, nch = (m + rh - 1) / rh;
    const size_t per = (size_t)ns * nch;
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      warp_pair(p0[j], p1[j]);
      if (lane == 0 && it.on[j]) {
        const size_t k = (size_t)it.b[j] * per + (size_t)it.chunk * ns + it.strip;
        part[2 * k] = p0[j];
        part[2 * k + 1] = p1[j];
      }
    }
  }
}

// ---------------------------------------------------------------- apply
// INIT = 0: p = first ? z : z + beta p_in -> p_out ; q = A p ; part += p^T q
// INIT = 1: r = b - A x (b in z, x in pin, r to q) ; part += (|b|^2, |r|^2)
// One fine-level stencil per node: rows of z and p_in staged through the
// ring, p formed at row yi, q (and the stored p) at row yi-1.
// XUPD: also the deferred solution update x += xa p_in of the previous
// iteration (fused Krylov update): x staged as a third vector; frequencies
// that converged last iteration (inactive, xa != 0) get only that update.
// p = z + beta p_in with the exact fma pattern of the complex recurrence
__device__ __forceinline__ cplx zpb(cplx bt, cplx pv, cplx zz) {
  return {fma(bt.re, pv.re, fma(-bt.im, pv.im, zz.re)), fma(bt.re, pv.im, fma(bt.im, pv.re, zz.im))};
}
__device__ __forceinline__ double zpb(double bt, double pv, double zz) { return fma(bt, pv, zz); }
__device__ __forceinline__ bool nonzero(cplx a) { return a.re != 0.0 || a.im != 0.0; }
__device__ __forceinline__ bool nonzero(double a) { return a != 0.0; }
// x + a p (the deferred solution update; complex: the same product order as before)
__device__ __forceinline__ cplx xpa(cplx xv, cplx a, cplx pv) {
  return {xv.re + (a.re * pv.re - a.im * pv.im), xv.im + (a.re * pv.im + a.im * pv.re)};
}
__device__ __forceinline__ double xpa(double xv, double a, double pv) { return xv + a * pv; }

template <class S, int INIT, int RA, int WPBK, bool XUPD = false>
__global__ void __launch_bounds__(WL * WPBK) k_stream_apply(FineOp op, const typename S::T* __restrict__ z,
                                                            const typename S::T* __restrict__ pin,
                                                            typename S::T* __restrict__ pout,
                                                            typename S::T* __restrict__ q,
                                                            const typename S::T* __restrict__ beta,
                                                            const int* __restrict__ active, int first, int nb,
                                                            double* __restrict__ part,
                                                            typename S::T* __restrict__ xs = nullptr,
                                                            const typename S::T* __restrict__ xa = nullptr,
                                                            ScalFuse sf = ScalFuse{}) {
  using T = typename S::T;
  constexpr int H = 1, OWN = WL - 2 * H;  // 30
  constexpr int RV = RA + 2, RC = RA + 2 + S::RETAIN, NVV = XUPD ? 3 : 2;
  extern __shared__ __align__(16) unsigned char fine_smem[];
  const int m = op.m;
  TP_PDL_ENTRY();
  const int rha = op.rha;
  const ItemNB<WPBK, 1> it = item_nb<WPBK, 1>(m, OWN, rha, nb, nullptr);
  const bool on = INIT || !active || active[it.b[0]];
  T xab{};
  if (XUPD) xab = xa[it.b[0]];
  const bool pend = XUPD && nonzero(xab);
  if (!it.ok || (!on && !pend)) return;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  VRowT<T, NVV>* const vring = reinterpret_cast<VRowT<T, NVV>*>(fine_smem) + wib * RV;
  WRow<S::NW>* const wring =
      reinterpret_cast<WRow<S::NW>*>(fine_smem + WPBK * RV * sizeof(VRowT<T, NVV>)) + wib * RC;
  const int x = it.xs - H + lane;
  const bool colok = x >= 0 && x < m;
  const bool own = lane >= H && lane < WL - H && colok;
  const int xc = min(max(x, 0), m - 1);
  const int b = it.b[0];
  const size_t o = (size_t)b * op.n;
  const T* const zp = z + o + xc;
  const T* const pp = pin + o + xc;
  T* const po = pout + o + xc;
  T* const qo = q + o + xc;
  T* const xo = XUPD ? xs + o + xc : nullptr;
  const cplx l = op.lam ? op.lam[b] : cplx{0, 0};
  const bool usep = INIT || !first;  // p_in is read
  T bt{};
  if constexpr (!INIT && std::is_same_v<T, cplx>) {
    if (sf.part) {
      // rho = r^T z (the up pass's partials), beta = rho / rho_prev
      if (on) {
        const cplx rn = warp_batch_sum(sf.part, sf.per, b);
        if (!first) bt = cdivv(rn, sf.rho_r[b]);
        if (it.chunk == 0 && it.strip == 0 && lane == 0) sf.rho_w[b] = rn;
      }
    } else if (!first) {
      bt = beta[b];
    }
  } else if (!INIT && !first) {
    bt = beta[b];
  }
  const int ys = it.ys, ye = it.ye;
  const int y0 = ys - 2, ylast = ye;  // staged rows
  const typename S::Src src = S::src(op, x, xc, y0, b);
  int vi = 0, wi = 0;
  auto issue = [&](int yr) {
    if (yr <= ylast) {
      const bool rowok = (unsigned)yr < (unsigned)m, rin = colok && rowok;
      const unsigned off = (unsigned)min(max(yr, 0), m - 1) * (unsigned)m;
      cpv(&vring[vi].v[0][lane], zp + off, rin);
      cpv(&vring[vi].v[1][lane], pp + off, rin && (usep || pend));
      if (XUPD) cpv(&vring[vi].v[2][lane], xo + off, rin && pend);
      S::stage(wring[wi], src, lane, yr, off, rowok);
      vi = wrap_inc(vi, RV);
      wi = wrap_inc(wi, RC);
    }
    cp_commit();
  };
#pragma unroll
  for (int j = 0; j <= RA; ++j) issue(y0 + j);
  int vr = 0, sr = 0;
  cp_wait<RA>();
  if (S::XLANE) __syncwarp();
  typename S::Reg k0 = S::first(wring[0], lane), k1 = k0;  // rows yi, yi-1
  // p at rows yi, yi-1, yi-2; b (INIT) at rows yi, yi-1
  T p0 = INIT ? vring[0].v[1][lane] : zpb(bt, vring[0].v[1][lane], vring[0].v[0][lane]), p1{}, p2{};
  T b0 = vring[0].v[0][lane], b1{};
  double s0 = 0, s1 = 0;
  TP_UNROLL(TPGPU_STREAM_UNROLL)
  for (int yi = ys - 1; yi <= ylast; ++yi) {
    issue(yi + RA);
    vr = wrap_inc(vr, RV);
    sr = wrap_inc(sr, RC);
    cp_wait<RA>();
    if (S::XLANE) __syncwarp();
    k1 = k0;
    k0 = S::load(wring[sr], lane, k1);
    const T zz = vring[vr].v[0][lane], pv = vring[vr].v[1][lane];
    if (XUPD && pend && own && yi >= ys && yi < ye) xo[(long)yi * m] = xpa(vring[vr].v[2][lane], xab, pv);
    p2 = p1; p1 = p0;
    b1 = b0; b0 = zz;
    p0 = INIT ? pv : zpb(bt, pv, zz);
    // q at row yi-1
    const T Ap = S::apply(k1, l, S::diag(k1, l), p2, p1, p0);
    const int y = yi - 1;
    if (on && own && y >= ys && y < ye) {
      const long i = (long)y * m;
      if (INIT) {
        const T r = b1 - Ap;
        qo[i] = r;
        s0 = sq_acc(b1, s0);
        s1 = sq_acc(r, s1);
      } else {
        po[i] = p1;
        qo[i] = Ap;
        dot_acc(p1, Ap, s0, s1);
      }
    }
  }
  cp_wait<0>();
  warp_pair(s0, s1);
  if (lane == 0 && on) {
    const int ns = (m + OWN - 1) / OWN, nch = (m + rha - 1) / rha;
    const size_t per = (size_t)ns * nch;
    const size_t k = (size_t)b * per + (size_t)it.chunk * ns + it.strip;
    part[2 * k] = s0;
    part[2 * k + 1] = s1;
  }
}

int items_per_batch(int m, int own, int rh = RH) { return ((m + own - 1) / own) * ((m + rh - 1) / rh); }

dim3 grid_for(int m, int own, int nb, int rh = RH, int wpb = WPB) {
  const long warps = (long)items_per_batch(m, own, rh) * nb;
  return dim3((unsigned)((warps + wpb - 1) / wpb));
}

// rows per warp item of the down/up passes: long chunks amortise the 5-6
// halo rows, short ones give the small grids enough warps
// (levels of 1000+ nodes per side: 128 rows -- cfg 3 sweeps 348 -> 331 ms at 64, 318 ms at 128,
// static_init 58.9 -> 57.0 s, profiles/r2l_ab.txt -- there are warps to spare
// and a chunk's six halo rows are amortised over twice the rows)
int rh_for(int m) {
  static const int envb = std::getenv("TPGPU_RHBIG") ? std::atoi(std::getenv("TPGPU_RHBIG")) : 128;
  static const int env = std::getenv("TPGPU_RH") ? std::atoi(std::getenv("TPGPU_RH")) : 0;
  static const int env1 = std::getenv("TPGPU_RH1") ? std::atoi(std::getenv("TPGPU_RH1")) : 0;
  static const int envm = std::getenv("TPGPU_RHMID") ? std::atoi(std::getenv("TPGPU_RHMID")) : 0;
  if (envm > 0 && m >= 1000 && m < 2000) return envm;  // A/B: the first Galerkin level of a 2048-cell grid
  if (m >= 1000) return envb;
  if (env > 0 && m >= 200) return env;
  if (env1 > 0 && m >= 100 && m < 200) return env1;
  return m >= 200 ? 32 : m >= 100 ? 16 : m >= 50 ? 16 : 8;
}

// rows per warp item of the apply pass: RHA, 64 on levels of 1000+ nodes per
// side (TPGPU_RHA_BIG overrides)
int rha_for(int m) {
  static const int envb = std::getenv("TPGPU_RHA_BIG") ? std::atoi(std::getenv("TPGPU_RHA_BIG")) : 64;
  return m >= 1000 ? envb : RHA;
}

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

template <class S, int NB, int RA, int WPBK, bool FUSED = false, bool BULK = false, class T = typename S::T>
void down_t(Problem& p, const FineOp& op, const T* r, T* z2, T* bc, int mc, const int* active, double om1,
            double om2, int nb, const T* q = nullptr, const T* alpha = nullptr, T* rout = nullptr,
            double* part = nullptr, const ScalFuse* sf = nullptr) {
  constexpr size_t sm = ring_smem<S, FUSED ? 2 : NB, RA, WPBK>() + (BULK ? (size_t)WPBK * (RA + 2) * 8 : 0);
  static bool attrs = [] {
    cudaFuncSetAttribute(k_stream_down<S, NB, RA, WPBK, FUSED, BULK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sm);
    return true;
  }();
  (void)attrs;
  const int rh = rh_for(op.m);
  launch_pdl(k_stream_down<S, NB, RA, WPBK, FUSED, BULK>, grid_for(op.m, 26, (nb + NB - 1) / NB, rh, WPBK), dim3(WL * WPBK),
             sm, p.cur_stream(), op, r, z2, bc, mc, rh, active, om1, om2, nb, q, alpha, rout, part,
             sf ? *sf : ScalFuse{});
}

template <class S, int NB, int RA, int WPBK, bool BULK = false, class T = typename S::T>
void up_t(Problem& p, const FineOp& op, const T* r, const T* z2, const T* xc, int mc, T* z, const int* active,
          double om1, double om2, int nb, int dot, double* part) {
  constexpr size_t sm = ring_smem<S, 4 * NB, RA, WPBK>() + (BULK ? (size_t)WPBK * (RA + 2) * 8 : 0);
  static bool attrs = [] {
    cudaFuncSetAttribute(k_stream_up<S, NB, RA, WPBK, BULK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    return true;
  }();
  (void)attrs;
  const int rh = rh_for(op.m);
  launch_pdl(k_stream_up<S, NB, RA, WPBK, BULK>, grid_for(op.m, 28, (nb + NB - 1) / NB, rh, WPBK), dim3(WL * WPBK), sm,
             p.cur_stream(), op, r, z2, xc, mc, rh, z, active, om1, om2, nb, dot, part);
}

template <class S, int RA, int W, class T = typename S::T>
void apply_t(Problem& p, const FineOp& op, const T* z, const T* pin, T* pout, T* q, const T* beta, const int* active,
             int first, int nb, double* part, bool init, T* x, const T* xa, const ScalFuse* sf = nullptr) {
  const ScalFuse sfv = sf ? *sf : ScalFuse{};
  constexpr size_t sm = ring_smem<S, 2, RA, W>();
  constexpr size_t sm3 = ring_smem<S, 3, RA, W>();
  static bool attrs = [] {
    cudaFuncSetAttribute(k_stream_apply<S, 0, RA, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaFuncSetAttribute(k_stream_apply<S, 1, RA, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaFuncSetAttribute(k_stream_apply<S, 0, RA, W, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm3);
    return true;
  }();
  (void)attrs;
  const int rha = rha_for(op.m);
  const dim3 g = grid_for(op.m, 30, nb, rha, W);
  cudaStream_t s = p.cur_stream();
  FineOp opa = op;
  opa.rha = rha;
  using T0 = T*;
  using C0 = const T*;
  if (init)
    launch_pdl(k_stream_apply<S, 1, RA, W>, g, dim3(WL * W), sm, s, opa, z, pin, pout, q, beta, active, first, nb, part,
               T0(nullptr), C0(nullptr), ScalFuse{});
  else if (xa)
    launch_pdl(k_stream_apply<S, 0, RA, W, true>, g, dim3(WL * W), sm3, s, opa, z, pin, pout, q, beta, active, first,
               nb, part, x, xa, sfv);
  else
    launch_pdl(k_stream_apply<S, 0, RA, W>, g, dim3(WL * W), sm, s, opa, z, pin, pout, q, beta, active, first, nb, part,
               T0(nullptr), C0(nullptr), sfv);
  TP_LAUNCHED(&p);
}

}  // namespace

int fine_partials(int m, int kind) {
  return kind == 0 ? items_per_batch(m, 30, rha_for(m)) : items_per_batch(m, kind == 1 ? 26 : 28, rh_for(m));
}

void launch_fine_apply(Problem& p, const FineOp& op, const cplx* z, const cplx* pin, cplx* pout, cplx* q,
                       const cplx* beta, const int* active, int first, int nb, double* part, bool init, cplx* x,
                       const cplx* xa, const ScalFuse* sf) {
  apply_t<Five, 4, 4>(p, op, z, pin, pout, q, beta, active, first, nb, part, init, x, xa, sf);
}

// slice mode: the fine-level Jacobian apply (p = z + beta p, q = J p, p^T q;
// or the initial residual; with xa: the deferred x update)
void launch_fine_apply(Problem& p, const FineOp& op, const double* z, const double* pin, double* pout, double* q,
                       const double* beta, const int* active, int first, int nb, double* part, bool init, double* x,
                       const double* xa) {
  apply_t<SevenJ, 4, 2>(p, op, z, pin, pout, q, beta, active, first, nb, part, init, x, xa);
}

// Down / up pass of one level: Five on the fine level (op.we set), Seven on
// the Galerkin levels (op.K / op.M set).  Frequencies per warp (NB), ring
// depth (RA rows in flight ahead) and warps per block are tuned per stencil
// (two frequencies per warp measured slower on B200: 10.1 vs 9.2 ms per cfg-1
// sweep -- 224 registers halve the resident warps); TPGPU_RA5 / TPGPU_RA5U
// override the ring depths for experiments.
void launch_stream_down(Problem& p, const FineOp& op, const cplx* r, cplx* z2, cplx* bc, int mc,
                        const int* active, double om1, double om2, int nb, const cplx* q, const cplx* alpha,
                        cplx* rout, double* part, const ScalFuse* sf) {
  if (op.we && q) {
    // vector rows by bulk copies (TPGPU_BULK=1; measured slower than the
    // per-lane cp.async rings: cfg 3 302-304 vs 294 ms per sweep, cfg 1 3.14
    // vs 2.89 ms, the fine down / up passes 82 / 64 vs 73 / 60 ms of kernel,
    // profiles/r2z_ab.txt -- one lane issuing after a __syncwarp and the
    // mbarrier wait sit on each row's critical path; default off)
    static const int bulk = env_int("TPGPU_BULK", 0);
    if (bulk) down_t<Five, 1, 6, 4, true, true>(p, op, r, z2, bc, mc, active, om1, om2, nb, q, alpha, rout, part, sf);
    else down_t<Five, 1, 6, 4, true>(p, op, r, z2, bc, mc, active, om1, om2, nb, q, alpha, rout, part, sf);
  } else if (op.we) {
    static const int ra = env_int("TPGPU_RA5", 6);
    if (ra == 4) down_t<Five, 1, 4, 4>(p, op, r, z2, bc, mc, active, om1, om2, nb);
    else down_t<Five, 1, 6, 4>(p, op, r, z2, bc, mc, active, om1, om2, nb);
  } else if (!op.M) {
    static const int nb7 = env_int("TPGPU_NB7", 1);
    if (nb7 == 2) down_t<SevenK, 2, 2, 2>(p, op, r, z2, bc, mc, active, om1, om2, nb);
    else down_t<SevenK, 1, 2, 2>(p, op, r, z2, bc, mc, active, om1, om2, nb);
  } else {
    static const int ra = env_int("TPGPU_RA7", 2), w = env_int("TPGPU_WPB7", 2);
    if (ra == 4) down_t<Seven, 1, 4, 2>(p, op, r, z2, bc, mc, active, om1, om2, nb);
    else if (w == 4) down_t<Seven, 1, 2, 4>(p, op, r, z2, bc, mc, active, om1, om2, nb);
    else if (w == 1) down_t<Seven, 1, 2, 1>(p, op, r, z2, bc, mc, active, om1, om2, nb);
    else down_t<Seven, 1, 2, 2>(p, op, r, z2, bc, mc, active, om1, om2, nb);
  }
  TP_LAUNCHED(&p);
}

void launch_stream_up(Problem& p, const FineOp& op, const cplx* r, const cplx* z2, const cplx* xc, int mc,
                      cplx* z, const int* active, double om1, double om2, int nb, int dot, double* part) {
  if (op.we) {
    static const int ra = env_int("TPGPU_RA5U", 2);
    static const int bulk = env_int("TPGPU_BULK", 0);
    if (ra == 4) up_t<Five, 1, 4, 4>(p, op, r, z2, xc, mc, z, active, om1, om2, nb, dot, part);
    else if (bulk) up_t<Five, 1, 2, 4, true>(p, op, r, z2, xc, mc, z, active, om1, om2, nb, dot, part);
    else up_t<Five, 1, 2, 4>(p, op, r, z2, xc, mc, z, active, om1, om2, nb, dot, part);
  } else if (!op.M) {
    static const int nb7 = env_int("TPGPU_NB7", 1);
    if (nb7 == 2) up_t<SevenK, 2, 2, 2>(p, op, r, z2, xc, mc, z, active, om1, om2, nb, dot, part);
    else up_t<SevenK, 1, 2, 2>(p, op, r, z2, xc, mc, z, active, om1, om2, nb, dot, part);
  } else {
    static const int ra = env_int("TPGPU_RA7U", 2), w = env_int("TPGPU_WPB7", 2);
    if (ra == 4) up_t<Seven, 1, 4, 2>(p, op, r, z2, xc, mc, z, active, om1, om2, nb, dot, part);
    else if (w == 4) up_t<Seven, 1, 2, 4>(p, op, r, z2, xc, mc, z, active, om1, om2, nb, dot, part);
    else if (w == 1) up_t<Seven, 1, 2, 1>(p, op, r, z2, xc, mc, z, active, om1, om2, nb, dot, part);
    else up_t<Seven, 1, 2, 2>(p, op, r, z2, xc, mc, z, active, om1, om2, nb, dot, part);
  }
  TP_LAUNCHED(&p);
}

// Slice mode (static_init Newton solves): the same passes on real vectors with
// per-slice symmetric Jacobian stencils (op.K = J of level l, op.kstride = 7n)
void launch_stream_down(Problem& p, const FineOp& op, const double* r, double* z2, double* bc, int mc,
                        const int* active, double om1, double om2, int nb, const double* q, const double* alpha,
                        double* rout, double* part) {
  if (q)
    down_t<SevenJ, 1, 4, 2, true>(p, op, r, z2, bc, mc, active, om1, om2, nb, q, alpha, rout, part);
  else if (op.Kf)
    down_t<SevenJF, 1, 4, 2>(p, op, r, z2, bc, mc, active, om1, om2, nb);
  else
    down_t<SevenJ, 1, 4, 2>(p, op, r, z2, bc, mc, active, om1, om2, nb);
  TP_LAUNCHED(&p);
}

void launch_stream_up(Problem& p, const FineOp& op, const double* r, const double* z2, const double* xc, int mc,
                      double* z, const int* active, double om1, double om2, int nb, int dot, double* part) {
  if (op.Kf) up_t<SevenJF, 1, 2, 2>(p, op, r, z2, xc, mc, z, active, om1, om2, nb, dot, part);
  else up_t<SevenJ, 1, 2, 2>(p, op, r, z2, xc, mc, z, active, om1, om2, nb, dot, part);
  TP_LAUNCHED(&p);
}

}  // namespace tpgpu
