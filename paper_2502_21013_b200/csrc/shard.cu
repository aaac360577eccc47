// Multi-GPU plumbing: partition, NCCL communicator, and the exchanges of
// the sharded sweep.
//
// An exact time DFT couples all N slices of every dof (periodic.hpp:161-167),
// so the sweep alternates two layouts:
//   strips      node rows [y0, y1) x all N slices  -- K(u), residual, RHS,
//               forward / inverse DFT (all local), one halo row each side;
//   frequencies k in [k0, k1) x all n dofs          -- the block solves
//               (periodic.hpp:168-170 decoupling: no communication).
// Per sweep: one halo exchange (2 rows x N slices to each neighbour), one
// all-to-all strips -> frequencies before the solves and one back after
// (grouped ncclSend/ncclRecv; every block is contiguous on one side and
// strided on the other, handled by cudaMemcpy2DAsync), and scalar norms
// gathered and summed in rank order (deterministic).  The static
// initialisation is independent per slice, so it runs slice-sharded on the
// full grid and is redistributed to strips by one all-to-all.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <string>

#include "tp_internal.cuh"

namespace tpgpu {

// NCCL is resolved at run time (dlopen on first use, reusing a libnccl
// already loaded by the host process, e.g. torch's), so loading libtpgpu.so
// never pins an NCCL version for the rest of the process.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

static NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(dlsym(h, "ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
    a.Send = reinterpret_cast<decltype(a.Send)>(dlsym(h, "ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(dlsym(h, "ncclRecv"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(dlsym(h, "ncclAllGather"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.GroupStart && a.GroupEnd && a.Send && a.Recv &&
           a.AllGather && a.GetErrorString;
    return a;
  }();
  if (!api.ok) throw Error(TP_ECUDA, "NCCL (libnccl.so.2) could not be loaded");
  return api;
}

#define ncclGetUniqueId(...) ::tpgpu::nccl().GetUniqueId(__VA_ARGS__)
#define ncclCommInitRank(...) ::tpgpu::nccl().CommInitRank(__VA_ARGS__)
#define ncclCommDestroy(...) ::tpgpu::nccl().CommDestroy(__VA_ARGS__)
#define ncclGroupStart() ::tpgpu::nccl().GroupStart()
#define ncclGroupEnd() ::tpgpu::nccl().GroupEnd()
#define ncclSend(...) ::tpgpu::nccl().Send(__VA_ARGS__)
#define ncclRecv(...) ::tpgpu::nccl().Recv(__VA_ARGS__)
#define ncclAllGather(...) ::tpgpu::nccl().AllGather(__VA_ARGS__)
#define ncclGetErrorString(...) ::tpgpu::nccl().GetErrorString(__VA_ARGS__)

#define TP_NCCL(x)                                                                              \
  do {                                                                                          \
    ncclResult_t tp_r_ = (x);                                                                   \
    if (tp_r_ != ncclSuccess)                                                                   \
      throw Error(TP_ECUDA, std::string("NCCL error ") + ncclGetErrorString(tp_r_) + " at " +   \
                                __FILE__ + ":" + std::to_string(__LINE__) + ": " #x);           \
  } while (0)

// ---------------------------------------------------------------- transport
// Every exchange of the sharded sweep is one of two patterns: a grouped set
// of point-to-point transfers (halo rows, the three all-to-alls) or an
// all-gather of a few doubles (rank-ordered norms, min/max).  tp_comm carries
// the backend: NCCL over NVLink (production, one process per GPU), or a
// host-staged exchange through a caller callback (tp_comm_create_host: device
// buffers are staged through pinned host memory, the callback moves bytes
// between processes, e.g. over gloo).  The host backend lets several ranks
// share one GPU without any kernel waiting on another process's kernel: the
// stream is drained before the callback and refilled after it.
struct P2P {
  int peer;
  void* buf;  // device
  size_t bytes;
};

static void host_stage_grow(tp_comm* c, size_t bytes) {
  if (bytes <= c->host_cap) return;
  if (c->host_buf) cudaFreeHost(c->host_buf);
  c->host_buf = nullptr;
  c->host_cap = 0;
  TP_CUDA(cudaMallocHost(&c->host_buf, bytes));
  c->host_cap = bytes;
}

// Grouped point-to-point exchange: sends[i] to sends[i].peer, recvs[i] from
// recvs[i].peer.  Transfers to self pair up in order.
static void comm_exchange(tp_comm* c, const std::vector<P2P>& sends, const std::vector<P2P>& recvs,
                          cudaStream_t stream) {
  if (c->kind == tp_comm::Kind::Nccl) {
    ncclComm_t nc = static_cast<ncclComm_t>(c->comm);
    TP_NCCL(ncclGroupStart());
    for (size_t i = 0; i < std::max(sends.size(), recvs.size()); ++i) {
      if (i < sends.size() && sends[i].bytes)
        TP_NCCL(ncclSend(sends[i].buf, sends[i].bytes, ncclChar, sends[i].peer, nc, stream));
      if (i < recvs.size() && recvs[i].bytes)
        TP_NCCL(ncclRecv(recvs[i].buf, recvs[i].bytes, ncclChar, recvs[i].peer, nc, stream));
    }
    TP_NCCL(ncclGroupEnd());
    return;
  }
  // host-staged: self transfers stay on the device; remote ones go through
  // one pinned staging area (sends first, then receives)
  std::vector<const P2P*> self_s, self_r, rs, rr;
  for (const P2P& t : sends) (t.peer == c->rank ? self_s : rs).push_back(&t);
  for (const P2P& t : recvs) (t.peer == c->rank ? self_r : rr).push_back(&t);
  require(self_s.size() == self_r.size(), "comm: unmatched self transfer");
  for (size_t i = 0; i < self_s.size(); ++i) {
    require(self_s[i]->bytes == self_r[i]->bytes, "comm: self transfer size mismatch");
    if (self_s[i]->bytes)
      TP_CUDA(cudaMemcpyAsync(self_r[i]->buf, self_s[i]->buf, self_s[i]->bytes, cudaMemcpyDeviceToDevice, stream));
  }
  size_t tot = 0;
  for (auto* t : rs) tot += t->bytes;
  for (auto* t : rr) tot += t->bytes;
  host_stage_grow(c, tot);
  char* h = static_cast<char*>(c->host_buf);
  std::vector<int32_t> sp, rp;
  std::vector<const void*> sb;
  std::vector<void*> rb;
  std::vector<size_t> sz, rz;
  size_t off = 0;
  for (auto* t : rs) {
    if (t->bytes) TP_CUDA(cudaMemcpyAsync(h + off, t->buf, t->bytes, cudaMemcpyDeviceToHost, stream));
    sp.push_back(t->peer);
    sb.push_back(h + off);
    sz.push_back(t->bytes);
    off += t->bytes;
  }
  for (auto* t : rr) {
    rp.push_back(t->peer);
    rb.push_back(h + off);
    rz.push_back(t->bytes);
    off += t->bytes;
  }
  TP_CUDA(cudaStreamSynchronize(stream));
  const int rc = c->host_fn(c->host_user, (int32_t)sp.size(), sp.data(), sb.data(), sz.data(), (int32_t)rp.size(),
                            rp.data(), rb.data(), rz.data());
  if (rc != 0) throw Error(TP_ECUDA, "host transport callback failed (" + std::to_string(rc) + ")");
  for (size_t i = 0; i < rr.size(); ++i)
    if (rr[i]->bytes) TP_CUDA(cudaMemcpyAsync(rr[i]->buf, rb[i], rr[i]->bytes, cudaMemcpyHostToDevice, stream));
  // the staging area is reused by the next exchange: drain the uploads
  TP_CUDA(cudaStreamSynchronize(stream));
}

// dst[q*bytes .. ] = rank q's src (bytes each), all device buffers
static void comm_allgather(tp_comm* c, const void* src, void* dst, size_t bytes, cudaStream_t stream) {
  if (c->kind == tp_comm::Kind::Nccl) {
    TP_NCCL(ncclAllGather(src, dst, bytes, ncclChar, static_cast<ncclComm_t>(c->comm), stream));
    return;
  }
  std::vector<P2P> s, r;
  for (int q = 0; q < c->nranks; ++q) {
    s.push_back({q, const_cast<void*>(src), bytes});
    r.push_back({q, static_cast<char*>(dst) + (size_t)q * bytes, bytes});
  }
  comm_exchange(c, s, r, stream);
}

// Frequencies are dealt to the ranks in boustrophedon ("snake") order --
// rounds of P consecutive frequencies, alternating direction: round 0 gives
// k = 0..P-1 to ranks 0..P-1, round 1 gives k = P..2P-1 to ranks P-1..0 --
// so every rank holds frequencies from the whole spectrum.  The block solves'
// cost falls steeply with k (cfg 3, measured: k = 1..20 take 7-8 COCG
// iterations, k > 140 none; odd-symmetric sources leave every even harmonic
// at round-off, so those take none either): a contiguous split would give rank
// 0 most of the work, and plain round-robin with an even P would give some
// ranks only even (free) harmonics.  In memory the spectrum is stored in
// slot order (slot s holds frequency kperm[s]): each rank's frequencies are
// a contiguous slot block [ks[r], ks[r+1]), so the all-to-alls stay block
// transfers; only the time-DFT kernels index by the permutation.
void make_partition(int m, int K, int N, int P, int r, ShardInfo& sh) {
  require(P >= 1 && r >= 0 && r < P, "shard: rank out of range");
  require(m >= P, "shard: more ranks than grid rows");
  require(K >= P, "shard: more ranks than frequencies");
  require(N >= P, "shard: more ranks than time slices");
  sh.P = P;
  sh.r = r;
  sh.ys.resize(P + 1);
  sh.ks.resize(P + 1);
  sh.ss.resize(P + 1);
  for (int q = 0; q <= P; ++q) {
    sh.ys[q] = (int)((long)m * q / P);
    sh.ss[q] = (int)((long)N * q / P);
  }
  std::vector<std::vector<int>> own(P);
  for (int k = 0; k < K; ++k) {
    const int round = k / P, pos = k % P;
    own[(round & 1) ? P - 1 - pos : pos].push_back(k);
  }
  sh.kperm.clear();
  sh.ks[0] = 0;
  for (int q = 0; q < P; ++q) {
    sh.kperm.insert(sh.kperm.end(), own[q].begin(), own[q].end());
    sh.ks[q + 1] = sh.ks[q] + (int)own[q].size();
  }
  if (P == 1) sh.kperm.clear();  // identity
  sh.y0 = sh.ys[r];
  sh.y1 = sh.ys[r + 1];
  sh.k0 = sh.ks[r];
  sh.k1 = sh.ks[r + 1];
  sh.s0 = sh.ss[r];
  sh.s1 = sh.ss[r + 1];
  sh.nr = (sh.y1 - sh.y0) * m;
}

// Halo rows of all N slices: my first owned row goes to rank r-1 (its hi),
// my last to rank r+1 (its lo).
void Problem::exchange_halo() {
  if (!sharded()) return;
  const int rows = sh.y1 - sh.y0;
  const size_t nm = (size_t)N * m;
  halo_lo.ensure(nm);
  halo_hi.ensure(nm);
  halo_send.ensure(2 * nm);
  // pack first and last rows of every slice (slice stride nr)
  TP_CUDA(cudaMemcpy2DAsync(halo_send.get(), m * sizeof(double), U.get(), (size_t)sh.nr * sizeof(double),
                            m * sizeof(double), N, cudaMemcpyDeviceToDevice, stream));
  TP_CUDA(cudaMemcpy2DAsync(halo_send.get() + nm, m * sizeof(double), U.get() + (size_t)(rows - 1) * m,
                            (size_t)sh.nr * sizeof(double), m * sizeof(double), N, cudaMemcpyDeviceToDevice,
                            stream));
  std::vector<P2P> sends, recvs;
  if (sh.r > 0) {
    sends.push_back({sh.r - 1, halo_send.get(), nm * sizeof(double)});
    recvs.push_back({sh.r - 1, halo_lo.get(), nm * sizeof(double)});
  }
  if (sh.r < sh.P - 1) {
    sends.push_back({sh.r + 1, halo_send.get() + nm, nm * sizeof(double)});
    recvs.push_back({sh.r + 1, halo_hi.get(), nm * sizeof(double)});
  }
  comm_exchange(sh.comm, sends, recvs, stream);
  // outer boundary ranks: no neighbour -> zero halo (Dirichlet)
  if (sh.r == 0) TP_CUDA(cudaMemsetAsync(halo_lo.get(), 0, nm * sizeof(double), stream));
  if (sh.r == sh.P - 1) TP_CUDA(cudaMemsetAsync(halo_hi.get(), 0, nm * sizeof(double), stream));
}

double Problem::global_sum(double local) {
  if (!sharded()) return local;
  red_all.ensure(sh.P + 1);
  double* d = red_all.get();
  TP_CUDA(cudaMemcpyAsync(d + sh.P, &local, sizeof(double), cudaMemcpyHostToDevice, stream));
  comm_allgather(sh.comm, d + sh.P, d, sizeof(double), stream);
  std::vector<double> h(sh.P);
  TP_CUDA(cudaMemcpyAsync(h.data(), d, sh.P * sizeof(double), cudaMemcpyDeviceToHost, stream));
  TP_CUDA(cudaStreamSynchronize(stream));
  double s = 0;
  for (int q = 0; q < sh.P; ++q) s += h[q];  // rank order: deterministic
  return s;
}

// Element-wise sum over ranks of an integer vector (each rank fills its own
// entries, zeros elsewhere): the per-slice Newton counts of the sharded
// static initialisation.
void Problem::global_sum_ints(std::vector<int>& v) {
  if (!sharded() || v.empty()) return;
  const size_t cnt = v.size();
  DevBuf<int> d((size_t)(sh.P + 1) * cnt);
  int* src = d.get() + (size_t)sh.P * cnt;
  TP_CUDA(cudaMemcpyAsync(src, v.data(), cnt * sizeof(int), cudaMemcpyHostToDevice, stream));
  comm_allgather(sh.comm, src, d.get(), cnt * sizeof(int), stream);
  std::vector<int> h((size_t)sh.P * cnt);
  TP_CUDA(cudaMemcpyAsync(h.data(), d.get(), h.size() * sizeof(int), cudaMemcpyDeviceToHost, stream));
  TP_CUDA(cudaStreamSynchronize(stream));
  for (size_t i = 0; i < cnt; ++i) {
    int acc = 0;
    for (int q = 0; q < sh.P; ++q) acc += h[(size_t)q * cnt + i];
    v[i] = acc;
  }
}

// out[i] = sum over ranks q (in rank order) of all[q * count + i]
__global__ void k_rank_sum(const double* __restrict__ all, int P, int count, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  double s = 0;
  for (int q = 0; q < P; ++q) s += all[(size_t)q * count + i];
  out[i] = s;
}

// Device-resident rank-ordered sum of `count` doubles: gather every rank's
// partials and sum them in rank order into d_out, without a host round trip
// on the NCCL path (deterministic: the same order on every rank).
void Problem::global_sum_dev(const double* d_in, int count, double* d_out) {
  if (!sharded()) {
    if (d_out != d_in) TP_CUDA(cudaMemcpyAsync(d_out, d_in, count * sizeof(double), cudaMemcpyDeviceToDevice, stream));
    return;
  }
  red_all.ensure((size_t)(sh.P + 1) * count);
  double* src = red_all.get() + (size_t)sh.P * count;
  TP_CUDA(cudaMemcpyAsync(src, d_in, count * sizeof(double), cudaMemcpyDeviceToDevice, stream));
  comm_allgather(sh.comm, src, red_all.get(), count * sizeof(double), stream);
  k_rank_sum<<<(count + 127) / 128, 128, 0, stream>>>(red_all.get(), sh.P, count, d_out);
  TP_LAUNCHED(this);
}

void Problem::global_minmax(double* lo, double* hi, int count) {
  if (!sharded()) return;
  red_all.ensure((size_t)2 * count * (sh.P + 1));
  double* d = red_all.get();
  std::vector<double> mine(2 * count);
  for (int i = 0; i < count; ++i) {
    mine[i] = lo[i];
    mine[count + i] = hi[i];
  }
  double* src = d + (size_t)2 * count * sh.P;
  TP_CUDA(cudaMemcpyAsync(src, mine.data(), 2 * count * sizeof(double), cudaMemcpyHostToDevice, stream));
  comm_allgather(sh.comm, src, d, 2 * count * sizeof(double), stream);
  std::vector<double> h((size_t)2 * count * sh.P);
  TP_CUDA(cudaMemcpyAsync(h.data(), d, h.size() * sizeof(double), cudaMemcpyDeviceToHost, stream));
  TP_CUDA(cudaStreamSynchronize(stream));
  for (int q = 0; q < sh.P; ++q)
    for (int i = 0; i < count; ++i) {
      lo[i] = std::fmin(lo[i], h[(size_t)q * 2 * count + i]);
      hi[i] = std::fmax(hi[i], h[(size_t)q * 2 * count + count + i]);
    }
}

// Ghat (K x nr, my strip) -> Ghat_f ((k1-k0) x n, my frequencies).
// To rank q: rows [ks[q], ks[q+1]) of my Ghat -- contiguous.  From rank q:
// its strip of my frequencies, (k1-k0) x n_q, received into staging and
// scattered into the columns [ys[q]*m, ys[q+1]*m) of Ghat_f.
void Problem::alltoall_to_freq(const cplx* src, cplx* dst) {
  if (!src) src = Ghat.get();
  if (!dst) dst = Ghat_f.get();
  const int Kr = sh.k1 - sh.k0;
  size_t off = 0;
  std::vector<size_t> soff(sh.P);
  for (int q = 0; q < sh.P; ++q) {
    soff[q] = off;
    off += (size_t)Kr * (sh.ys[q + 1] - sh.ys[q]) * m;
  }
  xstage.ensure(off);
  std::vector<P2P> sends, recvs;
  for (int q = 0; q < sh.P; ++q) {
    const size_t cnt_send = (size_t)(sh.ks[q + 1] - sh.ks[q]) * sh.nr * sizeof(cplx);
    const size_t cnt_recv = (size_t)Kr * (sh.ys[q + 1] - sh.ys[q]) * m * sizeof(cplx);
    sends.push_back({q, const_cast<cplx*>(src) + (size_t)sh.ks[q] * sh.nr, cnt_send});
    recvs.push_back({q, xstage.get() + soff[q], cnt_recv});
  }
  comm_exchange(sh.comm, sends, recvs, stream);
  for (int q = 0; q < sh.P; ++q) {
    const size_t nq = (size_t)(sh.ys[q + 1] - sh.ys[q]) * m;
    TP_CUDA(cudaMemcpy2DAsync(dst + (size_t)sh.ys[q] * m, (size_t)n * sizeof(cplx), xstage.get() + soff[q],
                              nq * sizeof(cplx), nq * sizeof(cplx), Kr, cudaMemcpyDeviceToDevice, stream));
  }
}

// Uhat_f ((k1-k0) x n) -> Uhat (K x nr): the reverse of alltoall_to_freq.
void Problem::alltoall_from_freq() {
  const int Kr = sh.k1 - sh.k0;
  size_t off = 0;
  std::vector<size_t> soff(sh.P);
  for (int q = 0; q < sh.P; ++q) {
    soff[q] = off;
    off += (size_t)Kr * (sh.ys[q + 1] - sh.ys[q]) * m;
  }
  xstage.ensure(off);
  for (int q = 0; q < sh.P; ++q) {
    const size_t nq = (size_t)(sh.ys[q + 1] - sh.ys[q]) * m;
    TP_CUDA(cudaMemcpy2DAsync(xstage.get() + soff[q], nq * sizeof(cplx), Uhat_f.get() + (size_t)sh.ys[q] * m,
                              (size_t)n * sizeof(cplx), nq * sizeof(cplx), Kr, cudaMemcpyDeviceToDevice, stream));
  }
  std::vector<P2P> sends, recvs;
  for (int q = 0; q < sh.P; ++q) {
    const size_t cnt_send = (size_t)Kr * (sh.ys[q + 1] - sh.ys[q]) * m * sizeof(cplx);
    const size_t cnt_recv = (size_t)(sh.ks[q + 1] - sh.ks[q]) * sh.nr * sizeof(cplx);
    sends.push_back({q, xstage.get() + soff[q], cnt_send});
    recvs.push_back({q, Uhat.get() + (size_t)sh.ks[q] * sh.nr, cnt_recv});
  }
  comm_exchange(sh.comm, sends, recvs, stream);
}

// Us: my static-init slices [s0, s1) on the full grid ((s1-s0) x n).  To
// rank q: rows of q's strip for my slices (strided, packed); from rank q:
// its slices of my strip, contiguous at U + ss[q]*nr.
void Problem::slices_to_strips(const double* Us) {
  const int Ns = sh.s1 - sh.s0;
  DevBuf<double> pack((size_t)Ns * n);
  size_t off = 0;
  std::vector<size_t> soff(sh.P);
  for (int q = 0; q < sh.P; ++q) {
    soff[q] = off;
    const size_t nq = (size_t)(sh.ys[q + 1] - sh.ys[q]) * m;
    TP_CUDA(cudaMemcpy2DAsync(pack.get() + off, nq * sizeof(double), Us + (size_t)sh.ys[q] * m, (size_t)n * sizeof(double),
                              nq * sizeof(double), Ns, cudaMemcpyDeviceToDevice, stream));
    off += (size_t)Ns * nq;
  }
  std::vector<P2P> sends, recvs;
  for (int q = 0; q < sh.P; ++q) {
    const size_t nq = (size_t)(sh.ys[q + 1] - sh.ys[q]) * m;
    sends.push_back({q, pack.get() + soff[q], (size_t)Ns * nq * sizeof(double)});
    recvs.push_back({q, U.get() + (size_t)sh.ss[q] * sh.nr, (size_t)(sh.ss[q + 1] - sh.ss[q]) * sh.nr * sizeof(double)});
  }
  comm_exchange(sh.comm, sends, recvs, stream);
  TP_CUDA(cudaStreamSynchronize(stream));
}

}  // namespace tpgpu

// =================================================================== C ABI

extern "C" {

int tp_shard_plan_make(int32_t cells, int32_t steps, int32_t nranks, int32_t rank, tp_shard_plan* out) {
  try {
    tpgpu::require(out != nullptr, "null plan");
    tpgpu::require(cells >= 2 && steps >= 1, "shard plan: bad sizes");
    tpgpu::ShardInfo sh;
    const int m = cells - 1;
    tpgpu::make_partition(m, steps / 2 + 1, steps, nranks, rank, sh);
    out->nranks = sh.P;
    out->rank = sh.r;
    out->row0 = sh.y0;
    out->row1 = sh.y1;
    out->freq0 = sh.k0;
    out->freq1 = sh.k1;
    out->slice0 = sh.s0;
    out->slice1 = sh.s1;
    out->n_local = sh.nr;
    return TP_OK;
  } catch (const std::exception& e) {
    tpgpu::set_last_error(e.what(), -1.0);
    return TP_EINVAL;
  }
}

int tp_shard_freq_order(int32_t cells, int32_t steps, int32_t nranks, int32_t* slot_to_freq) {
  try {
    tpgpu::require(slot_to_freq != nullptr, "null argument");
    tpgpu::require(cells >= 2 && steps >= 1, "shard plan: bad sizes");
    tpgpu::ShardInfo sh;
    const int K = steps / 2 + 1;
    tpgpu::make_partition(cells - 1, K, steps, nranks, 0, sh);
    for (int s = 0; s < K; ++s) slot_to_freq[s] = sh.kperm.empty() ? s : sh.kperm[s];
    return TP_OK;
  } catch (const std::exception& e) {
    tpgpu::set_last_error(e.what(), -1.0);
    return TP_EINVAL;
  }
}

int tp_nccl_unique_id(unsigned char id[128]) {
  try {
    ncclUniqueId u;
    if (ncclGetUniqueId(&u) != ncclSuccess) return TP_ECUDA;
    static_assert(sizeof(u.internal) == 128, "NCCL unique id size");
    std::memcpy(id, u.internal, 128);
    return TP_OK;
  } catch (const std::exception& e) {
    tpgpu::set_last_error(e.what(), -1.0);
    return TP_ECUDA;
  }
}

int tp_comm_create(const unsigned char id[128], int32_t nranks, int32_t rank, int32_t device, tp_comm** out) {
  if (!out || nranks < 1 || rank < 0 || rank >= nranks) return TP_EINVAL;
  if (cudaSetDevice(device) != cudaSuccess) return TP_ECUDA;
  try {
    ncclUniqueId u;
    std::memcpy(u.internal, id, 128);
    auto* c = new tp_comm;
    c->nranks = nranks;
    c->rank = rank;
    c->device = device;
    ncclComm_t nc = nullptr;
    if (ncclCommInitRank(&nc, nranks, u, rank) != ncclSuccess) {
      delete c;
      tpgpu::set_last_error("ncclCommInitRank failed", -1.0);
      return TP_ECUDA;
    }
    c->comm = nc;
    c->kind = tp_comm::Kind::Nccl;
    *out = c;
    return TP_OK;
  } catch (const std::exception& e) {
    tpgpu::set_last_error(e.what(), -1.0);
    return TP_ECUDA;
  }
}

int tp_comm_create_host(int32_t nranks, int32_t rank, int32_t device, tp_host_exchange_fn fn, void* user,
                        tp_comm** out) {
  if (!out || !fn || nranks < 1 || rank < 0 || rank >= nranks) return TP_EINVAL;
  if (cudaSetDevice(device) != cudaSuccess) return TP_ECUDA;
  auto* c = new tp_comm;
  c->kind = tp_comm::Kind::Host;
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  c->host_fn = fn;
  c->host_user = user;
  *out = c;
  return TP_OK;
}

void tp_comm_destroy(tp_comm* c) {
  if (!c) return;
  try {
    if (c->kind == tp_comm::Kind::Nccl && c->comm) ncclCommDestroy(static_cast<ncclComm_t>(c->comm));
  } catch (...) {
  }
  if (c->host_buf) cudaFreeHost(c->host_buf);
  delete c;
}

void* tp_comm_nccl(tp_comm* c) { return c && c->kind == tp_comm::Kind::Nccl ? c->comm : nullptr; }
int32_t tp_comm_rank(const tp_comm* c) { return c ? c->rank : -1; }
int32_t tp_comm_size(const tp_comm* c) { return c ? c->nranks : 0; }
int32_t tp_comm_device(const tp_comm* c) { return c ? c->device : -1; }

}  // extern "C"
