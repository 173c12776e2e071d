// Distributed DD/TD/QD LU with partial pivoting + solve of one n x n system
// (BASELINE config 4): a native, stream-ordered
// per-rank driver.
//
// Layout: 1-D column-block-cyclic, block b (columns [b*nb, (b+1)*nb)) on
// rank b % G; every rank also holds the right-hand side b as one extra
// local column (replicated), so the forward substitution L y = P b rides
// along the factorisation exactly as column n of the one-GPU [A | b] LU.
//
// Per panel P (owner o = P % G), all device-ordered -- the host only
// enqueues, pivots never leave the device until the end:
//   o, side stream S2: tall-block LU of rows [J, n) x the panel's columns
//      (the one-GPU blocked LU restricted to the block, lu_factor_async),
//      then the panel header (absolute pivots + singular status) and the
//      LIVE rows [J, n) x w packed into slot P % 2;
//   every rank, comm stream C: broadcast of that slot (header + live rows
//      only: (n - J) x w x k doubles, not the whole n x nb buffer);
//   every rank, main stream S (after the broadcast's event): the exchanges
//      on its local columns (composed on the device from the header), U12 =
//      L11^-1 A12 and A22 <- fold_j add(A22, mul(-L21_j, U12_j)) (K = w).
// Look-ahead: the owner of P+1 first brings that block up to date on S,
// then factors + packs it on S2 and its broadcast starts on C, while S runs
// the bulk of panel P's update.  Every element keeps the reference's chain
// (linalg.py:422-449 for A and the forward sweep of 496-509 for b), so
// pivots, factors and y are bitwise the one-GPU and the reference's.
//
// Back substitution (linalg.py:510-520) is column-cyclic too: blocks from
// last to first, the owner solves its diagonal block (the one-GPU sweep
// kernel) and applies its columns to the rows above, x_j in descending j
// as the reference does, then passes the vector [partial y | final x]
// (k x n) to the next block's owner; the last owner broadcasts x.
//
// Transport: NCCL (one process per GPU, the communicator bootstrapped from
// a unique id through the C ABI; libnccl is dlopen'ed so libmpcore loads
// without it), or a local world of G virtual ranks served by this process
// on one GPU (broadcast / send = device copies) -- the same host loop, used
// by the bitwise tests.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "dist.h"
#include "mc.cuh"

namespace mpk {

// ------------------------------------------------------------- NCCL ------
namespace {
struct NcclApi {
  bool tried = false, ok = false;
  std::string why;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclBroadcast) broadcast = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclGetErrorString) errorString = nullptr;
};
NcclApi &nccl() {
  static NcclApi a;
  if (a.tried) return a;
  a.tried = true;
  // the copy torch already loaded, if any (one libnccl per process), else
  // MPCORE_NCCL_LIB, else the loader's libnccl.so.2
  void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) {
    if (const char *p = std::getenv("MPCORE_NCCL_LIB")) h = dlopen(p, RTLD_NOW);
  }
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
  if (!h) {
    a.why = std::string("cannot load libnccl.so.2: ") + dlerror();
    return a;
  }
#define SYM(field, name)                                             \
  a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, name));     \
  if (!a.field) {                                                    \
    a.why = std::string("libnccl lacks ") + name;                    \
    return a;                                                        \
  }
  SYM(getUniqueId, "ncclGetUniqueId")
  SYM(commInitRank, "ncclCommInitRank")
  SYM(commDestroy, "ncclCommDestroy")
  SYM(broadcast, "ncclBroadcast")
  SYM(send, "ncclSend")
  SYM(recv, "ncclRecv")
  SYM(groupStart, "ncclGroupStart")
  SYM(groupEnd, "ncclGroupEnd")
  SYM(errorString, "ncclGetErrorString")
#undef SYM
  a.ok = true;
  return a;
}

cudaError_t nccl_err(ncclResult_t r, std::string &err, const char *what) {
  if (r == ncclSuccess) return cudaSuccess;
  err = std::string(what) + ": " + nccl().errorString(r);
  return cudaErrorUnknown;
}
}  // namespace

int nccl_unique_id(unsigned char *out, std::string &err) {
  NcclApi &a = nccl();
  if (!a.ok) { err = a.why; return 1; }
  ncclUniqueId id;
  ncclResult_t r = a.getUniqueId(&id);
  if (r != ncclSuccess) { err = a.errorString(r); return 1; }
  static_assert(sizeof(id.internal) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out, id.internal, 128);
  return 0;
}

struct NcclComm {
  ncclComm_t comm = nullptr;
  int world = 0, rank = 0;
};

void *nccl_comm_init(int world, int rank, const unsigned char *id_bytes,
                     std::string &err) {
  NcclApi &a = nccl();
  if (!a.ok) { err = a.why; return nullptr; }
  ncclUniqueId id;
  std::memcpy(id.internal, id_bytes, 128);
  auto *c = new NcclComm;
  ncclResult_t r = a.commInitRank(&c->comm, world, id, rank);
  if (r != ncclSuccess) {
    err = std::string("ncclCommInitRank: ") + a.errorString(r);
    delete c;
    return nullptr;
  }
  c->world = world;
  c->rank = rank;
  return c;
}

void nccl_comm_destroy(void *comm) {
  auto *c = static_cast<NcclComm *>(comm);
  if (!c) return;
  if (c->comm) nccl().commDestroy(c->comm);
  delete c;
}

// ------------------------------------------------------- transports ------
namespace {

struct Transport {
  virtual ~Transport() = default;
  // buffers[i] = the slot of served rank i (root's holds the data)
  // root: the root's global rank (NCCL) and its index among the buffers
  virtual cudaError_t bcast(std::vector<void *> &bufs, size_t bytes, int root,
                            int root_idx, std::vector<cudaStream_t> &streams,
                            std::string &err) = 0;
  // one message of `bytes` from rank src (buffer sbuf, stream ss) to rank
  // dst (buffer dbuf, stream ds); either side may be remote
  virtual cudaError_t p2p(int src, const void *sbuf, cudaStream_t ss, int dst,
                          void *dbuf, cudaStream_t ds, size_t bytes,
                          std::string &err) = 0;
};

// one process per GPU: the NCCL communicator (this process = one rank)
struct NcclTransport : Transport {
  NcclComm *c;
  explicit NcclTransport(NcclComm *c) : c(c) {}
  cudaError_t bcast(std::vector<void *> &bufs, size_t bytes, int root,
                    int root_idx, std::vector<cudaStream_t> &streams,
                    std::string &err) override {
    (void)root_idx;
    return nccl_err(nccl().broadcast(bufs[0], bufs[0], bytes, ncclUint8, root,
                                     c->comm, streams[0]),
                    err, "ncclBroadcast");
  }
  cudaError_t p2p(int src, const void *sbuf, cudaStream_t ss, int dst,
                  void *dbuf, cudaStream_t ds, size_t bytes,
                  std::string &err) override {
    if (src == c->rank)
      return nccl_err(nccl().send(sbuf, bytes, ncclUint8, dst, c->comm, ss),
                      err, "ncclSend");
    if (dst == c->rank)
      return nccl_err(nccl().recv(dbuf, bytes, ncclUint8, src, c->comm, ds),
                      err, "ncclRecv");
    return cudaSuccess;
  }
};

// G virtual ranks served by this process on one device
struct LocalTransport : Transport {
  std::vector<cudaEvent_t> evs;
  ~LocalTransport() override {
    for (auto e : evs) cudaEventDestroy(e);
  }
  cudaEvent_t ev() {
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    evs.push_back(e);
    return e;
  }
  cudaError_t bcast(std::vector<void *> &bufs, size_t bytes, int root_rank,
                    int root, std::vector<cudaStream_t> &streams,
                    std::string &err) override {
    (void)root_rank;
    cudaEvent_t done = ev();
    cudaError_t e = cudaEventRecord(done, streams[root]);
    for (size_t r = 0; r < bufs.size() && e == cudaSuccess; ++r) {
      if ((int)r == root) continue;
      e = cudaStreamWaitEvent(streams[r], done, 0);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(bufs[r], bufs[root], bytes,
                            cudaMemcpyDeviceToDevice, streams[r]);
    }
    if (e != cudaSuccess) err = cudaGetErrorString(e);
    return e;
  }
  cudaError_t p2p(int src, const void *sbuf, cudaStream_t ss, int dst,
                  void *dbuf, cudaStream_t ds, size_t bytes,
                  std::string &err) override {
    cudaEvent_t done = ev();
    cudaError_t e = cudaEventRecord(done, ss);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(ds, done, 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(dbuf, sbuf, bytes, cudaMemcpyDeviceToDevice, ds);
    if (e != cudaSuccess) err = cudaGetErrorString(e);
    return e;
  }
};

// ---------------------------------------------------------- kernels ------
constexpr int HDR_INTS = 1024;               // panel header: pivots, status
constexpr size_t HDR_BYTES = HDR_INTS * 4;
constexpr int W32 = LU_MAX_W, LIST = 4 * W32 + 1;

// header of the factored panel [J, J+w): absolute pivot rows, the tall LU's
// singular status (relative step or -1) at [HDR_INTS - 1].  After a
// singular step the remaining pivots are undefined in the LU's output: they
// become the identity so no later exchange can leave the matrix.
__global__ void panel_header_kernel(int32_t *hdr, const int32_t *swaps,
                                    const int32_t *status, int J, int w,
                                    int n) {
  const int st = status[0];
  for (int j = threadIdx.x; j < w; j += blockDim.x) {
    int p = J + swaps[j];
    if ((st >= 0 && j >= st) || p < J + j || p >= n) p = J + j;
    hdr[j] = p;
  }
  if (threadIdx.x == 0) hdr[HDR_INTS - 1] = st;
}

// compose the header's exchanges into laswp lists, one thread per chunk of
// 32 (mpcore_dev_laswp's host composition, on the device): after the
// swaps, row cur[i] holds what row src[i] held before
__global__ void compose_lists_kernel(const int32_t *hdr, int J, int w,
                                     int32_t *lists) {
  const int ch = blockIdx.x * blockDim.x + threadIdx.x;
  if (ch * W32 >= w) return;
  int32_t *cur = lists + (size_t)ch * LIST, *src = cur + 2 * W32;
  int cnt = 0;
  for (int i = ch * W32; i < min(w, (ch + 1) * W32); ++i) {
    const int a = J + i, b = hdr[i];
    if (a == b) continue;
    int ia = -1, ib = -1;
    for (int t = 0; t < cnt; ++t) {
      if (cur[t] == a) ia = t;
      if (cur[t] == b) ib = t;
    }
    if (ia < 0) { cur[cnt] = a; src[cnt] = a; ia = cnt++; }
    if (ib < 0) { cur[cnt] = b; src[cnt] = b; ib = cnt++; }
    const int t = src[ia];
    src[ia] = src[ib];
    src[ib] = t;
  }
  cur[4 * W32] = cnt;
}

// rows [0, J) of the back substitution after block [J, J+w) is solved:
// v_i <- add(v_i, mul(U_ij, neg(x_j))) for j = J+w-1 down to J (the
// reference's column sweep, linalg.py:512-519, operand order kept).  U is
// the owner's local block (columns [0, w) of the view), x = v[J .. J+w).
// A thread per row: its U values come in chunks of CH consecutive columns
// (a cache line per plane), the next chunk's loads in flight while the
// current chunk's madds run; the negated x in shared memory.
constexpr int BU_ROWS = 128;
template <int K>
__global__ void __launch_bounds__(BU_ROWS)
back_update_kernel(int J, int w, MatView U, double *__restrict__ v,
                   int64_t vplane) {
  constexpr int CH = K == 2 ? 16 : 8;
  extern __shared__ double xs[];  // [w][K] negated x
  for (int e = threadIdx.x; e < w * K; e += BU_ROWS) {
    const int j = e / K, c = e % K;
    xs[e] = -v[c * vplane + J + j];
  }
  __syncthreads();
  const int i = blockIdx.x * BU_ROWS + threadIdx.x;
  if (i >= J) return;
  double acc[K];
#pragma unroll
  for (int c = 0; c < K; ++c) acc[c] = v[c * vplane + i];
  const double *row = U.p + (int64_t)i * U.ld;
  double cur[CH][K], nxt[CH][K];
  // chunk t covers columns [c1 - CH, c1), c1 = w - t * CH, descending
  auto fetch = [&](int c1, double (&dst)[CH][K]) {
#pragma unroll
    for (int q = 0; q < CH; ++q) {
      const int col = c1 - CH + q;
#pragma unroll
      for (int c = 0; c < K; ++c)
        dst[q][c] = col >= 0 ? row[c * U.plane + col] : 0.0;
    }
  };
  fetch(w, cur);
  for (int c1 = w; c1 > 0; c1 -= CH) {
    if (c1 - CH > 0) fetch(c1 - CH, nxt);
#pragma unroll
    for (int q = CH - 1; q >= 0; --q) {
      const int col = c1 - CH + q;
      if (col < 0) break;
      double t[K], o[K];
      mc::mul<K>(cur[q], xs + (size_t)col * K, t);
      mc::add<K>(acc, t, o);
#pragma unroll
      for (int c = 0; c < K; ++c) acc[c] = o[c];
    }
#pragma unroll
    for (int q = 0; q < CH; ++q)
#pragma unroll
      for (int c = 0; c < K; ++c) cur[q][c] = nxt[q][c];
  }
#pragma unroll
  for (int c = 0; c < K; ++c) v[c * vplane + i] = acc[c];
}

template <int K>
cudaError_t back_update_k(int J, int w, MatView U, double *v, int64_t vplane,
                          cudaStream_t s) {
  const size_t smem = (size_t)w * K * sizeof(double);
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(
        back_update_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
        200 * 1024);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  back_update_kernel<K><<<(J + BU_ROWS - 1) / BU_ROWS, BU_ROWS, smem, s>>>(
      J, w, U, v, vplane);
  return cudaGetLastError();
}

cudaError_t back_update(int k, int J, int w, MatView U, double *v,
                        int64_t vplane, cudaStream_t s) {
  if (J <= 0) return cudaSuccess;
  switch (k) {
    case 2: return back_update_k<2>(J, w, U, v, vplane, s);
    case 3: return back_update_k<3>(J, w, U, v, vplane, s);
    case 4: return back_update_k<4>(J, w, U, v, vplane, s);
  }
  return cudaErrorInvalidValue;
}

MatView at(MatView A, int64_t i, int64_t j) {
  MatView v = A;
  v.p = A.p + i * A.ld + j;
  return v;
}

cudaError_t copy2d(int k, int rows, int cols, double *dst, int64_t ldd,
                   int64_t pd, const double *src, int64_t lds, int64_t ps,
                   cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  cudaError_t e = cudaSuccess;
  for (int c = 0; c < k && e == cudaSuccess; ++c)
    e = cudaMemcpy2DAsync(dst + c * pd, (size_t)ldd * 8, src + c * ps,
                          (size_t)lds * 8, (size_t)cols * 8, (size_t)rows,
                          cudaMemcpyDeviceToDevice, s);
  return e;
}

// U12 = L11^-1 A12 (unit lower L11, w x w, ld/plane of L), blocked by 32:
// each diagonal block by the wavefront kernel, then the rows below it in
// the block get that block's contributions (ascending order)
cudaError_t trsm_blocked(int k, int w, int ncols, MatView L, MatView U,
                         const int32_t *status, cudaStream_t s) {
  cudaError_t e = cudaSuccess;
  for (int sb = 0; sb < w && e == cudaSuccess; sb += W32) {
    const int wb = std::min(W32, w - sb);
    e = lu_trsm(k, at(L, sb, sb), at(U, sb, 0), wb, ncols, status, s);
    if (e == cudaSuccess && sb + wb < w)
      e = lu_update(k, w - sb - wb, ncols, wb, at(L, sb + wb, sb),
                    at(U, sb, 0), at(U, sb + wb, 0), status, s);
  }
  return e;
}

__global__ void never_singular_kernel(int32_t *p) { *p = -1; }

// ------------------------------------------------------- workspace -------
struct RankWork {
  cudaStream_t S = nullptr, C = nullptr;
  cudaEvent_t ev_recv[2] = {}, ev_consumed[2] = {}, ev_blk = nullptr,
              ev_start = nullptr;
  char *slot[2] = {};
  size_t slot_bytes = 0;
  int32_t *lists = nullptr, *swaps_all = nullptr, *status_all = nullptr,
          *tswaps = nullptr, *nosing = nullptr;
  double *v = nullptr, *tmp = nullptr;
  size_t nmax = 0, nbmax = 0;
  int kmax = 0;
};

struct DistWork {
  std::vector<std::unique_ptr<RankWork>> ranks;
  cudaStream_t S2 = nullptr;       // tall-block LUs (shared by local ranks)
  cudaEvent_t ev_packed = nullptr;
};

DistWork &dist_work() {
  static DistWork w;
  return w;
}

cudaError_t ensure_rank(RankWork &r, int k, int n, int nb) {
  cudaError_t e = cudaSuccess;
  if (!r.S) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if ((e = cudaStreamCreateWithFlags(&r.S, cudaStreamNonBlocking)) ||
        (e = cudaStreamCreateWithPriority(&r.C, cudaStreamNonBlocking, hi)))
      return e;
    cudaEvent_t *evs[] = {&r.ev_recv[0], &r.ev_recv[1], &r.ev_consumed[0],
                          &r.ev_consumed[1], &r.ev_blk, &r.ev_start};
    for (auto *p : evs)
      if ((e = cudaEventCreateWithFlags(p, cudaEventDisableTiming))) return e;
    if ((e = cudaMalloc(&r.nosing, sizeof(int32_t)))) return e;
    never_singular_kernel<<<1, 1, 0, r.S>>>(r.nosing);
  }
  if ((size_t)n <= r.nmax && (size_t)nb <= r.nbmax && k <= r.kmax)
    return cudaSuccess;
  // grow-only: the new sizes cover every earlier request
  const size_t nn = std::max((size_t)n, r.nmax),
               bb = std::max((size_t)nb, r.nbmax);
  const int kk = std::max(k, r.kmax);
  if ((e = cudaStreamSynchronize(r.S))) return e;
  if ((e = cudaStreamSynchronize(r.C))) return e;
  void **bufs[] = {(void **)&r.slot[0], (void **)&r.slot[1], (void **)&r.lists,
                   (void **)&r.swaps_all, (void **)&r.status_all,
                   (void **)&r.tswaps, (void **)&r.v, (void **)&r.tmp};
  for (void **p : bufs) {
    if (*p) cudaFree(*p);
    *p = nullptr;  // (a failed allocation below leaves no dangling pointer)
  }
  r.nmax = r.nbmax = 0;
  r.kmax = 0;
  r.slot_bytes = HDR_BYTES + (size_t)kk * nn * bb * sizeof(double);
  const size_t nblk = nn + 2;  // per-panel status (nb >= 1)
  if ((e = cudaMalloc(&r.slot[0], r.slot_bytes)) ||
      (e = cudaMalloc(&r.slot[1], r.slot_bytes)) ||
      (e = cudaMalloc(&r.lists, ((bb + W32 - 1) / W32) * LIST * 4)) ||
      (e = cudaMalloc(&r.swaps_all, nn * 4)) ||
      (e = cudaMalloc(&r.status_all, nblk * 4)) ||
      (e = cudaMalloc(&r.tswaps, bb * 4)) ||
      (e = cudaMalloc(&r.v, (size_t)kk * nn * 8)) ||
      (e = cudaMalloc(&r.tmp, (size_t)kk * bb * 8)))
    return e;
  cudaMemset(r.slot[0], 0, HDR_BYTES);
  cudaMemset(r.slot[1], 0, HDR_BYTES);
  r.nmax = nn;
  r.nbmax = bb;
  r.kmax = kk;
  return cudaDeviceSynchronize();
}

// phase timing (optional): event pairs per phase, summed at the end
struct Phases {
  bool on = false;
  int panel = -1;  // the panel the next records belong to
  std::vector<cudaEvent_t> pool;
  struct Rec {
    int ph, panel;
    cudaEvent_t a, b;
  };
  std::vector<Rec> recs;
  cudaEvent_t open_a[DIST_NPHASES] = {};
  int open_p[DIST_NPHASES] = {};
  cudaEvent_t mk() {
    cudaEvent_t e;
    cudaEventCreate(&e);
    pool.push_back(e);
    return e;
  }
  void begin(int ph, cudaStream_t s) {
    if (!on) return;
    open_a[ph] = mk();
    open_p[ph] = panel;
    cudaEventRecord(open_a[ph], s);
  }
  void end(int ph, cudaStream_t s) {
    if (!on || !open_a[ph]) return;
    cudaEvent_t b = mk();
    cudaEventRecord(b, s);
    recs.push_back({ph, open_p[ph], open_a[ph], b});
    open_a[ph] = nullptr;
  }
  // sums per phase; with MPCORE_DIST_TRACE=path also every record as
  // "phase panel start_ms end_ms" relative to the call's first event
  void collect(double *ms) {
    static const char *names[DIST_NPHASES] = {"total", "factor", "bcast",
                                              "exch_trsm", "update", "back"};
    for (int i = 0; i < DIST_NPHASES; ++i) ms[i] = 0;
    const char *path = std::getenv("MPCORE_DIST_TRACE");
    FILE *f = path ? std::fopen(path, "w") : nullptr;
    if (f) std::fprintf(f, "phase panel start_ms end_ms\n");
    cudaEvent_t origin = recs.empty() ? nullptr : recs.front().a;
    for (auto &r : recs)
      if (r.ph == DIST_TOTAL) origin = r.a;
    for (auto &r : recs) {
      float t = 0, t0 = 0, t1 = 0;
      if (cudaEventSynchronize(r.b) == cudaSuccess &&
          cudaEventElapsedTime(&t, r.a, r.b) == cudaSuccess)
        ms[r.ph] += t;
      if (f && origin && cudaEventElapsedTime(&t0, origin, r.a) == cudaSuccess &&
          cudaEventElapsedTime(&t1, origin, r.b) == cudaSuccess)
        std::fprintf(f, "%s %d %.4f %.4f\n", names[r.ph], r.panel, t0, t1);
    }
    if (f) std::fclose(f);
  }
  ~Phases() {
    for (auto e : pool) cudaEventDestroy(e);
  }
};

}  // namespace

// ---------------------------------------------------------- driver -------
int dist_lu_solve(void *comm, int k, int n, int nb, int G,
                  const std::vector<DistRankView> &views, LuWork &ws,
                  SolveWork &sw, cudaStream_t caller,
                  std::vector<int32_t> &swaps_out, int32_t *sing_step,
                  double *phase_ms, int64_t *launches, std::string &err) {
  cudaError_t e = cudaSuccess;
  const int R = (int)views.size();
  const int nbk = (n + nb - 1) / nb;
  auto fail = [&](cudaError_t ce, const char *what) {
    if (err.empty()) err = std::string(what) + ": " + cudaGetErrorString(ce);
    return 6;
  };
  if (nb < 1 || nb > HDR_INTS - 1 || k < 2 || k > 4 || n < 1 || G < 1 ||
      R < 1) {
    err = "bad distributed LU arguments";
    return 2;
  }
  std::unique_ptr<Transport> T;
  if (comm) {
    auto *c = static_cast<NcclComm *>(comm);
    if (R != 1 || c->world != G || views[0].rank != c->rank) {
      err = "NCCL world / rank do not match the layout";
      return 2;
    }
    T.reset(new NcclTransport(c));
  } else {
    if (R != G) {
      err = "a local world serves every rank";
      return 2;
    }
    T.reset(new LocalTransport);
  }
  DistWork &DW = dist_work();
  while ((int)DW.ranks.size() < R) DW.ranks.emplace_back(new RankWork);
  // diagnostics: MPCORE_DIST_SERIAL=1 runs every stream's work in order on
  // the main stream (no look-ahead overlap)
  static const bool serial = std::getenv("MPCORE_DIST_SERIAL") != nullptr;
  if (!DW.S2) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if ((e = cudaStreamCreateWithPriority(&DW.S2, cudaStreamNonBlocking, hi)) ||
        (e = cudaEventCreateWithFlags(&DW.ev_packed, cudaEventDisableTiming)))
      return fail(e, "streams");
  }
  std::vector<int> idx_of(G, -1);  // rank -> served index
  for (int i = 0; i < R; ++i) {
    if (views[i].rank < 0 || views[i].rank >= G || idx_of[views[i].rank] >= 0) {
      err = "ranks must be distinct and below the world size";
      return 2;
    }
    idx_of[views[i].rank] = i;
  }
  if (phase_ms)
    for (int i = 0; i < DIST_NPHASES; ++i) phase_ms[i] = 0.0;
  for (int i = 0; i < R; ++i)
    if ((e = ensure_rank(*DW.ranks[i], k, n, nb))) return fail(e, "workspace");
  Phases ph;
  ph.on = phase_ms != nullptr && R == 1;
  int64_t nlaunch = 0;
  auto width = [&](int b) { return std::min(nb, n - b * nb); };
  auto owner = [&](int b) { return b % G; };
  auto local_off = [&](int b) { return (b / G) * nb; };
  auto lcols = [&](int r) {
    int c = 0;
    for (int b = r; b < nbk; b += G) c += width(b);
    return c;
  };
  auto tstart = [&](int r, int P, int lc) {
    const int cnt = P < r ? 0 : (P - r) / G + 1;
    return std::min(cnt * nb, lc);
  };
  std::vector<int> lc(R);
  for (int i = 0; i < R; ++i) {
    lc[i] = lcols(views[i].rank);
    if (views[i].cols != lc[i] + 1) {
      err = "local matrix must hold the rank's columns plus b";
      return 2;
    }
  }
  // start: every stream after the caller's queued work (inputs ready)
  {
    cudaEvent_t start;
    cudaEventCreateWithFlags(&start, cudaEventDisableTiming);
    cudaEventRecord(start, caller);
    for (int i = 0; i < R; ++i) {
      cudaStreamWaitEvent(DW.ranks[i]->S, start, 0);
      cudaStreamWaitEvent(DW.ranks[i]->C, start, 0);
    }
    cudaStreamWaitEvent(DW.S2, start, 0);
    cudaEventDestroy(start);
  }
  for (int i = 0; i < R; ++i) ph.begin(DIST_TOTAL, DW.ranks[i]->S);

  auto slot_planes = [&](RankWork &rw, int s) {
    return reinterpret_cast<double *>(rw.slot[s] + HDR_BYTES);
  };
  auto slot_bytes_for = [&](int P) {
    const int J = P * nb, w = width(P);
    return HDR_BYTES + (size_t)k * (n - J) * w * sizeof(double);
  };
  // owner of P, on S2: tall LU, header, pack (after `after` on S)
  auto issue_factor = [&](int P, int i) -> int {
    RankWork &rw = *DW.ranks[i];
    const int J = P * nb, w = width(P), off = local_off(P), s = P % 2;
    const DistRankView &V = views[i];
    cudaStream_t S2 = serial ? rw.S : DW.S2;
    if ((e = cudaEventRecord(rw.ev_blk, rw.S)) ||
        (e = cudaStreamWaitEvent(S2, rw.ev_blk, 0)) ||
        (e = cudaStreamWaitEvent(S2, rw.ev_consumed[s], 0)))
      return fail(e, "factor order");
    ph.panel = P;
    ph.begin(DIST_FACTOR, S2);
    MatView blk = at(V.A, J, off);
    if ((e = lu_factor_async(k, n - J, w, blk, rw.tswaps, 32, ws, S2)))
      return fail(e, "tall-block LU");
    int32_t *hdr = reinterpret_cast<int32_t *>(rw.slot[s]);
    panel_header_kernel<<<1, 256, 0, S2>>>(hdr, rw.tswaps, ws.status, J,
                                              w, n);
    if ((e = cudaGetLastError())) return fail(e, "panel header");
    if ((e = copy2d(k, n - J, w, slot_planes(rw, s), w, (int64_t)(n - J) * w,
                    blk.p, V.A.ld, V.A.plane, S2)))
      return fail(e, "pack");
    ph.end(DIST_FACTOR, S2);
    if ((e = cudaEventRecord(DW.ev_packed, S2)) ||
        (e = cudaStreamWaitEvent(rw.C, DW.ev_packed, 0)))
      return fail(e, "pack order");
    nlaunch += 2;
    return 0;
  };
  // every rank, on C: broadcast of panel P's slot
  auto issue_bcast = [&](int P) -> int {
    const int s = P % 2, root = owner(P);
    std::vector<void *> bufs(R);
    std::vector<cudaStream_t> streams(R);
    for (int i = 0; i < R; ++i) {
      RankWork &rw = *DW.ranks[i];
      if ((e = cudaStreamWaitEvent(rw.C, rw.ev_consumed[s], 0)))
        return fail(e, "slot reuse");
      bufs[i] = rw.slot[s];
      streams[i] = rw.C;
      ph.panel = P;
      ph.begin(DIST_BCAST, rw.C);
    }
    const int root_idx = comm ? 0 : idx_of[root];
    if ((e = T->bcast(bufs, slot_bytes_for(P), root, root_idx, streams, err)))
      return fail(e, "broadcast");
    for (int i = 0; i < R; ++i) {
      RankWork &rw = *DW.ranks[i];
      ph.end(DIST_BCAST, rw.C);
      if ((e = cudaEventRecord(rw.ev_recv[s], rw.C)))
        return fail(e, "broadcast event");
    }
    nlaunch += 1;
    return 0;
  };
  // panel P applied on S to local column ranges: exchanges on `ex`,
  // U12 + update on [c0, c0 + nc)
  auto apply = [&](int P, int i, const std::vector<std::pair<int, int>> &ex,
                   int c0, int nc) -> int {
    RankWork &rw = *DW.ranks[i];
    const DistRankView &V = views[i];
    const int J = P * nb, w = width(P), s = P % 2;
    const double *pl = slot_planes(rw, s);
    MatView Ls{const_cast<double *>(pl), w, (int64_t)(n - J) * w};
    ph.panel = P;
    ph.begin(DIST_EXCH_TRSM, rw.S);
    for (auto &r : ex) {
      if (r.second <= 0) continue;
      for (int ch = 0; ch * W32 < w; ++ch) {
        if ((e = lu_laswp(k, V.A, r.first, r.first + r.second, 0, 0,
                          rw.lists + (size_t)ch * LIST, rw.nosing, rw.S)))
          return fail(e, "exchanges");
        ++nlaunch;
      }
    }
    if (nc > 0) {
      if ((e = trsm_blocked(k, w, nc, Ls, at(V.A, J, c0), rw.nosing, rw.S)))
        return fail(e, "U12");
      nlaunch += 2 * ((w + W32 - 1) / W32);
    }
    ph.end(DIST_EXCH_TRSM, rw.S);
    if (nc > 0 && n - J - w > 0) {
      ph.begin(DIST_UPDATE, rw.S);
      if ((e = gemm(k, true, false, n - J - w, nc, w, at(Ls, w, 0),
                    at(V.A, J, c0), at(V.A, J + w, c0), rw.S)))
        return fail(e, "update");
      ph.end(DIST_UPDATE, rw.S);
      ++nlaunch;
    }
    return 0;
  };

  int st = 0;
  // panel 0
  if (idx_of[owner(0)] >= 0 && (st = issue_factor(0, idx_of[owner(0)])))
    return st;
  if ((st = issue_bcast(0))) return st;
  for (int P = 0; P < nbk; ++P) {
    const int J = P * nb, w = width(P), s = P % 2;
    const bool nxt = P + 1 < nbk;
    for (int i = 0; i < R; ++i) {
      RankWork &rw = *DW.ranks[i];
      const int r = views[i].rank;
      if ((e = cudaStreamWaitEvent(rw.S, rw.ev_recv[s], 0)))
        return fail(e, "receive order");
      const int32_t *hdr = reinterpret_cast<const int32_t *>(rw.slot[s]);
      if ((e = cudaMemcpyAsync(rw.swaps_all + J, hdr, (size_t)w * 4,
                               cudaMemcpyDeviceToDevice, rw.S)) ||
          (e = cudaMemcpyAsync(rw.status_all + P, hdr + HDR_INTS - 1, 4,
                               cudaMemcpyDeviceToDevice, rw.S)))
        return fail(e, "pivots");
      compose_lists_kernel<<<1, 32, 0, rw.S>>>(hdr, J, w, rw.lists);
      if ((e = cudaGetLastError())) return fail(e, "compose");
      ++nlaunch;
      if (nxt && owner(P + 1) == r) {
        // look-ahead: block P+1 first, then its factorisation on S2
        const int off1 = local_off(P + 1), w1 = width(P + 1);
        const std::vector<std::pair<int, int>> blk{{off1, w1}};
        st = apply(P, i, blk, off1, w1);
        if (st) return st;
        if ((st = issue_factor(P + 1, i))) return st;
      }
    }
    if (nxt && (st = issue_bcast(P + 1))) return st;
    for (int i = 0; i < R; ++i) {
      RankWork &rw = *DW.ranks[i];
      const int r = views[i].rank;
      const int L1 = lc[i] + 1;  // local columns + b
      // exchanges: every local column except this panel's own block (the
      // tall LU exchanged it) and block P+1 when done ahead
      std::vector<std::pair<int, int>> ex{{0, L1}};
      auto cut = [&](int a0, int m0) {
        std::vector<std::pair<int, int>> out;
        for (auto &q : ex) {
          const int a = q.first, b = q.first + q.second;
          if (b <= a0 || a >= a0 + m0) {
            out.push_back(q);
            continue;
          }
          if (a < a0) out.push_back({a, a0 - a});
          if (b > a0 + m0) out.push_back({a0 + m0, b - a0 - m0});
        }
        ex.swap(out);
      };
      if (owner(P) == r) cut(local_off(P), w);
      int t0 = tstart(r, P, lc[i]), nt = L1 - t0;
      if (nxt && owner(P + 1) == r) {
        const int w1 = width(P + 1);
        cut(local_off(P + 1), w1);
        t0 += w1;
        nt -= w1;
      }
      if ((st = apply(P, i, ex, t0, nt))) return st;
      if ((e = cudaEventRecord(rw.ev_consumed[s], rw.S)))
        return fail(e, "slot event");
    }
  }
  // ---- back substitution, column-cyclic, blocks last to first ----
  for (int i = 0; i < R; ++i) {
    RankWork &rw = *DW.ranks[i];
    ph.panel = -1;
    ph.begin(DIST_BACK, rw.S);
    const DistRankView &V = views[i];
    if ((e = copy2d(k, n, 1, rw.v, 1, n, V.A.p + lc[i], V.A.ld, V.A.plane,
                    rw.S)))
      return fail(e, "y");
  }
  const size_t vbytes = (size_t)k * n * sizeof(double);
  if (G == 1) {
    // one rank holds all of U: the one-GPU pipelined sweep over the whole
    // triangle (the same per-element chain, rows in one cooperative launch
    // instead of one launch per block)
    RankWork &rw = *DW.ranks[0];
    if ((e = lu_solve_back(k, n, views[0].A, rw.v, sw, rw.S)))
      return fail(e, "back substitution");
    ++nlaunch;
  }
  for (int b = G == 1 ? -1 : nbk - 1; b >= 0; --b) {
    const int o = owner(b), J = b * nb, w = width(b), off = local_off(b);
    if (b < nbk - 1 && owner(b + 1) != o) {
      const int po = owner(b + 1), ip = idx_of[po], io = idx_of[o];
      if ((ip >= 0 || io >= 0) &&
          (e = T->p2p(po, ip >= 0 ? DW.ranks[ip]->v : nullptr,
                      ip >= 0 ? DW.ranks[ip]->S : nullptr, o,
                      io >= 0 ? DW.ranks[io]->v : nullptr,
                      io >= 0 ? DW.ranks[io]->S : nullptr, vbytes, err)))
        return fail(e, "back-substitution hand-off");
      ++nlaunch;
    }
    const int io = idx_of[o];
    if (io < 0) continue;
    RankWork &rw = *DW.ranks[io];
    const DistRankView &V = views[io];
    if ((e = copy2d(k, 1, w, rw.tmp, w, w, rw.v + J, n, n, rw.S)) ||
        (e = lu_solve_back(k, w, at(V.A, J, off), rw.tmp, sw, rw.S)) ||
        (e = copy2d(k, 1, w, rw.v + J, n, n, rw.tmp, w, w, rw.S)) ||
        (e = back_update(k, J, w, at(V.A, 0, off), rw.v, n, rw.S)))
      return fail(e, "back substitution");
    nlaunch += 2;
  }
  // x from the owner of block 0 to every rank
  {
    const int root = owner(0);
    std::vector<void *> bufs(R);
    std::vector<cudaStream_t> streams(R);
    for (int i = 0; i < R; ++i) {
      bufs[i] = DW.ranks[i]->v;
      streams[i] = DW.ranks[i]->S;
    }
    if (G > 1 &&
        (e = T->bcast(bufs, vbytes, root, comm ? 0 : idx_of[root], streams,
                      err)))
      return fail(e, "x broadcast");
    for (int i = 0; i < R; ++i) {
      RankWork &rw = *DW.ranks[i];
      if ((e = cudaMemcpyAsync(views[i].x, rw.v, vbytes,
                               cudaMemcpyDeviceToDevice, rw.S)))
        return fail(e, "x");
      ph.end(DIST_BACK, rw.S);
      ph.end(DIST_TOTAL, rw.S);
    }
  }
  // results: pivots and per-panel status from the first served rank
  RankWork &r0 = *DW.ranks[0];
  std::vector<int32_t> stat(nbk);
  swaps_out.assign(n, 0);
  if ((e = cudaMemcpyAsync(swaps_out.data(), r0.swaps_all, (size_t)n * 4,
                           cudaMemcpyDeviceToHost, r0.S)) ||
      (e = cudaMemcpyAsync(stat.data(), r0.status_all, (size_t)nbk * 4,
                           cudaMemcpyDeviceToHost, r0.S)))
    return fail(e, "results");
  // the caller's stream continues after every rank's work
  for (int i = 0; i < R; ++i) {
    cudaEvent_t done;
    cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
    cudaEventRecord(done, DW.ranks[i]->S);
    cudaStreamWaitEvent(caller, done, 0);
    cudaEventDestroy(done);
  }
  for (int i = 0; i < R; ++i)
    if ((e = cudaStreamSynchronize(DW.ranks[i]->S))) return fail(e, "sync");
  if ((e = cudaStreamSynchronize(DW.S2)) || (e = cudaGetLastError()))
    return fail(e, "sync");
  if (phase_ms) ph.collect(phase_ms);
  if (launches) *launches = nlaunch;
  *sing_step = -1;
  for (int P = 0; P < nbk; ++P)
    if (stat[P] >= 0) {
      *sing_step = P * nb + stat[P];
      err = "no nonzero pivot at elimination step " +
            std::to_string(*sing_step);
      return 3;
    }
  return 0;
}

}  // namespace mpk
