// Right-looking blocked LU with partial pivoting, bit-identical to the
// reference's unblocked lane path _lu_lanes (linalg.py:422-449).
//
// Per panel of w columns [J, J+w):
//   1. panel_kernel (cooperative): for each column j of the panel, pivot =
//      first max of |head| over rows >= j (linalg.py:429), swap of the panel
//      rows, singular check (433-436), recip = div(1, pivot) (439),
//      multipliers m_i = mul(A_ij, recip) (441) and the rank-1 update of the
//      remaining panel columns A_ic = add(A_ic, mul(-m_i, A_jc)) (444-448).
//   2. swap_trsm_kernel: the same row exchanges, composed, on every column
//      outside the panel (the reference swaps full rows, 430-431), and in
//      the same pass U12 rows J..J+w-1 of the trailing columns, continuing
//      each element's chain with the panel steps it had not seen yet.
//   3. lu_update (gemm.cu): A22 <- fold_j add(A22, mul(-L21_ij, U12_jc)).
// (laswp_kernel and trsm_kernel are the stand-alone pieces behind the
// distributed driver's mpcore_dev_laswp / mpcore_dev_trsm.)  Columns past
// the m pivoted ones (right-hand sides) take every exchange and update.
// Every element sees the same sequence of add(., mul(-m, u)) operations, in
// the same order, as in the reference; blocking only changes when each link
// runs (SURVEY finding 2).
//
// Panel protocol (per column, no grid barrier, no memory fences): every
// CTA owns a contiguous slice of the panel's rows in shared memory, and all
// cross-CTA data travels as self-validating 8-byte words (32-bit payload |
// 32-bit sequence number; aligned 8-byte accesses are single-copy atomic).
// For column j each CTA
//   (a) updates column j first (look-ahead), then publishes its local
//       first-max candidate: row index, |head| and the pivot value;
//   (b) finishes the rank-1 update of the remaining panel columns and
//       publishes its candidate row (and row j, if it owns it);
//   (c) polls every CTA's candidate words (one L2 round trip), takes the
//       global first max, computes recip = div(1, pivot) from the winner's
//       words (every CTA the same bits) while its other warps stream in the
//       winner's row, and applies the swap.
// Sequence numbers are unique per (LU call, column) and the word buffers are
// double-buffered by column parity, so a slow CTA's step is never
// overwritten before it has been consumed.
#include <climits>
#include <cstdlib>
#include <vector>

#include "internal.h"
#include "mc.cuh"

namespace mpk {

namespace {

constexpr int PANEL_THREADS = 256;
#ifndef POLL_NS
#define POLL_NS 32
#endif
typedef unsigned long long u64;

// GPU-scope relaxed accesses: single-copy atomic 8-byte words, no ordering
// needed beyond that (every word carries its own sequence number).
// (.volatile would be system scope.)
__device__ __forceinline__ void st_volatile(u64 *p, u64 v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v)
               : "memory");
}
__device__ __forceinline__ u64 ld_volatile(const u64 *p) {
  u64 v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ u64 ll_word(unsigned payload, unsigned seq) {
  return ((u64)payload << 32) | seq;
}

// Pivot order of np.argmax(|head|) (linalg.py:429): the first NaN if any,
// else the first maximum.  Magnitudes are >= 0, so their bit patterns order
// like the values; every NaN maps to one key above +inf.
__device__ __forceinline__ unsigned long long mag_key(double m) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(m);
  return b > 0x7FF0000000000000ull ? 0x7FF8000000000000ull : b;
}

// diagnostics (MPCORE_LU_STAMPS): per column index J, globaltimer at the
// first CTA entry / last CTA exit of the panel and exchange+U12 kernels:
// [0] panel entry (min) [1] panel exit (max) [2] swap_trsm entry (min)
// [3] swap_trsm exit (max); null when disabled
__device__ unsigned long long *g_lu_stamps = nullptr;
__device__ __forceinline__ void lu_stamp(int J, int slot, bool is_min) {
  unsigned long long *st = g_lu_stamps;
  if (st == nullptr) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (is_min)
    atomicMin(st + 4 * (int64_t)J + slot, t);
  else
    atomicMax(st + 4 * (int64_t)J + slot, t);
}

#include "panel.cuh"

// diagnostics: globaltimer into a trace slot (around the traced panel)
__global__ void stamp_kernel(unsigned long long *dst) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *dst = t;
}

// One block: advance the sequence base past the previous call's words; on
// 32-bit wrap restart at 0 and zero every exchange word first.
__global__ void __launch_bounds__(1024)
lu_begin_kernel(unsigned *epoch, int32_t *status, unsigned m,
                unsigned long long *w0, int n0, unsigned long long *w1, int n1,
                unsigned long long *w2, int n2) {
  const unsigned long long next =
      (unsigned long long)epoch[0] + epoch[1] + 2ull;
  const bool wrap = next + m + 2ull > 0xFFFFFFFFull;
  __syncthreads();  // every thread has read the old base
  if (wrap) {
    for (int i = threadIdx.x; i < n0; i += blockDim.x) w0[i] = 0ull;
    for (int i = threadIdx.x; i < n1; i += blockDim.x) w1[i] = 0ull;
    for (int i = threadIdx.x; i < n2; i += blockDim.x) w2[i] = 0ull;
  }
  if (threadIdx.x == 0) {
    epoch[0] = wrap ? 0u : (unsigned)next;
    epoch[1] = m;
    status[0] = -1;
  }
}

// Row exchanges of panel [J, J+w) on every column outside the panel, using
// the composition the panel kernel left in ws.swap_list (after the swaps,
// row cur[i] holds what row src[i] held before).  One thread per (column,
// plane): all loads, then all stores.
template <int K>
__global__ void __launch_bounds__(128)
laswp_kernel(MatView A, int c0, int c1, int c2, int c3,
             const int32_t *__restrict__ swap_list,
             const int32_t *__restrict__ status) {
  if (status[0] >= 0) return;
  __shared__ int cur[2 * LU_MAX_W], src[2 * LU_MAX_W];
  __shared__ int cnt;
  if (threadIdx.x < 2 * LU_MAX_W) {
    cur[threadIdx.x] = swap_list[threadIdx.x];
    src[threadIdx.x] = swap_list[2 * LU_MAX_W + threadIdx.x];
  }
  if (threadIdx.x == 0) cnt = swap_list[4 * LU_MAX_W];
  __syncthreads();
  const int m = cnt;
  if (m == 0) return;
  const int n1 = c1 - c0, n2 = c3 - c2, ncols = n1 + n2;
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ncols * K) return;
  int c = t / ncols, q = t % ncols;
  int col = q < n1 ? c0 + q : c2 + (q - n1);
  double *p = A.p + c * A.plane + col;
  double v[2 * LU_MAX_W];
#pragma unroll
  for (int i = 0; i < 2 * LU_MAX_W; ++i)
    if (i < m) v[i] = p[(int64_t)src[i] * A.ld];
#pragma unroll
  for (int i = 0; i < 2 * LU_MAX_W; ++i)
    if (i < m) p[(int64_t)cur[i] * A.ld] = v[i];
}

// U12 = panel rows [J, J+w) of the trailing columns.  Thread (jj, cl) owns
// element (J+jj, col); at step t every row jj > t applies
// add(U_jj, mul(-L_jj,t, U_t)) once U_t is final (wavefront over t).
template <int K, int W, int TC>
__global__ void __launch_bounds__(W *TC)
trsm_kernel(MatView L11, MatView U12, int w, int ncols,
            const int32_t *__restrict__ status) {
  if (status[0] >= 0) return;
  __shared__ double Ls[W][W][K];
  __shared__ double Ts[W][TC][K];
  const int tid = threadIdx.x;
  const int jj = tid / TC, cl = tid % TC;
  const int col = blockIdx.x * TC + cl;
  for (int e = tid; e < w * w; e += W * TC) {
    int r = e / w, q = e % w;
    if (q < r) {
#pragma unroll
      for (int c = 0; c < K; ++c)
        Ls[r][q][c] = -L11.p[c * L11.plane + (int64_t)r * L11.ld + q];
    }
  }
  const bool mine = jj < w && col < ncols;
  if (mine) {
#pragma unroll
    for (int c = 0; c < K; ++c)
      Ts[jj][cl][c] = U12.p[c * U12.plane + (int64_t)jj * U12.ld + col];
  }
  __syncthreads();
  for (int t = 0; t + 1 < w; ++t) {
    if (mine && jj > t) {
      double acc[K], l[K], u[K];
#pragma unroll
      for (int c = 0; c < K; ++c) {
        acc[c] = Ts[jj][cl][c];
        l[c] = Ls[jj][t][c];
        u[c] = Ts[t][cl][c];
      }
      mc::madd<K>(acc, l, u);
#pragma unroll
      for (int c = 0; c < K; ++c) Ts[jj][cl][c] = acc[c];
    }
    __syncthreads();
  }
  if (mine) {
#pragma unroll
    for (int c = 0; c < K; ++c)
      U12.p[c * U12.plane + (int64_t)jj * U12.ld + col] = Ts[jj][cl][c];
  }
}

// Row exchanges + U12 in one pass, one warp per column (lane = panel row):
// every read of the column (the composed exchange sources and the post-
// exchange panel rows) happens before any write, so the exchanges need no
// second sweep; U12 = L11^-1 A12 runs in registers, x_t broadcast by
// shuffles (no CTA barrier per step).  Columns [c2, c3) get both, [c0, c1)
// (the already factored L columns) only the exchanges.
template <int K, int LPC>
__global__ void __launch_bounds__(128)
swap_trsm_kernel(MatView A, int J, int w, int c0, int c1, int c2, int c3,
                 const int32_t *__restrict__ swap_list,
                 const int32_t *__restrict__ status) {
  // LPC lanes per column: 32 (one row per lane) or 16 (rows r and 31-r per
  // lane -- the triangle's shrinking work stays balanced, so a warp does
  // 46 madd steps for two columns instead of 62); the slot code below also
  // takes LPC = 8 (four rows per lane, 19 steps per column), measured no
  // faster than 16
  constexpr int CPW = 32 / LPC, CPB = 4 * CPW, NE = 2 * LU_MAX_W / LPC;
  if (threadIdx.x == 0) lu_stamp(J, 2, true);
  if (status[0] >= 0) return;
  __shared__ int cur[2 * LU_MAX_W], src[2 * LU_MAX_W], rsrc[LU_MAX_W];
  __shared__ double Ls[K][LU_MAX_W][LU_MAX_W + 1];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int sl = lane % LPC, gbase = lane - sl;   // sub-lane, group's lane 0
  const int nright = (c3 - c2 + CPB - 1) / CPB;
  const bool right = (int)blockIdx.x < nright;
  const int cslot = warp * CPW + lane / LPC;
  const int col = right ? c2 + blockIdx.x * CPB + cslot
                        : c0 + (blockIdx.x - nright) * CPB + cslot;
  const int cend = right ? c3 : c1;
  const int cnt = swap_list[4 * LU_MAX_W];
  if (tid < 2 * LU_MAX_W) {
    cur[tid] = swap_list[tid];
    src[tid] = swap_list[2 * LU_MAX_W + tid];
  }
  if (right) {
    // L11 (strictly lower part, negated): every load issued before the
    // first shared store, so the 8 x K loads per thread share one L2 trip
    constexpr int NIT = (LU_MAX_W * LU_MAX_W) / 128;
    double lv[NIT][K];
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
      const int e = tid + 128 * it, r = e / LU_MAX_W, q = e % LU_MAX_W;
      const bool ok = q < r && r < w;
#pragma unroll
      for (int k = 0; k < K; ++k)
        lv[it][k] = ok ? A.p[k * A.plane + (int64_t)(J + r) * A.ld + J + q]
                       : 0.0;
    }
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
      const int e = tid + 128 * it, r = e / LU_MAX_W, q = e % LU_MAX_W;
      if (q < r && r < w) {
#pragma unroll
        for (int k = 0; k < K; ++k) Ls[k][r][q] = -lv[it][k];
      }
    }
    if (tid < LU_MAX_W) rsrc[tid] = J + tid;
  }
  __syncthreads();
  // the post-exchange source of each panel row (cur entries are distinct)
  if (right && tid < cnt && cur[tid] < J + w) rsrc[cur[tid] - J] = src[tid];
  __syncthreads();
  const bool live = col < cend;   // (no early return: shuffles below)
  const int64_t ld = A.ld;
  double *pc = A.p + (live ? col : c2);
  // exchange entries sl + LPC*q; with U12 the panel rows are written by the
  // solve below, so only destinations below the panel are kept here
  bool ex[NE];
  double v[NE][K];
#pragma unroll
  for (int q = 0; q < NE; ++q) {
    const int i = sl + LPC * q;
    ex[q] = live && i < cnt && (!right || cur[i] >= J + w);
#pragma unroll
    for (int k = 0; k < K; ++k)
      v[q][k] = ex[q] ? pc[k * A.plane + (int64_t)src[i] * ld] : 0.0;
  }
  // rows of this lane, one per slot s: s LPC + sl for even s, s LPC +
  // LPC - 1 - sl for odd s (LPC = 32: sl; 16: sl, 31 - sl; 8: sl, 15 - sl,
  // 16 + sl, 31 - sl) -- every slot's rows shrink out of the triangle
  // together, so the lanes stay balanced
  constexpr int NS = LU_MAX_W / LPC;
  int rr[NS];
#pragma unroll
  for (int q = 0; q < NS; ++q)
    rr[q] = (q & 1) ? q * LPC + LPC - 1 - sl : q * LPC + sl;
  double u[NS][K];
#pragma unroll
  for (int q = 0; q < NS; ++q)
#pragma unroll
    for (int k = 0; k < K; ++k)
      u[q][k] = (live && right && rr[q] < w)
                    ? pc[k * A.plane + (int64_t)rsrc[rr[q]] * ld]
                    : 0.0;
  __syncwarp();
  if (right) {
    for (int t = 0; t + 1 < w; ++t) {
      // row t lives in slot t / LPC of the sub-lane holding it
      const int st = t / LPC;
      const int srcl =
          gbase + ((st & 1) ? st * LPC + LPC - 1 - t : t - st * LPC);
      double ut[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        double x = u[0][k];
#pragma unroll
        for (int q = 1; q < NS; ++q)
          if (q == st) x = u[q][k];
        ut[k] = __shfl_sync(0xffffffffu, x, srcl);
      }
#pragma unroll
      for (int q = 0; q < NS; ++q) {
        if (t < (q + 1) * LPC - 1) {  // some row of slot q is below t
          double l[K], o[K];
#pragma unroll
          for (int k = 0; k < K; ++k) {
            l[k] = Ls[k][rr[q]][t];
            o[k] = u[q][k];
          }
          mc::madd<K>(o, l, ut);
          const bool upd = rr[q] > t && rr[q] < w;
#pragma unroll
          for (int k = 0; k < K; ++k) u[q][k] = upd ? o[k] : u[q][k];
        }
      }
    }
#pragma unroll
    for (int q = 0; q < NS; ++q) {
      if (live && rr[q] < w) {
#pragma unroll
        for (int k = 0; k < K; ++k)
          pc[k * A.plane + (int64_t)(J + rr[q]) * ld] = u[q][k];
      }
    }
  }
#pragma unroll
  for (int q = 0; q < NE; ++q) {
    if (ex[q]) {
#pragma unroll
      for (int k = 0; k < K; ++k)
        pc[k * A.plane + (int64_t)cur[sl + LPC * q] * ld] = v[q][k];
    }
  }
  if (threadIdx.x == 0) lu_stamp(J, 3, false);
}

template <typename... KArgs, typename... Args>
cudaError_t launch_coop(void (*kern)(KArgs...), dim3 grid, dim3 block,
                        size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  // the panel is the critical path: highest priority so its CTAs are
  // dispatched ahead of a concurrently running trailing update's
  static const int prio = [] {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    return hi;
  }();
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributePriority;
  attr[1].val.priority = prio;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <int K, int W>
size_t panel_smem(int R) {
  return ((size_t)R * (W * K + 1) + W * K) * sizeof(double);
}

template <int K, int W, int SPL>
cudaError_t panel_launch(int G, size_t smem, int n, MatView A, int J, int w,
                         int32_t *d_swaps, LuWork &ws, int slot,
                         cudaStream_t s) {
  auto kern = panel_kernel<K, W, SPL>;
  static size_t configured = 0;
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(
        kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  return launch_coop(kern, dim3(G), dim3(PANEL_THREADS), smem, s, n, A, J, w,
                     d_swaps, ws, slot);
}

template <int K, int W>
cudaError_t panel_k(int n, MatView A, int J, int w, int32_t *d_swaps,
                    LuWork &ws, int slot, cudaStream_t s) {
  const int m = n - J;
  // Rows per CTA: the per-column candidate exchange costs ~0.6 us among 16
  // CTAs, ~0.9 us among 64 and ~1.9 us among 148 (tools/llbench.cu on
  // B200), while warp 0 handles up to 32 rows at the cost of one; so aim
  // for 32+ rows per CTA rather than spreading over every SM.
  static const int rows_target = [] {
    const char *e = std::getenv("MPCORE_PANEL_ROWS");
    int v = e ? std::atoi(e) : 32;
    return v > 0 ? v : 32;
  }();
  int G = min(ws.G, max(1, (m + rows_target - 1) / rows_target));
  const int R = (m + G - 1) / G;
  size_t smem = panel_smem<K, W>(R);
  // the poll keeps every slot's words in registers: size it to G so the
  // panel leaves room for update CTAs on its SMs (look-ahead overlap)
  if (G <= 64)
    return panel_launch<K, W, 2>(G, smem, n, A, J, w, d_swaps, ws, slot, s);
  return panel_launch<K, W, 5>(G, smem, n, A, J, w, d_swaps, ws, slot, s);
}

template <int K, int W>
cudaError_t trsm_k(MatView L11, MatView U12, int w, int ncols,
                   const int32_t *status, cudaStream_t s) {
  constexpr int TC = 256 / W;
  trsm_kernel<K, W, TC><<<(ncols + TC - 1) / TC, W * TC, 0, s>>>(
      L11, U12, w, ncols, status);
  return cudaGetLastError();
}


MatView sub(MatView A, int i, int j) {
  MatView v = A;
  v.p = A.p + (int64_t)i * A.ld + j;
  return v;
}

// -------------------------------------------------------- graph cache ----
struct GraphKey {
  const double *p;
  int64_t ld, plane;
  int k, m, ncols, nb;
  const int32_t *swaps;
  bool operator==(const GraphKey &o) const {
    return p == o.p && ld == o.ld && plane == o.plane && k == o.k &&
           m == o.m && ncols == o.ncols && nb == o.nb && swaps == o.swaps;
  }
};
struct GraphCache {
  struct Entry {
    GraphKey key;
    cudaGraphExec_t exec;
  };
  std::vector<Entry> entries;
};

// exchanges of the last panel (slot list) on [c0, c1) and, with U12, on
// [c2, c3)
cudaError_t lu_swap_trsm(int k, MatView A, int J, int w, int c0, int c1,
                         int c2, int c3, const int32_t *swap_list,
                         const int32_t *status, cudaStream_t s) {
  // CTAs of 4 warps: 4 columns (DD, a lane per row) or 8 (TD/QD)
  const int nl = (max(0, c1 - c0) + 3) / 4, nr = (max(0, c3 - c2) + 3) / 4;
  const int nl2 = (max(0, c1 - c0) + 7) / 8, nr2 = (max(0, c3 - c2) + 7) / 8;
  static const int lpc16_cols = [] {
    const char *e = std::getenv("MPCORE_TRSM_PAIR_COLS");
    return e ? std::atoi(e) : 800;
  }();

  if (nl + nr == 0) return cudaSuccess;
  cudaError_t e = cudaSuccess;
  prof_begin(PROF_TRSM, s);
  auto go = [&](void (*kern)(MatView, int, int, int, int, int, int,
                             const int32_t *, const int32_t *),
                int grid) {
    kern<<<grid, 128, 0, s>>>(A, J, w, c0, c1, c2, c3, swap_list, status);
    return cudaGetLastError();
  };
  switch (k) {
    case 2: e = go(swap_trsm_kernel<2, 32>, nl + nr); break;
    // TD/QD: two columns per warp (fewer madd steps) while the columns
    // fill the GPU; a lane per row (31 instead of 46 dependent steps) once
    // the trailing block is small and the solve is latency-bound
    case 3:
      e = c3 - c2 >= lpc16_cols ? go(swap_trsm_kernel<3, 16>, nl2 + nr2)
                                : go(swap_trsm_kernel<3, 32>, nl + nr);
      break;
    case 4:
      e = c3 - c2 >= lpc16_cols ? go(swap_trsm_kernel<4, 16>, nl2 + nr2)
                                : go(swap_trsm_kernel<4, 32>, nl + nr);
      break;
    default: return cudaErrorInvalidValue;
  }
  prof_end(PROF_TRSM, s);
  return e;
}

// LU of the m x ncols matrix A: ncols == m is the square factorisation;
// ncols < m factors a tall block (the distributed LU's panel), pivoting over
// all m rows and exchanging rows inside the block; ncols > m carries the
// columns beyond m as right-hand sides: they get every row exchange and
// every update (exactly the forward substitution of L y = P b, element by
// element in the reference's order) but no pivots.
//
// Look-ahead (HPL style): after panel P's exchanges and TRSM, the trailing
// update is split into the next panel's columns ("next") and the rest.  The
// next panel is factored on the high-priority side stream as soon as its
// columns are updated, concurrently with the rest of panel P's update on
// the main stream (disjoint columns); the main stream waits for it before
// panel P+1's exchanges.  Per element the order of operations is unchanged.
cudaError_t enqueue_lu(int k, int m, int ncols, MatView A, int32_t *d_swaps,
                       int nb, LuWork &ws, cudaStream_t s) {
  cudaError_t e;
  const bool ahead = ws.side != nullptr &&
                     std::getenv("MPCORE_NO_LOOKAHEAD") == nullptr;
  if ((e = lu_begin(ws, m, s)) != cudaSuccess) return e;
  bool panel_pending = false;  // panel J was factored on the side stream
  const int pc = min(m, ncols);  // columns that are pivoted
  for (int J = 0; J < pc; J += nb) {
    const int w = min(nb, pc - J);
    const int slot = (J / nb) & 1;
    int32_t *sl = ws.swap_list + slot * LU_SWAP_LIST;
    if (panel_pending) {
      if ((e = cudaStreamWaitEvent(s, ws.ev_panel, 0)) != cudaSuccess) return e;
      panel_pending = false;
    } else {
      if ((e = lu_panel(k, m, A, J, w, d_swaps, ws, slot, s)) != cudaSuccess)
        return e;
    }
    const int rest_r = m - J - w, rest_c = ncols - J - w;
    const int J2 = J + w, w2 = min(nb, max(0, pc - J2));
    // exchanges on every other column, U12 of the trailing columns
    if ((e = lu_swap_trsm(k, A, J, w, 0, J, J2, ncols, sl, ws.status, s)) !=
        cudaSuccess)
      return e;
    if (rest_c <= 0 || rest_r <= 0) continue;
    if (!ahead || w2 == 0) {
      if ((e = lu_update(k, rest_r, rest_c, w, sub(A, J2, J), sub(A, J, J2),
                         sub(A, J2, J2), ws.status, s)) != cudaSuccess)
        return e;
      continue;
    }
    // The next panel's columns are updated and factored on the high-priority
    // side stream, while the rest of this panel's update (disjoint
    // columns) runs here: the narrow update overlaps the wide one instead
    // of preceding it.
    // (measured: TD/QD gain from the overlap while the rest of the update is
    // long; DD -- panel-bound -- and the TD/QD tail, where the narrow update
    // is on the panel chain, do better with it ahead of the wide one on the
    // main stream: MPCORE_NEXT_MAIN_COLS, tools/nextcols_sweep.sh)
    static const char *nm_env = std::getenv("MPCORE_NEXT_ON_MAIN");
    static const int nm_cols = [] {
      const char *e = std::getenv("MPCORE_NEXT_MAIN_COLS");
      return e ? std::atoi(e) : 700;
    }();
    static const int nm_cols_dd = [] {
      const char *e = std::getenv("MPCORE_NEXT_MAIN_COLS_DD");
      return e ? std::atoi(e) : INT_MAX;
    }();
    const bool next_on_main =
        nm_env ? std::atoi(nm_env) != 0
               : rest_c - w2 < (k == 2 ? nm_cols_dd : nm_cols);
    cudaStream_t ns = next_on_main ? s : ws.side;
    if (next_on_main &&
        (e = lu_update(k, rest_r, w2, w, sub(A, J2, J), sub(A, J, J2),
                       sub(A, J2, J2), ws.status, s, PROF_UPDATE_NEXT)) !=
            cudaSuccess)
      return e;
    if ((e = cudaEventRecord(ws.ev_next, s)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(ws.side, ws.ev_next, 0)) != cudaSuccess)
      return e;
    if (!next_on_main &&
        (e = lu_update(k, rest_r, w2, w, sub(A, J2, J), sub(A, J, J2),
                       sub(A, J2, J2), ws.status, ns, PROF_UPDATE_NEXT)) !=
            cudaSuccess)
      return e;
    if ((e = lu_panel(k, m, A, J2, w2, d_swaps, ws, slot ^ 1, ws.side)) !=
        cudaSuccess)
      return e;
    if ((e = cudaEventRecord(ws.ev_panel, ws.side)) != cudaSuccess) return e;
    panel_pending = true;
    // ... while the rest of this panel's update runs here
    if (rest_c > w2) {
      if ((e = lu_update(k, rest_r, rest_c - w2, w, sub(A, J2, J),
                         sub(A, J, J2 + w2), sub(A, J2, J2 + w2), ws.status,
                         s)) != cudaSuccess)
        return e;
    }
  }
  if (panel_pending) {  // cannot happen (the last panel has no successor)
    if ((e = cudaStreamWaitEvent(s, ws.ev_panel, 0)) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace

cudaError_t LuWork::init(int sms) {
  G = sms;
  cudaError_t e;
  size_t cw = (size_t)2 * G * LU_CAND_WORDS * sizeof(u64);
  size_t rwb = (size_t)2 * G * LU_ROW_WORDS * sizeof(u64);
  size_t jw = (size_t)2 * LU_ROW_WORDS * sizeof(u64);
  if ((e = cudaMalloc(&cand_words, cw)) != cudaSuccess) return e;
  if ((e = cudaMalloc(&row_words, rwb)) != cudaSuccess) return e;
  if ((e = cudaMalloc(&rowj_words, jw)) != cudaSuccess) return e;
  if ((e = cudaMalloc(&epoch, 2 * sizeof(unsigned))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&status, sizeof(int32_t))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&swap_list, 2 * LU_SWAP_LIST * sizeof(int32_t))) !=
      cudaSuccess)
    return e;
  cudaMemset(swap_list, 0, 2 * LU_SWAP_LIST * sizeof(int32_t));
  cudaMemset(cand_words, 0, cw);
  cudaMemset(row_words, 0, rwb);
  cudaMemset(rowj_words, 0, jw);
  cudaMemset(epoch, 0, 2 * sizeof(unsigned));
  cudaMemset(status, 0xFF, sizeof(int32_t));
  graphs = new GraphCache();
  if (const char *pn = std::getenv("MPCORE_POLL_NS")) poll_ns = std::atoi(pn);
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  if ((e = cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, hi)) !=
      cudaSuccess)
    return e;
  if ((e = cudaEventCreateWithFlags(&ev_next, cudaEventDisableTiming)) !=
          cudaSuccess ||
      (e = cudaEventCreateWithFlags(&ev_panel, cudaEventDisableTiming)) !=
          cudaSuccess)
    return e;
  return cudaDeviceSynchronize();
}

cudaError_t lu_stamps_enable(unsigned long long *buf) {
  return cudaMemcpyToSymbol(g_lu_stamps, &buf, sizeof(buf));
}

cudaError_t lu_begin(LuWork &ws, int m, cudaStream_t s) {
  lu_begin_kernel<<<1, 1024, 0, s>>>(
      ws.epoch, ws.status, (unsigned)m, ws.cand_words,
      2 * ws.G * LU_CAND_WORDS, ws.row_words, 2 * ws.G * LU_ROW_WORDS,
      ws.rowj_words, 2 * LU_ROW_WORDS);
  return cudaGetLastError();
}

cudaError_t lu_panel(int k, int n, MatView A, int J, int w, int32_t *d_swaps,
                     LuWork &ws, int slot, cudaStream_t s) {
  prof_begin(PROF_PANEL, s);
  const bool mark = ws.trace != nullptr && ws.trace_J == J;
  if (mark) stamp_kernel<<<1, 1, 0, s>>>(ws.trace + 32 * 8 + 4);
  cudaError_t e = cudaErrorInvalidValue;
  if (w <= 16) {
    switch (k) {
      case 2: e = panel_k<2, 16>(n, A, J, w, d_swaps, ws, slot, s); break;
      case 3: e = panel_k<3, 16>(n, A, J, w, d_swaps, ws, slot, s); break;
      case 4: e = panel_k<4, 16>(n, A, J, w, d_swaps, ws, slot, s); break;
    }
  } else if (w <= 32) {
    switch (k) {
      case 2: e = panel_k<2, 32>(n, A, J, w, d_swaps, ws, slot, s); break;
      case 3: e = panel_k<3, 32>(n, A, J, w, d_swaps, ws, slot, s); break;
      case 4: e = panel_k<4, 32>(n, A, J, w, d_swaps, ws, slot, s); break;
    }
  }
  if (mark) stamp_kernel<<<1, 1, 0, s>>>(ws.trace + 32 * 8 + 5);
  prof_end(PROF_PANEL, s);
  return e;
}

cudaError_t lu_laswp(int k, MatView A, int c0, int c1, int c2, int c3,
                     const int32_t *swap_list, const int32_t *status,
                     cudaStream_t s) {
  int ncols = (c1 - c0) + (c3 - c2);
  if (ncols <= 0) return cudaSuccess;
  prof_begin(PROF_LASWP, s);
  int blocks = (ncols * k + 127) / 128;
  switch (k) {
    case 2: laswp_kernel<2><<<blocks, 128, 0, s>>>(A, c0, c1, c2, c3, swap_list, status); break;
    case 3: laswp_kernel<3><<<blocks, 128, 0, s>>>(A, c0, c1, c2, c3, swap_list, status); break;
    case 4: laswp_kernel<4><<<blocks, 128, 0, s>>>(A, c0, c1, c2, c3, swap_list, status); break;
    default: return cudaErrorInvalidValue;
  }
  prof_end(PROF_LASWP, s);
  return cudaGetLastError();
}

cudaError_t lu_trsm(int k, MatView L11, MatView U12, int w, int ncols,
                    const int32_t *status, cudaStream_t s) {
  if (ncols <= 0 || w <= 1) return cudaSuccess;
  prof_begin(PROF_TRSM, s);
  cudaError_t e = cudaErrorInvalidValue;
  if (w <= 16) {
    switch (k) {
      case 2: e = trsm_k<2, 16>(L11, U12, w, ncols, status, s); break;
      case 3: e = trsm_k<3, 16>(L11, U12, w, ncols, status, s); break;
      case 4: e = trsm_k<4, 16>(L11, U12, w, ncols, status, s); break;
    }
  } else {
    switch (k) {
      case 2: e = trsm_k<2, 32>(L11, U12, w, ncols, status, s); break;
      case 3: e = trsm_k<3, 32>(L11, U12, w, ncols, status, s); break;
      case 4: e = trsm_k<4, 32>(L11, U12, w, ncols, status, s); break;
    }
  }
  prof_end(PROF_TRSM, s);
  return e;
}

cudaError_t lu_factor_async(int k, int m, int ncols, MatView A,
                            int32_t *d_swaps, int nb, LuWork &ws,
                            cudaStream_t s) {
  cudaError_t e;
  if (nb > LU_MAX_W) nb = LU_MAX_W;
  if (nb < 1) nb = 1;
  static const bool no_graph = std::getenv("MPCORE_NO_GRAPH") != nullptr;
  if (prof_enabled() || no_graph) {
    // direct launches (per-kernel event timing needs them)
    if ((e = enqueue_lu(k, m, ncols, A, d_swaps, nb, ws, s)) != cudaSuccess)
      return e;
  } else {
    GraphCache &gc = *static_cast<GraphCache *>(ws.graphs);
    GraphKey key{A.p, A.ld, A.plane, k, m, ncols, nb, d_swaps};
    cudaGraphExec_t exec = nullptr;
    for (auto &en : gc.entries)
      if (en.key == key) exec = en.exec;
    if (!exec) {
      cudaGraph_t graph;
      if ((e = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal)) !=
          cudaSuccess)
        return e;
      cudaError_t ee = enqueue_lu(k, m, ncols, A, d_swaps, nb, ws, s);
      e = cudaStreamEndCapture(s, &graph);
      if (ee != cudaSuccess) return ee;
      if (e != cudaSuccess) return e;
      // node priorities (the panel's high-priority launch attribute) are
      // ignored by a graph unless asked for: without them the panel waits
      // behind the trailing update's CTAs for SM slots
      static const unsigned gflags =
          std::getenv("MPCORE_GRAPH_NO_PRIO") ? 0u
                                              : cudaGraphInstantiateFlagUseNodePriority;
      e = cudaGraphInstantiate(&exec, graph, gflags);
      cudaGraphDestroy(graph);
      if (e != cudaSuccess) return e;
      if (gc.entries.size() >= 512) {  // tall blocks: one shape per panel
        cudaGraphExecDestroy(gc.entries.front().exec);
        gc.entries.erase(gc.entries.begin());
      }
      gc.entries.push_back({key, exec});
    }
    if ((e = cudaGraphLaunch(exec, s)) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t lu_factor(int k, int m, int ncols, MatView A, int32_t *d_swaps,
                      int nb, LuWork &ws, int32_t *sing_step, cudaStream_t s) {
  cudaError_t e = lu_factor_async(k, m, ncols, A, d_swaps, nb, ws, s);
  if (e != cudaSuccess) return e;
  e = cudaMemcpyAsync(sing_step, ws.status, sizeof(int32_t),
                      cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(s);
}

}  // namespace mpk
