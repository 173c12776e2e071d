// Right-looking blocked LU with partial pivoting, bit-identical to the
// reference's unblocked lane path _lu_lanes (linalg.py:422-449).
//
// Per panel of w columns [J, J+w):
//   1. panel_kernel (cooperative): for each column j of the panel, pivot =
//      first max of |head| over rows >= j (linalg.py:429), swap of the panel
//      rows, singular check (433-436), recip = div(1, pivot) (439),
//      multipliers m_i = mul(A_ij, recip) (441) and the rank-1 update of the
//      remaining panel columns A_ic = add(A_ic, mul(-m_i, A_jc)) (444-448).
//   2. laswp_kernel: the same row exchanges, composed, on every column
//      outside the panel (the reference swaps full rows, 430-431).
//   3. trsm_kernel: U12 rows J..J+w-1 of the trailing columns, continuing
//      each element's chain with the panel steps it had not seen yet.
//   4. lu_update (gemm.cu): A22 <- fold_j add(A22, mul(-L21_ij, U12_jc)).
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
constexpr int NWARPS = PANEL_THREADS / 32;
typedef unsigned long long u64;

__device__ __forceinline__ void st_volatile(u64 *p, u64 v) {
  asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v)
               : "memory");
}
__device__ __forceinline__ u64 ld_volatile(const u64 *p) {
  u64 v;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ u64 ll_word(unsigned payload, unsigned seq) {
  return ((u64)payload << 32) | seq;
}

// (mag, row): larger magnitude wins; ties go to the smaller row
// (np.argmax returns the first maximum, linalg.py:429).
__device__ __forceinline__ bool better(double m1, int r1, double m2, int r2) {
  return m1 > m2 || (m1 == m2 && r1 < r2);
}

__device__ __forceinline__ void block_argmax(double &mag, int &row,
                                             double *s_mag, int *s_row) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    double om = __shfl_down_sync(0xffffffffu, mag, off);
    int orow = __shfl_down_sync(0xffffffffu, row, off);
    if (better(om, orow, mag, row)) { mag = om; row = orow; }
  }
  if (lane == 0) { s_mag[wid] = mag; s_row[wid] = row; }
  __syncthreads();
  if (wid == 0) {
    mag = lane < NWARPS ? s_mag[lane] : -1.0;
    row = lane < NWARPS ? s_row[lane] : INT_MAX;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      double om = __shfl_down_sync(0xffffffffu, mag, off);
      int orow = __shfl_down_sync(0xffffffffu, row, off);
      if (better(om, orow, mag, row)) { mag = om; row = orow; }
    }
    if (lane == 0) { s_mag[NWARPS] = mag; s_row[NWARPS] = row; }
  }
  __syncthreads();
  mag = s_mag[NWARPS];
  row = s_row[NWARPS];
}

struct PanelShared {
  double s_mag[NWARPS + 1];
  int s_row[NWARPS + 1];
  double recip[LU_MAX_K];
  int cand_row;        // local candidate (global row index) of the step
};

// LL word helpers: a double travels as two words (low half, high half)
__device__ __forceinline__ unsigned lo32(double v) {
  return (unsigned)((unsigned long long)__double_as_longlong(v) & 0xffffffffu);
}
__device__ __forceinline__ unsigned hi32(double v) {
  return (unsigned)((unsigned long long)__double_as_longlong(v) >> 32);
}

template <int K, int W>
__global__ void __launch_bounds__(PANEL_THREADS, 1)
panel_kernel(int n, MatView A, int J, int w, int32_t *__restrict__ swaps,
             LuWork ws) {
  const int G = gridDim.x, g = blockIdx.x, tid = threadIdx.x;
  if (ws.status[0] >= 0) return;
  // sequence numbers: unique per LU call (device epoch) and column
  const unsigned seq0 = ws.epoch[0] * 65536u + (unsigned)J + 1u;
  const int m = n - J;
  const int R = (m + G - 1) / G;
  const int rbeg = J + g * R;
  const int nr = max(0, min(rbeg + R, n) - rbeg);
  const int rw = 2 * w * K;  // LL words per panel row
  extern __shared__ double sm[];
  double *rows = sm;                  // [R][W][K]
  double *prow = rows + R * W * K;    // [W][K] pivot row of this step
  __shared__ PanelShared S;

  auto at = [&](int r, int col) -> double * { return rows + (r * W + col) * K; };

  for (int e = tid; e < nr * w; e += PANEL_THREADS) {
    int r = e / w, col = e % w;
#pragma unroll
    for (int c = 0; c < K; ++c)
      at(r, col)[c] = A.p[c * A.plane + (int64_t)(rbeg + r) * A.ld + J + col];
  }
  __syncthreads();

  // (a) local first-max candidate of column jj; words: idx, |head| (2),
  //     pivot value (2K) -- self-validating, no fence needed
  auto publish_candidate = [&](int jj, unsigned seq) {
    const int j = J + jj;
    double mag = -1.0;
    int row = INT_MAX;
    for (int r = tid; r < nr; r += PANEL_THREADS) {
      int gi = rbeg + r;
      if (gi >= j) {
        double v = fabs(at(r, jj)[0]);
        if (better(v, gi, mag, row)) { mag = v; row = gi; }
      }
    }
    block_argmax(mag, row, S.s_mag, S.s_row);
    u64 *wd = ws.cand_words + ((int64_t)(jj & 1) * G + g) * LU_CAND_WORDS;
    if (tid == 0) {
      S.cand_row = row;
      st_volatile(wd + 0, ll_word((unsigned)row, seq));
      st_volatile(wd + 1, ll_word(lo32(mag), seq));
      st_volatile(wd + 2, ll_word(hi32(mag), seq));
    } else if (tid <= 2 * K && row != INT_MAX) {
      const double v = at(row - rbeg, jj)[(tid - 1) >> 1];
      st_volatile(wd + 2 + tid, ll_word((tid & 1) ? lo32(v) : hi32(v), seq));
    }
  };
  // (b) candidate row and (if owned) row j, once every column is current
  auto publish_rows = [&](int jj, unsigned seq) {
    const int j = J + jj, par = jj & 1;
    const int row = S.cand_row;
    if (row != INT_MAX) {
      u64 *wd = ws.row_words + ((int64_t)par * G + g) * LU_ROW_WORDS;
      const double *src = at(row - rbeg, 0);
      for (int e = tid; e < rw; e += PANEL_THREADS) {
        double v = src[e >> 1];
        st_volatile(wd + e, ll_word((e & 1) ? hi32(v) : lo32(v), seq));
      }
    }
    if (j >= rbeg && j < rbeg + nr) {
      u64 *wd = ws.rowj_words + (int64_t)par * LU_ROW_WORDS;
      const double *src = at(j - rbeg, 0);
      for (int e = tid; e < rw; e += PANEL_THREADS) {
        double v = src[e >> 1];
        st_volatile(wd + e, ll_word((e & 1) ? hi32(v) : lo32(v), seq));
      }
    }
  };
  // poll one LL word until it carries `seq`; return its payload
  auto poll = [](const u64 *p, unsigned seq) -> unsigned {
    u64 v;
    do {
      v = ld_volatile(p);
    } while ((unsigned)v != seq);
    return (unsigned)(v >> 32);
  };

  publish_candidate(0, seq0);
  __syncthreads();
  publish_rows(0, seq0);

  for (int jj = 0; jj < w; ++jj) {
    const int j = J + jj, par = jj & 1;
    const unsigned seq = seq0 + jj;
    // (c) global first max over all candidates: one L2 round trip
    double gm = -1.0;
    int gr = INT_MAX;
    if (tid < G) {
      const u64 *wd = ws.cand_words + ((int64_t)par * G + tid) * LU_CAND_WORDS;
      unsigned a = poll(wd + 0, seq);
      unsigned b = poll(wd + 1, seq);
      unsigned c = poll(wd + 2, seq);
      gr = (int)a;
      gm = __longlong_as_double((long long)(((u64)c << 32) | b));
    }
    block_argmax(gm, gr, S.s_mag, S.s_row);
    const int r = gr;
    const int gw = (r - J) / R;
    const bool own_r = r >= rbeg && r < rbeg + nr;
    const bool own_j = j >= rbeg && j < rbeg + nr;
    const bool last = (j == n - 1);
    // warp 0: pivot value -> recip = div(1, pivot) (every CTA, same bits);
    // other warps: the winner's pivot row (and row j for the new owner of r)
    if (tid < 32) {
      if (!last) {
        const u64 *wd = ws.cand_words + ((int64_t)par * G + gw) * LU_CAND_WORDS;
        unsigned half = tid < 2 * K ? poll(wd + 3 + tid, seq) : 0u;
        double pv[K];
#pragma unroll
        for (int c = 0; c < K; ++c) {
          unsigned l = __shfl_sync(0xffffffffu, half, 2 * c);
          unsigned h = __shfl_sync(0xffffffffu, half, 2 * c + 1);
          pv[c] = __longlong_as_double((long long)(((u64)h << 32) | l));
        }
        if (tid == 0 && pv[0] != 0.0) {
          double one[K], q[K];
#pragma unroll
          for (int c = 0; c < K; ++c) one[c] = c == 0 ? 1.0 : 0.0;
          mc::div<K>(one, pv, q);
#pragma unroll
          for (int c = 0; c < K; ++c) S.recip[c] = q[c];
        }
      }
    } else {
      const u64 *wd = ws.row_words + ((int64_t)par * G + gw) * LU_ROW_WORDS;
      unsigned *pr = reinterpret_cast<unsigned *>(prow);
      for (int e = tid - 32; e < rw; e += PANEL_THREADS - 32)
        pr[e] = poll(wd + e, seq);
      if (r != j && own_r) {
        const u64 *wj = ws.rowj_words + (int64_t)par * LU_ROW_WORDS;
        unsigned *dst = reinterpret_cast<unsigned *>(at(r - rbeg, 0));
        for (int e = tid - 32; e < rw; e += PANEL_THREADS - 32)
          dst[e] = poll(wj + e, seq);
      }
    }
    __syncthreads();
    if (r != j && own_j) {
      double *dst = at(j - rbeg, 0);
      for (int e = tid; e < w * K; e += PANEL_THREADS) dst[e] = prow[e];
    }
    if (g == 0 && tid == 0) swaps[j] = r;
    if (prow[jj * K] == 0.0) {  // singular at step j (uniform decision)
      if (g == 0 && tid == 0) ws.status[0] = j;
      return;
    }
    if (last) break;  // linalg.py:437-438: no reciprocal at the end
    __syncthreads();
    // multipliers m_i = mul(A_ij, recip) for local rows i > j
    for (int rr = tid; rr < nr; rr += PANEL_THREADS) {
      if (rbeg + rr > j) {
        double a[K], rc[K], o[K];
#pragma unroll
        for (int c = 0; c < K; ++c) {
          a[c] = at(rr, jj)[c];
          rc[c] = S.recip[c];
        }
        mc::mul<K>(a, rc, o);
#pragma unroll
        for (int c = 0; c < K; ++c) at(rr, jj)[c] = o[c];
      }
    }
    __syncthreads();
    if (jj + 1 >= w) break;
    // look-ahead: column jj+1 first, then publish its candidate
    for (int rr = tid; rr < nr; rr += PANEL_THREADS) {
      if (rbeg + rr > j) {
        double negm[K], u[K], acc[K];
#pragma unroll
        for (int c = 0; c < K; ++c) {
          negm[c] = -at(rr, jj)[c];
          u[c] = prow[(jj + 1) * K + c];
          acc[c] = at(rr, jj + 1)[c];
        }
        mc::madd<K>(acc, negm, u);
#pragma unroll
        for (int c = 0; c < K; ++c) at(rr, jj + 1)[c] = acc[c];
      }
    }
    __syncthreads();
    publish_candidate(jj + 1, seq + 1);
    // remaining columns of step jj, then the rows of step jj+1
    const int ncol = w - jj - 2;
    for (int e = tid; e < nr * ncol; e += PANEL_THREADS) {
      int rr = e / ncol, cc = jj + 2 + e % ncol;
      if (rbeg + rr > j) {
        double negm[K], u[K], acc[K];
#pragma unroll
        for (int c = 0; c < K; ++c) {
          negm[c] = -at(rr, jj)[c];
          u[c] = prow[cc * K + c];
          acc[c] = at(rr, cc)[c];
        }
        mc::madd<K>(acc, negm, u);
#pragma unroll
        for (int c = 0; c < K; ++c) at(rr, cc)[c] = acc[c];
      }
    }
    __syncthreads();
    publish_rows(jj + 1, seq + 1);
  }

  for (int e = tid; e < nr * w; e += PANEL_THREADS) {
    int r = e / w, col = e % w;
#pragma unroll
    for (int c = 0; c < K; ++c)
      A.p[c * A.plane + (int64_t)(rbeg + r) * A.ld + J + col] = at(r, col)[c];
  }
}

__global__ void lu_begin_kernel(unsigned *epoch, int32_t *status) {
  epoch[0] += 1u;
  status[0] = -1;
}

// Row exchanges of panel [J, J+w), composed once per CTA in shared memory:
// after the swaps, row cur[i] holds what row src[i] held before.  Each
// thread then moves one column (of one plane): all loads, then all stores.
template <int K>
__global__ void __launch_bounds__(256)
laswp_kernel(MatView A, int J, int w, int c0, int c1, int c2, int c3,
             const int32_t *__restrict__ swaps,
             const int32_t *__restrict__ status) {
  if (status[0] >= 0) return;
  __shared__ int cur[2 * LU_MAX_W], src[2 * LU_MAX_W];
  __shared__ int cnt;
  if (threadIdx.x == 0) {
    int m = 0;
    for (int jj = 0; jj < w; ++jj) {
      int a = J + jj, b = swaps[a];
      if (a == b) continue;
      int ia = -1, ib = -1;
      for (int t = 0; t < m; ++t) {
        if (cur[t] == a) ia = t;
        if (cur[t] == b) ib = t;
      }
      if (ia < 0) { cur[m] = a; src[m] = a; ia = m++; }
      if (ib < 0) { cur[m] = b; src[m] = b; ib = m++; }
      int t = src[ia]; src[ia] = src[ib]; src[ib] = t;
    }
    cnt = m;
  }
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

template <typename... KArgs, typename... Args>
cudaError_t launch_coop(void (*kern)(KArgs...), dim3 grid, dim3 block,
                        size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <int K, int W>
size_t panel_smem(int R) {
  return ((size_t)R * W * K + W * K) * sizeof(double);
}

template <int K, int W>
cudaError_t panel_k(int n, MatView A, int J, int w, int32_t *d_swaps,
                    LuWork &ws, cudaStream_t s) {
  const int m = n - J;
  int G = min(ws.G, max(1, (m + 7) / 8));
  const int R = (m + G - 1) / G;
  size_t smem = panel_smem<K, W>(R);
  auto kern = panel_kernel<K, W>;
  static size_t configured = 0;
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(
        kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  return launch_coop(kern, dim3(G), dim3(PANEL_THREADS), smem, s, n, A, J, w,
                     d_swaps, ws);
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
  int k, n, nb;
  const int32_t *swaps;
  bool operator==(const GraphKey &o) const {
    return p == o.p && ld == o.ld && plane == o.plane && k == o.k &&
           n == o.n && nb == o.nb && swaps == o.swaps;
  }
};
struct GraphCache {
  struct Entry {
    GraphKey key;
    cudaGraphExec_t exec;
  };
  std::vector<Entry> entries;
};

cudaError_t enqueue_lu(int k, int n, MatView A, int32_t *d_swaps, int nb,
                       LuWork &ws, cudaStream_t s) {
  cudaError_t e;
  if ((e = lu_begin(ws, s)) != cudaSuccess) return e;
  for (int J = 0; J < n; J += nb) {
    const int w = min(nb, n - J);
    if ((e = lu_panel(k, n, A, J, w, d_swaps, ws, s)) != cudaSuccess) return e;
    if ((e = lu_laswp(k, A, J, w, 0, J, J + w, n, d_swaps, ws.status, s)) !=
        cudaSuccess)
      return e;
    const int rest = n - J - w;
    if (rest > 0) {
      if ((e = lu_trsm(k, sub(A, J, J), sub(A, J, J + w), w, rest, ws.status,
                       s)) != cudaSuccess)
        return e;
      if ((e = lu_update(k, rest, rest, w, sub(A, J + w, J), sub(A, J, J + w),
                         sub(A, J + w, J + w), ws.status, s)) != cudaSuccess)
        return e;
    }
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
  if ((e = cudaMalloc(&epoch, sizeof(unsigned))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&status, sizeof(int32_t))) != cudaSuccess) return e;
  cudaMemset(cand_words, 0, cw);
  cudaMemset(row_words, 0, rwb);
  cudaMemset(rowj_words, 0, jw);
  cudaMemset(epoch, 0, sizeof(unsigned));
  cudaMemset(status, 0xFF, sizeof(int32_t));
  graphs = new GraphCache();
  return cudaDeviceSynchronize();
}

cudaError_t lu_begin(LuWork &ws, cudaStream_t s) {
  lu_begin_kernel<<<1, 1, 0, s>>>(ws.epoch, ws.status);
  return cudaGetLastError();
}

cudaError_t lu_panel(int k, int n, MatView A, int J, int w, int32_t *d_swaps,
                     LuWork &ws, cudaStream_t s) {
  prof_begin(PROF_PANEL, s);
  cudaError_t e = cudaErrorInvalidValue;
  if (w <= 16) {
    switch (k) {
      case 2: e = panel_k<2, 16>(n, A, J, w, d_swaps, ws, s); break;
      case 3: e = panel_k<3, 16>(n, A, J, w, d_swaps, ws, s); break;
      case 4: e = panel_k<4, 16>(n, A, J, w, d_swaps, ws, s); break;
    }
  } else if (w <= 32) {
    switch (k) {
      case 2: e = panel_k<2, 32>(n, A, J, w, d_swaps, ws, s); break;
      case 3: e = panel_k<3, 32>(n, A, J, w, d_swaps, ws, s); break;
      case 4: e = panel_k<4, 32>(n, A, J, w, d_swaps, ws, s); break;
    }
  }
  prof_end(PROF_PANEL, s);
  return e;
}

cudaError_t lu_laswp(int k, MatView A, int J, int w, int c0, int c1, int c2,
                     int c3, const int32_t *d_swaps, const int32_t *status,
                     cudaStream_t s) {
  int ncols = (c1 - c0) + (c3 - c2);
  if (ncols <= 0) return cudaSuccess;
  prof_begin(PROF_LASWP, s);
  int blocks = (ncols * k + 255) / 256;
  switch (k) {
    case 2: laswp_kernel<2><<<blocks, 256, 0, s>>>(A, J, w, c0, c1, c2, c3, d_swaps, status); break;
    case 3: laswp_kernel<3><<<blocks, 256, 0, s>>>(A, J, w, c0, c1, c2, c3, d_swaps, status); break;
    case 4: laswp_kernel<4><<<blocks, 256, 0, s>>>(A, J, w, c0, c1, c2, c3, d_swaps, status); break;
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

cudaError_t lu_factor(int k, int n, MatView A, int32_t *d_swaps, int nb,
                      LuWork &ws, int32_t *sing_step, cudaStream_t s) {
  cudaError_t e;
  if (nb > LU_MAX_W) nb = LU_MAX_W;
  if (nb < 1) nb = 1;
  static const bool no_graph = std::getenv("MPCORE_NO_GRAPH") != nullptr;
  if (prof_enabled() || no_graph) {
    // direct launches (per-kernel event timing needs them)
    if ((e = enqueue_lu(k, n, A, d_swaps, nb, ws, s)) != cudaSuccess) return e;
  } else {
    GraphCache &gc = *static_cast<GraphCache *>(ws.graphs);
    GraphKey key{A.p, A.ld, A.plane, k, n, nb, d_swaps};
    cudaGraphExec_t exec = nullptr;
    for (auto &en : gc.entries)
      if (en.key == key) exec = en.exec;
    if (!exec) {
      cudaGraph_t graph;
      if ((e = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal)) !=
          cudaSuccess)
        return e;
      cudaError_t ee = enqueue_lu(k, n, A, d_swaps, nb, ws, s);
      e = cudaStreamEndCapture(s, &graph);
      if (ee != cudaSuccess) return ee;
      if (e != cudaSuccess) return e;
      e = cudaGraphInstantiate(&exec, graph, 0);
      cudaGraphDestroy(graph);
      if (e != cudaSuccess) return e;
      if (gc.entries.size() >= 16) {
        cudaGraphExecDestroy(gc.entries.front().exec);
        gc.entries.erase(gc.entries.begin());
      }
      gc.entries.push_back({key, exec});
    }
    if ((e = cudaGraphLaunch(exec, s)) != cudaSuccess) return e;
  }
  e = cudaMemcpyAsync(sing_step, ws.status, sizeof(int32_t),
                      cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(s);
}

}  // namespace mpk
