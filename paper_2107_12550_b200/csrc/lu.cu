// Right-looking blocked LU with partial pivoting, bit-identical to the
// reference's unblocked lane path _lu_lanes (linalg.py:422-449).
//
// Per panel of w columns [J, J+w):
//   1. panel_kernel  (cooperative, one grid barrier per column): for each
//      column j of the panel, pivot = first max of |head| over rows >= j
//      (linalg.py:429), swap of the panel rows, singular check
//      (linalg.py:433-436), recip = div(1, pivot) (439), multipliers
//      m_i = mul(A_ij, recip) (441) and the rank-1 update of the remaining
//      panel columns A_ic = add(A_ic, mul(-m_i, A_jc)) (444-448).
//   2. laswp_kernel: the same row exchanges, in order, on every column
//      outside the panel (the reference swaps full rows, 430-431).
//   3. trsm_kernel: U12 rows J..J+w-1 of the trailing columns, continuing
//      each element's chain with the panel steps it had not seen yet
//      (ascending j, so each element sees exactly the reference's chain).
//   4. lu_update (gemm.cu): A22 <- fold_j add(A22, mul(-L21_ij, U12_jc)).
// Every element of the matrix therefore sees the same sequence of
// add(., mul(-m, u)) operations, in the same order, as in the reference;
// blocking changes only when each link is executed (SURVEY finding 2).
#include <climits>
#include "internal.h"
#include "mc.cuh"

namespace mpk {

namespace {

constexpr int PANEL_THREADS = 256;
constexpr int NWARPS = PANEL_THREADS / 32;

__device__ __forceinline__ void grid_sync(unsigned *bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned *vgen = bar + 1;
    unsigned gen = *vgen;
    __threadfence();
    unsigned arrived = atomicAdd(bar, 1u);
    if (arrived == nblocks - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*vgen == gen) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// (mag, row) ordering: larger magnitude wins; ties go to the smaller row
// (np.argmax returns the first maximum).
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
    if (lane == 0) { s_mag[0] = mag; s_row[0] = row; }
  }
  __syncthreads();
  mag = s_mag[0];
  row = s_row[0];
  __syncthreads();
}

// Panel factorisation over rows [J, n), columns [J, J+w).  CTA g keeps rows
// [J + g*R, J + (g+1)*R) of the panel resident in shared memory.
template <int K, int W>
__global__ void __launch_bounds__(PANEL_THREADS, 1)
panel_kernel(int n, MatView A, int J, int w, int32_t *__restrict__ swaps,
             LuWork ws) {
  const int G = gridDim.x, g = blockIdx.x, tid = threadIdx.x;
  if (ws.status[0] >= 0) return;
  const int m = n - J;
  const int R = (m + G - 1) / G;
  const int rbeg = J + g * R;
  const int nr = max(0, min(rbeg + R, n) - rbeg);
  extern __shared__ double sm[];
  double *rows = sm;                 // [R][W][K]
  double *prow = rows + R * W * K;   // [W][K]
  double *recip = prow + W * K;      // [K]
  __shared__ double s_mag[NWARPS];
  __shared__ int s_row[NWARPS];

  for (int e = tid; e < nr * w; e += PANEL_THREADS) {
    int r = e / w, col = e % w;
#pragma unroll
    for (int c = 0; c < K; ++c)
      rows[(r * W + col) * K + c] =
          A.p[c * A.plane + (int64_t)(rbeg + r) * A.ld + J + col];
  }
  __syncthreads();

  for (int jj = 0; jj < w; ++jj) {
    const int j = J + jj, par = jj & 1;
    double mag = -1.0;
    int row = INT_MAX;
    for (int r = tid; r < nr; r += PANEL_THREADS) {
      int gi = rbeg + r;
      if (gi >= j) {
        double v = fabs(rows[(r * W + jj) * K]);
        if (better(v, gi, mag, row)) { mag = v; row = gi; }
      }
    }
    block_argmax(mag, row, s_mag, s_row);
    // publish this CTA's candidate row (and row j if owned)
    double *cand = ws.cand_rows + ((int64_t)par * G + g) * (W * K);
    if (row != INT_MAX) {
      int r = row - rbeg;
      for (int e = tid; e < w * K; e += PANEL_THREADS)
        cand[e] = rows[r * W * K + e];
    }
    if (j >= rbeg && j < rbeg + nr) {
      int r = j - rbeg;
      double *rj = ws.rowj + (int64_t)par * (W * K);
      for (int e = tid; e < w * K; e += PANEL_THREADS) rj[e] = rows[r * W * K + e];
    }
    if (tid == 0) {
      ws.cand_mag[par * G + g] = mag;
      ws.cand_idx[par * G + g] = row;
    }
    grid_sync(ws.bar, G);
    // global first-max over the published candidates
    double gm = -1.0;
    int gr = INT_MAX, gw = 0;
    for (int t = tid; t < G; t += PANEL_THREADS) {
      double cm = __ldcg(ws.cand_mag + par * G + t);
      int cr = __ldcg(ws.cand_idx + par * G + t);
      if (better(cm, cr, gm, gr)) { gm = cm; gr = cr; }
    }
    block_argmax(gm, gr, s_mag, s_row);
    const int r = gr;
    // the winner CTA is the owner of row r
    gw = (r - J) / R;
    const double *wrow = ws.cand_rows + ((int64_t)par * G + gw) * (W * K);
    for (int e = tid; e < w * K; e += PANEL_THREADS) prow[e] = __ldcg(wrow + e);
    __syncthreads();
    if (r != j) {
      if (r >= rbeg && r < rbeg + nr) {
        const double *rj = ws.rowj + (int64_t)par * (W * K);
        int lr = r - rbeg;
        for (int e = tid; e < w * K; e += PANEL_THREADS)
          rows[lr * W * K + e] = __ldcg(rj + e);
      }
      if (j >= rbeg && j < rbeg + nr) {
        int lr = j - rbeg;
        for (int e = tid; e < w * K; e += PANEL_THREADS)
          rows[lr * W * K + e] = prow[e];
      }
    }
    if (g == 0 && tid == 0) swaps[j] = r;
    if (prow[jj * K] == 0.0) {  // singular at step j (uniform decision)
      if (g == 0 && tid == 0) ws.status[0] = j;
      return;
    }
    if (j == n - 1) break;  // linalg.py:437-438: no reciprocal at the end
    if (tid == 0) {
      double one[K], pv[K], q[K];
#pragma unroll
      for (int c = 0; c < K; ++c) {
        one[c] = c == 0 ? 1.0 : 0.0;
        pv[c] = prow[jj * K + c];
      }
      mc::div<K>(one, pv, q);
#pragma unroll
      for (int c = 0; c < K; ++c) recip[c] = q[c];
    }
    __syncthreads();
    // multipliers m_i = mul(A_ij, recip)
    for (int rr = tid; rr < nr; rr += PANEL_THREADS) {
      if (rbeg + rr > j) {
        double a[K], rc[K], o[K];
#pragma unroll
        for (int c = 0; c < K; ++c) {
          a[c] = rows[(rr * W + jj) * K + c];
          rc[c] = recip[c];
        }
        mc::mul<K>(a, rc, o);
#pragma unroll
        for (int c = 0; c < K; ++c) rows[(rr * W + jj) * K + c] = o[c];
      }
    }
    __syncthreads();
    // rank-1 update of the remaining panel columns
    const int ncol = w - jj - 1;
    for (int e = tid; e < nr * ncol; e += PANEL_THREADS) {
      int rr = e / ncol, cc = jj + 1 + e % ncol;
      if (rbeg + rr > j) {
        double negm[K], u[K], acc[K];
#pragma unroll
        for (int c = 0; c < K; ++c) {
          negm[c] = -rows[(rr * W + jj) * K + c];
          u[c] = prow[cc * K + c];
          acc[c] = rows[(rr * W + cc) * K + c];
        }
        mc::madd<K>(acc, negm, u);
#pragma unroll
        for (int c = 0; c < K; ++c) rows[(rr * W + cc) * K + c] = acc[c];
      }
    }
    __syncthreads();
  }

  for (int e = tid; e < nr * w; e += PANEL_THREADS) {
    int r = e / w, col = e % w;
#pragma unroll
    for (int c = 0; c < K; ++c)
      A.p[c * A.plane + (int64_t)(rbeg + r) * A.ld + J + col] =
          rows[(r * W + col) * K + c];
  }
}

// Row exchanges of panel [J, J+w) applied in order to columns [c0, c1) and
// [c2, c3) (everything outside the panel).  One thread per (column, plane).
template <int K>
__global__ void laswp_kernel(MatView A, int J, int w, int c0, int c1, int c2,
                             int c3, const int32_t *__restrict__ swaps,
                             const int32_t *__restrict__ status) {
  if (status[0] >= 0) return;
  const int n1 = c1 - c0, n2 = c3 - c2, ncols = n1 + n2;
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ncols * K) return;
  int c = t / ncols, q = t % ncols;
  int col = q < n1 ? c0 + q : c2 + (q - n1);
  double *p = A.p + c * A.plane + col;
  for (int jj = 0; jj < w; ++jj) {
    int j = J + jj, r = swaps[j];
    if (r != j) {
      double a = p[(int64_t)j * A.ld], b = p[(int64_t)r * A.ld];
      p[(int64_t)j * A.ld] = b;
      p[(int64_t)r * A.ld] = a;
    }
  }
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

template <int K, int W>
size_t panel_smem(int R) {
  return ((size_t)R * W * K + W * K + K) * sizeof(double);
}

template <int K, int W>
cudaError_t panel_k(int n, MatView A, int J, int w, int32_t *d_swaps,
                    LuWork &ws, cudaStream_t s) {
  const int m = n - J;
  int G = min(ws.G, max(1, (m + 7) / 8));
  const int R = (m + G - 1) / G;
  size_t smem = panel_smem<K, W>(R);
  auto kern = panel_kernel<K, W>;
  cudaError_t e = cudaFuncSetAttribute(
      kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  LuWork wcopy = ws;
  void *args[] = {(void *)&n, (void *)&A, (void *)&J, (void *)&w,
                  (void *)&d_swaps, (void *)&wcopy};
  return cudaLaunchCooperativeKernel((const void *)kern, dim3(G),
                                     dim3(PANEL_THREADS), args, smem, s);
}

template <int K, int W>
cudaError_t trsm_k(MatView L11, MatView U12, int w, int ncols,
                   const int32_t *status, cudaStream_t s) {
  constexpr int TC = 256 / W;
  trsm_kernel<K, W, TC><<<(ncols + TC - 1) / TC, W * TC, 0, s>>>(
      L11, U12, w, ncols, status);
  return cudaGetLastError();
}

}  // namespace

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

cudaError_t lu_laswp(int k, int n, MatView A, int J, int w, int c0, int c1,
                     const int32_t *d_swaps, const int32_t *status,
                     cudaStream_t s) {
  // columns [0, J) and [J+w, n)
  (void)c0; (void)c1;
  int ncols = J + (n - J - w);
  if (ncols <= 0) return cudaSuccess;
  prof_begin(PROF_LASWP, s);
  int total = ncols * k;
  int blocks = (total + 255) / 256;
  switch (k) {
    case 2: laswp_kernel<2><<<blocks, 256, 0, s>>>(A, J, w, 0, J, J + w, n, d_swaps, status); break;
    case 3: laswp_kernel<3><<<blocks, 256, 0, s>>>(A, J, w, 0, J, J + w, n, d_swaps, status); break;
    case 4: laswp_kernel<4><<<blocks, 256, 0, s>>>(A, J, w, 0, J, J + w, n, d_swaps, status); break;
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

static MatView sub(MatView A, int i, int j) {
  MatView v = A;
  v.p = A.p + (int64_t)i * A.ld + j;
  return v;
}

cudaError_t lu_factor(int k, int n, MatView A, int32_t *d_swaps, int nb,
                      LuWork &ws, int32_t *sing_step, cudaStream_t s) {
  cudaError_t e;
  if (nb > 32) nb = 32;
  if (nb < 1) nb = 1;
  e = cudaMemsetAsync(ws.status, 0xFF, sizeof(int32_t), s);  // -1
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(ws.bar, 0, 2 * sizeof(unsigned), s);
  if (e != cudaSuccess) return e;
  for (int J = 0; J < n; J += nb) {
    const int w = min(nb, n - J);
    if ((e = lu_panel(k, n, A, J, w, d_swaps, ws, s)) != cudaSuccess) return e;
    if ((e = lu_laswp(k, n, A, J, w, 0, 0, d_swaps, ws.status, s)) !=
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
  e = cudaMemcpyAsync(sing_step, ws.status, sizeof(int32_t),
                      cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(s);
}

}  // namespace mpk
