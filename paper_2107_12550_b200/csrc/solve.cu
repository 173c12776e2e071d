// Forward/back substitution with the LU factors, bit-identical to the
// reference's _solve_lanes (linalg.py:496-521):
//   swaps applied in order (501-503);
//   forward (unit L), column sweeps j ascending:
//       x_i = add(x_i, mul(-L_ij, x_j))            i > j      (504-509)
//   backward, j descending:
//       x_j = div(x_j, U_jj);  x_i = add(x_i, mul(U_ij, -x_j))   i < j (510-520)
// Each x_i's chain keeps the reference's order (ascending j forward,
// descending j backward); threads only parallelise over i.
#include "internal.h"
#include "mc.cuh"

namespace mpk {

namespace {

constexpr int SOLVE_THREADS = 1024;

template <int K, bool SMEM>
__global__ void __launch_bounds__(SOLVE_THREADS, 1)
solve_kernel(int n, MatView LU, const int32_t *__restrict__ swaps,
             double *__restrict__ xg) {
  extern __shared__ double sx[];
  double *x = SMEM ? sx : xg;  // planar [K][n]
  const int tid = threadIdx.x;
  if (SMEM) {
    for (int i = tid; i < n; i += SOLVE_THREADS)
#pragma unroll
      for (int c = 0; c < K; ++c) x[c * n + i] = xg[(int64_t)c * n + i];
  }
  __syncthreads();
  if (tid == 0) {
    for (int j = 0; j < n; ++j) {
      int r = swaps[j];
      if (r != j) {
#pragma unroll
        for (int c = 0; c < K; ++c) {
          double t = x[c * n + j];
          x[c * n + j] = x[c * n + r];
          x[c * n + r] = t;
        }
      }
    }
  }
  __syncthreads();
  // forward
  for (int j = 0; j + 1 < n; ++j) {
    double xj[K];
#pragma unroll
    for (int c = 0; c < K; ++c) xj[c] = x[c * n + j];
    for (int i = j + 1 + tid; i < n; i += SOLVE_THREADS) {
      double l[K], acc[K];
#pragma unroll
      for (int c = 0; c < K; ++c) {
        l[c] = -LU.p[c * LU.plane + (int64_t)i * LU.ld + j];
        acc[c] = x[c * n + i];
      }
      mc::madd<K>(acc, l, xj);
#pragma unroll
      for (int c = 0; c < K; ++c) x[c * n + i] = acc[c];
    }
    __syncthreads();
  }
  // backward
  __shared__ double sxj[K];
  for (int j = n - 1; j >= 0; --j) {
    if (tid == 0) {
      double a[K], u[K], q[K];
#pragma unroll
      for (int c = 0; c < K; ++c) {
        a[c] = x[c * n + j];
        u[c] = LU.p[c * LU.plane + (int64_t)j * LU.ld + j];
      }
      mc::div<K>(a, u, q);
#pragma unroll
      for (int c = 0; c < K; ++c) {
        x[c * n + j] = q[c];
        sxj[c] = -q[c];
      }
    }
    __syncthreads();
    if (j == 0) break;
    double nx[K];
#pragma unroll
    for (int c = 0; c < K; ++c) nx[c] = sxj[c];
    for (int i = tid; i < j; i += SOLVE_THREADS) {
      double u[K], acc[K];
#pragma unroll
      for (int c = 0; c < K; ++c) {
        u[c] = LU.p[c * LU.plane + (int64_t)i * LU.ld + j];
        acc[c] = x[c * n + i];
      }
      mc::madd<K>(acc, u, nx);
#pragma unroll
      for (int c = 0; c < K; ++c) x[c * n + i] = acc[c];
    }
    __syncthreads();
  }
  if (SMEM) {
    for (int i = tid; i < n; i += SOLVE_THREADS)
#pragma unroll
      for (int c = 0; c < K; ++c) xg[(int64_t)c * n + i] = x[c * n + i];
  }
}

template <int K>
cudaError_t solve_k(int n, MatView LU, const int32_t *swaps, double *x,
                    cudaStream_t s) {
  size_t bytes = (size_t)n * K * sizeof(double);
  if (bytes <= 200 * 1024) {
    auto kern = solve_kernel<K, true>;
    cudaError_t e = cudaFuncSetAttribute(
        kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    kern<<<1, SOLVE_THREADS, bytes, s>>>(n, LU, swaps, x);
  } else {
    solve_kernel<K, false><<<1, SOLVE_THREADS, 0, s>>>(n, LU, swaps, x);
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t lu_solve(int k, int n, MatView LU, const int32_t *d_swaps,
                     double *x, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  prof_begin(PROF_SOLVE, s);
  cudaError_t e = cudaErrorInvalidValue;
  switch (k) {
    case 2: e = solve_k<2>(n, LU, d_swaps, x, s); break;
    case 3: e = solve_k<3>(n, LU, d_swaps, x, s); break;
    case 4: e = solve_k<4>(n, LU, d_swaps, x, s); break;
  }
  prof_end(PROF_SOLVE, s);
  return e;
}

}  // namespace mpk
