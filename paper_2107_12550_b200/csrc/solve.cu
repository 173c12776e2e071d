// Forward/back substitution with the LU factors, bit-identical to the
// reference's _solve_lanes (linalg.py:496-521):
//   swaps applied in order (501-503)  == gather by the final permutation;
//   forward (unit L), column sweeps j ascending:
//       x_i = add(x_i, mul(-L_ij, x_j))            i > j      (504-509)
//   backward, j descending:
//       x_j = div(x_j, U_jj);  x_i = add(x_i, mul(U_ij, -x_j))   i < j (510-520)
// Each x_i's chain keeps the reference's order (ascending j forward,
// descending j backward).
//
// Parallel structure: rows are cut into blocks of RB; one CTA thread owns
// one row and runs its chain in registers.  A block consumes the columns of
// every earlier block as soon as that block has published its final x
// values (flag per block, epoch-tagged), staging L/U tiles through shared
// memory with coalesced loads, then resolves its own diagonal triangle and
// publishes.  CTAs are persistent (cooperative launch => co-resident) and
// take blocks in dependency order, so the wavefront pipelines across SMs.
#include "internal.h"
#include "mc.cuh"

namespace mpk {

namespace {

constexpr int RB = 128;  // rows per block (= threads per CTA)
constexpr int CB = 16;   // columns per staged tile

__device__ __forceinline__ void wait_flag(const int *flags, int blk,
                                          int epoch) {
  if (threadIdx.x == 0) {
    const volatile int *f = flags + blk;
    while (*f < epoch) {
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ void publish_flag(int *flags, int blk, int epoch) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) atomicExch(flags + blk, epoch);
}

// Stage rows [r0, r0+RB) x cols [c0, c0+cw) of M into Ts[c][r][CB+1].
template <int K>
__device__ __forceinline__ void stage_tile(double *Ts, MatView M, int n,
                                           int r0, int c0, int cw) {
  for (int e = threadIdx.x; e < RB * CB; e += RB) {
    int r = e / CB, cc = e % CB;
    if (r0 + r < n && cc < cw) {
#pragma unroll
      for (int c = 0; c < K; ++c)
        Ts[(c * RB + r) * (CB + 1) + cc] =
            M.p[c * M.plane + (int64_t)(r0 + r) * M.ld + c0 + cc];
    }
  }
}

template <int K>
__device__ __forceinline__ void stage_x(double *xs, const double *x, int n,
                                        int c0, int cw) {
  for (int e = threadIdx.x; e < cw * K; e += RB) {
    int c = e / cw, cc = e % cw;
    xs[c * CB + cc] = __ldcg(x + (int64_t)c * n + c0 + cc);
  }
}

// xw[i] = b[perm[i]]  (the reference's in-order swaps, composed)
template <int K>
__global__ void permute_kernel(int n, const int32_t *__restrict__ perm,
                               const double *__restrict__ b,
                               double *__restrict__ xw) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int src = perm[i];
#pragma unroll
  for (int c = 0; c < K; ++c) xw[(int64_t)c * n + i] = b[(int64_t)c * n + src];
}

template <int K>
__global__ void __launch_bounds__(RB)
forward_kernel(int n, MatView LU, double *__restrict__ x, int *flags,
               int epoch) {
  extern __shared__ double sm[];
  double *Ls = sm;                          // [K][RB][CB+1]
  double *xs = Ls + K * RB * (CB + 1);      // [K][CB]
  double *xown = xs + K * CB;               // [K][RB]
  const int nblk = (n + RB - 1) / RB;
  const int tid = threadIdx.x;
  for (int blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const int r0 = blk * RB, i = r0 + tid;
    const bool live = i < n;
    double acc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) acc[c] = live ? x[(int64_t)c * n + i] : 0.0;
    // columns of earlier blocks, ascending
    int waited = -1;
    for (int c0 = 0; c0 < r0; c0 += CB) {
      const int cb = c0 / RB;
      if (cb != waited) {
        wait_flag(flags, cb, epoch);
        waited = cb;
      }
      stage_tile<K>(Ls, LU, n, r0, c0, CB);
      stage_x<K>(xs, x, n, c0, CB);
      __syncthreads();
      if (live) {
#pragma unroll 1
        for (int jj = 0; jj < CB; ++jj) {
          double l[K], xj[K];
#pragma unroll
          for (int c = 0; c < K; ++c) {
            l[c] = -Ls[(c * RB + tid) * (CB + 1) + jj];
            xj[c] = xs[c * CB + jj];
          }
          mc::madd<K>(acc, l, xj);
        }
      }
      __syncthreads();
    }
    // own triangle: columns r0 .. min(n, r0+RB)-2
    const int rend = min(n, r0 + RB);
    for (int c0 = r0; c0 < rend - 1; c0 += CB) {
      const int cw = min(CB, rend - 1 - c0);
      stage_tile<K>(Ls, LU, n, r0, c0, cw);
      __syncthreads();
      for (int jj = 0; jj < cw; ++jj) {
        const int j = c0 + jj;
        if (i == j) {
#pragma unroll
          for (int c = 0; c < K; ++c) xown[c * RB + tid] = acc[c];
        }
        __syncthreads();
        if (live && i > j) {
          double l[K], xj[K];
#pragma unroll
          for (int c = 0; c < K; ++c) {
            l[c] = -Ls[(c * RB + tid) * (CB + 1) + jj];
            xj[c] = xown[c * RB + (j - r0)];
          }
          mc::madd<K>(acc, l, xj);
        }
      }
      __syncthreads();
    }
    if (live) {
#pragma unroll
      for (int c = 0; c < K; ++c) x[(int64_t)c * n + i] = acc[c];
    }
    publish_flag(flags, blk, epoch);
  }
}

template <int K>
__global__ void __launch_bounds__(RB)
backward_kernel(int n, MatView LU, double *__restrict__ x, int *flags,
                int epoch) {
  extern __shared__ double sm[];
  double *Us = sm;
  double *xs = Us + K * RB * (CB + 1);
  double *xown = xs + K * CB;               // [K][RB]: -x_j of own block
  const int nblk = (n + RB - 1) / RB;
  const int tid = threadIdx.x;
  for (int q = blockIdx.x; q < nblk; q += gridDim.x) {
    const int blk = nblk - 1 - q;
    const int r0 = blk * RB, i = r0 + tid;
    const int rend = min(n, r0 + RB);
    const bool live = i < n;
    double acc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) acc[c] = live ? x[(int64_t)c * n + i] : 0.0;
    // columns of later blocks, descending: tiles [c0, c0+cw) from the right
    int waited = -1;
    for (int cend = n; cend > rend; cend -= CB) {
      const int c0 = max(rend, cend - CB), cw = cend - c0;
      const int cb = (cend - 1) / RB;
      // a tile never straddles blocks: block edges are multiples of RB and
      // tiles are cut back from n; wait on every block the tile touches
      for (int b = c0 / RB; b <= cb; ++b) {
        if (b != waited) {
          wait_flag(flags, b, epoch);
          waited = b;
        }
      }
      stage_tile<K>(Us, LU, n, r0, c0, cw);
      stage_x<K>(xs, x, n, c0, cw);
      __syncthreads();
      if (live) {
#pragma unroll 1
        for (int jj = cw - 1; jj >= 0; --jj) {
          double u[K], nx[K];
#pragma unroll
          for (int c = 0; c < K; ++c) {
            u[c] = Us[(c * RB + tid) * (CB + 1) + jj];
            nx[c] = -xs[c * CB + jj];
          }
          mc::madd<K>(acc, u, nx);
        }
      }
      __syncthreads();
    }
    // own triangle, j descending from rend-1 to r0
    for (int cend = rend; cend > r0; cend -= CB) {
      const int c0 = max(r0, cend - CB), cw = cend - c0;
      stage_tile<K>(Us, LU, n, r0, c0, cw);
      __syncthreads();
      for (int jj = cw - 1; jj >= 0; --jj) {
        const int j = c0 + jj;
        if (i == j) {
          double u[K], qv[K];
#pragma unroll
          for (int c = 0; c < K; ++c) u[c] = Us[(c * RB + tid) * (CB + 1) + jj];
          mc::div<K>(acc, u, qv);
#pragma unroll
          for (int c = 0; c < K; ++c) {
            acc[c] = qv[c];
            xown[c * RB + tid] = -qv[c];
          }
        }
        __syncthreads();
        if (live && i < j) {
          double u[K], nx[K];
#pragma unroll
          for (int c = 0; c < K; ++c) {
            u[c] = Us[(c * RB + tid) * (CB + 1) + jj];
            nx[c] = xown[c * RB + (j - r0)];
          }
          mc::madd<K>(acc, u, nx);
        }
      }
      __syncthreads();
    }
    if (live) {
#pragma unroll
      for (int c = 0; c < K; ++c) x[(int64_t)c * n + i] = acc[c];
    }
    publish_flag(flags, blk, epoch);
  }
}

template <int K>
size_t solve_smem() {
  return ((size_t)K * RB * (CB + 1) + K * CB + K * RB) * sizeof(double);
}

template <typename F>
int coop_grid(F kern, size_t smem, int want) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, RB, smem);
  int cap = per_sm * num_sms();
  if (cap < 1) cap = 1;
  return want < cap ? want : cap;
}

template <int K>
cudaError_t solve_k(int n, MatView LU, const int32_t *perm, const double *b,
                    double *x, SolveWork &sw, cudaStream_t s) {
  const size_t smem = solve_smem<K>();
  auto fk = forward_kernel<K>;
  auto bk = backward_kernel<K>;
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(fk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem)) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(bk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem)) != cudaSuccess)
    return e;
  const int nblk = (n + RB - 1) / RB;
  if ((e = sw.ensure(nblk)) != cudaSuccess) return e;
  permute_kernel<K><<<(n + 255) / 256, 256, 0, s>>>(n, perm, b, x);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  int epoch = sw.next_epoch();
  int G = coop_grid(fk, smem, nblk);
  int *flags = sw.flags;
  void *fargs[] = {(void *)&n, (void *)&LU, (void *)&x, (void *)&flags,
                   (void *)&epoch};
  e = cudaLaunchCooperativeKernel((const void *)fk, dim3(G), dim3(RB), fargs,
                                  smem, s);
  if (e != cudaSuccess) return e;
  int epoch2 = sw.next_epoch();
  G = coop_grid(bk, smem, nblk);
  void *bargs[] = {(void *)&n, (void *)&LU, (void *)&x, (void *)&flags,
                   (void *)&epoch2};
  return cudaLaunchCooperativeKernel((const void *)bk, dim3(G), dim3(RB),
                                     bargs, smem, s);
}

}  // namespace

cudaError_t SolveWork::ensure(int nblk) {
  if (nblk <= cap) return cudaSuccess;
  if (flags) cudaFree(flags);
  flags = nullptr;
  cap = 0;
  epoch = 0;
  cudaError_t e = cudaMalloc(&flags, (size_t)nblk * sizeof(int));
  if (e != cudaSuccess) return e;
  e = cudaMemset(flags, 0, (size_t)nblk * sizeof(int));
  if (e != cudaSuccess) return e;
  cap = nblk;
  return cudaSuccess;
}

cudaError_t lu_solve(int k, int n, MatView LU, const int32_t *d_perm,
                     const double *b, double *x, SolveWork &sw,
                     cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  prof_begin(PROF_SOLVE, s);
  cudaError_t e = cudaErrorInvalidValue;
  switch (k) {
    case 2: e = solve_k<2>(n, LU, d_perm, b, x, sw, s); break;
    case 3: e = solve_k<3>(n, LU, d_perm, b, x, sw, s); break;
    case 4: e = solve_k<4>(n, LU, d_perm, b, x, sw, s); break;
  }
  prof_end(PROF_SOLVE, s);
  return e;
}

}  // namespace mpk
