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
// one row and runs its chain in registers.  Columns are consumed in tiles of
// CB: a tile of x becomes readable as soon as the CB rows it covers are
// final (per-tile flag, epoch-tagged), so the next block starts on a tile
// while the producing block is still resolving later rows of its diagonal
// triangle.  L/U tiles are staged through shared memory with coalesced,
// double-buffered cp.async loads.  CTAs are persistent (cooperative launch
// => co-resident) and take blocks in dependency order.
#include "internal.h"
#include "mc.cuh"

namespace mpk {

namespace {

constexpr int RB = 128;  // rows per block (= threads per CTA)
constexpr int CB = 16;   // columns per staged tile (= rows per flag)

__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s),
               "l"(gmem));
}
__device__ __forceinline__ void cp_commit() {
  asm volatile("cp.async.commit_group;\n" ::);
}
template <int N> __device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void wait_flag(const int *flags, int t,
                                          int epoch) {
  if (threadIdx.x == 0) {
    const volatile int *f = flags + t;
    while (*f < epoch) __nanosleep(20);
    __threadfence();
  }
  __syncthreads();
}

// the x rows of tile t are final: make them visible, then raise its flag
__device__ __forceinline__ void publish(int *flags, int t, int epoch) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) atomicExch(flags + t, epoch);
}

// Stage rows [r0, r0+RB) x cols [c0, c0+cw) of M into Ts[c][r][CB+1]
// (asynchronous; caller commits / waits)
template <int K>
__device__ __forceinline__ void stage_tile(double *Ts, MatView M, int n,
                                           int r0, int c0, int cw) {
  for (int e = threadIdx.x; e < RB * CB; e += RB) {
    int r = e / CB, cc = e % CB;
    if (r0 + r < n && cc < cw) {
#pragma unroll
      for (int c = 0; c < K; ++c)
        cp_async8(Ts + (c * RB + r) * (CB + 1) + cc,
                  M.p + c * M.plane + (int64_t)(r0 + r) * M.ld + c0 + cc);
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

constexpr int TILE_ELEMS = RB * (CB + 1);

template <int K>
__global__ void __launch_bounds__(RB)
forward_kernel(int n, MatView LU, double *__restrict__ x, int *flags,
               int epoch) {
  extern __shared__ double sm[];
  double *Ls0 = sm;                          // [2][K][RB][CB+1]
  double *xs = Ls0 + 2 * K * TILE_ELEMS;     // [K][CB]
  double *xown = xs + K * CB;                // [K][RB]
  const int nblk = (n + RB - 1) / RB;
  const int tid = threadIdx.x;
  for (int blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const int r0 = blk * RB, i = r0 + tid;
    const bool live = i < n;
    const int rend = min(n, r0 + RB);
    double acc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) acc[c] = live ? x[(int64_t)c * n + i] : 0.0;
    // off-diagonal tiles, ascending; L tiles prefetched one ahead
    const int ntile = r0 / CB;
    if (ntile > 0) {
      stage_tile<K>(Ls0, LU, n, r0, 0, CB);
      cp_commit();
    }
    for (int t = 0; t < ntile; ++t) {
      double *Ls = Ls0 + (t & 1) * K * TILE_ELEMS;
      if (t + 1 < ntile) {
        stage_tile<K>(Ls0 + ((t + 1) & 1) * K * TILE_ELEMS, LU, n, r0,
                      (t + 1) * CB, CB);
        cp_commit();
      }
      wait_flag(flags, t, epoch);
      stage_x<K>(xs, x, n, t * CB, CB);
      if (t + 1 < ntile) cp_wait<1>(); else cp_wait<0>();
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
    // diagonal triangle, tile by tile; each finished tile is published
    for (int c0 = r0; c0 < rend; c0 += CB) {
      const int cw = min(CB, rend - c0);
      stage_tile<K>(Ls0, LU, n, r0, c0, cw);
      cp_commit();
      cp_wait<0>();
      __syncthreads();
      for (int jj = 0; jj < cw; ++jj) {
        const int j = c0 + jj;
        if (i == j) {
#pragma unroll
          for (int c = 0; c < K; ++c) {
            xown[c * RB + tid] = acc[c];
            x[(int64_t)c * n + i] = acc[c];   // final
          }
        }
        __syncthreads();
        if (live && i > j) {
          double l[K], xj[K];
#pragma unroll
          for (int c = 0; c < K; ++c) {
            l[c] = -Ls0[(c * RB + tid) * (CB + 1) + jj];
            xj[c] = xown[c * RB + (j - r0)];
          }
          mc::madd<K>(acc, l, xj);
        }
      }
      publish(flags, c0 / CB, epoch);
    }
  }
}

template <int K>
__global__ void __launch_bounds__(RB)
backward_kernel(int n, MatView LU, double *__restrict__ x, int *flags,
                int epoch) {
  extern __shared__ double sm[];
  double *Us0 = sm;
  double *xs = Us0 + 2 * K * TILE_ELEMS;
  double *xown = xs + K * CB;                // [K][RB]: -x_j of own block
  const int nblk = (n + RB - 1) / RB;
  const int ntile_all = (n + CB - 1) / CB;
  const int tid = threadIdx.x;
  for (int q = blockIdx.x; q < nblk; q += gridDim.x) {
    const int blk = nblk - 1 - q;
    const int r0 = blk * RB, i = r0 + tid;
    const int rend = min(n, r0 + RB);
    const bool live = i < n;
    double acc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) acc[c] = live ? x[(int64_t)c * n + i] : 0.0;
    // off-diagonal tiles of later rows, descending (tile index from the top
    // tile of the matrix down to the first tile after this block)
    const int t_lo = (rend + CB - 1) / CB;     // first tile after the block
    const int nt = ntile_all - t_lo;
    auto tile_c0 = [&](int q2) { return (ntile_all - 1 - q2) * CB; };
    if (nt > 0) {
      int c0 = tile_c0(0);
      stage_tile<K>(Us0, LU, n, r0, c0, min(CB, n - c0));
      cp_commit();
    }
    for (int q2 = 0; q2 < nt; ++q2) {
      const int c0 = tile_c0(q2), cw = min(CB, n - c0);
      double *Us = Us0 + (q2 & 1) * K * TILE_ELEMS;
      if (q2 + 1 < nt) {
        int c1 = tile_c0(q2 + 1);
        stage_tile<K>(Us0 + ((q2 + 1) & 1) * K * TILE_ELEMS, LU, n, r0, c1,
                      min(CB, n - c1));
        cp_commit();
      }
      wait_flag(flags, c0 / CB, epoch);
      stage_x<K>(xs, x, n, c0, cw);
      if (q2 + 1 < nt) cp_wait<1>(); else cp_wait<0>();
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
    // diagonal triangle, tiles from the bottom; j descending
    const int last_tile = (rend - 1) / CB;
    for (int tt = last_tile; tt >= r0 / CB; --tt) {
      const int c0 = tt * CB, cw = min(CB, rend - c0);
      stage_tile<K>(Us0, LU, n, r0, c0, cw);
      cp_commit();
      cp_wait<0>();
      __syncthreads();
      for (int jj = cw - 1; jj >= 0; --jj) {
        const int j = c0 + jj;
        if (i == j) {
          double u[K], qv[K];
#pragma unroll
          for (int c = 0; c < K; ++c) u[c] = Us0[(c * RB + tid) * (CB + 1) + jj];
          mc::div<K>(acc, u, qv);
#pragma unroll
          for (int c = 0; c < K; ++c) {
            acc[c] = qv[c];
            xown[c * RB + tid] = -qv[c];
            x[(int64_t)c * n + i] = qv[c];    // final
          }
        }
        __syncthreads();
        if (live && i < j) {
          double u[K], nx[K];
#pragma unroll
          for (int c = 0; c < K; ++c) {
            u[c] = Us0[(c * RB + tid) * (CB + 1) + jj];
            nx[c] = xown[c * RB + (j - r0)];
          }
          mc::madd<K>(acc, u, nx);
        }
      }
      publish(flags, tt, epoch);
    }
  }
}

template <int K>
size_t solve_smem() {
  return ((size_t)2 * K * TILE_ELEMS + K * CB + K * RB) * sizeof(double);
}

template <typename F>
int coop_grid(F kern, size_t smem, int want) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, RB, smem);
  int cap = per_sm * num_sms();
  if (cap < 1) cap = 1;
  return want < cap ? want : cap;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_coop(void (*kern)(KArgs...), int grid, size_t smem,
                        cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(RB);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <int K>
cudaError_t solve_k(int n, MatView LU, const int32_t *perm, const double *b,
                    double *x, SolveWork &sw, cudaStream_t s) {
  const size_t smem = solve_smem<K>();
  auto fk = forward_kernel<K>;
  auto bk = backward_kernel<K>;
  static bool configured = false;
  cudaError_t e;
  if (!configured) {
    if ((e = cudaFuncSetAttribute(
             fk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) !=
        cudaSuccess)
      return e;
    if ((e = cudaFuncSetAttribute(
             bk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) !=
        cudaSuccess)
      return e;
    configured = true;
  }
  const int nblk = (n + RB - 1) / RB;
  const int ntile = (n + CB - 1) / CB;
  if ((e = sw.ensure(ntile)) != cudaSuccess) return e;
  permute_kernel<K><<<(n + 255) / 256, 256, 0, s>>>(n, perm, b, x);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  int epoch = sw.next_epoch();
  int *flags = sw.flags;
  e = launch_coop(fk, coop_grid(fk, smem, nblk), smem, s, n, LU, x, flags,
                  epoch);
  if (e != cudaSuccess) return e;
  int epoch2 = sw.next_epoch();
  return launch_coop(bk, coop_grid(bk, smem, nblk), smem, s, n, LU, x, flags,
                     epoch2);
}

}  // namespace

cudaError_t SolveWork::ensure(int nflags) {
  if (nflags <= cap) return cudaSuccess;
  if (flags) cudaFree(flags);
  flags = nullptr;
  cap = 0;
  epoch = 0;
  cudaError_t e = cudaMalloc(&flags, (size_t)nflags * sizeof(int));
  if (e != cudaSuccess) return e;
  e = cudaMemset(flags, 0, (size_t)nflags * sizeof(int));
  if (e != cudaSuccess) return e;
  cap = nflags;
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
