// Forward/back substitution with the LU factors, bit-identical to the
// reference's _solve_lanes (linalg.py:496-521):
//   swaps applied in order (501-503)  == gather by the final permutation;
//   forward (unit L), column sweeps j ascending:
//       x_i = add(x_i, mul(-L_ij, x_j))            i > j      (504-509)
//   backward, j descending:
//       x_j = div(x_j, U_jj);  x_i = add(x_i, mul(U_ij, -x_j))   i < j (510-520)
// Every x_i's chain keeps the reference's order (ascending j forward,
// descending j backward); madd = add(acc, mul(a, b)), so a product may be
// formed by another thread ahead of time and added in order.
//
// Parallel structure.  Rows are cut into blocks of 32; a CTA (persistent,
// cooperative => co-resident) takes blocks in dependency order.  In a CTA:
//   warp 0, the owner: lane = row, the row's accumulator in registers.  It
//     adds the products of every completed source block in order, runs the
//     critical source block (the neighbour still being solved) with full
//     madds as its x values appear, then the diagonal triangle with the
//     x_j broadcast by shuffles (no CTA barrier on the per-row chain);
//   warps 1-3, producers: for each completed source block, products
//     P[r][c] = mul(-L_rc, x_c) (coalesced: lane = column) into a
//     double-buffered shared-memory ring (named barriers FULL/EMPTY), and
//     the L tiles of the critical source block and of the diagonal.
// Products cost ~60 % of a madd (TD: 133 of 214 FP64 instructions), so the
// owner's per-row chain is only the adds.  Every final x_i is published as
// 2K self-validating 8-byte words (payload | sequence), so a consumer needs
// no flag, no fence and a single L2 round trip per chunk of rows.
#include <cstdlib>

#include "internal.h"
#include "mc.cuh"

namespace mpk {

namespace {

constexpr int SB = 32;         // rows per block (owner lanes)
constexpr int NPW = 3;         // producer warps
constexpr int ST = 32 * (1 + NPW);
constexpr int PS = SB + 1;     // padded row stride of the shared tiles
constexpr int NSLOT = 2;
constexpr int BAR_FULL = 1, BAR_EMPTY = 3, BAR_STAGED = 5;

using u64 = unsigned long long;

__device__ __forceinline__ void st_word(u64 *p, u64 v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v)
               : "memory");
}
__device__ __forceinline__ u64 ld_word(const u64 *p) {
  u64 v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ void nb_sync(int id) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(ST) : "memory");
}
__device__ __forceinline__ void nb_arrive(int id) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(ST) : "memory");
}

// x_i (K doubles) -> words [2c][i] = lo, [2c+1][i] = hi, each | seq
template <int K>
__device__ __forceinline__ void publish_x(u64 *W, int64_t n, int i,
                                          const double *v, unsigned seq) {
#pragma unroll
  for (int c = 0; c < K; ++c) {
    const u64 b = (u64)__double_as_longlong(v[c]);
    st_word(W + (2 * c) * n + i, (b << 32) | seq);
    st_word(W + (2 * c + 1) * n + i, (b & 0xffffffff00000000ull) | seq);
  }
}
// publish_x under a predicate, without a branch (keeps the per-row chain of
// the triangle free of divergent blocks)
template <int K>
__device__ __forceinline__ void publish_x_if(bool p, u64 *W, int64_t n, int i,
                                             const double *v, unsigned seq) {
#pragma unroll
  for (int c = 0; c < K; ++c) {
    const u64 b = (u64)__double_as_longlong(v[c]);
    const u64 lo = (b << 32) | seq, hi = (b & 0xffffffff00000000ull) | seq;
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %0, 0;\n\t"
        "@q st.relaxed.gpu.global.u64 [%1], %2;\n\t"
        "@q st.relaxed.gpu.global.u64 [%3], %4;\n\t}" ::"r"((unsigned)p),
        "l"(W + (2 * c) * n + i), "l"(lo), "l"(W + (2 * c + 1) * n + i),
        "l"(hi)
        : "memory");
  }
}
// poll row i's words until all carry seq; returns the K doubles
template <int K>
__device__ __forceinline__ void fetch_x(const u64 *W, int64_t n, int i,
                                        unsigned seq, double *v) {
  u64 w[2 * K];
  for (;;) {
#pragma unroll
    for (int x = 0; x < 2 * K; ++x) w[x] = ld_word(W + x * n + i);
    bool ok = true;
#pragma unroll
    for (int x = 0; x < 2 * K; ++x) ok &= (unsigned)w[x] == seq;
    if (ok) break;
    __nanosleep(16);
  }
#pragma unroll
  for (int c = 0; c < K; ++c)
    v[c] = __longlong_as_double(
        (long long)((w[2 * c + 1] & 0xffffffff00000000ull) | (w[2 * c] >> 32)));
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

constexpr int TILE = SB * PS;  // one plane of a shared tile

// One kernel for both sweeps (BACK = false: forward with unit L).
template <int K, bool BACK>
__global__ void __launch_bounds__(ST, 1)
sweep_kernel(int n, MatView LU, double *__restrict__ x, u64 *__restrict__ W,
             unsigned seq, u64 *trace) {
  extern __shared__ double sm[];
  double *P = sm;                        // [NSLOT][K][SB][PS] products
  double *Lc = P + NSLOT * K * TILE;     // [K][SB][PS] critical source tile
  double *Ld = Lc + K * TILE;            // [K][SB][PS] diagonal tile
  const int nblk = (n + SB - 1) / SB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t N = n;

  for (int q = blockIdx.x; q < nblk; q += gridDim.x) {
    const int blk = BACK ? nblk - 1 - q : q;
    const int r0 = blk * SB;
    const int rows = min(SB, n - r0);
    // completed source blocks, in fold order, and the critical one
    const int crit = BACK ? blk + 1 : blk - 1;
    const bool has_crit = crit >= 0 && crit < nblk;
    const int nfull = BACK ? max(0, nblk - blk - 2) : max(0, blk - 1);
    auto src_of = [&](int t) { return BACK ? nblk - 1 - t : t; };
    __syncthreads();  // the previous block's tiles are no longer read

    if (warp > 0) {
      // ============================================================ producers
      const int pw = warp - 1;
      // stage the critical source tile and the diagonal tile (lane = column)
      for (int r = pw; r < rows; r += NPW) {
        const int64_t row = (int64_t)(r0 + r) * LU.ld;
        if (has_crit) {
          const int c = crit * SB + lane;
          if (c < n) {
#pragma unroll
            for (int k = 0; k < K; ++k)
              Lc[k * TILE + r * PS + lane] = LU.p[k * LU.plane + row + c];
          }
        }
        if (r0 + lane < n) {
#pragma unroll
          for (int k = 0; k < K; ++k)
            Ld[k * TILE + r * PS + lane] = LU.p[k * LU.plane + row + r0 + lane];
          // the row's division hint RN(1/U_rr) in the tile's pad column
          if (BACK && lane == r)
            Ld[r * PS + SB] = mc::recip_hint(LU.p[row + r0 + lane]);
        }
      }
      nb_arrive(BAR_STAGED);
      for (int t = 0; t < nfull; ++t) {
        const int s = t & 1;
        const int sb = src_of(t), c = sb * SB + lane;
        if (t >= NSLOT) nb_sync(BAR_EMPTY + s);
        if (c < n) {
          // the tile's L/U values do not depend on x: load them first, so
          // their latency overlaps the wait for the source block's x
          constexpr int RPW = (SB + NPW - 1) / NPW;
          double lv[RPW][K];
#pragma unroll
          for (int q = 0; q < RPW; ++q) {
            const int r = pw + q * NPW;
#pragma unroll
            for (int k = 0; k < K; ++k) {
              const double v =
                  r < rows ? LU.p[k * LU.plane + (int64_t)(r0 + r) * LU.ld + c]
                           : 0.0;
              lv[q][k] = BACK ? v : -v;
            }
          }
          double xv[K];
          fetch_x<K>(W, N, c, seq, xv);
          if (BACK) {
#pragma unroll
            for (int k = 0; k < K; ++k) xv[k] = -xv[k];
          }
          double *Ps = P + s * K * TILE;
#pragma unroll
          for (int q = 0; q < RPW; ++q) {
            const int r = pw + q * NPW;
            if (r < rows) {
              double o[K];
              mc::mul<K>(lv[q], xv, o);  // fwd mul(-L, x); back mul(U, -x)
#pragma unroll
              for (int k = 0; k < K; ++k) Ps[k * TILE + r * PS + lane] = o[k];
            }
          }
        }
        nb_arrive(BAR_FULL + s);
      }
    } else {
      // ================================================================ owner
      auto mark = [&](int slot) {
        if (trace && lane == 0) {
          u64 t;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
          trace[(int64_t)blk * 8 + slot] = t;
        }
      };
      mark(0);
      const int i = r0 + lane;
      const bool live = lane < rows;
      double acc[K];
#pragma unroll
      for (int k = 0; k < K; ++k) acc[k] = live ? x[k * N + i] : 0.0;
      for (int t = 0; t < nfull; ++t) {
        const int s = t & 1;
        const int sb = src_of(t);
        const int cols = min(SB, n - sb * SB);
        nb_sync(BAR_FULL + s);
        const double *Ps = P + s * K * TILE + lane * PS;
        if (live) {
          if (BACK) {
            for (int c = cols - 1; c >= 0; --c) {
              double p[K], o[K];
#pragma unroll
              for (int k = 0; k < K; ++k) p[k] = Ps[k * TILE + c];
              mc::add<K>(acc, p, o);
#pragma unroll
              for (int k = 0; k < K; ++k) acc[k] = o[k];
            }
          } else {
            for (int c = 0; c < cols; ++c) {
              double p[K], o[K];
#pragma unroll
              for (int k = 0; k < K; ++k) p[k] = Ps[k * TILE + c];
              mc::add<K>(acc, p, o);
#pragma unroll
              for (int k = 0; k < K; ++k) acc[k] = o[k];
            }
          }
        }
        __syncwarp();
        if (t + NSLOT < nfull) nb_arrive(BAR_EMPTY + s);
      }
      mark(1);
      nb_sync(BAR_STAGED);
      // critical source block: full madds as its rows become final.  Every
      // lane polls its own row of the block; each poll brings in all rows
      // published so far, and the ready ones are consumed in fold order.
      if (has_crit) {
        const int c0 = crit * SB, cols = min(SB, n - c0);
        double xv[K];
        bool have = lane >= cols;
        unsigned ready = __ballot_sync(0xffffffffu, have);
        int done = 0, iters = 0;
        mark(4);
        while (done < cols) {
          ++iters;
          // re-poll the missing rows; the loads fly while the ready
          // columns are consumed
          u64 w[2 * K];
          const bool polled = !have;
          if (polled) {
#pragma unroll
            for (int x = 0; x < 2 * K; ++x) w[x] = ld_word(W + x * N + c0 + lane);
          }
          for (; done < cols; ++done) {
            const int cc = BACK ? cols - 1 - done : done;
            if (!(ready >> cc & 1u)) break;
            double xj[K], a[K], o[K];
#pragma unroll
            for (int k = 0; k < K; ++k) {
              const double v = __shfl_sync(0xffffffffu, xv[k], cc);
              const double l = Lc[k * TILE + lane * PS + cc];
              xj[k] = BACK ? -v : v;
              a[k] = BACK ? l : -l;
              o[k] = acc[k];
            }
            mc::madd<K>(o, a, xj);
#pragma unroll
            for (int k = 0; k < K; ++k) acc[k] = live ? o[k] : acc[k];
          }
          if (polled) {
            bool ok = true;
#pragma unroll
            for (int x = 0; x < 2 * K; ++x) ok &= (unsigned)w[x] == seq;
            if (ok) {
              have = true;
#pragma unroll
              for (int k = 0; k < K; ++k)
                xv[k] = __longlong_as_double((long long)(
                    (w[2 * k + 1] & 0xffffffff00000000ull) | (w[2 * k] >> 32)));
            }
          }
          const unsigned prev = ready;
          ready = __ballot_sync(0xffffffffu, have);
          if (prev != ready && __popc(ready) == 32) mark(5);
          if (iters == 1) mark(7);
        }
        if (trace && lane == 0) trace[(int64_t)blk * 8 + 6] = iters;
      }
      mark(2);
      // diagonal triangle; each row is published the moment it is final
      for (int e = 0; e < rows; ++e) {
        const int jj = BACK ? rows - 1 - e : e;
        if (BACK && lane == jj) {
          double u[K], qv[K];
#pragma unroll
          for (int k = 0; k < K; ++k) u[k] = Ld[k * TILE + lane * PS + lane];
          mc::div_y<K>(acc, u, Ld[lane * PS + SB], qv);
#pragma unroll
          for (int k = 0; k < K; ++k) acc[k] = qv[k];
          publish_x<K>(W, N, i, acc, seq);
        }
        double xj[K], a[K], o[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const double v = __shfl_sync(0xffffffffu, acc[k], jj);
          const double l = Ld[k * TILE + lane * PS + jj];
          xj[k] = BACK ? -v : v;
          a[k] = BACK ? l : -l;
          o[k] = acc[k];
        }
        // forward: row jj is final; publish it (predicated, off the chain)
        if (!BACK) publish_x_if<K>(lane == jj, W, N, i, acc, seq);
        mc::madd<K>(o, a, xj);
        const bool upd = live && (BACK ? lane < jj : lane > jj);
#pragma unroll
        for (int k = 0; k < K; ++k) acc[k] = upd ? o[k] : acc[k];
      }
      if (live) {
#pragma unroll
        for (int k = 0; k < K; ++k) x[k * N + i] = acc[k];
      }
      mark(3);
    }
  }
}

template <int K>
size_t sweep_smem() {
  return (size_t)(NSLOT + 2) * K * TILE * sizeof(double);
}

template <typename F>
int coop_grid(F kern, size_t smem, int want) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, ST, smem);
  int cap = per_sm * num_sms();
  if (cap < 1) cap = 1;
  return want < cap ? want : cap;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_coop(void (*kern)(KArgs...), int grid, size_t smem,
                        cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(ST);
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
  const size_t smem = sweep_smem<K>();
  auto fk = sweep_kernel<K, false>;
  auto bk = sweep_kernel<K, true>;
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
  const int nblk = (n + SB - 1) / SB;
  if ((e = sw.ensure(n)) != cudaSuccess) return e;
  permute_kernel<K><<<(n + 255) / 256, 256, 0, s>>>(n, perm, b, x);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  u64 *tf = sw.trace, *tb = sw.trace ? sw.trace + (int64_t)8 * nblk : nullptr;
  e = launch_coop(fk, coop_grid(fk, smem, nblk), smem, s, n, LU, x, sw.words,
                  sw.next_seq(s), tf);
  if (e != cudaSuccess) return e;
  return launch_coop(bk, coop_grid(bk, smem, nblk), smem, s, n, LU, x,
                     sw.words, sw.next_seq(s), tb);
}

template <int K>
cudaError_t back_k(int n, MatView LU, double *x, SolveWork &sw,
                   cudaStream_t s) {
  const size_t smem = sweep_smem<K>();
  auto bk = sweep_kernel<K, true>;
  static bool configured = false;
  cudaError_t e;
  if (!configured) {
    if ((e = cudaFuncSetAttribute(
             bk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) !=
        cudaSuccess)
      return e;
    configured = true;
  }
  const int nblk = (n + SB - 1) / SB;
  if ((e = sw.ensure(n)) != cudaSuccess) return e;
  u64 *tb = sw.trace ? sw.trace + (int64_t)8 * nblk : nullptr;
  return launch_coop(bk, coop_grid(bk, smem, nblk), smem, s, n, LU, x,
                     sw.words, sw.next_seq(s), tb);
}

}  // namespace

cudaError_t lu_solve_back(int k, int n, MatView LU, double *x, SolveWork &sw,
                          cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  prof_begin(PROF_SOLVE, s);
  cudaError_t e = cudaErrorInvalidValue;
  switch (k) {
    case 2: e = back_k<2>(n, LU, x, sw, s); break;
    case 3: e = back_k<3>(n, LU, x, sw, s); break;
    case 4: e = back_k<4>(n, LU, x, sw, s); break;
  }
  prof_end(PROF_SOLVE, s);
  return e;
}

cudaError_t SolveWork::ensure(int64_t rows) {
  if (rows <= cap) return cudaSuccess;
  if (words) cudaFree(words);
  words = nullptr;
  cap = 0;
  const size_t bytes = (size_t)2 * LU_MAX_K * rows * sizeof(u64);
  cudaError_t e = cudaMalloc(&words, bytes);
  if (e != cudaSuccess) return e;
  // sequence 0 is never used, so zeroed words are never valid
  e = cudaMemset(words, 0, bytes);
  if (e != cudaSuccess) return e;
  cap = rows;
  if (std::getenv("MPCORE_TRACE_SOLVE")) {
    // diagnostics: [2 sweeps][blocks][4] globaltimer stamps of each owner
    if (trace) cudaFree(trace);
    trace_len = 2 * 8 * ((rows + SB - 1) / SB);
    e = cudaMalloc(&trace, trace_len * sizeof(u64));
    if (e != cudaSuccess) return e;
  }
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
