// IR residual r = b - A x at the long precision p on the GPU (SURVEY §8(f)
// row 1; refine.py:163-172 with the scalar mat_vec order of
// linalg.py:564-574): per row i, acc = fold_j add(acc, mul(A_ij, x_j)) in
// ascending j from zero, then r_i = add(b_i, -acc) -- every operation
// correctly rounded to p bits (longfloat.cuh), so r is the host's (and
// the reference's) residual bit for bit.  Each row is one sequential chain
// of n dependent long multiply-adds: a thread per row, one warp per block
// so the warps spread over the SMs.
#include <cstdlib>

#include "internal.h"
#include "longfloat.cuh"
#include "longwarp.cuh"
#include "longseg.cuh"

namespace mpk {

namespace {

template <int N>
__global__ void __launch_bounds__(32)
long_residual_kernel(const lf::DF *__restrict__ A, const lf::DF *__restrict__ x,
                     const lf::DF *__restrict__ b, lf::DF *__restrict__ res,
                     int n, int p) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const lf::DF *row = A + (int64_t)i * n;
  lf::DF acc = lf::zero();
  for (int j = 0; j < n; ++j) {
    const lf::DF prod = lf::mul<N>(row[j], x[j], p);
    acc = lf::add<N>(acc, prod, p);
  }
  res[i] = lf::add<N>(b[i], lf::neg(acc), p);
}

// The same chain, one warp per row: lane t holds limb t (longwarp.cuh),
// so each long multiply-add costs a few hundred cycles of lane-parallel
// steps instead of thousands of sequential limb operations.  The next
// step's operands are loaded while the current one is computed.
__global__ void __launch_bounds__(128)
long_residual_warp_kernel(const lf::DF *__restrict__ A,
                          const lf::DF *__restrict__ x,
                          const lf::DF *__restrict__ b,
                          lf::DF *__restrict__ res, int n, int p) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (lw::uni(row >= n)) return;  // warp-uniform
  const int t = threadIdx.x & 31;
  auto load = [&](const lf::DF &v) {
    lw::WV w;
    w.m = t < lf::NL ? v.m[t] : 0ull;
    w.exp = v.exp;
    w.sign = v.sign;
    return w;
  };
  const lf::DF *arow = A + (int64_t)row * n;
  lw::WV acc = lw::zero();
  lw::WV an = load(arow[0]), xn = load(x[0]);
  for (int j = 0; j < n; ++j) {
    const lw::WV aj = an, xj = xn;
    if (j + 1 < n) {
      an = load(arow[j + 1]);
      xn = load(x[j + 1]);
    }
    acc = lw::add(acc, lw::mul(aj, xj, p), p);
  }
  const lw::WV r = lw::add(load(b[row]), lw::neg(acc), p);
  if (t < lf::NL) res[row].m[t] = r.m;
  if (t == 0) {
    res[row].sign = r.sign;
    res[row].exp = r.sign == 0 ? 0 : r.exp;
  }
}

// The same chain with its products moved off it: acc_i = add(acc_i,
// mul(A_ij, x_j)) needs each product only when it is added, and the
// products do not depend on acc.  One CTA per row: warp 0 runs the chain of
// correctly rounded adds in ascending j; warps 1..LR_PROD form the products
// (the same warp-cooperative mul) ahead of it into a shared-memory ring,
// published by a per-slot sequence flag.  Every operation and its order are
// unchanged, so the result is the same bits; the chain is the adds only.
constexpr int LR_RING = 8;

template <int NP>  // producer warps

__global__ void __launch_bounds__(32 * (1 + NP))
long_residual_split_kernel(const lf::DF *__restrict__ A,
                           const lf::DF *__restrict__ x,
                           const lf::DF *__restrict__ b,
                           lf::DF *__restrict__ res, int n, int p) {
  __shared__ uint64_t ring_m[LR_RING][32];
  __shared__ int64_t ring_e[LR_RING];
  __shared__ int ring_s[LR_RING];
  __shared__ volatile int ready[LR_RING];  // j + 1 once product j is in
  __shared__ volatile int consumed;        // products taken by the chain
  const int row = blockIdx.x, warp = threadIdx.x >> 5, t = threadIdx.x & 31;
  if (threadIdx.x < LR_RING) ready[threadIdx.x] = 0;
  if (threadIdx.x == 0) consumed = 0;
  __syncthreads();
  auto load = [&](const lf::DF &v) {
    lw::WV w;
    w.m = t < lf::NL ? v.m[t] : 0ull;
    w.exp = v.exp;
    w.sign = v.sign;
    return w;
  };
  const lf::DF *arow = A + (int64_t)row * n;
  if (warp == 0) {
    lw::WV acc = lw::zero();
    for (int j = 0; j < n; ++j) {
      const int s = j % LR_RING;
      while (lw::uni(ready[s] != j + 1)) {
      }
      __threadfence_block();
      lw::WV pr;
      pr.m = ring_m[s][t];
      pr.exp = ring_e[s];
      pr.sign = ring_s[s];
      __threadfence_block();
      __syncwarp();
      if (t == 0) consumed = j + 1;  // the slot may be refilled
      acc = lw::add(acc, pr, p);
    }
    const lw::WV r = lw::add(load(b[row]), lw::neg(acc), p);
    if (t < lf::NL) res[row].m[t] = r.m;
    if (t == 0) {
      res[row].sign = r.sign;
      res[row].exp = r.sign == 0 ? 0 : r.exp;
    }
  } else {
    const int pw = warp - 1;
    int j = pw;
    lw::WV an, xn;
    if (j < n) {
      an = load(arow[j]);
      xn = load(x[j]);
    }
    for (; j < n; j += NP) {
      const lw::WV aj = an, xj = xn;
      if (j + NP < n) {
        an = load(arow[j + NP]);
        xn = load(x[j + NP]);
      }
      const lw::WV pr = lw::mul(aj, xj, p);
      const int s = j % LR_RING;
      // slot s last held product j - LR_RING
      while (lw::uni(consumed <= j - LR_RING)) __nanosleep(64);
      __threadfence_block();
      ring_m[s][t] = pr.m;
      if (t == 0) {
        ring_e[s] = pr.exp;
        ring_s[s] = pr.sign;
      }
      __threadfence_block();
      __syncwarp();
      if (t == 0) ready[s] = j + 1;
    }
  }
}

// Variant 5 (production): the products and the chains in two kernels.
// Every product mul(A_ij, x_j) is independent, so a first kernel forms all
// n^2 of them -- two per warp, one per 16-lane segment (longseg.cuh: the
// 2p-bit product needs 16 limbs, so a full warp left half its lanes idle) --
// into a scratch matrix at full occupancy; then one warp per row runs only
// its chain of correctly rounded adds over its row of products, the next
// product's load in flight -- no producer/consumer hand-off inside the
// chain.  (Fused into one cooperative launch, with the chains trailing the
// production column block by column block, it was slower: the chains then
// compete with the producers for issue slots.)
// two products per warp (one per 16-lane segment, longseg.cuh)
__global__ void __launch_bounds__(256)
long_products2_kernel(const lf::DF *__restrict__ A,
                      const lf::DF *__restrict__ x, lf::DF *__restrict__ P,
                      int n, int p) {
  const int t = threadIdx.x & 15, sg = (threadIdx.x >> 4) & 1;
  const int64_t nn = (int64_t)n * n;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t e0 = 2 * wid; e0 < nn; e0 += 2 * nw) {
    const int64_t e = e0 + sg;
    if (e < nn) {  // (segment-uniform)
      const lf::DF &a = A[e], &xv = x[e % n];
      ls::WV wa, wx;
      wa.m = t < lf::NL ? a.m[t] : 0ull;
      wa.exp = a.exp;
      wa.sign = a.sign;
      wx.m = t < lf::NL ? xv.m[t] : 0ull;
      wx.exp = xv.exp;
      wx.sign = xv.sign;
      const ls::WV pr = ls::mul(wa, wx, p);
      if (t < lf::NL) P[e].m[t] = pr.m;
      if (t == 0) {
        P[e].sign = pr.sign;
        P[e].exp = pr.exp;
      }
    }
  }
}

__global__ void __launch_bounds__(128)
long_chain_kernel(const lf::DF *__restrict__ P, const lf::DF *__restrict__ b,
                  lf::DF *__restrict__ res, int n, int p) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (lw::uni(row >= n)) return;
  const int t = threadIdx.x & 31;
  auto load = [&](const lf::DF &v) {
    lw::WV w;
    w.m = t < lf::NL ? v.m[t] : 0ull;
    w.exp = v.exp;
    w.sign = v.sign;
    return w;
  };
  const lf::DF *prow = P + (int64_t)row * n;
  lw::WV acc = lw::zero();
  lw::WV nx = load(prow[0]);
  for (int j = 0; j < n; ++j) {
    const lw::WV pj = nx;
    if (j + 1 < n) nx = load(prow[j + 1]);
    acc = lw::add(acc, pj, p);
  }
  const lw::WV r = lw::add(load(b[row]), lw::neg(acc), p);
  if (t < lf::NL) res[row].m[t] = r.m;
  if (t == 0) {
    res[row].sign = r.sign;
    res[row].exp = r.sign == 0 ? 0 : r.exp;
  }
}

}  // namespace

cudaError_t long_residual(int p, int n, const void *A, const void *x,
                          const void *b, void *res, cudaStream_t s,
                          int variant) {
  if (n <= 0) return cudaSuccess;
  if (variant == 5 && p <= 512) {
    // scratch for the n^2 products (grow-only, kept)
    static void *scratch = nullptr;
    static size_t cap = 0;
    const size_t need = (size_t)n * n * sizeof(lf::DF);
    if (cap < need) {
      if (scratch) cudaFree(scratch);
      scratch = nullptr;
      cap = 0;
      cudaError_t e = cudaMalloc(&scratch, need);
      if (e != cudaSuccess) return e;
      cap = need;
    }
    auto *P = static_cast<lf::DF *>(scratch);
    long_products2_kernel<<<148 * 8, 256, 0, s>>>(
        static_cast<const lf::DF *>(A), static_cast<const lf::DF *>(x), P, n,
        p);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    long_chain_kernel<<<(n + 3) / 4, 128, 0, s>>>(
        P, static_cast<const lf::DF *>(b), static_cast<lf::DF *>(res), n, p);
    return cudaGetLastError();
  }
  if (variant == 2 && p <= 512) {
    // producer warps per row (MPCORE_RESIDUAL_PRODUCERS, default 2)
    static const int np = [] {
      const char *e = std::getenv("MPCORE_RESIDUAL_PRODUCERS");
      const int v = e ? std::atoi(e) : 2;
      return v < 1 ? 1 : (v > 3 ? 3 : v);
    }();
    auto a2 = static_cast<const lf::DF *>(A);
    auto x2 = static_cast<const lf::DF *>(x);
    auto b2 = static_cast<const lf::DF *>(b);
    auto r2 = static_cast<lf::DF *>(res);
    if (np == 1)
      long_residual_split_kernel<1><<<n, 64, 0, s>>>(a2, x2, b2, r2, n, p);
    else if (np == 2)
      long_residual_split_kernel<2><<<n, 96, 0, s>>>(a2, x2, b2, r2, n, p);
    else
      long_residual_split_kernel<3><<<n, 128, 0, s>>>(a2, x2, b2, r2, n, p);
    return cudaGetLastError();
  }
  if (variant == 0 && p <= 512) {
    long_residual_warp_kernel<<<(n + 3) / 4, 128, 0, s>>>(
        static_cast<const lf::DF *>(A), static_cast<const lf::DF *>(x),
        static_cast<const lf::DF *>(b), static_cast<lf::DF *>(res), n, p);
    return cudaGetLastError();
  }
  const int N = (p + 63) >> 6;
  const dim3 grid((n + 31) / 32), block(32);
  auto a = static_cast<const lf::DF *>(A);
  auto xv = static_cast<const lf::DF *>(x);
  auto bv = static_cast<const lf::DF *>(b);
  auto r = static_cast<lf::DF *>(res);
  switch (N) {
#define LR_CASE(NN)                                                        \
  case NN:                                                                 \
    long_residual_kernel<NN><<<grid, block, 0, s>>>(a, xv, bv, r, n, p);   \
    break;
    LR_CASE(1) LR_CASE(2) LR_CASE(3) LR_CASE(4)
    LR_CASE(5) LR_CASE(6) LR_CASE(7) LR_CASE(8)
#undef LR_CASE
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace mpk
