// IR residual r = b - A x at the long precision p on the GPU (SURVEY §8(f)
// row 1; refine.py:163-172 with the scalar mat_vec order of
// linalg.py:564-574): per row i, acc = fold_j add(acc, mul(A_ij, x_j)) in
// ascending j from zero, then r_i = add(b_i, -acc) -- every operation
// correctly rounded to p bits (longfloat.cuh), so r is the host's (and
// the reference's) residual bit for bit.  Each row is one sequential chain
// of n dependent long multiply-adds: a thread per row, one warp per block
// so the warps spread over the SMs.
#include "internal.h"
#include "longfloat.cuh"
#include "longwarp.cuh"

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

}  // namespace

cudaError_t long_residual(int p, int n, const void *A, const void *x,
                          const void *b, void *res, cudaStream_t s,
                          int variant) {
  if (n <= 0) return cudaSuccess;
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
