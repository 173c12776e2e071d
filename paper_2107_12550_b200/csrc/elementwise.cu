// Elementwise batch kernels (linalg.py:624-673: axpy_batch,
// elementwise_add/mul_batch), elementwise division (mcfloat.py:304-318) and
// square root (mcfloat.py:324-340, mc_sqrt 596-601),
// mat_vec (linalg.py:545-574) and the seeded planar input generator.
#include "internal.h"
#include "mc.cuh"

namespace mpk {

namespace {

constexpr int EW_THREADS = 256;

template <int K, int OP>
__global__ void __launch_bounds__(EW_THREADS)
ew_kernel(int64_t n, const double *__restrict__ x,
          const double *__restrict__ y, double *__restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double a[K], b[K], o[K];
#pragma unroll
    for (int c = 0; c < K; ++c) {
      a[c] = x[c * n + i];
      b[c] = OP == 3 ? 0.0 : y[c * n + i];
    }
    if constexpr (OP == 0) mc::add<K>(a, b, o);
    else if constexpr (OP == 1) mc::mul<K>(a, b, o);
    else if constexpr (OP == 2) mc::div<K>(a, b, o);
    else mc::sqrt<K>(a, o);  // (unary: y is not read)
#pragma unroll
    for (int c = 0; c < K; ++c) out[c * n + i] = o[c];
  }
}

template <int K> struct Alpha { double c[K]; };

// y_i <- add(y_i, mul(x_i, alpha))   (linalg.py:636-642; alpha from the right)
template <int K>
__global__ void __launch_bounds__(EW_THREADS)
axpy_kernel(int64_t n, Alpha<K> alpha, const double *__restrict__ x,
            double *__restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double a[K], acc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) {
      a[c] = x[c * n + i];
      acc[c] = y[c * n + i];
    }
    mc::madd<K>(acc, a, alpha.c);
#pragma unroll
    for (int c = 0; c < K; ++c) y[c * n + i] = acc[c];
  }
}

// splitmix64 finaliser (testgen.py:57-59) and the [-1, 1) mapping
// (testgen.py:100-101): RN(double(u)) * 2^-63 - 1.
__device__ __forceinline__ double uniform_at(uint64_t seed, uint64_t i) {
  uint64_t z = seed + 0x9E3779B97F4A7C15ull * (i + 1);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z = z ^ (z >> 31);
  return __dsub_rn(__dmul_rn(__ull2double_rn(z), 0x1p-63), 1.0);
}

template <int K>
__global__ void __launch_bounds__(EW_THREADS)
gen_kernel(double *__restrict__ out, int64_t count, int64_t plane,
           uint64_t base_index, uint64_t seed) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x) {
    uint64_t idx = (base_index + (uint64_t)e) * 4ull;
    double raw[K], zero[K], o[K];
    raw[0] = uniform_at(seed, idx);
#pragma unroll
    for (int c = 1; c < K; ++c)
      raw[c] = __dmul_rn(__dmul_rn(raw[c - 1], 0x1p-53),
                         uniform_at(seed, idx + c));
#pragma unroll
    for (int c = 0; c < K; ++c) zero[c] = 0.0;
    mc::add<K>(raw, zero, o);  // renormalise: add_k(raw, 0)
#pragma unroll
    for (int c = 0; c < K; ++c) out[c * plane + e] = o[c];
  }
}

// The same recipe for the local columns of a column-block-cyclic layout:
// local column lc of rank `rank` is global column
// ((lc / nb) * world + rank) * nb + lc % nb of a size-n system.
template <int K>
__global__ void __launch_bounds__(EW_THREADS)
gen_cyclic_kernel(double *__restrict__ out, int64_t ld, int64_t plane,
                  int rows, int local_cols, int nb, int world, int rank,
                  uint64_t base_index, int64_t n, uint64_t seed) {
  const int64_t count = (int64_t)rows * local_cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / local_cols), lc = (int)(e % local_cols);
    const int64_t gc = ((int64_t)(lc / nb) * world + rank) * nb + lc % nb;
    double o[K];
    if (gc < n) {
      uint64_t idx = (base_index + (uint64_t)r * (uint64_t)n + (uint64_t)gc) * 4ull;
      double raw[K], zero[K];
      raw[0] = uniform_at(seed, idx);
#pragma unroll
      for (int c = 1; c < K; ++c)
        raw[c] = __dmul_rn(__dmul_rn(raw[c - 1], 0x1p-53),
                           uniform_at(seed, idx + c));
#pragma unroll
      for (int c = 0; c < K; ++c) zero[c] = 0.0;
      mc::add<K>(raw, zero, o);
    } else {
#pragma unroll
      for (int c = 0; c < K; ++c) o[c] = 0.0;
    }
#pragma unroll
    for (int c = 0; c < K; ++c) out[c * plane + (int64_t)r * ld + lc] = o[c];
  }
}

// mat_vec: one thread per row; the row chain runs over column tiles staged
// through shared memory with coalesced loads.
constexpr int MV_ROWS = 128;
template <int K> constexpr int mv_cols() { return K == 2 ? 16 : 8; }

template <int K>
__global__ void __launch_bounds__(MV_ROWS)
matvec_kernel(int rows, int cols, MatView A, const double *__restrict__ x,
              double *__restrict__ y) {
  constexpr int MV_COLS = mv_cols<K>();
  __shared__ double tile[K][MV_ROWS][MV_COLS + 1];
  __shared__ double xs[K][MV_COLS];
  const int r0 = blockIdx.x * MV_ROWS;
  const int row = r0 + threadIdx.x;
  double acc[K];
#pragma unroll
  for (int c = 0; c < K; ++c) acc[c] = 0.0;
  for (int j0 = 0; j0 < cols; j0 += MV_COLS) {
    const int jn = min(MV_COLS, cols - j0);
    __syncthreads();
    for (int t = threadIdx.x; t < MV_ROWS * MV_COLS; t += MV_ROWS) {
      int rr = t / MV_COLS, cc = t % MV_COLS;
      if (r0 + rr < rows && cc < jn) {
#pragma unroll
        for (int c = 0; c < K; ++c)
          tile[c][rr][cc] = A.p[c * A.plane + (int64_t)(r0 + rr) * A.ld + j0 + cc];
      }
    }
    if (threadIdx.x < jn) {
#pragma unroll
      for (int c = 0; c < K; ++c) xs[c][threadIdx.x] = x[c * (int64_t)cols + j0 + threadIdx.x];
    }
    __syncthreads();
    if (row < rows) {
      for (int cc = 0; cc < jn; ++cc) {
        double a[K], b[K];
#pragma unroll
        for (int c = 0; c < K; ++c) {
          a[c] = tile[c][threadIdx.x][cc];
          b[c] = xs[c][cc];
        }
        mc::madd<K>(acc, a, b);
      }
    }
  }
  if (row < rows) {
#pragma unroll
    for (int c = 0; c < K; ++c) y[c * (int64_t)rows + row] = acc[c];
  }
}

int grid_for(int64_t n) {
  int64_t g = (n + EW_THREADS - 1) / EW_THREADS;
  int64_t cap = (int64_t)num_sms() * 8;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

template <int K>
cudaError_t ew_dispatch(int op, int64_t n, const double *x, const double *y,
                        double *out, cudaStream_t s) {
  int g = grid_for(n);
  if (op == 0) ew_kernel<K, 0><<<g, EW_THREADS, 0, s>>>(n, x, y, out);
  else if (op == 1) ew_kernel<K, 1><<<g, EW_THREADS, 0, s>>>(n, x, y, out);
  else if (op == 2) ew_kernel<K, 2><<<g, EW_THREADS, 0, s>>>(n, x, y, out);
  else ew_kernel<K, 3><<<g, EW_THREADS, 0, s>>>(n, x, y, out);
  return cudaGetLastError();
}

}  // namespace

#define KSWITCH(k, expr)                                  \
  switch (k) {                                            \
    case 2: { constexpr int K = 2; return expr; }         \
    case 3: { constexpr int K = 3; return expr; }         \
    case 4: { constexpr int K = 4; return expr; }         \
    default: return cudaErrorInvalidValue;                \
  }

cudaError_t elementwise(int k, int op, int64_t n, const double *x,
                        const double *y, double *out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  prof_begin(PROF_ELEMENTWISE, s);
  cudaError_t e;
  switch (k) {
    case 2: e = ew_dispatch<2>(op, n, x, y, out, s); break;
    case 3: e = ew_dispatch<3>(op, n, x, y, out, s); break;
    case 4: e = ew_dispatch<4>(op, n, x, y, out, s); break;
    default: return cudaErrorInvalidValue;
  }
  prof_end(PROF_ELEMENTWISE, s);
  return e;
}

template <int K>
static cudaError_t axpy_k(int64_t n, const double *alpha, const double *x,
                          double *y, cudaStream_t s) {
  Alpha<K> al;
  for (int c = 0; c < K; ++c) al.c[c] = alpha[c];
  axpy_kernel<K><<<grid_for(n), EW_THREADS, 0, s>>>(n, al, x, y);
  return cudaGetLastError();
}

cudaError_t axpy(int k, int64_t n, const double *alpha, const double *x,
                 double *y, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  KSWITCH(k, axpy_k<K>(n, alpha, x, y, s));
}

template <int K>
static cudaError_t gen_k(double *out, int64_t count, int64_t plane, int slot,
                         int64_t n, uint64_t seed, cudaStream_t s) {
  uint64_t base = (uint64_t)slot * (uint64_t)n * (uint64_t)n;
  prof_begin(PROF_GEN, s);
  gen_kernel<K><<<grid_for(count), EW_THREADS, 0, s>>>(out, count, plane, base,
                                                       seed);
  prof_end(PROF_GEN, s);
  return cudaGetLastError();
}

cudaError_t generate(int k, double *out, int64_t count, int64_t plane,
                     int slot, int64_t n, uint64_t seed, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  KSWITCH(k, gen_k<K>(out, count, plane, slot, n, seed, s));
}

template <int K>
static cudaError_t gen_cyclic_k(MatView out, int rows, int local_cols, int nb,
                                int world, int rank, int slot, int64_t n,
                                uint64_t seed, cudaStream_t s) {
  uint64_t base = (uint64_t)slot * (uint64_t)n * (uint64_t)n;
  gen_cyclic_kernel<K><<<grid_for((int64_t)rows * local_cols), EW_THREADS, 0,
                         s>>>(out.p, out.ld, out.plane, rows, local_cols, nb,
                              world, rank, base, n, seed);
  return cudaGetLastError();
}

cudaError_t generate_cyclic(int k, MatView out, int rows, int local_cols,
                            int nb, int world, int rank, int slot, int64_t n,
                            uint64_t seed, cudaStream_t s) {
  if ((int64_t)rows * local_cols <= 0) return cudaSuccess;
  KSWITCH(k, gen_cyclic_k<K>(out, rows, local_cols, nb, world, rank, slot, n,
                             seed, s));
}

template <int K>
static cudaError_t matvec_k(int rows, int cols, MatView A, const double *x,
                            double *y, cudaStream_t s) {
  prof_begin(PROF_MATVEC, s);
  matvec_kernel<K><<<(rows + MV_ROWS - 1) / MV_ROWS, MV_ROWS, 0, s>>>(
      rows, cols, A, x, y);
  prof_end(PROF_MATVEC, s);
  return cudaGetLastError();
}

cudaError_t matvec(int k, int rows, int cols, MatView A, const double *x,
                   double *y, cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  KSWITCH(k, matvec_k<K>(rows, cols, A, x, y, s));
}

}  // namespace mpk
