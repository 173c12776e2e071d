// FP64 issue-rate microbenchmark (the roofline denominator; MEASURED_PEAKS
// has no FP64 figure).  Each thread runs 8 independent dependency chains so
// the FP64 pipe, not latency, bounds the rate.
#include <cuda_runtime.h>
#include "../../include/mpcore.h"
#include "internal.h"

namespace {
constexpr int CH = 8, ITERS = 4096, THREADS = 256;

__global__ void __launch_bounds__(THREADS) dadd_loop(double *out, double s) {
  double a[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) a[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = __dadd_rn(a[c], s);
  }
  double t = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) t += a[c];
  if (t == 12345.678) out[0] = t;
}

__global__ void __launch_bounds__(THREADS) dfma_loop(double *out, double s) {
  double a[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) a[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = __fma_rn(a[c], s, s);
  }
  double t = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) t += a[c];
  if (t == 12345.678) out[0] = t;
}
}  // namespace

extern "C" int32_t mpcore_fp64_peak(double *dadd_per_s, double *dfma_per_s) {
  if (!dadd_per_s || !dfma_per_s) return MPCORE_BAD_DIMENSION;
  int32_t sms = 0;
  int st = mpcore_sm_count(&sms);
  if (st) return st;
  double *d = nullptr;
  if (cudaMalloc(&d, sizeof(double)) != cudaSuccess) return MPCORE_INTERNAL;
  const int blocks = sms * 8;
  const double instr = (double)blocks * THREADS * ITERS * CH;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best_add = 1e30f, best_fma = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(a);
    dadd_loop<<<blocks, THREADS>>>(d, 1e-300);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float t;
    cudaEventElapsedTime(&t, a, b);
    if (rep && t < best_add) best_add = t;
    cudaEventRecord(a);
    dfma_loop<<<blocks, THREADS>>>(d, 1e-300);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&t, a, b);
    if (rep && t < best_fma) best_fma = t;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaError_t e = cudaGetLastError();
  cudaFree(d);
  if (e != cudaSuccess) return MPCORE_INTERNAL;
  *dadd_per_s = instr / (best_add * 1e-3);
  *dfma_per_s = instr / (best_fma * 1e-3);
  return MPCORE_OK;
}
