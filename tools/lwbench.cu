// Latency of one warp-cooperative 512-bit correctly rounded add / mul
// (longwarp.cuh) in a dependent chain: cycles per operation.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -I paper_2107_12550_b200/csrc tools/lwbench.cu -o /tmp/lwbench
#include <cstdio>
#include <cstdint>
#include "longfloat.cuh"
#include "longwarp.cuh"

__global__ void bench(int iters, int p, long long *out, uint64_t *sink) {
  const int t = threadIdx.x;
  // operands: mantissas with the top bit at p - 1, varying exponents
  lw::WV a, b;
  a.m = t < 8 ? 0x9E3779B97F4A7C15ull * (t + 1) : 0ull;
  b.m = t < 8 ? 0xBF58476D1CE4E5B9ull * (t + 3) : 0ull;
  if (t == 7) { a.m |= 1ull << 63; b.m |= 1ull << 63; }
  a.exp = -512; b.exp = -530;
  a.sign = 1; b.sign = 1;
  lw::WV acc = a;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    b.exp = -530 - (i & 7);
    acc = lw::add(acc, b, p);
    acc.exp = -512;  // keep the magnitude steady
  }
  long long t1 = clock64();
  lw::WV m = a;
  for (int i = 0; i < iters; ++i) {
    m = lw::mul(m, b, p);
    m.exp = -512;
  }
  long long t2 = clock64();
  if (t == 0) { out[0] = t1 - t0; out[1] = t2 - t1; }
  sink[t] = acc.m ^ m.m;
}

int main() {
  long long *d, h[2];
  uint64_t *s;
  cudaMalloc(&d, 16);
  cudaMalloc(&s, 32 * 8);
  const int iters = 2000;
  bench<<<1, 32>>>(iters, 512, d, s);
  bench<<<1, 32>>>(iters, 512, d, s);
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("lw::add %.0f cycles, lw::mul %.0f cycles (512 bits, dependent chain, one warp)\n",
         (double)h[0] / iters, (double)h[1] / iters);
  return 0;
}
