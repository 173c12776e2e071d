// Microbenchmark: latency of an all-to-all exchange of sequence-tagged
// 8-byte words among G co-resident CTAs (the panel's per-column pattern).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o llbench llbench.cu
#include <cstdio>
#include <cuda_runtime.h>

typedef unsigned long long u64;

__device__ __forceinline__ void st_rel(u64 *p, u64 v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ u64 ld_rel(const u64 *p) {
  u64 v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ u64 gtime() {
  u64 t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// mode 0: all-to-all, every CTA polls every slot (one warp, <=5 per lane)
// mode 1: tree: CTA 0 polls all, publishes a single word, all poll it
// stride: words per slot (padding)
__global__ void exchange(u64 *slots, u64 *out, int steps, int mode, int stride,
                         int sleep_ns) {
  const int G = gridDim.x, g = blockIdx.x, lane = threadIdx.x;
  u64 t0 = gtime();
  for (int s = 1; s <= steps; ++s) {
    unsigned seq = (unsigned)s;
    u64 *mine = slots + (size_t)((s & 1) * G + g) * stride;
    if (lane == 0) st_rel(mine, ((u64)g << 32) | seq);
    if (mode == 0 || g == 0) {
      unsigned done = 0;
      for (int q = 0; q < 5; ++q)
        if (lane + 32 * q >= G) done |= 1u << q;
      for (;;) {
        for (int q = 0; q < 5; ++q)
          if (!(done & (1u << q))) {
            u64 v = ld_rel(slots + (size_t)((s & 1) * G + lane + 32 * q) * stride);
            if ((unsigned)v == seq) done |= 1u << q;
          }
        if (__all_sync(0xffffffffu, done == 31u)) break;
        if (sleep_ns) __nanosleep(sleep_ns);
      }
      if (mode == 1 && lane == 0)
        st_rel(slots + (size_t)(2 * G + (s & 1)) * stride, seq);
    }
    if (mode == 1 && g != 0) {
      if (lane == 0) {
        while ((unsigned)ld_rel(slots + (size_t)(2 * G + (s & 1)) * stride) != seq)
          if (sleep_ns) __nanosleep(sleep_ns);
      }
      __syncwarp();
    }
  }
  u64 t1 = gtime();
  if (lane == 0) out[g] = t1 - t0;
}

int main() {
  int dev = 0;
  cudaSetDevice(dev);
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, dev);
  u64 *slots, *out;
  cudaMalloc(&slots, 1 << 22);
  cudaMalloc(&out, 4096 * 8);
  const int steps = 2000;
  for (int mode = 0; mode < 2; ++mode)
    for (int G : {16, 64, 148})
      for (int stride : {1, 16})
        for (int sl : {0, 32}) {
          cudaMemset(slots, 0, 1 << 22);
          void *args[] = {&slots, &out, (void *)&steps, &mode, &stride, &sl};
          cudaLaunchCooperativeKernel((void *)exchange, G, 32, args, 0, 0);
          cudaError_t e = cudaDeviceSynchronize();
          u64 h[4096];
          cudaMemcpy(h, out, G * 8, cudaMemcpyDeviceToHost);
          u64 mx = 0;
          for (int i = 0; i < G; ++i) mx = h[i] > mx ? h[i] : mx;
          printf("mode %d G %3d stride %2d sleep %2d: %.0f ns/step %s\n", mode,
                 G, stride, sl, (double)mx / steps,
                 e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
  return 0;
}
