// Microbenchmark: all-to-all exchange of sequence-tagged 8-byte words among
// the CTAs of one thread-block cluster through distributed shared memory
// (remote st.shared::cluster, local polling) -- the panel's per-column
// pattern without the L2 round trip.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmembench dsmembench.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;

__device__ __forceinline__ unsigned cluster_ctarank() {
  unsigned r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r;
}
__device__ __forceinline__ unsigned cluster_nctarank() {
  unsigned r; asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r)); return r;
}
__device__ __forceinline__ u64 gtime() {
  u64 t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t;
}
// address of my shared variable in CTA `rank` of the cluster
__device__ __forceinline__ unsigned remote(const void *p, unsigned rank) {
  unsigned s = (unsigned)__cvta_generic_to_shared(p), r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(s), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_remote(unsigned addr, u64 v) {
  asm volatile("st.relaxed.cluster.shared::cluster.u64 [%0], %1;" :: "r"(addr), "l"(v) : "memory");
}
__device__ __forceinline__ u64 ld_local(const u64 *p) {
  u64 v; unsigned s = (unsigned)__cvta_generic_to_shared(p);
  asm volatile("ld.relaxed.cluster.shared::cta.u64 %0, [%1];" : "=l"(v) : "r"(s) : "memory");
  return v;
}

__global__ void exchange(u64 *out, int steps, int words) {
  __shared__ u64 slots[2][16][8];
  const unsigned C = cluster_nctarank(), g = cluster_ctarank();
  const int lane = threadIdx.x;
  for (int i = lane; i < 2 * 16 * 8; i += 32) (&slots[0][0][0])[i] = 0;
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  u64 t0 = gtime();
  for (int s = 1; s <= steps; ++s) {
    const unsigned seq = (unsigned)s;
    // lane (c, x): word x of my slot into CTA c
    for (int e = lane; e < (int)C * words; e += 32) {
      const unsigned c = e / words, x = e % words;
      st_remote(remote(&slots[s & 1][g][x], c), ((u64)g << 32) | seq);
    }
    // poll every slot locally: lane = (slot, word)
    for (;;) {
      bool ok = true;
      for (int e = lane; e < (int)C * words; e += 32) {
        const int c = e / words, x = e % words;
        ok &= (unsigned)ld_local(&slots[s & 1][c][x]) == seq;
      }
      if (__all_sync(0xffffffffu, ok)) break;
    }
  }
  u64 t1 = gtime();
  if (lane == 0) out[blockIdx.x] = t1 - t0;
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

int main() {
  u64 *d, h[16];
  cudaMalloc(&d, 16 * sizeof(u64));
  cudaFuncSetAttribute(exchange, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const int steps = 2000;
  for (int C : {2, 4, 8, 16}) for (int words : {1, 5}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C); cfg.blockDim = dim3(32);
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = C; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    cfg.attrs = a; cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, exchange, d, steps, words);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("C=%d: %s\n", C, cudaGetErrorString(e)); cudaGetLastError(); continue; }
    cudaMemcpy(h, d, C * sizeof(u64), cudaMemcpyDeviceToHost);
    u64 mx = 0; for (int i = 0; i < C; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("cluster %2d, %d words/slot: %.1f ns per all-to-all exchange\n", C, words, (double)mx / steps);
  }
  return 0;
}
