// Stress check of mc::ddiv_y (division from a reciprocal hint) against
// __ddiv_rn on random and constructed hard cases: quotients next to rounding
// midpoints, divisors at both ends of the binade, wide exponent spreads.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -fmad=false \
//        -I paper_2107_12550_b200/csrc tools/divcheck.cu -o /tmp/divcheck
//   /tmp/divcheck [rounds]
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "mc.cuh"

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double mk(uint64_t sign, int e, uint64_t man) {
  return __longlong_as_double((long long)((sign << 63) |
                                          ((uint64_t)(e + 1023) << 52) |
                                          (man & 0xFFFFFFFFFFFFFull)));
}

__global__ void check(uint64_t seed, unsigned long long *bad,
                      double *first) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t s = mix(seed ^ (t * 0xD1B54A32D192ED03ull));
  for (int it = 0; it < 64; ++it) {
    s = mix(s);
    const uint64_t u1 = s, u2 = mix(s ^ 1), u3 = mix(s ^ 2);
    const int kind = (int)(u3 & 7);
    double a, b;
    const int ea = (int)((u3 >> 8) % 847) - 423;
    const int eb = (int)((u3 >> 20) % 847) - 423;
    uint64_t mb = u2;
    if (kind == 1) mb |= 0xFFFFFFFFFF000ull;         // b near 2
    if (kind == 2) mb &= 0x0000000000FFFull;         // b near 1
    if (kind == 3) mb = 0x6A09E667F3BCDull ^ (u2 & 0xFFF);  // b near sqrt 2
    b = mk(u2 >> 63, eb, mb);
    if (kind >= 4) {
      // a = RN(m b) + d ulps with m a midpoint of the quotient's binade
      const double q = mk(0, ea - eb > 400 ? 400 - 0 : (ea - eb < -400 ? -400 : ea - eb), u1);
      const double m = __dadd_rn(q, __dmul_rn(q, 0x1p-53));  // ~ q + ulp/2
      double am = __dmul_rn(m, b);
      const int d = (int)((u3 >> 40) % 5) - 2;
      long long bits = __double_as_longlong(am) + d;
      a = __longlong_as_double(bits);
      if (kind == 5) a = __longlong_as_double(__double_as_longlong(am) ^ 1);
    } else {
      a = mk(u1 >> 63, ea, u1);
    }
    const double y = mc::recip_hint(b);
    const double f = mc::ddiv_y(a, b, y);
    const double r = __ddiv_rn(a, b);
    if (__double_as_longlong(f) != __double_as_longlong(r)) {
      unsigned long long k = atomicAdd(bad, 1ull);
      if (k < 4) {
        first[3 * k] = a;
        first[3 * k + 1] = b;
        first[3 * k + 2] = f;
      }
    }
  }
}

int main(int argc, char **argv) {
  const int rounds = argc > 1 ? atoi(argv[1]) : 200;
  unsigned long long *bad;
  double *first;
  cudaMallocManaged(&bad, 8);
  cudaMallocManaged(&first, 12 * 8);
  *bad = 0;
  const int blocks = 148 * 16, threads = 256;
  for (int r = 0; r < rounds; ++r)
    check<<<blocks, threads>>>(0x5eed0000ull + r, bad, first);
  cudaError_t e = cudaDeviceSynchronize();
  const double total = (double)rounds * blocks * threads * 64;
  printf("divcheck: %s, %.3g pairs, %llu mismatches\n", cudaGetErrorString(e),
         total, *bad);
  for (unsigned long long k = 0; k < *bad && k < 4; ++k)
    printf("  a=%a b=%a fast=%a\n", first[3 * k], first[3 * k + 1],
           first[3 * k + 2]);
  return (e == cudaSuccess && *bad == 0) ? 0 : 1;
}
