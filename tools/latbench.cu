// FP64 dependent-latency microbenchmark (one warp, clock64).
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2107_12550_b200/csrc/mc.cuh"

__global__ void lat(double *out, long long *cyc, double s) {
  double a = threadIdx.x * 1e-9 + 1.0, b = s;
  long long t0 = clock64();
  for (int i = 0; i < 1000; ++i) a = __dadd_rn(a, b);
  long long t1 = clock64();
  double c = a;
  for (int i = 0; i < 1000; ++i) c = __fma_rn(c, b, b);
  long long t2 = clock64();
  double d = c;
  for (int i = 0; i < 100; ++i) d = __ddiv_rn(d, b + 1.0);
  long long t3 = clock64();
  // one TD madd chain: acc = add(acc, mul(x, y)) with acc dependence
  double acc[3] = {d, 0, 0}, x[3] = {1.0000001, 1e-17, 1e-34}, y[3] = {0.999, 2e-18, 0};
  for (int i = 0; i < 100; ++i) mc::madd<3>(acc, x, y);
  long long t4 = clock64();
  double q[3];
  for (int i = 0; i < 20; ++i) { mc::div<3>(acc, x, q); acc[0] = q[0]; acc[1] = q[1]; acc[2] = q[2]; }
  long long t5 = clock64();
  double acc2[2] = {acc[0], acc[1]}, x2[2] = {1.0000001, 1e-17}, y2[2] = {0.999, 2e-18};
  for (int i = 0; i < 100; ++i) mc::madd<2>(acc2, x2, y2);
  long long t6 = clock64();
  double q2[2];
  for (int i = 0; i < 20; ++i) { mc::div<2>(acc2, x2, q2); acc2[0] = q2[0]; acc2[1] = q2[1]; }
  long long t7 = clock64();
  for (int i = 0; i < 20; ++i) { mc::div<2>(acc2, x2, q2); x2[0] = acc2[0]; x2[1] = acc2[1]; acc2[0] = q2[0]; acc2[1] = q2[1]; }
  long long t8 = clock64();
  for (int i = 0; i < 20; ++i) { mc::div<3>(acc, x, q); x[0] = acc[0]; x[1] = acc[1]; x[2] = acc[2]; acc[0] = q[0]; acc[1] = q[1]; acc[2] = q[2]; }
  long long t9 = clock64();
  const double y3 = mc::recip_hint(x[0]);
  for (int i = 0; i < 20; ++i) { mc::div_y<3>(acc, x, y3, q); acc[0] = q[0]; acc[1] = q[1]; acc[2] = q[2]; }
  long long t10 = clock64();
  for (int i = 0; i < 20; ++i) { mc::recip<2>(acc2, q2); acc2[0] = q2[0]; acc2[1] = q2[1]; }
  long long t11 = clock64();
  for (int i = 0; i < 100; ++i) d = mc::ddiv_y(d, 1.37, 0.72992700729927);
  long long t12 = clock64();
  // full madd chain: the product's operand is the previous result
  double u3[3] = {0.5, 1e-18, 1e-35}, l3[3] = {-0.999, 1e-17, 0};
  for (int i = 0; i < 50; ++i) { double o3[3] = {u3[0] * 0 + 1.0, 1e-17, 0}; mc::madd<3>(o3, l3, u3); u3[0] = o3[0]; u3[1] = o3[1]; u3[2] = o3[2]; }
  long long t13 = clock64();
  double u2[2] = {0.5, 1e-18}, l2[2] = {-0.999, 1e-17};
  for (int i = 0; i < 50; ++i) { double o2[2] = {1.0, 1e-17}; mc::madd<2>(o2, l2, u2); u2[0] = o2[0]; u2[1] = o2[1]; }
  long long t14 = clock64();
  double w3[3] = {0.5, 1e-18, 1e-35}, m3[3];
  for (int i = 0; i < 50; ++i) { mc::mul<3>(w3, l3, m3); w3[0] = m3[0]; w3[1] = m3[1]; w3[2] = m3[2]; }
  long long t15 = clock64();
  out[threadIdx.x] = acc2[0] + acc2[1] + q[2] + acc[0] + d + u3[0] + u2[0] + w3[0];
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3;
    cyc[4] = t5 - t4; cyc[5] = t6 - t5; cyc[6] = t7 - t6; cyc[7] = t8 - t7; cyc[8] = t9 - t8;
    cyc[9] = t10 - t9; cyc[10] = t11 - t10; cyc[11] = t12 - t11; cyc[12] = t13 - t12; cyc[13] = t14 - t13; cyc[14] = t15 - t14;
  }
}

int main() {
  double *o; long long *c, h[32];
  cudaMalloc(&o, 1024); cudaMalloc(&c, 256);
  lat<<<1, 32>>>(o, c, 1e-20);
  lat<<<1, 32>>>(o, c, 1e-20);
  cudaMemcpy(h, c, 256, cudaMemcpyDeviceToHost);
  printf("DADD dep latency  %.1f cyc\n", h[0] / 1000.0);
  printf("DFMA dep latency  %.1f cyc\n", h[1] / 1000.0);
  printf("DDIV dep latency  %.1f cyc\n", h[2] / 100.0);
  printf("TD madd (acc-dep) %.1f cyc\n", h[3] / 100.0);
  printf("TD div            %.1f cyc\n", h[4] / 20.0);
  printf("DD madd (acc-dep) %.1f cyc\n", h[5] / 100.0);
  printf("DD div            %.1f cyc\n", h[6] / 20.0);
  printf("DD div (var b)    %.1f cyc\n", h[7] / 20.0);
  printf("TD div (var b)    %.1f cyc\n", h[8] / 20.0);
  printf("TD div_y (hinted) %.1f cyc\n", h[9] / 20.0);
  printf("DD recip (var b)  %.1f cyc\n", h[10] / 20.0);
  printf("ddiv_y dep        %.1f cyc\n", h[11] / 100.0);
  printf("TD madd (b-dep)   %.1f cyc\n", h[12] / 50.0);
  printf("DD madd (b-dep)   %.1f cyc\n", h[13] / 50.0);
  printf("TD mul dep        %.1f cyc\n", h[14] / 50.0);
  return 0;
}
