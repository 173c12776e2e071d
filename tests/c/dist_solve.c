/* A plain C host of libmpcore's distributed LU + solve (include/mpcore.h):
 * one rank, NCCL communicator from a unique id, DD system of the config-4
 * recipe generated on the device, solved through mpcore_dist_lu_solve and
 * through the one-call mpcore_dev_solve_system; the two must agree bit for
 * bit (pivots and x).  Built and run by tests/test_gpu_c_host.py:
 *   gcc -O2 dist_solve.c -I include -L <pkg> -lmpcore -lcudart
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "mpcore.h"

#define CHECK(call)                                                    \
  do {                                                                 \
    int32_t st_ = (call);                                              \
    if (st_ != 0) {                                                    \
      char msg[256];                                                   \
      mpcore_last_error(msg, sizeof msg);                              \
      fprintf(stderr, "%s -> %d: %s\n", #call, st_, msg);              \
      return 1;                                                        \
    }                                                                  \
  } while (0)

int main(int argc, char **argv) {
  const int k = 2, n = argc > 1 ? atoi(argv[1]) : 512, nb = 256;
  const uint64_t seed = 210712554;
  const size_t ld = (size_t)n + 1, plane = (size_t)n * ld;
  double *A0, *A1, *ones, *b, *x1, *x2;
  if (cudaMalloc((void **)&A0, k * plane * 8) || cudaMalloc((void **)&A1, k * plane * 8) ||
      cudaMalloc((void **)&ones, k * (size_t)n * 8) || cudaMalloc((void **)&b, k * (size_t)n * 8) ||
      cudaMalloc((void **)&x1, k * (size_t)n * 8) || cudaMalloc((void **)&x2, k * (size_t)n * 8))
    return 2;
  cudaMemset(ones, 0, k * (size_t)n * 8);
  double *h1 = malloc((size_t)n * 8);
  for (int i = 0; i < n; ++i) h1[i] = 1.0;
  cudaMemcpy(ones, h1, (size_t)n * 8, cudaMemcpyHostToDevice);
  cudaDeviceSynchronize();
  /* A (n x n inside an n x (n+1) layout), b = A * ones in DD, b as column n */
  CHECK(mpcore_dev_generate_cyclic(k, (uint64_t)A0, ld, plane, n, n, nb, 1, 0,
                                   0, n, seed));
  CHECK(mpcore_dev_matvec(k, n, n, (uint64_t)A0, ld, plane, (uint64_t)ones,
                          (uint64_t)b));
  CHECK(mpcore_dev_copy2d(k, n, 1, (uint64_t)(A0 + n), ld, plane, (uint64_t)b,
                          1, n));
  CHECK(mpcore_dev_copy2d(k, n, n + 1, (uint64_t)A1, ld, plane, (uint64_t)A0,
                          ld, plane));
  /* the distributed driver, one rank, its own NCCL communicator */
  uint8_t id[128];
  uint64_t comm = 0;
  CHECK(mpcore_dist_unique_id(id, sizeof id));
  CHECK(mpcore_dist_comm_init(1, 0, id, sizeof id, &comm));
  int32_t rank = 0, cols = n + 1, step = -1;
  uint64_t base = (uint64_t)A0, xs = (uint64_t)x1;
  int64_t lds = (int64_t)ld, planes = (int64_t)plane, launches = 0;
  int32_t *sw1 = malloc((size_t)n * 4), *sw2 = malloc((size_t)n * 4);
  double phases[6];
  CHECK(mpcore_dist_lu_solve(comm, k, n, nb, 1, 1, &rank, &base, &lds, &planes,
                             &cols, &xs, 0, sw1, &step, phases, &launches));
  CHECK(mpcore_dist_comm_destroy(comm));
  /* the one-call LU + solve on the copy */
  CHECK(mpcore_dev_solve_system(k, n, (uint64_t)A1, ld, plane, 0, (uint64_t)x2,
                                sw2, &step));
  double *hx1 = malloc(k * (size_t)n * 8), *hx2 = malloc(k * (size_t)n * 8);
  cudaMemcpy(hx1, x1, k * (size_t)n * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(hx2, x2, k * (size_t)n * 8, cudaMemcpyDeviceToHost);
  double err = 0.0;
  for (int i = 0; i < n; ++i) err = fmax(err, fabs((hx1[i] - 1.0) + hx1[n + i]));
  const int same = memcmp(sw1, sw2, (size_t)n * 4) == 0 &&
                   memcmp(hx1, hx2, k * (size_t)n * 8) == 0;
  printf("n=%d dist %.3f ms (%lld launches) max|x-1| %.3g bitwise-vs-one-call %s\n",
         n, phases[0], (long long)launches, err, same ? "yes" : "NO");
  return same && err < 1e-20 ? 0 : 3;
}
