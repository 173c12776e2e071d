// Internal launch interface between the C-ABI layer (cabi.cu) and the
// sm_100a kernels.  All device matrices are planar: K planes, row-major in
// each plane, element (i, j) of plane c at base[c*plane + i*ld + j].
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace mpk {

struct MatView {
  double *p;       // element (0, 0) of plane 0
  int64_t ld;      // row stride (elements)
  int64_t plane;   // plane stride (elements)
};

// Kernel timing accumulator (CUDA events on the library stream).
enum ProfSlot {
  PROF_PANEL = 0, PROF_LASWP, PROF_TRSM, PROF_UPDATE, PROF_SOLVE,
  PROF_GEMM, PROF_MATVEC, PROF_ELEMENTWISE, PROF_GEN, PROF_NSLOTS
};
void prof_begin(int slot, cudaStream_t s);
void prof_end(int slot, cudaStream_t s);
bool prof_enabled();

// Shared scratch used by the panel factorisation.
struct LuWork {
  double *cand_rows = nullptr;    // [2][G][W*K]
  double *rowj = nullptr;         // [2][W*K]
  double *cand_mag = nullptr;     // [2][G]
  int32_t *cand_idx = nullptr;    // [2][G]
  unsigned *bar = nullptr;        // [0] count, [1] generation
  int32_t *status = nullptr;      // [0] singular step (or -1)
  int G = 0;                      // CTAs of the cooperative panel launch
  int cap_w = 0, cap_k = 0;
};

int num_sms();

// elementwise op: 0 add(x,y), 1 mul(x,y), 2 div(x,y); n lanes, planar
cudaError_t elementwise(int k, int op, int64_t n, const double *x,
                        const double *y, double *out, cudaStream_t s);
// y <- add(y, mul(x, alpha)); alpha: k host values
cudaError_t axpy(int k, int64_t n, const double *alpha, const double *x,
                 double *y, cudaStream_t s);
// seeded planar generator; count elements at flat offsets
// 0..count-1 of object `slot` in a size-n system; writes renormalised planes
// with plane stride `plane` (>= count)
cudaError_t generate(int k, double *out, int64_t count, int64_t plane,
                     int slot, int64_t n, uint64_t seed, cudaStream_t s);
// y = A x (mat_vec), A rows x cols
cudaError_t matvec(int k, int rows, int cols, MatView A, const double *x,
                   double *y, cudaStream_t s);
// C = fold_p add(C, mul(opA(A_ip), B_pj)); opA = -A when neg_a; C starts at
// 0 when zero_init
cudaError_t gemm(int k, bool neg_a, bool zero_init, int M, int N, int KK,
                 MatView A, MatView B, MatView C, cudaStream_t s);
// LU with partial pivoting in place; swaps (device, n entries).  Returns
// cudaSuccess; *sing_step = first singular step or -1.  nb = panel width.
cudaError_t lu_factor(int k, int n, MatView A, int32_t *d_swaps, int nb,
                      LuWork &w, int32_t *sing_step, cudaStream_t s);
// x (device, in: b) <- solve with LU factors and swaps
cudaError_t lu_solve(int k, int n, MatView LU, const int32_t *d_swaps,
                     double *x, cudaStream_t s);

// panel pieces (exposed for the distributed driver)
cudaError_t lu_panel(int k, int n, MatView A, int J, int w, int32_t *d_swaps,
                     LuWork &ws, cudaStream_t s);
cudaError_t lu_laswp(int k, int n, MatView A, int J, int w, int c0, int c1,
                     const int32_t *d_swaps, const int32_t *status,
                     cudaStream_t s);
cudaError_t lu_trsm(int k, MatView L11, MatView U12, int w, int ncols,
                    const int32_t *status, cudaStream_t s);
cudaError_t lu_update(int k, int M, int N, int w, MatView L21, MatView U12,
                      MatView A22, const int32_t *status, cudaStream_t s);

}  // namespace mpk
