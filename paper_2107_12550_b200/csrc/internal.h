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
  PROF_GEMM, PROF_MATVEC, PROF_ELEMENTWISE, PROF_GEN, PROF_UPDATE_NEXT,
  PROF_NSLOTS
};
void prof_begin(int slot, cudaStream_t s);
void prof_end(int slot, cudaStream_t s);
bool prof_enabled();

// Shared scratch used by the panel factorisation (lu.cu).  The panel's CTAs
// exchange per-column pivot candidates through sequence-tagged 8-byte words
// (payload | seq, single-copy atomic), and pivot rows through plain stores
// published by a release word; parity double-buffering keeps a slow reader's
// step intact while fast CTAs publish the next one.
constexpr int LU_MAX_W = 32, LU_MAX_K = 4;
constexpr int LU_CAND_WORDS = 16;                    // idx, mag(2), pivot(2K)
constexpr int LU_ROW_WORDS = 2 * LU_MAX_W * LU_MAX_K;  // a panel row, 2/double
constexpr int LU_SWAP_LIST = 4 * LU_MAX_W + 1;         // one composed list
struct LuWork {
  unsigned long long *cand_words = nullptr;  // [2][G][LU_CAND_WORDS]
  unsigned long long *row_words = nullptr;   // [2][G][LU_ROW_WORDS]
  unsigned long long *rowj_words = nullptr;  // [2][LU_ROW_WORDS]
  // [0] sequence base of the current LU call, [1] its row count: a call's
  // words carry base + J + 1 + jj <= base + m + 1; the next call's base
  // is base + m + 2, and before the 32-bit sequence space would wrap the base
  // restarts at 0 with every word zeroed (lu_begin_kernel), so no stale
  // word of an earlier call can ever validate
  unsigned *epoch = nullptr;
  int32_t *status = nullptr;                 // [0] singular step (or -1)
  int32_t *swap_list = nullptr;  // [2 slots][64 cur | 64 src | count]
  int G = 0;                                 // max CTAs of the panel launch
  void *graphs = nullptr;                    // host-side graph cache
  cudaStream_t side = nullptr;   // high-priority stream: look-ahead panels
  cudaEvent_t ev_next = nullptr, ev_panel = nullptr;
  unsigned long long *trace = nullptr;       // diagnostics: [G][32][8] ns
  int trace_J = -1;                          // panel to trace (-1: none)
  unsigned poll_ns = 32;                     // back-off between polls
  cudaError_t init(int sms);
};

int num_sms();
// IR residual b - A x at long precision p <= 512 on the device (residual.cu):
// A row-major n x n, x, b, res length n, all as fixed-width long floats
// (longfloat.cuh lf::DF = the host's ff::F); variant 5 (production): the
// n^2 products in one kernel (two per warp, longseg.cuh), then a warp per
// row for the chain of adds; 2: the products on producer warps beside each
// row's chain; 0: a warp per row doing both (longwarp.cuh); 1: a thread
// per row (longfloat.cuh)
cudaError_t long_residual(int p, int n, const void *A, const void *x,
                          const void *b, void *res, cudaStream_t s,
                          int variant = 0);
// the IR's long -> short conversion (convert.cu), in row chunks: A (n x n
// lf::DF; rows [r0, r1) flat exact values in, rounded to p out, in place),
// their k heads into the planes (ld, plane), *d_bad when a head leaves the
// binary64 range and the largest head exponent (*d_emax); then the
// long_to_short_partials() per-block sums of the heads' squares scaled by
// 2^-emax
// A's exact values as uploaded when every mantissa fits 576 bits (80 B
// instead of lf::DF's 96): es = exponent * 4 + sign + 1
struct LongFlat9 {
  int64_t es;
  uint64_t m[9];
};
cudaError_t long_to_short_init(int *d_bad, int *d_emax, cudaStream_t s);
// in == null: A holds the flat values (lf::DF) and is converted in place;
// else in (LongFlat9, rows [r0, r1)) is converted into A
cudaError_t long_to_short_rows(int k, int n, int p, void *A, const void *in,
                               int r0, int r1, double *planes, int64_t ld,
                               int64_t plane, int *d_bad, int *d_emax,
                               cudaStream_t s);
cudaError_t long_to_short_stats(int n, const double *planes, int64_t ld,
                                const int *d_emax, double *d_partials,
                                cudaStream_t s);
int long_to_short_partials();
cudaError_t long_to_short_selftest(int k, int p, void *A, const void *in9,
                                   int64_t count, double *heads, int *ok,
                                   cudaStream_t s);
// diagnostics: per-panel kernel stamps into buf ([4 * n] u64) or off (null)
cudaError_t lu_stamps_enable(unsigned long long *buf);

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
// the recipe on the local columns of a column-block-cyclic layout
cudaError_t generate_cyclic(int k, MatView out, int rows, int local_cols,
                            int nb, int world, int rank, int slot, int64_t n,
                            uint64_t seed, cudaStream_t s);
// y = A x (mat_vec), A rows x cols
cudaError_t matvec(int k, int rows, int cols, MatView A, const double *x,
                   double *y, cudaStream_t s);
// C = fold_p add(C, mul(opA(A_ip), B_pj)); opA = -A when neg_a; C starts at
// 0 when zero_init
cudaError_t gemm(int k, bool neg_a, bool zero_init, int M, int N, int KK,
                 MatView A, MatView B, MatView C, cudaStream_t s);
// LU with partial pivoting in place of the m x ncols matrix A (ncols <= m;
// ncols < m factors a tall block, exchanging rows inside it only); swaps
// (device, ncols entries, row indices relative to A).  *sing_step = first
// singular step or -1.  nb = panel width (<= 32).
cudaError_t lu_factor(int k, int m, int ncols, MatView A, int32_t *d_swaps,
                      int nb, LuWork &w, int32_t *sing_step, cudaStream_t s);
// the same, stream-ordered only: no host synchronisation; the singular step
// (or -1) stays in w.status[0] on the device
cudaError_t lu_factor_async(int k, int m, int ncols, MatView A,
                            int32_t *d_swaps, int nb, LuWork &w,
                            cudaStream_t s);
// Scratch of the pipelined triangular solves: every final x_i is published
// as 2K self-validating words (32-bit payload | 32-bit sequence), [2K][rows].
struct SolveWork {
  unsigned long long *words = nullptr;
  int64_t cap = 0;           // rows
  unsigned seq = 0;
  unsigned long long *trace = nullptr;  // MPCORE_TRACE_SOLVE diagnostics
  int64_t trace_len = 0;
  cudaError_t ensure(int64_t rows);
  // a fresh sequence number for one sweep; on 32-bit wrap the words are
  // zeroed first (stream-ordered), so sequence 0 stays invalid and no
  // word of a sweep 2^32 calls ago can validate
  unsigned next_seq(cudaStream_t s) {
    if (++seq == 0) {
      cudaMemsetAsync(words, 0, (size_t)2 * LU_MAX_K * cap * sizeof(unsigned long long), s);
      seq = 1;
    }
    return seq;
  }
};
// x <- solve(LU, perm, b): x[i] = b[perm[i]] (the reference's swaps,
// composed), then forward and back substitution.  b and x must not alias.
cudaError_t lu_solve(int k, int n, MatView LU, const int32_t *d_perm,
                     const double *b, double *x, SolveWork &sw,
                     cudaStream_t s);

// back substitution only: x (planar k x n) holds L^-1 P b on entry (e.g.
// the right-hand-side column of an augmented LU) and x on exit
cudaError_t lu_solve_back(int k, int n, MatView LU, double *x, SolveWork &sw,
                          cudaStream_t s);

// panel pieces (exposed for the distributed driver)
cudaError_t lu_begin(LuWork &ws, int m, cudaStream_t s);
// factor panel [J, J+w); its composed row exchanges go to swap-list slot
cudaError_t lu_panel(int k, int n, MatView A, int J, int w, int32_t *d_swaps,
                     LuWork &ws, int slot, cudaStream_t s);
// row exchanges of the last factored panel (composed in ws.swap_list by the
// panel kernel) on columns [c0, c1) and [c2, c3)
cudaError_t lu_laswp(int k, MatView A, int c0, int c1, int c2, int c3,
                     const int32_t *swap_list, const int32_t *status,
                     cudaStream_t s);
cudaError_t lu_trsm(int k, MatView L11, MatView U12, int w, int ncols,
                    const int32_t *status, cudaStream_t s);
cudaError_t lu_update(int k, int M, int N, int w, MatView L21, MatView U12,
                      MatView A22, const int32_t *status, cudaStream_t s,
                      int prof_slot = PROF_UPDATE);

}  // namespace mpk
