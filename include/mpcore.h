/*
 * libmpcore — B200-native (sm_100a) DD/TD/QD dense direct solver, C ABI.
 *
 * Drop-in for the reference's C-ABI shared library
 * (/root/reference/pkg/src/mpcore/build_lib.py:31-57, behaviour in
 * /root/reference/pkg/src/mpcore/ffi.py).  The first 16 entry points below
 * are the reference's exported symbols with identical prototypes, status
 * codes and handle semantics; the rest are extensions (bulk planar I/O,
 * products, device generator, profiling, distributed LU) that a foreign host
 * needs to move n = 2048 .. 32768 systems, which the reference's
 * one-element-at-a-time text interface cannot do.
 *
 * Conventions (ffi.py:1-21, build_lib.py:70-101):
 *   - every function returns an int32 status:
 *       0 ok, 1 invalid handle (unknown, released or wrong kind),
 *       2 dimension/argument mismatch, NULL out-pointer or truncated buffer,
 *       3 singular matrix, 4 parse / file error, 5 arithmetic overflow,
 *       6 internal error (CUDA failure, or a concurrent mutation of the same
 *         object: mutators latch their target).
 *   - handles are sequential uint64 ids < 2^53 and are never reused;
 *   - text crosses as NUL-terminated ASCII in caller-owned buffers,
 *     truncated with status 2 when the buffer is too small;
 *   - nothing unwinds across the boundary; no callbacks.
 *   - planar layout: a k-component rows x cols object is k planes of
 *     rows*cols binary64, row-major within each plane (simd.py:36-48).
 * Objects live in device (HBM) memory; there is no CPU fallback: without a
 * usable CUDA device every compute entry point returns 6 and
 * mpcore_last_error() says why.
 */
#ifndef MPCORE_H
#define MPCORE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPCORE_OK 0
#define MPCORE_BAD_HANDLE 1
#define MPCORE_BAD_DIMENSION 2
#define MPCORE_SINGULAR 3
#define MPCORE_BAD_PARSE 4
#define MPCORE_OVERFLOW 5
#define MPCORE_INTERNAL 6

/* ---- reference ABI (build_lib.py:31-57) -------------------------------- */

/* build_lib.py:32 / ffi.py:127 */
int32_t mpcore_version(char *out, int32_t cap);
/* build_lib.py:33 / ffi.py:131.  Mirrors MPCORE_SIMD (simd.py:17-28); the
 * device path is the only execution path, so it selects nothing. */
int32_t mpcore_simd_enabled(void);
/* build_lib.py:34-35 / ffi.py:135-141: zero-filled k-component matrix */
int32_t mpcore_matrix_new(int32_t k, int32_t rows, int32_t cols,
                          uint64_t *out);
/* build_lib.py:36 / ffi.py:144-149 */
int32_t mpcore_vector_new(int32_t k, int32_t n, uint64_t *out);
/* build_lib.py:37 / ffi.py:152-154 */
int32_t mpcore_release(uint64_t h);
/* build_lib.py:38-39 / ffi.py:167-186: decimal (rounded to 53k+64 bits,
 * then to k components) or exact hex-float text; vectors use (i, 0) */
int32_t mpcore_set_element_from_decimal(uint64_t h, int32_t i, int32_t j,
                                        const char *text);
/* build_lib.py:40-41 / ffi.py:189-197 */
int32_t mpcore_get_element_components(uint64_t h, int32_t i, int32_t j,
                                      double *out, int32_t cap);
/* build_lib.py:42 / ffi.py:203-214: in-place P*A = L*U on the GPU; on a
 * singular matrix returns 3 and writes 0 to *piv_out */
int32_t mpcore_lu_factor(uint64_t h, uint64_t *piv_out);
/* build_lib.py:43-44 / ffi.py:217-240: x <- solve(LU, piv, b) on the GPU */
int32_t mpcore_lu_solve(uint64_t lu_h, uint64_t piv_h, uint64_t b_h,
                        uint64_t x_h);
/* build_lib.py:45-48 / ffi.py:243-258: load .mpmat system, run the
 * mixed-precision iterative refinement, return a report handle */
int32_t mpcore_refine(const char *a_path, const char *b_path,
                      int32_t short_k, int32_t long_bits, const char *rtol,
                      const char *atol, int32_t max_iter,
                      uint64_t *report_out);
/* build_lib.py:49-56 / ffi.py:266-306 */
int32_t mpcore_report_iterations(uint64_t h, int32_t *out);
int32_t mpcore_report_stop_reason(uint64_t h, char *out, int32_t cap);
int32_t mpcore_report_residual_count(uint64_t h, int32_t *out);
int32_t mpcore_report_residual_entry(uint64_t h, int32_t idx,
                                     int32_t digits, char *out, int32_t cap);
int32_t mpcore_report_solution_count(uint64_t h, int32_t *out);
int32_t mpcore_report_solution_entry(uint64_t h, int32_t idx,
                                     int32_t digits, char *out, int32_t cap);

/* ---- extension: one-call solve ----------------------------------------
 * x = A^-1 b with A's factors left in A and the pivot record returned, as
 * mpcore_lu_factor + mpcore_lu_solve do (bit for bit); b rides along as an
 * extra column of the factorisation (its exchanges and updates are the
 * forward substitution, element by element in the reference's order), so
 * only the back substitution runs after the LU.  nb <= 0: default. */
int32_t mpcore_solve_system(uint64_t a_h, uint64_t b_h, uint64_t x_h,
                            int32_t nb, uint64_t *piv_out,
                            int32_t *singular_step);
/* the same on a caller-owned augmented device matrix [A | b] (k planes of
 * n x ld, ld >= n+1, b in column n): factors in place, x (k x n planar)
 * out, swaps_out (n entries, may be NULL) */
int32_t mpcore_dev_solve_system(int32_t k, int32_t n, uint64_t aug,
                                int64_t ld, int64_t plane, int32_t nb,
                                uint64_t x, int32_t *swaps_out,
                                int32_t *singular_step);

/* ---- extension: BASELINE config 3 (TD-mpmath IR, n = 1024, κ = 1e30) ---
 * Builds A = U diag(σ) W (σ geometric 1 .. 10^-kappa_exp10, U, W seeded
 * butterfly-orthogonal at 576-bit fixed point) and b = A ones at long_bits
 * on the host (threads <= 0: all), then runs the mpcore_refine loop on it
 * (short side on the GPU).  Returns a report handle as mpcore_refine does. */
int32_t mpcore_refine_config3(int32_t n, uint64_t seed, double kappa_exp10,
                              int32_t short_k, int32_t long_bits,
                              const char *rtol, const char *atol,
                              int32_t max_iter, int32_t threads,
                              uint64_t *report_out);
/* the same system written as .mpmat files (BigFloat hex, matfile.py
 * layout) for mpcore_refine or the reference's own driver; host only */
int32_t mpcore_write_config3(int32_t n, uint64_t seed, double kappa_exp10,
                             int32_t long_bits, int32_t threads,
                             const char *a_path, const char *b_path);
/* seconds: [generate, convert, factor, refinement loop, residuals, solves]
 * (generate only for mpcore_refine_config3; mpcore_refine reports 5) */
int32_t mpcore_report_timings(uint64_t h, double *out, int32_t cap,
                              int32_t *count);

/* ---- extensions: object introspection and bulk planar transfer --------- */

/* kind: 1 matrix, 2 vector, 3 pivot record, 4 report */
int32_t mpcore_object_info(uint64_t h, int32_t *kind, int32_t *k,
                           int32_t *rows, int32_t *cols);
/* host planar (k*rows*cols doubles) -> device object; count must match */
int32_t mpcore_set_planes(uint64_t h, const double *planes, int64_t count);
/* device object -> host planar; cap in doubles */
/* Asynchronous mpcore_set_planes: the copy runs on its own stream and
   overlaps the library's computation; every later call that touches the
   device is ordered after it.  `planes` (page-locked for a truly
   asynchronous copy) must stay unchanged until such a call returns.
   Extension (pipelined solves). */
int32_t mpcore_set_planes_async(uint64_t h, const double *planes,
                                int64_t count);
int32_t mpcore_get_planes(uint64_t h, double *out, int64_t cap);
/* Asynchronous mpcore_get_planes: on the copy stream, after the library's
   queued work on the object; `out` (page-locked for a truly asynchronous
   copy) is valid after mpcore_sync.  Later writes to the object wait for
   the copy.  Extension (pipelined products). */
int32_t mpcore_get_planes_async(uint64_t h, double *out, int64_t cap);
/* device-to-device copy between objects of identical shape */
int32_t mpcore_copy(uint64_t src, uint64_t dst);
/* pivot record from a host swap list (PivotRecord(swaps), linalg.py:348-366) */
int32_t mpcore_pivot_new(int32_t n, const int32_t *swaps, uint64_t *out);
/* swaps[j] = r, 0-based (linalg.py:348-354) */
int32_t mpcore_pivot_get(uint64_t h, int32_t *out, int32_t cap);
/* page-locked host buffers for fast H2D/D2H of planes */
int32_t mpcore_host_alloc(int64_t bytes, void **out);
int32_t mpcore_host_free(void *p);

/* ---- extensions: compute entry points ---------------------------------- */

/* lu_factor with explicit panel width (0 = default) and the singular step
 * (SingularMatrixError.step, errors.py:21-30; -1 when nonsingular) */
int32_t mpcore_lu_factor_ex(uint64_t h, int32_t nb, uint64_t *piv_out,
                            int32_t *singular_step);
/* C = A*B, mat_mul_blocked (linalg.py:577-617); C must be A.rows x B.cols */
int32_t mpcore_mat_mul(uint64_t a, uint64_t b, uint64_t c);
/* y = A*x, mat_vec (linalg.py:545-574) */
int32_t mpcore_mat_vec(uint64_t a, uint64_t x, uint64_t y);
/* out = x op y elementwise: op 0 add, 1 mul (linalg.py:648-673), 2 div
 * (mcfloat.py:304-318; a zero divisor head returns 6), 3 sqrt of x
 * (_sqrt_t, mcfloat.py:324-340; y is not read; a negative head returns 6) */
int32_t mpcore_elementwise(int32_t op, uint64_t x, uint64_t y, uint64_t out);
/* y <- y + x*alpha (axpy_batch, linalg.py:624-645); alpha: k doubles */
int32_t mpcore_axpy(const double *alpha, int32_t k, uint64_t x, uint64_t y);
/* fill a matrix/vector with the seeded planar recipe:
 * slot 0 = A, 1 = B, 2 = x of a size-system_n system, seed S */
int32_t mpcore_generate(uint64_t h, int32_t slot, int64_t system_n,
                        uint64_t seed);

/* ---- extensions: one-shot host-buffer entry points (paper names:
 * DD/TD/QD LUdecompPM and SolveDD/TD/QDLSPM) ---------- */

/* factor host planar a (k*n*n, in place) -> swaps (n int32) */
int32_t mpcore_lu_decomp_pm(int32_t k, int32_t n, double *a_planes,
                            int32_t *swaps, int32_t *singular_step);
/* solve with host factors/swaps/b -> host x (k*n) */
int32_t mpcore_solve_ls_pm(int32_t k, int32_t n, const double *lu_planes,
                           const int32_t *swaps, const double *b_planes,
                           double *x_planes);

/* ---- extensions: device-pointer building blocks (expert) ---------------
 * For hosts that lay out and move device memory themselves -- the
 * column-block-cyclic distributed LU (paper_2107_12550_b200/dist.py).
 * Pointers are device addresses of planar views (base, ld, plane stride,
 * all in elements); they are not checked beyond NULL. */

/* device address of a matrix/vector object's planes */
int32_t mpcore_object_device_ptr(uint64_t h, uint64_t *ptr);
/* in-place LU with partial pivoting of an m x ncols block (ncols <= m):
 * pivots over all m rows, exchanges rows inside the block only; swaps_out
 * (host, ncols) are row indices relative to the block (linalg.py:422-449) */
int32_t mpcore_dev_lu_block(int32_t k, int32_t m, int32_t ncols, uint64_t base,
                            int64_t ld, int64_t plane, int32_t nb,
                            int32_t *swaps_out, int32_t *singular_step);
/* row exchanges (row0+i) <-> swaps[i], i ascending, on columns
 * [col0, col0+ncols) of the view (linalg.py:430-431) */
int32_t mpcore_dev_laswp(int32_t k, uint64_t base, int64_t ld, int64_t plane,
                         int32_t col0, int32_t ncols, int32_t row0,
                         const int32_t *swaps, int32_t nswaps);
/* U <- L11^-1 U for unit-lower L11 (w x w) and U (w x ncols), each element
 * continuing its chain add(u, mul(-l, u')) in ascending order */
int32_t mpcore_dev_trsm(int32_t k, int32_t w, int32_t ncols, uint64_t l11,
                        int64_t ldl, int64_t planel, uint64_t u12, int64_t ldu,
                        int64_t planeu);
/* C <- fold_p add(C, mul(opA(A_ip), B_pj)), opA = -A if neg_a, C from 0 if
 * zero_init (linalg.py:577-617 and the LU trailing update) */
int32_t mpcore_dev_gemm(int32_t k, int32_t neg_a, int32_t zero_init, int32_t M,
                        int32_t N, int32_t Kd, uint64_t a, int64_t lda,
                        int64_t pa, uint64_t b, int64_t ldb, int64_t pb,
                        uint64_t c, int64_t ldc, int64_t pc);
/* strided rows x cols copy of every plane */
int32_t mpcore_dev_copy2d(int32_t k, int32_t rows, int32_t cols, uint64_t dst,
                          int64_t ldd, int64_t pd, uint64_t src, int64_t lds,
                          int64_t ps);
/* x <- solve(LU, swaps, b) for device LU (n x n view), host swaps (n),
 * device b and x (k*n, planar, not aliased) (linalg.py:496-538) */
int32_t mpcore_dev_lu_solve(int32_t k, int32_t n, uint64_t lu, int64_t ld,
                            int64_t plane, const int32_t *swaps, uint64_t b,
                            uint64_t x);
/* y <- A x (mat_vec, linalg.py:545-574) on device views; x, y planar k*n */
int32_t mpcore_dev_matvec(int32_t k, int32_t rows, int32_t cols, uint64_t a,
                          int64_t ld, int64_t plane, uint64_t x, uint64_t y);
/* the seeded recipe on the local columns of a column-block-cyclic layout */
int32_t mpcore_dev_generate_cyclic(int32_t k, uint64_t base, int64_t ld,
                                   int64_t plane, int32_t rows,
                                   int32_t local_cols, int32_t nb,
                                   int32_t world, int32_t rank, int32_t slot,
                                   int64_t system_n, uint64_t seed);

/* ---- extensions: the distributed LU + solve (BASELINE config 4) --------
 * One process per GPU.  Rank 0 draws an NCCL unique id (128 bytes) and the
 * host shares it over its own channel (torch.distributed, MPI, a file);
 * every rank then creates its communicator.  libnccl.so.2 is loaded on
 * first use (the copy already in the process if any, else MPCORE_NCCL_LIB,
 * else the loader's); without it these calls return 6. */
int32_t mpcore_dist_unique_id(uint8_t *out, int32_t cap);
int32_t mpcore_dist_comm_init(int32_t world, int32_t rank, const uint8_t *id,
                              int32_t len, uint64_t *comm_out);
int32_t mpcore_dist_comm_destroy(uint64_t comm);
/* Factor A (n x n, column-block-cyclic: block b of nb columns on rank
 * b % world) with partial pivoting and solve A x = b, stream-ordered on the
 * device (linalg.py:422-538 per element; pivots, factors and x bitwise the
 * one-GPU result).  comm = a communicator (this process serves one rank,
 * nlocal = 1) or 0 (this process serves every rank of the world on its
 * device: nlocal = world, broadcasts become device copies).  Per served
 * rank i: ranks[i], the local matrix at bases[i] (lds[i], planes[i]) with
 * cols[i] = its local column count + 1, the last column holding b on
 * entry (y = L^-1 P b on exit), and xs[i] (device, k*n planar) for x.
 * The work starts after `stream`'s queued work (0: the library stream; 1:
 * cudaStreamLegacy) and that stream waits for its end.  swaps_out (host, n) = PivotRecord.swaps;
 * phase_ms (6, optional, one served rank only): total, tall-block factor +
 * pack, broadcasts, exchanges + U12, trailing update, back substitution;
 * launches (optional): kernels + collectives enqueued.  3 = singular. */
int32_t mpcore_dist_lu_solve(uint64_t comm, int32_t k, int32_t n, int32_t nb,
                             int32_t world, int32_t nlocal,
                             const int32_t *ranks, const uint64_t *bases,
                             const int64_t *lds, const int64_t *planes,
                             const int32_t *cols, const uint64_t *xs,
                             uint64_t stream, int32_t *swaps_out,
                             int32_t *singular_step, double *phase_ms,
                             int64_t *launches);

/* ---- extensions: device, diagnostics, profiling ------------------------ */

/* debug (the substitute for compute-sanitizer memcheck, which this pool
 * does not allow): with MPCORE_DEBUG_GUARD=1 in the environment when an
 * object is created, its planes sit between two 64 KiB guard zones filled
 * with 0xA5; this checks every live guarded object: *checked of them,
 * *bad with a written zone */
int32_t mpcore_debug_check_guards(int64_t *checked, int64_t *bad);
/* selftest: the GPU long -> short conversion of the refinement driver
 * (round to prec bits, k binary64 heads) against the host's on iters
 * random values; *mismatches = values differing in any bit */
int32_t mpcore_debug_convert_selftest(int64_t iters, uint64_t seed,
                                      int32_t prec, int32_t k,
                                      int64_t *mismatches);

/* select the CUDA device for this process (before any other call) */
int32_t mpcore_set_device(int32_t device);
int32_t mpcore_device_name(char *out, int32_t cap);
int32_t mpcore_sm_count(int32_t *out);
/* last error text of the calling thread */
int32_t mpcore_last_error(char *out, int32_t cap);
/* wait for all device work of the library stream */
int32_t mpcore_sync(void);
/* per-kernel-family CUDA-event timing on the library stream:
 * slots 0 panel, 1 laswp, 2 trsm, 3 trailing update, 4 solve, 5 gemm,
 * 6 mat_vec, 7 elementwise, 8 generator, 9 the look-ahead's next-panel
 * update (the rest of the trailing update is slot 3) */
int32_t mpcore_prof_enable(int32_t on);
int32_t mpcore_prof_reset(void);
int32_t mpcore_prof_read(double *ms, int64_t *launches, int32_t cap);
/* diagnostics: per-CTA, per-column phase timestamps (ns) of the panel
 * selected by the MPCORE_TRACE_PANEL environment variable; [SMs][32][8] */
int32_t mpcore_debug_panel_trace(uint64_t *out_ns, int64_t cap);
/* Diagnostics: per-panel kernel entry/exit stamps (globaltimer ns) of the
   next LUs.  out == NULL arms / resets a len-entry buffer (4 per column
   index J: panel entry, panel exit, exchange+U12 entry, exit); otherwise
   copies len entries to out.  Extension (no reference counterpart). */
int32_t mpcore_debug_lu_stamps(int64_t len, uint64_t *out);
/* Device timing on the library's stream (all compute and copies run there):
   record CUDA event `slot` (0..7); elapsed milliseconds from slot a to slot
   b (waits for b).  Extension (bench.py). */
int32_t mpcore_stream_event_record(int32_t slot);
int32_t mpcore_stream_event_elapsed(int32_t a, int32_t b, double *ms);
/* diagnostics: owner timestamps (ns) of every row block of the last solve
 * (MPCORE_TRACE_SOLVE set): [forward, backward][blocks][4] = start, completed
 * source blocks added, critical source block done, diagonal done */
int32_t mpcore_debug_solve_trace(uint64_t *out_ns, int64_t cap);
/* diagnostics: the refinement loop's fixed-width long arithmetic against
 * the generic big-integer path on random operands at precision prec
 * (<= 640); host only */
/* Diagnostics: the device long residual b - A x
   against the host's on a random n x n system at precision prec <= 512
   (variant 0: warp per row, the production kernel; 1: thread per row);
   mismatching rows in *mismatches.  Extension. */
int32_t mpcore_debug_long_residual_selftest(int32_t n, int32_t prec,
                                            uint64_t seed, int32_t variant,
                                            int64_t *mismatches);
int32_t mpcore_debug_longfloat_selftest(int64_t iters, uint64_t seed,
                                        int32_t prec, int64_t *mismatches);
/* diagnostics: timeline of the profiled launches since mpcore_prof_reset,
 * (slot, start us, end us) per launch in enqueue order */
int32_t mpcore_debug_timeline(double *out, int64_t cap, int64_t *count);
/* FP64 issue-rate microbenchmark: DADD instructions per second */
int32_t mpcore_fp64_peak(double *dadd_per_s, double *dfma_per_s);

#ifdef __cplusplus
}
#endif
#endif /* MPCORE_H */
