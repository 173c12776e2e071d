// Host-side mixed-precision iterative refinement behind mpcore_refine
// (ffi.py:243-258 -> refine.py:121-197): .mpmat loading (matfile.py), the
// long-precision residual loop in correctly rounded big-float arithmetic
// (bignum.h; same single-rounding semantics as bigfloat.py), and the
// short-precision factor/solve on the GPU through ShortSolver.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <string>
#include <vector>

#include "bignum.h"

namespace mpr {

struct Report {
  int iterations = 0;
  std::string stop_reason = "max_iter";
  std::vector<bn::BF> residuals;   // residual 2-norm per iteration
  std::vector<bn::BF> solution;    // final x at long precision
  int64_t prec = 0;                // precision of residuals / solution
  // seconds: generate (config 3 only), convert, factor, refinement loop,
  // residuals (inside the loop), short solves (inside the loop)
  std::vector<double> timings;
};

// The short side: factor once, solve many (implemented on the GPU by
// cabi.cu).  Planes are k x n (vectors) / k x n x n (matrix), planar.
class ShortSolver {
 public:
  virtual ~ShortSolver() = default;
  // -> status (0 ok, 3 singular, 6 other)
  virtual int factor(int k, int n, const double *a_planes,
                     std::string &err) = 0;
  virtual int solve(const std::vector<double> &b_planes,
                    std::vector<double> &x_planes, std::string &err) = 0;
  // factor and the first solve in one call (a GPU solver carries b along
  // the factorisation); the same results as factor() + solve()
  virtual int factor_solve(int k, int n, const double *a_planes,
                           const std::vector<double> &b_planes,
                           std::vector<double> &x_planes, std::string &err) {
    const int st = factor(k, n, a_planes, err);
    return st ? st : solve(b_planes, x_planes, err);
  }
  // Optional, asynchronous form of factor_solve: begin enqueues the
  // factorisation and the first solve and returns (a_planes and b_planes
  // must stay valid until end); end waits and delivers x.  begin returning
  // -1 means "not supported" (the caller uses factor_solve).
  virtual int factor_solve_begin(int k, int n, const double *a_planes,
                                 const std::vector<double> &b_planes,
                                 std::string &err) { return -1; }
  virtual int factor_solve_end(std::vector<double> &x_planes,
                               std::string &err) { return 6; }
  // Optional: the long -> short conversion on the device (SURVEY §8(f)
  // row 2).  `flat` (staging slot 0, n x n ff::F) holds A's exact values
  // (un-normalised limbs); on return the device holds them rounded to p
  // (for the device residual) and their k binary64 heads (the planes of
  // the next factor_solve_begin, which then uploads only b), and *emax /
  // *hsum are the heads' largest exponent (INT_MIN: all zero) and sum of
  // squares scaled by 2^-2emax.  -> 0; 5 when a head leaves the binary64
  // range (convert on the host instead); other: error
  virtual bool device_convert_supported(int p) { return false; }
  // in row chunks: begin, then rows [r0, r1) of `flat` once the host has
  // written them (their upload and conversion overlap the host's next
  // chunk), then end
  // compact: `flat` holds mpk::LongFlat9 records (80 B, mantissas of at
  // most 576 bits) instead of ff::F ones
  virtual int device_convert_begin(int k, int n, int p, const void *flat,
                                   bool compact, std::string &err) {
    return 6;
  }
  virtual int device_convert_rows(int r0, int r1, std::string &err) {
    return 6;
  }
  virtual int device_convert_end(int *emax, double *hsum, std::string &err) {
    return 6;
  }
  // the device's rounded long A into host memory (n x n ff::F)
  virtual int download_long_A(void *dst, std::string &err) { return 6; }
  // Optional: the long residual b - A x on the device.
  // Values travel as fixed-width long floats (fastfloat.h ff::F, p <= 512).
  virtual bool residual_supported(int p) { return false; }
  // a host buffer of `bytes` the solver keeps (page-locked, reused across
  // calls), or null: slot 0 the fixed-width A, slot 1 the short planes
  virtual void *staging(int slot, size_t bytes) { return nullptr; }
  // A (n x n, row-major, in staging memory) and b; the upload may proceed
  // asynchronously, overlapping the factorisation
  virtual int residual_setup(int n, int p, const void *A, const void *b,
                             std::string &err) { return 6; }
  virtual int residual(const void *x, void *res, std::string &err) { return 6; }
};

// -> status (0 ok, 2 dims, 3 singular, 4 parse/file, 5 overflow, 6 other)
int refine_files(const char *a_path, const char *b_path, int short_k,
                 int long_bits, const char *rtol, const char *atol,
                 int max_iter, ShortSolver &short_side, Report &out,
                 std::string &err);

// the refinement loop on long-precision values already in memory (A
// row-major n x n, B length n); threads <= 0: all host threads
int refine_core(std::vector<bn::BF> &A, std::vector<bn::BF> &B, int n,
                int short_k, int long_bits, const char *rtol, const char *atol,
                int max_iter, int threads, ShortSolver &short_side, Report &out,
                std::string &err);

// the device conversion (convert.cu) against the host's ff::from_bf +
// to_multicomp on iters random values at precision p, k heads: mismatches
int64_t convert_selftest(int64_t iters, uint64_t seed, int p, int k,
                         cudaStream_t s);

// fastfloat.h against the generic big-integer path: mismatches over iters
// random operand pairs at precision p (-1: p out of the fixed-width range)
int64_t longfloat_selftest(int64_t iters, uint64_t seed, int p);

// the device long residual (residual.cu) against the host's on a random
// n x n system at precision p <= 512 (variant: see mpk::long_residual):
// mismatching rows, -1 on error
int64_t long_residual_selftest(int n, int p, uint64_t seed, cudaStream_t s,
                               int variant);

// bf_format_hex (bigfloat.py:524-537) and a .mpmat writer (matfile.py
// layout: header "mpmat rows cols bf bits", one row per line)
std::string format_hex(const bn::BF &v);
int write_mpmat(const char *path, const std::vector<bn::BF> &vals, int rows,
                int cols, int64_t bits, std::string &err);

// bf_format_decimal (bigfloat.py:483-509); digits <= 0: the default for prec
std::string format_decimal(const bn::BF &v, int digits, int64_t prec);

// correctly rounded long arithmetic at precision p (bigfloat.py:239-326)
bn::BF lf_add(const bn::BF &a, const bn::BF &b, int64_t p);
bn::BF lf_sub(const bn::BF &a, const bn::BF &b, int64_t p);
bn::BF lf_mul(const bn::BF &a, const bn::BF &b, int64_t p);
bn::BF lf_div(const bn::BF &a, const bn::BF &b, int64_t p);
bn::BF lf_sqrt(const bn::BF &a, int64_t p);
bn::BF lf_round(const bn::BF &a, int64_t p);
int lf_cmp(const bn::BF &a, const bn::BF &b);

}  // namespace mpr
