// Host-side mixed-precision iterative refinement behind mpcore_refine
// (ffi.py:243-258 -> refine.py:121-197): .mpmat loading (matfile.py), the
// long-precision residual loop in correctly rounded big-float arithmetic, and
// the short-precision factor/solve on the GPU.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "bignum.h"

namespace mpr {

struct Report {
  int iterations = 0;
  std::string stop_reason = "max_iter";
  std::vector<bn::BF> residuals;   // residual 2-norm per iteration
  std::vector<bn::BF> solution;    // final x at long precision
  int64_t prec = 0;
};

// -> status (0 ok, 2 dims, 3 singular, 4 parse/file, 5 overflow, 6 other)
int refine_files(const char *a_path, const char *b_path, int short_k,
                 int long_bits, const char *rtol, const char *atol,
                 int max_iter, Report &out, std::string &err);

// bf_format_decimal (bigfloat.py:483-509); digits <= 0 = default for prec
std::string format_decimal(const bn::BF &v, int digits, int64_t prec = 0);

}  // namespace mpr
