// BASELINE config 3 test system (testsys.cpp).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "bignum.h"

namespace mpr {

// A = U diag(σ) W (n x n, row-major) and b = A * ones, entries rounded to
// long_bits; σ geometric from 1 to 10^-kappa_exp10.  threads <= 0: all host
// threads.  -> status (0 ok, 2 bad n)
int config3_system(int n, uint64_t seed, int64_t long_bits, double kappa_exp10,
                   int threads, std::vector<bn::BF> &A, std::vector<bn::BF> &b,
                   std::string &err);

}  // namespace mpr
