// Minimal unsigned big integer + exact binary-float helpers for the C-ABI's
// text paths.  Mirrors the rounding rules of the reference's BigFloat
// (/root/reference/pkg/src/mpcore/bigfloat.py): _round_to (RNE to p bits,
// 172-187), _round_ratio (p+2 quotient bits + sticky, 263-273),
// bf_to_binary64 (RNE to 53 bits then ldexp, 375-387) and bf_to_multicomp
// (peel k rounded heads, 419-432).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace bn {

struct UBig {
  std::vector<uint32_t> w;  // little-endian limbs, no leading zero limbs

  UBig() = default;
  explicit UBig(uint64_t v) {
    while (v) { w.push_back((uint32_t)v); v >>= 32; }
  }
  bool zero() const { return w.empty(); }
  void trim() { while (!w.empty() && w.back() == 0) w.pop_back(); }
  int64_t bits() const;
  bool bit(int64_t i) const;
  bool low_bits_nonzero(int64_t nbits) const;  // any of bits [0, nbits) set
  void mul_small(uint32_t m);
  void add_small(uint32_t a);
  UBig shl(int64_t s) const;
  UBig shr(int64_t s) const;
  uint64_t low64() const;
  static int cmp(const UBig &a, const UBig &b);
  static UBig add(const UBig &a, const UBig &b);
  static UBig sub(const UBig &a, const UBig &b);  // requires a >= b
  static UBig mul(const UBig &a, const UBig &b);
  static void divmod(const UBig &a, const UBig &b, UBig &q, UBig &r);
  static UBig isqrt(const UBig &a);
  static UBig pow10(int64_t e);
  std::string to_dec() const;
};

// sign * man * 2^exp  (sign 0 => zero)
struct BF {
  int sign = 0;
  UBig man;
  int64_t exp = 0;
};

// Round man*2^exp to p bits, half to even (bigfloat.py:_round_to).
void round_to(UBig &man, int64_t &exp, int64_t p);
BF mk(int sign, UBig man, int64_t exp, int64_t p);            // _mk
BF round_ratio(int sign, const UBig &num, const UBig &den, int64_t exp,
               int64_t p);                                    // _round_ratio
BF add_exact(const BF &a, const BF &b);
BF neg(const BF &a);

// status: 0 ok, 4 parse error, 5 overflow
int parse_decimal(const std::string &text, int64_t p, BF &out);
int parse_hex(const std::string &text, BF &out);
// Nearest binary64 (RNE); returns 5 on overflow.
int to_binary64(const BF &a, double &out);
BF from_binary64(double x);
// Peel k heads (bf_to_multicomp). Returns 0 or 5 (overflow).
int to_multicomp(const BF &a, int k, double *out);

}  // namespace bn
