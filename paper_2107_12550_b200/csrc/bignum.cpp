// Exact big-integer helpers for the C-ABI text paths (see bignum.h).
#include "bignum.h"

#include <algorithm>
#include <cctype>
#include <cmath>

namespace bn {

int64_t UBig::bits() const {
  if (w.empty()) return 0;
  return 32 * (int64_t)(w.size() - 1) + (32 - __builtin_clz(w.back()));
}

bool UBig::bit(int64_t i) const {
  size_t l = (size_t)(i / 32);
  if (i < 0 || l >= w.size()) return false;
  return (w[l] >> (i % 32)) & 1u;
}

bool UBig::low_bits_nonzero(int64_t nbits) const {
  if (nbits <= 0) return false;
  size_t full = (size_t)(nbits / 32);
  for (size_t l = 0; l < full && l < w.size(); ++l)
    if (w[l]) return true;
  int rem = (int)(nbits % 32);
  if (rem && full < w.size()) return (w[full] & ((1u << rem) - 1u)) != 0;
  return false;
}

void UBig::mul_small(uint32_t m) {
  uint64_t carry = 0;
  for (auto &x : w) {
    uint64_t t = (uint64_t)x * m + carry;
    x = (uint32_t)t;
    carry = t >> 32;
  }
  if (carry) w.push_back((uint32_t)carry);
  trim();
}

void UBig::add_small(uint32_t a) {
  uint64_t carry = a;
  for (size_t i = 0; i < w.size() && carry; ++i) {
    uint64_t t = (uint64_t)w[i] + carry;
    w[i] = (uint32_t)t;
    carry = t >> 32;
  }
  if (carry) w.push_back((uint32_t)carry);
}

UBig UBig::shl(int64_t s) const {
  if (zero() || s == 0) return *this;
  UBig r;
  size_t limbs = (size_t)(s / 32);
  int b = (int)(s % 32);
  r.w.assign(limbs, 0u);
  uint32_t carry = 0;
  for (uint32_t x : w) {
    if (b) {
      r.w.push_back((x << b) | carry);
      carry = x >> (32 - b);
    } else {
      r.w.push_back(x);
    }
  }
  if (carry) r.w.push_back(carry);
  r.trim();
  return r;
}

UBig UBig::shr(int64_t s) const {
  if (s <= 0) return *this;
  size_t limbs = (size_t)(s / 32);
  if (limbs >= w.size()) return UBig();
  int b = (int)(s % 32);
  UBig r;
  r.w.resize(w.size() - limbs);
  for (size_t i = 0; i < r.w.size(); ++i) {
    uint64_t lo = w[i + limbs];
    uint64_t hi = (i + limbs + 1 < w.size()) ? w[i + limbs + 1] : 0;
    r.w[i] = (uint32_t)(((hi << 32) | lo) >> b);
  }
  r.trim();
  return r;
}

uint64_t UBig::low64() const {
  uint64_t v = 0;
  if (w.size() > 0) v |= w[0];
  if (w.size() > 1) v |= (uint64_t)w[1] << 32;
  return v;
}

int UBig::cmp(const UBig &a, const UBig &b) {
  if (a.w.size() != b.w.size()) return a.w.size() < b.w.size() ? -1 : 1;
  for (size_t i = a.w.size(); i-- > 0;)
    if (a.w[i] != b.w[i]) return a.w[i] < b.w[i] ? -1 : 1;
  return 0;
}

UBig UBig::add(const UBig &a, const UBig &b) {
  UBig r;
  size_t n = std::max(a.w.size(), b.w.size());
  r.w.resize(n);
  uint64_t carry = 0;
  for (size_t i = 0; i < n; ++i) {
    uint64_t t = carry;
    if (i < a.w.size()) t += a.w[i];
    if (i < b.w.size()) t += b.w[i];
    r.w[i] = (uint32_t)t;
    carry = t >> 32;
  }
  if (carry) r.w.push_back((uint32_t)carry);
  return r;
}

UBig UBig::sub(const UBig &a, const UBig &b) {
  UBig r;
  r.w.resize(a.w.size());
  int64_t borrow = 0;
  for (size_t i = 0; i < a.w.size(); ++i) {
    int64_t t = (int64_t)a.w[i] - borrow - (i < b.w.size() ? (int64_t)b.w[i] : 0);
    borrow = t < 0;
    if (t < 0) t += ((int64_t)1 << 32);
    r.w[i] = (uint32_t)t;
  }
  r.trim();
  return r;
}

UBig UBig::mul(const UBig &a, const UBig &b) {
  if (a.zero() || b.zero()) return UBig();
  std::vector<uint64_t> acc(a.w.size() + b.w.size() + 1, 0);
  UBig r;
  r.w.assign(a.w.size() + b.w.size(), 0u);
  for (size_t i = 0; i < a.w.size(); ++i) {
    uint64_t carry = 0;
    for (size_t j = 0; j < b.w.size(); ++j) {
      uint64_t t = (uint64_t)a.w[i] * b.w[j] + r.w[i + j] + carry;
      r.w[i + j] = (uint32_t)t;
      carry = t >> 32;
    }
    size_t k = i + b.w.size();
    while (carry) {
      uint64_t t = (uint64_t)r.w[k] + carry;
      r.w[k] = (uint32_t)t;
      carry = t >> 32;
      ++k;
    }
  }
  r.trim();
  return r;
}

// Schoolbook long division on 32-bit limbs (Knuth's Algorithm D: normalise
// the divisor's top bit, estimate each quotient limb from the top two limbs
// and correct at most twice, multiply-subtract, add back on a borrow).
void UBig::divmod(const UBig &a, const UBig &b, UBig &q, UBig &r) {
  q = UBig();
  r = UBig();
  if (b.zero() || cmp(a, b) < 0) {  // (division by zero: callers exclude it)
    r = a;
    return;
  }
  const size_t n = b.w.size(), na = a.w.size();
  if (n == 1) {
    const uint64_t d = b.w[0];
    uint64_t rem = 0;
    q.w.assign(na, 0u);
    for (size_t i = na; i-- > 0;) {
      const uint64_t cur = (rem << 32) | a.w[i];
      q.w[i] = (uint32_t)(cur / d);
      rem = cur % d;
    }
    q.trim();
    r = UBig(rem);
    return;
  }
  const int s = __builtin_clz(b.w[n - 1]);
  std::vector<uint32_t> vn(n), un(na + 1);
  for (size_t i = n - 1; i > 0; --i)
    vn[i] = (b.w[i] << s) | (s ? (uint32_t)((uint64_t)b.w[i - 1] >> (32 - s)) : 0u);
  vn[0] = b.w[0] << s;
  un[na] = s ? (uint32_t)((uint64_t)a.w[na - 1] >> (32 - s)) : 0u;
  for (size_t i = na - 1; i > 0; --i)
    un[i] = (a.w[i] << s) | (s ? (uint32_t)((uint64_t)a.w[i - 1] >> (32 - s)) : 0u);
  un[0] = a.w[0] << s;
  const uint64_t B = 1ull << 32;
  q.w.assign(na - n + 1, 0u);
  for (size_t j = na - n + 1; j-- > 0;) {
    const uint64_t num = ((uint64_t)un[j + n] << 32) | un[j + n - 1];
    uint64_t qhat = num / vn[n - 1], rhat = num % vn[n - 1];
    while (qhat >= B || qhat * vn[n - 2] > ((rhat << 32) | un[j + n - 2])) {
      --qhat;
      rhat += vn[n - 1];
      if (rhat >= B) break;
    }
    int64_t k = 0, t;
    for (size_t i = 0; i < n; ++i) {
      const uint64_t p = qhat * vn[i];
      t = (int64_t)un[i + j] - k - (int64_t)(p & 0xffffffffull);
      un[i + j] = (uint32_t)t;
      k = (int64_t)(p >> 32) - (t >> 32);
    }
    t = (int64_t)un[j + n] - k;
    un[j + n] = (uint32_t)t;
    if (t < 0) {  // qhat one too large: add the divisor back
      --qhat;
      uint64_t c = 0;
      for (size_t i = 0; i < n; ++i) {
        const uint64_t s2 = (uint64_t)un[i + j] + vn[i] + c;
        un[i + j] = (uint32_t)s2;
        c = s2 >> 32;
      }
      un[j + n] += (uint32_t)c;
    }
    q.w[j] = (uint32_t)qhat;
  }
  r.w.assign(n, 0u);
  for (size_t i = 0; i < n; ++i)
    r.w[i] = (un[i] >> s) | (s ? (uint32_t)((uint64_t)un[i + 1] << (32 - s)) : 0u);
  q.trim();
  r.trim();
}

UBig UBig::isqrt(const UBig &a) {
  if (a.zero()) return UBig();
  // Newton from above converges to floor(sqrt(a)) from any start >=
  // sqrt(a); start from the binary64 root of the leading bits (rounded up
  // with margin), so a few iterations suffice instead of ~log2(bits)
  const int64_t nb = a.bits();
  UBig x;
  if (nb > 64) {
    int64_t sh = nb - 62;
    if (sh & 1) sh += 1;                       // even: sqrt(2^sh) exact
    const uint64_t top = a.shr(sh).low64();    // a < (top + 1) 2^sh
    const double r = std::sqrt((double)top + 2.0) * (1.0 + 0x1p-40) + 2.0;
    x = UBig((uint64_t)std::ceil(r)).shl(sh / 2);
  } else {
    x = UBig(1).shl((nb + 1) / 2 + 1);
  }
  for (;;) {
    UBig q, r;
    divmod(a, x, q, r);
    UBig y = add(x, q).shr(1);
    if (cmp(y, x) >= 0) break;
    x = y;
  }
  return x;
}

UBig UBig::pow10(int64_t e) {
  UBig r(1);
  while (e >= 9) { r.mul_small(1000000000u); e -= 9; }
  while (e-- > 0) r.mul_small(10u);
  return r;
}

std::string UBig::to_dec() const {
  if (zero()) return "0";
  std::string s;
  UBig t = *this;
  UBig ten9(1000000000u);
  while (!t.zero()) {
    UBig q, r;
    divmod(t, ten9, q, r);
    uint32_t chunk = (uint32_t)r.low64();
    for (int i = 0; i < 9; ++i) {
      s.push_back((char)('0' + chunk % 10));
      chunk /= 10;
      if (q.zero() && chunk == 0) break;
    }
    t = q;
  }
  while (s.size() > 1 && s.back() == '0') s.pop_back();
  std::reverse(s.begin(), s.end());
  return s;
}

void round_to(UBig &man, int64_t &exp, int64_t p) {
  int64_t excess = man.bits() - p;
  if (excess > 0) {
    bool half_bit = man.bit(excess - 1);
    bool below = man.low_bits_nonzero(excess - 1);
    man = man.shr(excess);
    exp += excess;
    if (half_bit && (below || man.bit(0))) {
      man.add_small(1);
      if (man.bits() > p) {
        man = man.shr(1);
        exp += 1;
      }
    }
  }
}

BF mk(int sign, UBig man, int64_t exp, int64_t p) {
  BF r;
  if (man.zero()) return r;
  round_to(man, exp, p);
  r.sign = sign;
  r.man = man;
  r.exp = exp;
  return r;
}

BF round_ratio(int sign, const UBig &num, const UBig &den, int64_t exp,
               int64_t p) {
  int64_t shift = p + 2 - (num.bits() - den.bits());
  if (shift < 0) shift = 0;
  UBig q, r;
  UBig::divmod(num.shl(shift), den, q, r);
  exp -= shift;
  if (!r.zero()) {
    q = q.shl(1);
    q.add_small(1);
    exp -= 1;
  }
  return mk(sign, q, exp, p);
}

BF neg(const BF &a) {
  BF r = a;
  r.sign = -a.sign;
  return r;
}

BF add_exact(const BF &a, const BF &b) {
  if (a.sign == 0) return b;
  if (b.sign == 0) return a;
  int64_t e = std::min(a.exp, b.exp);
  UBig A = a.man.shl(a.exp - e), B = b.man.shl(b.exp - e);
  BF r;
  r.exp = e;
  if (a.sign == b.sign) {
    r.sign = a.sign;
    r.man = UBig::add(A, B);
  } else {
    int c = UBig::cmp(A, B);
    if (c == 0) return BF();
    if (c > 0) {
      r.sign = a.sign;
      r.man = UBig::sub(A, B);
    } else {
      r.sign = b.sign;
      r.man = UBig::sub(B, A);
    }
  }
  return r;
}

int to_binary64(const BF &a, double &out) {
  if (a.sign == 0) {
    out = 0.0;
    return 0;
  }
  UBig m = a.man;
  int64_t e = a.exp;
  round_to(m, e, 53);
  if (e > 2000) return 5;
  if (e < -3000) {
    out = a.sign < 0 ? -0.0 : 0.0;  // ldexp underflows to (signed) zero
    return 0;
  }
  double r = std::ldexp((double)m.low64(), (int)e);
  if (std::isinf(r)) return 5;
  out = a.sign < 0 ? -r : r;
  return 0;
}

BF from_binary64(double x) {
  BF r;
  if (x == 0.0) return r;
  int e;
  double f = std::frexp(std::fabs(x), &e);
  uint64_t man = (uint64_t)std::ldexp(f, 53);
  r.sign = x > 0 ? 1 : -1;
  r.man = UBig(man);
  r.exp = e - 53;
  return r;
}

int to_multicomp(const BF &a, int k, double *out) {
  BF r = a;
  for (int c = 0; c < k; ++c) {
    double v;
    int st = to_binary64(r, v);
    if (st) return st;
    out[c] = v;
    if (v != 0.0) r = add_exact(r, neg(from_binary64(v)));
  }
  return 0;
}

static std::string strip(const std::string &s) {
  size_t b = 0, e = s.size();
  while (b < e && std::isspace((unsigned char)s[b])) ++b;
  while (e > b && std::isspace((unsigned char)s[e - 1])) --e;
  return s.substr(b, e - b);
}

static bool parse_exp10(const std::string &s, size_t &i, int64_t &out) {
  // [+-]?\d+ to the end of the string
  int sg = 1;
  if (i < s.size() && (s[i] == '+' || s[i] == '-')) {
    if (s[i] == '-') sg = -1;
    ++i;
  }
  if (i >= s.size()) return false;
  int64_t v = 0;
  bool big = false;
  for (; i < s.size(); ++i) {
    if (!std::isdigit((unsigned char)s[i])) return false;
    if (v > (int64_t)1e15) big = true;
    else v = v * 10 + (s[i] - '0');
  }
  out = big ? sg * (int64_t)4e15 : sg * v;
  return true;
}

int parse_decimal(const std::string &text, int64_t p, BF &out) {
  std::string s = strip(text);
  size_t i = 0;
  int sign = 1;
  if (i < s.size() && (s[i] == '+' || s[i] == '-')) {
    if (s[i] == '-') sign = -1;
    ++i;
  }
  std::string int_s, frac_s;
  while (i < s.size() && std::isdigit((unsigned char)s[i])) int_s += s[i++];
  bool dot = false;
  if (i < s.size() && s[i] == '.') {
    dot = true;
    ++i;
    while (i < s.size() && std::isdigit((unsigned char)s[i])) frac_s += s[i++];
  }
  if (int_s.empty() && (!dot || frac_s.empty())) return 4;
  int64_t e = 0;
  if (i < s.size()) {
    if (s[i] != 'e' && s[i] != 'E') return 4;
    ++i;
    if (!parse_exp10(s, i, e)) return 4;
  }
  std::string digits = int_s + frac_s;
  size_t nz = digits.find_first_not_of('0');
  if (nz == std::string::npos) {
    out = BF();
    return 0;
  }
  digits = digits.substr(nz);
  int64_t e10 = e - (int64_t)frac_s.size();
  // beyond any binary64-representable magnitude: report overflow / zero
  // exactly as the reference's bf_to_binary64 would downstream
  int64_t mag10 = e10 + (int64_t)digits.size();
  if (mag10 > 400) return 5;
  if (mag10 < -400) {  // rounds to a signed zero downstream
    out.sign = sign;
    out.man = UBig(1);
    out.exp = -5000;
    return 0;
  }
  UBig d;
  for (char ch : digits) {
    d.mul_small(10);
    d.add_small((uint32_t)(ch - '0'));
  }
  if (e10 >= 0) {
    out = mk(sign, UBig::mul(d, UBig::pow10(e10)), 0, p);
  } else {
    out = round_ratio(sign, d, UBig::pow10(-e10), 0, p);
  }
  return 0;
}

static int hexval(char c) {
  if (c >= '0' && c <= '9') return c - '0';
  if (c >= 'a' && c <= 'f') return c - 'a' + 10;
  if (c >= 'A' && c <= 'F') return c - 'A' + 10;
  return -1;
}

int parse_hex(const std::string &text, BF &out) {
  std::string s = strip(text);
  size_t i = 0;
  int sign = 1;
  if (i < s.size() && (s[i] == '+' || s[i] == '-')) {
    if (s[i] == '-') sign = -1;
    ++i;
  }
  if (i + 1 >= s.size() || s[i] != '0' || (s[i + 1] != 'x' && s[i + 1] != 'X'))
    return 4;
  i += 2;
  UBig man;
  int nint = 0, nfrac = 0;
  while (i < s.size() && hexval(s[i]) >= 0) {
    man.mul_small(16);
    man.add_small((uint32_t)hexval(s[i++]));
    ++nint;
  }
  if (nint == 0) return 4;
  if (i < s.size() && s[i] == '.') {
    ++i;
    while (i < s.size() && hexval(s[i]) >= 0) {
      man.mul_small(16);
      man.add_small((uint32_t)hexval(s[i++]));
      ++nfrac;
    }
  }
  if (i >= s.size() || (s[i] != 'p' && s[i] != 'P')) return 4;
  ++i;
  int64_t e;
  if (!parse_exp10(s, i, e)) return 4;
  if (man.zero()) {
    out = BF();
    return 0;
  }
  out.sign = sign;
  out.man = man;
  out.exp = e - 4 * (int64_t)nfrac;
  return 0;
}

}  // namespace bn
