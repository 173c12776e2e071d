// Fixed-width correctly rounded long floats for the refinement loop's hot
// operations (the residual b - A x, norms, the x update; refine.py:163-190).
//
// Same arithmetic as lf_add / lf_mul (bigfloat.py:239-274: the exact result
// rounded once to p bits, half to even), without heap traffic: the mantissa
// is held normalised to exactly p bits in NL 64-bit limbs (p <= 64 * NL).
// tests/test_longside.py checks every operation against the generic
// big-integer path (mpcore_debug_longfloat_selftest).
#pragma once
#include <cstdint>
#include <cstring>

#include "bignum.h"

namespace ff {

constexpr int NL = 10;            // p <= 640
constexpr int WL = 2 * NL + 2;    // exact sums / products

struct F {
  int sign = 0;       // 0: zero
  int64_t exp = 0;    // value = sign * m * 2^exp, m has exactly p bits
  uint64_t m[NL];
};

inline int bitlen(const uint64_t *a, int n) {
  for (int i = n - 1; i >= 0; --i)
    if (a[i]) return 64 * i + 64 - __builtin_clzll(a[i]);
  return 0;
}
inline bool getbit(const uint64_t *a, int n, int64_t i) {
  if (i < 0 || i >= 64 * (int64_t)n) return false;
  return (a[i >> 6] >> (i & 63)) & 1u;
}
inline bool any_below(const uint64_t *a, int n, int64_t nbits) {
  if (nbits <= 0) return false;
  const int64_t full = nbits >> 6;
  for (int64_t l = 0; l < full && l < n; ++l)
    if (a[l]) return true;
  const int rem = (int)(nbits & 63);
  return rem && full < n && (a[full] & ((1ull << rem) - 1ull)) != 0;
}
// out[0..nout) = a >> s
inline void shr_into(const uint64_t *a, int n, int64_t s, uint64_t *out,
                     int nout) {
  const int64_t q = s >> 6;
  const int r = (int)(s & 63);
  for (int i = 0; i < nout; ++i) {
    const int64_t j = i + q;
    uint64_t lo = j < n ? a[j] : 0, hi = j + 1 < n ? a[j + 1] : 0;
    out[i] = r ? (lo >> r) | (hi << (64 - r)) : lo;
  }
}
// out[0..nout) = a << s (bits beyond nout limbs dropped)
inline void shl_into(const uint64_t *a, int n, int64_t s, uint64_t *out,
                     int nout) {
  const int64_t q = s >> 6;
  const int r = (int)(s & 63);
  for (int i = nout - 1; i >= 0; --i) {
    const int64_t j = i - q;
    uint64_t hi = (j >= 0 && j < n) ? a[j] : 0;
    uint64_t lo = (j - 1 >= 0 && j - 1 < n) ? a[j - 1] : 0;
    out[i] = r ? (hi << r) | (lo >> (64 - r)) : hi;
  }
}
inline int cmp_n(const uint64_t *a, const uint64_t *b, int n) {
  for (int i = n - 1; i >= 0; --i)
    if (a[i] != b[i]) return a[i] > b[i] ? 1 : -1;
  return 0;
}
inline void add_n(uint64_t *a, const uint64_t *b, int n) {
  unsigned __int128 c = 0;
  for (int i = 0; i < n; ++i) {
    c += (unsigned __int128)a[i] + b[i];
    a[i] = (uint64_t)c;
    c >>= 64;
  }
}
inline void sub_n(uint64_t *a, const uint64_t *b, int n) {  // a -= b, a >= b
  uint64_t borrow = 0;
  for (int i = 0; i < n; ++i) {
    const uint64_t bi = b[i] + borrow;
    const uint64_t nb = (bi < borrow) || (a[i] < bi);
    a[i] -= bi;
    borrow = nb;
  }
}

// the exact value sign * w * 2^e rounded to p bits (half to even)
inline F round_to(int sign, const uint64_t *w, int n, int64_t e, int p) {
  F r;
  const int L = bitlen(w, n);
  if (L == 0) return r;
  r.sign = sign;
  if (L <= p) {
    shl_into(w, n, p - L, r.m, NL);
    r.exp = e - (p - L);
    return r;
  }
  const int64_t ex = L - p;
  const bool half = getbit(w, n, ex - 1);
  const bool below = any_below(w, n, ex - 1);
  shr_into(w, n, ex, r.m, NL);
  r.exp = e + ex;
  if (half && (below || (r.m[0] & 1u))) {
    bool carry = true;
    for (int i = 0; i < NL && carry; ++i) carry = ++r.m[i] == 0;
    if (carry || bitlen(r.m, NL) > p) {
      // rounded up to 2^p: the mantissa becomes 2^(p-1), one binade up
      std::memset(r.m, 0, sizeof r.m);
      r.m[(p - 1) >> 6] = 1ull << ((p - 1) & 63);
      r.exp += 1;
    }
  }
  return r;
}

inline F mul(const F &a, const F &b, int p) {
  if (a.sign == 0 || b.sign == 0) return F();
  const int nl = (p + 63) >> 6;
  uint64_t w[2 * NL] = {0};
  for (int i = 0; i < nl; ++i) {
    unsigned __int128 c = 0;
    const uint64_t ai = a.m[i];
    for (int j = 0; j < nl; ++j) {
      c += (unsigned __int128)ai * b.m[j] + w[i + j];
      w[i + j] = (uint64_t)c;
      c >>= 64;
    }
    w[i + nl] = (uint64_t)c;
  }
  return round_to(a.sign * b.sign, w, 2 * nl, a.exp + b.exp, p);
}

inline F add(const F &a, const F &b, int p) {
  if (a.sign == 0) return b;
  if (b.sign == 0) return a;
  const F &x = a.exp >= b.exp ? a : b;
  const F &y = a.exp >= b.exp ? b : a;
  const int64_t d = x.exp - y.exp;
  // y below a quarter ulp of x never moves the rounded result (even when
  // x is a power of two and y is subtracted)
  if (d >= p + 3) return x;
  const int nl = (p + 63) >> 6;
  const int nw = ((p + (int)d + 1) >> 6) + 1;
  uint64_t w[WL], v[WL];
  shl_into(x.m, nl, d, w, nw);
  for (int i = 0; i < nw; ++i) v[i] = i < nl ? y.m[i] : 0;
  int sign = x.sign;
  if (x.sign == y.sign) {
    add_n(w, v, nw);
  } else {
    const int c = cmp_n(w, v, nw);
    if (c == 0) return F();
    if (c > 0) {
      sub_n(w, v, nw);
    } else {
      sub_n(v, w, nw);
      std::memcpy(w, v, sizeof(uint64_t) * nw);
      sign = y.sign;
    }
  }
  return round_to(sign, w, nw, y.exp, p);
}

inline F neg(const F &a) {
  F r = a;
  r.sign = -a.sign;
  return r;
}

inline F from_bf(const bn::BF &v, int p) {
  if (v.sign == 0) return F();
  uint64_t w[WL] = {0};
  const auto &l = v.man.w;  // 32-bit limbs
  const int n = (int)((l.size() + 1) / 2);
  if (n > WL) {  // wider than any p handled here: round via the slow path
    bn::UBig m = v.man;
    int64_t e = v.exp;
    bn::round_to(m, e, p);
    bn::BF t;
    t.sign = v.sign;
    t.man = m;
    t.exp = e;
    return from_bf(t, p);
  }
  for (size_t i = 0; i < l.size(); ++i)
    w[i / 2] |= (uint64_t)l[i] << (32 * (i & 1));
  return round_to(v.sign, w, n, v.exp, p);
}

inline bn::BF to_bf(const F &a) {
  bn::BF r;
  if (a.sign == 0) return r;
  r.sign = a.sign;
  int tz = 0;
  int i = 0;
  while (i < NL && a.m[i] == 0) {
    tz += 64;
    ++i;
  }
  if (i < NL) tz += __builtin_ctzll(a.m[i]);
  uint64_t t[NL];
  shr_into(a.m, NL, tz, t, NL);
  for (int k = 0; k < NL; ++k) {
    r.man.w.push_back((uint32_t)t[k]);
    r.man.w.push_back((uint32_t)(t[k] >> 32));
  }
  r.man.trim();
  r.exp = a.exp + tz;
  return r;
}

}  // namespace ff
