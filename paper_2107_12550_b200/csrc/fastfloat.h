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
#include <cmath>
#include <cstring>
#include <x86intrin.h>

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
    if (L == p) {  // already p bits (the common case for inputs at p)
      for (int i = 0; i < NL; ++i) r.m[i] = i < n ? w[i] : 0ull;
    } else {
      shl_into(w, n, p - L, r.m, NL);
    }
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

// ---- compile-time-width kernels (N = ceil(p / 64) limbs) -----------------
// Same results as add / mul above (the exact value rounded once to p bits,
// half to even), computed the way a floating-point adder does it: the
// smaller operand is shifted right into a frame with one 64-bit guard limb
// and a sticky bit, instead of shifting the larger one left into a window
// of p + d bits.  In the frame, bit i of x's mantissa sits at i + 64.

// top set bit of a (W limbs), -1 if zero
template <int W> inline int top_bit(const uint64_t *a) {
  for (int i = W - 1; i >= 0; --i)
    if (a[i]) return 64 * i + 63 - __builtin_clzll(a[i]);
  return -1;
}
// out[0..N) = a[0..W) >> s (0 <= s < 64 W), rounded to nearest even using
// the bits shifted out plus `sticky`; returns true when the increment
// carried to bit p (the caller renormalises)
template <int W, int N>
inline bool shr_round(const uint64_t *a, int s, bool sticky, int p,
                      uint64_t *out) {
  // zero-padded copy: out limb i reads pad[i + q], pad[i + q + 1]
  uint64_t pad[W + N + 2];
#pragma GCC unroll 32
  for (int i = 0; i < W; ++i) pad[i] = a[i];
#pragma GCC unroll 32
  for (int i = W; i < W + N + 2; ++i) pad[i] = 0;
  const int q = s >> 6, r = s & 63;
  const uint64_t *src = pad + q;
  if (r) {
#pragma GCC unroll 16
    for (int i = 0; i < N; ++i)
      out[i] = (src[i] >> r) | (src[i + 1] << (64 - r));
  } else {
#pragma GCC unroll 16
    for (int i = 0; i < N; ++i) out[i] = src[i];
  }
  if (s == 0) return false;
  const int rb = s - 1;  // round bit position
  if (!((a[rb >> 6] >> (rb & 63)) & 1u)) return false;
  bool below = sticky;
  if (!below) {
    const int full = rb >> 6, rem = rb & 63;
    for (int l = 0; l < full && !below; ++l) below = a[l] != 0;
    if (!below && rem) below = (a[full] & ((1ull << rem) - 1ull)) != 0;
  }
  if (!below && !(out[0] & 1u)) return false;
  bool carry = true;
  for (int i = 0; i < N && carry; ++i) carry = ++out[i] == 0;
  // rounded up to 2^p?
  const int pl = p >> 6, pb = p & 63;
  return carry || (pl < N && ((out[pl] >> pb) & 1u));
}
inline void set_pow2(F &r, int p) {  // mantissa 2^(p-1)
  for (int i = 0; i < NL; ++i) r.m[i] = 0;
  r.m[(p - 1) >> 6] = 1ull << ((p - 1) & 63);
}

template <int N> inline F add_t(const F &a, const F &b, int p) {
  if (a.sign == 0) return b;
  if (b.sign == 0) return a;
  const F &x = a.exp >= b.exp ? a : b;
  const F &y = a.exp >= b.exp ? b : a;
  const int64_t d64 = x.exp - y.exp;
  // y below a quarter ulp of x never moves the rounded result
  if (d64 >= p + 3) return x;
  const int d = (int)d64;
  constexpr int W = N + 2;
  uint64_t X[W], Y[W], S[W];
  X[0] = 0;
#pragma GCC unroll 16
  for (int i = 0; i < N; ++i) X[i + 1] = x.m[i];
  X[N + 1] = 0;
  // Y = (y.m << 64) >> d, sticky = the bits shifted out.  ys[j] = limb j
  // of y.m << 64, zero-padded so ys[i + q + 1] is in range (q <= N + 1)
  const int q = d >> 6, r = d & 63;
  uint64_t ys[2 * W + 2];
  ys[0] = 0;
#pragma GCC unroll 16
  for (int i = 0; i < N; ++i) ys[i + 1] = y.m[i];
#pragma GCC unroll 32
  for (int i = N + 1; i < 2 * W + 2; ++i) ys[i] = 0;
  const uint64_t *src = ys + q;
  if (r) {
#pragma GCC unroll 16
    for (int i = 0; i < W; ++i) Y[i] = (src[i] >> r) | (src[i + 1] << (64 - r));
  } else {
#pragma GCC unroll 16
    for (int i = 0; i < W; ++i) Y[i] = src[i];
  }
  bool sticky = false;
  for (int j = 1; j < q; ++j) sticky |= ys[j] != 0;
  if (r) sticky |= (ys[q] & ((1ull << r) - 1ull)) != 0;
  int sign = x.sign;
  if (x.sign == y.sign) {
    unsigned char cf = 0;
#pragma GCC unroll 16
    for (int i = 0; i < W; ++i)
      cf = _addcarry_u64(cf, X[i], Y[i], (unsigned long long *)&S[i]);
  } else {
    const uint64_t *P = X, *M = Y;
    if (d == 0) {  // equal exponents: order the mantissas
      int c = 0;
      for (int i = W - 1; i >= 0 && c == 0; --i)
        if (X[i] != Y[i]) c = X[i] > Y[i] ? 1 : -1;
      if (c == 0) return F();
      if (c < 0) {
        P = Y;
        M = X;
        sign = y.sign;
      }
    }
    // P - M - sticky: a lost fraction of M borrows one unit (the remaining
    // fraction is still nonzero, so sticky stays set)
    unsigned char bf = sticky ? 1 : 0;
#pragma GCC unroll 16
    for (int i = 0; i < W; ++i)
      bf = _subborrow_u64(bf, P[i], M[i], (unsigned long long *)&S[i]);
  }
  const int t = top_bit<W>(S);
  F res;
  if (t < 0) return res;
  res.sign = sign;
  for (int i = N; i < NL; ++i) res.m[i] = 0;
  if (t < p) {
    // fewer than p + 1 bits: exact (bits are lost only for d > 64, and
    // then the result keeps at least p + 62 bits in the frame)
    const int sh = p - 1 - t;
    shl_into(S, W, sh, res.m, N);
    res.exp = x.exp - 64 - sh;
    return res;
  }
  const int sh = t - p + 1;
  res.exp = x.exp - 64 + sh;
  if (shr_round<W, N>(S, sh, sticky, p, res.m)) {
    set_pow2(res, p);
    res.exp += 1;
  }
  return res;
}

template <int N> inline F mul_t(const F &a, const F &b, int p) {
  if (a.sign == 0 || b.sign == 0) return F();
  // column-wise (Comba): the partial products of a column are independent
  // and accumulate into a three-word sum
  uint64_t w[2 * N];
  unsigned long long c0 = 0, c1 = 0, c2 = 0;
#pragma GCC unroll 16
  for (int k = 0; k < 2 * N - 1; ++k) {
#pragma GCC unroll 16
    for (int i = 0; i < N; ++i) {
      const int j = k - i;
      if (j < 0 || j >= N) continue;
      const unsigned __int128 pr = (unsigned __int128)a.m[i] * b.m[j];
      unsigned char cf = _addcarry_u64(0, c0, (uint64_t)pr, &c0);
      cf = _addcarry_u64(cf, c1, (uint64_t)(pr >> 64), &c1);
      c2 += cf;
    }
    w[k] = c0;
    c0 = c1;
    c1 = c2;
    c2 = 0;
  }
  w[2 * N - 1] = c0;
  // the product of two p-bit mantissas has 2p or 2p - 1 bits
  const int top = 2 * p - 1;
  const bool full = (w[top >> 6] >> (top & 63)) & 1u;
  const int sh = full ? p : p - 1;
  F res;
  res.sign = a.sign * b.sign;
  for (int i = N; i < NL; ++i) res.m[i] = 0;
  res.exp = a.exp + b.exp + sh;
  if (shr_round<2 * N, N>(w, sh, false, p, res.m)) {
    set_pow2(res, p);
    res.exp += 1;
  }
  return res;
}

// bf_to_multicomp on a fixed-width value (bigfloat.py:419-432, as
// bn::to_multicomp): k heads, each the nearest binary64 (half to even),
// peeled off exactly.  Returns false, leaving `out` undefined, when a head
// would fall outside the normal binary64 range (the caller then takes the
// generic path, which reproduces ldexp's subnormal rounding and overflow).
template <int N>
inline bool to_multicomp_t(const F &r0, int k, int p, double *out) {
  // The value is sign * M * 2^e with the integer M in N limbs; each head is
  // M's top 53 bits rounded to nearest even, and M keeps the exact signed
  // remainder (no renormalisation: only its bit length is tracked).
  uint64_t M[N];
  for (int i = 0; i < N; ++i) M[i] = r0.m[i];
  int sign = r0.sign;
  const int64_t e = r0.exp;
  int len = r0.sign == 0 ? 0 : p;
  for (int c = 0; c < k; ++c) {
    if (len == 0) {
      out[c] = 0.0;
      continue;
    }
    uint64_t h;
    int sh = 0;
    bool up = false;
    if (len <= 53) {
      h = M[0];
    } else {
      sh = len - 53;
      const int q = sh >> 6, rr = sh & 63;
      const uint64_t lo = M[q], hi = q + 1 < N ? M[q + 1] : 0;
      h = (rr ? (lo >> rr) | (hi << (64 - rr)) : lo) & ((1ull << 53) - 1ull);
      const int rb = sh - 1;
      const bool half = (M[rb >> 6] >> (rb & 63)) & 1u;
      if (half) {
        bool below = (rb & 63) &&
                     (M[rb >> 6] & ((1ull << (rb & 63)) - 1ull)) != 0;
        for (int l = 0; l < (rb >> 6) && !below; ++l) below = M[l] != 0;
        up = below || (h & 1u);
      }
      if (up) ++h;  // may reach 2^53 (exact)
    }
    const int64_t E = e + sh;
    const int top = 63 - __builtin_clzll(h);
    if (E + top < -1022 || E + top > 1023) return false;
    // h 2^E in the normal range: the binary64 bits directly (h != 0)
    const int sh52 = 52 - top;  // h << sh52 has its top bit at 52 (may be < 0)
    const uint64_t frac =
        (sh52 >= 0 ? h << sh52 : h >> -sh52) & ((1ull << 52) - 1ull);
    const uint64_t bits = ((uint64_t)(E + top + 1023) << 52) | frac |
                          (sign < 0 ? (1ull << 63) : 0ull);
    std::memcpy(&out[c], &bits, 8);
    if (c + 1 == k) break;
    if (len <= 53) {  // the head took everything
      len = 0;
      continue;
    }
    // remainder: the low sh bits, or 2^sh minus them after rounding up
    const int qs = sh >> 6, rs = sh & 63;
    for (int i = 0; i < N; ++i) {
      if (i > qs || (i == qs && rs == 0)) M[i] = 0;
      else if (i == qs) M[i] &= (1ull << rs) - 1ull;
    }
    if (up) {
      unsigned char cf = 1;  // two's complement, masked to sh bits
      for (int i = 0; i < N; ++i)
        cf = _addcarry_u64(cf, ~M[i], 0ull, (unsigned long long *)&M[i]);
      for (int i = 0; i < N; ++i) {
        if (i > qs || (i == qs && rs == 0)) M[i] = 0;
        else if (i == qs) M[i] &= (1ull << rs) - 1ull;
      }
      sign = -sign;
    }
    len = 0;
    for (int i = N - 1; i >= 0; --i)
      if (M[i]) {
        len = 64 * i + 64 - __builtin_clzll(M[i]);
        break;
      }
  }
  return true;
}

// runtime dispatch on the limb count
#define FF_DISPATCH(FN, ...)             \
  switch ((p + 63) >> 6) {               \
    case 1: return FN<1>(__VA_ARGS__);   \
    case 2: return FN<2>(__VA_ARGS__);   \
    case 3: return FN<3>(__VA_ARGS__);   \
    case 4: return FN<4>(__VA_ARGS__);   \
    case 5: return FN<5>(__VA_ARGS__);   \
    case 6: return FN<6>(__VA_ARGS__);   \
    case 7: return FN<7>(__VA_ARGS__);   \
    case 8: return FN<8>(__VA_ARGS__);   \
    case 9: return FN<9>(__VA_ARGS__);   \
    default: return FN<10>(__VA_ARGS__); \
  }
inline F fadd(const F &a, const F &b, int p) { FF_DISPATCH(add_t, a, b, p) }
inline F fmul(const F &a, const F &b, int p) { FF_DISPATCH(mul_t, a, b, p) }
inline bool to_multicomp(const F &r, int k, int p, double *out) {
  FF_DISPATCH(to_multicomp_t, r, k, p, out)
}
#undef FF_DISPATCH

// a binary64 value exactly, as a p-bit fixed-width value (p >= 53)
inline F from_double(double x, int p) {
  F r;
  if (x == 0.0) return r;
  int e;
  const double f = std::frexp(std::fabs(x), &e);  // f in [0.5, 1)
  uint64_t m = (uint64_t)std::ldexp(f, 53);         // exact, 53 bits
  r.sign = x < 0 ? -1 : 1;
  const int tz = __builtin_ctzll(m);
  m >>= tz;
  const int len = 64 - __builtin_clzll(m);
  const uint64_t w[1] = {m};
  for (int i = 0; i < NL; ++i) r.m[i] = 0;
  shl_into(w, 1, p - len, r.m, NL);
  r.exp = (int64_t)e - 53 + tz - (p - len);
  return r;
}
// a value held at precision q, rounded once to p <= q bits
inline F round(const F &a, int q, int p) {
  if (a.sign == 0 || q == p) return a;
  return round_to(a.sign, a.m, NL, a.exp, p);
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
