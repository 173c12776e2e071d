// Correctly rounded long floats on the device: the IR residual b - A x at
// the working precision p (refine.py:163-172, linalg.py:564-574), SURVEY
// §8(f) row 1.  Same arithmetic as the host's fastfloat.h (add_t / mul_t):
// the exact result rounded once to p bits, half to even -- the
// single-rounding rules of bigfloat.py:239-274 -- so the residual is bit
// for bit the host's (and the reference's).
//
// A value is sign * m * 2^exp with the mantissa m normalised to exactly p
// bits in N = ceil(p / 64) 64-bit limbs (DF mirrors the host struct ff::F
// byte for byte, so arrays of it upload unchanged).  Every limb array is
// indexed with compile-time indices only (shifts by a runtime amount go
// through log-step limb shifters and selects), so the values stay in
// registers.
#pragma once
#include <cstdint>

namespace lf {

constexpr int NL = 10;  // limbs in the struct (the host's ff::NL)
struct DF {
  int sign;      // 0: zero
  int64_t exp;
  uint64_t m[NL];
};

#define LFI __device__ __forceinline__

// in place: a >>= 64 q (q >= 0; q >= W clears)
template <int W> LFI void shr_limbs(uint64_t (&a)[W], int q) {
#pragma unroll
  for (int b = 1; b < 2 * W; b <<= 1) {
    const bool on = (q & b) != 0;
#pragma unroll
    for (int i = 0; i < W; ++i) a[i] = on ? (i + b < W ? a[i + b] : 0ull) : a[i];
  }
}
// in place: a <<= 64 q (bits beyond W limbs dropped)
template <int W> LFI void shl_limbs(uint64_t (&a)[W], int q) {
#pragma unroll
  for (int b = 1; b < 2 * W; b <<= 1) {
    const bool on = (q & b) != 0;
#pragma unroll
    for (int i = W - 1; i >= 0; --i) a[i] = on ? (i - b >= 0 ? a[i - b] : 0ull) : a[i];
  }
}
// in place: a >>= r bits, 0 <= r < 64
template <int W> LFI void shr_bits(uint64_t (&a)[W], int r) {
  if (r == 0) return;
#pragma unroll
  for (int i = 0; i < W; ++i)
    a[i] = (a[i] >> r) | (i + 1 < W ? a[i + 1] << (64 - r) : 0ull);
}
template <int W> LFI void shl_bits(uint64_t (&a)[W], int r) {
  if (r == 0) return;
#pragma unroll
  for (int i = W - 1; i >= 0; --i)
    a[i] = (a[i] << r) | (i > 0 ? a[i - 1] >> (64 - r) : 0ull);
}
// bit `pos` of a (0 beyond the array)
template <int W> LFI bool get_bit(const uint64_t (&a)[W], int pos) {
  const int l = pos >> 6, b = pos & 63;
  uint64_t v = 0;
#pragma unroll
  for (int i = 0; i < W; ++i) v = (i == l) ? a[i] : v;
  return pos >= 0 && l < W && ((v >> b) & 1ull);
}
// any set bit of a strictly below position pos
template <int W> LFI bool any_below(const uint64_t (&a)[W], int pos) {
  const int l = pos >> 6, b = pos & 63;
  bool r = false;
#pragma unroll
  for (int i = 0; i < W; ++i) {
    const uint64_t mask = i < l ? ~0ull : (i == l ? ((1ull << b) - 1ull) : 0ull);
    r |= (a[i] & mask) != 0;
  }
  return pos > 0 && r;
}
template <int W> LFI int top_bit(const uint64_t (&a)[W]) {
  int t = -1;
#pragma unroll
  for (int i = 0; i < W; ++i)
    if (a[i]) t = 64 * i + 63 - __clzll((long long)a[i]);
  return t;
}

LFI DF zero() {
  DF r;
  r.sign = 0;
  r.exp = 0;
#pragma unroll
  for (int i = 0; i < NL; ++i) r.m[i] = 0;
  return r;
}

// a (W limbs) >> s, rounded to nearest even into N limbs (plus `sticky`
// for bits already lost); true when the increment reached bit p
template <int W, int N>
LFI bool shr_round(const uint64_t (&a)[W], int s, bool sticky, int p,
                   uint64_t (&out)[N]) {
  uint64_t t[W];
#pragma unroll
  for (int i = 0; i < W; ++i) t[i] = a[i];
  shr_limbs<W>(t, s >> 6);
  shr_bits<W>(t, s & 63);
#pragma unroll
  for (int i = 0; i < N; ++i) out[i] = t[i];
  if (s == 0) return false;
  const bool half = get_bit<W>(a, s - 1);
  const bool below = sticky || any_below<W>(a, s - 1);
  if (!(half && (below || (out[0] & 1ull)))) return false;
  bool carry = true;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const uint64_t v = out[i] + (carry ? 1ull : 0ull);
    carry = carry && v == 0ull;
    out[i] = v;
  }
  return carry || get_bit<N>(out, p);
}
template <int N> LFI void set_pow2(DF &r, int p) {
#pragma unroll
  for (int i = 0; i < NL; ++i) r.m[i] = 0;
  const int l = (p - 1) >> 6;
#pragma unroll
  for (int i = 0; i < N; ++i) r.m[i] = (i == l) ? (1ull << ((p - 1) & 63)) : 0ull;
}

template <int N> LFI DF add(const DF &a, const DF &b, int p) {
  if (a.sign == 0) return b;
  if (b.sign == 0) return a;
  const bool ax = a.exp >= b.exp;
  const DF &x = ax ? a : b;
  const DF &y = ax ? b : a;
  const int64_t d64 = x.exp - y.exp;
  if (d64 >= p + 3) return x;
  const int d = (int)d64;
  constexpr int W = N + 2;
  uint64_t X[W], Y[W], S[W];
  X[0] = 0ull;
  Y[0] = 0ull;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    X[i + 1] = x.m[i];
    Y[i + 1] = y.m[i];
  }
  X[N + 1] = 0ull;
  Y[N + 1] = 0ull;
  // sticky: bits of (y.m << 64) below position d
  const bool sticky = any_below<W>(Y, d);
  shr_limbs<W>(Y, d >> 6);
  shr_bits<W>(Y, d & 63);
  int sign = x.sign;
  if (x.sign == y.sign) {
    uint64_t c = 0;
#pragma unroll
    for (int i = 0; i < W; ++i) {
      const uint64_t s1 = X[i] + Y[i];
      const uint64_t c1 = s1 < X[i];
      S[i] = s1 + c;
      c = c1 | (S[i] < s1);
    }
  } else {
    bool swap = false;
    if (d == 0) {  // equal exponents: order the mantissas
      int c = 0;
#pragma unroll
      for (int i = W - 1; i >= 0; --i)
        if (c == 0 && X[i] != Y[i]) c = X[i] > Y[i] ? 1 : -1;
      if (c == 0) return zero();
      swap = c < 0;
      if (swap) sign = y.sign;
    }
    // P - M - sticky (a lost fraction of M borrows one unit)
    uint64_t bw = sticky ? 1ull : 0ull;
#pragma unroll
    for (int i = 0; i < W; ++i) {
      const uint64_t P = swap ? Y[i] : X[i], M = swap ? X[i] : Y[i];
      const uint64_t mi = M + bw;
      const uint64_t nb = (mi < bw) | (P < mi);
      S[i] = P - mi;
      bw = nb;
    }
  }
  const int t = top_bit<W>(S);
  DF res = zero();
  if (t < 0) return res;
  res.sign = sign;
  if (t < p) {  // exact (see fastfloat.h add_t)
    const int sh = p - 1 - t;
    shl_limbs<W>(S, sh >> 6);
    shl_bits<W>(S, sh & 63);
#pragma unroll
    for (int i = 0; i < N; ++i) res.m[i] = S[i];
    res.exp = x.exp - 64 - sh;
    return res;
  }
  const int sh = t - p + 1;
  res.exp = x.exp - 64 + sh;
  uint64_t o[N];
  const bool up = shr_round<W, N>(S, sh, sticky, p, o);
#pragma unroll
  for (int i = 0; i < N; ++i) res.m[i] = o[i];
  if (up) {
    set_pow2<N>(res, p);
    res.exp += 1;
  }
  return res;
}

template <int N> LFI DF mul(const DF &a, const DF &b, int p) {
  if (a.sign == 0 || b.sign == 0) return zero();
  // column-wise product into 2N limbs; the 128-bit partial products via
  // __umul64hi, carries in a three-word accumulator
  uint64_t w[2 * N];
  uint64_t c0 = 0, c1 = 0, c2 = 0;
#pragma unroll
  for (int k = 0; k < 2 * N - 1; ++k) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const int j = k - i;
      if (j < 0 || j >= N) continue;
      const uint64_t lo = a.m[i] * b.m[j], hi = __umul64hi(a.m[i], b.m[j]);
      c0 += lo;
      const uint64_t k1 = c0 < lo;
      const uint64_t h = hi + k1;   // hi <= 2^64 - 2: no overflow
      c1 += h;
      c2 += c1 < h;
    }
    w[k] = c0;
    c0 = c1;
    c1 = c2;
    c2 = 0;
  }
  w[2 * N - 1] = c0;
  const bool full = get_bit<2 * N>(w, 2 * p - 1);
  const int sh = full ? p : p - 1;
  DF res = zero();
  res.sign = a.sign * b.sign;
  res.exp = a.exp + b.exp + sh;
  uint64_t o[N];
  const bool up = shr_round<2 * N, N>(w, sh, false, p, o);
#pragma unroll
  for (int i = 0; i < N; ++i) res.m[i] = o[i];
  if (up) {
    set_pow2<N>(res, p);
    res.exp += 1;
  }
  return res;
}

LFI DF neg(const DF &a) {
  DF r = a;
  r.sign = -a.sign;
  return r;
}

}  // namespace lf
