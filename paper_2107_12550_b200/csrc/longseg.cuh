// longwarp.cuh on half warps: two values per warp, each on a 16-lane
// segment (lane t of a segment holds limb t; the 2p-bit product of p <= 512
// needs 16 limbs), so the residual's product kernel forms two products per
// instruction stream.  Every collective uses the segment's mask (segments
// may take different branches); the arithmetic is longwarp.cuh's, step for
// step -- the same bits.
//
// (longwarp.cuh:) Warp-cooperative correctly rounded long floats for the
// device residual: one warp per value, lane t holding 64-bit limb t of the
// mantissa (limbs beyond the value's are zero).  Same results as longfloat.cuh / the host's
// fastfloat.h (exact result rounded once to p bits, half to even), with
// the limb loops replaced by lane-parallel steps: shuffles for limb shifts,
// ballots for sticky bits, and carry-lookahead over the lanes (generate /
// propagate masks) for multi-limb addition.  Sign and exponent are
// uniform across the warp, so control flow is warp-uniform.
#pragma once
#include <cstdint>

namespace ls {

#define LSI __device__ __forceinline__
constexpr int SEG = 16;
// this lane's segment mask and base lane
LSI unsigned seg_mask() { return (threadIdx.x & 16) ? 0xffff0000u : 0x0000ffffu; }
LSI int seg_base() { return threadIdx.x & 16; }

struct WV {        // this lane's view of a long float
  uint64_t m;      // limb `lane` of the mantissa (p bits, top bit p - 1)
  int64_t exp;     // value = sign * mantissa * 2^exp
  int sign;        // 0: zero
};

LSI int lane_id() { return threadIdx.x & 15; }
LSI uint64_t shfl(uint64_t v, int src) {
  const uint64_t r = __shfl_sync(seg_mask(), v, src & 15, SEG);
  return (src >= 0 && src < SEG) ? r : 0ull;
}
// the segment's 16 vote bits
LSI unsigned ballot(bool p) {
  return (__ballot_sync(seg_mask(), p) >> seg_base()) & 0xffffu;
}
// a condition every lane evaluates alike, as a vote: branches on it are
// warp-uniform to the compiler too, so the shuffles after them need no
// divergence handling
LSI bool uni(bool p) { return __all_sync(seg_mask(), p); }

// limbs >> s bits (s >= 0)
LSI uint64_t shr(uint64_t v, int s) {
  const int q = s >> 6, r = s & 63, t = lane_id();
  const uint64_t lo = shfl(v, t + q), hi = shfl(v, t + q + 1);
  return r ? (lo >> r) | (hi << (64 - r)) : lo;
}
// limbs << s bits (s >= 0)
LSI uint64_t shl(uint64_t v, int s) {
  const int q = s >> 6, r = s & 63, t = lane_id();
  const uint64_t hi = shfl(v, t - q), lo = shfl(v, t - q - 1);
  return r ? (hi << r) | (lo >> (64 - r)) : hi;
}
LSI bool get_bit(uint64_t v, int pos) {
  const uint64_t w = shfl(v, pos >> 6);
  return pos >= 0 && ((w >> (pos & 63)) & 1ull);
}
// any set bit strictly below bit position pos
LSI bool any_below(uint64_t v, int pos) {
  const int lo = 64 * lane_id();
  const uint64_t mask = pos >= lo + 64 ? ~0ull
                        : (pos > lo ? ((1ull << (pos - lo)) - 1ull) : 0ull);
  return ballot((v & mask) != 0ull) != 0u;
}
LSI int top_bit(uint64_t v) {
  const unsigned nz = ballot(v != 0ull);
  if (uni(nz == 0u)) return -1;
  const int h = 31 - __clz((int)nz);
  return 64 * h + 63 - __clzll((long long)shfl(v, h));
}
// carries into every lane from generate / propagate masks and a carry
// into lane 0 (disjoint g and p): ((g << 1 | cin) + p) ^ p
LSI bool carry_in(bool g, bool p, bool cin) {
  const unsigned G = ballot(g), P = ballot(p);
  const unsigned C = ((((G << 1) | (cin ? 1u : 0u)) + P) ^ P) & 0xffffu;
  return (C >> lane_id()) & 1u;
}
// x + y + cin over the lanes
LSI uint64_t add_limbs(uint64_t x, uint64_t y, bool cin) {
  const uint64_t s = x + y;
  return s + (carry_in(s < x, s == ~0ull, cin) ? 1ull : 0ull);
}
// x - y - bin over the lanes (x >= y + bin as numbers)
LSI uint64_t sub_limbs(uint64_t x, uint64_t y, bool bin) {
  const uint64_t d = x - y;
  return d - (carry_in(x < y, d == 0ull, bin) ? 1ull : 0ull);
}

LSI WV zero() { return WV{0ull, 0, 0}; }

// S (exact, top bit t >= p - 1 ... any) rounded to p bits: the mantissa
// limbs and the exponent adjustment; `sticky` marks bits lost before
LSI void round_into(uint64_t S, int t, bool sticky, int p, int64_t base_exp,
                    WV &r) {
  if (uni(t < p)) {  // fits: exact
    const int sh = p - 1 - t;
    r.m = shl(S, sh);
    r.exp = base_exp - sh;
    return;
  }
  const int sh = t - p + 1;
  uint64_t o = shr(S, sh);
  r.exp = base_exp + sh;
  const bool half = get_bit(S, sh - 1);
  const bool below = sticky || any_below(S, sh - 1);
  const bool lsb = shfl(o, 0) & 1ull;
  if (uni(half && (below || lsb))) {
    o = add_limbs(o, 0ull, true);
    if (uni(get_bit(o, p))) {  // rounded up to 2^p
      const int l = (p - 1) >> 6;
      o = lane_id() == l ? (1ull << ((p - 1) & 63)) : 0ull;
      r.exp += 1;
    }
  }
  r.m = o;
}

LSI WV add(const WV &a, const WV &b, int p) {
  if (uni(a.sign == 0)) return b;
  if (uni(b.sign == 0)) return a;
  const bool ax = a.exp >= b.exp;
  const WV &x = ax ? a : b;
  const WV &y = ax ? b : a;
  const int64_t d64 = x.exp - y.exp;
  if (uni(d64 >= p + 3)) return x;
  const int d = (int)d64;
  // frame: one guard limb below the mantissas
  const uint64_t X = shfl(x.m, lane_id() - 1);
  const uint64_t Yf = shfl(y.m, lane_id() - 1);
  const bool sticky = any_below(Yf, d);
  const uint64_t Y = shr(Yf, d);
  int sign = x.sign;
  uint64_t S;
  if (uni(x.sign == y.sign)) {
    S = add_limbs(X, Y, false);
  } else {
    bool swap = false;
    if (uni(d == 0)) {
      const unsigned D = ballot(X != Y);
      if (uni(D == 0u)) return zero();
      const int h = 31 - __clz((int)D);
      swap = shfl(X, h) < shfl(Y, h);
      if (swap) sign = y.sign;
    }
    S = swap ? sub_limbs(Y, X, sticky) : sub_limbs(X, Y, sticky);
  }
  WV r;
  r.sign = sign;
  const int t = top_bit(S);
  if (uni(t < 0)) return zero();
  round_into(S, t, sticky, p, x.exp - 64, r);
  return r;
}

LSI WV mul(const WV &a, const WV &b, int p) {
  if (uni(a.sign == 0 || b.sign == 0)) return zero();
  const int t = lane_id();
  // lane t: row products a_t * b_s for the 8 limbs s of b (limbs >= 8 are
  // zero for p <= 512); column t + s gets lo, t + s + 1 gets hi.  Round s:
  // lane u collects lo from lane u - s and hi from lane u - s - 1.
  uint64_t c0 = 0ull, c1 = 0ull, c2 = 0ull;
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const uint64_t bs = shfl(b.m, s);
    const uint64_t lo = a.m * bs, hi = __umul64hi(a.m, bs);
    const uint64_t vlo = shfl(lo, t - s), vhi = shfl(hi, t - s - 1);
    c0 += vlo;
    uint64_t k = c0 < vlo;
    c1 += k;
    c2 += c1 < k;
    c0 += vhi;
    k = c0 < vhi;
    c1 += k;
    c2 += c1 < k;
  }
  // column t = c0 + 2^64 c1 + 2^128 c2: limbs of the product
  const uint64_t x1 = shfl(c1, t - 1), x2 = shfl(c2, t - 2);
  uint64_t s1 = c0 + x1;
  uint64_t k = s1 < x1;
  const uint64_t s2 = s1 + x2;
  k += s2 < x2;                        // 0..2 into the next column
  const uint64_t kin = shfl(k, t - 1);
  const uint64_t s3 = s2 + kin;
  const uint64_t P = s3 + (carry_in(s3 < kin, s3 == ~0ull, false) ? 1ull : 0ull);
  // round the 2p- or (2p-1)-bit product to p bits
  const bool full = get_bit(P, 2 * p - 1);
  WV r;
  r.sign = a.sign * b.sign;
  round_into(P, full ? 2 * p - 1 : 2 * p - 2, false, p, a.exp + b.exp, r);
  return r;
}

LSI WV neg(const WV &a) { return WV{a.m, a.exp, -a.sign}; }

}  // namespace ls
