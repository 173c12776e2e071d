// Multi-component (DD/TD/QD) binary64 arithmetic as sm_100a device inlines.
//
// Every routine reproduces, operation for operation, the kernels of the
// reference (/root/reference/pkg/src/mpcore/mcfloat.py) so results are
// bit-identical:
//   two_sum        mcfloat.py:55-65     (Knuth, 6 DADD)
//   quick_two_sum  mcfloat.py:68-76     (3 DADD)
//   two_prod       mcfloat.py:79-102    Dekker in the reference; here DMUL +
//                                       DFMA, which yields the identical
//                                       (p, e) pair for every operand pair
//                                       whose product neither overflows nor
//                                       underflows (SURVEY finding 3).
//   sweep/cascade/compress            mcfloat.py:109-143
//   add2/mul2/add3/mul3/add4/mul4     mcfloat.py:189-257 (term lists verbatim)
//   mul_scalar / div                  mcfloat.py:286-318
//
// Every operation goes through an explicit round-to-nearest intrinsic
// (__dadd_rn/__dmul_rn/__fma_rn), so no contraction can change a bit even if
// the file were built without -fmad=false (the build uses it anyway).
#pragma once
#include <cstdint>

namespace mc {

#define MCI __device__ __forceinline__

MCI double add_(double a, double b) { return __dadd_rn(a, b); }
MCI double sub_(double a, double b) { return __dsub_rn(a, b); }
MCI double mul_(double a, double b) { return __dmul_rn(a, b); }

MCI void two_sum(double a, double b, double &s, double &e) {
  s = add_(a, b);
  double bb = sub_(s, a);
  e = add_(sub_(a, sub_(s, bb)), sub_(b, bb));
}
MCI double fsum_head(double a, double b) { return add_(a, b); }
MCI void quick_two_sum(double a, double b, double &s, double &e) {
  s = add_(a, b);
  e = sub_(b, sub_(s, a));
}
MCI void two_prod(double a, double b, double &p, double &e) {
  p = mul_(a, b);
  e = __fma_rn(a, b, -p);
}
// The reference's two_prod is Dekker's splitting form (mcfloat.py:79-102).
// Its error term equals the FMA form's RN(a b - p) whenever the split cannot
// overflow (|a|, |b| < 2**996) and no partial product underflows (a, b
// normal, |p| >= 2**-959), and both are +0 when an operand is +-0 and the
// other's split cannot overflow (tests/test_range_edges.py).
// The default build relies on that band (every BASELINE input lies deep
// inside it).  libmpcore_exact.so (MPCORE_EXACT_RANGE=1) is compiled with
// MPCORE_EXACT_TWO_PROD: each multiplication routine forms its products the
// FMA way, tests all its pairs on the integer pipe (exponent fields), and
// only outside the band re-forms its error terms with tp_ref -- the
// reference's own sequence (NaN error terms for huge operands, its tails
// near underflow) -- so every result keeps the reference's bits everywhere,
// for 12-19 % of the FP64-bound throughput.
#ifdef MPCORE_EXACT_TWO_PROD
MCI bool tp_ok(double a, double b, double p) {
  const unsigned ma = (unsigned)__double2hiint(a) & 0x7ff00000u,
                 mb = (unsigned)__double2hiint(b) & 0x7ff00000u,
                 mp = (unsigned)__double2hiint(p) & 0x7ff00000u;
  return (ma - 0x00100000u < (2018u << 20)) &
         (mb - 0x00100000u < (2018u << 20)) &
         (mp - (64u << 20) < (1983u << 20));
}
static __device__ __noinline__ double tp_ref(double a, double b, double p) {
  const unsigned ha = (unsigned)__double2hiint(a),
                 hb = (unsigned)__double2hiint(b);
  const bool za = ((ha & 0x7fffffffu) | (unsigned)__double2loint(a)) == 0u;
  const bool zb = ((hb & 0x7fffffffu) | (unsigned)__double2loint(b)) == 0u;
  if ((za && (hb & 0x7ff00000u) < (2019u << 20)) ||
      (zb && (ha & 0x7ff00000u) < (2019u << 20)) || tp_ok(a, b, p))
    return __fma_rn(a, b, -p);
  const double S = 134217729.0;  // _SPLIT = 2**27 + 1
  double t = __dmul_rn(S, a);
  const double ahi = __dsub_rn(t, __dsub_rn(t, a)), alo = __dsub_rn(a, ahi);
  t = __dmul_rn(S, b);
  const double bhi = __dsub_rn(t, __dsub_rn(t, b)), blo = __dsub_rn(b, bhi);
  return __dadd_rn(__dadd_rn(__dadd_rn(__dsub_rn(__dmul_rn(ahi, bhi), p),
                                       __dmul_rn(ahi, blo)),
                             __dmul_rn(alo, bhi)),
                   __dmul_rn(alo, blo));
}
#define MC_EXACT_1(A0, B0, P, Q)                                  \
  if (__builtin_expect(!tp_ok(A0, B0, P), 0)) Q = tp_ref(A0, B0, P);
#define MC_EXACT_6(a, b)                                                   \
  if (__builtin_expect(!(tp_ok(a[0], b[0], p00) & tp_ok(a[0], b[1], p01) & \
                         tp_ok(a[1], b[0], p10) & tp_ok(a[0], b[2], p02) & \
                         tp_ok(a[1], b[1], p11) & tp_ok(a[2], b[0], p20)), \
                       0)) {                                              \
    q00 = tp_ref(a[0], b[0], p00);                                        \
    q01 = tp_ref(a[0], b[1], p01);                                        \
    q10 = tp_ref(a[1], b[0], p10);                                        \
    q02 = tp_ref(a[0], b[2], p02);                                        \
    q11 = tp_ref(a[1], b[1], p11);                                        \
    q20 = tp_ref(a[2], b[0], p20);                                        \
  }
#else
#define MC_EXACT_1(A0, B0, P, Q)
#define MC_EXACT_6(a, b)
#endif

// _sweep: bottom-up two_sum chain; residuals overwrite t[0..M-2].
template <int M> MCI double sweep(double (&t)[M]) {
  double s = t[M - 1];
#pragma unroll
  for (int i = M - 2; i >= 0; --i) {
    double e;
    two_sum(t[i], s, s, e);
    t[i] = e;
  }
  return s;
}
// The final sweep of a cascade discards its residuals: only the running sum.
template <int M> MCI double sweep_last(const double (&t)[M]) {
  double s = t[M - 1];
#pragma unroll
  for (int i = M - 2; i >= 0; --i) s = add_(t[i], s);
  return s;
}
// _cascade(terms, K) followed by _compress, for M input terms.
template <int M, int K> struct Cascade {
  static MCI void run(double (&t)[M], double *o) {
    if constexpr (K == 1) {
      o[0] = sweep_last<M>(t);
    } else {
      o[0] = sweep<M>(t);
      double r[M - 1];
#pragma unroll
      for (int i = 0; i < M - 1; ++i) r[i] = t[i];
      Cascade<M - 1, K - 1>::run(r, o + 1);
    }
  }
};
template <int K> MCI void compress(double *c) {
  double carry = c[0];
#pragma unroll
  for (int i = 1; i < K; ++i) {
    double s;
    quick_two_sum(carry, c[i], s, carry);
    c[i - 1] = s;
  }
  c[K - 1] = carry;
}
template <int M, int K> MCI void cascade_compress(double (&t)[M], double *o) {
  Cascade<M, K>::run(t, o);
  compress<K>(o);
}

// ------------------------------------------------------------ add / mul ----
template <int K> struct V { double c[K]; };

MCI void add2(const double *a, const double *b, double *o) {
  double s0, e0, s1, e1;
  two_sum(a[0], b[0], s0, e0);
  two_sum(a[1], b[1], s1, e1);
  e0 = add_(e0, s1);
  quick_two_sum(s0, e0, s0, e0);
  e0 = add_(e0, e1);
  quick_two_sum(s0, e0, o[0], o[1]);
}
MCI void mul2(const double *a, const double *b, double *o) {
  double p, e;
  two_prod(a[0], b[0], p, e);
  MC_EXACT_1(a[0], b[0], p, e)
  e = add_(e, add_(mul_(a[0], b[1]), mul_(a[1], b[0])));
  quick_two_sum(p, e, o[0], o[1]);
}
MCI void add3(const double *a, const double *b, double *o) {
  double s0, e0, s1, e1, s2, e2;
  two_sum(a[0], b[0], s0, e0);
  two_sum(a[1], b[1], s1, e1);
  two_sum(a[2], b[2], s2, e2);
  double t[6] = {s0, s1, e0, s2, e1, e2};
  cascade_compress<6, 3>(t, o);
}
MCI void mul3(const double *a, const double *b, double *o) {
  double p00, q00, p01, q01, p10, q10, p02, q02, p11, q11, p20, q20;
  two_prod(a[0], b[0], p00, q00);
  two_prod(a[0], b[1], p01, q01);
  two_prod(a[1], b[0], p10, q10);
  two_prod(a[0], b[2], p02, q02);
  two_prod(a[1], b[1], p11, q11);
  two_prod(a[2], b[0], p20, q20);
  MC_EXACT_6(a, b)
  double t3 = add_(add_(add_(q02, q11), q20),
                   add_(mul_(a[1], b[2]), mul_(a[2], b[1])));
  double t[10] = {p00, p01, p10, q00, p02, p11, p20, q01, q10, t3};
  cascade_compress<10, 3>(t, o);
}
MCI void add4(const double *a, const double *b, double *o) {
  double s0, e0, s1, e1, s2, e2, s3, e3;
  two_sum(a[0], b[0], s0, e0);
  two_sum(a[1], b[1], s1, e1);
  two_sum(a[2], b[2], s2, e2);
  two_sum(a[3], b[3], s3, e3);
  double t[8] = {s0, s1, e0, s2, e1, s3, e2, e3};
  cascade_compress<8, 4>(t, o);
}
MCI void mul4(const double *a, const double *b, double *o) {
  double p00, q00, p01, q01, p10, q10, p02, q02, p11, q11, p20, q20;
  two_prod(a[0], b[0], p00, q00);
  two_prod(a[0], b[1], p01, q01);
  two_prod(a[1], b[0], p10, q10);
  two_prod(a[0], b[2], p02, q02);
  two_prod(a[1], b[1], p11, q11);
  two_prod(a[2], b[0], p20, q20);
  MC_EXACT_6(a, b)
  double t3 = add_(add_(add_(q02, q11), q20),
                   add_(add_(mul_(a[0], b[3]), mul_(a[3], b[0])),
                        add_(mul_(a[1], b[2]), mul_(a[2], b[1]))));
  double t[10] = {p00, p01, p10, q00, p02, p11, p20, q01, q10, t3};
  cascade_compress<10, 4>(t, o);
}

template <int K> MCI void add(const double *a, const double *b, double *o) {
  if constexpr (K == 2) add2(a, b, o);
  else if constexpr (K == 3) add3(a, b, o);
  else add4(a, b, o);
}
template <int K> MCI void mul(const double *a, const double *b, double *o) {
  if constexpr (K == 2) mul2(a, b, o);
  else if constexpr (K == 3) mul3(a, b, o);
  else mul4(a, b, o);
}
// acc <- add(acc, mul(a, b))   (the reference's madd; accumulator first)
template <int K> MCI void madd(double *acc, const double *a, const double *b) {
  double t[K], o[K];
  mul<K>(a, b, t);
  add<K>(acc, t, o);
#pragma unroll
  for (int c = 0; c < K; ++c) acc[c] = o[c];
}
// _mul_scalar_t: terms = [p_0..p_{K-1}], tails = [q_0..q_{K-1}]
template <int K> MCI void mul_scalar(const double *a, double x, double *o) {
  double t[2 * K];
#pragma unroll
  for (int c = 0; c < K; ++c) two_prod(a[c], x, t[c], t[K + c]);
#ifdef MPCORE_EXACT_TWO_PROD
  bool ok = true;
#pragma unroll
  for (int c = 0; c < K; ++c) ok &= tp_ok(a[c], x, t[c]);
  if (__builtin_expect(!ok, 0)) {
#pragma unroll
    for (int c = 0; c < K; ++c) t[K + c] = tp_ref(a[c], x, t[c]);
  }
#endif
  cascade_compress<2 * K, K>(t, o);
}
// RN(1/b) when b lies well inside the normal range (|exponent| <= 423), else
// 0: the hint that lets ddiv_y skip the division routine.
MCI double recip_hint(double b) {
  const unsigned eb = ((unsigned)__double2hiint(b) >> 20) & 0x7ffu;
  return eb - 600u <= 846u ? __ddiv_rn(1.0, b) : 0.0;
}
// RN(a / b) given y = recip_hint(b), bit-identical to __ddiv_rn(a, b).
// With y = RN(1/b): q0 = RN(a y) is within 1.5 ulp of a/b, one correction
// q1 = RN(q0 + RN(a - q0 b) y) is within 1/2 ulp plus ~2^-51 ulp, and from
// there r = a - q1 b is exact and RN(q1 + r y) = RN(a/b) (Markstein's
// theorem: a/b is at least 2^-53 ulp / b from any midpoint, the error term
// (a/b - q1)(by - 1) stays below it for b in [1, 2)).  Both operands within
// 2^+-423 keep every intermediate normal; anything else (zero remainders,
// huge/tiny values, Inf, NaN) takes __ddiv_rn.  tests/test_gpu_div.py and
// tools/divcheck.cu check it against __ddiv_rn on hard cases.
// (out of line: inlined, the compiler if-converts the routine's own fast
// path into the caller and the select waits for it)
static __device__ __noinline__ double ddiv_slow(double a, double b) {
  return __ddiv_rn(a, b);
}
MCI double ddiv_y(double a, double b, double y) {
  // the corrections run unconditionally; the range test overlaps them and
  // only a rejected operand pays for the division routine
  double q = __dmul_rn(a, y);
  double r = __fma_rn(-q, b, a);
  q = __fma_rn(r, y, q);
  r = __fma_rn(-q, b, a);
  q = __fma_rn(r, y, q);
  const unsigned ea = ((unsigned)__double2hiint(a) >> 20) & 0x7ffu;
  if (y == 0.0 || ea - 600u > 846u) q = ddiv_slow(a, b);
  return q;
}
// _div_t: K+1 head-quotient digits of long division; b[0] != 0 required.
// y = recip_hint(b[0]) (one division per divisor, off the digit chain).
template <int K>
MCI void div_y(const double *a, const double *b, double y, double *o) {
  double digits[K + 1], r[K];
#pragma unroll
  for (int c = 0; c < K; ++c) r[c] = a[c];
#pragma unroll
  for (int i = 0; i < K + 1; ++i) {
    double qi = ddiv_y(r[0], b[0], y);
    digits[i] = qi;
    if (i < K) {
      double t[K], nr[K];
      mul_scalar<K>(b, qi, t);
#pragma unroll
      for (int c = 0; c < K; ++c) t[c] = -t[c];
      add<K>(r, t, nr);
#pragma unroll
      for (int c = 0; c < K; ++c) r[c] = nr[c];
    }
  }
  cascade_compress<K + 1, K>(digits, o);
}
template <int K> MCI void div(const double *a, const double *b, double *o) {
  div_y<K>(a, b, recip_hint(b[0]), o);
}
// div(1, b): the first digit RN(1/b[0]) is the hint itself
template <int K> MCI void recip(const double *b, double *o) {
  double digits[K + 1], r[K];
  const double y = recip_hint(b[0]);
  r[0] = 1.0;
#pragma unroll
  for (int c = 1; c < K; ++c) r[c] = 0.0;
#pragma unroll
  for (int i = 0; i < K + 1; ++i) {
    double qi = i == 0 ? (y != 0.0 ? y : __ddiv_rn(1.0, b[0]))
                       : ddiv_y(r[0], b[0], y);
    digits[i] = qi;
    if (i < K) {
      double t[K], nr[K];
      mul_scalar<K>(b, qi, t);
#pragma unroll
      for (int c = 0; c < K; ++c) t[c] = -t[c];
      add<K>(r, t, nr);
#pragma unroll
      for (int c = 0; c < K; ++c) r[c] = nr[c];
    }
  }
  cascade_compress<K + 1, K>(digits, o);
}

// _sqrt_t (mcfloat.py:324-340): Newton on y ~ 1/sqrt(a) seeded from
// RN(1 / RN(sqrt(a0))) (both IEEE correctly rounded, as Python's
// 1.0 / math.sqrt), 2/2/3 steps for DD/TD/QD, then one Heron correction;
// every step in the reference's operand order.  a0 >= 0 is the caller's
// check (the reference raises DomainError); an exact zero gives zeros.
template <int K> MCI void sqrt(const double *a, double *o) {
  if (a[0] == 0.0) {
#pragma unroll
    for (int c = 0; c < K; ++c) o[c] = 0.0;
    return;
  }
  constexpr int STEPS = K == 4 ? 3 : 2;
  double one[K], y[K];
#pragma unroll
  for (int c = 0; c < K; ++c) one[c] = y[c] = 0.0;
  one[0] = 1.0;
  y[0] = __ddiv_rn(1.0, __dsqrt_rn(a[0]));
#pragma unroll 1
  for (int it = 0; it < STEPS; ++it) {
    double yy[K], ayy[K], r[K], yr[K], h[K], ny[K];
    mul<K>(y, y, yy);
    mul<K>(a, yy, ayy);
#pragma unroll
    for (int c = 0; c < K; ++c) ayy[c] = -ayy[c];
    add<K>(one, ayy, r);
    mul<K>(y, r, yr);
    mul_scalar<K>(yr, 0.5, h);
    add<K>(y, h, ny);
#pragma unroll
    for (int c = 0; c < K; ++c) y[c] = ny[c];
  }
  double s[K], ss[K], e[K], yh[K], ey[K];
  mul<K>(a, y, s);
  mul<K>(s, s, ss);
#pragma unroll
  for (int c = 0; c < K; ++c) ss[c] = -ss[c];
  add<K>(a, ss, e);
  mul_scalar<K>(y, 0.5, yh);
  mul<K>(e, yh, ey);
  add<K>(s, ey, o);
}

// Exact FP64 instruction counts per op (FMA two_prod).
template <int K> struct Cost;
template <> struct Cost<2> { static constexpr int madd = 29, mul = 9, add = 20; };
template <> struct Cost<3> { static constexpr int madd = 264, mul = 168, add = 96; };
template <> struct Cost<4> { static constexpr int madd = 376, mul = 211, add = 165; };

}  // namespace mc
