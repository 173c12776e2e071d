// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the reference's short-precision (DD/TD/QD) hot path:
// the error-free transformations and k-component kernels of
// /root/reference/pkg/src/mpcore/mcfloat.py and the lane-path dense kernels
// of /root/reference/pkg/src/mpcore/linalg.py.  Only tests/, bench.py's
// cpu_baseline / --impl reference leg and __graft_entry__.smoke() may load
// this library, and only as the checker (or the timed CPU baseline).  The
// product (paper_2107_12550_b200/) never links or calls it.
//
// Parity pin: tests/test_oracle_golden.py checks every entry point against
// golden vectors produced by the reference itself (tests/golden/, made by
// tests/golden/make_golden.py importing /root/reference/pkg/src/mpcore).
//
// Arithmetic discipline: IEEE binary64 round-to-nearest,
// built with -ffp-contract=off (no FMA contraction), two_prod in Dekker's
// split form exactly as the reference writes it (mcfloat.py:79-102).  The
// product's device code uses the FMA form; the two agree bitwise in range,
// which the parity tests re-check on every run.
//
// Layout: planar, component-major.  A k-component n x m matrix is k planes of
// n*m doubles, row-major within a plane (simd.py:36-48).
//
// Loops that are independent per output element are OpenMP-parallel and
// written so gcc vectorises them (AVX2 here): every element still sees the
// reference's operation chain in the reference's order, so threading and
// vectorisation do not change a bit.

#include <cmath>
#include <cstdint>
#include <cstring>
#include <cstdlib>
#include <vector>
#include <algorithm>
#ifdef _OPENMP
#include <omp.h>
#endif

#define RESTRICT __restrict__
#define INL static inline __attribute__((always_inline))

namespace {

// ---------------------------------------------------------------- EFTs ----
// mcfloat.py:55-65
INL void two_sum(double a, double b, double &s, double &e) {
  s = a + b;
  double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}
// mcfloat.py:68-76
INL void quick_two_sum(double a, double b, double &s, double &e) {
  s = a + b;
  e = b - (s - a);
}
// mcfloat.py:82-89 (_SPLIT = 2**27 + 1)
INL void split(double a, double &hi, double &lo) {
  double t = 134217729.0 * a;
  hi = t - (t - a);
  lo = a - hi;
}
// mcfloat.py:92-102 (Dekker)
INL void two_prod(double a, double b, double &p, double &e) {
  p = a * b;
#ifdef MCREF_FMA_TWO_PROD
  // (libmcref_fma.so only: the FMA form the CUDA path uses)
  e = std::fma(a, b, -p);
  return;
#endif
  double ahi, alo, bhi, blo;
  split(a, ahi, alo);
  split(b, bhi, blo);
  e = ((ahi * bhi - p) + ahi * blo + alo * bhi) + alo * blo;
}

// ------------------------------------------------------ renormalisation ----
// _sweep (mcfloat.py:109-117): bottom-up two_sum chain over t[0..m).
// Overwrites t[0..m-1) with the residuals (rest[i]) and returns the head.
INL double sweep(double *t, int m) {
  double s = t[m - 1];
  for (int i = m - 2; i >= 0; --i) {
    double e;
    two_sum(t[i], s, s, e);
    t[i] = e;
  }
  return s;
}
// _cascade (mcfloat.py:120-132): peel k heads; t is consumed.
INL void cascade(double *t, int m, int k, double *out) {
  for (int c = 0; c < k; ++c) {
    out[c] = sweep(t, m);
    --m;
  }
}
// _compress (mcfloat.py:135-143): top-down quick_two_sum polish.
INL void compress(double *c, int k) {
  double carry = c[0];
  for (int i = 1; i < k; ++i) {
    double s;
    quick_two_sum(carry, c[i], s, carry);
    c[i - 1] = s;
  }
  c[k - 1] = carry;
}

// ------------------------------------------------------------- kernels ----
// _add2 (mcfloat.py:189-197)
INL void add2(const double *a, const double *b, double *o) {
  double s0, e0, s1, e1;
  two_sum(a[0], b[0], s0, e0);
  two_sum(a[1], b[1], s1, e1);
  e0 = e0 + s1;
  quick_two_sum(s0, e0, s0, e0);
  e0 = e0 + e1;
  quick_two_sum(s0, e0, s0, e0);
  o[0] = s0;
  o[1] = e0;
}
// _mul2 (mcfloat.py:200-204)
INL void mul2(const double *a, const double *b, double *o) {
  double p, e;
  two_prod(a[0], b[0], p, e);
  e = e + (a[0] * b[1] + a[1] * b[0]);
  quick_two_sum(p, e, o[0], o[1]);
}
// _add3 (mcfloat.py:207-214)
INL void add3(const double *a, const double *b, double *o) {
  double s0, e0, s1, e1, s2, e2;
  two_sum(a[0], b[0], s0, e0);
  two_sum(a[1], b[1], s1, e1);
  two_sum(a[2], b[2], s2, e2);
  double t[6] = {s0, s1, e0, s2, e1, e2};
  cascade(t, 6, 3, o);
  compress(o, 3);
}
// _mul3 (mcfloat.py:217-229)
INL void mul3(const double *a, const double *b, double *o) {
  double p00, q00, p01, q01, p10, q10, p02, q02, p11, q11, p20, q20;
  two_prod(a[0], b[0], p00, q00);
  two_prod(a[0], b[1], p01, q01);
  two_prod(a[1], b[0], p10, q10);
  two_prod(a[0], b[2], p02, q02);
  two_prod(a[1], b[1], p11, q11);
  two_prod(a[2], b[0], p20, q20);
  double t3 = (q02 + q11 + q20) + (a[1] * b[2] + a[2] * b[1]);
  double t[10] = {p00, p01, p10, q00, p02, p11, p20, q01, q10, t3};
  cascade(t, 10, 3, o);
  compress(o, 3);
}
// _add4 (mcfloat.py:232-241)
INL void add4(const double *a, const double *b, double *o) {
  double s0, e0, s1, e1, s2, e2, s3, e3;
  two_sum(a[0], b[0], s0, e0);
  two_sum(a[1], b[1], s1, e1);
  two_sum(a[2], b[2], s2, e2);
  two_sum(a[3], b[3], s3, e3);
  double t[8] = {s0, s1, e0, s2, e1, s3, e2, e3};
  cascade(t, 8, 4, o);
  compress(o, 4);
}
// _mul4 (mcfloat.py:244-257)
INL void mul4(const double *a, const double *b, double *o) {
  double p00, q00, p01, q01, p10, q10, p02, q02, p11, q11, p20, q20;
  two_prod(a[0], b[0], p00, q00);
  two_prod(a[0], b[1], p01, q01);
  two_prod(a[1], b[0], p10, q10);
  two_prod(a[0], b[2], p02, q02);
  two_prod(a[1], b[1], p11, q11);
  two_prod(a[2], b[0], p20, q20);
  double t3 = (q02 + q11 + q20) +
              ((a[0] * b[3] + a[3] * b[0]) + (a[1] * b[2] + a[2] * b[1]));
  double t[10] = {p00, p01, p10, q00, p02, p11, p20, q01, q10, t3};
  cascade(t, 10, 4, o);
  compress(o, 4);
}

template <int K> INL void add(const double *a, const double *b, double *o) {
  if (K == 2) add2(a, b, o);
  else if (K == 3) add3(a, b, o);
  else add4(a, b, o);
}
template <int K> INL void mul(const double *a, const double *b, double *o) {
  if (K == 2) mul2(a, b, o);
  else if (K == 3) mul3(a, b, o);
  else mul4(a, b, o);
}

// _mul_scalar_t (mcfloat.py:286-296)
template <int K> INL void mul_scalar(const double *a, double x, double *o) {
  double t[2 * K];
  for (int c = 0; c < K; ++c) two_prod(a[c], x, t[c], t[K + c]);
  cascade(t, 2 * K, K, o);
  compress(o, K);
}
// _div_t (mcfloat.py:304-318); caller guarantees b[0] != 0.
template <int K> static void divk(const double *a, const double *b, double *o) {
  double digits[K + 1], r[K], tmp[K];
  for (int c = 0; c < K; ++c) r[c] = a[c];
  for (int i = 0; i < K + 1; ++i) {
    double qi = r[0] / b[0];
    digits[i] = qi;
    if (i < K) {
      mul_scalar<K>(b, qi, tmp);
      for (int c = 0; c < K; ++c) tmp[c] = -tmp[c];
      double nr[K];
      add<K>(r, tmp, nr);
      for (int c = 0; c < K; ++c) r[c] = nr[c];
    }
  }
  cascade(digits, K + 1, K, o);
  compress(o, K);
}

// _sqrt_t (mcfloat.py:324-340); caller guarantees a[0] >= 0.
template <int K> static void sqrtk(const double *a, double *o) {
  if (a[0] == 0.0) {
    for (int c = 0; c < K; ++c) o[c] = 0.0;
    return;
  }
  const int steps = K == 4 ? 3 : 2;  // _SQRT_STEPS
  double one[K] = {}, y[K] = {};
  one[0] = 1.0;
  y[0] = 1.0 / std::sqrt(a[0]);
  for (int it = 0; it < steps; ++it) {
    double yy[K], ayy[K], r[K], yr[K], h[K], ny[K];
    mul<K>(y, y, yy);
    mul<K>(a, yy, ayy);
    for (int c = 0; c < K; ++c) ayy[c] = -ayy[c];
    add<K>(one, ayy, r);
    mul<K>(y, r, yr);
    mul_scalar<K>(yr, 0.5, h);
    add<K>(y, h, ny);
    for (int c = 0; c < K; ++c) y[c] = ny[c];
  }
  double s[K], ss[K], e[K], yh[K], ey[K];
  mul<K>(a, y, s);
  mul<K>(s, s, ss);
  for (int c = 0; c < K; ++c) ss[c] = -ss[c];
  add<K>(a, ss, e);
  mul_scalar<K>(y, 0.5, yh);
  mul<K>(e, yh, ey);
  add<K>(s, ey, o);
}

// --------------------------------------------------------- dense kernels ----
// Element (i, j) of plane c: p[c * plane + i * ld + j].

// _lu_lanes (linalg.py:422-449).  Returns 0, or 3 with *sing = step.
// np.argmax over |head| (linalg.py:429): the first NaN if any, else the
// first maximum -- "m beats the best so far" in that order
static inline bool pivot_better(double m, double best) {
  if (std::isnan(best)) return false;
  if (std::isnan(m)) return true;
  return m > best;
}

template <int K>
static int lu(int n, double *d, int32_t *swaps, int32_t *sing) {
  const size_t plane = (size_t)n * n;
  double one[K] = {1.0};
  for (int j = 0; j < n; ++j) {
    // pivot: first max of |head| over rows j..n-1 (linalg.py:429)
    int r = j;
    double best = std::fabs(d[(size_t)j * n + j]);
    for (int i = j + 1; i < n; ++i) {
      double m = std::fabs(d[(size_t)i * n + j]);
      if (pivot_better(m, best)) { best = m; r = i; }
    }
    if (r != j) {  // full-row swap (linalg.py:430-431)
      for (int c = 0; c < K; ++c) {
        double *pj = d + c * plane + (size_t)j * n;
        double *pr = d + c * plane + (size_t)r * n;
        for (int q = 0; q < n; ++q) std::swap(pj[q], pr[q]);
      }
    }
    swaps[j] = r;
    double piv[K];
    for (int c = 0; c < K; ++c) piv[c] = d[c * plane + (size_t)j * n + j];
    if (piv[0] == 0.0) { *sing = j; return 3; }   // linalg.py:433-436
    if (j + 1 == n) break;                       // linalg.py:437-438
    double recip[K];
    divk<K>(one, piv, recip);                    // linalg.py:439
    const int rows = n - j - 1;
#pragma omp parallel for schedule(static) if (rows > 64)
    for (int i = j + 1; i < n; ++i) {
      double a[K], m[K], negm[K];
      for (int c = 0; c < K; ++c) a[c] = d[c * plane + (size_t)i * n + j];
      mul<K>(a, recip, m);                       // linalg.py:441
      for (int c = 0; c < K; ++c) {
        d[c * plane + (size_t)i * n + j] = m[c];
        negm[c] = -m[c];
      }
      double *RESTRICT ri[K];
      const double *RESTRICT rj[K];
      for (int c = 0; c < K; ++c) {
        ri[c] = d + c * plane + (size_t)i * n;
        rj[c] = d + c * plane + (size_t)j * n;
      }
      // linalg.py:444-448: A_ic = add(A_ic, mul(-m_i, A_jc))
#pragma GCC ivdep
      for (int q = j + 1; q < n; ++q) {
        double u[K], t[K], x[K], o[K];
        for (int c = 0; c < K; ++c) { u[c] = rj[c][q]; x[c] = ri[c][q]; }
        mul<K>(negm, u, t);
        add<K>(x, t, o);
        for (int c = 0; c < K; ++c) ri[c][q] = o[c];
      }
    }
  }
  return 0;
}

// _lu_lanes restricted to an m x w block (row stride ld, plane stride pl):
// pivot over all m rows, exchange rows inside the block, update inside the
// block only.  The blocked/distributed factorisations are checked against
// compositions of this, trsm() and gemm_update() (all in the reference's
// per-element chain order).
template <int K>
static int lu_block(int m, int w, double *d, int64_t ld, int64_t pl,
                    int32_t *swaps, int32_t *sing) {
  double one[K] = {1.0};
  for (int j = 0; j < w; ++j) {
    int r = j;
    double best = std::fabs(d[(int64_t)j * ld + j]);
    for (int i = j + 1; i < m; ++i) {
      double v = std::fabs(d[(int64_t)i * ld + j]);
      if (pivot_better(v, best)) { best = v; r = i; }
    }
    if (r != j)
      for (int c = 0; c < K; ++c)
        for (int q = 0; q < w; ++q)
          std::swap(d[c * pl + (int64_t)j * ld + q], d[c * pl + (int64_t)r * ld + q]);
    swaps[j] = r;
    if (d[(int64_t)j * ld + j] == 0.0) { *sing = j; return 3; }
    if (j + 1 == m) break;
    double piv[K], recip[K];
    for (int c = 0; c < K; ++c) piv[c] = d[c * pl + (int64_t)j * ld + j];
    divk<K>(one, piv, recip);
#pragma omp parallel for schedule(static) if (m - j > 256)
    for (int i = j + 1; i < m; ++i) {
      double a[K], mm[K], negm[K];
      for (int c = 0; c < K; ++c) a[c] = d[c * pl + (int64_t)i * ld + j];
      mul<K>(a, recip, mm);
      for (int c = 0; c < K; ++c) {
        d[c * pl + (int64_t)i * ld + j] = mm[c];
        negm[c] = -mm[c];
      }
      for (int q = j + 1; q < w; ++q) {
        double u[K], t[K], x[K], o[K];
        for (int c = 0; c < K; ++c) {
          u[c] = d[c * pl + (int64_t)j * ld + q];
          x[c] = d[c * pl + (int64_t)i * ld + q];
        }
        mul<K>(negm, u, t);
        add<K>(x, t, o);
        for (int c = 0; c < K; ++c) d[c * pl + (int64_t)i * ld + q] = o[c];
      }
    }
  }
  return 0;
}

// U (w x ncols) <- chains add(U_jc, mul(-L_jt, U_tc)), t ascending (t < j)
template <int K>
static void trsm(int w, int ncols, const double *l, int64_t ldl, int64_t pl,
                 double *u, int64_t ldu, int64_t pu) {
#pragma omp parallel for schedule(static) if (ncols > 64)
  for (int q = 0; q < ncols; ++q)
    for (int j = 1; j < w; ++j)
      for (int t = 0; t < j; ++t) {
        double a[K], b[K], x[K], tt[K], o[K];
        for (int c = 0; c < K; ++c) {
          a[c] = -l[c * pl + (int64_t)j * ldl + t];
          b[c] = u[c * pu + (int64_t)t * ldu + q];
          x[c] = u[c * pu + (int64_t)j * ldu + q];
        }
        mul<K>(a, b, tt);
        add<K>(x, tt, o);
        for (int c = 0; c < K; ++c) u[c * pu + (int64_t)j * ldu + q] = o[c];
      }
}

// C (M x N) <- fold_p add(C_ij, mul(-A_ip, B_pj)), p ascending
template <int K>
static void gemm_update(int M, int N, int KK, const double *a, int64_t lda,
                        int64_t pa, const double *b, int64_t ldb, int64_t pb,
                        double *cm, int64_t ldc, int64_t pc) {
#pragma omp parallel for schedule(static) if (M > 16)
  for (int i = 0; i < M; ++i)
    for (int p = 0; p < KK; ++p) {
      double x[K];
      for (int c = 0; c < K; ++c) x[c] = -a[c * pa + (int64_t)i * lda + p];
      for (int j = 0; j < N; ++j) {
        double y[K], t[K], z[K], o[K];
        for (int c = 0; c < K; ++c) {
          y[c] = b[c * pb + (int64_t)p * ldb + j];
          z[c] = cm[c * pc + (int64_t)i * ldc + j];
        }
        mul<K>(x, y, t);
        add<K>(z, t, o);
        for (int c = 0; c < K; ++c) cm[c * pc + (int64_t)i * ldc + j] = o[c];
      }
    }
}

// _solve_lanes (linalg.py:496-521); x holds b on entry.
template <int K>
static void solve(int n, const double *d, const int32_t *swaps, double *x) {
  const size_t plane = (size_t)n * n;
  for (int j = 0; j < n; ++j) {
    int r = swaps[j];
    if (r != j)
      for (int c = 0; c < K; ++c) std::swap(x[c * n + j], x[c * n + r]);
  }
  // forward, column sweeps: x_i = add(x_i, mul(-L_ij, x_j))  (504-509)
  for (int j = 0; j < n - 1; ++j) {
    double xj[K];
    for (int c = 0; c < K; ++c) xj[c] = x[c * n + j];
    for (int i = j + 1; i < n; ++i) {
      double l[K], t[K], xi[K], o[K];
      for (int c = 0; c < K; ++c) {
        l[c] = -d[c * plane + (size_t)i * n + j];
        xi[c] = x[c * n + i];
      }
      mul<K>(l, xj, t);
      add<K>(xi, t, o);
      for (int c = 0; c < K; ++c) x[c * n + i] = o[c];
    }
  }
  // backward: x_j = div(x_j, U_jj); x_i = add(x_i, mul(U_ij, -x_j)) (510-520)
  for (int j = n - 1; j >= 0; --j) {
    double xj[K], ujj[K], q[K];
    for (int c = 0; c < K; ++c) {
      xj[c] = x[c * n + j];
      ujj[c] = d[c * plane + (size_t)j * n + j];
    }
    divk<K>(xj, ujj, q);
    for (int c = 0; c < K; ++c) x[c * n + j] = q[c];
    if (j == 0) break;
    double negq[K];
    for (int c = 0; c < K; ++c) negq[c] = -q[c];
    for (int i = 0; i < j; ++i) {
      double u[K], t[K], xi[K], o[K];
      for (int c = 0; c < K; ++c) {
        u[c] = d[c * plane + (size_t)i * n + j];
        xi[c] = x[c * n + i];
      }
      mul<K>(u, negq, t);
      add<K>(xi, t, o);
      for (int c = 0; c < K; ++c) x[c * n + i] = o[c];
    }
  }
}

// mat_vec lane path (linalg.py:562-574): y_i = fold_j add(y_i, mul(A_ij, x_j))
template <int K>
static void matvec(int rows, int cols, const double *a, const double *x,
                   double *y) {
  const size_t plane = (size_t)rows * cols;
#pragma omp parallel for schedule(static) if (rows > 256)
  for (int i = 0; i < rows; ++i) {
    double acc[K] = {0.0};
    for (int j = 0; j < cols; ++j) {
      double aij[K], xj[K], t[K], o[K];
      for (int c = 0; c < K; ++c) {
        aij[c] = a[c * plane + (size_t)i * cols + j];
        xj[c] = x[c * cols + j];
      }
      mul<K>(aij, xj, t);
      add<K>(acc, t, o);
      for (int c = 0; c < K; ++c) acc[c] = o[c];
    }
    for (int c = 0; c < K; ++c) y[c * rows + i] = acc[c];
  }
}

// mat_mul_blocked lane path (linalg.py:589-600):
//   C_ij = fold over p ascending of add(C_ij, mul(A_ip, B_pj)), C = 0.
template <int K>
static void gemm(int m, int kk, int nn, const double *A, const double *B,
                 double *C) {
  const size_t pa = (size_t)m * kk, pb = (size_t)kk * nn, pc = (size_t)m * nn;
  for (size_t t = 0; t < (size_t)K * pc; ++t) C[t] = 0.0;
#pragma omp parallel for schedule(dynamic, 4) if ((size_t)m * nn > 4096)
  for (int i = 0; i < m; ++i) {
    double *RESTRICT ci[K];
    for (int c = 0; c < K; ++c) ci[c] = C + c * pc + (size_t)i * nn;
    for (int p = 0; p < kk; ++p) {
      double aip[K];
      for (int c = 0; c < K; ++c) aip[c] = A[c * pa + (size_t)i * kk + p];
      const double *RESTRICT bp[K];
      for (int c = 0; c < K; ++c) bp[c] = B + c * pb + (size_t)p * nn;
#pragma GCC ivdep
      for (int q = 0; q < nn; ++q) {
        double b[K], t[K], x[K], o[K];
        for (int c = 0; c < K; ++c) { b[c] = bp[c][q]; x[c] = ci[c][q]; }
        mul<K>(aip, b, t);
        add<K>(x, t, o);
        for (int c = 0; c < K; ++c) ci[c][q] = o[c];
      }
    }
  }
}

// Elementwise kernels over n lanes (linalg.py:624-673, mcfloat.py:304-318).
// op: 0 add(x, y), 1 mul(x, y), 2 div(x, y), 4 sqrt(x) (y unused)
template <int K>
static void elementwise(int op, int64_t n, const double *x, const double *y,
                        double *out) {
#pragma omp parallel for schedule(static) if (n > 4096)
  for (int64_t i = 0; i < n; ++i) {
    double a[K], b[K], o[K];
    for (int c = 0; c < K; ++c) { a[c] = x[c * n + i]; b[c] = y[c * n + i]; }
    if (op == 0) add<K>(a, b, o);
    else if (op == 1) mul<K>(a, b, o);
    else if (op == 2) divk<K>(a, b, o);
    else sqrtk<K>(a, o);
    for (int c = 0; c < K; ++c) out[c * n + i] = o[c];
  }
}

template <int K>
static void axpy(int64_t n, const double *alpha, const double *x, double *y) {
  for (int64_t i = 0; i < n; ++i) {
    double a[K], b[K], t[K], o[K];
    for (int c = 0; c < K; ++c) { a[c] = x[c * n + i]; b[c] = y[c * n + i]; }
    mul<K>(a, alpha, t);
    add<K>(b, t, o);
    for (int c = 0; c < K; ++c) y[c * n + i] = o[c];
  }
}

}  // namespace

#define DISPATCH(k, call)                         \
  switch (k) {                                    \
    case 2: { constexpr int K = 2; call; } break; \
    case 3: { constexpr int K = 3; call; } break; \
    case 4: { constexpr int K = 4; call; } break; \
    default: return 2;                            \
  }

extern "C" {

int mcref_two_sum(int64_t n, const double *a, const double *b, double *s,
                  double *e) {
  for (int64_t i = 0; i < n; ++i) two_sum(a[i], b[i], s[i], e[i]);
  return 0;
}
int mcref_two_prod(int64_t n, const double *a, const double *b, double *p,
                   double *e) {
  for (int64_t i = 0; i < n; ++i) two_prod(a[i], b[i], p[i], e[i]);
  return 0;
}
int mcref_elementwise(int k, int op, int64_t n, const double *x,
                      const double *y, double *out) {
  if (op < 0 || op > 4 || op == 3) return 2;
  DISPATCH(k, elementwise<K>(op, n, x, y, out));
  return 0;
}
int mcref_axpy(int k, int64_t n, const double *alpha, const double *x,
               double *y) {
  DISPATCH(k, axpy<K>(n, alpha, x, y));
  return 0;
}
int mcref_lu(int k, int n, double *a, int32_t *swaps, int32_t *sing_step) {
  int st = 0;
  *sing_step = -1;
  DISPATCH(k, st = lu<K>(n, a, swaps, sing_step));
  return st;
}
int mcref_solve(int k, int n, const double *lu, const int32_t *swaps,
                double *x) {
  DISPATCH(k, solve<K>(n, lu, swaps, x));
  return 0;
}
int mcref_matvec(int k, int rows, int cols, const double *a, const double *x,
                 double *y) {
  DISPATCH(k, matvec<K>(rows, cols, a, x, y));
  return 0;
}
int mcref_gemm(int k, int m, int kk, int nn, const double *a, const double *b,
               double *c) {
  DISPATCH(k, gemm<K>(m, kk, nn, a, b, c));
  return 0;
}
int mcref_lu_block(int k, int m, int w, double *a, int64_t ld, int64_t pl,
                   int32_t *swaps, int32_t *sing_step) {
  int st = 0;
  *sing_step = -1;
  DISPATCH(k, st = lu_block<K>(m, w, a, ld, pl, swaps, sing_step));
  return st;
}
int mcref_trsm(int k, int w, int ncols, const double *l, int64_t ldl,
               int64_t pl, double *u, int64_t ldu, int64_t pu) {
  DISPATCH(k, trsm<K>(w, ncols, l, ldl, pl, u, ldu, pu));
  return 0;
}
int mcref_gemm_update(int k, int M, int N, int KK, const double *a,
                      int64_t lda, int64_t pa, const double *b, int64_t ldb,
                      int64_t pb, double *c, int64_t ldc, int64_t pc) {
  DISPATCH(k, gemm_update<K>(M, N, KK, a, lda, pa, b, ldb, pb, c, ldc, pc));
  return 0;
}
int mcref_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
void mcref_set_threads(int t) {
#ifdef _OPENMP
  if (t > 0) omp_set_num_threads(t);
#else
  (void)t;
#endif
}

}  // extern "C"
