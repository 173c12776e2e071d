// The IR's long -> short conversion on the GPU (
// linalg.py:761-770 convert_matrix, bigfloat.py:419-432 bf_to_multicomp):
// every element of the long matrix, uploaded as its exact value (sign,
// exponent, up to 640 mantissa bits), is rounded once to the working
// precision p (the reference re-rounds A into the long context on entry),
// kept in that fixed-width form for the device residual, and peeled into
// its k binary64 heads -- the planes the short factorisation starts from,
// written straight into the [A | b] workspace.  Also the heads' largest
// exponent and scaled sum of squares for the rigorous ||A||_F bounds.
//
// These are device ports of the host's fastfloat.h round_to and
// to_multicomp_t, operation for operation (bitwise the same; checked by
// mpcore_debug_convert_selftest against the host on random and constructed
// values).
#include <algorithm>
#include <climits>

#include "internal.h"
#include "longfloat.cuh"

namespace mpk {

namespace {

constexpr int CL = lf::NL;  // limbs of the flat input and of lf::DF

__device__ __forceinline__ int bitlen(const uint64_t *a, int n) {
  for (int i = n - 1; i >= 0; --i)
    if (a[i]) return 64 * i + 64 - __clzll((long long)a[i]);
  return 0;
}
__device__ __forceinline__ bool getbit(const uint64_t *a, int n, int64_t i) {
  if (i < 0 || i >= 64 * (int64_t)n) return false;
  return (a[i >> 6] >> (i & 63)) & 1u;
}
__device__ __forceinline__ bool any_below(const uint64_t *a, int n,
                                          int64_t nbits) {
  if (nbits <= 0) return false;
  const int64_t full = nbits >> 6;
  for (int64_t l = 0; l < full && l < n; ++l)
    if (a[l]) return true;
  const int rem = (int)(nbits & 63);
  return rem && full < n && (a[full] & ((1ull << rem) - 1ull)) != 0;
}
__device__ __forceinline__ void shr_into(const uint64_t *a, int n, int64_t s,
                                         uint64_t *out, int nout) {
  const int64_t q = s >> 6;
  const int r = (int)(s & 63);
  for (int i = 0; i < nout; ++i) {
    const int64_t j = i + q;
    const uint64_t lo = j < n ? a[j] : 0, hi = j + 1 < n ? a[j + 1] : 0;
    out[i] = r ? (lo >> r) | (hi << (64 - r)) : lo;
  }
}
__device__ __forceinline__ void shl_into(const uint64_t *a, int n, int64_t s,
                                         uint64_t *out, int nout) {
  const int64_t q = s >> 6;
  const int r = (int)(s & 63);
  for (int i = nout - 1; i >= 0; --i) {
    const int64_t j = i - q;
    const uint64_t hi = (j >= 0 && j < n) ? a[j] : 0;
    const uint64_t lo = (j - 1 >= 0 && j - 1 < n) ? a[j - 1] : 0;
    out[i] = r ? (hi << r) | (lo >> (64 - r)) : hi;
  }
}

// fastfloat.h round_to: the exact value sign * w * 2^e rounded to p bits,
// half to even (a zero has sign 0 and zero limbs)
__device__ lf::DF round_to(int sign, const uint64_t *w, int n, int64_t e,
                           int p) {
  lf::DF r;
  for (int i = 0; i < CL; ++i) r.m[i] = 0;
  r.sign = 0;
  r.exp = 0;
  const int L = bitlen(w, n);
  if (L == 0) return r;
  r.sign = sign;
  if (L <= p) {
    if (L == p) {
      for (int i = 0; i < CL; ++i) r.m[i] = i < n ? w[i] : 0ull;
    } else {
      shl_into(w, n, p - L, r.m, CL);
    }
    r.exp = e - (p - L);
    return r;
  }
  const int64_t ex = L - p;
  const bool half = getbit(w, n, ex - 1);
  const bool below = any_below(w, n, ex - 1);
  shr_into(w, n, ex, r.m, CL);
  r.exp = e + ex;
  if (half && (below || (r.m[0] & 1u))) {
    bool carry = true;
    for (int i = 0; i < CL && carry; ++i) carry = ++r.m[i] == 0;
    if (carry || bitlen(r.m, CL) > p) {
      for (int i = 0; i < CL; ++i) r.m[i] = 0;
      r.m[(p - 1) >> 6] = 1ull << ((p - 1) & 63);
      r.exp += 1;
    }
  }
  return r;
}

// fastfloat.h to_multicomp_t: k heads of r0 (k binary64 values), false when
// a head leaves the normal binary64 range
template <int N>
__device__ bool to_multicomp(const lf::DF &r0, int k, int p, double *out) {
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
      if (up) ++h;
    }
    const int64_t E = e + sh;
    const int top = 63 - __clzll((long long)h);
    if (E + top < -1022 || E + top > 1023) return false;
    const int sh52 = 52 - top;
    const uint64_t frac =
        (sh52 >= 0 ? h << sh52 : h >> -sh52) & ((1ull << 52) - 1ull);
    const uint64_t bits = ((uint64_t)(E + top + 1023) << 52) | frac |
                          (sign < 0 ? (1ull << 63) : 0ull);
    out[c] = __longlong_as_double((long long)bits);
    if (c + 1 == k) break;
    if (len <= 53) {
      len = 0;
      continue;
    }
    const int qs = sh >> 6, rs = sh & 63;
    for (int i = 0; i < N; ++i) {
      if (i > qs || (i == qs && rs == 0)) M[i] = 0;
      else if (i == qs) M[i] &= (1ull << rs) - 1ull;
    }
    if (up) {
      uint64_t cf = 1;  // two's complement, masked to sh bits
      for (int i = 0; i < N; ++i) {
        const uint64_t v = ~M[i] + cf;
        cf = (cf && v == 0ull) ? 1ull : 0ull;
        M[i] = v;
      }
      for (int i = 0; i < N; ++i) {
        if (i > qs || (i == qs && rs == 0)) M[i] = 0;
        else if (i == qs) M[i] &= (1ull << rs) - 1ull;
      }
      sign = -sign;
    }
    len = 0;
    for (int i = N - 1; i >= 0; --i)
      if (M[i]) {
        len = 64 * i + 64 - __clzll((long long)M[i]);
        break;
      }
  }
  return true;
}

// A[e] (flat exact value) -> A[e] rounded to p; its k heads into the planes
// (element (i, j) of plane c at pl[c * plane + i * ld + j]); the largest
// head exponent into *emax; *bad when a head leaves the binary64 range
template <int N, bool COMPACT>
__global__ void __launch_bounds__(256)
convert_kernel(lf::DF *__restrict__ A, const LongFlat9 *__restrict__ in,
               int64_t e0, int64_t e1, int n, int k, int p,
               double *__restrict__ pl, int64_t ld, int64_t plane,
               int *__restrict__ bad, int *__restrict__ emax) {
  int my_emax = INT_MIN;
  for (int64_t e = e0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < e1;
       e += (int64_t)gridDim.x * blockDim.x) {
    lf::DF v;
    if constexpr (COMPACT) {
      const LongFlat9 f = in[e];
      uint64_t w[CL];
      for (int i = 0; i < CL; ++i) w[i] = i < 9 ? f.m[i] : 0ull;
      v = round_to((int)(f.es & 3) - 1, w, CL, f.es >> 2, p);
    } else {
      const lf::DF raw = A[e];
      v = round_to(raw.sign, raw.m, CL, raw.exp, p);
    }
    A[e] = v;
    double c[4] = {0.0, 0.0, 0.0, 0.0};
    if (!to_multicomp<N>(v, k, p, c)) atomicOr(bad, 1);
    const int64_t i = e / n, j = e % n;
    for (int q = 0; q < k; ++q) pl[q * plane + i * ld + j] = c[q];
    if (c[0] != 0.0) {
      const int ex =
          (int)((__double_as_longlong(c[0]) >> 52) & 0x7ff) - 1023;
      my_emax = max(my_emax, ex);
    }
  }
  my_emax = __reduce_max_sync(0xffffffffu, my_emax);
  if ((threadIdx.x & 31) == 0 && my_emax != INT_MIN) atomicMax(emax, my_emax);
}

__global__ void conv_init_kernel(int *bad, int *emax) {
  *bad = 0;
  *emax = INT_MIN;
}

// per-block sums of (head * 2^-emax)^2 over plane 0 (the ||A||_F bounds)
__global__ void __launch_bounds__(256)
headsum_kernel(const double *__restrict__ pl, int64_t ld, int n,
               const int *__restrict__ emax, double *__restrict__ partials) {
  __shared__ double red[256];
  const double scale = *emax == INT_MIN ? 1.0 : ldexp(1.0, -*emax);
  const int64_t count = (int64_t)n * n;
  double s = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double v = pl[(e / n) * ld + e % n] * scale;
    s += v * v;
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partials[blockIdx.x] = red[0];
}

// selftest: the device round + peel of flat values (in place, or from the
// compact records when in9 is set), for the host to compare
template <int N>
__global__ void convert_only_kernel(lf::DF *A, const LongFlat9 *in9,
                                    int64_t count, int k, int p,
                                    double *heads, int *ok) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x) {
    lf::DF v;
    if (in9) {
      const LongFlat9 f = in9[e];
      uint64_t w[CL];
      for (int i = 0; i < CL; ++i) w[i] = i < 9 ? f.m[i] : 0ull;
      v = round_to((int)(f.es & 3) - 1, w, CL, f.es >> 2, p);
    } else {
      const lf::DF raw = A[e];
      v = round_to(raw.sign, raw.m, CL, raw.exp, p);
    }
    A[e] = v;
    ok[e] = to_multicomp<N>(v, k, p, heads + 4 * e) ? 1 : 0;
  }
}

#define CONV_SWITCH(NN, CALL)                                   \
  switch (NN) {                                                 \
    case 1: { constexpr int N = 1; CALL; } break;               \
    case 2: { constexpr int N = 2; CALL; } break;               \
    case 3: { constexpr int N = 3; CALL; } break;               \
    case 4: { constexpr int N = 4; CALL; } break;               \
    case 5: { constexpr int N = 5; CALL; } break;               \
    case 6: { constexpr int N = 6; CALL; } break;               \
    case 7: { constexpr int N = 7; CALL; } break;               \
    case 8: { constexpr int N = 8; CALL; } break;               \
    case 9: { constexpr int N = 9; CALL; } break;               \
    default: { constexpr int N = 10; CALL; } break;             \
  }

}  // namespace

constexpr int CONV_PARTIALS = 296;  // headsum blocks (2 per SM)

cudaError_t long_to_short_init(int *d_bad, int *d_emax, cudaStream_t s) {
  conv_init_kernel<<<1, 1, 0, s>>>(d_bad, d_emax);
  return cudaGetLastError();
}

cudaError_t long_to_short_rows(int k, int n, int p, void *A, const void *in,
                               int r0, int r1, double *planes, int64_t ld,
                               int64_t plane, int *d_bad, int *d_emax,
                               cudaStream_t s) {
  const int64_t e0 = (int64_t)r0 * n, e1 = (int64_t)r1 * n;
  if (e1 <= e0) return cudaSuccess;
  const int grid = (int)std::min<int64_t>((e1 - e0 + 255) / 256, 148 * 16);
  auto *a = static_cast<lf::DF *>(A);
  auto *f = static_cast<const LongFlat9 *>(in);
  if (f) {
    CONV_SWITCH((p + 63) >> 6,
                (convert_kernel<N, true><<<grid, 256, 0, s>>>(
                    a, f, e0, e1, n, k, p, planes, ld, plane, d_bad, d_emax)))
  } else {
    CONV_SWITCH((p + 63) >> 6,
                (convert_kernel<N, false><<<grid, 256, 0, s>>>(
                    a, f, e0, e1, n, k, p, planes, ld, plane, d_bad, d_emax)))
  }
  return cudaGetLastError();
}

cudaError_t long_to_short_stats(int n, const double *planes, int64_t ld,
                                const int *d_emax, double *d_partials,
                                cudaStream_t s) {
  headsum_kernel<<<CONV_PARTIALS, 256, 0, s>>>(planes, ld, n, d_emax,
                                               d_partials);
  return cudaGetLastError();
}

int long_to_short_partials() { return CONV_PARTIALS; }

cudaError_t long_to_short_selftest(int k, int p, void *A, const void *in9,
                                   int64_t count, double *heads, int *ok,
                                   cudaStream_t s) {
  auto *a = static_cast<lf::DF *>(A);
  auto *f9 = static_cast<const LongFlat9 *>(in9);
  const int grid = (int)std::min<int64_t>((count + 255) / 256, 148 * 8);
  CONV_SWITCH((p + 63) >> 6,
              (convert_only_kernel<N><<<grid, 256, 0, s>>>(a, f9, count, k, p,
                                                           heads, ok)))
  return cudaGetLastError();
}

}  // namespace mpk
