// BASELINE config 3 test system (SURVEY §7 "config 3 generation"; the
// reference's own generator, testgen.py:229-274, builds R·D·R⁻¹ instead):
//
//   A = U · diag(σ) · W,   σ_k = r^k,  r = (1e-30)^(1/(n-1))  (κ = 1e30),
//   b = A · ones  at the long precision (mat_vec order, linalg.py:566-574).
//
// U and W are random orthogonal matrices.  The config asks for QR of a
// Gaussian at 512 bits; SURVEY notes that any deterministic 512-bit
// orthogonalisation is acceptable (only reproducibility of A matters) and
// that two mpmath QRs take hours at n = 1024.  Here each is a product of
// ceil(log2 n) butterfly layers of plane rotations (layer l rotates rows
// (i, i + 2^l)): dense after all layers, exactly orthogonal up to the
// working precision, and O(n^2 log n) to apply.  The rotation angles come
// from the seeded splitmix64 stream of SURVEY §8(d) (slots 5 and 6):
// t = w(i) in [-1, 1), c = (1 - t^2)/(1 + t^2), s = 2t/(1 + t^2).
//
// Working precision: 576-bit two's-complement fixed point (scale 2^576) for
// the O(n^2 log n) rotation sweeps, column-parallel on host threads; σ and
// the rotation coefficients come from correctly rounded 640-bit big floats.
// Entries of A are then rounded once (RNE) to the long precision.
#include "testsys.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <thread>

#include "refine_host.h"

namespace mpr {

using bn::BF;
using bn::UBig;

namespace {

constexpr int L = 10;          // limbs; value = (signed int) / 2^(64*(L-1))
constexpr int FRAC = 64 * (L - 1);
constexpr int64_t PW = 640;    // precision of σ and rotation coefficients

struct Fx {
  uint64_t w[L];  // little-endian two's complement
};

inline void fx_zero(Fx &a) { std::memset(a.w, 0, sizeof a.w); }
inline bool fx_neg_p(const Fx &a) { return (int64_t)a.w[L - 1] < 0; }
inline void fx_negate(Fx &a) {
  unsigned __int128 c = 1;
  for (int i = 0; i < L; ++i) {
    c += (uint64_t)~a.w[i];
    a.w[i] = (uint64_t)c;
    c >>= 64;
  }
}
inline void fx_add(const Fx &a, const Fx &b, Fx &o) {
  unsigned __int128 c = 0;
  for (int i = 0; i < L; ++i) {
    c += (unsigned __int128)a.w[i] + b.w[i];
    o.w[i] = (uint64_t)c;
    c >>= 64;
  }
}
inline void fx_sub(const Fx &a, const Fx &b, Fx &o) {
  Fx nb = b;
  fx_negate(nb);
  fx_add(a, nb, o);
}
// a*b / 2^FRAC, truncated toward zero in magnitude (|a|, |b| < 2^63)
inline void fx_mul(const Fx &a, const Fx &b, Fx &o) {
  Fx x = a, y = b;
  const bool neg = fx_neg_p(x) != fx_neg_p(y);
  if (fx_neg_p(x)) fx_negate(x);
  if (fx_neg_p(y)) fx_negate(y);
  uint64_t p[2 * L] = {0};
  for (int i = 0; i < L; ++i) {
    if (!x.w[i]) continue;
    unsigned __int128 c = 0;
    for (int j = 0; j < L; ++j) {
      c += (unsigned __int128)x.w[i] * y.w[j] + p[i + j];
      p[i + j] = (uint64_t)c;
      c >>= 64;
    }
    p[i + L] = (uint64_t)c;
  }
  for (int i = 0; i < L; ++i) o.w[i] = p[i + L - 1];
  if (neg) fx_negate(o);
}

Fx fx_from_bf(const BF &v) {
  Fx r;
  fx_zero(r);
  if (v.sign == 0) return r;
  // |v| * 2^FRAC = man * 2^(exp + FRAC), truncated
  const int64_t sh = v.exp + FRAC;
  UBig m = sh >= 0 ? v.man.shl(sh) : v.man.shr(-sh);
  for (int i = 0; i < L && 2 * i < (int)m.w.size(); ++i) {
    uint64_t lo = m.w[2 * i];
    uint64_t hi = 2 * i + 1 < (int)m.w.size() ? m.w[2 * i + 1] : 0;
    r.w[i] = lo | (hi << 32);
  }
  if (v.sign < 0) fx_negate(r);
  return r;
}

BF fx_to_bf(const Fx &a, int64_t p) {
  Fx x = a;
  BF r;
  const bool neg = fx_neg_p(x);
  if (neg) fx_negate(x);
  UBig m;
  for (int i = 0; i < L; ++i) {
    m.w.push_back((uint32_t)x.w[i]);
    m.w.push_back((uint32_t)(x.w[i] >> 32));
  }
  m.trim();
  if (m.zero()) return r;
  return bn::mk(neg ? -1 : 1, m, -FRAC, p);
}

BF bf_from_double(double d, int64_t p) { return lf_round(bn::from_binary64(d), p); }

// x^e (e >= 0) by squaring, every product rounded to p
BF bf_pow(const BF &x, int64_t e, int64_t p) {
  BF r = bf_from_double(1.0, p), b = x;
  while (e > 0) {
    if (e & 1) r = lf_mul(r, b, p);
    e >>= 1;
    if (e) b = lf_mul(b, b, p);
  }
  return r;
}

// the seeded recipe of SURVEY §8(d): w(i) = RN(mix(S + G(i+1))) 2^-63 - 1
uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
double w_of(uint64_t seed, uint64_t i) {
  const uint64_t u = mix64(seed + 0x9E3779B97F4A7C15ull * (i + 1));
  return std::ldexp((double)u, -63) - 1.0;
}

struct Rot {
  Fx c, s;
};

// rotation coefficients of every layer of one butterfly (slot picks the
// stream segment), layer-major, pair index = position of i among the rows
// with bit l clear
std::vector<Rot> make_rotations(int n, int layers, uint64_t seed, int slot) {
  std::vector<Rot> rot((size_t)layers * n);
  const BF one = bf_from_double(1.0, PW), two = bf_from_double(2.0, PW);
  for (int l = 0; l < layers; ++l)
    for (int i = 0; i < n; ++i) {
      const uint64_t idx = ((uint64_t)slot * n * n + (uint64_t)l * n + i) * 4;
      const BF t = bf_from_double(w_of(seed, idx), PW);
      const BF t2 = lf_mul(t, t, PW);
      const BF den = lf_add(one, t2, PW);
      rot[(size_t)l * n + i].c = fx_from_bf(lf_div(lf_sub(one, t2, PW), den, PW));
      rot[(size_t)l * n + i].s = fx_from_bf(lf_div(lf_mul(two, t, PW), den, PW));
    }
  return rot;
}

// M <- B_{L-1} ... B_0 M for the butterfly of `rot`, columns [c0, c1)
void apply_butterfly(std::vector<Fx> &M, int n, int layers,
                     const std::vector<Rot> &rot, int c0, int c1) {
  Fx t0, t1, u0, u1;
  for (int l = 0; l < layers; ++l) {
    const int h = 1 << l;
    for (int i = 0; i < n; ++i) {
      if ((i & h) || i + h >= n) continue;
      const Rot &R = rot[(size_t)l * n + i];
      Fx *ri = &M[(size_t)i * n], *rj = &M[(size_t)(i + h) * n];
      for (int c = c0; c < c1; ++c) {
        // (x, y) -> (c x - s y, s x + c y)
        fx_mul(R.c, ri[c], t0);
        fx_mul(R.s, rj[c], t1);
        fx_mul(R.s, ri[c], u0);
        fx_mul(R.c, rj[c], u1);
        fx_sub(t0, t1, ri[c]);
        fx_add(u0, u1, rj[c]);
      }
    }
  }
}

template <class F>
void parallel_for(int n, int threads, F f) {
  threads = std::max(1, std::min(threads, n));
  if (threads == 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> ts;
  for (int t = 0; t < threads; ++t) {
    const int a = (int)((int64_t)n * t / threads), b = (int)((int64_t)n * (t + 1) / threads);
    ts.emplace_back([=] { f(a, b); });
  }
  for (auto &t : ts) t.join();
}

}  // namespace

int config3_system(int n, uint64_t seed, int64_t long_bits, double kappa_exp10,
                   int threads, std::vector<BF> &A, std::vector<BF> &b,
                   std::string &err) {
  if (n < 1) {
    err = "n must be positive";
    return 2;
  }
  if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
  int layers = 0;
  while ((1 << layers) < n) ++layers;
  // σ_k = r^k, r^(n-1) = 10^-kappa (Newton on x^(n-1) = y at PW bits)
  std::vector<Fx> sigma(n);
  {
    BF y;
    char buf[64];
    std::snprintf(buf, sizeof buf, "1e-%d", (int)kappa_exp10);
    bn::parse_decimal(buf, PW, y);
    const int64_t m = n - 1;
    BF r = bf_from_double(1.0, PW);
    if (m > 0) {
      r = bf_from_double(std::pow(10.0, -kappa_exp10 / (double)m), PW);
      const BF mm = bf_from_double((double)m, PW);
      for (int it = 0; it < 6; ++it) {
        const BF pm1 = bf_pow(r, m - 1, PW);
        const BF pm = lf_mul(pm1, r, PW);
        r = lf_sub(r, lf_div(lf_sub(pm, y, PW), lf_mul(mm, pm1, PW), PW), PW);
      }
    }
    BF s = bf_from_double(1.0, PW);
    for (int k = 0; k < n; ++k) {
      sigma[k] = fx_from_bf(s);
      s = lf_mul(s, r, PW);
    }
  }
  const std::vector<Rot> ru = make_rotations(n, layers, seed, 5);
  const std::vector<Rot> rw = make_rotations(n, layers, seed, 6);
  // M = W (butterfly applied to the identity), rows scaled by σ, then U M
  std::vector<Fx> M((size_t)n * n);
  for (auto &v : M) fx_zero(v);
  const Fx one = fx_from_bf(bf_from_double(1.0, PW));
  for (int i = 0; i < n; ++i) M[(size_t)i * n + i] = one;
  parallel_for(n, threads, [&](int c0, int c1) {
    apply_butterfly(M, n, layers, rw, c0, c1);
  });
  parallel_for(n, threads, [&](int r0, int r1) {
    for (int i = r0; i < r1; ++i)
      for (int c = 0; c < n; ++c) {
        Fx t;
        fx_mul(sigma[i], M[(size_t)i * n + c], t);
        M[(size_t)i * n + c] = t;
      }
  });
  parallel_for(n, threads, [&](int c0, int c1) {
    apply_butterfly(M, n, layers, ru, c0, c1);
  });
  // round to the long precision; b = A * ones in mat_vec order
  A.assign((size_t)n * n, BF());
  b.assign(n, BF());
  const BF bone = bf_from_double(1.0, long_bits);
  parallel_for(n, threads, [&](int r0, int r1) {
    for (int i = r0; i < r1; ++i) {
      BF acc;
      for (int c = 0; c < n; ++c) {
        BF &a = A[(size_t)i * n + c];
        a = fx_to_bf(M[(size_t)i * n + c], long_bits);
        acc = lf_add(acc, lf_mul(a, bone, long_bits), long_bits);
      }
      b[i] = acc;
    }
  });
  return 0;
}

}  // namespace mpr
