// Native mixed-precision iterative refinement for mpcore_refine.
//
//   .mpmat loading            matfile.py:67-151
//   long arithmetic           bigfloat.py:239-326 (every op rounds once, RNE)
//   long <-> short            linalg.py:740-770, bigfloat.py:404-432
//   the refinement loop       refine.py:121-197 (operation order verbatim)
// The short factorisation and every correction solve run on the GPU through
// ShortSolver (cabi.cu).
#include "refine_host.h"
#include "internal.h"

#include "fastfloat.h"

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <climits>
#include <cstddef>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <memory>
#include <sstream>
#include <thread>

namespace mpr {

using bn::BF;
using bn::UBig;

// ------------------------------------------------------ long arithmetic ----
BF lf_round(const BF &a, int64_t p) {
  if (a.sign == 0) return BF();
  return bn::mk(a.sign, a.man, a.exp, p);
}
BF lf_add(const BF &a, const BF &b, int64_t p) {
  return lf_round(bn::add_exact(a, b), p);
}
BF lf_sub(const BF &a, const BF &b, int64_t p) {
  return lf_round(bn::add_exact(a, bn::neg(b)), p);
}
BF lf_mul(const BF &a, const BF &b, int64_t p) {
  if (a.sign == 0 || b.sign == 0) return BF();
  return bn::mk(a.sign * b.sign, UBig::mul(a.man, b.man), a.exp + b.exp, p);
}
BF lf_div(const BF &a, const BF &b, int64_t p) {
  if (a.sign == 0) return BF();
  return bn::round_ratio(a.sign * b.sign, a.man, b.man, a.exp - b.exp, p);
}
// bf_sqrt (bigfloat.py:304-326); a >= 0
BF lf_sqrt(const BF &a, int64_t p) {
  if (a.sign == 0) return BF();
  int64_t shift = 2 * (p + 2) - a.man.bits();
  if (shift < 0) shift = 0;
  if ((a.exp - shift) & 1) shift += 1;
  UBig m2 = a.man.shl(shift);
  UBig s = UBig::isqrt(m2);
  int64_t e = (a.exp - shift) >> 1;  // exact: a.exp - shift is even
  if (UBig::cmp(UBig::mul(s, s), m2) != 0) {
    s = s.shl(1);
    s.add_small(1);
    e -= 1;
  }
  return bn::mk(1, s, e, p);
}
int lf_cmp(const BF &a, const BF &b) {
  if (a.sign != b.sign) return a.sign > b.sign ? 1 : -1;
  if (a.sign == 0) return 0;
  int64_t ta = a.exp + a.man.bits(), tb = b.exp + b.man.bits();
  if (ta != tb) return (ta > tb ? 1 : -1) * a.sign;
  int c;
  if (a.exp >= b.exp)
    c = UBig::cmp(a.man.shl(a.exp - b.exp), b.man);
  else
    c = UBig::cmp(a.man, b.man.shl(b.exp - a.exp));
  return c * a.sign;
}

static BF from_int(int64_t v, int64_t p) {
  BF r;
  if (v == 0) return r;
  r.sign = v > 0 ? 1 : -1;
  r.man = UBig((uint64_t)(v > 0 ? v : -v));
  r.exp = 0;
  return lf_round(r, p);
}

// exact sum of binary64 components, rounded once to p (bf_from_multicomp)
static BF from_components(const double *c, int k, int64_t p) {
  BF acc;
  for (int i = 0; i < k; ++i)
    if (c[i] != 0.0) acc = bn::add_exact(acc, bn::from_binary64(c[i]));
  return lf_round(acc, p);
}

// ------------------------------------------------------------ formatting ----
static UBig rn_int(const UBig &num, const UBig &den) {
  UBig q, r;
  UBig::divmod(num, den, q, r);
  UBig r2 = r.shl(1);
  int c = UBig::cmp(r2, den);
  if (c > 0 || (c == 0 && q.bit(0))) q.add_small(1);
  return q;
}

std::string format_decimal(const BF &a, int digits, int64_t prec) {
  if (digits <= 0) digits = (int)std::ceil((double)prec * 0.3010299956639812) + 2;
  if (a.sign == 0) {
    std::string frac((size_t)(digits - 1), '0');
    return frac.empty() ? "0.e+0" : "0." + frac + "e+0";
  }
  const int64_t top = a.exp + a.man.bits();
  int64_t d_exp = (int64_t)std::floor((double)top * 0.30102999566398114);
  UBig scaled;
  const UBig lo = UBig::pow10(digits - 1), hi = UBig::pow10(digits);
  for (int it = 0; it < 4; ++it) {
    int64_t t = digits - 1 - d_exp;
    UBig num = a.man, den(1);
    if (t >= 0) num = UBig::mul(num, UBig::pow10(t));
    else den = UBig::pow10(-t);
    if (a.exp >= 0) num = num.shl(a.exp);
    else den = den.shl(-a.exp);
    scaled = rn_int(num, den);
    if (UBig::cmp(scaled, hi) >= 0) d_exp += 1;
    else if (UBig::cmp(scaled, lo) < 0) d_exp -= 1;
    else break;
  }
  std::string s = scaled.to_dec();
  std::string out = a.sign < 0 ? "-" : "";
  out += s[0];
  out += ".";
  out += s.substr(1);
  char eb[32];
  std::snprintf(eb, sizeof eb, "e%+lld", (long long)d_exp);
  return out + eb;
}

// --------------------------------------------------------------- .mpmat ----
struct Loaded {
  int rows = 0, cols = 0;
  bool bf = false;
  int k = 1;
  int64_t bits = 0;
  std::vector<BF> vals;   // bf entries, row-major
};

static int load_mpmat(const char *path, Loaded &L, std::string &err) {
  std::ifstream fh(path);
  if (!fh) {
    err = std::string(path) + ": cannot open";
    return 4;
  }
  std::string line;
  if (!std::getline(fh, line)) {
    err = std::string(path) + ":1: bad header";
    return 4;
  }
  std::istringstream hs(line);
  std::vector<std::string> parts;
  for (std::string t; hs >> t;) parts.push_back(t);
  if (parts.size() != 5 || parts[0] != "mpmat") {
    err = std::string(path) + ":1: bad header";
    return 4;
  }
  try {
    L.rows = std::stoi(parts[1]);
    L.cols = std::stoi(parts[2]);
    L.bits = std::stoll(parts[4]);
  } catch (...) {
    err = std::string(path) + ":1: non-integer dimensions in header";
    return 4;
  }
  const std::string &tag = parts[3];
  if (L.rows < 1 || L.cols < 1) {
    err = std::string(path) + ":1: dimensions must be positive";
    return 4;
  }
  if (tag == "bf") {
    if (L.bits < 2) {
      err = std::string(path) + ":1: bad precision";
      return 4;
    }
    L.bf = true;
    L.k = 1;
  } else if (tag == "dd" || tag == "td" || tag == "qd") {
    L.k = tag == "dd" ? 2 : tag == "td" ? 3 : 4;
    if (L.bits != 53 * L.k) {
      err = std::string(path) + ":1: tag/bits mismatch";
      return 4;
    }
  } else {
    err = std::string(path) + ":1: unknown scalar tag " + tag;
    return 4;
  }
  const size_t want = (size_t)L.cols * L.k;
  if (L.bf) L.vals.reserve((size_t)L.rows * L.cols);
  for (int i = 0; i < L.rows; ++i) {
    if (!std::getline(fh, line)) {
      err = std::string(path) + ": file ends early";
      return 4;
    }
    std::istringstream ls(line);
    std::vector<std::string> toks;
    for (std::string t; ls >> t;) toks.push_back(t);
    if (toks.size() != want) {
      err = std::string(path) + ": wrong token count";
      return 4;
    }
    for (auto &t : toks) {
      BF v;
      if (bn::parse_hex(t, v)) {
        err = std::string(path) + ": bad hex-float " + t;
        return 4;
      }
      if (L.bf) L.vals.push_back(lf_round(v, L.bits));
    }
  }
  for (std::string extra; std::getline(fh, extra);) {
    for (char ch : extra)
      if (!std::isspace((unsigned char)ch)) {
        err = std::string(path) + ": trailing content";
        return 4;
      }
  }
  return 0;
}

// bf_format_hex (bigfloat.py:524-537): (+-)0x1.<nibbles>p(+-)E, exact
std::string format_hex(const BF &a) {
  if (a.sign == 0) return "0x0.0p+0";
  const int64_t nbits = a.man.bits() - 1;
  const int64_t e = a.exp + nbits;
  std::string out = a.sign < 0 ? "-" : "";
  char eb[32];
  std::snprintf(eb, sizeof eb, "p%+lld", (long long)e);
  if (nbits == 0) return out + "0x1" + eb;
  const int64_t pad = (4 - nbits % 4) % 4;
  // frac = (man - 2^nbits) << pad, printed as (nbits + pad) / 4 nibbles
  const UBig frac = a.man.shl(pad);
  const int64_t width = (nbits + pad) / 4;
  std::string hex((size_t)width, '0');
  static const char *dig = "0123456789abcdef";
  for (int64_t i = 0; i < width; ++i) {
    int v = 0;
    for (int b = 0; b < 4; ++b) v |= (int)frac.bit(4 * i + b) << b;
    hex[(size_t)(width - 1 - i)] = dig[v];
  }
  return out + "0x1." + hex + eb;
}

int write_mpmat(const char *path, const std::vector<BF> &vals, int rows,
                int cols, int64_t bits, std::string &err) {
  std::ofstream fh(path);
  if (!fh) {
    err = std::string(path) + ": cannot open for writing";
    return 4;
  }
  fh << "mpmat " << rows << " " << cols << " bf " << bits << "\n";
  for (int i = 0; i < rows; ++i) {
    for (int j = 0; j < cols; ++j) {
      if (j) fh << " ";
      fh << format_hex(vals[(size_t)i * cols + j]);
    }
    fh << "\n";
  }
  if (!fh) {
    err = std::string(path) + ": write failed";
    return 4;
  }
  return 0;
}

// -------------------------------------------------------- the IR driver ----
// rows [0, n) split over host threads; every row keeps its own chain, so the
// result does not depend on the thread count
template <class F>
static void par_rows(size_t n, int threads, F f) {
  threads = (int)std::max<size_t>(1, std::min<size_t>((size_t)threads, n));
  if (threads == 1) {
    f((size_t)0, n);
    return;
  }
  std::vector<std::thread> ts;
  for (int t = 0; t < threads; ++t)
    ts.emplace_back(f, n * t / threads, n * (t + 1) / threads);
  for (auto &t : ts) t.join();
}

static int to_planes(const std::vector<BF> &v, int k, double *out,
                     size_t count, std::string &err, int threads = 1) {
  std::vector<char> bad(1, 0);
  par_rows(count, threads, [&](size_t a, size_t b) {
    double c[4];
    for (size_t e = a; e < b; ++e) {
      if (bn::to_multicomp(v[e], k, c)) {
        bad[0] = 1;  // any thread: the value is reported below
        return;
      }
      for (int q = 0; q < k; ++q) out[q * count + e] = c[q];
    }
  });
  if (bad[0]) {
    err = "value does not fit in binary64";
    return 5;
  }
  return 0;
}

// uninitialised heap buffer (no zero fill: first touch by the filling
// threads); alloc() -> false when out of memory
template <class T> struct RawBuf {
  T *p = nullptr;
  bool owned = false;
  bool alloc(size_t n) {
    p = static_cast<T *>(std::malloc(n * sizeof(T) + 1));
    owned = p != nullptr;
    return owned;
  }
  void adopt(T *ext) { p = ext; }   // memory owned elsewhere
  T &operator[](size_t i) { return p[i]; }
  const T &operator[](size_t i) const { return p[i]; }
  ~RawBuf() {
    if (owned) std::free(p);
  }
};
// the device residual takes the host layout unchanged (longfloat.cuh DF)
static_assert(sizeof(ff::F) == 96 && offsetof(ff::F, exp) == 8 &&
                  offsetof(ff::F, m) == 16,
              "ff::F layout must match lf::DF");

static BF norm2(const std::vector<BF> &v, int64_t p) {
  BF acc;
  for (const BF &s : v) acc = lf_add(acc, lf_mul(s, s, p), p);
  return lf_sqrt(acc, p);
}

using Clock = std::chrono::steady_clock;
static double secs(Clock::time_point a, Clock::time_point b) {
  return std::chrono::duration<double>(b - a).count();
}

// MPCORE_REFINE_TIMERS=1: per-phase host times on stderr (diagnostics)
struct PhaseLog {
  bool on = std::getenv("MPCORE_REFINE_TIMERS") != nullptr;
  Clock::time_point t = Clock::now();
  void mark(const char *what) {
    const auto u = Clock::now();
    if (on) std::fprintf(stderr, "[refine] %-22s %8.2f ms\n", what, secs(t, u) * 1e3);
    t = u;
  }
};

// exact value of v into the flat fixed-width form the device conversion
// reads (ff::F layout, limbs not normalised); false when wider than NL limbs
static bool flat_from_bf(const BF &v, ff::F &f) {
  f.sign = v.sign;
  f.exp = v.exp;
  const size_t n32 = v.man.w.size();
  if (n32 > 2 * (size_t)ff::NL) return false;
  std::memset(f.m, 0, sizeof f.m);
  if (n32) std::memcpy(f.m, v.man.w.data(), n32 * sizeof(uint32_t));
  if (v.sign == 0) f.exp = 0;
  return true;
}

// Worker threads kept for one refinement: the per-iteration loops over n
// values (tens of microseconds of work) cannot pay a thread start-up each.
// Workers spin briefly on a generation counter, then sleep on a condition
// variable; run() splits [0, n) into contiguous chunks, the caller takes
// the first.
class SpinPool {
 public:
  explicit SpinPool(int threads) : T_(std::max(1, threads)) {
    for (int t = 1; t < T_; ++t) ts_.emplace_back([this, t] { loop(t); });
  }
  ~SpinPool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_.store(true);
      gen_.fetch_add(1);
    }
    cv_.notify_all();
    for (auto &t : ts_) t.join();
  }
  template <class F> void run(size_t n, F f) {
    if (T_ == 1 || n < 64) {
      f((size_t)0, n);
      return;
    }
    job_ = [&](int t) { f(n * t / T_, n * (t + 1) / T_); };
    done_.store(0);
    {
      std::lock_guard<std::mutex> g(m_);
      gen_.fetch_add(1);
    }
    cv_.notify_all();
    job_(0);
    while (done_.load() < T_ - 1) {
    }
  }

 private:
  void loop(int t) {
    uint64_t seen = 0;
    for (;;) {
      int spins = 0;
      while (gen_.load() == seen && ++spins < 200000) {
      }
      if (gen_.load() == seen) {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return gen_.load() != seen; });
      }
      seen = gen_.load();
      if (stop_.load()) return;
      job_(t);
      done_.fetch_add(1);
    }
  }
  int T_;
  std::vector<std::thread> ts_;
  std::function<void(int)> job_;
  std::atomic<uint64_t> gen_{0};
  std::atomic<int> done_{0};
  std::atomic<bool> stop_{false};
  std::mutex m_;
  std::condition_variable cv_;
};

// the compact record (mpk::LongFlat9: exponent and sign in one word, 9
// limbs); false when the mantissa is wider than 576 bits
static bool flat9_from_bf(const BF &v, mpk::LongFlat9 &f) {
  const size_t n32 = v.man.w.size();
  if (n32 > 18) return false;
  f.es = (v.sign == 0 ? (int64_t)0 : v.exp) * 4 + (v.sign + 1);
  std::memset(f.m, 0, sizeof f.m);
  if (n32 && v.sign != 0)
    std::memcpy(f.m, v.man.w.data(), n32 * sizeof(uint32_t));
  return true;
}

// software prefetch of a value's heap-allocated mantissa limbs
constexpr size_t kPrefetch = 24;
static inline void prefetch_bf(const BF &v) {
  const uint32_t *p = v.man.w.data();
  __builtin_prefetch(p);
  __builtin_prefetch(p + 16);
}

int refine_core(std::vector<BF> &Avals, std::vector<BF> &Bvals, int n,
                int short_k, int long_bits, const char *rtol_s,
                const char *atol_s, int max_iter, int threads, ShortSolver &S,
                Report &out, std::string &err) {
  if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
  int st;
  // RefineConfig validation (refine.py:70-77): DomainError -> 6
  if (short_k < 2 || short_k > 4) { err = "short_k must be 2, 3, or 4"; return 6; }
  if (long_bits <= 53 * short_k) { err = "long_bits must exceed 53 * short_k"; return 6; }
  if (max_iter < 1) { err = "max_iter must be >= 1"; return 6; }
  const int k = short_k;
  const int64_t p = long_bits;
  BF rtol, atol;
  if (bn::parse_decimal(rtol_s, p, rtol) || bn::parse_decimal(atol_s, p, atol)) {
    err = "malformed tolerance";
    return 4;
  }
  if (rtol.sign < 0 || atol.sign < 0) { err = "tolerances must be nonnegative"; return 6; }
  if (rtol.sign == 0 && atol.sign == 0) { err = "rtol and atol cannot both be zero"; return 6; }
  const auto t0 = Clock::now();
  PhaseLog plog;
  // short copies; transfer precision max(long, 53k+64)+8 (linalg.py:743)
  const int64_t p_in = std::max<int64_t>(p, 53 * k + 64) + 8;
  const bool fast = p_in <= 64 * ff::NL;   // fixed-width path (fastfloat.h)
  // re-round into the working context (convert_* BfDomain -> BfDomain);
  // the fixed-width path rounds A once in its conversion pass (from_bf)
  if (!fast) {
    par_rows(Avals.size(), threads, [&](size_t a, size_t b) {
      for (size_t e = a; e < b; ++e) Avals[e] = lf_round(Avals[e], p);
    });
  }
  for (auto &v : Bvals) v = lf_round(v, p);
  plog.mark("round A, b");
  const int pi = (int)p;
  const size_t nn = (size_t)n * n;
  // n x n buffers are first touched by the threads that fill them (a
  // zero-filled std::vector would page them in on one thread)
  RawBuf<double> a_pl;
  RawBuf<ff::F> Af;
  // the residual on the GPU when the short side offers it (p <= 512): the
  // fixed-width A is then written straight into its page-locked staging
  const bool dev_res = fast && S.residual_supported(pi);
  if (dev_res) {
    if (void *st_buf = S.staging(0, nn * sizeof(ff::F)))
      Af.adopt(static_cast<ff::F *>(st_buf));
  }
  // the short planes too (the factorisation's upload from page-locked
  // memory runs at the link's rate)
  if (fast && S.residual_supported(pi)) {
    if (void *st_buf = S.staging(1, (size_t)k * nn * sizeof(double)))
      a_pl.adopt(static_cast<double *>(st_buf));
  }
  if ((a_pl.p == nullptr && !a_pl.alloc((size_t)k * nn)) ||
      (fast && Af.p == nullptr && !Af.alloc(nn))) {
    err = "out of host memory";
    return 6;
  }
  std::vector<double> b_pl((size_t)k * n), x_pl;
  // ||A||_F, row-major accumulation (linalg.py:692-700).  check_stop only
  // compares against a threshold monotone in ||A||_F, so rigorous bounds
  // from the binary64 heads (below) decide every comparison that does not
  // land within ~2^-40 (relative) of the threshold; the exact, sequentially
  // rounded sum is formed only for one that does (exact_fro).
  BF a_fro;
  const int T = (int)std::max<size_t>(1, std::min<size_t>((size_t)threads, nn));
  bool fro_exact = !fast;     // a_fro holds the exact ||A||_F
  bool af_on_host = true;  // Af holds the rounded A (else the flat input)
  auto exact_fro = [&]() {
    if (!af_on_host) {  // the rounded A lives on the device
      std::string e2;
      if (S.download_long_A(Af.p, e2)) return false;
      af_on_host = true;
    }
    RawBuf<ff::F> sq;  // squares on all threads, summed in order
    if (!sq.alloc(nn)) return false;
    par_rows(nn, threads, [&](size_t a, size_t b) {
      for (size_t e = a; e < b; ++e) sq[e] = ff::fmul(Af[e], Af[e], pi);
    });
    ff::F acc;
    for (size_t e = 0; e < nn; ++e) acc = ff::fadd(acc, sq[e], pi);
    a_fro = lf_sqrt(ff::to_bf(acc), p);
    fro_exact = true;
    return true;
  };
  std::vector<int> head_emax(T, INT_MIN);
  std::vector<double> head_sum(T, 0.0);
  // the factorisation can start as soon as the short planes exist: with an
  // asynchronous short side the fixed-width copy of A (for the device
  // residual) is written in a second pass while the GPU factors
  const bool split_factor = std::getenv("MPCORE_REFINE_SPLIT_FACTOR") != nullptr;
  const bool overlap = fast && dev_res && !split_factor &&
                       std::getenv("MPCORE_REFINE_NO_OVERLAP") == nullptr;
  // the conversion on the GPU: the host only lays the
  // exact values out flat in the staging buffer (one copy of each
  // mantissa), the device rounds them to p, keeps them for the residual and
  // peels the heads straight into the factorisation's workspace
  bool dev_conv = overlap && S.device_convert_supported(pi) &&
                  std::getenv("MPCORE_REFINE_HOST_CONVERT") == nullptr;
  if (dev_conv) {
    // row chunks: the host flattens chunk c + 1 while chunk c uploads and
    // converts.  First in the compact 80-byte records (every mantissa of at
    // most 576 bits, the common case); a wider value restarts the pass in
    // the full ff::F layout.
    bool ok = false;
    static const int chunk_env = [] {
      const char *e = std::getenv("MPCORE_CONVERT_CHUNKS");
      return e ? std::atoi(e) : 8;
    }();
    const int chunks = std::max(1, std::min(chunk_env, n / 64));
    auto chunk_rows = [&](int c, int &r0, int &r1) {
      r0 = (int)((int64_t)n * c / chunks);
      r1 = (int)((int64_t)n * (c + 1) / chunks);
    };
    auto *flat9 = reinterpret_cast<mpk::LongFlat9 *>(Af.p);
    for (int attempt = 0; attempt < 2 && !ok; ++attempt) {
      const bool compact = attempt == 0;
      std::atomic<bool> wide{false};
      st = S.device_convert_begin(k, n, pi, Af.p, compact, err);
      if (st) return st;
      // every thread flattens its share of each chunk in turn; thread 0
      // then waits for the chunk's other shares and hands it to the
      // device, while the others already work on the next chunk
      std::vector<std::atomic<int>> done(chunks);
      for (auto &d : done) d.store(0);
      std::atomic<int> dev_st{0};
      std::string dev_err;
      std::vector<std::thread> ws;
      for (int t = 0; t < T; ++t)
        ws.emplace_back([&, t] {
          for (int c = 0; c < chunks; ++c) {
            int r0, r1;
            chunk_rows(c, r0, r1);
            const size_t e0 = (size_t)r0 * n, m = (size_t)(r1 - r0) * n;
            const size_t a = e0 + m * t / T, b = e0 + m * (t + 1) / T;
            for (size_t e = a; e < b && !wide.load(std::memory_order_relaxed);
                 ++e) {
              if (e + kPrefetch < b) prefetch_bf(Avals[e + kPrefetch]);
              const bool fits = compact ? flat9_from_bf(Avals[e], flat9[e])
                                        : flat_from_bf(Avals[e], Af[e]);
              if (!fits) {
                wide.store(true);
                break;
              }
            }
            done[c].fetch_add(1);
            if (t == 0) {
              while (done[c].load() < T) std::this_thread::yield();
              if (!wide.load() && dev_st.load() == 0) {
                std::string e2;
                const int r = S.device_convert_rows(r0, r1, e2);
                if (r) {
                  dev_err = e2;
                  dev_st.store(r);
                }
              }
            }
          }
        });
      for (auto &w : ws) w.join();
      if (dev_st.load()) {
        err = dev_err;
        return dev_st.load();
      }
      ok = !wide.load();
    }
    plog.mark("A -> flat (host), chunked upload + convert");
    int emax = INT_MIN;
    double hs = 0.0;
    if (ok) {
      st = S.device_convert_end(&emax, &hs, err);
      if (st != 0 && st != 5) return st;
      ok = st == 0;
      plog.mark("device convert");
    }
    if (ok) {
      af_on_host = false;
      head_emax.assign(T, INT_MIN);
      head_sum.assign(T, 0.0);
      head_emax[0] = emax;
      head_sum[0] = hs;
    } else {
      dev_conv = false;  // a value wider than 640 bits or a head out of
                         // range: the host pass below (bn fallback inside)
    }
  }
  if (fast && !dev_conv) {
    // one pass: fixed-width value, its k binary64 heads (bf_to_multicomp),
    // the fixed-width copy (unless a second pass writes it) and, per
    // thread, the largest head exponent with the sum of the heads' squares
    // scaled by it (for the ||A||_F bounds below)
    std::vector<char> bad(T, 0);
    std::vector<std::thread> ws;
    for (int t = 0; t < T; ++t)
      ws.emplace_back([&, t] {
        const size_t a = nn * t / T, b = nn * (t + 1) / T;
        double c[4];
        int hmax = INT_MIN;
        double hsum = 0.0, hscale = 0.0;
        for (size_t e = a; e < b; ++e) {
          // the mantissas live on the heap, one allocation each: fetch a
          // few elements ahead (the pass is bound by those misses)
          if (e + kPrefetch < b) prefetch_bf(Avals[e + kPrefetch]);
          const ff::F v = ff::from_bf(Avals[e], pi);
          if (!overlap) Af[e] = v;
          if (!ff::to_multicomp(v, k, pi, c) &&
              bn::to_multicomp(ff::to_bf(v), k, c)) {
            bad[t] = 1;
            break;
          }
          for (int q = 0; q < k; ++q) a_pl[(size_t)q * nn + e] = c[q];
          if (c[0] != 0.0) {
            const int eh = std::ilogb(c[0]);
            if (eh > hmax) {  // rescale (powers of two)
              if (hmax != INT_MIN) hsum = std::ldexp(hsum, 2 * (hmax - eh));
              hmax = eh;
              hscale = std::ldexp(1.0, -eh);
            }
            const double v = c[0] * hscale;
            hsum += v * v;
          }
        }
        head_emax[t] = hmax;
        head_sum[t] = hsum;
      });
    for (auto &w : ws) w.join();
    for (int t = 0; t < T; ++t)
      if (bad[t]) {
        err = "value does not fit in binary64";
        return 5;
      }
  } else if (!fast) {
    if ((st = to_planes(Avals, k, a_pl.p, nn, err, threads))) return st;
    std::vector<BF> sq(Avals.size());
    par_rows(Avals.size(), threads, [&](size_t a, size_t b) {
      for (size_t e = a; e < b; ++e) sq[e] = lf_mul(Avals[e], Avals[e], p);
    });
    BF acc;
    for (const BF &s : sq) acc = lf_add(acc, s, p);
    a_fro = lf_sqrt(acc, p);
  }
  // Rigorous bounds on ||A||_F from the binary64 heads (a_pl plane 0):
  // check_stop's threshold is monotone in ||A||_F, so a comparison that
  // falls outside [threshold(a_lo), threshold(a_hi)) is decided without the
  // exact (sequentially rounded) sum, which is formed only when a
  // comparison lands inside the bracket (exact_fro).
  BF a_lo, a_hi;
  bool have_bounds = false;
  // MPCORE_REFINE_EXACT_FRO=1: always form the exact ||A||_F (tests)
  const bool force_exact = std::getenv("MPCORE_REFINE_EXACT_FRO") != nullptr;
  if (fast && !force_exact) {
    int emax = INT_MIN;
    for (int e : head_emax) emax = std::max(emax, e);
    const double eps = (double)(nn + 64) * 0x1p-52 + 0x1p-50;
    // (heads far from the subnormal range: each within 2^-53 of its value,
    // and subnormal heads of tiny elements negligible against the slack)
    if (emax != INT_MIN && emax > -900 && eps < 0x1p-12) {
      double S = 0.0;
      for (int t = 0; t < T; ++t)
        if (head_emax[t] != INT_MIN)
          S += std::ldexp(head_sum[t], 2 * (head_emax[t] - emax));
      // heads: relative error 2^-53 each (squares 2^-52); sums of nn terms
      // (nn + T) u; underflowed squares at most nn 2^-1022 in total
      const double lo2 = S * (1.0 - eps) - (double)nn * 0x1p-1000;
      const double hi2 = S * (1.0 + eps) + (double)nn * 0x1p-1000;
      const double lo = lo2 > 0.0 ? std::sqrt(lo2) * (1.0 - 0x1p-40) : 0.0;
      const double hi = std::sqrt(hi2) * (1.0 + 0x1p-40);
      if (std::isfinite(hi)) {
        a_lo = bn::from_binary64(lo);
        a_hi = bn::from_binary64(hi);
        if (a_lo.sign) a_lo.exp += emax;
        a_hi.exp += emax;
        have_bounds = true;
      }
    }
  }
  plog.mark(dev_conv ? "A -> flat, GPU convert" :
            overlap ? "A -> planes" : "A -> fixed, planes");
  if ((st = to_planes(Bvals, k, b_pl.data(), (size_t)n, err))) return st;
  std::vector<ff::F> Bf;
  bool use_dev = false;
  bool begun = false;
  if (overlap) {
    st = S.factor_solve_begin(k, n, a_pl.p, b_pl, err);
    if (st > 0) return st;
    begun = st == 0;
  }
  auto t1 = Clock::now();
  if (overlap && !dev_conv) {
    // the fixed-width A, while the GPU factors (or before the synchronous
    // factorisation when the short side cannot overlap)
    par_rows(nn, threads, [&](size_t a, size_t b) {
      for (size_t e = a; e < b; ++e) {
        if (e + kPrefetch < b) prefetch_bf(Avals[e + kPrefetch]);
        Af[e] = ff::from_bf(Avals[e], pi);
      }
    });
    plog.mark("A -> fixed (overlapping the factorisation)");
    if (!begun) t1 = Clock::now();
  }
  if (fast) {
    Bf.resize(n);
    for (int i = 0; i < n; ++i) Bf[i] = ff::from_bf(Bvals[i], pi);
    if (dev_res) {  // upload (asynchronous) overlaps the factorisation
      if ((st = S.residual_setup(n, pi, Af.p, Bf.data(), err))) return st;
      use_dev = true;
    }
  }
  // the factorisation and the first solve (b along the LU on the GPU);
  // MPCORE_REFINE_SPLIT_FACTOR=1 takes factor() + solve() instead (tests:
  // both give the same bits)
  if (begun) {
    if ((st = S.factor_solve_end(x_pl, err))) return st;
  } else if (split_factor) {
    if ((st = S.factor(k, n, a_pl.p, err))) return st;
    if ((st = S.solve(b_pl, x_pl, err))) return st;
  } else if ((st = S.factor_solve(k, n, a_pl.p, b_pl, x_pl, err))) {
    return st;
  }
  const auto t2 = Clock::now();
  plog.mark("factor + first solve");
  double t_solve = 0, t_res = 0;
  auto timed_solve = [&](const std::vector<double> &rhs) {
    const auto a = Clock::now();
    const int r = S.solve(rhs, x_pl, err);
    t_solve += secs(a, Clock::now());
    return r;
  };
  // bf_from_multicomp at p_in, then into the working precision
  auto lift = [&](const std::vector<double> &pl, std::vector<BF> &x) {
    x.resize(n);
    double c[4];
    for (int i = 0; i < n; ++i) {
      for (int q = 0; q < k; ++q) c[q] = pl[(size_t)q * n + i];
      x[i] = lf_round(from_components(c, k, p_in), p);
    }
  };
  // the same on fixed-width values: the components are summed at p_in,
  // exactly whenever they span fewer than p_in - 56 bits (always, for the
  // renormalised values the GPU returns); otherwise the generic path
  const int pin = (int)p_in;
  SpinPool pool(std::min(T, std::max(1, n / 64)));
  auto lift_f = [&](const std::vector<double> &pl, std::vector<ff::F> &x) {
    x.resize(n);
    pool.run((size_t)n, [&](size_t i0, size_t i1) {
      for (size_t i = i0; i < i1; ++i) {
        double c[4];
        int emax = INT_MIN, emin = INT_MAX;
        for (int q = 0; q < k; ++q) {
          c[q] = pl[(size_t)q * n + i];
          if (c[q] != 0.0) {
            const int e = std::ilogb(c[q]);
            emax = std::max(emax, e);
            emin = std::min(emin, e);
          }
        }
        if (emax != INT_MIN && emax - emin > pin - 56) {
          x[i] = ff::from_bf(lf_round(from_components(c, k, p_in), p), pi);
          continue;
        }
        ff::F acc;
        for (int q = 0; q < k; ++q)
          if (c[q] != 0.0)
            acc = ff::fadd(acc, ff::from_double(c[q], pin), pin);
        x[i] = ff::round(acc, pin, pi);
      }
    });
  };
  std::vector<BF> x;
  std::vector<ff::F> xf, resf, zf;
  if (fast) {
    lift_f(x_pl, xf);
  } else {
    lift(x_pl, x);
  }
  plog.mark("lift x");
  const BF one = from_int(1, p);
  const BF sqrt_n = lf_sqrt(from_int(n, p), p);
  std::vector<BF> res(n), work(n), z;
  // (the squares in parallel, their sum in the reference's order)
  std::vector<ff::F> sqv;
  auto norm2_f = [&](const std::vector<ff::F> &v) {
    sqv.resize(v.size());
    pool.run(v.size(), [&](size_t i0, size_t i1) {
      for (size_t i = i0; i < i1; ++i) sqv[i] = ff::fmul(v[i], v[i], pi);
    });
    ff::F acc;
    for (const ff::F &q : sqv) acc = ff::fadd(acc, q, pi);
    return lf_sqrt(ff::to_bf(acc), p);
  };
  std::string reason = "max_iter";
  int corrections = 0;
  out.residuals.clear();
  for (int it = 0; it < max_iter; ++it) {
    // res = b - A x  (scalar mat_vec order per row, linalg.py:566-574)
    const auto ta = Clock::now();
    BF res_norm, x_norm;
    if (use_dev) {
      resf.resize(n);
      if ((st = S.residual(xf.data(), resf.data(), err))) return st;
      t_res += secs(ta, Clock::now());
      res_norm = norm2_f(resf);
      x_norm = norm2_f(xf);
    } else if (fast) {
      resf.resize(n);
      par_rows((size_t)n, threads, [&](size_t r0, size_t r1) {
        for (size_t i = r0; i < r1; ++i) {
          ff::F acc;
          const ff::F *row = &Af[i * n];
          for (int j = 0; j < n; ++j)
            acc = ff::fadd(acc, ff::fmul(row[j], xf[j], pi), pi);
          resf[i] = ff::fadd(Bf[i], ff::neg(acc), pi);
        }
      });
      t_res += secs(ta, Clock::now());
      res_norm = norm2_f(resf);
      x_norm = norm2_f(xf);
    } else {
      par_rows((size_t)n, threads, [&](size_t r0, size_t r1) {
        for (size_t i = r0; i < r1; ++i) {
          BF acc;
          const BF *row = &Avals[i * n];
          for (int j = 0; j < n; ++j)
            acc = lf_add(acc, lf_mul(row[j], x[j], p), p);
          res[i] = lf_sub(Bvals[i], acc, p);
        }
      });
      t_res += secs(ta, Clock::now());
      res_norm = norm2(res, p);
      x_norm = norm2(x, p);
    }
    plog.mark("residual + norms");
    out.residuals.push_back(res_norm);
    if (res_norm.sign == 0) { reason = "converged"; break; }
    // check_stop (refine.py:104-118): res < sqrt(n) rtol ||A||_F ||x|| + atol
    auto threshold = [&](const BF &af) {
      BF t = sqrt_n;
      t = lf_mul(t, rtol, p);
      t = lf_mul(t, af, p);
      t = lf_mul(t, x_norm, p);
      return lf_add(t, atol, p);
    };
    bool conv;
    if (!fro_exact && have_bounds && lf_cmp(res_norm, threshold(a_lo)) < 0) {
      conv = true;
    } else if (!fro_exact && have_bounds &&
               lf_cmp(res_norm, threshold(a_hi)) >= 0) {
      conv = false;
    } else {
      if (!fro_exact) {
        if (!exact_fro()) {
          err = "out of host memory";
          return 6;
        }
        plog.mark("||A||_F (exact)");
      }
      conv = lf_cmp(res_norm, threshold(a_fro)) < 0;
    }
    if (conv) { reason = "converged"; break; }
    const size_t h = out.residuals.size();
    if (h >= 4 && lf_cmp(out.residuals[h - 1], out.residuals[h - 2]) >= 0 &&
        lf_cmp(out.residuals[h - 2], out.residuals[h - 3]) >= 0 &&
        lf_cmp(out.residuals[h - 3], out.residuals[h - 4]) >= 0) {
      reason = "stagnated";
      break;
    }
    // z = solve(r / ||r||), x += z * ||r||  (refine.py:184-190)
    BF coef = lf_div(one, res_norm, p);
    std::vector<double> w_pl((size_t)k * n);
    if (fast) {
      const ff::F cf = ff::from_bf(coef, pi);
      std::atomic<bool> overflow{false};
      pool.run((size_t)n, [&](size_t i0, size_t i1) {
        for (size_t i = i0; i < i1; ++i) {
          const ff::F w = ff::fmul(resf[i], cf, pi);
          double c[4];
          if (!ff::to_multicomp(w, k, pi, c) &&
              bn::to_multicomp(ff::to_bf(w), k, c)) {
            overflow.store(true);
            return;
          }
          for (int q = 0; q < k; ++q) w_pl[(size_t)q * n + i] = c[q];
        }
      });
      if (overflow.load()) {
        err = "value does not fit in binary64";
        return 5;
      }
    } else {
      for (int i = 0; i < n; ++i) work[i] = lf_mul(res[i], coef, p);
      if ((st = to_planes(work, k, w_pl.data(), (size_t)n, err))) return st;
    }
    if ((st = timed_solve(w_pl))) return st;
    if (fast) {
      lift_f(x_pl, zf);
      const ff::F rn = ff::from_bf(res_norm, pi);
      pool.run((size_t)n, [&](size_t i0, size_t i1) {
        for (size_t i = i0; i < i1; ++i)
          xf[i] = ff::fadd(xf[i], ff::fmul(zf[i], rn, pi), pi);
      });
    } else {
      lift(x_pl, z);
      for (int i = 0; i < n; ++i) x[i] = lf_add(x[i], lf_mul(z[i], res_norm, p), p);
    }
    ++corrections;
    plog.mark("correction");
  }
  if (fast) {
    x.resize(n);
    for (int i = 0; i < n; ++i) x[i] = ff::to_bf(xf[i]);
  }
  const auto t3 = Clock::now();
  out.iterations = corrections;
  out.stop_reason = reason;
  out.solution = x;
  out.prec = p;
  // convert, factor (+ the first solve), refinement loop, residuals, solves
  out.timings = {secs(t0, t1), secs(t1, t2), secs(t2, t3), t_res, t_solve};
  return 0;
}

// fastfloat.h vs the generic path on random operands (diagnostics / tests)
int64_t longfloat_selftest(int64_t iters, uint64_t seed, int p) {
  if (p < 2 || p > 64 * ff::NL) return -1;
  uint64_t z = seed;
  auto rnd = [&]() {
    z += 0x9E3779B97F4A7C15ull;
    uint64_t x = z;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
  };
  auto rand_bf = [&](int64_t e_center) {
    // random p-bit (or shorter) mantissa, exponent near e_center
    bn::BF v;
    const int bits = 1 + (int)(rnd() % (uint64_t)p);
    bn::UBig m;
    for (int b = 0; b < bits; b += 32) m.w.push_back((uint32_t)rnd());
    m = m.shr((int64_t)m.w.size() * 32 - bits);
    if (m.w.empty()) m = bn::UBig(1);
    if (!m.bit(bits - 1)) m = bn::UBig::add(m.shl(0), bn::UBig(1).shl(bits - 1));
    if (rnd() % 8 == 0) {  // runs of ones: carries through every limb
      m = bn::UBig(1).shl(bits);
      m = bn::UBig::sub(m, bn::UBig(1 + rnd() % 3));
    }
    v.sign = (rnd() & 1) ? 1 : -1;
    v.man = m;
    v.exp = e_center - bits + (int64_t)(rnd() % 7) - 3;
    v.man.trim();
    return v;
  };
  int64_t bad = 0;
  for (int64_t it = 0; it < iters; ++it) {
    const int64_t gap_kind = rnd() % 6;
    int64_t gap = gap_kind == 0 ? 0
                  : gap_kind == 1 ? (int64_t)(rnd() % 4)
                  : gap_kind == 2 ? (int64_t)(rnd() % (uint64_t)(p + 8))
                  : gap_kind == 3 ? p + (int64_t)(rnd() % 6) - 3
                  : (int64_t)(rnd() % 3000);
    BF a = lf_round(rand_bf(0), p), b = lf_round(rand_bf(-gap), p);
    if (rnd() % 16 == 0) b = bn::neg(a);          // exact cancellation
    if (rnd() % 16 == 1) b = lf_round(bn::neg(a), p - 1 > 1 ? p - 1 : p);
    const ff::F fa = ff::from_bf(a, p), fb = ff::from_bf(b, p);
    const BF s_ref = lf_add(a, b, p), s = ff::to_bf(ff::add(fa, fb, p));
    const BF d_ref = lf_sub(a, b, p), d = ff::to_bf(ff::add(fa, ff::neg(fb), p));
    const BF m_ref = lf_mul(a, b, p), mm = ff::to_bf(ff::mul(fa, fb, p));
    if (lf_cmp(s, s_ref) != 0 || s.sign != s_ref.sign) ++bad;
    if (lf_cmp(d, d_ref) != 0 || d.sign != d_ref.sign) ++bad;
    if (lf_cmp(mm, m_ref) != 0 || mm.sign != m_ref.sign) ++bad;
    // big-integer division (Knuth D): q b + r == a, r < b
    if (!b.man.zero()) {
      bn::UBig q, r;
      const bn::UBig num = bn::UBig::mul(a.man, a.man.shl(rnd() % 70));
      bn::UBig::divmod(num, b.man, q, r);
      if (bn::UBig::cmp(bn::UBig::add(bn::UBig::mul(q, b.man), r), num) != 0 ||
          bn::UBig::cmp(r, b.man) >= 0)
        ++bad;
    }
    // the compile-time-width kernels (fadd / fmul) on the same operands
    const BF s2 = ff::to_bf(ff::fadd(fa, fb, p));
    const BF d2 = ff::to_bf(ff::fadd(fa, ff::neg(fb), p));
    const BF m2 = ff::to_bf(ff::fmul(fa, fb, p));
    if (lf_cmp(s2, s_ref) != 0 || s2.sign != s_ref.sign) ++bad;
    if (lf_cmp(d2, d_ref) != 0 || d2.sign != d_ref.sign) ++bad;
    if (lf_cmp(m2, m_ref) != 0 || m2.sign != m_ref.sign) ++bad;
    // bf_to_multicomp on the fixed-width value (when it takes the fast path)
    for (int k = 2; k <= 4; ++k) {
      double c1[4], c2[4];
      if (ff::to_multicomp(fa, k, p, c1)) {
        if (bn::to_multicomp(a, k, c2) != 0 ||
            std::memcmp(c1, c2, sizeof(double) * k) != 0)
          ++bad;
      }
    }
    // the lift of k binary64 components: exact sum at p + 64, then p
    if (p + 64 <= 64 * ff::NL) {
      double c[4];
      if (bn::to_multicomp(a, 4, c) == 0) {
        const int pin = p + 64;
        ff::F acc;
        BF ex;
        for (int q = 0; q < 4; ++q) {
          if (c[q] == 0.0) continue;
          acc = ff::fadd(acc, ff::from_double(c[q], pin), pin);
          ex = bn::add_exact(ex, bn::from_binary64(c[q]));
        }
        const BF l1 = ff::to_bf(ff::round(acc, pin, p));
        const BF l2 = lf_round(lf_round(ex, pin), p);
        if (lf_cmp(l1, l2) != 0 || l1.sign != l2.sign) ++bad;
      }
    }
  }
  return bad;
}

// The device long residual (residual.cu) against the host's fixed-width
// one on a random n x n system at precision p: rows whose residual differs
// in any bit (sign, exponent or mantissa limb).  -1: bad arguments / CUDA.
int64_t long_residual_selftest(int n, int p, uint64_t seed, cudaStream_t s,
                               int variant) {
  if (n <= 0 || p < 2 || p > 512) return -1;
  uint64_t z = seed;
  auto rnd = [&]() {
    z += 0x9E3779B97F4A7C15ull;
    uint64_t x = z;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
  };
  const int nl = (p + 63) >> 6;
  auto rand_f = [&](int64_t ec) {
    ff::F v;
    v.sign = (rnd() & 1) ? 1 : -1;
    for (int i = 0; i < ff::NL; ++i) v.m[i] = i < nl ? rnd() : 0;
    if (rnd() % 8 == 0)  // runs of ones: carries through every limb
      for (int i = 0; i < nl; ++i) v.m[i] = ~0ull;
    for (int b = p; b < 64 * nl; ++b) v.m[b >> 6] &= ~(1ull << (b & 63));
    v.m[(p - 1) >> 6] |= 1ull << ((p - 1) & 63);
    v.exp = ec - p;
    if (rnd() % 64 == 0) v = ff::F();  // zeros
    return v;
  };
  const size_t nn = (size_t)n * n;
  std::vector<ff::F> A(nn), x(n), b(n), r_host(n), r_dev(n);
  for (auto &v : A) v = rand_f((int64_t)(rnd() % 40) - 20);
  for (auto &v : x) v = rand_f((int64_t)(rnd() % 40) - 20);
  // b close to A x in some rows (cancellation), random elsewhere
  for (int i = 0; i < n; ++i) {
    ff::F acc;
    for (int j = 0; j < n; ++j)
      acc = ff::fadd(acc, ff::fmul(A[(size_t)i * n + j], x[j], p), p);
    if (i % 3 == 0) {
      b[i] = acc;
      if (i % 6 == 0 && acc.sign != 0) b[i].m[0] ^= 1ull << ((nl * 64 - p) & 63);
    } else {
      b[i] = rand_f((int64_t)(rnd() % 40) - 10);
    }
    r_host[i] = ff::fadd(b[i], ff::neg(acc), p);
  }
  void *dA = nullptr, *dx = nullptr, *db = nullptr, *dr = nullptr;
  const size_t fb = sizeof(ff::F);
  int64_t bad = -1;
  if (cudaMalloc(&dA, nn * fb) == cudaSuccess &&
      cudaMalloc(&dx, n * fb) == cudaSuccess &&
      cudaMalloc(&db, n * fb) == cudaSuccess &&
      cudaMalloc(&dr, n * fb) == cudaSuccess &&
      cudaMemcpy(dA, A.data(), nn * fb, cudaMemcpyHostToDevice) == cudaSuccess &&
      cudaMemcpy(dx, x.data(), n * fb, cudaMemcpyHostToDevice) == cudaSuccess &&
      cudaMemcpy(db, b.data(), n * fb, cudaMemcpyHostToDevice) == cudaSuccess &&
      mpk::long_residual(p, n, dA, dx, db, dr, s, variant) == cudaSuccess &&
      cudaStreamSynchronize(s) == cudaSuccess &&
      cudaMemcpy(r_dev.data(), dr, n * fb, cudaMemcpyDeviceToHost) == cudaSuccess) {
    bad = 0;
    for (int i = 0; i < n; ++i) {
      const ff::F &u = r_host[i], &v = r_dev[i];
      bool same = u.sign == v.sign;
      if (same && u.sign != 0) {
        same = u.exp == v.exp;
        for (int l = 0; l < nl; ++l) same = same && u.m[l] == v.m[l];
      }
      if (!same) ++bad;
    }
  }
  for (void *q : {dA, dx, db, dr})
    if (q) cudaFree(q);
  return bad;
}

int refine_files(const char *a_path, const char *b_path, int short_k,
                 int long_bits, const char *rtol_s, const char *atol_s,
                 int max_iter, ShortSolver &S, Report &out, std::string &err) {
  Loaded A, B;
  int st = load_mpmat(a_path, A, err);
  if (st) return st;
  st = load_mpmat(b_path, B, err);
  if (st) return st;
  if (B.cols != 1) {
    err = std::string(b_path) + ": vector file must have 1 column";
    return 4;
  }
  if (short_k < 2 || short_k > 4) { err = "short_k must be 2, 3, or 4"; return 6; }
  if (long_bits <= 53 * short_k) { err = "long_bits must exceed 53 * short_k"; return 6; }
  if (max_iter < 1) { err = "max_iter must be >= 1"; return 6; }
  if (!A.bf || !B.bf) { err = "refinement expects BigFloat matrix and vector"; return 6; }
  if (A.rows != A.cols) { err = "matrix must be square"; return 2; }
  if (B.rows != A.rows) { err = "rhs length does not match n"; return 2; }
  return refine_core(A.vals, B.vals, A.rows, short_k, long_bits, rtol_s,
                     atol_s, max_iter, 0, S, out, err);
}

}  // namespace mpr

namespace mpr {
// The device long -> short conversion (convert.cu) against the host's
// ff::from_bf + ff::to_multicomp: values of 1 .. 640 bits, exponents across
// the binary64 range edges, runs of ones (rounding carries), exact halves.
int64_t convert_selftest(int64_t iters, uint64_t seed, int p, int k,
                         cudaStream_t s) {
  if (iters <= 0 || p < 2 || p > 64 * ff::NL || k < 2 || k > 4) return -1;
  uint64_t z = seed;
  auto rnd = [&]() {
    z += 0x9E3779B97F4A7C15ull;
    uint64_t x = z;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
  };
  std::vector<ff::F> flat(iters);
  std::vector<ff::F> host_f(iters);
  std::vector<double> host_c(4 * iters, 0.0);
  std::vector<int> host_ok(iters);
  for (int64_t it = 0; it < iters; ++it) {
    BF v;
    const int bits = 1 + (int)(rnd() % (64 * ff::NL));
    bn::UBig m;
    for (int b = 0; b < bits; b += 32) m.w.push_back((uint32_t)rnd());
    m = m.shr((int64_t)m.w.size() * 32 - bits);
    m.trim();
    if (rnd() % 6 == 0) {  // runs of ones / exact halves
      m = bn::UBig::sub(bn::UBig(1).shl(bits), bn::UBig(1 + rnd() % 2));
      if (rnd() & 1) m = bn::UBig::add(m.shl(0), bn::UBig(1).shl(bits / 2));
      m.trim();
    }
    if (m.zero() || rnd() % 50 == 0) {
      v = BF();
    } else {
      v.sign = (rnd() & 1) ? 1 : -1;
      v.man = m;
      const int64_t kind = rnd() % 10;
      const int64_t top = kind == 0 ? 1020 + (int64_t)(rnd() % 8)
                          : kind == 1 ? -1015 - (int64_t)(rnd() % 12)
                                      : (int64_t)(rnd() % 200) - 100;
      v.exp = top - bits;
    }
    if (!flat_from_bf(v, flat[it])) {  // > 640 bits: the host path's
      flat[it] = ff::F();               // (not compared)
      flat[it].sign = 0;
      std::memset(flat[it].m, 0, sizeof flat[it].m);
      host_ok[it] = -1;
      continue;
    }
    host_f[it] = ff::from_bf(v, p);
    host_ok[it] = ff::to_multicomp(host_f[it], k, p, &host_c[4 * it]) ? 1 : 0;
  }
  // the compact records too (values of at most 576 bits)
  std::vector<mpk::LongFlat9> flat9(iters);
  std::vector<int> has9(iters, 0);
  for (int64_t it = 0; it < iters; ++it) {
    if (host_ok[it] < 0) continue;
    BF v;
    v.sign = flat[it].sign;
    v.exp = flat[it].exp;
    for (int l = 0; l < ff::NL; ++l) {
      v.man.w.push_back((uint32_t)flat[it].m[l]);
      v.man.w.push_back((uint32_t)(flat[it].m[l] >> 32));
    }
    v.man.trim();
    has9[it] = flat9_from_bf(v, flat9[it]) ? 1 : 0;
  }
  void *dA = nullptr, *dh = nullptr, *dok = nullptr, *d9 = nullptr;
  std::vector<ff::F> dev_f(iters);
  std::vector<double> dev_c(4 * iters);
  std::vector<int> dev_ok(iters);
  int64_t bad = -1;
  const size_t fb = sizeof(ff::F) * iters;
  // pass 0: the full records converted in place; pass 1: the compact ones
  for (int pass = 0; pass < 2; ++pass) {
    bool okc = true;
    if (pass == 0)
      okc = cudaMalloc(&dA, fb) == cudaSuccess &&
            cudaMalloc(&dh, sizeof(double) * 4 * iters) == cudaSuccess &&
            cudaMalloc(&dok, sizeof(int) * iters) == cudaSuccess &&
            cudaMalloc(&d9, sizeof(mpk::LongFlat9) * iters) == cudaSuccess &&
            cudaMemcpy(dA, flat.data(), fb, cudaMemcpyHostToDevice) ==
                cudaSuccess &&
            mpk::long_to_short_selftest(k, p, dA, nullptr, iters,
                                        static_cast<double *>(dh),
                                        static_cast<int *>(dok), s) ==
                cudaSuccess;
    else
      okc = cudaMemcpy(d9, flat9.data(), sizeof(mpk::LongFlat9) * iters,
                       cudaMemcpyHostToDevice) == cudaSuccess &&
            mpk::long_to_short_selftest(k, p, dA, d9, iters,
                                        static_cast<double *>(dh),
                                        static_cast<int *>(dok), s) ==
                cudaSuccess;
    okc = okc && cudaStreamSynchronize(s) == cudaSuccess &&
          cudaMemcpy(dev_f.data(), dA, fb, cudaMemcpyDeviceToHost) ==
              cudaSuccess &&
          cudaMemcpy(dev_c.data(), dh, sizeof(double) * 4 * iters,
                     cudaMemcpyDeviceToHost) == cudaSuccess &&
          cudaMemcpy(dev_ok.data(), dok, sizeof(int) * iters,
                     cudaMemcpyDeviceToHost) == cudaSuccess;
    if (!okc) {
      bad = -1;
      break;
    }
    if (pass == 0) bad = 0;
    const int nl = (p + 63) >> 6;
    for (int64_t it = 0; it < iters; ++it) {
      if (host_ok[it] < 0 || (pass == 1 && !has9[it])) continue;
      const ff::F &u = host_f[it], &w = dev_f[it];
      bool same = u.sign == w.sign;
      if (same && u.sign != 0) {
        same = u.exp == w.exp;
        for (int l = 0; l < ff::NL; ++l)
          same = same && (l < nl ? u.m[l] == w.m[l] : w.m[l] == 0);
      }
      same = same && host_ok[it] == dev_ok[it];
      if (same && host_ok[it])
        same = std::memcmp(&host_c[4 * it], &dev_c[4 * it],
                           sizeof(double) * k) == 0;
      if (!same && bad < 3 && std::getenv("MPCORE_SELFTEST_VERBOSE"))
        std::fprintf(stderr, "convert mismatch (pass %d) at %lld\n", pass,
                     (long long)it);
      if (!same) ++bad;
    }
  }
  for (void *q : {dA, dh, dok, d9})
    if (q) cudaFree(q);
  return bad;
}
}  // namespace mpr
