// DD/TD/QD GEMM on the FP64 pipe: mat_mul_blocked (linalg.py:577-617) and
// the LU trailing update (linalg.py:444-448 regrouped per panel).
//
//   C_ij <- fold over p = 0..KK-1 (ascending) of add(C_ij, mul(opA(A_ip), B_pj))
//
// opA = identity for mat_mul_blocked (C starts at exact +0.0, linalg.py:
// 586-597) and opA = negation for the trailing update A22 += (-L21) U12,
// whose chain per element continues the reference's rank-1 sequence
// A_ic = add(A_ic, mul(-m_i, A_jc)) over the panel's steps j in ascending
// order.  Each output element's chain is sequential in p (no split-K, no
// Strassen) so results are bitwise those of the reference.
//
// Tiling: a CTA owns a BM x BN output tile; K-slices of BK are staged through
// shared memory with cp.async (double-buffered); each thread keeps a TM x TN
// register micro-tile of accumulators (strided over the CTA tile so shared
// loads are broadcast / conflict-free).  The work is FP64-issue bound: per
// madd 29 / 264 / 376 FP64 instructions (DD/TD/QD) against (TM+TN)/(TM*TN)
// operand loads from shared memory.
#include "internal.h"
#include "mc.cuh"

namespace mpk {

namespace {

__device__ __forceinline__ void cp_async8(void *smem, const void *gmem,
                                          bool pred) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s),
               "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::);
}
template <int N> __device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

template <int K, int BM, int BN, int BK, int TM, int TN>
struct GemmCfg {
  static constexpr int TX = BN / TN, TY = BM / TM, NT = TX * TY;
  static constexpr int A_ELEMS = BM * BK, B_ELEMS = BK * BN;
  static constexpr int STAGE = K * (A_ELEMS + B_ELEMS);
  static constexpr size_t SMEM = 2 * STAGE * sizeof(double);
};

template <int K, int BM, int BN, int BK, int TM, int TN, bool NEG_A,
          bool ZERO, int MINB>
__global__ void __launch_bounds__((BM / TM) * (BN / TN), MINB)
gemm_kernel(int M, int N, int KK, MatView A, MatView B, MatView C,
            const int32_t *__restrict__ status) {
  using Cfg = GemmCfg<K, BM, BN, BK, TM, TN>;
  constexpr int TX = Cfg::TX, TY = Cfg::TY, NT = Cfg::NT;
  if (status != nullptr && status[0] >= 0) return;  // singular: stop
  extern __shared__ double smem[];
  const int tid = threadIdx.x;
  const int tx = tid % TX, ty = tid / TX;
  const int i0 = blockIdx.y * BM, j0 = blockIdx.x * BN;

  auto load_a = [&](int stage, int k0) {
    double *As = smem + stage * Cfg::STAGE;
    for (int e = tid; e < Cfg::A_ELEMS; e += NT) {
      int r = e / BK, q = e % BK;
      int gi = i0 + r, gq = k0 + q;
      bool ok = gi < M && gq < KK;
      int64_t off = ok ? (int64_t)gi * A.ld + gq : 0;
#pragma unroll
      for (int c = 0; c < K; ++c)
        cp_async8(As + c * Cfg::A_ELEMS + e, A.p + c * A.plane + off, ok);
    }
  };
  auto load_b = [&](int stage, int k0) {
    double *Bs = smem + stage * Cfg::STAGE + K * Cfg::A_ELEMS;
    for (int e = tid; e < Cfg::B_ELEMS; e += NT) {
      int q = e / BN, cc = e % BN;
      int gq = k0 + q, gj = j0 + cc;
      bool ok = gq < KK && gj < N;
      int64_t off = ok ? (int64_t)gq * B.ld + gj : 0;
#pragma unroll
      for (int c = 0; c < K; ++c)
        cp_async8(Bs + c * Cfg::B_ELEMS + e, B.p + c * B.plane + off, ok);
    }
  };
  auto load_tile = [&](int stage, int k0) {
    load_a(stage, k0);
    load_b(stage, k0);
    cp_async_commit();
  };
  const int ntiles = (KK + BK - 1) / BK;
  if (ntiles > 0) load_tile(0, 0);

  double acc[TM][TN][K];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      int gi = i0 + ty + i * TY, gj = j0 + tx + j * TX;
      bool ok = gi < M && gj < N;
#pragma unroll
      for (int c = 0; c < K; ++c)
        acc[i][j][c] = (ZERO || !ok)
                           ? 0.0
                           : C.p[c * C.plane + (int64_t)gi * C.ld + gj];
    }

  for (int kt = 0; kt < ntiles; ++kt) {
    if (kt + 1 < ntiles) {
      load_tile((kt + 1) & 1, (kt + 1) * BK);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double *As = smem + (kt & 1) * Cfg::STAGE;
    const double *Bs = As + K * Cfg::A_ELEMS;
    const int kmax = min(BK, KK - kt * BK);
    // small micro-tiles expose the accumulator chain: unroll so the products
    // of the next steps overlap it
#pragma unroll(TM * TN <= 2 ? 4 : 1)
    for (int kk = 0; kk < kmax; ++kk) {
      double a[TM][K], b[TN][K];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int c = 0; c < K; ++c) {
          double v = As[c * Cfg::A_ELEMS + (ty + i * TY) * BK + kk];
          a[i][c] = NEG_A ? -v : v;
        }
#pragma unroll
      for (int j = 0; j < TN; ++j)
#pragma unroll
        for (int c = 0; c < K; ++c)
          b[j][c] = Bs[c * Cfg::B_ELEMS + kk * BN + tx + j * TX];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) mc::madd<K>(acc[i][j], a[i], b[j]);
    }
    __syncthreads();
  }

#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      int gi = i0 + ty + i * TY, gj = j0 + tx + j * TX;
      if (gi < M && gj < N) {
#pragma unroll
        for (int c = 0; c < K; ++c)
          C.p[c * C.plane + (int64_t)gi * C.ld + gj] = acc[i][j][c];
      }
    }
}

template <int BM_, int BN_, int BK_, int TM_, int TN_, int MINB_>
struct TileT {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, TM = TM_, TN = TN_,
                       MINB = MINB_;
};

template <int K, class T, bool NEG_A, bool ZERO>
struct Launcher {
  using Cfg = GemmCfg<K, T::BM, T::BN, T::BK, T::TM, T::TN>;
  static constexpr auto kern =
      gemm_kernel<K, T::BM, T::BN, T::BK, T::TM, T::TN, NEG_A, ZERO, T::MINB>;
  // resident CTAs per SM (0 if the shape cannot launch)
  static int slots() {
    static const int v = [] {
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)Cfg::SMEM) != cudaSuccess)
        return 0;
      int per = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, Cfg::NT,
                                                    Cfg::SMEM);
      return per;
    }();
    return v;
  }
  static cudaError_t run(int M, int N, int KK, MatView A, MatView B, MatView C,
                         const int32_t *status, cudaStream_t s) {
    if (slots() <= 0) return cudaErrorInvalidConfiguration;
    dim3 grid((N + T::BN - 1) / T::BN, (M + T::BM - 1) / T::BM);
    kern<<<grid, Cfg::NT, Cfg::SMEM, s>>>(M, N, KK, A, B, C, status);
    return cudaGetLastError();
  }
};

// Candidate tiles per precision: (index, BM, BN, BK, TM, TN, min CTAs/SM),
// 256 threads each; 6 and 7 are the 128- and 64-thread tiles for launches
// too small to give every SM a 256-thread tile.
#define MPK_TILES_DD(X)                                                       \
  X(0, 64, 64, 16, 4, 4, 2) X(1, 32, 64, 16, 2, 4, 2)                         \
  X(2, 64, 32, 16, 4, 2, 2) X(3, 32, 32, 16, 2, 2, 2)                         \
  X(4, 16, 32, 16, 1, 2, 2) X(5, 32, 32, 16, 2, 2, 3)                         \
  X(6, 8, 16, 16, 1, 1, 4) X(7, 8, 8, 16, 1, 1, 8)
#define MPK_TILES_XD(X)                                                       \
  X(0, 32, 32, 16, 2, 2, 1) X(1, 32, 16, 16, 2, 1, 2)                         \
  X(2, 16, 32, 16, 1, 2, 2) X(3, 16, 16, 16, 1, 1, 2)                         \
  X(4, 8, 32, 16, 1, 1, 2) X(5, 32, 32, 16, 2, 2, 2)                          \
  X(6, 8, 16, 16, 1, 1, 4) X(7, 8, 8, 16, 1, 1, 8)
// Their FP64 issue efficiency at a many-wave update shape (M = N = 8192,
// KK = 32; tools/tile_sweep.py on B200), which the wave-aware chooser
// weighs against tile quantisation.  (6, 7: only used below one tile per
// SM, where the SM count, not the efficiency, decides.)
constexpr double TILE_EFF[3][8] = {
    {0.940, 0.924, 0.918, 0.902, 0.852, 0.910, 0.8, 0.8},    // DD
    {0.987, 0.981, 0.981, 0.976, 0.965, 0.990, 0.95, 0.95},  // TD
    {0.975, 0.984, 0.987, 0.984, 0.976, 0.998, 0.95, 0.95}}; // QD
constexpr int NTILES = 8;
constexpr unsigned SMALL_TILES = 0xc0u;

struct TileInfo {
  int bm, bn, slots;
  double eff;
};

template <int K, bool NEG_A, bool ZERO>
TileInfo tile_info(int idx) {
#define MPK_INFO(I, BM, BN, BK, TM, TN, MB)                                  \
  case I:                                                                    \
    return {BM, BN,                                                          \
            Launcher<K, TileT<BM, BN, BK, TM, TN, MB>, NEG_A, ZERO>::slots(), \
            TILE_EFF[K - 2][I]};
  if constexpr (K == 2) {
    switch (idx) { MPK_TILES_DD(MPK_INFO) }
  } else {
    switch (idx) { MPK_TILES_XD(MPK_INFO) }
  }
#undef MPK_INFO
  return {1, 1, 0, 1.0};
}

template <int K, bool NEG_A, bool ZERO>
cudaError_t launch_idx(int idx, int M, int N, int KK, MatView A, MatView B,
                       MatView C, const int32_t *status, cudaStream_t s) {
#define MPK_RUN(I, BM, BN, BK, TM, TN, MB)                                    \
  case I:                                                                    \
    return Launcher<K, TileT<BM, BN, BK, TM, TN, MB>, NEG_A, ZERO>::run(      \
        M, N, KK, A, B, C, status, s);
  if constexpr (K == 2) {
    switch (idx) { MPK_TILES_DD(MPK_RUN) }
  } else {
    switch (idx) { MPK_TILES_XD(MPK_RUN) }
  }
#undef MPK_RUN
  return cudaErrorInvalidValue;
}

// MPCORE_GEMM_TILE=i forces candidate i (tuning sweeps); -1 = choose
int tile_override() {
  static const int v = [] {
    const char *e = std::getenv("MPCORE_GEMM_TILE");
    return e ? std::atoi(e) : -1;
  }();
  return v;
}

// Every CTA of a wave costs the same (same KK), so the time of an M x N
// product is ~ ceil(tiles / resident slots) * tile area / efficiency; pick
// the candidate minimising it (the trailing update shrinks every panel, so
// a fixed tile wastes up to a wave per launch).
//
// A launch with fewer tiles than SMs leaves SMs idle and the busy ones run
// a whole tile each: then the 128/64-thread tiles (SMALL_TILES) compete on
// the outputs of the busiest SM, ceil(tiles / SMs) * tile area.
template <int K, bool NEG_A, bool ZERO>
int choose_tile(int M, int N, unsigned mask = 0x3fu) {
  const int forced = tile_override();
  if (forced >= 0 && forced < NTILES) return forced;
  const int sms = num_sms();
  static const bool small_ok = std::getenv("MPCORE_NO_SMALL_TILES") == nullptr;
  int best = 0;
  double best_cost = 1e300;
  for (int i = 0; i < NTILES; ++i) {
    if (!(mask >> i & 1u)) continue;
    const TileInfo t = tile_info<K, NEG_A, ZERO>(i);
    if (t.slots <= 0) continue;
    const int64_t tiles =
        (int64_t)((M + t.bm - 1) / t.bm) * ((N + t.bn - 1) / t.bn);
    if (tiles < sms && small_ok) {
      // under one tile per SM: the busiest SM's outputs decide
      int sbest = i;
      double scost = (double)t.bm * t.bn / t.eff;
      for (int q = 0; q < NTILES; ++q) {
        if (!(SMALL_TILES >> q & 1u)) continue;
        const TileInfo u = tile_info<K, NEG_A, ZERO>(q);
        if (u.slots <= 0) continue;
        const int64_t ut =
            (int64_t)((M + u.bm - 1) / u.bm) * ((N + u.bn - 1) / u.bn);
        const double c = (double)((ut + sms - 1) / sms) * u.bm * u.bn / u.eff;
        if (c < scost * 0.999) {
          scost = c;
          sbest = q;
        }
      }
      return sbest;
    }
  }
  for (int i = 0; i < NTILES; ++i) {
    if (!(mask >> i & 1u)) continue;
    const TileInfo t = tile_info<K, NEG_A, ZERO>(i);
    if (t.slots <= 0) continue;
    const int64_t tiles =
        (int64_t)((M + t.bm - 1) / t.bm) * ((N + t.bn - 1) / t.bn);
    const int64_t slots = (int64_t)t.slots * sms;
    const double waves = (double)((tiles + slots - 1) / slots);
    const double cost = waves * t.bm * t.bn * t.slots / t.eff;
    if (cost < best_cost * 0.999) {
      best_cost = cost;
      best = i;
    }
  }
  return best;
}

template <int K, bool NEG_A, bool ZERO>
cudaError_t launch(int M, int N, int KK, MatView A, MatView B, MatView C,
                   const int32_t *status, cudaStream_t s,
                   unsigned mask = 0x3fu) {
  // (mask selects among the 256-thread tiles; small ones are added below
  // one tile per SM)
  return launch_idx<K, NEG_A, ZERO>(choose_tile<K, NEG_A, ZERO>(M, N, mask),
                                    M, N, KK, A, B, C, status, s);
}

// Candidates for the LU trailing update, which shares the GPU with the
// look-ahead panel: measured over whole LUs (tools/tile_mask.sh, n = 2048)
// the short-lived tiles win -- 16 x 16 for TD/QD, everything but 64 x 64
// for DD.  MPCORE_UPDATE_TILES=mask overrides.
unsigned update_mask(int k) {
  static const unsigned v = [] {
    const char *e = std::getenv("MPCORE_UPDATE_TILES");
    return e ? (unsigned)std::strtoul(e, nullptr, 0) : 0u;
  }();
  if (v) return v;
  return k == 2 ? 0x3eu : 0x08u;
}

}  // namespace

cudaError_t gemm(int k, bool neg_a, bool zero_init, int M, int N, int KK,
                 MatView A, MatView B, MatView C, cudaStream_t s) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  prof_begin(PROF_GEMM, s);
  cudaError_t e = cudaErrorInvalidValue;
#define GEMM_CASE(KV)                                                       \
  case KV:                                                                  \
    if (neg_a)                                                              \
      e = zero_init ? launch<KV, true, true>(M, N, KK, A, B, C, nullptr, s) \
                    : launch<KV, true, false>(M, N, KK, A, B, C, nullptr, s); \
    else                                                                    \
      e = zero_init ? launch<KV, false, true>(M, N, KK, A, B, C, nullptr, s) \
                    : launch<KV, false, false>(M, N, KK, A, B, C, nullptr, s); \
    break;
  switch (k) {
    GEMM_CASE(2)
    GEMM_CASE(3)
    GEMM_CASE(4)
    default: break;
  }
#undef GEMM_CASE
  prof_end(PROF_GEMM, s);
  return e;
}

cudaError_t lu_update(int k, int M, int N, int w, MatView L21, MatView U12,
                      MatView A22, const int32_t *status, cudaStream_t s,
                      int prof_slot) {
  if (M <= 0 || N <= 0 || w <= 0) return cudaSuccess;
  prof_begin(prof_slot, s);
  cudaError_t e = cudaErrorInvalidValue;
  switch (k) {
    case 2: e = launch<2, true, false>(M, N, w, L21, U12, A22, status, s, update_mask(2)); break;
    case 3: e = launch<3, true, false>(M, N, w, L21, U12, A22, status, s, update_mask(3)); break;
    case 4: e = launch<4, true, false>(M, N, w, L21, U12, A22, status, s, update_mask(4)); break;
    default: break;
  }
  prof_end(prof_slot, s);
  return e;
}

}  // namespace mpk
