// Panel factorisation kernel (included by lu.cu; see the protocol notes at
// the top of lu.cu).  Warp-specialised:
//   warp 0 ("W0") runs the per-column critical chain with warp-level
//     synchronisation only: poll every CTA's candidate words, global first
//     max (redux.sync), recip = div(1, pivot) (all lanes, same bits),
//     multipliers, look-ahead update of the next column, local first max of
//     that column, publish the next candidate;
//   warps 1..7 ("H") stream the winner's pivot row, apply the row exchange,
//     run the rank-1 update of the remaining panel columns and publish the
//     candidate rows;
// coupled by named barriers (bar.arrive by the producer, bar.sync by the
// consumer, 256 threads per barrier):
//   B_WIN  W0 -> H : winner of column jj known (smem)
//   B_ROW  H -> W0 : pivot row staged, swap applied
//   B_MUL  W0 -> H : multipliers of column jj + next candidate row known
//   B_REM  H -> W0 : remaining update of column jj done, rows published
//
// Included inside namespace mpk::{anonymous} of lu.cu (uses its helpers).
#pragma once

constexpr int B_WIN = 1, B_ROW = 2, B_MUL = 3, B_REM = 4, B_H = 5;
constexpr int H_THREADS = PANEL_THREADS - 32;

// a double travels as two LL words (low half, high half)
__device__ __forceinline__ unsigned lo32(double v) {
  return (unsigned)((unsigned long long)__double_as_longlong(v) & 0xffffffffu);
}
__device__ __forceinline__ unsigned hi32(double v) {
  return (unsigned)((unsigned long long)__double_as_longlong(v) >> 32);
}

__device__ __forceinline__ void nb_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void nb_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// warp-wide first max of (key, row): larger mag_key first (NaN above
// everything), then the smaller row (np.argmax); row INT_MAX = no candidate.
// Three integer reductions decide it exactly.
__device__ __forceinline__ void warp_argmax(unsigned long long key, int row,
                                            int &out_row) {
  const bool valid = row != INT_MAX;
  const unsigned long long b = valid ? key : 0ull;
  unsigned hi = (unsigned)(b >> 32), lo = (unsigned)b;
  unsigned vmask = __ballot_sync(0xffffffffu, valid);
  if (!valid) hi = 0u;
  unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  unsigned lo_c = (valid && hi == mhi) ? lo : 0u;
  unsigned mlo = __reduce_max_sync(0xffffffffu, lo_c);
  unsigned rc = (valid && hi == mhi && lo == mlo) ? (unsigned)row : 0xffffffffu;
  unsigned mrow = __reduce_min_sync(0xffffffffu, rc);
  out_row = vmask == 0u ? INT_MAX : (int)mrow;
}

struct PanelSmem {
  double recip[LU_MAX_K];
  int winner;      // global row of the pivot of the current column
  int gw;          // CTA owning it
  int cand_row;    // this CTA's candidate for the next column
  int flag;        // 1 singular / last column: stop after B_WIN
  int singular;    // 1: stop without write-back
  int piv[LU_MAX_W];                 // winner of every column of the panel
};

template <int K, int W, int SPL>
__global__ void __launch_bounds__(PANEL_THREADS, 1)
panel_kernel(int n, MatView A, int J, int w, int32_t *__restrict__ swaps,
             LuWork ws, int slot) {
  const int G = gridDim.x, g = blockIdx.x, tid = threadIdx.x;
  const int lane = tid & 31;
  if (tid == 0) lu_stamp(J, 0, true);
  if (ws.status[0] >= 0) return;
  if (ws.trace != nullptr && ws.trace_J == J && tid == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    ws.trace[((int64_t)g * 33 + 32) * 8 + 0] = t;
  }
  const unsigned seq0 = ws.epoch[0] + (unsigned)J + 1u;  // (LuWork::epoch)
  const int m = n - J;
  const int R = (m + G - 1) / G;
  const int rbeg = J + g * R;
  const int nr = max(0, min(rbeg + R, n) - rbeg);
  const int rw = 2 * w * K;
  extern __shared__ double sm[];
  // [R][W*K + 1]: the odd row stride keeps warp 0's column accesses (lane =
  // row) free of shared-memory bank conflicts
  constexpr int RS = W * K + 1;
  double *rows = sm;
  double *prow = rows + R * RS;       // [W][K]
  __shared__ PanelSmem S;
  auto at = [&](int r, int col) -> double * { return rows + r * RS + col * K; };

  for (int e = tid; e < nr * w; e += PANEL_THREADS) {
    int r = e / w, col = e % w;
#pragma unroll
    for (int c = 0; c < K; ++c)
      at(r, col)[c] = A.p[c * A.plane + (int64_t)(rbeg + r) * A.ld + J + col];
  }
  if (tid == 0) {
    S.flag = 0;
    S.singular = 0;
  }
  __syncthreads();

  // W0: local first max of column jj (rows >= J+jj) and its candidate words
  auto w0_publish_max = [&](int jj, unsigned seq, unsigned long long key,
                            int row) {
    int br;
    warp_argmax(key, row, br);
    u64 *wd = ws.cand_words + ((int64_t)(jj & 1) * G + g) * LU_CAND_WORDS;
    if (lane == 0) {
      S.cand_row = br;
      st_volatile(wd, ll_word((unsigned)br, seq));
    } else if (lane <= 2 * K) {
      // the candidate's value (its |head| is the magnitude): 2K words
      const double v = br != INT_MAX ? at(br - rbeg, jj)[(lane - 1) >> 1] : 0.0;
      st_volatile(wd + lane, ll_word((lane & 1) ? lo32(v) : hi32(v), seq));
    }
  };
  // (each lane scans its rows in increasing order, so "strictly larger"
  // keeps the first maximum; warp_argmax breaks ties across lanes by row)
  auto w0_publish_candidate = [&](int jj, unsigned seq) {
    const int j = J + jj;
    unsigned long long key = 0ull;
    int row = INT_MAX;
    for (int r = lane; r < nr; r += 32) {
      int gi = rbeg + r;
      if (gi >= j) {
        const unsigned long long kv = mag_key(fabs(at(r, jj)[0]));
        if (row == INT_MAX || kv > key) { key = kv; row = gi; }
      }
    }
    w0_publish_max(jj, seq, key, row);
  };
  // H: publish the candidate row of column jj (+ row J+jj if owned)
  auto h_publish_rows = [&](int jj, unsigned seq, int row) {
    const int j = J + jj, par = jj & 1, ht = tid - 32;
    if (row != INT_MAX) {
      u64 *wd = ws.row_words + ((int64_t)par * G + g) * LU_ROW_WORDS;
      const double *src = at(row - rbeg, 0);
      for (int e = ht; e < rw; e += H_THREADS) {
        double v = src[e >> 1];
        st_volatile(wd + e, ll_word((e & 1) ? hi32(v) : lo32(v), seq));
      }
    }
    if (j >= rbeg && j < rbeg + nr) {
      u64 *wd = ws.rowj_words + (int64_t)par * LU_ROW_WORDS;
      const double *src = at(j - rbeg, 0);
      for (int e = ht; e < rw; e += H_THREADS) {
        double v = src[e >> 1];
        st_volatile(wd + e, ll_word((e & 1) ? hi32(v) : lo32(v), seq));
      }
    }
  };
  const bool tracing = ws.trace != nullptr && ws.trace_J == J && tid == 0;
  auto trace = [&](int jj, int slot) {
    if (tracing) {
      unsigned long long t;
      if (slot == 0) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        ws.trace[((int64_t)g * 33 + jj) * 8 + 7] = t;
      }
      t = clock64();
      ws.trace[((int64_t)g * 33 + jj) * 8 + slot] = t;
    }
  };
  auto poll = [&](const u64 *p, unsigned seq) -> unsigned {
    u64 v = ld_volatile(p);
    while ((unsigned)v != seq) {
      __nanosleep(ws.poll_ns);
      v = ld_volatile(p);
    }
    return (unsigned)(v >> 32);
  };

  auto stamp = [&](int slot) {
    if (tracing) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      ws.trace[((int64_t)g * 33 + 32) * 8 + slot] = t;
    }
  };
  stamp(1);
  // prologue: candidate and rows of column 0 (all columns current)
  if (tid < 32) w0_publish_candidate(0, seq0);
  __syncthreads();
  if (tid >= 32) h_publish_rows(0, seq0, S.cand_row);

  if (tid < 32) {
    // ================================================================ W0 ==
    for (int jj = 0; jj < w; ++jj) {
      const int j = J + jj, par = jj & 1;
      const unsigned seq = seq0 + jj;
      trace(jj, 0);
      // every slot's row and value words (1 + 2K); the magnitude is the
      // value's |head|, so the winner's pivot arrives with the poll itself
      // SPL slots per lane (G <= 32 * SPL)
      constexpr int NW = 1 + 2 * K;
      u64 wv[SPL][NW];
      unsigned done = 0;  // bit q: slot lane+32q complete (or absent)
#pragma unroll
      for (int q = 0; q < SPL; ++q)
        if (lane + 32 * q >= G) done |= 1u << q;
      for (;;) {
#pragma unroll
        for (int q = 0; q < SPL; ++q) {
          if (!(done & (1u << q))) {
            const u64 *wd = ws.cand_words +
                            ((int64_t)par * G + lane + 32 * q) * LU_CAND_WORDS;
#pragma unroll
            for (int x = 0; x < NW; ++x) wv[q][x] = ld_volatile(wd + x);
          }
        }
#pragma unroll
        for (int q = 0; q < SPL; ++q) {
          if (!(done & (1u << q))) {
            bool all = true;
#pragma unroll
            for (int x = 0; x < NW; ++x)
              if ((unsigned)wv[q][x] != seq) all = false;
            if (all) done |= 1u << q;
          }
        }
        if (__all_sync(0xffffffffu, done == (1u << SPL) - 1u)) break;
        __nanosleep(ws.poll_ns);
      }
      // (a lane's slots hold increasing row ranges: "strictly larger"
      // keeps the first maximum)
      unsigned long long bk = 0ull;
      int br = INT_MAX;
      unsigned bw[2 * K];
#pragma unroll
      for (int x = 0; x < 2 * K; ++x) bw[x] = 0u;
#pragma unroll
      for (int q = 0; q < SPL; ++q) {
        if (lane + 32 * q < G) {
          const int rr = (int)(wv[q][0] >> 32);
          const unsigned long long kk = mag_key(fabs(__longlong_as_double(
              (long long)((wv[q][2] & 0xffffffff00000000ull) | (wv[q][1] >> 32)))));
          if (rr != INT_MAX && (br == INT_MAX || kk > bk)) {
            bk = kk;
            br = rr;
#pragma unroll
            for (int x = 0; x < 2 * K; ++x) bw[x] = (unsigned)(wv[q][1 + x] >> 32);
          }
        }
      }
      int r;
      warp_argmax(bk, br, r);
      trace(jj, 1);
      const int gw = (r - J) / R;
      if (g == 0 && lane == 0) swaps[j] = r;
      // pivot value of the winner: from the lane whose best slot won
      const int src = __ffs(__ballot_sync(0xffffffffu, br == r)) - 1;
      double pv[K];
#pragma unroll
      for (int c = 0; c < K; ++c) {
        unsigned l = __shfl_sync(0xffffffffu, bw[2 * c], src);
        unsigned h = __shfl_sync(0xffffffffu, bw[2 * c + 1], src);
        pv[c] = __longlong_as_double((long long)(((u64)h << 32) | l));
      }
      const bool singular = pv[0] == 0.0;
      const bool last = (j == n - 1);
      if (lane == 0) {
        S.winner = r;
        S.piv[jj] = r;
        S.gw = gw;
        S.flag = (singular || last) ? 1 : 0;
        S.singular = singular ? 1 : 0;
        if (singular && g == 0) ws.status[0] = j;
      }
      __syncwarp();
      nb_arrive(B_WIN, PANEL_THREADS);
      if (singular) return;
      if (last) break;
      // recip = div(1, pivot): every lane computes the same value
      double rc[K];
      mc::recip<K>(pv, rc);
      trace(jj, 2);
      nb_sync(B_ROW, PANEL_THREADS);  // pivot row staged, swap applied
      trace(jj, 3);
      // (H finished column jj-1 before it staged this pivot row, so this
      // wait is only the barrier's bookkeeping)
      if (jj >= 1) nb_sync(B_REM, PANEL_THREADS);
      // one pass over the rows i > j: multiplier m_i = mul(A_ij, recip),
      // look-ahead update of column jj+1 and its local first max
      const bool ahead = jj + 1 < w;
      unsigned long long mkey = 0ull;
      int mrow = INT_MAX;
      for (int rr = lane; rr < nr; rr += 32) {
        const int gi = rbeg + rr;
        if (gi > j) {
          double a[K], m[K];
#pragma unroll
          for (int c = 0; c < K; ++c) a[c] = at(rr, jj)[c];
          mc::mul<K>(a, rc, m);
#pragma unroll
          for (int c = 0; c < K; ++c) at(rr, jj)[c] = m[c];
          if (ahead) {
            double negm[K], u[K], acc[K];
#pragma unroll
            for (int c = 0; c < K; ++c) {
              negm[c] = -m[c];
              u[c] = prow[(jj + 1) * K + c];
              acc[c] = at(rr, jj + 1)[c];
            }
            mc::madd<K>(acc, negm, u);
#pragma unroll
            for (int c = 0; c < K; ++c) at(rr, jj + 1)[c] = acc[c];
            const unsigned long long kv = mag_key(fabs(acc[0]));
            if (mrow == INT_MAX || kv > mkey) { mkey = kv; mrow = gi; }
          }
        }
      }
      trace(jj, 4);
      trace(jj, 5);
      if (ahead) {
        __syncwarp();
        w0_publish_max(jj + 1, seq + 1, mkey, mrow);
        trace(jj, 6);
      }
      __syncwarp();
      nb_arrive(B_MUL, PANEL_THREADS);
      if (jj + 1 >= w) break;
    }
  } else {
    // ================================================================= H ==
    const int ht = tid - 32;
    unsigned *pr = reinterpret_cast<unsigned *>(prow);
    for (int jj = 0; jj < w; ++jj) {
      const int j = J + jj, par = jj & 1;
      const unsigned seq = seq0 + jj;
      nb_sync(B_WIN, PANEL_THREADS);
      if (S.flag) break;  // singular (W0 has returned) or last column
      const int r = S.winner, gw = S.gw;
      const bool own_r = r >= rbeg && r < rbeg + nr;
      const bool own_j = j >= rbeg && j < rbeg + nr;
      const u64 *wd = ws.row_words + ((int64_t)par * G + gw) * LU_ROW_WORDS;
      for (int e = ht; e < rw; e += H_THREADS) pr[e] = poll(wd + e, seq);
      if (r != j && own_r) {
        const u64 *wj = ws.rowj_words + (int64_t)par * LU_ROW_WORDS;
        unsigned *dst = reinterpret_cast<unsigned *>(at(r - rbeg, 0));
        for (int e = ht; e < rw; e += H_THREADS) dst[e] = poll(wj + e, seq);
      }
      nb_sync(B_H, H_THREADS);
      if (r != j && own_j) {
        double *dst = at(j - rbeg, 0);
        for (int e = ht; e < w * K; e += H_THREADS) dst[e] = prow[e];
      }
      nb_sync(B_H, H_THREADS);
      nb_arrive(B_ROW, PANEL_THREADS);
      nb_sync(B_MUL, PANEL_THREADS);   // multipliers + next candidate known
      if (jj + 1 >= w) break;
      // remaining rank-1 update, columns jj+2 .. w-1 of the rows i > j: a
      // thread keeps one column's pivot-row value and walks a strided set of
      // rows (independent madds, unrolled for ILP)
      const int ncol = w - jj - 2;
      if (ncol > 0) {
        const int ng = H_THREADS / ncol;
        const int cc = jj + 2 + ht % ncol, g0 = ht / ncol;
        const int r_first = max(0, j + 1 - rbeg);
        if (g0 < ng) {
          double u[K];
#pragma unroll
          for (int c = 0; c < K; ++c) u[c] = prow[cc * K + c];
#pragma unroll 4
          for (int rr = r_first + g0; rr < nr; rr += ng) {
            double negm[K], acc[K];
#pragma unroll
            for (int c = 0; c < K; ++c) {
              negm[c] = -at(rr, jj)[c];
              acc[c] = at(rr, cc)[c];
            }
            mc::madd<K>(acc, negm, u);
#pragma unroll
            for (int c = 0; c < K; ++c) at(rr, cc)[c] = acc[c];
          }
        }
      }
      nb_sync(B_H, H_THREADS);
      h_publish_rows(jj + 1, seq + 1, S.cand_row);
      nb_arrive(B_REM, PANEL_THREADS);
    }
  }
  stamp(2);
  if (S.singular) return;  // uniform across the grid: no write-back
  __syncthreads();
  for (int e = tid; e < nr * w; e += PANEL_THREADS) {
    int r = e / w, col = e % w;
#pragma unroll
    for (int c = 0; c < K; ++c)
      A.p[c * A.plane + (int64_t)(rbeg + r) * A.ld + J + col] = at(r, col)[c];
  }
  // Epilogue: CTA 0 composes the panel's row exchanges for the exchange
  // kernel: after the exchanges, row cur[i] holds what row src[i] held
  // before.  Each lane traces one candidate position back through the
  // swaps (J+jj <-> piv[jj], jj descending) -- no serial pass over columns.
  if (g == 0 && tid < 32) {
    const int pv = lane < w ? S.piv[lane] : -1;
    auto origin = [&](int p) {
      int x = p;
#pragma unroll 4
      for (int jj = w - 1; jj >= 0; --jj) {
        const int b = __shfl_sync(0xffffffffu, pv, jj), a = J + jj;
        x = x == a ? b : (x == b ? a : x);
      }
      return x;
    };
    // positions: the panel rows J+lane, and each distinct pivot row below
    const int pa = lane < w ? J + lane : -1;
    int pb = -1;
    if (lane < w && pv >= J + w) {
      bool first = true;
      for (int q = 0; q < lane; ++q)
        if (S.piv[q] == pv) first = false;
      if (first) pb = pv;
    }
    const int sa = origin(pa), sb = origin(pb);
    const bool ka = pa >= 0 && sa != pa, kb = pb >= 0 && sb != pb;
    const unsigned ma = __ballot_sync(0xffffffffu, ka);
    const unsigned mb = __ballot_sync(0xffffffffu, kb);
    const unsigned lt = (1u << lane) - 1u;
    int32_t *sl = ws.swap_list + slot * LU_SWAP_LIST;
    if (ka) {
      const int i = __popc(ma & lt);
      sl[i] = pa;
      sl[2 * LU_MAX_W + i] = sa;
    }
    if (kb) {
      const int i = __popc(ma) + __popc(mb & lt);
      sl[i] = pb;
      sl[2 * LU_MAX_W + i] = sb;
    }
    if (lane == 0) sl[4 * LU_MAX_W] = __popc(ma) + __popc(mb);
  }
  stamp(3);
  if (tid == 0) lu_stamp(J, 1, false);
}
