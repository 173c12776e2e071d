// Distributed LU driver (dist.cu) <-> C-ABI layer (cabi.cu).
#pragma once
#include <string>
#include <vector>

#include "internal.h"

namespace mpk {

// one rank's local storage: n rows x (local columns + 1); the last column
// holds b (replicated) on entry; x (k x n planar, device) receives the
// solution
struct DistRankView {
  int rank = 0;
  MatView A{};
  int cols = 0;
  double *x = nullptr;
};

enum DistPhase {
  DIST_TOTAL = 0,      // whole call, main stream
  DIST_FACTOR,         // tall-block LU + header + pack (side stream)
  DIST_BCAST,          // panel broadcasts (comm stream, incl. waiting)
  DIST_EXCH_TRSM,      // exchanges + U12 (main stream)
  DIST_UPDATE,         // trailing update (main stream)
  DIST_BACK,           // column-cyclic back substitution (main stream)
  DIST_NPHASES
};

int nccl_unique_id(unsigned char *out128, std::string &err);
void *nccl_comm_init(int world, int rank, const unsigned char *id128,
                     std::string &err);
void nccl_comm_destroy(void *comm);

// comm = an nccl_comm_init handle (one served rank) or null (every rank of
// the world served here, on this device).  -> 0, 2 bad arguments,
// 3 singular (*sing_step), 6 CUDA / NCCL failure (err)
int dist_lu_solve(void *comm, int k, int n, int nb, int G,
                  const std::vector<DistRankView> &views, LuWork &ws,
                  SolveWork &sw, cudaStream_t caller,
                  std::vector<int32_t> &swaps_out, int32_t *sing_step,
                  double *phase_ms, int64_t *launches, std::string &err);

}  // namespace mpk
