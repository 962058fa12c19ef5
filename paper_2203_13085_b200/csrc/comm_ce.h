// Copy-engine two-shot mean (ALGO_CE): the data moves through the GPUs' copy engines
// (cudaMemcpyAsync over the IPC-mapped peer regions) and the SMs only reduce the own
// chunk and flip flags (comm_ce.cu).
#ifndef LASGD_COMM_CE_H
#define LASGD_COMM_CE_H

#include "comm_launch.cuh"

namespace lasgd {

// This rank's and its peers' buffers for one CE mean.  stage_peer[q]: owner q's staging
// region (parity 0, [source rank][stage_elems]); xbar_peer[q]: q's mean buffer.
struct CeRound {
  const char* snap_local;
  char* xbar_local;
  const char* stage_local;
  char* stage_peer[kMaxR];
  char* xbar_peer[kMaxR];
  size_t stage_elems;
};

int launch_ce_mean(int dtype, int P, const CommArgs& a, const CeRound& r, cudaStream_t s);
// One-warp device barrier on rank-level slot kind 5 (epoch = a.epoch): lasgd_comm_barrier.
int launch_rank_barrier(int P, const CommArgs& a, cudaStream_t s);

}  // namespace lasgd

#endif  // LASGD_COMM_CE_H
