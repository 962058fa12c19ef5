// Copy-engine two-shot mean (ALGO_CE, the side-stream all-reduce of the overlap
// pipeline with the NVLink traffic off the SMs).  Same result as K3, bit for bit:
// owner q of chunk q (partition_chunks, params.py:130-147) sums the P contributions
// in the ring order of collective.py:154-203 and divides by P; only the transport differs.
//
//   1. k_gate: every rank has entered this launch, so every peer finished its previous
//      one (its staging and mean buffers are free, its compute stream consumed its mean);
//   2. P-1 copies: my snapshot's chunk q -> owner q's staging slot [me] (copy engine);
//   3. k_ce_signal(kind 3): my copies are complete (stream order) -> flag every peer,
//      wait for every peer's flag: my staging holds all contributions;
//   4. k_ce_reduce: ring-order sum of my chunk / P -> my mean buffer (HBM-bound, 1+1/P B);
//   5. P-1 copies: my mean chunk -> every peer's mean buffer at the same offset;
//   6. k_ce_signal(kind 4): flag + wait, then publish done_seq.
// Per rank: 2(P-1)/P B out and in over NVLink (as K3), moved by the copy engines; the
// SMs hold one warp while waiting and one short reduce kernel.
#include "comm_ce.h"

namespace lasgd {

// Rank-level signal + wait on slot kind (3: contributions delivered, 4: means delivered).
// Every copy this rank enqueued before this kernel has completed (stream order); the
// system-scope fence orders them before the flags.
template <int P>
__global__ void __launch_bounds__(32) k_ce_signal(CommArgs a, int kind, int publish) {
  __threadfence_system();
  const size_t slot = (size_t)2 * kMaxB * kMaxR + (size_t)kind * kMaxR;
  const bool skip = (kind == 3 && a.skip_signal_phase == 1) || (kind == 4 && a.skip_signal_phase == 2);
  if (threadIdx.x < P && !skip) st_release_sys(a.pad[threadIdx.x] + slot + a.rank, a.epoch);
  // a failure earlier in this launch (or an injected one) already poisoned the round:
  // do not wait out another timeout
  if (*(volatile uint32_t*)&a.status[ST_ERR] != ERR_NONE) return;
  const bool ok = rank_wait<P>(a, kind, a.epoch, 0, a.rank);
  if (publish && ok && threadIdx.x == 0) {
    __threadfence();
    st_relaxed_sys64(a.done_seq, a.seq);
  }
}

template <int P>
__global__ void __launch_bounds__(32) k_ce_gate(CommArgs a) {
  const size_t slot = (size_t)2 * kMaxB * kMaxR + (size_t)2 * kMaxR;
  if (threadIdx.x < P) st_release_sys(a.pad[threadIdx.x] + slot + a.rank, a.epoch);
  rank_wait<P>(a, 2, a.epoch, 0, a.rank);
}

// Own chunk [cs, cs + len): xbar = (v_r + v_{r+1} + ... + v_{r-1}) / P with v_rank read
// from the local snapshot and v_q from staging slot q; the sources are put in ring order
// once, so every index below is a compile-time constant (registers, no local memory).
template <typename T, int P>
__global__ void __launch_bounds__(256) k_ce_reduce(const T* __restrict__ own, const T* __restrict__ stage,
                                                   size_t stage_elems, T* __restrict__ xbar, size_t len, int rank) {
  constexpr int U = 4;
  const T* src[P];
#pragma unroll
  for (int k = 0; k < P; ++k) {
    const int q = (rank + k) % P;
    src[k] = q == rank ? own : stage + (size_t)q * stage_elems;
  }
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i0 = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i0 + (U - 1) * stride < len; i0 += U * stride) {  // U elements in flight per thread
    T v[U][P];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int k = 0; k < P; ++k) v[u][k] = __ldcs(src[k] + i0 + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      T acc = v[u][0];
#pragma unroll
      for (int k = 1; k < P; ++k) acc = add_rn(acc, v[u][k]);
      __stcs(xbar + i0 + u * stride, mean_div<T, P>(acc));
    }
  }
  for (; i0 < len; i0 += stride) {
    T acc = __ldcs(src[0] + i0);
#pragma unroll
    for (int k = 1; k < P; ++k) acc = add_rn(acc, __ldcs(src[k] + i0));
    __stcs(xbar + i0, mean_div<T, P>(acc));
  }
}

static size_t bound_host(size_t n, int P, int c) {
  const size_t base = n / (size_t)P, rem = n % (size_t)P;
  return (size_t)c * base + ((size_t)c < rem ? (size_t)c : rem);
}

template <typename T, int P>
static int ce_mean(const CommArgs& a, const CeRound& r, cudaStream_t s) {
  const size_t E = sizeof(T), n = a.n;
  const int me = a.rank;
  k_ce_gate<P><<<1, 32, 0, s>>>(a);
  LASGD_CUDA_TRY(cudaGetLastError());
  for (int k = 1; k < P; ++k) {  // rotated: every rank starts at a different owner
    const int q = (me + k) % P;
    const size_t cs = bound_host(n, P, q), ce = bound_host(n, P, q + 1);
    if (ce > cs)
      LASGD_CUDA_TRY(cudaMemcpyAsync(r.stage_peer[q] + (size_t)me * r.stage_elems * E, r.snap_local + cs * E,
                                     (ce - cs) * E, cudaMemcpyDeviceToDevice, s));
  }
  k_ce_signal<P><<<1, 32, 0, s>>>(a, 3, 0);
  LASGD_CUDA_TRY(cudaGetLastError());
  const size_t cs = bound_host(n, P, me), len = bound_host(n, P, me + 1) - cs;
  if (len > 0) {
    // a short HBM-bound pass: 2 CTAs per SM whatever the communicator's SM budget
    // (at 1 GB, P=4: 2.408 ms with 296 CTAs vs 2.480 with 128)
    size_t blocks = (len + 4 * 256 - 1) / (4 * 256);
    const size_t cap = 2 * (size_t)num_sms();
    if (blocks > cap) blocks = cap;
    k_ce_reduce<T, P><<<(unsigned)blocks, 256, 0, s>>>(reinterpret_cast<const T*>(r.snap_local) + cs,
                                                      reinterpret_cast<const T*>(r.stage_local), r.stage_elems,
                                                      reinterpret_cast<T*>(r.xbar_local) + cs, len, me);
    LASGD_CUDA_TRY(cudaGetLastError());
    for (int k = 1; k < P; ++k) {
      const int q = (me + k) % P;
      LASGD_CUDA_TRY(cudaMemcpyAsync(r.xbar_peer[q] + cs * E, r.xbar_local + cs * E, len * E,
                                     cudaMemcpyDeviceToDevice, s));
    }
  }
  k_ce_signal<P><<<1, 32, 0, s>>>(a, 4, 1);
  LASGD_CUDA_TRY(cudaGetLastError());
  return LASGD_OK;
}

template <typename T>
static int ce_mean_t(int P, const CommArgs& a, const CeRound& r, cudaStream_t s) {
  switch (P) {
    case 2: return ce_mean<T, 2>(a, r, s);
    case 3: return ce_mean<T, 3>(a, r, s);
    case 4: return ce_mean<T, 4>(a, r, s);
    case 5: return ce_mean<T, 5>(a, r, s);
    case 6: return ce_mean<T, 6>(a, r, s);
    case 7: return ce_mean<T, 7>(a, r, s);
    case 8: return ce_mean<T, 8>(a, r, s);
    default: return fail(LASGD_ERR_UNSUPPORTED, "the copy-engine mean needs 2 <= P <= %d, got %d", kMaxR, P);
  }
}

template <int P>
__global__ void __launch_bounds__(32) k_rank_barrier(CommArgs a) {
  const size_t slot = (size_t)2 * kMaxB * kMaxR + (size_t)5 * kMaxR;
  if (threadIdx.x < P) st_release_sys(a.pad[threadIdx.x] + slot + a.rank, a.epoch);
  rank_wait<P>(a, 5, a.epoch, 0, a.rank);
}

int launch_rank_barrier(int P, const CommArgs& a, cudaStream_t s) {
  switch (P) {
    case 2: k_rank_barrier<2><<<1, 32, 0, s>>>(a); break;
    case 3: k_rank_barrier<3><<<1, 32, 0, s>>>(a); break;
    case 4: k_rank_barrier<4><<<1, 32, 0, s>>>(a); break;
    case 5: k_rank_barrier<5><<<1, 32, 0, s>>>(a); break;
    case 6: k_rank_barrier<6><<<1, 32, 0, s>>>(a); break;
    case 7: k_rank_barrier<7><<<1, 32, 0, s>>>(a); break;
    case 8: k_rank_barrier<8><<<1, 32, 0, s>>>(a); break;
    default: return fail(LASGD_ERR_UNSUPPORTED, "device barrier needs 2 <= P <= %d, got %d", kMaxR, P);
  }
  LASGD_CUDA_TRY(cudaGetLastError());
  return LASGD_OK;
}

int launch_ce_mean(int dtype, int P, const CommArgs& a, const CeRound& r, cudaStream_t s) {
  return dtype == LASGD_F64 ? ce_mean_t<double>(P, a, r, s) : ce_mean_t<float>(P, a, r, s);
}

}  // namespace lasgd
