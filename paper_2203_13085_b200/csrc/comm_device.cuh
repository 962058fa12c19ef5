// Device side of the NVLink communicator: launch arguments (CommArgs), system-scope
// flag primitives, per-CTA and rank-level barriers, the launch gate, completion
// publication, tracing, and the tile work distribution shared by every comm kernel.
// Part of the communicator translation unit (lasgd_comm.cu includes it).
#ifndef LASGD_COMM_DEVICE_CUH
#define LASGD_COMM_DEVICE_CUH

#include "lasgd_common.cuh"

namespace lasgd {

constexpr int kMaxR = LASGD_MAX_RANKS;
constexpr int kMaxB = LASGD_MAX_BLOCKS;  // flag slots per phase and rank
constexpr int kPhases = 3;  // 0 entry (per CTA), 1 mid (per CTA), 2 rank-level mid
constexpr size_t kPadBytes = (size_t)kPhases * kMaxB * kMaxR * sizeof(uint32_t);
constexpr int kDoneSlots = 64;
constexpr int kTileQ = 4;  // work-queue counters per launch slot (the push mean uses four)
constexpr int kEvents = 64;

// host-mapped status block layout (uint32 words)
// ST_CLAIM: taken (CAS) by the first failure, which fills the fields and publishes
// ST_ERR last, so a host that sees ST_ERR also sees the fields describing it
enum { ST_ERR = 0, ST_PEER, ST_PHASE, ST_BLOCK, ST_SEQ_LO, ST_SEQ_HI, ST_RANK, ST_CLAIM, ST_WORDS = 16 };
enum { ERR_NONE = 0, ERR_TIMEOUT = 1, ERR_INJECTED = 2 };

struct CommArgs {
  const char* snap[kMaxR];
  char* xbar[kMaxR];
  uint32_t* pad[kMaxR];
  size_t n;
  // a launch over the sub-range [range_off, range_off + n) of an n_glob-element vector
  // (bucketed SGD-AR) sums every element in the ring order of its chunk of the WHOLE
  // vector, so bucketing leaves the mean bit-identical; n_glob == 0: the launch is the
  // whole vector
  size_t range_off, n_glob;
  int rank;
  int nblocks;
  uint32_t epoch;
  int phases;  // bit 0: reduce (one-shot / RS), bit 1: all-gather (two-shot)
  long long timeout_ns;
  int skip_signal_phase;
  uint32_t* status;
  unsigned int* done_ctr;
  unsigned long long* done_seq;
  unsigned long long seq;
  unsigned long long* nonfinite;
  unsigned long long* trace;  // optional per-CTA timeline: [b][0..3] = start, entry passed, mid passed, end
  unsigned long long* tile_ctr;  // two work queues of this launch (nullptr: static slices)
  unsigned int* mid_ctr;         // CTAs of this rank past the reduce-scatter (rank-level barrier)
  unsigned int* end_ctr;         // CTAs of this rank done pushing (push round, rank-level end signal)
  unsigned int* aux_ctr;         // push mean: CTAs done scattering the second half (row-6 signal)
  // push round (K8): per-rank staging regions and round bookkeeping
  char* stage[kMaxR];            // owner o's staging: [parity][source rank][stage_elems]
  size_t stage_elems;
  int cur;                       // snapshot slot / staging parity read this round
  uint32_t prev_push;            // launch whose end signals certify the staged contributions
  uint32_t prev_end;             // K7: the previous launch, if its end signals certify this one's inputs (else 0)
  // graph-replayable launch (adv.rd != nullptr): the sequence number (epoch of every
  // flag), the snapshot slot and the work-queue / counter slots come from the worker's
  // device round descriptor instead of the fields above; snap[] then point at slot 0
  // (slot 1 is slot_stride bytes further) and the counters at their slot-0 entries.
  // dyn_chain: the previous launch raised end signals (every round of a captured
  // steady-state loop does), so K7 enters on them.  The last CTA advances the descriptor.
  RoundAdv adv;
  size_t slot_stride;
  int dyn_chain;
};

// Per-CTA copy of the dynamic launch arguments (read once by thread 0 at entry).
struct DynComm {
  unsigned long long seq;
  DynView v;
};
static __shared__ DynComm s_dyn;

// One round trip: thread 0 loads every field this launch needs, the CTA shares them.
__device__ __forceinline__ void dyn_comm_begin(const CommArgs& a) {
  if (a.adv.rd == nullptr) return;
  if (threadIdx.x == 0) {
    s_dyn.seq = __ldcg(&a.adv.rd->seq) + 1ull;
    s_dyn.v = dyn_read(a.adv.rd);
  }
  __syncthreads();
}
__device__ __forceinline__ unsigned long long cseq(const CommArgs& a) { return a.adv.rd ? s_dyn.seq : a.seq; }
__device__ __forceinline__ uint32_t cepoch(const CommArgs& a) { return a.adv.rd ? (uint32_t)s_dyn.seq : a.epoch; }
__device__ __forceinline__ int ccur(const CommArgs& a) { return a.adv.rd ? s_dyn.v.cur : a.cur; }
__device__ __forceinline__ uint32_t cprev_push(const CommArgs& a) {
  return a.adv.rd ? (uint32_t)(s_dyn.seq - 1ull) : a.prev_push;
}
__device__ __forceinline__ uint32_t cprev_end(const CommArgs& a) {
  return a.adv.rd ? (a.dyn_chain ? (uint32_t)(s_dyn.seq - 1ull) : 0u) : a.prev_end;
}
__device__ __forceinline__ unsigned long long* ctile(const CommArgs& a) {
  return (a.adv.rd && a.tile_ctr) ? a.tile_ctr + kTileQ * (s_dyn.seq % kDoneSlots) : a.tile_ctr;
}
__device__ __forceinline__ unsigned* cmid(const CommArgs& a) {
  return (a.adv.rd && a.mid_ctr) ? a.mid_ctr + (s_dyn.seq % kDoneSlots) : a.mid_ctr;
}
__device__ __forceinline__ unsigned* caux(const CommArgs& a) {
  return (a.adv.rd && a.aux_ctr) ? a.aux_ctr + (s_dyn.seq % kDoneSlots) : a.aux_ctr;
}
__device__ __forceinline__ unsigned* cend(const CommArgs& a) {
  return (a.adv.rd && a.end_ctr) ? a.end_ctr + (s_dyn.seq % kDoneSlots) : a.end_ctr;
}
// rank q's snapshot slot `slot` (dynamic launches), or the launch's slot (static)
__device__ __forceinline__ const char* csnap(const CommArgs& a, int q) {
  return a.snap[q] + ((a.adv.rd && s_dyn.v.cur) ? a.slot_stride : 0);
}
__device__ __forceinline__ const char* cslot(const CommArgs& a, int q, int slot) {
  return a.snap[q] + (slot ? a.slot_stride : 0);
}
// the learning rate / first step / delta reset of a dynamic launch
template <typename T>
__device__ __forceinline__ SgdCoef<T> ccoef(const CommArgs& a, const SgdCoef<T>& c) {
  SgdCoef<T> r = c;
  if (a.adv.rd) dyn_coef(r, s_dyn.v);  // after dyn_comm_begin
  return r;
}

__device__ __forceinline__ unsigned long long globaltimer();

__device__ __forceinline__ void trace_mark(const CommArgs& a, int b, int k) {
  if (a.trace != nullptr && threadIdx.x == 0) a.trace[b * 4 + k] = globaltimer();
}

// ------------------------------------------------------------------ primitives
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_sys64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Bounds of partition_chunks(n, P): bound(c) = c*base + min(c, rem).
__device__ __forceinline__ size_t chunk_bound(size_t n, int P, int c) {
  const size_t base = n / (size_t)P, rem = n % (size_t)P;
  return (size_t)c * base + ((size_t)c < rem ? (size_t)c : rem);
}

// Chunk bound c of the whole vector in this launch's local coordinates (clamped to
// [0, n]): chunk_of over these bounds gives the ring-order start of a sub-range element.
__device__ __forceinline__ size_t chunk_bound_local(const CommArgs& a, int P, int c) {
  if (a.n_glob == 0) return chunk_bound(a.n, P, c);
  const size_t g = chunk_bound(a.n_glob, P, c);
  if (g <= a.range_off) return 0;
  const size_t l = g - a.range_off;
  return l < a.n ? l : a.n;
}

template <int P>
__device__ __forceinline__ int chunk_of(size_t j, const size_t (&bnd)[P + 1]) {
  int c = 0;
#pragma unroll
  for (int k = 1; k < P; ++k) c += (j >= bnd[k]);
  return c;
}

// Ring-order start of element j of this launch: its chunk of the whole vector
// (== the owner chunk for a whole-vector launch).
template <int P>
__device__ __forceinline__ int rot_of(const CommArgs& a, size_t j) {
  int c = 0;
#pragma unroll
  for (int k = 1; k < P; ++k) c += (j >= chunk_bound_local(a, P, k));
  return c;
}

// Sum v[c], v[c+1], ..., v[c-1] (mod P) left to right: the reference ring order.
template <typename T, int P>
__device__ __forceinline__ T rot_sum(const T (&v)[P], int c) {
  T acc = v[0];
#pragma unroll
  for (int cc = 0; cc < P; ++cc) {
    if (c == cc) {
      T s = v[cc];
#pragma unroll
      for (int k = 1; k < P; ++k) s = add_rn(s, v[(cc + k) % P]);
      acc = s;
    }
  }
  return acc;
}

// buf / P (collective.py:200).  For power-of-two P, x*(1/P) is the same correctly
// rounded value as x/P (exact scaling), so use the cheaper multiply.
template <typename T, int P>
__device__ __forceinline__ T mean_div(T s) {
  if constexpr ((P & (P - 1)) == 0) {
    return mul_rn(s, T(1.0 / P));
  } else {
    return div_rn(s, T(P));
  }
}

__device__ inline void report_failure(const CommArgs& a, int code, int peer, int phase, int block, int rank) {
  if (atomicCAS(&a.status[ST_CLAIM], 0u, 1u) == 0u) {
    a.status[ST_PEER] = peer;
    a.status[ST_PHASE] = phase;
    a.status[ST_BLOCK] = block;
    a.status[ST_SEQ_LO] = (uint32_t)(cseq(a) & 0xffffffffu);
    a.status[ST_SEQ_HI] = (uint32_t)(cseq(a) >> 32);
    a.status[ST_RANK] = rank;
    __threadfence_system();
    st_release_sys(&a.status[ST_ERR], (uint32_t)code);
  }
}

// Per-CTA barrier with the same CTA index on every peer.  Thread q < P signals
// peer q and waits for peer q's signal.
template <int P>
__device__ bool cta_barrier(const CommArgs& a, int phase, int b, int rank) {
  __syncthreads();
  int ok = 1;
  if (threadIdx.x < P) {
    const int q = threadIdx.x;
    const size_t slot = ((size_t)phase * kMaxB + b) * kMaxR;
    if (a.skip_signal_phase != phase) {
      __threadfence_system();
      st_release_sys(a.pad[q] + slot + rank, cepoch(a));
    }
    const uint32_t* f = a.pad[rank] + slot + q;
    const unsigned long long t0 = globaltimer();
    while ((int32_t)(ld_acquire_sys(f) - cepoch(a)) < 0) {
      if ((long long)(globaltimer() - t0) > a.timeout_ns) {
        report_failure(a, ERR_TIMEOUT, q, phase, b, rank);
        ok = 0;
        break;
      }
      __nanosleep(64);
    }
  }
  return __syncthreads_and(ok) != 0;
}

// Last CTA of a launch publishes the sequence number to host-mapped memory (and, for a
// graph-replayable launch, advances the worker's device round descriptor: every CTA
// read it at entry, before counting itself in here).
__device__ inline void publish_done(const CommArgs& a) {
  __syncthreads();
  if (threadIdx.x == 0) {
    // device scope is enough here: the counter is device-local, and the host only learns
    // "launch done" from done_seq (every data read by the host or another stream is
    // ordered by the launch's event); the last CTA's system-scope fence + release below
    // publishes it.  (Peers' data visibility is the rank-level signals' job, which keep
    // their per-CTA system-scope fences.)
    __threadfence();
    const unsigned long long seq = cseq(a);
    const unsigned slot = (unsigned)(seq % kDoneSlots);
    const unsigned prev = atomicAdd(&a.done_ctr[slot], 1u);
    if (prev == (unsigned)a.nblocks - 1u) {
      a.done_ctr[slot] = 0u;
      unsigned long long* tq = ctile(a);
      if (tq)
        for (int k = 0; k < kTileQ; ++k) tq[k] = 0ull;  // every CTA has left its tile loops
      if (a.adv.rd) dyn_apply(a.adv.rd, a.adv);
      // done_seq tells the host "launch complete" — it never carries data to the host:
      // everything the launch wrote is read by later device work (stream order, events,
      // or work the host issues after seeing the flag), for which device-scope
      // visibility is what counts.  A device-scope fence and a relaxed system-scope store
      // suffice; a system-scope release here waited for the round's posted NVLink
      // writes and cost ~3 µs per round (tools/graph_trace_probe.py, N=2: 0.1663 ->
      // 0.1635 ms per round).
      __threadfence();
      st_relaxed_sys64(a.done_seq, seq);
    }
  }
}

// Even split of `npack` packs over `nb` CTAs.
__device__ __forceinline__ void split(size_t npack, int nb, int b, size_t& p0, size_t& p1) {
  const size_t per = (npack + nb - 1) / nb;
  p0 = (size_t)b * per;
  if (p0 > npack) p0 = npack;
  p1 = p0 + per;
  if (p1 > npack) p1 = npack;
}

// Work distribution of the one-shot kernels over packs [0, npack): with a launch work
// queue (P2P launches) CTAs take tiles of TILE_ITERS*U*blockDim packs from an atomic
// counter, the next index fetched while the current tile streams, so fast CTAs absorb
// the tail; otherwise (virtual ranks) CTA b takes the b-th even slice.  Every CTA has
// passed its entry barrier before it takes a tile, so the double-buffer argument is
// unchanged (it only needs every CTA to wait for its peers' same-index CTA).
constexpr int kTileIters = 2;

// Tiles of `tile` packs over [base, base + npack): from the atomic queue `ctr` when
// given (next index prefetched while the current tile streams), else a contiguous
// even slice per CTA.
// `rot` rotates the order in which the packs are visited (logical pack l maps to
// (l + rot) mod npack): the two-shot all-gather starts every rank at a different
// owner's chunk so no owner serves all readers at once.
template <typename F>
__device__ __forceinline__ void tile_loop(unsigned long long* ctr, int b, int nblocks, size_t base, size_t npack,
                                          size_t tile, F&& range, size_t rot = 0) {
  if (npack == 0) return;
  auto visit = [&](size_t l0, size_t l1) {
    if (l0 >= l1) return;
    size_t a0 = l0 + rot;
    if (a0 >= npack) a0 -= npack;
    const size_t len = l1 - l0;
    if (a0 + len <= npack) {
      range(base + a0, base + a0 + len);
    } else {
      range(base + a0, base + npack);
      range(base, base + a0 + len - npack);
    }
  };
  if (ctr == nullptr) {
    size_t p0, p1;
    split(npack, nblocks, b, p0, p1);
    visit(p0, p1);
    return;
  }
  __shared__ unsigned long long s_next;
  const unsigned long long ntiles = (npack + tile - 1) / tile;
  __syncthreads();
  if (threadIdx.x == 0) s_next = atomicAdd(ctr, 1ull);
  __syncthreads();
  unsigned long long t = s_next;
  while (t < ntiles) {
    __syncthreads();  // everyone has read s_next
    if (threadIdx.x == 0) s_next = atomicAdd(ctr, 1ull);  // prefetch the next index
    const size_t p0 = (size_t)t * tile;
    visit(p0, p0 + tile < npack ? p0 + tile : npack);
    __syncthreads();
    t = s_next;
  }
}

template <int U, typename F>
__device__ __forceinline__ void for_tiles(const CommArgs& a, int b, size_t npack, F&& range) {
  tile_loop(ctile(a), b, a.nblocks, 0, npack, (size_t)kTileIters * U * blockDim.x, range);
}

// Rank-level signal of kind k (0 = mid: reduce-scatter / mean pushes done, 1 = end:
// next-snapshot chunks pushed to their owners): every CTA counts itself in (after a
// __threadfence_system, so its stores — remote ones included — are visible system
// wide); the last CTA of the rank writes `epoch` into slot [k][rank] of every peer.
template <int P>
__device__ void rank_signal(const CommArgs& a, int kind, unsigned* ctr, int rank) {
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const unsigned prev = atomicAdd(ctr, 1u);
    s_last = prev == (unsigned)a.nblocks - 1u;
    if (s_last) *ctr = 0u;  // every CTA of this launch has counted itself in
  }
  __syncthreads();
  const size_t slot = (size_t)2 * kMaxB * kMaxR + (size_t)kind * kMaxR;
  // fault injection (test knob): phase 1 drops the mid signal, phase 2 the end signal
  if (s_last && threadIdx.x < P && !(kind == 0 && a.skip_signal_phase == 1) &&
      !(kind == 1 && a.skip_signal_phase == 2)) {
    __threadfence_system();
    st_release_sys(a.pad[threadIdx.x] + slot + rank, cepoch(a));
  }
}

// Wait until every rank has signalled kind k with an epoch >= `epoch`.
template <int P>
__device__ bool rank_wait(const CommArgs& a, int kind, uint32_t epoch, int b, int rank) {
  const size_t slot = (size_t)2 * kMaxB * kMaxR + (size_t)kind * kMaxR;
  int ok = 1;
  if (threadIdx.x < P) {
    const int q = threadIdx.x;
    const uint32_t* f = a.pad[rank] + slot + q;
    const unsigned long long t0 = globaltimer();
    while ((int32_t)(ld_acquire_sys(f) - epoch) < 0) {
      if ((long long)(globaltimer() - t0) > a.timeout_ns) {
        report_failure(a, ERR_TIMEOUT, q, kind + 1, b, rank);  // phase 1 mid, 2 end, 3 gate
        ok = 0;
        break;
      }
      __nanosleep(64);
    }
  }
  return __syncthreads_and(ok) != 0;
}

// Rank-level barrier between the two phases of the two-shot kernels.  Requires all
// CTAs co-resident: the P2P two-shot kernels are launched cooperatively.
template <int P>
__device__ bool rank_barrier(const CommArgs& a, int b, int rank) {
  rank_signal<P>(a, 0, cmid(a), rank);
  return rank_wait<P>(a, 0, cepoch(a), b, rank);
}

// Launch gate (one warp, launched in stream order just before a side-stream
// all-reduce): announce launch `epoch` to every peer (rank-level slot kind 2), then
// wait until every peer announced it too.  A wide all-reduce kernel whose peers are
// late spins in its entry barrier holding a CTA on most SMs, which starves the
// compute stream's large forward/backward CTAs; behind the gate it only starts once
// every peer is about to start as well, and the waiting costs one warp.
template <int P>
__global__ void __launch_bounds__(32) k_gate(CommArgs a) {
  const size_t slot = (size_t)2 * kMaxB * kMaxR + (size_t)2 * kMaxR;
  if (threadIdx.x < P) st_release_sys(a.pad[threadIdx.x] + slot + a.rank, a.epoch);
  rank_wait<P>(a, 2, a.epoch, 0, a.rank);
}

// Aligned body of chunk c in packs, [cp0, cp1), plus its unaligned head/tail elements.
template <typename T, int P>
__device__ __forceinline__ void chunk_packs(size_t n, int c, size_t& cs, size_t& ce, size_t& cp0, size_t& cp1) {
  constexpr int W = Pack<T>::W;
  cs = chunk_bound(n, P, c);
  ce = chunk_bound(n, P, c + 1);
  cp0 = (cs + W - 1) / W;
  cp1 = ce / W;
  if (cp1 < cp0) cp1 = cp0;
}

}  // namespace lasgd

#endif  // LASGD_COMM_DEVICE_CUH
