// Mean all-reduce of the LASGD snapshot over NVLink P2P (K2 one-shot, K3 two-shot)
// with epoch-tagged per-CTA flags in IPC-mapped signal pads (K6) and a
// host-mapped completion word for flag polling.
//
// Replaces collective.py:154-203 (`execute_allreduce`) and the
// LoopbackTransport round (collective.py:229-287).  The arithmetic reproduces the
// reference ring's per-chunk summation order bit for bit: element j of chunk c
// (partition_chunks(n, P), params.py:130-147) is summed x_c, x_{c+1}, ..., x_{c-1}
// (mod P) and the sum is divided by P once (collective.py:200).  Every rank
// therefore ends with identical bits, like the reference's per_rank copies.
//
// One-shot: every rank reads all P snapshots (P-1 over NVLink) and reduces every
// element itself.   NVLink in-bytes per rank: (P-1)*B.
// Two-shot: rank c reduces chunk c (reduce-scatter, same order), then copies the
// other ranks' reduced chunks (all-gather).  NVLink in-bytes: 2(P-1)/P*B — the
// reference's bytes_per_node (collective.py:206-226).
//
// Synchronisation is per CTA: CTA b of every rank slices the data identically, so
// CTA b only ever waits for CTA b of its peers (no grid-wide barrier).  The entry
// barrier publishes "my snapshot slot is final"; the two-shot mid barrier publishes
// "my reduced chunk slice is final" and, implicitly, "I have finished reading your
// snapshot slice".  Snapshot slots are double-buffered by round parity by the
// caller, so the next round's writes never race a peer's reads (a peer can only
// enter round r+1 after finishing round r, and our round r+1 launch completes only
// after every peer entered it).  A %globaltimer watchdog turns a dead peer into a
// CollectiveFailure instead of a hung GPU.
#include <stdarg.h>
#include <string.h>
#include <time.h>

#include <map>
#include <mutex>
#include <utility>

#include "lasgd_common.cuh"

namespace lasgd {

constexpr int kMaxR = LASGD_MAX_RANKS;
constexpr int kMaxB = LASGD_MAX_BLOCKS;  // flag slots per phase and rank
constexpr int kPhases = 3;  // 0 entry (per CTA), 1 mid (per CTA), 2 rank-level mid
constexpr size_t kPadBytes = (size_t)kPhases * kMaxB * kMaxR * sizeof(uint32_t);
constexpr int kDoneSlots = 64;
constexpr int kEvents = 64;

// host-mapped status block layout (uint32 words)
enum { ST_ERR = 0, ST_PEER, ST_PHASE, ST_BLOCK, ST_SEQ_LO, ST_SEQ_HI, ST_RANK, ST_WORDS = 16 };
enum { ERR_NONE = 0, ERR_TIMEOUT = 1, ERR_INJECTED = 2 };

struct CommArgs {
  const char* snap[kMaxR];
  char* xbar[kMaxR];
  uint32_t* pad[kMaxR];
  size_t n;
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
  // push round (K8): per-rank staging regions and round bookkeeping
  char* stage[kMaxR];            // owner o's staging: [parity][source rank][stage_elems]
  size_t stage_elems;
  int cur;                       // snapshot slot / staging parity read this round
  uint32_t prev_push;            // launch whose end signals certify the staged contributions
  uint32_t prev_end;             // K7: the previous launch, if its end signals certify this one's inputs (else 0)
};

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

template <int P>
__device__ __forceinline__ int chunk_of(size_t j, const size_t (&bnd)[P + 1]) {
  int c = 0;
#pragma unroll
  for (int k = 1; k < P; ++k) c += (j >= bnd[k]);
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

__device__ void report_failure(const CommArgs& a, int code, int peer, int phase, int block, int rank) {
  if (atomicCAS(&a.status[ST_ERR], 0u, (uint32_t)code) == 0u) {
    a.status[ST_PEER] = peer;
    a.status[ST_PHASE] = phase;
    a.status[ST_BLOCK] = block;
    a.status[ST_SEQ_LO] = (uint32_t)(a.seq & 0xffffffffu);
    a.status[ST_SEQ_HI] = (uint32_t)(a.seq >> 32);
    a.status[ST_RANK] = rank;
    __threadfence_system();
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
      st_release_sys(a.pad[q] + slot + rank, a.epoch);
    }
    const uint32_t* f = a.pad[rank] + slot + q;
    const unsigned long long t0 = globaltimer();
    while ((int32_t)(ld_acquire_sys(f) - a.epoch) < 0) {
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

// Last CTA of a launch publishes the sequence number to host-mapped memory.
__device__ void publish_done(const CommArgs& a) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const unsigned slot = (unsigned)(a.seq % kDoneSlots);
    const unsigned prev = atomicAdd(&a.done_ctr[slot], 1u);
    if (prev == (unsigned)a.nblocks - 1u) {
      a.done_ctr[slot] = 0u;
      if (a.tile_ctr) a.tile_ctr[0] = a.tile_ctr[1] = 0ull;  // every CTA has left its tile loops
      __threadfence_system();
      st_release_sys64(a.done_seq, a.seq);
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
  tile_loop(a.tile_ctr, b, a.nblocks, 0, npack, (size_t)kTileIters * U * blockDim.x, range);
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
  if (s_last && threadIdx.x < P && !(kind == 0 && a.skip_signal_phase == 1)) {
    __threadfence_system();
    st_release_sys(a.pad[threadIdx.x] + slot + rank, a.epoch);
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
        report_failure(a, ERR_TIMEOUT, q, 1, b, rank);
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
  rank_signal<P>(a, 0, a.mid_ctr, rank);
  return rank_wait<P>(a, 0, a.epoch, b, rank);
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

// ------------------------------------------------------------------ one-shot (K2)
template <typename T, int P, bool VIRTUAL, int U>
__global__ void __launch_bounds__(256, 2) k_oneshot(CommArgs a) {
  constexpr int W = Pack<T>::W;
  const int rank = VIRTUAL ? (int)blockIdx.y : a.rank;
  const int b = blockIdx.x;
  bool ok = true;
  trace_mark(a, b, 0);
  if (!VIRTUAL) ok = cta_barrier<P>(a, 0, b, rank);
  trace_mark(a, b, 1);
  unsigned bad = 0;
  if (ok) {
    const size_t n = a.n;
    size_t bnd[P + 1];
#pragma unroll
    for (int c = 0; c <= P; ++c) bnd[c] = chunk_bound(n, P, c);
    const T* src[P];
#pragma unroll
    for (int q = 0; q < P; ++q) src[q] = reinterpret_cast<const T*>(a.snap[q]);
    T* out = reinterpret_cast<T*>(a.xbar[rank]);
    auto range = [&](size_t p0, size_t p1) {
    for (size_t p = p0 + threadIdx.x; p < p1; p += (size_t)U * blockDim.x) {
      Pack<T> v[U][P];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const size_t pu = p + (size_t)u * blockDim.x;
        if (pu < p1) {
#pragma unroll
          for (int q = 0; q < P; ++q) v[u][q] = ld_cg(src[q] + pu * W);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const size_t pu = p + (size_t)u * blockDim.x;
        if (pu < p1) {
          const size_t j0 = pu * W;
          const int c0 = chunk_of<P>(j0, bnd), c1 = chunk_of<P>(j0 + W - 1, bnd);
          Pack<T> o;
#pragma unroll
          for (int k = 0; k < W; ++k) {
            T lane[P];
#pragma unroll
            for (int q = 0; q < P; ++q) lane[q] = v[u][q].v[k];
            const int c = (c0 == c1) ? c0 : chunk_of<P>(j0 + k, bnd);
            o.v[k] = mean_div<T, P>(rot_sum<T, P>(lane, c));
            bad += !finite(o.v[k]);
          }
          st_stream(out + j0, o);
        }
      }
    }
    };
    for_tiles<U>(a, b, n / W, range);
    if (b == a.nblocks - 1) {  // scalar tail n % W
      for (size_t j = (n / W) * W + threadIdx.x; j < n; j += blockDim.x) {
        T lane[P];
#pragma unroll
        for (int q = 0; q < P; ++q) lane[q] = src[q][j];
        T r = mean_div<T, P>(rot_sum<T, P>(lane, chunk_of<P>(j, bnd)));
        out[j] = r;
        bad += !finite(r);
      }
    }
  }
  report_nonfinite(a.nonfinite, bad);
  trace_mark(a, b, 3);
  if (!VIRTUAL) publish_done(a);
}

// ------------------------------------------------------------------ two-shot (K3)
template <typename T, int P>
__device__ __forceinline__ T ordered_sum(const T* const (&src)[P], int rank, size_t j) {
  T v[P];
#pragma unroll
  for (int q = 0; q < P; ++q) v[q] = src[q][j];
  return rot_sum<T, P>(v, rank);
}

// Visit tiles 0..ntiles-1 from the atomic queue `ctr` (next index prefetched), or
// statically strided over the CTAs when there is no queue (virtual ranks).
template <typename V>
__device__ __forceinline__ void queue_loop(unsigned long long* ctr, int b, int nblocks, unsigned long long ntiles,
                                           V&& visit) {
  if (ctr == nullptr) {
    for (unsigned long long t = b; t < ntiles; t += nblocks) visit(t);
    return;
  }
  __shared__ unsigned long long s_next;
  __syncthreads();
  if (threadIdx.x == 0) s_next = atomicAdd(ctr, 1ull);
  __syncthreads();
  unsigned long long t = s_next;
  while (t < ntiles) {
    __syncthreads();
    if (threadIdx.x == 0) s_next = atomicAdd(ctr, 1ull);
    visit(t);
    __syncthreads();
    t = s_next;
  }
}

// Phase-2 work of the two-shot kernels: the aligned body of every chunk c (minus the
// own chunk when skip_own) in tiles interleaved across chunks and rotated per rank —
// tile t is the (t / P)-th tile of chunk (rank + 1 + t) % P — so at any moment the
// CTAs are spread over every owner (NVLink) and over the own chunk (HBM only), and
// no owner serves all readers at once.  CTA 0 then does the unaligned head/tail
// elements of every chunk (at most 2W-2 per chunk boundary).
template <typename T, int P, typename FB, typename FS>
__device__ __forceinline__ void chunk_tiles(unsigned long long* ctr, int b, int nblocks, size_t n, int rank,
                                            bool skip_own, size_t tile, FB&& body, FS&& scalar) {
  constexpr int W = Pack<T>::W;
  size_t tmax = 0;
#pragma unroll
  for (int c = 0; c < P; ++c) {
    size_t cs, ce, cp0, cp1;
    chunk_packs<T, P>(n, c, cs, ce, cp0, cp1);
    const size_t tc = (cp1 - cp0 + tile - 1) / tile;
    tmax = tc > tmax ? tc : tmax;
  }
  queue_loop(ctr, b, nblocks, (unsigned long long)tmax * P, [&](unsigned long long t) {
    const int c = (rank + 1 + (int)(t % P)) % P;
    if (skip_own && c == rank) return;
    size_t cs, ce, cp0, cp1;
    chunk_packs<T, P>(n, c, cs, ce, cp0, cp1);
    const size_t a0 = cp0 + (size_t)(t / P) * tile;
    if (a0 >= cp1) return;
    body(c, a0, a0 + tile < cp1 ? a0 + tile : cp1);
  });
  if (b == 0) {
    for (int c = 0; c < P; ++c) {
      if (skip_own && c == rank) continue;
      size_t cs, ce, cp0, cp1;
      chunk_packs<T, P>(n, c, cs, ce, cp0, cp1);
      const size_t he = cp0 * W < ce ? cp0 * W : ce;
      const size_t ts = cp1 * W > he ? cp1 * W : he;
      for (size_t j = cs + threadIdx.x; j < he; j += blockDim.x) scalar(c, j);
      for (size_t j = ts + threadIdx.x; j < ce; j += blockDim.x) scalar(c, j);
    }
  }
}

// Reduce-scatter of this rank's chunk (ring order x_rank, x_rank+1, ..., x_rank-1)
// into its xbar buffer: aligned packs from work queue 0, head/tail elements on CTA 0.
template <typename T, int P, int U>
__device__ __forceinline__ unsigned reduce_own_chunk(const CommArgs& a, int b, int rank, unsigned long long* q0) {
  constexpr int W = Pack<T>::W;
  const size_t n = a.n;
  unsigned bad = 0;
  T* own = reinterpret_cast<T*>(a.xbar[rank]);
  const T* src[P];
#pragma unroll
  for (int q = 0; q < P; ++q) src[q] = reinterpret_cast<const T*>(a.snap[q]);
  size_t cs, ce, cp0, cp1;
  chunk_packs<T, P>(n, rank, cs, ce, cp0, cp1);
  auto range = [&](size_t p0, size_t p1) {
    for (size_t p = p0 + threadIdx.x; p < p1; p += (size_t)U * blockDim.x) {
      Pack<T> v[U][P];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const size_t pu = p + (size_t)u * blockDim.x;
        if (pu < p1) {
#pragma unroll
          for (int q = 0; q < P; ++q) v[u][q] = ld_cg(src[q] + pu * W);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const size_t pu = p + (size_t)u * blockDim.x;
        if (pu < p1) {
          Pack<T> o;
#pragma unroll
          for (int k = 0; k < W; ++k) {
            T lane[P];
#pragma unroll
            for (int q = 0; q < P; ++q) lane[q] = v[u][q].v[k];
            o.v[k] = mean_div<T, P>(rot_sum<T, P>(lane, rank));
            bad += !finite(o.v[k]);
          }
          st_plain(own + pu * W, o);
        }
      }
    }
  };
  tile_loop(q0, b, a.nblocks, cp0, cp1 - cp0, (size_t)kTileIters * U * blockDim.x, range);
  if (b == 0) {  // unaligned head / tail of the chunk (and tiny chunks)
    const size_t hs = cs, he = cp0 * W < ce ? cp0 * W : ce;
    const size_t ts = cp1 * W > hs ? (cp1 * W > he ? cp1 * W : he) : he;
    for (size_t j = hs + threadIdx.x; j < he; j += blockDim.x) {
      T r = mean_div<T, P>(ordered_sum<T, P>(src, rank, j));
      own[j] = r;
      bad += !finite(r);
    }
    for (size_t j = ts + threadIdx.x; j < ce; j += blockDim.x) {
      T r = mean_div<T, P>(ordered_sum<T, P>(src, rank, j));
      own[j] = r;
      bad += !finite(r);
    }
  }
  return bad;
}

template <typename T, int P, bool VIRTUAL, int U, int UAG>
__global__ void __launch_bounds__(256, 2) k_twoshot(CommArgs a) {
  constexpr int W = Pack<T>::W;
  const int rank = VIRTUAL ? (int)blockIdx.y : a.rank;
  const int b = blockIdx.x;
  const size_t n = a.n;
  bool ok = true;
  unsigned bad = 0;
  T* out = reinterpret_cast<T*>(a.xbar[rank]);
  unsigned long long* q0 = a.tile_ctr ? a.tile_ctr : nullptr;
  unsigned long long* q1 = a.tile_ctr ? a.tile_ctr + 1 : nullptr;
  trace_mark(a, b, 0);
  if (a.phases & 1) {
    if (!VIRTUAL) ok = cta_barrier<P>(a, 0, b, rank);
    trace_mark(a, b, 1);
    if (ok) bad += reduce_own_chunk<T, P, U>(a, b, rank, q0);
  }
  if (a.phases & 2) {
    if (!VIRTUAL && ok) ok = rank_barrier<P>(a, b, rank);
    trace_mark(a, b, 2);
    if (ok) {
      // all-gather: every pack outside the own chunk comes from its owner's xbar
      chunk_tiles<T, P>(q1, b, a.nblocks, n, rank, true, (size_t)kTileIters * UAG * blockDim.x,
        [&](int c, size_t p0, size_t p1) {
          const T* zc = reinterpret_cast<const T*>(a.xbar[c]);
          for (size_t p = p0 + threadIdx.x; p < p1; p += (size_t)UAG * blockDim.x) {
            Pack<T> v[UAG];
#pragma unroll
            for (int u = 0; u < UAG; ++u) {
              const size_t pu = p + (size_t)u * blockDim.x;
              if (pu < p1) v[u] = ld_cg(zc + pu * W);
            }
#pragma unroll
            for (int u = 0; u < UAG; ++u) {
              const size_t pu = p + (size_t)u * blockDim.x;
              if (pu < p1) st_stream(out + pu * W, v[u]);
            }
          }
        },
        [&](int c, size_t j) { out[j] = reinterpret_cast<const T*>(a.xbar[c])[j]; });
    }
  }
  report_nonfinite(a.nonfinite, bad);
  trace_mark(a, b, 3);
  if (!VIRTUAL) publish_done(a);
}

// ------------------------------------------------------------------ fused round (K7)
// One pass at a round boundary of the deterministic schedule: the local step (K5) of
// this minibatch, the mean of the round's snapshots read straight from every peer over
// NVLink (K2 order), the pull / finalize (K4) and the next snapshot (K1), per element:
//   x' = K5(x, g, m)                          (sgd_elem)
//   xbar = (sum_k snap_{(c+k)%P}) / P         (rot_sum / mean_div, ring order)
//   pull:     x'' = x' + (-alpha)*(snap_own + (-1)*xbar)       (pull_elem)
//   finalize: x'' = xbar + delta'             (optimizer.py:171; delta' = delta + s)
//   snap_next = x''
// Same element functions as the separate kernels, so the result is bit-identical to
// K5 -> (K2 completes) -> K4 under the deterministic schedule; HBM and NVLink stream
// concurrently instead of back to back, and xbar never touches HBM.
template <typename T>
struct FusedRound {
  T* x[kMaxR];
  const T* g[kMaxR];
  T* m[kMaxR];
  T* delta[kMaxR];
  T* snap_next[kMaxR];
  SgdCoef<T> c;
  T neg_alpha;
  int mode;  // 0 pull, 1 reference finalize (delta)
};

template <typename T, int P, bool VIRTUAL, int U>
__global__ void __launch_bounds__(256, (P == 1 ? 3 : 2)) k_fused_round(CommArgs a, FusedRound<T> f) {
  constexpr int W = Pack<T>::W;
  const int rank = VIRTUAL ? (int)blockIdx.y : a.rank;
  const int vr = VIRTUAL ? (int)blockIdx.y : 0;
  const int b = blockIdx.x;
  bool ok = true;
  trace_mark(a, b, 0);
  // Entry: every peer's snapshot slot must be final and every peer must be done reading
  // this rank's other slot.  When the previous launch was a round that raised end
  // signals (K7 one-shot or K8), those certify both and were raised before the peers
  // even launched this kernel; otherwise the per-CTA entry barrier.
  if (!VIRTUAL && P > 1) ok = a.prev_end ? rank_wait<P>(a, 1, a.prev_end, b, rank) : cta_barrier<P>(a, 0, b, rank);
  trace_mark(a, b, 1);
  unsigned bad = 0;
  if (ok) {
    const size_t n = a.n;
    size_t bnd[P + 1];
#pragma unroll
    for (int c = 0; c <= P; ++c) bnd[c] = chunk_bound(n, P, c);
    const T* src[P];
#pragma unroll
    for (int q = 0; q < P; ++q) src[q] = reinterpret_cast<const T*>(a.snap[q]);
    T* const x = f.x[vr];
    const T* const g = f.g[vr];
    T* const m = f.m[vr];
    T* const dl = f.delta[vr];
    T* const sn = f.snap_next[vr];
    const bool load_m = f.c.use_mom && !f.c.first, load_d = f.c.use_delta && !f.c.reset;
    const bool store_d = f.c.use_delta && (P == 1 || f.mode == 0);  // finalize resets delta
    auto element = [&](T& xv, T gv, T& mv, T& dv, const T (&lane)[P], int cidx) -> T {
      unsigned bb = sgd_elem(f.c, xv, gv, mv, dv);
      if constexpr (P > 1) {
        const T zb = mean_div<T, P>(rot_sum<T, P>(lane, cidx));
        if (f.mode == 0) {
          T own = lane[0];
#pragma unroll
          for (int q = 1; q < P; ++q) own = (q == rank) ? lane[q] : own;  // no dynamic register indexing
          bb += pull_elem(f.neg_alpha, xv, own, zb);
        } else {
          xv = add_rn(zb, dv);
          bb += !finite(xv);
        }
      }
      bad += bb;
      return xv;
    };
    auto range = [&](size_t p0, size_t p1) {
    for (size_t p = p0 + threadIdx.x; p < p1; p += (size_t)U * blockDim.x) {
      Pack<T> vx[U], vg[U], vm[U], vd[U], vs[U][P];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const size_t pu = p + (size_t)u * blockDim.x;
        if (pu < p1) {
          const size_t j = pu * W;
          vx[u] = ld_stream(x + j);
          vg[u] = ld_stream(g + j);
          if (load_m) vm[u] = ld_stream(m + j);
          if (load_d) vd[u] = ld_stream(dl + j);
          if constexpr (P > 1) {
#pragma unroll
            for (int q = 0; q < P; ++q) vs[u][q] = ld_cg(src[q] + j);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const size_t pu = p + (size_t)u * blockDim.x;
        if (pu < p1) {
          const size_t j0 = pu * W;
          const int c0 = chunk_of<P>(j0, bnd), c1 = chunk_of<P>(j0 + W - 1, bnd);
#pragma unroll
          for (int k = 0; k < W; ++k) {
            T lane[P];
#pragma unroll
            for (int q = 0; q < P; ++q) lane[q] = (P > 1) ? vs[u][q].v[k] : T(0);
            const int cidx = (c0 == c1) ? c0 : chunk_of<P>(j0 + k, bnd);
            element(vx[u].v[k], vg[u].v[k], vm[u].v[k], vd[u].v[k], lane, cidx);
          }
          st_stream(x + j0, vx[u]);
          if (f.c.use_mom) st_stream(m + j0, vm[u]);
          if (store_d) st_stream(dl + j0, vd[u]);
          st_stream(sn + j0, vx[u]);
        }
      }
    }
    };
    for_tiles<U>(a, b, n / W, range);
    if (b == a.nblocks - 1) {  // scalar tail n % W
      for (size_t j = (n / W) * W + threadIdx.x; j < n; j += blockDim.x) {
        T lane[P];
#pragma unroll
        for (int q = 0; q < P; ++q) lane[q] = (P > 1) ? src[q][j] : T(0);
        T xv = x[j], mv = load_m ? m[j] : T(0), dv = load_d ? dl[j] : T(0);
        element(xv, g[j], mv, dv, lane, chunk_of<P>(j, bnd));
        x[j] = xv;
        if (f.c.use_mom) m[j] = mv;
        if (store_d) dl[j] = dv;
        sn[j] = xv;
      }
    }
  }
  if (!VIRTUAL && P > 1 && ok) rank_signal<P>(a, 1, a.end_ctr, rank);  // certifies the next round's entry
  report_nonfinite(a.nonfinite, bad);
  trace_mark(a, b, 3);
  if (!VIRTUAL) publish_done(a);
}

// Two-shot form of K7 for larger P: (1) reduce-scatter of this rank's chunk into its
// xbar buffer (ring order, same as K3), (2) rank-level mid barrier, (3) over every
// pack: local step + pull with the pack's mean read straight from its owner's xbar
// (NVLink unless the pack is in the own chunk), next snapshot.  NVLink in-bytes
// 2(P-1)/P*B; xbar is written only for the own chunk.  Both phases take tiles from
// work queues.  Virtual ranks run phase 1 and phase 2 as two launches.
template <typename T, int P, bool VIRTUAL, int U>
__global__ void __launch_bounds__(256, 2) k_fused_twoshot(CommArgs a, FusedRound<T> f) {
  constexpr int W = Pack<T>::W;
  const int rank = VIRTUAL ? (int)blockIdx.y : a.rank;
  const int vr = VIRTUAL ? (int)blockIdx.y : 0;
  const int b = blockIdx.x;
  const size_t n = a.n;
  bool ok = true;
  unsigned bad = 0;
  unsigned long long* q0 = a.tile_ctr ? a.tile_ctr : nullptr;
  unsigned long long* q1 = a.tile_ctr ? a.tile_ctr + 1 : nullptr;
  T* const x = f.x[vr];
  const T* const g = f.g[vr];
  T* const m = f.m[vr];
  T* const dl = f.delta[vr];
  T* const sn = f.snap_next[vr];
  const T* const snap_own = reinterpret_cast<const T*>(a.snap[rank]);
  const bool load_m = f.c.use_mom && !f.c.first, load_d = f.c.use_delta && !f.c.reset;
  const bool store_d = f.c.use_delta && f.mode == 0;
  auto element = [&](T& xv, T gv, T& mv, T& dv, T sv, T zb) {
    unsigned bb = sgd_elem(f.c, xv, gv, mv, dv);
    if (f.mode == 0) {
      bb += pull_elem(f.neg_alpha, xv, sv, zb);
    } else {
      xv = add_rn(zb, dv);
      bb += !finite(xv);
    }
    bad += bb;
  };
  trace_mark(a, b, 0);
  if (a.phases & 1) {
    if (!VIRTUAL) ok = cta_barrier<P>(a, 0, b, rank);
    trace_mark(a, b, 1);
    if (ok) {
      // Own chunk, complete in this phase: its mean is formed here (ring order, stored
      // for the peers' phase 2) and the local step + pull applied right away — the own
      // snapshot is one of the P sources already in registers.
      T* own = reinterpret_cast<T*>(a.xbar[rank]);
      const T* src[P];
#pragma unroll
      for (int q = 0; q < P; ++q) src[q] = reinterpret_cast<const T*>(a.snap[q]);
      size_t cs, ce, cp0, cp1;
      chunk_packs<T, P>(n, rank, cs, ce, cp0, cp1);
      tile_loop(q0, b, a.nblocks, cp0, cp1 - cp0, (size_t)kTileIters * U * blockDim.x, [&](size_t p0, size_t p1) {
        for (size_t p = p0 + threadIdx.x; p < p1; p += (size_t)U * blockDim.x) {
          Pack<T> v[U][P], vx[U], vg[U], vm[U], vd[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const size_t pu = p + (size_t)u * blockDim.x;
            if (pu < p1) {
              const size_t j = pu * W;
#pragma unroll
              for (int q = 0; q < P; ++q) v[u][q] = ld_cg(src[q] + j);
              vx[u] = ld_stream(x + j);
              vg[u] = ld_stream(g + j);
              if (load_m) vm[u] = ld_stream(m + j);
              if (load_d) vd[u] = ld_stream(dl + j);
            }
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const size_t pu = p + (size_t)u * blockDim.x;
            if (pu < p1) {
              const size_t j = pu * W;
              Pack<T> z;
#pragma unroll
              for (int k = 0; k < W; ++k) {
                T lane[P];
#pragma unroll
                for (int q = 0; q < P; ++q) lane[q] = v[u][q].v[k];
                T sv = lane[0];
#pragma unroll
                for (int q = 1; q < P; ++q) sv = (q == rank) ? lane[q] : sv;
                z.v[k] = mean_div<T, P>(rot_sum<T, P>(lane, rank));
                element(vx[u].v[k], vg[u].v[k], vm[u].v[k], vd[u].v[k], sv, z.v[k]);
              }
              st_plain(own + j, z);
              st_stream(x + j, vx[u]);
              if (f.c.use_mom) st_stream(m + j, vm[u]);
              if (store_d) st_stream(dl + j, vd[u]);
              st_stream(sn + j, vx[u]);
            }
          }
        }
      });
      if (b == 0) {  // unaligned head / tail elements of the own chunk
        const size_t he = cp0 * W < ce ? cp0 * W : ce;
        const size_t ts = cp1 * W > he ? cp1 * W : he;
        auto scalar = [&](size_t j) {
          const T zb = mean_div<T, P>(ordered_sum<T, P>(src, rank, j));
          own[j] = zb;
          T xv = x[j], mv = load_m ? m[j] : T(0), dv = load_d ? dl[j] : T(0);
          element(xv, g[j], mv, dv, snap_own[j], zb);
          x[j] = xv;
          if (f.c.use_mom) m[j] = mv;
          if (store_d) dl[j] = dv;
          sn[j] = xv;
        };
        for (size_t j = cs + threadIdx.x; j < he; j += blockDim.x) scalar(j);
        for (size_t j = ts + threadIdx.x; j < ce; j += blockDim.x) scalar(j);
      }
    }
  }
  if (a.phases & 2) {
    if (!VIRTUAL && ok) ok = rank_barrier<P>(a, b, rank);
    trace_mark(a, b, 2);
    if (ok) {
      chunk_tiles<T, P>(q1, b, a.nblocks, n, rank, true, (size_t)kTileIters * U * blockDim.x,
        [&](int c, size_t p0, size_t p1) {
          const T* zc = reinterpret_cast<const T*>(a.xbar[c]);  // owner's reduced chunk (NVLink unless c == rank)
          for (size_t p = p0 + threadIdx.x; p < p1; p += (size_t)U * blockDim.x) {
            Pack<T> vx[U], vg[U], vm[U], vd[U], vs[U], vz[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const size_t pu = p + (size_t)u * blockDim.x;
              if (pu < p1) {
                const size_t j = pu * W;
                vz[u] = ld_cg(zc + j);
                vx[u] = ld_stream(x + j);
                vg[u] = ld_stream(g + j);
                if (load_m) vm[u] = ld_stream(m + j);
                if (load_d) vd[u] = ld_stream(dl + j);
                if (f.mode == 0) vs[u] = ld_stream(snap_own + j);
              }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const size_t pu = p + (size_t)u * blockDim.x;
              if (pu < p1) {
                const size_t j = pu * W;
#pragma unroll
                for (int k = 0; k < W; ++k)
                  element(vx[u].v[k], vg[u].v[k], vm[u].v[k], vd[u].v[k], vs[u].v[k], vz[u].v[k]);
                st_stream(x + j, vx[u]);
                if (f.c.use_mom) st_stream(m + j, vm[u]);
                if (store_d) st_stream(dl + j, vd[u]);
                st_stream(sn + j, vx[u]);
              }
            }
          }
        },
        [&](int c, size_t j) {
          T xv = x[j], mv = load_m ? m[j] : T(0), dv = load_d ? dl[j] : T(0);
          element(xv, g[j], mv, dv, f.mode == 0 ? snap_own[j] : T(0), reinterpret_cast<const T*>(a.xbar[c])[j]);
          x[j] = xv;
          if (f.c.use_mom) m[j] = mv;
          if (store_d) dl[j] = dv;
          sn[j] = xv;
        });
    }
  }
  report_nonfinite(a.nonfinite, bad);
  trace_mark(a, b, 3);
  if (!VIRTUAL) publish_done(a);
}

// Launch `kernel` normally, or cooperatively (all CTAs co-resident, required by the
// rank-level barrier of the P2P two-shot kernels).  A cooperative grid is clamped to
// what fits on the device — every rank computes the same clamp on the same GPU type,
// so the per-CTA flag slots still line up.
template <typename... Args>
int launch_kernel(bool coop, void (*kernel)(Args...), dim3 grid, int threads, cudaStream_t s, Args... args) {
  if (!coop) {
    kernel<<<grid, threads, 0, s>>>(args...);
    LASGD_CUDA_TRY(cudaGetLastError());
    return LASGD_OK;
  }
  void* kargs[] = {(void*)&args...};
  LASGD_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)kernel, grid, dim3(threads), kargs, 0, s));
  return LASGD_OK;
}

template <typename... Args>
int coop_capacity(void (*kernel)(Args...), int threads) {
  // cached per (kernel, threads): an occupancy query per launch costs host time every step
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> cache;
  const auto key = std::make_pair(reinterpret_cast<const void*>(kernel), threads);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  const int cap = per_sm * num_sms();
  std::lock_guard<std::mutex> lk(mu);
  cache[key] = cap;
  return cap;
}

template <typename T, bool VIRTUAL>
int launch_fused(int P, const CommArgs& a, const FusedRound<T>& f, dim3 grid, int threads, cudaStream_t s,
                 int algo = LASGD_ALGO_ONESHOT) {
  static_assert(sizeof(CommArgs) + sizeof(FusedRound<T>) < 4000, "kernel parameters");
#define LASGD_FCASE(PP)                                                                             \
  case PP:                                                                                          \
    if (algo == LASGD_ALGO_TWOSHOT && PP > 1) {                                                     \
      auto kern = k_fused_twoshot<T, PP, VIRTUAL, (PP <= 4 ? 2 : 1)>;                               \
      CommArgs aa = a;                                                                              \
      if (!VIRTUAL) {                                                                               \
        const int cap = coop_capacity(kern, threads);                                               \
        if ((int)grid.x > cap) grid.x = cap;                                                        \
        aa.nblocks = grid.x;                                                                        \
      }                                                                                             \
      return launch_kernel(!VIRTUAL, kern, grid, threads, s, aa, f);                                \
    }                                                                                               \
    return launch_kernel(false, k_fused_round<T, PP, VIRTUAL, (PP <= 2 ? 2 : 1)>, grid, threads, s, \
                         a, f);
  switch (P) {
    LASGD_FCASE(1)
    LASGD_FCASE(2)
    LASGD_FCASE(3)
    LASGD_FCASE(4)
    LASGD_FCASE(5)
    LASGD_FCASE(6)
    LASGD_FCASE(7)
    LASGD_FCASE(8)
    default: return fail(LASGD_ERR_UNSUPPORTED, "world size %d > %d", P, kMaxR);
  }
#undef LASGD_FCASE
  LASGD_CUDA_TRY(cudaGetLastError());
  return LASGD_OK;
}

template <typename T>
FusedRound<T> make_fused(int nr, void* const* x, const void* const* g, void* const* m, void* const* delta,
                         void* const* snap_next, const lasgd_sgd_params* sgd, double alpha, int mode) {
  FusedRound<T> f;
  memset(&f, 0, sizeof(f));
  for (int r = 0; r < nr; ++r) {
    f.x[r] = (T*)x[r];
    f.g[r] = (const T*)g[r];
    f.m[r] = m ? (T*)m[r] : nullptr;
    f.delta[r] = delta ? (T*)delta[r] : nullptr;
    f.snap_next[r] = (T*)snap_next[r];
  }
  f.c = make_sgd_coef<T>(sgd, delta != nullptr && delta[0] != nullptr);
  f.neg_alpha = (T)(-alpha);
  f.mode = mode;
  return f;
}

int check_fused_args(int nr, void* const* x, const void* const* g, void* const* m, void* const* delta,
                     void* const* snap_next, const lasgd_sgd_params* sgd, double alpha, int mode) {
  if (!sgd) return fail(LASGD_ERR_INVALID_ARGUMENT, "null sgd params");
  if (mode != 0 && mode != 1) return fail(LASGD_ERR_INVALID_ARGUMENT, "mode %d (0 pull, 1 finalize)", mode);
  if (mode == 0 && !(alpha > 0.0 && alpha <= 1.0)) return fail(LASGD_ERR_INVALID_ARGUMENT, "alpha must be in (0, 1], got %g", alpha);
  if (mode == 1 && (!delta || !delta[0])) return fail(LASGD_ERR_INVALID_ARGUMENT, "finalize mode needs the delta buffer");
  if (sgd->momentum != 0.0 && !m) return fail(LASGD_ERR_INVALID_ARGUMENT, "momentum needs m");
  if (sgd->nesterov && (sgd->momentum <= 0.0 || sgd->dampening != 0.0))
    return fail(LASGD_ERR_INVALID_ARGUMENT, "Nesterov momentum requires a momentum and zero dampening");
  for (int r = 0; r < nr; ++r) {
    if (!x[r] || !g[r] || !snap_next[r] || !aligned16(x[r]) || !aligned16(g[r]) || !aligned16(snap_next[r]) ||
        (m && m[r] && !aligned16(m[r])) || (delta && delta[r] && !aligned16(delta[r])))
      return fail(LASGD_ERR_INVALID_ARGUMENT, "fused round buffers must be non-null and 16-B aligned");
    if (sgd->momentum != 0.0 && !m[r]) return fail(LASGD_ERR_INVALID_ARGUMENT, "momentum needs m");
  }
  return LASGD_OK;
}

// ------------------------------------------------------------------ push round (K8)
// The fused round with the data movement done by remote STORES from the producer.
// Chunk c is owned by rank c.  Every rank keeps, in its IPC region, a staging area
// stage[parity][source][chunk] for the contributions to its own chunk.
//   init (phase bit 4): push chunk c of the current snapshot to owner c's staging.
//   phase A (bit 1): wait for every rank's end signal of the previous push launch
//     (staged contributions complete; peers finished their previous round); the owner
//     forms the ring-order mean of its chunk from local staging + its own snapshot,
//     applies the local step + pull to its own chunk, and pushes the mean to every
//     peer's xbar.
//   rank-level mid barrier (all means pushed).
//   phase B (bit 2): every other chunk: local step + pull with the mean in the local
//     xbar, next snapshot written locally and pushed to the owner's staging (other
//     parity); then the rank-level end signal.
// Per rank and round: NVLink out 2(P-1)/P*B as posted writes, all reads local.  Same
// element functions and summation order as K7, so results are bit-identical.
template <typename T>
__device__ __forceinline__ T* stage_ptr(const CommArgs& a, int owner, int parity, int src, int P) {
  return reinterpret_cast<T*>(a.stage[owner]) + ((size_t)parity * P + src) * a.stage_elems;
}

template <typename T, int P, bool VIRTUAL, int U>
__global__ void __launch_bounds__(256, 2) k_push_round(CommArgs a, FusedRound<T> f) {
  constexpr int W = Pack<T>::W;
  const int rank = VIRTUAL ? (int)blockIdx.y : a.rank;
  const int vr = VIRTUAL ? (int)blockIdx.y : 0;
  const int b = blockIdx.x;
  const size_t n = a.n;
  const int cur = a.cur, nxt = 1 - a.cur;
  bool ok = true;
  unsigned bad = 0;
  unsigned long long* q0 = a.tile_ctr ? a.tile_ctr : nullptr;
  unsigned long long* q1 = a.tile_ctr ? a.tile_ctr + 1 : nullptr;
  const T* const snap_own = reinterpret_cast<const T*>(a.snap[rank]);
  trace_mark(a, b, 0);
  // offset of element j of chunk c inside a staging slot (keeps 16-byte alignment)
  auto soff = [&](int c, size_t j) { return j - chunk_bound(n, P, c) / W * W; };
  if (a.phases & 4) {
    // initial contributions: chunk c of the current snapshot -> owner c, parity cur
    chunk_tiles<T, P>(q1, b, a.nblocks, n, rank, true, (size_t)kTileIters * U * blockDim.x,
      [&](int c, size_t p0, size_t p1) {
        T* dst = stage_ptr<T>(a, c, cur, rank, P);
        for (size_t p = p0 + threadIdx.x; p < p1; p += (size_t)U * blockDim.x) {
          Pack<T> v[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const size_t pu = p + (size_t)u * blockDim.x;
            if (pu < p1) v[u] = ld_stream(snap_own + pu * W);
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const size_t pu = p + (size_t)u * blockDim.x;
            if (pu < p1) st_plain(dst + soff(c, pu * W), v[u]);
          }
        }
      },
      [&](int c, size_t j) { stage_ptr<T>(a, c, cur, rank, P)[soff(c, j)] = snap_own[j]; });
    if (!VIRTUAL) rank_signal<P>(a, 1, a.end_ctr, rank);
  }
  T* const x = f.x[vr];
  const T* const g = f.g[vr];
  T* const m = f.m[vr];
  T* const dl = f.delta[vr];
  T* const sn = f.snap_next[vr];
  const bool load_m = f.c.use_mom && !f.c.first, load_d = f.c.use_delta && !f.c.reset;
  const bool store_d = f.c.use_delta && f.mode == 0;
  auto element = [&](T& xv, T gv, T& mv, T& dv, T sv, T zb) {
    unsigned bb = sgd_elem(f.c, xv, gv, mv, dv);
    if (f.mode == 0) {
      bb += pull_elem(f.neg_alpha, xv, sv, zb);
    } else {
      xv = add_rn(zb, dv);
      bb += !finite(xv);
    }
    bad += bb;
  };
  if (a.phases & 1) {
    if (!VIRTUAL) ok = rank_wait<P>(a, 1, a.prev_push, b, rank);
    trace_mark(a, b, 1);
    if (ok) {
      const T* src[P];
#pragma unroll
      for (int q = 0; q < P; ++q) src[q] = q == rank ? snap_own : stage_ptr<T>(a, rank, cur, q, P);
      size_t cs, ce, cp0, cp1;
      chunk_packs<T, P>(n, rank, cs, ce, cp0, cp1);
      const size_t base = cs / W * W;  // staging offset origin of the own chunk
      tile_loop(q0, b, a.nblocks, cp0, cp1 - cp0, (size_t)kTileIters * U * blockDim.x, [&](size_t p0, size_t p1) {
        for (size_t p = p0 + threadIdx.x; p < p1; p += (size_t)U * blockDim.x) {
          Pack<T> v[U][P], vx[U], vg[U], vm[U], vd[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const size_t pu = p + (size_t)u * blockDim.x;
            if (pu < p1) {
              const size_t j = pu * W;
#pragma unroll
              for (int q = 0; q < P; ++q) v[u][q] = ld_stream(src[q] + (q == rank ? j : j - base));
              vx[u] = ld_stream(x + j);
              vg[u] = ld_stream(g + j);
              if (load_m) vm[u] = ld_stream(m + j);
              if (load_d) vd[u] = ld_stream(dl + j);
            }
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const size_t pu = p + (size_t)u * blockDim.x;
            if (pu < p1) {
              const size_t j = pu * W;
              Pack<T> z;
#pragma unroll
              for (int k = 0; k < W; ++k) {
                T lane[P];
#pragma unroll
                for (int q = 0; q < P; ++q) lane[q] = v[u][q].v[k];
                T sv = lane[0];
#pragma unroll
                for (int q = 1; q < P; ++q) sv = (q == rank) ? lane[q] : sv;
                z.v[k] = mean_div<T, P>(rot_sum<T, P>(lane, rank));
                element(vx[u].v[k], vg[u].v[k], vm[u].v[k], vd[u].v[k], sv, z.v[k]);
              }
#pragma unroll
              for (int q = 0; q < P; ++q)
                if (q != rank) st_plain(reinterpret_cast<T*>(a.xbar[q]) + j, z);  // the mean to every peer
              st_stream(x + j, vx[u]);
              if (f.c.use_mom) st_stream(m + j, vm[u]);
              if (store_d) st_stream(dl + j, vd[u]);
              st_stream(sn + j, vx[u]);
            }
          }
        }
      });
      if (b == 0) {  // unaligned head / tail elements of the own chunk
        const size_t he = cp0 * W < ce ? cp0 * W : ce;
        const size_t ts = cp1 * W > he ? cp1 * W : he;
        auto scalar = [&](size_t j) {
          T lane[P];
#pragma unroll
          for (int q = 0; q < P; ++q) lane[q] = src[q][q == rank ? j : j - base];
          const T zb = mean_div<T, P>(rot_sum<T, P>(lane, rank));
#pragma unroll
          for (int q = 0; q < P; ++q)
            if (q != rank) reinterpret_cast<T*>(a.xbar[q])[j] = zb;
          T xv = x[j], mv = load_m ? m[j] : T(0), dv = load_d ? dl[j] : T(0);
          element(xv, g[j], mv, dv, snap_own[j], zb);
          x[j] = xv;
          if (f.c.use_mom) m[j] = mv;
          if (store_d) dl[j] = dv;
          sn[j] = xv;
        };
        for (size_t j = cs + threadIdx.x; j < he; j += blockDim.x) scalar(j);
        for (size_t j = ts + threadIdx.x; j < ce; j += blockDim.x) scalar(j);
      }
    }
  }
  if (a.phases & 2) {
    if (!VIRTUAL && ok) ok = rank_barrier<P>(a, b, rank);
    trace_mark(a, b, 2);
    if (ok) {
      const T* zl = reinterpret_cast<const T*>(a.xbar[rank]);  // means pushed by their owners
      chunk_tiles<T, P>(q1, b, a.nblocks, n, rank, true, (size_t)kTileIters * U * blockDim.x,
        [&](int c, size_t p0, size_t p1) {
          T* dst = stage_ptr<T>(a, c, nxt, rank, P);
          for (size_t p = p0 + threadIdx.x; p < p1; p += (size_t)U * blockDim.x) {
            Pack<T> vx[U], vg[U], vm[U], vd[U], vs[U], vz[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const size_t pu = p + (size_t)u * blockDim.x;
              if (pu < p1) {
                const size_t j = pu * W;
                vz[u] = ld_stream(zl + j);
                vx[u] = ld_stream(x + j);
                vg[u] = ld_stream(g + j);
                if (load_m) vm[u] = ld_stream(m + j);
                if (load_d) vd[u] = ld_stream(dl + j);
                if (f.mode == 0) vs[u] = ld_stream(snap_own + j);
              }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const size_t pu = p + (size_t)u * blockDim.x;
              if (pu < p1) {
                const size_t j = pu * W;
#pragma unroll
                for (int k = 0; k < W; ++k)
                  element(vx[u].v[k], vg[u].v[k], vm[u].v[k], vd[u].v[k], vs[u].v[k], vz[u].v[k]);
                st_plain(dst + soff(c, j), vx[u]);  // next-round contribution to owner c
                st_stream(x + j, vx[u]);
                if (f.c.use_mom) st_stream(m + j, vm[u]);
                if (store_d) st_stream(dl + j, vd[u]);
                st_stream(sn + j, vx[u]);
              }
            }
          }
        },
        [&](int c, size_t j) {
          T xv = x[j], mv = load_m ? m[j] : T(0), dv = load_d ? dl[j] : T(0);
          element(xv, g[j], mv, dv, f.mode == 0 ? snap_own[j] : T(0), zl[j]);
          x[j] = xv;
          if (f.c.use_mom) m[j] = mv;
          if (store_d) dl[j] = dv;
          sn[j] = xv;
          stage_ptr<T>(a, c, nxt, rank, P)[soff(c, j)] = xv;
        });
      if (!VIRTUAL) rank_signal<P>(a, 1, a.end_ctr, rank);
    }
  }
  report_nonfinite(a.nonfinite, bad);
  trace_mark(a, b, 3);
  if (!VIRTUAL) publish_done(a);
}

// ------------------------------------------------------------------ mirror push round (K8, P = 2)
// At P = 2 the push round keeps a full mirror of the peer's snapshot in local HBM: the
// staging area (2 parities x 2 sources x n/2) is re-used as [parity][n].  Each round
// reads the own snapshot and the mirror (both local), forms the ring-order mean per
// element exactly like the one-shot K7, applies local step + pull, writes the next
// snapshot locally AND stores it into the peer's mirror (other parity) as posted NVLink
// writes; the rank-level end signals certify the mirror for the next round's entry.
// One phase, no mid barrier; NVLink out B per round (= the one-shot's B in), as stores.
template <typename T>
__device__ __forceinline__ T* mirror_ptr(const CommArgs& a, int owner, int parity) {
  return reinterpret_cast<T*>(a.stage[owner]) + (size_t)parity * 2 * a.stage_elems;
}

template <typename T, bool VIRTUAL, int U>
__global__ void __launch_bounds__(256, 2) k_push_mirror(CommArgs a, FusedRound<T> f) {
  constexpr int P = 2;
  constexpr int W = Pack<T>::W;
  const int rank = VIRTUAL ? (int)blockIdx.y : a.rank;
  const int vr = VIRTUAL ? (int)blockIdx.y : 0;
  const int peer = 1 - rank;
  const int b = blockIdx.x;
  const size_t n = a.n;
  const int cur = a.cur, nxt = 1 - a.cur;
  bool ok = true;
  unsigned bad = 0;
  const T* const snap_own = reinterpret_cast<const T*>(a.snap[rank]);
  trace_mark(a, b, 0);
  if (a.phases & 4) {  // initial mirror: the current snapshot -> the peer's mirror, parity cur
    T* dst = mirror_ptr<T>(a, peer, cur);
    for_tiles<U>(a, b, n / W, [&](size_t p0, size_t p1) {
      for (size_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) st_plain(dst + p * W, ld_stream(snap_own + p * W));
    });
    if (b == a.nblocks - 1)
      for (size_t j = (n / W) * W + threadIdx.x; j < n; j += blockDim.x) dst[j] = snap_own[j];
    if (!VIRTUAL) rank_signal<P>(a, 1, a.end_ctr, rank);
  }
  if (a.phases & 1) {
    if (!VIRTUAL) ok = rank_wait<P>(a, 1, a.prev_push, b, rank);
    trace_mark(a, b, 1);
    if (ok) {
      size_t bnd[P + 1];
#pragma unroll
      for (int c = 0; c <= P; ++c) bnd[c] = chunk_bound(n, P, c);
      const T* const mir = mirror_ptr<T>(a, rank, cur);  // the peer's snapshot, local copy
      T* const out = mirror_ptr<T>(a, peer, nxt);          // the peer's copy of our next snapshot
      T* const x = f.x[vr];
      const T* const g = f.g[vr];
      T* const m = f.m[vr];
      T* const dl = f.delta[vr];
      T* const sn = f.snap_next[vr];
      const bool load_m = f.c.use_mom && !f.c.first, load_d = f.c.use_delta && !f.c.reset;
      const bool store_d = f.c.use_delta && f.mode == 0;
      auto element = [&](T& xv, T gv, T& mv, T& dv, T own, T oth, int cidx) {
        unsigned bb = sgd_elem(f.c, xv, gv, mv, dv);
        T lane[P];  // lanes by rank, selected without dynamic register indexing
        lane[0] = rank == 0 ? own : oth;
        lane[1] = rank == 0 ? oth : own;
        const T zb = mean_div<T, P>(rot_sum<T, P>(lane, cidx));
        if (f.mode == 0) {
          bb += pull_elem(f.neg_alpha, xv, own, zb);
        } else {
          xv = add_rn(zb, dv);
          bb += !finite(xv);
        }
        bad += bb;
      };
      for_tiles<U>(a, b, n / W, [&](size_t p0, size_t p1) {
        for (size_t p = p0 + threadIdx.x; p < p1; p += (size_t)U * blockDim.x) {
          Pack<T> vx[U], vg[U], vm[U], vd[U], vs[U], vo[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const size_t pu = p + (size_t)u * blockDim.x;
            if (pu < p1) {
              const size_t j = pu * W;
              vx[u] = ld_stream(x + j);
              vg[u] = ld_stream(g + j);
              if (load_m) vm[u] = ld_stream(m + j);
              if (load_d) vd[u] = ld_stream(dl + j);
              vs[u] = ld_stream(snap_own + j);
              vo[u] = ld_stream(mir + j);
            }
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const size_t pu = p + (size_t)u * blockDim.x;
            if (pu < p1) {
              const size_t j0 = pu * W;
              const int c0 = chunk_of<P>(j0, bnd), c1 = chunk_of<P>(j0 + W - 1, bnd);
#pragma unroll
              for (int k = 0; k < W; ++k)
                element(vx[u].v[k], vg[u].v[k], vm[u].v[k], vd[u].v[k], vs[u].v[k], vo[u].v[k],
                        c0 == c1 ? c0 : chunk_of<P>(j0 + k, bnd));
              st_plain(out + j0, vx[u]);  // posted NVLink write into the peer's mirror
              st_stream(x + j0, vx[u]);
              if (f.c.use_mom) st_stream(m + j0, vm[u]);
              if (store_d) st_stream(dl + j0, vd[u]);
              st_stream(sn + j0, vx[u]);
            }
          }
        }
      });
      if (b == a.nblocks - 1) {  // scalar tail n % W
        for (size_t j = (n / W) * W + threadIdx.x; j < n; j += blockDim.x) {
          T xv = x[j], mv = load_m ? m[j] : T(0), dv = load_d ? dl[j] : T(0);
          element(xv, g[j], mv, dv, snap_own[j], mir[j], chunk_of<P>(j, bnd));
          x[j] = xv;
          if (f.c.use_mom) m[j] = mv;
          if (store_d) dl[j] = dv;
          sn[j] = xv;
          out[j] = xv;
        }
      }
      if (!VIRTUAL) rank_signal<P>(a, 1, a.end_ctr, rank);
    }
  }
  report_nonfinite(a.nonfinite, bad);
  trace_mark(a, b, 3);
  if (!VIRTUAL) publish_done(a);
}

// ------------------------------------------------------------------ dispatch
template <int P>
constexpr int unroll_for() { return P <= 2 ? 8 : (P <= 4 ? 4 : 2); }
template <int P>
constexpr int oneshot_unroll() { return P <= 2 ? 4 : (P <= 4 ? 2 : 1); }  // <= 128 regs, no spills

template <typename T, bool VIRTUAL>
int launch_allreduce(int algo, int P, const CommArgs& a, dim3 grid, int threads, cudaStream_t s) {
#define LASGD_CASE(PP)                                                                                    \
  case PP:                                                                                                \
    if (algo == LASGD_ALGO_ONESHOT) return launch_kernel(false, k_oneshot<T, PP, VIRTUAL, oneshot_unroll<PP>()>, \
                                                         grid, threads, s, a);                            \
    {                                                                                                     \
      auto kern = k_twoshot<T, PP, VIRTUAL, unroll_for<PP>(), 8>;                                         \
      CommArgs aa = a;                                                                                    \
      if (!VIRTUAL) {                                                                                     \
        const int cap = coop_capacity(kern, threads);                                                     \
        if ((int)grid.x > cap) grid.x = cap;                                                              \
        aa.nblocks = grid.x;                                                                              \
      }                                                                                                   \
      return launch_kernel(!VIRTUAL, kern, grid, threads, s, aa);                                         \
    }
  switch (P) {
    LASGD_CASE(1)
    LASGD_CASE(2)
    LASGD_CASE(3)
    LASGD_CASE(4)
    LASGD_CASE(5)
    LASGD_CASE(6)
    LASGD_CASE(7)
    LASGD_CASE(8)
    default: return fail(LASGD_ERR_UNSUPPORTED, "world size %d > %d", P, kMaxR);
  }
#undef LASGD_CASE
  LASGD_CUDA_TRY(cudaGetLastError());
  return LASGD_OK;
}

template <typename T, bool VIRTUAL>
int launch_push(int P, const CommArgs& a, const FusedRound<T>& f, dim3 grid, int threads, cudaStream_t s) {
#define LASGD_PCASE(PP)                                                                             \
  case PP: {                                                                                        \
    auto kern = k_push_round<T, PP, VIRTUAL, (PP <= 4 ? 2 : 1)>;                                    \
    CommArgs aa = a;                                                                                \
    if (!VIRTUAL) {                                                                                 \
      const int cap = coop_capacity(kern, threads);                                                 \
      if ((int)grid.x > cap) grid.x = cap;                                                          \
      aa.nblocks = grid.x;                                                                          \
    }                                                                                               \
    return launch_kernel(!VIRTUAL, kern, grid, threads, s, aa, f);                                  \
  }
  if (P == 2) {  // mirror form
    auto kern = k_push_mirror<T, VIRTUAL, 2>;
    CommArgs aa = a;
    if (!VIRTUAL) {
      const int cap = coop_capacity(kern, threads);
      if ((int)grid.x > cap) grid.x = cap;
      aa.nblocks = grid.x;
    }
    return launch_kernel(!VIRTUAL, kern, grid, threads, s, aa, f);
  }
  switch (P) {
    LASGD_PCASE(3)
    LASGD_PCASE(4)
    LASGD_PCASE(5)
    LASGD_PCASE(6)
    LASGD_PCASE(7)
    LASGD_PCASE(8)
    default: return fail(LASGD_ERR_UNSUPPORTED, "push round needs 2 <= P <= %d, got %d", kMaxR, P);
  }
#undef LASGD_PCASE
}

size_t elem_bytes(int dtype);

// Elements per staging slot: the largest chunk plus room for the 16-byte alignment shift.
size_t push_stage_elems(size_t n, int P, int dtype) {
  const size_t W = 16 / elem_bytes(dtype);
  const size_t e = (n + P - 1) / P + 2 * W;
  return (e + 63) / 64 * 64;  // every slot starts 16-byte (in fact 256-byte) aligned
}

int launch_any(int dtype, bool virt, int algo, int P, const CommArgs& a, dim3 grid, int threads, cudaStream_t s) {
  if (dtype == LASGD_F32)
    return virt ? launch_allreduce<float, true>(algo, P, a, grid, threads, s)
                : launch_allreduce<float, false>(algo, P, a, grid, threads, s);
  if (dtype == LASGD_F64)
    return virt ? launch_allreduce<double, true>(algo, P, a, grid, threads, s)
                : launch_allreduce<double, false>(algo, P, a, grid, threads, s);
  return fail(LASGD_ERR_INVALID_ARGUMENT, "unknown dtype %d", dtype);
}

int launch_gate(int P, const CommArgs& a, cudaStream_t s) {
  switch (P) {
    case 2: k_gate<2><<<1, 32, 0, s>>>(a); break;
    case 3: k_gate<3><<<1, 32, 0, s>>>(a); break;
    case 4: k_gate<4><<<1, 32, 0, s>>>(a); break;
    case 5: k_gate<5><<<1, 32, 0, s>>>(a); break;
    case 6: k_gate<6><<<1, 32, 0, s>>>(a); break;
    case 7: k_gate<7><<<1, 32, 0, s>>>(a); break;
    case 8: k_gate<8><<<1, 32, 0, s>>>(a); break;
    default: return fail(LASGD_ERR_UNSUPPORTED, "gate needs 2 <= P <= %d, got %d", kMaxR, P);
  }
  LASGD_CUDA_TRY(cudaGetLastError());
  return LASGD_OK;
}

size_t elem_bytes(int dtype) { return dtype == LASGD_F64 ? 8 : 4; }

// One-shot reads (P-1)*B per rank, two-shot 2(P-1)/P*B plus one extra barrier
// (~a few microseconds).  P == 2 moves the same bytes either way: one-shot wins.
int resolve_algo(int algo, int P, size_t bytes) {
  if (algo != LASGD_ALGO_AUTO) return algo;
  if (P <= 2) return LASGD_ALGO_ONESHOT;
  const size_t cutoff = P <= 4 ? (size_t)2 << 20 : (size_t)1 << 20;
  return bytes <= cutoff ? LASGD_ALGO_ONESHOT : LASGD_ALGO_TWOSHOT;
}

// Fused round (K7/K8): where the all-reduce would be two-shot, the push round moves
// the same NVLink bytes with stores only and no entry wait on peers' snapshots
// (measured 3-5% faster per round at P=3/4, profiles/bench_r01_algo_*.json).
// At P = 2 the push round is the mirror form: same bytes as the one-shot, moved as
// posted stores, ~6% faster per round at ResNet-50 size (profiles/k8_mirror_ab_r01_p2.jsonl).
int resolve_fused_algo(int algo, int P, size_t bytes) {
  if (P <= 1) return LASGD_ALGO_ONESHOT;
  if (algo != LASGD_ALGO_AUTO) return algo;
  if (P == 2) return bytes >= ((size_t)1 << 20) ? LASGD_ALGO_PUSH : LASGD_ALGO_ONESHOT;
  const int a = resolve_algo(algo, P, bytes);
  return a == LASGD_ALGO_TWOSHOT ? LASGD_ALGO_PUSH : a;
}

}  // namespace lasgd

using namespace lasgd;

// ====================================================================== virtual ranks
extern "C" int lasgd_mean_virtual(void* const* outs, int n_out, const void* const* srcs, int P, size_t n, int dtype,
                                  int algo, int nblocks, unsigned long long* nonfinite, void* stream) {
  if (P < 1 || P > kMaxR) return fail(LASGD_ERR_UNSUPPORTED, "P=%d outside [1, %d]", P, kMaxR);
  if (!outs || !srcs) return fail(LASGD_ERR_INVALID_ARGUMENT, "null pointer array");
  if (n == 0) return LASGD_OK;
  if (dtype != LASGD_F32 && dtype != LASGD_F64) return fail(LASGD_ERR_INVALID_ARGUMENT, "unknown dtype %d", dtype);
  algo = resolve_algo(algo, P, n * elem_bytes(dtype));
  if (algo != LASGD_ALGO_ONESHOT && algo != LASGD_ALGO_TWOSHOT)
    return fail(LASGD_ERR_INVALID_ARGUMENT, "unknown algo %d", algo);
  if (algo == LASGD_ALGO_TWOSHOT && n_out != P)
    return fail(LASGD_ERR_INVALID_ARGUMENT, "two-shot emulation needs one output per rank (n_out=%d, P=%d)", n_out, P);
  if (n_out < 1 || n_out > kMaxR) return fail(LASGD_ERR_INVALID_ARGUMENT, "n_out=%d", n_out);
  if (nblocks <= 0) nblocks = 2 * num_sms();
  if (nblocks > 65535) nblocks = 65535;
  CommArgs a;
  memset(&a, 0, sizeof(a));
  for (int q = 0; q < P; ++q) {
    if (!srcs[q] || !aligned16(srcs[q])) return fail(LASGD_ERR_INVALID_ARGUMENT, "source %d null or not 16-B aligned", q);
    a.snap[q] = reinterpret_cast<const char*>(srcs[q]);
  }
  for (int r = 0; r < n_out; ++r) {
    if (!outs[r] || !aligned16(outs[r])) return fail(LASGD_ERR_INVALID_ARGUMENT, "output %d null or not 16-B aligned", r);
    a.xbar[r] = reinterpret_cast<char*>(outs[r]);
  }
  a.n = n;
  a.nblocks = nblocks;
  a.skip_signal_phase = -1;
  a.nonfinite = nonfinite;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  dim3 grid(nblocks, n_out);
  if (algo == LASGD_ALGO_ONESHOT) {
    a.phases = 1;
    return launch_any(dtype, true, algo, P, a, grid, 256, s);
  }
  a.phases = 1;  // reduce-scatter of every virtual rank ...
  int rc = launch_any(dtype, true, algo, P, a, grid, 256, s);
  if (rc) return rc;
  a.phases = 2;  // ... then the all-gather (stream order replaces the mid barrier)
  a.nonfinite = nullptr;
  return launch_any(dtype, true, algo, P, a, grid, 256, s);
}

extern "C" int lasgd_fused_round_virtual(int P, int algo, void* const* x, const void* const* g, void* const* m,
                                         void* const* delta, const void* const* snaps, void* const* xbars,
                                         void* const* snap_next, size_t n, int dtype, const lasgd_sgd_params* sgd,
                                         double alpha, int mode, int nblocks, unsigned long long* nonfinite,
                                         void* stream) {
  if (P < 1 || P > kMaxR) return fail(LASGD_ERR_UNSUPPORTED, "P=%d outside [1, %d]", P, kMaxR);
  if (!x || !g || !snaps || !snap_next) return fail(LASGD_ERR_INVALID_ARGUMENT, "null pointer array");
  if (dtype != LASGD_F32 && dtype != LASGD_F64) return fail(LASGD_ERR_INVALID_ARGUMENT, "unknown dtype %d", dtype);
  int rc = check_fused_args(P, x, g, m, delta, snap_next, sgd, alpha, mode);
  if (rc) return rc;
  if (P == 1)  // no peers: the streaming local step with the snapshot store fused in
    return sgd_step_snapshot(dtype, x[0], g[0], m ? m[0] : nullptr, delta ? delta[0] : nullptr, snap_next[0], n, sgd,
                             nonfinite, stream);
  algo = resolve_algo(algo, P, n * elem_bytes(dtype));
  if (algo != LASGD_ALGO_ONESHOT && algo != LASGD_ALGO_TWOSHOT) return fail(LASGD_ERR_INVALID_ARGUMENT, "algo %d", algo);
  if (algo == LASGD_ALGO_TWOSHOT && !xbars) return fail(LASGD_ERR_INVALID_ARGUMENT, "two-shot needs per-rank mean buffers");
  if (n == 0) return LASGD_OK;
  // P == 1 (local step + snapshot) fits 3 CTAs per SM (<= 85 registers); otherwise 2
  if (nblocks <= 0) nblocks = (P == 1 ? 3 : 2) * num_sms();
  CommArgs a;
  memset(&a, 0, sizeof(a));
  for (int q = 0; q < P; ++q) {
    if (!snaps[q] || !aligned16(snaps[q])) return fail(LASGD_ERR_INVALID_ARGUMENT, "snapshot %d null or unaligned", q);
    a.snap[q] = reinterpret_cast<const char*>(snaps[q]);
    if (xbars) {
      if (!xbars[q] || !aligned16(xbars[q])) return fail(LASGD_ERR_INVALID_ARGUMENT, "mean buffer %d null or unaligned", q);
      a.xbar[q] = reinterpret_cast<char*>(xbars[q]);
    }
  }
  a.n = n;
  a.nblocks = nblocks;
  a.skip_signal_phase = -1;
  a.nonfinite = nonfinite;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int nph = algo == LASGD_ALGO_TWOSHOT ? 2 : 1;
  for (int ph = 0; ph < nph; ++ph) {  // two-shot: reduce-scatter launch, then the pull launch
    a.phases = algo == LASGD_ALGO_TWOSHOT ? (1 << ph) : 3;
    if (dtype == LASGD_F32)
      rc = launch_fused<float, true>(P, a, make_fused<float>(P, x, g, m, delta, snap_next, sgd, alpha, mode),
                                     dim3(nblocks, P), 256, s, algo);
    else
      rc = launch_fused<double, true>(P, a, make_fused<double>(P, x, g, m, delta, snap_next, sgd, alpha, mode),
                                      dim3(nblocks, P), 256, s, algo);
    if (rc) return rc;
  }
  return LASGD_OK;
}

extern "C" size_t lasgd_push_stage_elems(size_t n, int P, int dtype) { return push_stage_elems(n, P, dtype); }

// K8 over P virtual ranks on one device: (init) staging launch, then phase A for every
// rank, then phase B for every rank (stream order replaces the rank-level barriers).
extern "C" int lasgd_fused_push_virtual(int P, void* const* x, const void* const* g, void* const* m,
                                        void* const* delta, const void* const* snaps, void* const* snap_next,
                                        void* const* xbars, void* const* stages, int cur, int init, size_t n,
                                        int dtype, const lasgd_sgd_params* sgd, double alpha, int mode, int nblocks,
                                        unsigned long long* nonfinite, void* stream) {
  if (P < 2 || P > kMaxR) return fail(LASGD_ERR_UNSUPPORTED, "push round needs 2 <= P <= %d", kMaxR);
  if (!x || !g || !snaps || !snap_next || !xbars || !stages) return fail(LASGD_ERR_INVALID_ARGUMENT, "null pointer array");
  if (dtype != LASGD_F32 && dtype != LASGD_F64) return fail(LASGD_ERR_INVALID_ARGUMENT, "unknown dtype %d", dtype);
  if (cur != 0 && cur != 1) return fail(LASGD_ERR_INVALID_ARGUMENT, "parity %d", cur);
  int rc = check_fused_args(P, x, g, m, delta, snap_next, sgd, alpha, mode);
  if (rc) return rc;
  if (n == 0) return LASGD_OK;
  if (nblocks <= 0) nblocks = 2 * num_sms();
  CommArgs a;
  memset(&a, 0, sizeof(a));
  for (int q = 0; q < P; ++q) {
    if (!snaps[q] || !xbars[q] || !stages[q] || !aligned16(snaps[q]) || !aligned16(xbars[q]) || !aligned16(stages[q]))
      return fail(LASGD_ERR_INVALID_ARGUMENT, "rank %d buffers null or unaligned", q);
    a.snap[q] = reinterpret_cast<const char*>(snaps[q]);
    a.xbar[q] = reinterpret_cast<char*>(xbars[q]);
    a.stage[q] = reinterpret_cast<char*>(stages[q]);
  }
  a.n = n;
  a.nblocks = nblocks;
  a.skip_signal_phase = -1;
  a.stage_elems = push_stage_elems(n, P, dtype);
  a.cur = cur;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  for (int ph : {4, 1, 2}) {
    if (ph == 4 && !init) continue;
    a.phases = ph;
    a.nonfinite = ph == 4 ? nullptr : nonfinite;
    if (dtype == LASGD_F32)
      rc = launch_push<float, true>(P, a, make_fused<float>(P, x, g, m, delta, snap_next, sgd, alpha, mode),
                                    dim3(nblocks, P), 256, s);
    else
      rc = launch_push<double, true>(P, a, make_fused<double>(P, x, g, m, delta, snap_next, sgd, alpha, mode),
                                     dim3(nblocks, P), 256, s);
    if (rc) return rc;
  }
  return LASGD_OK;
}

// ====================================================================== communicator
struct lasgd_comm {
  int rank = 0, world = 1, device = 0, dtype = LASGD_F32;
  size_t n = 0, elem = 4;
  int nblocks = 96, threads = 256;
  long long timeout_ns = 30LL * 1000000000LL;
  long long fault_seq = -1;
  int fault_phase = 0;
  char* base = nullptr;
  size_t region_bytes = 0, off_snap[2] = {0, 0}, off_xbar = 0, off_stage = 0, stage_elems = 0;
  int push_slot = -1;            // staging parity that holds the current contributions (-1: none)
  unsigned long long last_push = 0;  // launch whose end signals certify them
  unsigned long long end_seq = 0;    // last launch that raised end signals (K7 one-shot, K8)
  unsigned int* end_ctr = nullptr;   // [kDoneSlots] rank-level end-signal counters
  char* peer_base[kMaxR] = {nullptr};
  bool opened = false;
  bool poisoned = false;
  uint32_t* status_host = nullptr;  // ST_WORDS uint32 + u64 done_seq (host-mapped)
  uint32_t* status_dev = nullptr;
  unsigned long long* done_host = nullptr;
  unsigned long long* done_dev = nullptr;
  unsigned int* done_ctr = nullptr;
  unsigned long long* tile_ctr = nullptr;  // [kDoneSlots][2] work queues
  unsigned int* mid_ctr = nullptr;         // [kDoneSlots] rank-level barrier counters
  unsigned long long* trace_buf = nullptr;  // [kMaxB][4] globaltimer stamps of the last traced launch
  bool trace_on = false;
  bool gate = false;           // launch k_gate ahead of every all-reduce (side-stream use)
  unsigned long long seq = 0;  // launches issued
  cudaEvent_t ev[kEvents];
  int nev = 0;
};

static size_t round_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

extern "C" int lasgd_comm_create(int rank, int world, int device, size_t n, int dtype, const lasgd_comm_config* cfg,
                                 lasgd_comm** out) {
  if (!out) return fail(LASGD_ERR_INVALID_ARGUMENT, "null out");
  *out = nullptr;
  if (world < 1 || world > kMaxR) return fail(LASGD_ERR_UNSUPPORTED, "world size %d outside [1, %d]", world, kMaxR);
  if (rank < 0 || rank >= world) return fail(LASGD_ERR_INVALID_ARGUMENT, "rank %d outside [0, %d)", rank, world);
  if (n < 1) return fail(LASGD_ERR_INVALID_ARGUMENT, "d must be positive");
  if (dtype != LASGD_F32 && dtype != LASGD_F64) return fail(LASGD_ERR_INVALID_ARGUMENT, "unknown dtype %d", dtype);
  lasgd_comm* c = new lasgd_comm();
  c->rank = rank;
  c->world = world;
  c->device = device;
  c->dtype = dtype;
  c->n = n;
  c->elem = elem_bytes(dtype);
  if (cfg) {
    if (cfg->nblocks > 0) c->nblocks = cfg->nblocks;
    if (cfg->threads > 0) c->threads = cfg->threads;
    if (cfg->timeout_s > 0) c->timeout_ns = (long long)(cfg->timeout_s * 1e9);
    c->fault_seq = cfg->fault_seq;
    c->fault_phase = cfg->fault_phase;
  }
  if (c->nblocks < 1 || c->nblocks > kMaxB) {
    int nb = c->nblocks;
    delete c;
    return fail(LASGD_ERR_INVALID_ARGUMENT, "nblocks=%d outside [1, %d]", nb, kMaxB);
  }
  if (c->threads < 64 || c->threads > 256 || c->threads % 32) {
    int t = c->threads;
    delete c;
    return fail(LASGD_ERR_INVALID_ARGUMENT, "threads=%d must be a multiple of 32 in [64, 256]", t);
  }
  DeviceGuard g(device);
  const size_t bytes = n * c->elem;
  c->off_snap[0] = round_up(kPadBytes, 4096);
  c->off_snap[1] = round_up(c->off_snap[0] + bytes, 4096);
  c->off_xbar = round_up(c->off_snap[1] + bytes, 4096);
  // staging for the push round: [2 parities][world sources][stage_elems]
  c->stage_elems = world > 1 ? push_stage_elems(n, world, dtype) : 0;
  c->off_stage = round_up(c->off_xbar + bytes, 4096);
  c->region_bytes = round_up(c->off_stage + 2 * (size_t)world * c->stage_elems * c->elem, (size_t)2 << 20);
  cudaError_t e = cudaMalloc(&c->base, c->region_bytes);
  if (e != cudaSuccess) {
    delete c;
    return cuda_fail(e, "cudaMalloc(comm region)");
  }
  e = cudaMemset(c->base, 0, c->region_bytes);
  if (e == cudaSuccess) e = cudaHostAlloc((void**)&c->status_host, 4096, cudaHostAllocMapped);
  if (e == cudaSuccess) {
    memset(c->status_host, 0, 4096);
    e = cudaHostGetDevicePointer((void**)&c->status_dev, c->status_host, 0);
  }
  if (e == cudaSuccess) e = cudaMalloc(&c->done_ctr, kDoneSlots * sizeof(unsigned int));
  if (e == cudaSuccess) e = cudaMalloc(&c->tile_ctr, 2 * kDoneSlots * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(c->tile_ctr, 0, 2 * kDoneSlots * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMalloc(&c->mid_ctr, kDoneSlots * sizeof(unsigned int));
  if (e == cudaSuccess) e = cudaMemset(c->mid_ctr, 0, kDoneSlots * sizeof(unsigned int));
  if (e == cudaSuccess) e = cudaMalloc(&c->end_ctr, kDoneSlots * sizeof(unsigned int));
  if (e == cudaSuccess) e = cudaMemset(c->end_ctr, 0, kDoneSlots * sizeof(unsigned int));
  if (e == cudaSuccess) e = cudaMemset(c->done_ctr, 0, kDoneSlots * sizeof(unsigned int));
  if (e == cudaSuccess) e = cudaMalloc(&c->trace_buf, (size_t)kMaxB * 4 * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(c->trace_buf, 0, (size_t)kMaxB * 4 * sizeof(unsigned long long));
  for (int i = 0; e == cudaSuccess && i < kEvents; ++i) {
    e = cudaEventCreateWithFlags(&c->ev[i], cudaEventDisableTiming);
    if (e == cudaSuccess) c->nev++;
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    int rc = cuda_fail(e, "lasgd_comm_create");
    lasgd_comm_destroy(c);
    return rc;
  }
  c->done_host = reinterpret_cast<unsigned long long*>(c->status_host + 64);
  c->done_dev = reinterpret_cast<unsigned long long*>(c->status_dev + 64);
  c->peer_base[rank] = c->base;
  *out = c;
  return LASGD_OK;
}

extern "C" int lasgd_comm_ipc_handle(lasgd_comm* c, void* out) {
  if (!c || !out) return fail(LASGD_ERR_INVALID_ARGUMENT, "null argument");
  static_assert(sizeof(cudaIpcMemHandle_t) == LASGD_IPC_HANDLE_BYTES, "IPC handle size");
  DeviceGuard g(c->device);
  cudaIpcMemHandle_t h;
  LASGD_CUDA_TRY(cudaIpcGetMemHandle(&h, c->base));
  memcpy(out, &h, sizeof(h));
  return LASGD_OK;
}

extern "C" int lasgd_comm_open(lasgd_comm* c, const void* handles) {
  if (!c || !handles) return fail(LASGD_ERR_INVALID_ARGUMENT, "null argument");
  if (c->opened) return fail(LASGD_ERR_STATE, "communicator already opened");
  DeviceGuard g(c->device);
  for (int r = 0; r < c->world; ++r) {
    if (r == c->rank) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, (const char*)handles + (size_t)r * LASGD_IPC_HANDLE_BYTES, sizeof(h));
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle(peer region)");
    c->peer_base[r] = (char*)p;
  }
  c->opened = true;
  return LASGD_OK;
}

extern "C" int lasgd_comm_buffer(lasgd_comm* c, int which, void** ptr) {
  if (!c || !ptr) return fail(LASGD_ERR_INVALID_ARGUMENT, "null argument");
  if (which == 0 || which == 1) *ptr = c->base + c->off_snap[which];
  else if (which == 2) *ptr = c->base + c->off_xbar;
  else return fail(LASGD_ERR_INVALID_ARGUMENT, "buffer index %d", which);
  return LASGD_OK;
}

extern "C" int lasgd_comm_resolve_algo(lasgd_comm* c, int algo) {
  if (!c) return fail(LASGD_ERR_INVALID_ARGUMENT, "null comm");
  return resolve_algo(algo, c->world, c->n * c->elem);
}

extern "C" int lasgd_comm_resolve_fused_algo(lasgd_comm* c, int algo) {
  if (!c) return fail(LASGD_ERR_INVALID_ARGUMENT, "null comm");
  return resolve_fused_algo(algo, c->world, c->n * c->elem);
}

// Latest launch each peer has reached, from this rank's signal pad: the entry flags
// of the first `rows` CTA slots and the gate slots (a gated launch announces itself
// in its gate before its wide kernel writes entry flags).  Copied on a private
// non-blocking stream, so it never waits behind the caller's (possibly stalled)
// streams.  out[q] = epoch of peer q's latest launch (u32, wrapping compare).
static int read_peer_epochs(lasgd_comm* c, int rows, uint32_t* out) {
  static thread_local uint32_t* host = nullptr;
  static thread_local cudaStream_t s = nullptr;
  const size_t entry_words = (size_t)kMaxB * kMaxR;
  if (!host) LASGD_CUDA_TRY(cudaHostAlloc((void**)&host, (entry_words + kMaxR) * sizeof(uint32_t), cudaHostAllocDefault));
  if (!s) LASGD_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  const size_t gate_word = (size_t)2 * kMaxB * kMaxR + (size_t)2 * kMaxR;  // k_gate's rank-level slots
  LASGD_CUDA_TRY(cudaMemcpyAsync(host, c->base, (size_t)rows * kMaxR * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  LASGD_CUDA_TRY(cudaMemcpyAsync(host + entry_words, c->base + gate_word * sizeof(uint32_t), kMaxR * sizeof(uint32_t),
                                 cudaMemcpyDeviceToHost, s));
  LASGD_CUDA_TRY(cudaStreamSynchronize(s));
  for (int q = 0; q < kMaxR; ++q) {
    uint32_t best = host[entry_words + q];
    for (int b = 0; b < rows; ++b) {
      const uint32_t v = host[(size_t)b * kMaxR + q];
      if ((int32_t)(v - best) > 0) best = v;
    }
    out[q] = best;
  }
  return LASGD_OK;
}

// Highest launch sequence number any peer has started (drain of adaptive runs).
extern "C" int lasgd_comm_peer_max_seq(lasgd_comm* c, unsigned long long* out) {
  if (!c || !out) return fail(LASGD_ERR_INVALID_ARGUMENT, "null argument");
  DeviceGuard g(c->device);
  uint32_t ep[kMaxR];
  int rc = read_peer_epochs(c, kMaxB, ep);
  if (rc) return rc;
  uint32_t best = 0;
  for (int q = 0; q < c->world; ++q)
    if (q != c->rank && ep[q] > best) best = ep[q];
  *out = best;
  return LASGD_OK;
}

extern "C" int lasgd_comm_set_gate(lasgd_comm* c, int on) {
  if (!c) return fail(LASGD_ERR_INVALID_ARGUMENT, "null comm");
  c->gate = on != 0;
  return LASGD_OK;
}

extern "C" int lasgd_comm_peers_ahead(lasgd_comm* c, unsigned long long seq) {
  if (!c) return fail(LASGD_ERR_INVALID_ARGUMENT, "null comm");
  if (c->world <= 1) return 0;
  DeviceGuard g(c->device);
  // CTA 0 of every K2/K3 launch writes its entry flag first, so the CTA-0 row (plus
  // the gate row) holds each peer's latest launch: 64 bytes instead of the whole pad
  uint32_t ep[kMaxR];
  int rc = read_peer_epochs(c, 1, ep);
  if (rc) return rc;
  for (int q = 0; q < c->world; ++q)
    if (q != c->rank && (int32_t)(ep[q] - (uint32_t)seq) > 0) return 1;
  return 0;
}

extern "C" int lasgd_comm_invalidate_staging(lasgd_comm* c) {
  if (!c) return fail(LASGD_ERR_INVALID_ARGUMENT, "null comm");
  c->push_slot = -1;
  return LASGD_OK;
}

extern "C" int lasgd_comm_launches(lasgd_comm* c, unsigned long long* out) {
  if (!c || !out) return fail(LASGD_ERR_INVALID_ARGUMENT, "null argument");
  *out = c->seq;
  return LASGD_OK;
}

extern "C" int lasgd_comm_info(lasgd_comm* c, int* rank, int* world, void** xbar) {
  if (!c) return fail(LASGD_ERR_INVALID_ARGUMENT, "null comm");
  if (rank) *rank = c->rank;
  if (world) *world = c->world;
  if (xbar) *xbar = c->base + c->off_xbar;
  return LASGD_OK;
}

extern "C" int lasgd_comm_set_trace(lasgd_comm* c, int on) {
  if (!c) return fail(LASGD_ERR_INVALID_ARGUMENT, "null comm");
  c->trace_on = on != 0;
  return LASGD_OK;
}

extern "C" int lasgd_comm_read_trace(lasgd_comm* c, unsigned long long* out, int max_ctas) {
  if (!c || !out) return fail(LASGD_ERR_INVALID_ARGUMENT, "null argument");
  const int nb = max_ctas < c->nblocks ? max_ctas : c->nblocks;
  DeviceGuard g(c->device);
  LASGD_CUDA_TRY(cudaDeviceSynchronize());
  LASGD_CUDA_TRY(cudaMemcpy(out, c->trace_buf, (size_t)nb * 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  return nb;
}

extern "C" int lasgd_comm_set_nblocks(lasgd_comm* c, int nblocks) {
  if (!c) return fail(LASGD_ERR_INVALID_ARGUMENT, "null comm");
  if (nblocks < 1 || nblocks > kMaxB) return fail(LASGD_ERR_INVALID_ARGUMENT, "nblocks=%d outside [1, %d]", nblocks, kMaxB);
  c->nblocks = nblocks;
  return LASGD_OK;
}

// Common launch preparation: validates the communicator state, assigns the next
// sequence number (the epoch of every flag written by this launch) and fills the
// pointer tables for snapshot slot `snap_slot`.
static int prepare_launch(lasgd_comm* c, int snap_slot, CommArgs& a, unsigned long long& s) {
  if (!c) return fail(LASGD_ERR_INVALID_ARGUMENT, "null comm");
  if (!c->opened && c->world > 1) return fail(LASGD_ERR_STATE, "lasgd_comm_open has not been called");
  if (snap_slot != 0 && snap_slot != 1) return fail(LASGD_ERR_INVALID_ARGUMENT, "snapshot slot %d", snap_slot);
  if (c->poisoned || c->status_host[ST_ERR] != ERR_NONE) {
    c->poisoned = true;
    return fail(LASGD_ERR_COLLECTIVE, "communicator failed earlier; re-create it");
  }
  s = ++c->seq;
  memset(&a, 0, sizeof(a));
  for (int r = 0; r < c->world; ++r) {
    a.snap[r] = c->peer_base[r] + c->off_snap[snap_slot];
    a.xbar[r] = c->peer_base[r] + c->off_xbar;
    a.pad[r] = reinterpret_cast<uint32_t*>(c->peer_base[r]);
  }
  a.n = c->n;
  a.rank = c->rank;
  a.nblocks = c->nblocks;
  a.epoch = (uint32_t)s;
  a.phases = 3;
  a.timeout_ns = c->timeout_ns;
  a.skip_signal_phase = -1;
  if ((long long)s == c->fault_seq) {
    a.skip_signal_phase = c->fault_phase;
    // collective.py:271-279: the faulting round fails on every rank, this one included
    uint32_t* st = c->status_host;
    st[ST_PEER] = c->rank;
    st[ST_PHASE] = c->fault_phase;
    st[ST_BLOCK] = 0;
    st[ST_SEQ_LO] = (uint32_t)(s & 0xffffffffu);
    st[ST_SEQ_HI] = (uint32_t)(s >> 32);
    st[ST_RANK] = c->rank;
    __atomic_store_n(&st[ST_ERR], (uint32_t)ERR_INJECTED, __ATOMIC_SEQ_CST);
  }
  a.status = c->status_dev;
  a.done_ctr = c->done_ctr;
  a.tile_ctr = c->tile_ctr + 2 * (s % kDoneSlots);
  a.mid_ctr = c->mid_ctr + (s % kDoneSlots);
  a.end_ctr = c->end_ctr + (s % kDoneSlots);
  for (int r = 0; r < c->world; ++r) a.stage[r] = c->peer_base[r] + c->off_stage;
  a.stage_elems = c->stage_elems;
  a.cur = snap_slot;
  a.done_seq = c->done_dev;
  a.seq = s;
  a.nonfinite = nullptr;
  a.trace = c->trace_on ? c->trace_buf : nullptr;
  return LASGD_OK;
}

extern "C" int lasgd_comm_allreduce(lasgd_comm* c, int snap_slot, int algo, void* stream, unsigned long long* seq) {
  if (!c) return fail(LASGD_ERR_INVALID_ARGUMENT, "null comm");
  algo = resolve_algo(algo, c->world, c->n * c->elem);
  if (algo != LASGD_ALGO_ONESHOT && algo != LASGD_ALGO_TWOSHOT) return fail(LASGD_ERR_INVALID_ARGUMENT, "algo %d", algo);
  DeviceGuard g(c->device);
  CommArgs a;
  unsigned long long s = 0;
  int rc = prepare_launch(c, snap_slot, a, s);
  if (rc) return rc;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  c->push_slot = -1;  // the caller rewrote a snapshot slot: staged push contributions are stale
  if (c->gate && c->world > 1 && (rc = launch_gate(c->world, a, cs))) return rc;
  rc = launch_any(c->dtype, false, algo, c->world, a, dim3(c->nblocks, 1), c->threads, cs);
  if (rc) return rc;
  LASGD_CUDA_TRY(cudaEventRecord(c->ev[s % kEvents], cs));
  if (seq) *seq = s;
  return LASGD_OK;
}

extern "C" int lasgd_comm_fused_round(lasgd_comm* c, int snap_slot, int algo, void* x, const void* g, void* m,
                                      void* delta, const lasgd_sgd_params* sgd, double alpha, int mode, int nblocks,
                                      unsigned long long* nonfinite, void* stream, unsigned long long* seq) {
  if (!c) return fail(LASGD_ERR_INVALID_ARGUMENT, "null comm");
  algo = resolve_fused_algo(algo, c->world, c->n * c->elem);
  const bool push = algo == LASGD_ALGO_PUSH;
  if (!push && algo != LASGD_ALGO_ONESHOT && algo != LASGD_ALGO_TWOSHOT)
    return fail(LASGD_ERR_INVALID_ARGUMENT, "algo %d", algo);
  void* xs[1] = {x};
  const void* gs[1] = {g};
  void* ms[1] = {m};
  void* ds[1] = {delta};
  void* ns[1] = {nullptr};
  if (snap_slot != 0 && snap_slot != 1) return fail(LASGD_ERR_INVALID_ARGUMENT, "snapshot slot %d", snap_slot);
  ns[0] = c->base + c->off_snap[1 - snap_slot];
  int rc = check_fused_args(1, xs, gs, m ? ms : nullptr, delta ? ds : nullptr, ns, sgd, alpha, mode);
  if (rc) return rc;
  // default: 2 CTAs per SM (the fused pass owns the GPU at a round boundary); every
  // rank computes the same value, so the per-CTA flag slots line up
  if (nblocks <= 0) nblocks = 2 * num_sms() <= kMaxB ? 2 * num_sms() : kMaxB;
  if (nblocks > kMaxB) return fail(LASGD_ERR_INVALID_ARGUMENT, "nblocks=%d > %d", nblocks, kMaxB);
  DeviceGuard dg(c->device);
  CommArgs a;
  unsigned long long s = 0;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  if (push) {
    auto fl = make_fused<float>(1, xs, gs, m ? ms : nullptr, delta ? ds : nullptr, ns, sgd, alpha, mode);
    auto fd = make_fused<double>(1, xs, gs, m ? ms : nullptr, delta ? ds : nullptr, ns, sgd, alpha, mode);
    if (c->push_slot != snap_slot) {
      // first push round (or after other use of the slots): stage the current snapshot's
      // chunks at their owners (one extra launch, certified by its end signals)
      rc = prepare_launch(c, snap_slot, a, s);
      if (rc) return rc;
      a.nblocks = nblocks;
      a.phases = 4;
      rc = c->dtype == LASGD_F32 ? launch_push<float, false>(c->world, a, fl, dim3(nblocks, 1), c->threads, cs)
                                 : launch_push<double, false>(c->world, a, fd, dim3(nblocks, 1), c->threads, cs);
      if (rc) return rc;
      LASGD_CUDA_TRY(cudaEventRecord(c->ev[s % kEvents], cs));
      c->last_push = s;
      c->end_seq = s;
    }
    rc = prepare_launch(c, snap_slot, a, s);
    if (rc) return rc;
    a.nblocks = nblocks;
    a.nonfinite = nonfinite;
    a.phases = 3;
    a.prev_push = (uint32_t)c->last_push;
    rc = c->dtype == LASGD_F32 ? launch_push<float, false>(c->world, a, fl, dim3(nblocks, 1), c->threads, cs)
                               : launch_push<double, false>(c->world, a, fd, dim3(nblocks, 1), c->threads, cs);
    if (rc) return rc;
    c->last_push = s;
    c->end_seq = s;
    c->push_slot = 1 - snap_slot;
    LASGD_CUDA_TRY(cudaEventRecord(c->ev[s % kEvents], cs));
    if (seq) *seq = s;
    return LASGD_OK;
  }
  rc = prepare_launch(c, snap_slot, a, s);
  if (rc) return rc;
  a.nblocks = nblocks;
  a.nonfinite = nonfinite;
  if (algo == LASGD_ALGO_ONESHOT && c->end_seq != 0 && c->end_seq + 1 == s) a.prev_end = (uint32_t)c->end_seq;
  c->push_slot = -1;  // this round writes the next snapshot without staging it
  if (c->dtype == LASGD_F32)
    rc = launch_fused<float, false>(c->world, a, make_fused<float>(1, xs, gs, m ? ms : nullptr, delta ? ds : nullptr, ns, sgd, alpha, mode), dim3(nblocks, 1), c->threads, cs, algo);
  else
    rc = launch_fused<double, false>(c->world, a, make_fused<double>(1, xs, gs, m ? ms : nullptr, delta ? ds : nullptr, ns, sgd, alpha, mode), dim3(nblocks, 1), c->threads, cs, algo);
  if (rc) return rc;
  c->end_seq = algo == LASGD_ALGO_ONESHOT ? s : 0;  // the one-shot K7 raises end signals
  LASGD_CUDA_TRY(cudaEventRecord(c->ev[s % kEvents], cs));
  if (seq) *seq = s;
  return LASGD_OK;
}

extern "C" int lasgd_comm_query(lasgd_comm* c, unsigned long long seq) {
  if (!c) return fail(LASGD_ERR_INVALID_ARGUMENT, "null comm");
  const uint32_t err = __atomic_load_n(&c->status_host[ST_ERR], __ATOMIC_ACQUIRE);
  if (err != ERR_NONE) {
    const unsigned long long fs =
        (unsigned long long)c->status_host[ST_SEQ_LO] | ((unsigned long long)c->status_host[ST_SEQ_HI] << 32);
    if (seq >= fs) {
      c->poisoned = true;
      char buf[256];
      lasgd_comm_diagnostic(c, buf, sizeof(buf));
      return fail(LASGD_ERR_COLLECTIVE, "%s", buf);
    }
  }
  if (seq == 0 || seq > c->seq) return fail(LASGD_ERR_INVALID_ARGUMENT, "unknown launch %llu", seq);
  const unsigned long long done = __atomic_load_n(c->done_host, __ATOMIC_ACQUIRE);
  return done >= seq ? 1 : 0;
}

extern "C" int lasgd_comm_stream_wait(lasgd_comm* c, unsigned long long seq, void* stream) {
  if (!c) return fail(LASGD_ERR_INVALID_ARGUMENT, "null comm");
  if (seq == 0 || seq > c->seq) return fail(LASGD_ERR_INVALID_ARGUMENT, "unknown launch %llu", seq);
  DeviceGuard g(c->device);
  LASGD_CUDA_TRY(cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(stream), c->ev[seq % kEvents], 0));
  return LASGD_OK;
}

extern "C" int lasgd_comm_wait(lasgd_comm* c, unsigned long long seq, double timeout_s) {
  struct timespec t0, t;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  for (;;) {
    int rc = lasgd_comm_query(c, seq);
    if (rc != 0) return rc;
    clock_gettime(CLOCK_MONOTONIC, &t);
    double el = (t.tv_sec - t0.tv_sec) + 1e-9 * (t.tv_nsec - t0.tv_nsec);
    if (timeout_s >= 0 && el > timeout_s) return fail(LASGD_ERR_TIMEOUT, "launch %llu not complete after %.3fs", seq, el);
    struct timespec ns = {0, 20000};
    nanosleep(&ns, nullptr);
  }
}

extern "C" int lasgd_comm_diagnostic(lasgd_comm* c, char* buf, size_t len) {
  if (!c || !buf || !len) return fail(LASGD_ERR_INVALID_ARGUMENT, "null argument");
  const uint32_t* st = c->status_host;
  const unsigned long long fs = (unsigned long long)st[ST_SEQ_LO] | ((unsigned long long)st[ST_SEQ_HI] << 32);
  const char* phase = st[ST_PHASE] == 0 ? "entry" : "mid";
  switch (st[ST_ERR]) {
    case ERR_NONE: snprintf(buf, len, "ok"); break;
    case ERR_TIMEOUT:
      snprintf(buf, len, "rank %u timed out waiting for rank %u at the %s barrier of launch %llu (CTA %u)", st[ST_RANK],
               st[ST_PEER], phase, fs, st[ST_BLOCK]);
      break;
    case ERR_INJECTED:
      snprintf(buf, len, "injected fault in launch %llu at the %s barrier (rank %u)", fs, phase, st[ST_RANK]);
      break;
    default: snprintf(buf, len, "unknown failure code %u", st[ST_ERR]);
  }
  return LASGD_OK;
}

extern "C" unsigned long long lasgd_comm_bytes_per_node(lasgd_comm* c, int algo) {
  if (!c || c->world <= 1) return 0;
  algo = resolve_algo(algo, c->world, c->n * c->elem);
  const unsigned long long B = (unsigned long long)c->n * c->elem;
  if (algo == LASGD_ALGO_ONESHOT) return (unsigned long long)(c->world - 1) * B;
  return lasgd_bytes_per_node(c->n, c->world, (int)c->elem, -1);
}

extern "C" int lasgd_comm_destroy(lasgd_comm* c) {
  if (!c) return LASGD_OK;
  DeviceGuard g(c->device);
  cudaDeviceSynchronize();
  for (int r = 0; r < c->world; ++r)
    if (r != c->rank && c->peer_base[r]) cudaIpcCloseMemHandle(c->peer_base[r]);
  for (int i = 0; i < c->nev; ++i) cudaEventDestroy(c->ev[i]);
  if (c->done_ctr) cudaFree(c->done_ctr);
  if (c->tile_ctr) cudaFree(c->tile_ctr);
  if (c->mid_ctr) cudaFree(c->mid_ctr);
  if (c->end_ctr) cudaFree(c->end_ctr);
  if (c->trace_buf) cudaFree(c->trace_buf);
  if (c->status_host) cudaFreeHost(c->status_host);
  if (c->base) cudaFree(c->base);
  delete c;
  return LASGD_OK;
}
