// Mean all-reduce kernels: K2 one-shot and K3 two-shot (ring-order sum, bit-identical on every rank).
// Part of the communicator translation unit (lasgd_comm.cu includes it); see the
// overview there.
#ifndef LASGD_COMM_ALLREDUCE_CUH
#define LASGD_COMM_ALLREDUCE_CUH

#include "comm_device.cuh"

namespace lasgd {

// ------------------------------------------------------------------ one-shot (K2)
template <typename T, int P, bool VIRTUAL, int U>
__global__ void __launch_bounds__(256, 2) k_oneshot(CommArgs a) {
  pdl_entry();
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
  pdl_entry();
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

}  // namespace lasgd

#endif  // LASGD_COMM_ALLREDUCE_CUH
