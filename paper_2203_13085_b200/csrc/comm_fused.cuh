// Fused round kernels (K7): local step + NVLink mean + pull + next snapshot in one pass, one-shot and two-shot forms.
// Part of the communicator translation unit (lasgd_comm.cu includes it); see the
// overview there.
#ifndef LASGD_COMM_FUSED_CUH
#define LASGD_COMM_FUSED_CUH

#include "comm_allreduce.cuh"  // chunk_tiles, ordered_sum, tile loops

namespace lasgd {

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
  int mode;  // 0 pull, 1 reference finalize (delta), 2 SGD-AR (step with the mean of the slots)
};

template <typename T, int P, bool VIRTUAL, int U>
__global__ void __launch_bounds__(256, (P == 1 ? 3 : 2)) k_fused_round(CommArgs a, FusedRound<T> f) {
  pdl_entry();
  constexpr int W = Pack<T>::W;
  const int rank = VIRTUAL ? (int)blockIdx.y : a.rank;
  const int vr = VIRTUAL ? (int)blockIdx.y : 0;
  const int b = blockIdx.x;
  bool ok = true;
  dyn_comm_begin(a);
  const SgdCoef<T> cf = ccoef(a, f.c);
  trace_mark(a, b, 0);
  // Entry: every peer's snapshot slot must be final and every peer must be done reading
  // this rank's other slot.  When the previous launch was a round that raised end
  // signals (K7 one-shot or K8), those certify both and were raised before the peers
  // even launched this kernel; otherwise the per-CTA entry barrier.
  if (!VIRTUAL && P > 1) ok = cprev_end(a) ? rank_wait<P>(a, 1, cprev_end(a), b, rank) : cta_barrier<P>(a, 0, b, rank);
  trace_mark(a, b, 1);
  unsigned bad = 0;
  if (ok) {
    const size_t n = a.n;
    size_t bnd[P + 1];
#pragma unroll
    for (int c = 0; c <= P; ++c) bnd[c] = chunk_bound_local(a, P, c);
    const T* src[P];
#pragma unroll
    for (int q = 0; q < P; ++q) src[q] = reinterpret_cast<const T*>(csnap(a, q));
    T* const x = f.x[vr];
    const T* const g = f.g[vr];
    T* const m = f.m[vr];
    T* const dl = f.delta[vr];
    T* const sn = a.adv.rd ? reinterpret_cast<T*>(const_cast<char*>(cslot(a, rank, 1 - ccur(a)))) : f.snap_next[vr];
    const bool load_m = cf.use_mom && !cf.first, load_d = cf.use_delta && !cf.reset;
    const bool store_d = cf.use_delta && (P == 1 || f.mode == 0);  // finalize resets delta
    auto element = [&](T& xv, T gv, T& mv, T& dv, const T (&lane)[P], int cidx) -> T {
      if constexpr (P > 1) {
        if (f.mode == 2) {  // SGD-AR: the local step with the ring-order mean of the gradients
          bad += sgd_elem(cf, xv, mean_div<T, P>(rot_sum<T, P>(lane, cidx)), mv, dv);
          return xv;
        }
      }
      unsigned bb = sgd_elem(cf, xv, gv, mv, dv);
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
          if (f.mode != 2) vg[u] = ld_stream(g + j);
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
          if (cf.use_mom) st_stream(m + j0, vm[u]);
          if (store_d) st_stream(dl + j0, vd[u]);
          if (f.mode != 2) st_stream(sn + j0, vx[u]);
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
        element(xv, f.mode == 2 ? T(0) : g[j], mv, dv, lane, chunk_of<P>(j, bnd));
        x[j] = xv;
        if (cf.use_mom) m[j] = mv;
        if (store_d) dl[j] = dv;
        if (f.mode != 2) sn[j] = xv;
      }
    }
  }
  if (!VIRTUAL && P > 1 && ok) rank_signal<P>(a, 1, cend(a), rank);  // certifies the next round's entry
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
  pdl_entry();
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
  const bool ranged = a.n_glob != 0;  // bucket of a bucketed SGD-AR step
  auto element = [&](T& xv, T gv, T& mv, T& dv, T sv, T zb) {
    if (f.mode == 2) {  // SGD-AR: the local step with the mean gradient
      bad += sgd_elem(f.c, xv, zb, mv, dv);
      return;
    }
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
              if (f.mode != 2) vg[u] = ld_stream(g + j);
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
              // ring-order start: the owner chunk, or for a bucket (sub-range launch) the
              // element's chunk of the whole vector
              const int r0 = ranged ? rot_of<P>(a, j) : rank, r1 = ranged ? rot_of<P>(a, j + W - 1) : rank;
#pragma unroll
              for (int k = 0; k < W; ++k) {
                T lane[P];
#pragma unroll
                for (int q = 0; q < P; ++q) lane[q] = v[u][q].v[k];
                T sv = lane[0];
#pragma unroll
                for (int q = 1; q < P; ++q) sv = (q == rank) ? lane[q] : sv;
                z.v[k] = mean_div<T, P>(rot_sum<T, P>(lane, r0 == r1 ? r0 : rot_of<P>(a, j + k)));
                element(vx[u].v[k], vg[u].v[k], vm[u].v[k], vd[u].v[k], sv, z.v[k]);
              }
              st_plain(own + j, z);
              st_stream(x + j, vx[u]);
              if (f.c.use_mom) st_stream(m + j, vm[u]);
              if (store_d) st_stream(dl + j, vd[u]);
              if (f.mode != 2) st_stream(sn + j, vx[u]);
            }
          }
        }
      });
      if (b == 0) {  // unaligned head / tail elements of the own chunk
        const size_t he = cp0 * W < ce ? cp0 * W : ce;
        const size_t ts = cp1 * W > he ? cp1 * W : he;
        auto scalar = [&](size_t j) {
          const T zb = mean_div<T, P>(ordered_sum<T, P>(src, ranged ? rot_of<P>(a, j) : rank, j));
          own[j] = zb;
          T xv = x[j], mv = load_m ? m[j] : T(0), dv = load_d ? dl[j] : T(0);
          element(xv, f.mode == 2 ? T(0) : g[j], mv, dv, snap_own[j], zb);
          x[j] = xv;
          if (f.c.use_mom) m[j] = mv;
          if (store_d) dl[j] = dv;
          if (f.mode != 2) sn[j] = xv;
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
                if (f.mode != 2) vg[u] = ld_stream(g + j);
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
                if (f.mode != 2) st_stream(sn + j, vx[u]);
              }
            }
          }
        },
        [&](int c, size_t j) {
          T xv = x[j], mv = load_m ? m[j] : T(0), dv = load_d ? dl[j] : T(0);
          element(xv, f.mode == 2 ? T(0) : g[j], mv, dv, f.mode == 0 ? snap_own[j] : T(0),
                  reinterpret_cast<const T*>(a.xbar[c])[j]);
          x[j] = xv;
          if (f.c.use_mom) m[j] = mv;
          if (store_d) dl[j] = dv;
          if (f.mode != 2) sn[j] = xv;
        });
    }
  }
  report_nonfinite(a.nonfinite, bad);
  trace_mark(a, b, 3);
  if (!VIRTUAL) publish_done(a);
}


}  // namespace lasgd

#endif  // LASGD_COMM_FUSED_CUH
