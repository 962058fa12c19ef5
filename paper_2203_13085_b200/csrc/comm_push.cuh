// Push round kernels (K8): data moved by remote stores; staged-chunk form for P >= 3, mirror form for P = 2.
// Part of the communicator translation unit (lasgd_comm.cu includes it); see the
// overview there.
#ifndef LASGD_COMM_PUSH_CUH
#define LASGD_COMM_PUSH_CUH

#include "comm_fused.cuh"

namespace lasgd {

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
//   split (bit 8, P2P, large buffers): phase A does its chunk in two halves and signals
//     each (rank-level rows 0 and 6) instead of the mid barrier; phase B does half 0 of
//     every other chunk once every owner's row 0 is in, then half 1 after row 6 — the
//     second half's mean stores drain while phase B already works.
// Per rank and round: NVLink out 2(P-1)/P*B as posted writes, all reads local.  Same
// element functions and summation order as K7, so results are bit-identical.
template <typename T>
__device__ __forceinline__ T* stage_ptr(const CommArgs& a, int owner, int parity, int src, int P) {
  return reinterpret_cast<T*>(a.stage[owner]) + ((size_t)parity * P + src) * a.stage_elems;
}

template <typename T, int P, bool VIRTUAL, int U>
__global__ void __launch_bounds__(256, 2) k_push_round(CommArgs a, FusedRound<T> f) {
  pdl_entry();
  constexpr int W = Pack<T>::W;
  const int rank = VIRTUAL ? (int)blockIdx.y : a.rank;
  const int vr = VIRTUAL ? (int)blockIdx.y : 0;
  const int b = blockIdx.x;
  const size_t n = a.n;
  dyn_comm_begin(a);
  const SgdCoef<T> cf = ccoef(a, f.c);
  const int cur = ccur(a), nxt = 1 - cur;
  bool ok = true;
  unsigned bad = 0;
  unsigned long long* q0 = ctile(a);
  unsigned long long* q1 = ctile(a) ? ctile(a) + 1 : nullptr;
  // split (phases bit 8, large buffers, P2P only): phase A signals its first half's means
  // before doing the second, so phase B's first half overlaps the second half's drain
  const bool split = !VIRTUAL && (a.phases & 8) != 0;
  unsigned long long* const qA1 = ctile(a) ? ctile(a) + 2 : nullptr;
  unsigned long long* const qB1 = ctile(a) ? ctile(a) + 3 : nullptr;
  const size_t tile = (size_t)kTileIters * U * blockDim.x;
  const T* const snap_own = reinterpret_cast<const T*>(csnap(a, rank));
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
    if (!VIRTUAL) rank_signal<P>(a, 1, cend(a), rank);
  }
  T* const x = f.x[vr];
  const T* const g = f.g[vr];
  T* const m = f.m[vr];
  T* const dl = f.delta[vr];
  T* const sn = a.adv.rd ? reinterpret_cast<T*>(const_cast<char*>(cslot(a, rank, nxt))) : f.snap_next[vr];
  const bool load_m = cf.use_mom && !cf.first, load_d = cf.use_delta && !cf.reset;
  const bool store_d = cf.use_delta && f.mode == 0;
  auto element = [&](T& xv, T gv, T& mv, T& dv, T sv, T zb) {
    unsigned bb = sgd_elem(cf, xv, gv, mv, dv);
    if (f.mode == 0) {
      bb += pull_elem(f.neg_alpha, xv, sv, zb);
    } else {
      xv = add_rn(zb, dv);
      bb += !finite(xv);
    }
    bad += bb;
  };
  if (a.phases & 1) {
    if (!VIRTUAL) ok = rank_wait<P>(a, 1, cprev_push(a), b, rank);
    trace_mark(a, b, 1);
    if (ok) {
      size_t cs, ce, cp0, cp1;
      chunk_packs<T, P>(n, rank, cs, ce, cp0, cp1);
      const size_t base = cs / W * W;  // staging offset origin of the own chunk
      // contribution of rank q to the own chunk: the own snapshot, or q's staged copy
      // (addresses computed per use: P pointers would cost 2P registers at large P)
      const T* const stage0 = stage_ptr<T>(a, rank, cur, 0, P);
      const size_t selems = a.stage_elems;
      auto src = [&](int q, size_t j) -> const T* {
        return q == rank ? snap_own + j : stage0 + (size_t)q * selems + (j - base);
      };
      auto bodyA = [&](size_t p0, size_t p1) {
        for (size_t p = p0 + threadIdx.x; p < p1; p += (size_t)U * blockDim.x) {
          Pack<T> v[U][P], vx[U], vg[U], vm[U], vd[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const size_t pu = p + (size_t)u * blockDim.x;
            if (pu < p1) {
              const size_t j = pu * W;
#pragma unroll
              for (int q = 0; q < P; ++q) v[u][q] = ld_stream(src(q, j));
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
              if (cf.use_mom) st_stream(m + j, vm[u]);
              if (store_d) st_stream(dl + j, vd[u]);
              st_stream(sn + j, vx[u]);
            }
          }
        }
      };
      if (split) {  // half 0's means pushed and signalled before half 1 starts
        const size_t mid = cp0 + (cp1 - cp0) / 2;
        tile_loop(q0, b, a.nblocks, cp0, mid - cp0, tile, bodyA);
        rank_signal<P>(a, 0, cmid(a), rank);
        tile_loop(qA1, b, a.nblocks, mid, cp1 - mid, tile, bodyA);
      } else {
        tile_loop(q0, b, a.nblocks, cp0, cp1 - cp0, tile, bodyA);
      }
      if (b == 0) {  // unaligned head / tail elements of the own chunk
        const size_t he = cp0 * W < ce ? cp0 * W : ce;
        const size_t ts = cp1 * W > he ? cp1 * W : he;
        auto scalar = [&](size_t j) {
          T lane[P];
#pragma unroll
          for (int q = 0; q < P; ++q) lane[q] = *src(q, j);
          const T zb = mean_div<T, P>(rot_sum<T, P>(lane, rank));
#pragma unroll
          for (int q = 0; q < P; ++q)
            if (q != rank) reinterpret_cast<T*>(a.xbar[q])[j] = zb;
          T xv = x[j], mv = load_m ? m[j] : T(0), dv = load_d ? dl[j] : T(0);
          element(xv, g[j], mv, dv, snap_own[j], zb);
          x[j] = xv;
          if (cf.use_mom) m[j] = mv;
          if (store_d) dl[j] = dv;
          sn[j] = xv;
        };
        for (size_t j = cs + threadIdx.x; j < he; j += blockDim.x) scalar(j);
        for (size_t j = ts + threadIdx.x; j < ce; j += blockDim.x) scalar(j);
      }
      if (split) rank_signal<P>(a, 6, caux(a), rank);  // half 1's means pushed
    }
  }
  if (a.phases & 2) {
    if (split) {
      if (ok) ok = rank_wait<P>(a, 0, cepoch(a), b, rank);  // every owner's half-0 means landed
    } else if (!VIRTUAL && ok) {
      ok = rank_barrier<P>(a, b, rank);
    }
    trace_mark(a, b, 2);
    if (ok) {
      const T* zl = reinterpret_cast<const T*>(a.xbar[rank]);  // means pushed by their owners
      auto bodyB =
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
                if (cf.use_mom) st_stream(m + j, vm[u]);
                if (store_d) st_stream(dl + j, vd[u]);
                st_stream(sn + j, vx[u]);
              }
            }
          }
        };
      auto scalarB = [&](int c, size_t j) {
          T xv = x[j], mv = load_m ? m[j] : T(0), dv = load_d ? dl[j] : T(0);
          element(xv, g[j], mv, dv, f.mode == 0 ? snap_own[j] : T(0), zl[j]);
          x[j] = xv;
          if (cf.use_mom) m[j] = mv;
          if (store_d) dl[j] = dv;
          sn[j] = xv;
          stage_ptr<T>(a, c, nxt, rank, P)[soff(c, j)] = xv;
        };
      if (split) {
        // half h of every other chunk, tiles interleaved across owners like chunk_tiles
        auto half_tiles = [&](unsigned long long* qq, int h) {
          auto hr = [&](int c, size_t& lo, size_t& hi) {
            size_t ccs, cce, ccp0, ccp1;
            chunk_packs<T, P>(n, c, ccs, cce, ccp0, ccp1);
            const size_t mid = ccp0 + (ccp1 - ccp0) / 2;
            lo = h ? mid : ccp0;
            hi = h ? ccp1 : mid;
          };
          size_t tmax = 0;
#pragma unroll
          for (int c = 0; c < P; ++c) {
            size_t lo, hi;
            hr(c, lo, hi);
            const size_t tc = (hi - lo + tile - 1) / tile;
            tmax = tc > tmax ? tc : tmax;
          }
          queue_loop(qq, b, a.nblocks, (unsigned long long)tmax * P, [&](unsigned long long t) {
            const int c = (rank + 1 + (int)(t % P)) % P;
            if (c == rank) return;
            size_t lo, hi;
            hr(c, lo, hi);
            const size_t p0 = lo + (size_t)(t / P) * tile;
            if (p0 >= hi) return;
            bodyB(c, p0, p0 + tile < hi ? p0 + tile : hi);
          });
        };
        half_tiles(q1, 0);
        ok = rank_wait<P>(a, 6, cepoch(a), b, rank);  // every owner's half-1 means landed
        if (ok) {
          half_tiles(qB1, 1);
          if (b == 0) {  // unaligned head / tail elements of every other chunk
            for (int c = 0; c < P; ++c) {
              if (c == rank) continue;
              size_t ccs, cce, ccp0, ccp1;
              chunk_packs<T, P>(n, c, ccs, cce, ccp0, ccp1);
              const size_t he = ccp0 * W < cce ? ccp0 * W : cce;
              const size_t ts = ccp1 * W > he ? ccp1 * W : he;
              for (size_t j = ccs + threadIdx.x; j < he; j += blockDim.x) scalarB(c, j);
              for (size_t j = ts + threadIdx.x; j < cce; j += blockDim.x) scalarB(c, j);
            }
          }
        }
      } else {
        chunk_tiles<T, P>(q1, b, a.nblocks, n, rank, true, tile, bodyB, scalarB);
      }
      if (ok && !VIRTUAL) rank_signal<P>(a, 1, cend(a), rank);
    }
  }
  report_nonfinite(a.nonfinite, bad);
  trace_mark(a, b, 3);
  if (!VIRTUAL) publish_done(a);
}

// ------------------------------------------------------------------ push mean (ALGO_PUSH all-reduce)
// K3's result with every byte moved by remote STORES, one cooperative launch, the chunks
// split into two halves so the second half's scatter covers the first half's drain and
// signal latency:
//   scatter half 0: chunk c of my snapshot -> owner c's staging [cur][me] (posted NVLink
//     writes), rank-level signal row 1; scatter half 1 (+ the unaligned head/tail
//     elements), signal row 6;
//   reduce half 0 once every rank's row-1 signal is in: my chunk in ring order from my
//     snapshot + the staged contributions, / P, stored into my xbar and every peer's;
//     reduce half 1 (+ head/tail) once row 6 is in;
//   rank-level mid barrier: every rank's means have landed everywhere.
// Per rank: NVLink out 2(P-1)/P B as stores (as the push round), all loads local.  Four
// work queues (kTileQ).  The staging slots are the push round's: lasgd_comm_allreduce marks
// them as not holding round contributions afterwards.
template <typename T, int P, int U>
__global__ void __launch_bounds__(256, 2) k_push_mean(CommArgs a) {
  constexpr int W = Pack<T>::W;
  const int rank = a.rank;
  const int b = blockIdx.x;
  const size_t n = a.n;
  const int cur = a.cur;
  const T* const snap_own = reinterpret_cast<const T*>(a.snap[rank]);
  unsigned long long* const qt = a.tile_ctr;  // [0], [1]: scatter halves; [2], [3]: reduce halves
  auto q = [&](int k) -> unsigned long long* { return qt ? qt + k : nullptr; };
  const size_t tile = (size_t)kTileIters * U * blockDim.x;
  auto soff = [&](int c, size_t j) { return j - chunk_bound(n, P, c) / W * W; };
  // aligned packs of half h of chunk c
  // split (phases bit 8, large buffers): two halves; otherwise half 0 is the whole chunk
  // and there is no second signal (small buffers: one signal less beats the overlap)
  const bool split = (a.phases & 8) != 0;
  auto half = [&](int c, int h, size_t& lo, size_t& hi) {
    size_t cs, ce, cp0, cp1;
    chunk_packs<T, P>(n, c, cs, ce, cp0, cp1);
    const size_t mid = split ? cp0 + (cp1 - cp0) / 2 : cp1;
    lo = h ? mid : cp0;
    hi = h ? cp1 : mid;
  };
  auto scatter = [&](int h) {
    size_t tmax = 0;
#pragma unroll
    for (int c = 0; c < P; ++c) {
      size_t lo, hi;
      half(c, h, lo, hi);
      const size_t tc = (hi - lo + tile - 1) / tile;
      tmax = tc > tmax ? tc : tmax;
    }
    queue_loop(q(h), b, a.nblocks, (unsigned long long)tmax * P, [&](unsigned long long t) {
      const int c = (rank + 1 + (int)(t % P)) % P;  // every rank starts at a different owner
      if (c == rank) return;
      size_t lo, hi;
      half(c, h, lo, hi);
      const size_t p0 = lo + (size_t)(t / P) * tile;
      if (p0 >= hi) return;
      const size_t p1 = p0 + tile < hi ? p0 + tile : hi;
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
    });
  };
  size_t cs, ce, cp0, cp1;
  chunk_packs<T, P>(n, rank, cs, ce, cp0, cp1);
  const size_t base = cs / W * W;
  const T* const stage0 = stage_ptr<T>(a, rank, cur, 0, P);
  const size_t selems = a.stage_elems;
  auto src = [&](int qq, size_t j) -> const T* {
    return qq == rank ? snap_own + j : stage0 + (size_t)qq * selems + (j - base);
  };
  auto reduce = [&](int h) {
    size_t lo, hi;
    half(rank, h, lo, hi);
    tile_loop(q(2 + h), b, a.nblocks, lo, hi - lo, tile, [&](size_t p0, size_t p1) {
      for (size_t p = p0 + threadIdx.x; p < p1; p += (size_t)U * blockDim.x) {
        Pack<T> v[U][P];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const size_t pu = p + (size_t)u * blockDim.x;
          if (pu < p1) {
#pragma unroll
            for (int qq = 0; qq < P; ++qq) v[u][qq] = ld_stream(src(qq, pu * W));
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
              for (int qq = 0; qq < P; ++qq) lane[qq] = v[u][qq].v[k];
              z.v[k] = mean_div<T, P>(rot_sum<T, P>(lane, rank));
            }
#pragma unroll
            for (int qq = 0; qq < P; ++qq) st_plain(reinterpret_cast<T*>(a.xbar[qq]) + j, z);
          }
        }
      }
    });
  };
  trace_mark(a, b, 0);
  scatter(0);
  if (split) rank_signal<P>(a, 1, a.end_ctr, rank);
  scatter(1);
  if (b == 0) {  // unaligned head / tail elements of every other chunk
    for (int c = 0; c < P; ++c) {
      if (c == rank) continue;
      size_t ccs, cce, ccp0, ccp1;
      chunk_packs<T, P>(n, c, ccs, cce, ccp0, ccp1);
      const size_t he = ccp0 * W < cce ? ccp0 * W : cce;
      const size_t ts = ccp1 * W > he ? ccp1 * W : he;
      T* dst = stage_ptr<T>(a, c, cur, rank, P);
      for (size_t j = ccs + threadIdx.x; j < he; j += blockDim.x) dst[soff(c, j)] = snap_own[j];
      for (size_t j = ts + threadIdx.x; j < cce; j += blockDim.x) dst[soff(c, j)] = snap_own[j];
    }
  }
  if (split) {
    rank_signal<P>(a, 6, a.aux_ctr, rank);
  } else {
    rank_signal<P>(a, 1, a.end_ctr, rank);
  }
  bool ok = rank_wait<P>(a, 1, a.epoch, b, rank);
  trace_mark(a, b, 1);
  if (ok) reduce(0);
  if (ok && split) ok = rank_wait<P>(a, 6, a.epoch, b, rank);
  if (ok) {
    reduce(1);
    if (b == 0) {  // unaligned head / tail elements of the own chunk
      const size_t he = cp0 * W < ce ? cp0 * W : ce;
      const size_t ts = cp1 * W > he ? cp1 * W : he;
      auto scalar = [&](size_t j) {
        T lane[P];
#pragma unroll
        for (int qq = 0; qq < P; ++qq) lane[qq] = *src(qq, j);
        const T zb = mean_div<T, P>(rot_sum<T, P>(lane, rank));
#pragma unroll
        for (int qq = 0; qq < P; ++qq) reinterpret_cast<T*>(a.xbar[qq])[j] = zb;
      };
      for (size_t j = cs + threadIdx.x; j < he; j += blockDim.x) scalar(j);
      for (size_t j = ts + threadIdx.x; j < ce; j += blockDim.x) scalar(j);
    }
  }
  trace_mark(a, b, 2);  // this CTA's means issued
  if (ok) ok = rank_barrier<P>(a, b, rank);
  trace_mark(a, b, 3);
  publish_done(a);
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
  pdl_entry();
  constexpr int P = 2;
  constexpr int W = Pack<T>::W;
  const int rank = VIRTUAL ? (int)blockIdx.y : a.rank;
  const int vr = VIRTUAL ? (int)blockIdx.y : 0;
  const int peer = 1 - rank;
  const int b = blockIdx.x;
  const size_t n = a.n;
  dyn_comm_begin(a);
  const SgdCoef<T> cf = ccoef(a, f.c);
  const int cur = ccur(a), nxt = 1 - cur;
  bool ok = true;
  unsigned bad = 0;
  const T* const snap_own = reinterpret_cast<const T*>(csnap(a, rank));
  trace_mark(a, b, 0);
  if (a.phases & 4) {  // initial mirror: the current snapshot -> the peer's mirror, parity cur
    T* dst = mirror_ptr<T>(a, peer, cur);
    for_tiles<U>(a, b, n / W, [&](size_t p0, size_t p1) {
      for (size_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) st_plain(dst + p * W, ld_stream(snap_own + p * W));
    });
    if (b == a.nblocks - 1)
      for (size_t j = (n / W) * W + threadIdx.x; j < n; j += blockDim.x) dst[j] = snap_own[j];
    if (!VIRTUAL) rank_signal<P>(a, 1, cend(a), rank);
  }
  if (a.phases & 1) {
    if (!VIRTUAL) ok = rank_wait<P>(a, 1, cprev_push(a), b, rank);
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
      T* const sn = a.adv.rd ? reinterpret_cast<T*>(const_cast<char*>(cslot(a, rank, nxt))) : f.snap_next[vr];
      const bool load_m = cf.use_mom && !cf.first, load_d = cf.use_delta && !cf.reset;
      const bool store_d = cf.use_delta && f.mode == 0;
      auto element = [&](T& xv, T gv, T& mv, T& dv, T own, T oth, int cidx) {
        unsigned bb = sgd_elem(cf, xv, gv, mv, dv);
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
              if (cf.use_mom) st_stream(m + j0, vm[u]);
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
          if (cf.use_mom) m[j] = mv;
          if (store_d) dl[j] = dv;
          sn[j] = xv;
          out[j] = xv;
        }
      }
      if (!VIRTUAL) rank_signal<P>(a, 1, cend(a), rank);
    }
  }
  report_nonfinite(a.nonfinite, bad);
  trace_mark(a, b, 3);
  if (!VIRTUAL) publish_done(a);
}

}  // namespace lasgd

#endif  // LASGD_COMM_PUSH_CUH
