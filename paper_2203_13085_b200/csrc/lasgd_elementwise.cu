// Rank-local streaming kernels of the LASGD sync path: K0 blend, K1 snapshot,
// K4 elastic pull / reference finalize, K5 fused local SGD step.
//
// All are HBM-bound elementwise passes over the flat parameter buffer: 128-bit
// evict-first loads/stores, U independent packs in flight per thread,
// grid = 2 CTAs x 256 threads per SM by default (<= 64 registers per thread: half of
// each SM stays free for the side-stream all-reduce), scalar tail for n % W,
// warp-aggregated non-finite counter fused into the pass (the reference checks
// every blend result, params.py:88).  No tensor cores: there is no reuse.
//
// Reference anchors: blend params.py:80-89; sgd_local_step optimizer.py:136-149;
// lasgd_finalize_round optimizer.py:152-178; pull = blend order of
// optimizer.py:256-257 (Algorithm 1 line 9a, PAPER.md:182 for alpha = 1).

#include <stdarg.h>
#include <string.h>

#include "lasgd_common.cuh"

namespace lasgd {

// ------------------------------------------------------------- generic driver
constexpr int kThreads = 256;
// Each Op declares U, the packs in flight per thread, sized so the loaded data stays
// near 32 registers (<= 64 total under __launch_bounds__(256, 4), no spills).

template <typename T, typename Op, int U>
__device__ __forceinline__ void stream_body(Op& op, size_t n, unsigned long long* nonfinite) {
  constexpr int W = Pack<T>::W;
  const size_t npack = n / W;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned bad = 0;
  for (; i + (U - 1) * stride < npack; i += U * stride) {
    typename Op::Loaded L[U];
#pragma unroll
    for (int u = 0; u < U; ++u) op.load(L[u], (i + u * stride) * W);
#pragma unroll
    for (int u = 0; u < U; ++u) bad += op.compute_store(L[u], (i + u * stride) * W);
  }
  for (; i < npack; i += stride) {
    typename Op::Loaded L;
    op.load(L, i * W);
    bad += op.compute_store(L, i * W);
  }
  const size_t t = npack * W + (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) bad += op.scalar(t);
  report_nonfinite(nonfinite, bad);
}

template <typename T, typename Op, int U>
__global__ void __launch_bounds__(kThreads, 4) k_stream(Op op, size_t n, unsigned long long* nonfinite) {
  pdl_entry();
  stream_body<T, Op, U>(op, n, nonfinite);
}

// Fallback for buffers that are not 16-byte aligned (e.g. arbitrary views).
template <typename T, typename Op>
__global__ void __launch_bounds__(kThreads, 4) k_scalar(Op op, size_t n, unsigned long long* nonfinite) {
  unsigned bad = 0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    bad += op.scalar(i);
  report_nonfinite(nonfinite, bad);
}

template <typename T, typename Op>
int launch(const Op& op, size_t n, bool aligned, unsigned long long* nonfinite, void* stream) {
  if (n == 0) return LASGD_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (aligned) {
    const size_t npack = n / Pack<T>::W;
    const size_t work = npack > (size_t)kThreads ? npack : (size_t)kThreads;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(stream_grid(work, kThreads));
    cfg.blockDim = dim3(kThreads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    LASGD_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_stream<T, Op, Op::U>, op, n, nonfinite));
  } else {
    k_scalar<T, Op><<<stream_grid(n, kThreads), kThreads, 0, s>>>(op, n, nonfinite);
  }
  LASGD_CUDA_TRY(cudaGetLastError());
  return LASGD_OK;
}

// ------------------------------------------------------------- K0 blend
template <typename T>
struct BlendOp {
  T* out;
  const T* u;
  const T* v;
  T a, b;
  static constexpr int U = 4;
  struct Loaded { Pack<T> u, v; };
  __device__ __forceinline__ unsigned elem(T uu, T vv, T& o) const {
    o = add_rn(mul_rn(a, uu), mul_rn(b, vv));
    return !finite(o);
  }
  __device__ __forceinline__ void load(Loaded& L, size_t j) const {
    L.u = ld_stream(u + j);
    L.v = ld_stream(v + j);
  }
  __device__ __forceinline__ unsigned compute_store(const Loaded& L, size_t j) const {
    Pack<T> o;
    unsigned bad = 0;
#pragma unroll
    for (int k = 0; k < Pack<T>::W; ++k) bad += elem(L.u.v[k], L.v.v[k], o.v[k]);
    st_stream(out + j, o);
    return bad;
  }
  __device__ __forceinline__ unsigned scalar(size_t j) const {
    T o;
    unsigned bad = elem(u[j], v[j], o);
    out[j] = o;
    return bad;
  }
};

// ------------------------------------------------------------- K1 snapshot
template <typename T>
struct CopyOp {
  T* dst;
  const T* src;
  static constexpr int U = 4;
  struct Loaded { Pack<T> s; };
  __device__ __forceinline__ void load(Loaded& L, size_t j) const { L.s = ld_stream(src + j); }
  __device__ __forceinline__ unsigned compute_store(const Loaded& L, size_t j) const {
    st_stream(dst + j, L.s);
    return 0;
  }
  __device__ __forceinline__ unsigned scalar(size_t j) const {
    dst[j] = src[j];
    return 0;
  }
};

// ------------------------------------------------------------- K5 local step
template <typename T>
struct SgdOp {
  T* x;
  const T* g;
  T* m;
  T* delta;
  T* snap;  // optional: also write the updated x here (K7 at P = 1: local step + next snapshot)
  SgdCoef<T> c;
  // load m / delta whenever they exist (their values are ignored on a first step / after
  // a reset): the loads then do not wait for first / reset, which the graph-replayable
  // kernel reads from the device round descriptor at entry
  bool load_all = false;
  static constexpr int U = 2;
  struct Loaded { Pack<T> x, g, m, d; };

  __device__ __forceinline__ void load(Loaded& L, size_t j) const {
    L.x = ld_stream(x + j);
    L.g = ld_stream(g + j);
    if (c.use_mom && (load_all || !c.first)) L.m = ld_stream(m + j);
    if (c.use_delta && (load_all || !c.reset)) L.d = ld_stream(delta + j);
  }
  __device__ __forceinline__ unsigned compute_store(Loaded& L, size_t j) const {
    unsigned bad = 0;
#pragma unroll
    for (int k = 0; k < Pack<T>::W; ++k) bad += sgd_elem(c, L.x.v[k], L.g.v[k], L.m.v[k], L.d.v[k]);
    st_stream(x + j, L.x);
    if (c.use_mom) st_stream(m + j, L.m);
    if (c.use_delta) st_stream(delta + j, L.d);
    if (snap) st_stream(snap + j, L.x);
    return bad;
  }
  __device__ __forceinline__ unsigned scalar(size_t j) const {
    T xv = x[j], mv = (c.use_mom && !c.first) ? m[j] : T(0), dv = (c.use_delta && !c.reset) ? delta[j] : T(0);
    unsigned bad = sgd_elem(c, xv, g[j], mv, dv);
    x[j] = xv;
    if (c.use_mom) m[j] = mv;
    if (c.use_delta) delta[j] = dv;
    if (snap) snap[j] = xv;
    return bad;
  }
};

// ------------------------------------------------------------- K4 pull / finalize
template <typename T>
struct PullOp {
  T* x;
  T* snap_next;
  const T* snap;
  const T* xbar;
  T neg_alpha;
  static constexpr int U = 2;
  struct Loaded { Pack<T> x, s, z; };
  __device__ __forceinline__ unsigned elem(T& xv, T sv, T zv) const { return pull_elem(neg_alpha, xv, sv, zv); }
  __device__ __forceinline__ void load(Loaded& L, size_t j) const {
    L.x = ld_stream(x + j);
    L.s = ld_stream(snap + j);
    L.z = ld_stream(xbar + j);
  }
  __device__ __forceinline__ unsigned compute_store(Loaded& L, size_t j) const {
    unsigned bad = 0;
#pragma unroll
    for (int k = 0; k < Pack<T>::W; ++k) bad += elem(L.x.v[k], L.s.v[k], L.z.v[k]);
    st_stream(x + j, L.x);
    if (snap_next) st_stream(snap_next + j, L.x);
    return bad;
  }
  __device__ __forceinline__ unsigned scalar(size_t j) const {
    T xv = x[j];
    unsigned bad = elem(xv, snap[j], xbar[j]);
    x[j] = xv;
    if (snap_next) snap_next[j] = xv;
    return bad;
  }
};

template <typename T>
struct FinalizeOp {
  T* x;
  T* snap_next;
  const T* z;
  const T* delta;
  static constexpr int U = sizeof(T) == 8 ? 1 : 2;
  struct Loaded { Pack<T> z, d; };
  __device__ __forceinline__ void load(Loaded& L, size_t j) const {
    L.z = ld_stream(z + j);
    if (delta) {
      L.d = ld_stream(delta + j);
    } else {
#pragma unroll
      for (int k = 0; k < Pack<T>::W; ++k) L.d.v[k] = T(0);
    }
  }
  __device__ __forceinline__ unsigned compute_store(Loaded& L, size_t j) const {
    Pack<T> o;
    unsigned bad = 0;
#pragma unroll
    for (int k = 0; k < Pack<T>::W; ++k) {
      o.v[k] = add_rn(L.z.v[k], L.d.v[k]);  // blend(1, z, 1, delta), optimizer.py:171
      bad += !finite(o.v[k]);
    }
    st_stream(x + j, o);
    if (snap_next) st_stream(snap_next + j, o);
    return bad;
  }
  __device__ __forceinline__ unsigned scalar(size_t j) const {
    T o = add_rn(z[j], delta ? delta[j] : T(0));
    x[j] = o;
    if (snap_next) snap_next[j] = o;
    return !finite(o);
  }
};

// ------------------------------------------------------------- K5 + K4 in one pass
// The round boundary of the deterministic overlap pipeline: the local step, then the
// pull towards the (stale) mean that the side stream has already delivered (mode 0), or
// the reference finalize new = xbar + delta' (mode 1); the next snapshot written in the
// same pass.  The element function is K7's, so the bits equal K5 followed by K4.  8B
// (x, g, m, snap, xbar in; x, m, snap_next out) instead of 5B + 5B.
template <typename T>
struct SgdPullOp {
  T* x;
  const T* g;
  T* m;
  T* delta;
  T* snap_next;
  const T* snap;
  const T* xbar;
  SgdCoef<T> c;
  T neg_alpha;
  int mode;
  static constexpr int U = 1;
  struct Loaded { Pack<T> x, g, m, d, s, z; };
  __device__ __forceinline__ unsigned elem(T& xv, T gv, T& mv, T& dv, T sv, T zv) const {
    unsigned bad = sgd_elem(c, xv, gv, mv, dv);
    if (mode == 0) {
      bad += pull_elem(neg_alpha, xv, sv, zv);
    } else {
      xv = add_rn(zv, dv);  // blend(1, z, 1, delta), optimizer.py:171
      bad += !finite(xv);
    }
    return bad;
  }
  __device__ __forceinline__ void load(Loaded& L, size_t j) const {
    L.x = ld_stream(x + j);
    L.g = ld_stream(g + j);
    if (c.use_mom && !c.first) L.m = ld_stream(m + j);
    if (c.use_delta && !c.reset) L.d = ld_stream(delta + j);
    if (mode == 0) L.s = ld_stream(snap + j);
    L.z = ld_stream(xbar + j);
  }
  __device__ __forceinline__ unsigned compute_store(Loaded& L, size_t j) const {
    unsigned bad = 0;
#pragma unroll
    for (int k = 0; k < Pack<T>::W; ++k) bad += elem(L.x.v[k], L.g.v[k], L.m.v[k], L.d.v[k], L.s.v[k], L.z.v[k]);
    st_stream(x + j, L.x);
    if (c.use_mom) st_stream(m + j, L.m);
    if (c.use_delta && mode == 0) st_stream(delta + j, L.d);  // finalize resets delta (lazily)
    st_stream(snap_next + j, L.x);
    return bad;
  }
  __device__ __forceinline__ unsigned scalar(size_t j) const {
    T xv = x[j], mv = (c.use_mom && !c.first) ? m[j] : T(0), dv = (c.use_delta && !c.reset) ? delta[j] : T(0);
    unsigned bad = elem(xv, g[j], mv, dv, mode == 0 ? snap[j] : T(0), xbar[j]);
    x[j] = xv;
    if (c.use_mom) m[j] = mv;
    if (c.use_delta && mode == 0) delta[j] = dv;
    snap_next[j] = xv;
    return bad;
  }
};

template <typename T>
int sgd_pull_t(void* x, const void* g, void* m, void* delta, void* snap_next, const void* snap, const void* xbar,
               size_t n, const lasgd_sgd_params* p, double alpha, int mode, unsigned long long* nf, void* s) {
  SgdPullOp<T> op;
  op.x = (T*)x;
  op.g = (const T*)g;
  op.m = (T*)m;
  op.delta = (T*)delta;
  op.snap_next = (T*)snap_next;
  op.snap = (const T*)snap;
  op.xbar = (const T*)xbar;
  op.c = make_sgd_coef<T>(p, delta != nullptr);
  op.neg_alpha = (T)(-alpha);
  op.mode = mode;
  const bool al = aligned16(x) && aligned16(g) && (!op.c.use_mom || aligned16(m)) &&
                  (!op.c.use_delta || aligned16(delta)) && aligned16(snap_next) && (mode != 0 || aligned16(snap)) &&
                  aligned16(xbar);
  return launch<T>(op, n, al, nf, s);
}

// ------------------------------------------------------------- typed entry points
template <typename T>
int blend_t(void* out, double a, const void* u, double b, const void* v, size_t n, unsigned long long* nf,
            void* s) {
  BlendOp<T> op{(T*)out, (const T*)u, (const T*)v, (T)a, (T)b};
  return launch<T>(op, n, aligned16(out) && aligned16(u) && aligned16(v), nf, s);
}

template <typename T>
int copy_t(void* dst, const void* src, size_t n, void* s) {
  CopyOp<T> op{(T*)dst, (const T*)src};
  return launch<T>(op, n, aligned16(dst) && aligned16(src), nullptr, s);
}

template <typename T>
int sgd_t(void* x, const void* g, void* m, void* delta, size_t n, const lasgd_sgd_params* p,
          unsigned long long* nf, void* s, void* snap = nullptr) {
  SgdOp<T> op;
  op.x = (T*)x;
  op.g = (const T*)g;
  op.m = (T*)m;
  op.delta = (T*)delta;
  op.snap = (T*)snap;
  op.c = make_sgd_coef<T>(p, delta != nullptr);
  bool al = aligned16(x) && aligned16(g) && (!op.c.use_mom || aligned16(m)) && (!op.c.use_delta || aligned16(delta)) &&
            (!snap || aligned16(snap));
  return launch<T>(op, n, al, nf, s);
}

// K7 at P = 1 (no peers, no mean, no pull — optimizer.py:168-169): the local step with
// the next snapshot written in the same streaming pass (6B instead of K5 5B + K1 2B).
int sgd_step_snapshot(int dtype, void* x, const void* g, void* m, void* delta, void* snap, size_t n,
                      const lasgd_sgd_params* p, unsigned long long* nf, void* s) {
  if (dtype == LASGD_F32) return sgd_t<float>(x, g, m, delta, n, p, nf, s, snap);
  if (dtype == LASGD_F64) return sgd_t<double>(x, g, m, delta, n, p, nf, s, snap);
  return fail(LASGD_ERR_INVALID_ARGUMENT, "unknown dtype %d", dtype);
}

// K5 (and the P = 1 round: K5 + next snapshot) with lr / first_step / delta reset /
// snapshot slot from the device round descriptor: the graph-replayable form.
template <typename T, int U>
__global__ void __launch_bounds__(kThreads, 4) k_sgd_dyn(SgdOp<T> op, T* snap0, T* snap1, size_t n,
                                                        unsigned long long* nonfinite, RoundAdv adv, bool aligned) {
  // Programmatic dependent launch: let the next step's kernel get its CTAs onto the SMs
  // now (they wait in griddepcontrol.wait below until this grid has completed and its
  // writes are visible), then wait for the previous step's grid the same way.  Saves the
  // launch ramp between back-to-back steps of a replayed graph.
  pdl_entry();
  const DynView v = dyn_read(adv.rd);
  dyn_coef(op.c, v);
  op.snap = snap0 == nullptr ? nullptr : (v.cur ? snap0 : snap1);  // next slot = 1 - cur
  if (aligned)
    stream_body<T, SgdOp<T>, U>(op, n, nonfinite);
  else {  // unaligned views: the scalar loop
    unsigned bad = 0;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
      bad += op.scalar(i);
    report_nonfinite(nonfinite, bad);
  }
  dyn_advance(adv, gridDim.x);
}

template <typename T>
int sgd_dyn_t(void* x, const void* g, void* m, void* delta, void* const* snaps, size_t n, const lasgd_sgd_params* p,
              unsigned long long* nf, void* s, const RoundAdv& adv) {
  SgdOp<T> op;
  op.x = (T*)x;
  op.g = (const T*)g;
  op.m = (T*)m;
  op.delta = (T*)delta;
  op.snap = nullptr;
  op.c = make_sgd_coef<T>(p, delta != nullptr);
  op.load_all = true;
  const size_t npack = n / Pack<T>::W;
  const size_t work = npack > (size_t)kThreads ? npack : (size_t)kThreads;
  const bool al = aligned16(x) && aligned16(g) && (!op.c.use_mom || aligned16(m)) &&
                  (!op.c.use_delta || aligned16(delta)) && (!snaps || (aligned16(snaps[0]) && aligned16(snaps[1])));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(stream_grid(work, kThreads));
  cfg.blockDim = dim3(kThreads);
  cfg.stream = reinterpret_cast<cudaStream_t>(s);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  LASGD_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_sgd_dyn<T, SgdOp<T>::U>, op, snaps ? (T*)snaps[0] : nullptr,
                                    snaps ? (T*)snaps[1] : nullptr, n, nf, adv, al));
  return LASGD_OK;
}

int sgd_step_dyn(int dtype, void* x, const void* g, void* m, void* delta, void* const* snaps, size_t n,
                 const lasgd_sgd_params* p, unsigned long long* nf, void* s, const RoundAdv& adv) {
  if (!adv.rd) return fail(LASGD_ERR_INVALID_ARGUMENT, "sgd_step_dyn: no round descriptor");
  if (dtype == LASGD_F32) return sgd_dyn_t<float>(x, g, m, delta, snaps, n, p, nf, s, adv);
  if (dtype == LASGD_F64) return sgd_dyn_t<double>(x, g, m, delta, snaps, n, p, nf, s, adv);
  return fail(LASGD_ERR_INVALID_ARGUMENT, "unknown dtype %d", dtype);
}

template <typename T>
int pull_t(void* x, void* snap_next, const void* snap, const void* xbar, size_t n, double alpha,
           unsigned long long* nf, void* s) {
  PullOp<T> op{(T*)x, (T*)snap_next, (const T*)snap, (const T*)xbar, (T)(-alpha)};
  bool al = aligned16(x) && aligned16(snap) && aligned16(xbar) && (!snap_next || aligned16(snap_next));
  return launch<T>(op, n, al, nf, s);
}

template <typename T>
int finalize_t(void* x, void* snap_next, const void* z, const void* delta, size_t n, unsigned long long* nf,
               void* s) {
  FinalizeOp<T> op{(T*)x, (T*)snap_next, (const T*)z, (const T*)delta};
  bool al = aligned16(x) && aligned16(z) && (!delta || aligned16(delta)) && (!snap_next || aligned16(snap_next));
  return launch<T>(op, n, al, nf, s);
}

}  // namespace lasgd

// ============================================================== C ABI
using namespace lasgd;

#define DISPATCH_DTYPE(dtype, CALL_F32, CALL_F64)                                   \
  do {                                                                              \
    if ((dtype) == LASGD_F32) return CALL_F32;                                      \
    if ((dtype) == LASGD_F64) return CALL_F64;                                      \
    return fail(LASGD_ERR_INVALID_ARGUMENT, "unknown dtype %d", (int)(dtype));      \
  } while (0)

extern "C" int lasgd_blend(void* out, double a, const void* u, double b, const void* v, size_t n, int dtype,
                           unsigned long long* nonfinite, void* stream) {
  if (n && (!out || !u || !v)) return fail(LASGD_ERR_INVALID_ARGUMENT, "lasgd_blend: null buffer");
  DISPATCH_DTYPE(dtype, blend_t<float>(out, a, u, b, v, n, nonfinite, stream),
                 blend_t<double>(out, a, u, b, v, n, nonfinite, stream));
}

extern "C" int lasgd_snapshot(void* snap, const void* x, size_t n, int dtype, void* stream) {
  if (n && (!snap || !x)) return fail(LASGD_ERR_INVALID_ARGUMENT, "lasgd_snapshot: null buffer");
  if (snap == x) return LASGD_OK;
  DISPATCH_DTYPE(dtype, copy_t<float>(snap, x, n, stream), copy_t<double>(snap, x, n, stream));
}

extern "C" int lasgd_sgd_step(void* x, const void* g, void* m, void* delta, size_t n, int dtype,
                              const lasgd_sgd_params* p, unsigned long long* nonfinite, void* stream) {
  if (!p) return fail(LASGD_ERR_INVALID_ARGUMENT, "lasgd_sgd_step: null params");
  if (n && (!x || !g)) return fail(LASGD_ERR_INVALID_ARGUMENT, "lasgd_sgd_step: null buffer");
  if (p->momentum != 0.0 && !m) return fail(LASGD_ERR_INVALID_ARGUMENT, "lasgd_sgd_step: momentum needs m");
  if (p->momentum < 0.0 || p->weight_decay < 0.0 || p->dampening < 0.0 || p->dampening > 1.0)
    return fail(LASGD_ERR_INVALID_ARGUMENT, "lasgd_sgd_step: invalid hyper-parameters");
  if (p->nesterov && (p->momentum <= 0.0 || p->dampening != 0.0))
    return fail(LASGD_ERR_INVALID_ARGUMENT, "Nesterov momentum requires a momentum and zero dampening");
  DISPATCH_DTYPE(dtype, sgd_t<float>(x, g, m, delta, n, p, nonfinite, stream),
                 sgd_t<double>(x, g, m, delta, n, p, nonfinite, stream));
}

extern "C" int lasgd_elastic_pull(void* x, void* snap_next, const void* snap, const void* xbar, size_t n,
                                  int dtype, double alpha, unsigned long long* nonfinite, void* stream) {
  if (n && (!x || !snap || !xbar)) return fail(LASGD_ERR_INVALID_ARGUMENT, "lasgd_elastic_pull: null buffer");
  if (!(alpha >= 0.0 && alpha <= 1.0)) return fail(LASGD_ERR_INVALID_ARGUMENT, "alpha must be in [0, 1], got %g", alpha);
  DISPATCH_DTYPE(dtype, pull_t<float>(x, snap_next, snap, xbar, n, alpha, nonfinite, stream),
                 pull_t<double>(x, snap_next, snap, xbar, n, alpha, nonfinite, stream));
}

extern "C" int lasgd_sgd_pull(void* x, const void* g, void* m, void* delta, void* snap_next, const void* snap,
                              const void* xbar, size_t n, int dtype, const lasgd_sgd_params* p, double alpha, int mode,
                              unsigned long long* nonfinite, void* stream) {
  if (!p) return fail(LASGD_ERR_INVALID_ARGUMENT, "lasgd_sgd_pull: null params");
  if (n && (!x || !g || !snap_next || !xbar || (mode == 0 && !snap)))
    return fail(LASGD_ERR_INVALID_ARGUMENT, "lasgd_sgd_pull: null buffer");
  if (mode != 0 && mode != 1) return fail(LASGD_ERR_INVALID_ARGUMENT, "mode %d (0 pull, 1 finalize)", mode);
  if (mode == 1 && !delta) return fail(LASGD_ERR_INVALID_ARGUMENT, "finalize mode needs the delta buffer");
  if (mode == 0 && !(alpha > 0.0 && alpha <= 1.0)) return fail(LASGD_ERR_INVALID_ARGUMENT, "alpha must be in (0, 1]");
  if (p->momentum != 0.0 && !m) return fail(LASGD_ERR_INVALID_ARGUMENT, "lasgd_sgd_pull: momentum needs m");
  if (p->nesterov && (p->momentum <= 0.0 || p->dampening != 0.0))
    return fail(LASGD_ERR_INVALID_ARGUMENT, "Nesterov momentum requires a momentum and zero dampening");
  DISPATCH_DTYPE(dtype, sgd_pull_t<float>(x, g, m, delta, snap_next, snap, xbar, n, p, alpha, mode, nonfinite, stream),
                 sgd_pull_t<double>(x, g, m, delta, snap_next, snap, xbar, n, p, alpha, mode, nonfinite, stream));
}

extern "C" int lasgd_finalize(void* x, void* snap_next, const void* z, const void* delta, size_t n, int dtype,
                              unsigned long long* nonfinite, void* stream) {
  // delta == NULL: the accumulator is zero (no local step since the last finalize,
  // optimizer.py:174), so new = z + 0 without reading it
  if (n && (!x || !z)) return fail(LASGD_ERR_INVALID_ARGUMENT, "lasgd_finalize: null buffer");
  DISPATCH_DTYPE(dtype, finalize_t<float>(x, snap_next, z, delta, n, nonfinite, stream),
                 finalize_t<double>(x, snap_next, z, delta, n, nonfinite, stream));
}
