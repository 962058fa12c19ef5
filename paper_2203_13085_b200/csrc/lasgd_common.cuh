// Shared device/host helpers for the LASGD sync kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "lasgd_sync.h"

namespace lasgd {

// ---------------------------------------------------------------- errors
void set_last_error(const char* fmt, ...);
int fail(int code, const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what);

#define LASGD_CUDA_TRY(expr)                                 \
  do {                                                       \
    cudaError_t _e = (expr);                                 \
    if (_e != cudaSuccess) return ::lasgd::cuda_fail(_e, #expr); \
  } while (0)

int num_sms();  // SM count of the current device (cached per device)

// K5 with the next snapshot written in the same pass (lasgd_elementwise.cu).
int sgd_step_snapshot(int dtype, void* x, const void* g, void* m, void* delta, void* snap, size_t n,
                      const lasgd_sgd_params* p, unsigned long long* nf, void* s);
struct RoundAdv;
// K5 with the per-launch scalars read from the device round descriptor (graph replay);
// snaps != nullptr also writes the next snapshot slot snaps[1 - cur] (P = 1 round).
int sgd_step_dyn(int dtype, void* x, const void* g, void* m, void* delta, void* const* snaps, size_t n,
                 const lasgd_sgd_params* p, unsigned long long* nf, void* s, const RoundAdv& adv);

// ---------------------------------------------------------------- arithmetic
// Separately rounded ops (the reference's numpy never contracts a*b+c).
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ bool finite(float a) { return isfinite(a); }
__device__ __forceinline__ bool finite(double a) { return isfinite(a); }

// ---------------------------------------------------------------- 128-bit packs
template <typename T>
struct alignas(16) Pack {
  static constexpr int W = 16 / sizeof(T);
  T v[W];
};

// Streaming loads/stores (evict-first): the sync path touches every byte once per
// launch and every buffer is >> L2 at ResNet-50 size.
template <typename T>
__device__ __forceinline__ Pack<T> ld_stream(const T* p) {
  uint4 r = __ldcs(reinterpret_cast<const uint4*>(p));
  return *reinterpret_cast<Pack<T>*>(&r);
}
template <typename T>
__device__ __forceinline__ void st_stream(T* p, const Pack<T>& v) {
  __stcs(reinterpret_cast<uint4*>(p), *reinterpret_cast<const uint4*>(&v));
}
// L2-only (L1-bypassing) load, used for peer (NVLink-mapped) memory.
template <typename T>
__device__ __forceinline__ Pack<T> ld_cg(const T* p) {
  uint4 r = __ldcg(reinterpret_cast<const uint4*>(p));
  return *reinterpret_cast<Pack<T>*>(&r);
}
template <typename T>
__device__ __forceinline__ void st_plain(T* p, const Pack<T>& v) {
  *reinterpret_cast<uint4*>(p) = *reinterpret_cast<const uint4*>(&v);
}

// Warp-aggregated non-finite counter (one atomic per warp, only when non-zero).
__device__ __forceinline__ void report_nonfinite(unsigned long long* ctr, unsigned bad) {
  if (ctr == nullptr) return;
  unsigned total = __reduce_add_sync(0xffffffffu, bad);
  if (total != 0 && (threadIdx.x & 31) == 0) atomicAdd(ctr, (unsigned long long)total);
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ---------------------------------------------------------------- element math
// Shared by the standalone kernels and the fused round kernel, so both produce the
// same bits by construction.

// K5 coefficients, already rounded to T on the host side of the launch.
template <typename T>
struct SgdCoef {
  T neg_lr, mu, omd, wd;
  bool use_wd, use_mom, nesterov, first, use_delta, reset;
};

template <typename T>
SgdCoef<T> make_sgd_coef(const lasgd_sgd_params* p, bool use_delta) {
  SgdCoef<T> c;
  c.neg_lr = (T)(-p->lr);
  c.mu = (T)p->momentum;
  c.omd = (T)(1.0 - p->dampening);
  c.wd = (T)p->weight_decay;
  c.use_wd = p->weight_decay != 0.0;
  c.use_mom = p->momentum != 0.0;
  c.nesterov = p->nesterov != 0;
  c.first = p->first_step != 0;
  c.use_delta = use_delta;
  c.reset = p->delta_reset != 0;
  return c;
}

// One local step on one element (optimizer.py:145-146 at momentum = wd = 0):
//   d = g (+ wd*x); m = first ? d : mu*m + (1-damp)*d; d = nesterov ? d + mu*m : m;
//   s = (-lr)*d; x = x + s; delta = (reset ? 0 : delta) + s.   Returns #non-finite.
template <typename T>
__device__ __forceinline__ unsigned sgd_elem(const SgdCoef<T>& c, T& xv, T gv, T& mv, T& dv) {
  T dir = gv;
  if (c.use_wd) dir = add_rn(dir, mul_rn(c.wd, xv));
  if (c.use_mom) {
    mv = c.first ? dir : add_rn(mul_rn(c.mu, mv), mul_rn(c.omd, dir));
    dir = c.nesterov ? add_rn(dir, mul_rn(c.mu, mv)) : mv;
  }
  const T s = mul_rn(c.neg_lr, dir);
  xv = add_rn(xv, s);
  unsigned bad = !finite(xv);
  if (c.use_delta) {
    dv = add_rn(c.reset ? T(0) : dv, s);
    bad += !finite(dv);
  }
  return bad;
}

// Elastic pull on one element: diff = 1*snap + (-1)*xbar; x = 1*x + (-alpha)*diff
// (blend order of optimizer.py:256-257).  Returns #non-finite.
template <typename T>
__device__ __forceinline__ unsigned pull_elem(T neg_alpha, T& xv, T sv, T zv) {
  const T diff = add_rn(sv, mul_rn(T(-1), zv));
  xv = add_rn(xv, mul_rn(neg_alpha, diff));
  return !finite(diff) + !finite(xv);
}

// ---------------------------------------------------------------- programmatic dependent launch
// First statement of every sync kernel: let a dependent grid (launched with programmatic
// stream serialization) get onto the SMs as soon as this grid's CTAs exit, then wait
// until the previous grid in the stream has completed and its writes are visible.  With
// a plain launch both are no-ops; nothing is read before the wait.
__device__ __forceinline__ void pdl_entry() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// ---------------------------------------------------------------- device round descriptor
// The per-launch scalars of the deterministic schedule (optimizer.py:181-207 with
// collective_complete = (tau_i == k)) live in device memory so that a captured loop of
// worker steps replays as one CUDA graph: every CTA of a launch reads the learning
// rate (table indexed by the local clock, problems.py:322-365), first_step, the delta
// reset flag and the snapshot slot at entry, and the last CTA to finish advances the
// descriptor for the next launch (RoundAdv says how: baked into the graph node, the
// same on every replay because a graph holds a whole number of rounds).
struct DevRound {
  unsigned long long clock;         // local steps taken (NodeState.local_clock)
  unsigned long long seq;           // communicator launches issued (epoch of the next one - 1)
  double lr_now;                    // lr[min(clock, lr_len - 1)]: one load at kernel entry
  const double* lr;                 // learning rate per local clock
  unsigned long long lr_len;        // clock >= lr_len reads the last entry
  int snap_idx;                     // current snapshot slot
  int mom_started;                  // momentum buffer initialised (first_step = !mom_started)
  int delta_fresh;                  // delta is logically zero (reset at the last finalize)
  unsigned int arrive;              // CTAs of the running launch that have finished
};

struct RoundAdv {
  DevRound* rd;   // nullptr: static launch arguments (eager path)
  int steps;      // local steps this launch takes (0 or 1)
  int close;      // this launch closes a round (snapshot slot flips, delta reset)
  int has_mom;    // momentum buffer in use
  int has_delta;  // delta accumulator in use
  int seq_inc;    // communicator launches this kernel counts as
};

struct DynView {
  double lr;
  int first, reset, cur;
};

// Every thread reads the descriptor (independent loads of one L2 line written by the
// previous kernel: a single round trip).
__device__ __forceinline__ DynView dyn_read(const DevRound* r) {
  DynView v;
  v.lr = __ldcg(&r->lr_now);
  v.first = !__ldcg(&r->mom_started);
  v.reset = __ldcg(&r->delta_fresh);
  v.cur = __ldcg(&r->snap_idx);
  return v;
}

// Advance by `ad` (the last CTA of a launch): clock, launch count, flags, and the rate of
// the new clock.
__device__ __forceinline__ void dyn_apply(DevRound* r, const RoundAdv& ad) {
  r->clock += (unsigned long long)ad.steps;
  r->seq += (unsigned long long)ad.seq_inc;
  if (ad.steps) {
    const unsigned long long k = r->clock, len = r->lr_len;
    r->lr_now = r->lr[k < len ? k : len - 1];
  }
  if (ad.steps && ad.has_mom) r->mom_started = 1;
  if (ad.close) {
    r->snap_idx ^= 1;
    r->delta_fresh = ad.has_delta;
  } else if (ad.steps) {
    r->delta_fresh = 0;
  }
}

template <typename T>
__device__ __forceinline__ void dyn_coef(SgdCoef<T>& c, const DynView& v) {
  c.neg_lr = (T)(-v.lr);  // the host's (T)(-lr) of make_sgd_coef
  c.first = v.first != 0;
  c.reset = c.use_delta && v.reset != 0;
}

// Last CTA of the launch (of `total` CTAs) advances the descriptor.  Every CTA read it
// at entry, before counting itself in, so the update cannot race a reader.
__device__ __forceinline__ void dyn_advance(const RoundAdv& ad, unsigned total) {
  if (ad.rd == nullptr) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    DevRound* r = ad.rd;
    if (atomicAdd(&r->arrive, 1u) == total - 1u) {
      r->arrive = 0u;
      dyn_apply(r, ad);
      __threadfence();
    }
  }
}

// Host-side communicator bookkeeping a graph replay must advance like the captured
// launches did (lasgd_comm.cu): launches issued, the last push round, the last launch
// that raised end-of-round signals, the staging parity that holds valid contributions.
struct CommMirror {
  unsigned long long seq, last_push, end_seq;
  int push_slot;
};
int comm_mirror_get(lasgd_comm* c, CommMirror* m);
int comm_mirror_set(lasgd_comm* c, const CommMirror& m);
// Record the completion event of launch c->seq on `stream` (after a graph replay).
int comm_record_last(lasgd_comm* c, void* stream);
// Algorithm of the overlap pipeline's side-stream mean for `algo` (AUTO: the copy-engine
// two-shot where it interferes least with forward/backward, else as lasgd_comm_allreduce).
int comm_side_algo(lasgd_comm* c, int algo);
// The fused round (K7 one-shot or K8 push) in graph-replayable form: sequence number,
// snapshot slot, learning rate, first step and delta reset from adv.rd; requires the
// steady state of a deterministic loop (the previous launch was a round of the same
// kind).  Issues no event (the captured graph is the unit of completion).
int comm_fused_round_dyn(lasgd_comm* c, int snap_slot, int algo, void* x, const void* g, void* m, void* delta,
                         const lasgd_sgd_params* sgd, double alpha, int mode, int nblocks,
                         unsigned long long* nonfinite, void* stream, const RoundAdv& adv, unsigned long long* seq);

// CTAs per SM of the streaming kernels (tunable, lasgd_set_stream_ctas_per_sm).  The
// default leaves half of every SM's registers/threads free so the all-reduce CTAs on
// the side stream can co-reside with a local step instead of queueing behind it.
int stream_ctas_per_sm();

// Grid for a streaming kernel: enough CTAs to fill every SM `per_sm` times, never more
// than the work needs.
inline int stream_grid(size_t work_items, int threads, int per_sm = 0) {
  if (per_sm <= 0) per_sm = stream_ctas_per_sm();
  size_t need = (work_items + threads - 1) / threads;
  size_t cap = (size_t)num_sms() * per_sm;
  if (need < 1) need = 1;
  return (int)(need < cap ? need : cap);
}

// RAII device switch for comm calls.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace lasgd
