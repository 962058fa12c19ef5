// Native per-rank LASGD worker: the round protocol of Algorithm 1 (
// optimizer.py:181-207) as a host-side state machine over CUDA streams and events,
// so one C call issues a whole local step (the Python layer only forwards the
// gradient pointer and the learning rate).
//
// pipeline OVERLAP: compute stream K5 every step; at a round boundary the compute
//   stream waits for the previous launch (event), applies K4 (pull or reference
//   finalize, writing the next snapshot slot) and hands the snapshot to the side
//   stream, where K2/K3 runs while the next minibatches proceed.
// pipeline FUSED (deterministic only): the boundary step is one fused launch (local
//   step + NVLink mean + pull + next snapshot: K7, or the K8 push round — mirror form at
//   P = 2, staged form at P >= 3 — as lasgd_comm_resolve_fused_algo picks); other steps
//   are K5.
// adaptive: a round closes as soon as the host-mapped completion flag of the
//   in-flight launch is set, when the peers are already ahead (this rank is the
//   round's laggard, lasgd_comm_peers_ahead), or when tau_max local steps have been
//   taken (then the compute stream waits on the event; the host never blocks except
//   for the bounded run-ahead throttle).  Side-stream all-reduces are gated (k_gate)
//   so they do not hold SMs while a late peer catches up.
#include <string.h>
#include <time.h>

#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges show up in Nsight timelines, free otherwise

#include "lasgd_common.cuh"

namespace lasgd {

enum Kind { K_SGD = 0, K_SNAPSHOT, K_PULL, K_FINALIZE, K_ALLREDUCE, K_FUSED, K_SGD_PULL, K_KINDS };

struct TimingRec {
  int kind;
  cudaEvent_t e0, e1;
};

}  // namespace lasgd

using namespace lasgd;

struct lasgd_worker {
  lasgd_comm* comm = nullptr;
  int world = 1, rank = 0, dtype = LASGD_F32;
  size_t n = 0;
  void* x = nullptr;
  void* m = nullptr;
  void* delta = nullptr;
  void* snap[2] = {nullptr, nullptr};
  void* xbar = nullptr;
  lasgd_worker_config cfg;
  cudaStream_t compute = nullptr, side = nullptr;
  unsigned long long* nonfinite = nullptr;
  // protocol state (mirrors NodeState, optimizer.py:79-104)
  int tau = 0, snap_idx = 0;
  long long local_clock = 0, global_clock = 0;
  bool mom_started = false, delta_fresh = false;
  unsigned long long seq = 0;
  cudaEvent_t ev_snap = nullptr;
  std::vector<cudaEvent_t> lead;  // adaptive run-ahead throttle ring
  size_t lead_pos = 0;
  long long lead_count = 0;
  // graph replay (deterministic schedule): the device round descriptor the captured
  // launches read and advance, and the learning-rate table it indexes
  DevRound* rd = nullptr;
  double* lr_dev = nullptr;
  size_t lr_len = 0;
  bool dyn = false;       // issuing into a capture: launches take their scalars from rd
  cudaStream_t cap_stream = nullptr;  // lasgd_worker_graph_capture records here
  bool rd_dirty = true;   // eager launches ran since rd was last written
  unsigned long long rd_seq = 0;  // communicator launches rd accounts for
  // instrumentation
  bool timed = false;
  std::vector<TimingRec> recs;
  std::vector<cudaEvent_t> pool;
  long long launches[K_KINDS] = {0};
  long long tau_hist[LASGD_TAU_HIST] = {0};
};

namespace {
struct NvtxRange {  // one named range per worker call
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

static cudaEvent_t pool_get(lasgd_worker* w) {
  if (!w->pool.empty()) {
    cudaEvent_t e = w->pool.back();
    w->pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// Issue one kernel launch with optional timing events around it on `s`.
template <typename F>
static int issue(lasgd_worker* w, int kind, cudaStream_t s, F&& fn) {
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (w->timed) {
    e0 = pool_get(w);
    e1 = pool_get(w);
    cudaEventRecord(e0, s);
  }
  int rc = fn();
  if (rc) return rc;
  if (w->timed) {
    cudaEventRecord(e1, s);
    w->recs.push_back({kind, e0, e1});
  }
  w->launches[kind]++;
  return LASGD_OK;
}

static lasgd_sgd_params sgd_params(const lasgd_worker* w, double lr) {
  lasgd_sgd_params p;
  p.lr = lr;
  p.momentum = w->cfg.momentum;
  p.dampening = w->cfg.dampening;
  p.weight_decay = w->cfg.weight_decay;
  p.nesterov = w->cfg.nesterov;
  p.first_step = !w->mom_started;
  p.delta_reset = w->delta_fresh;
  return p;
}

static bool finalize_mode(const lasgd_worker* w) { return w->cfg.mode == 1 && w->cfg.alpha == 1.0; }

static int submit_allreduce(lasgd_worker* w, int slot) {
  LASGD_CUDA_TRY(cudaEventRecord(w->ev_snap, w->compute));
  LASGD_CUDA_TRY(cudaStreamWaitEvent(w->side, w->ev_snap, 0));
  unsigned long long s = 0;
  // (ALGO_PUSH here is the push mean: the all-reduce with every byte moved by stores)
  const int algo = comm_side_algo(w->comm, w->cfg.algo);
  int rc = issue(w, K_ALLREDUCE, w->side,
                 [&] { return lasgd_comm_allreduce(w->comm, slot, algo, (void*)w->side, &s); });
  if (rc) return rc;
  w->seq = s;
  return LASGD_OK;
}

static void close_round_bookkeeping(lasgd_worker* w, int closed_tau) {
  w->tau_hist[closed_tau < LASGD_TAU_HIST ? closed_tau : LASGD_TAU_HIST - 1]++;
  w->snap_idx = 1 - w->snap_idx;
  w->delta_fresh = w->delta != nullptr;
  w->tau = 0;
  w->global_clock++;
}

// Round boundary of the overlap pipeline (optimizer.py:152-178 + the next submit).
static int close_round(lasgd_worker* w) {
  NvtxRange range("lasgd.close_round");
  const int cur = w->snap_idx, nxt = 1 - cur;
  int rc;
  if (w->world == 1) {
    // optimizer.py:168-169: P == 1 keeps the live model; only the snapshot moves
    rc = issue(w, K_SNAPSHOT, w->compute,
               [&] { return lasgd_snapshot(w->snap[nxt], w->x, w->n, w->dtype, (void*)w->compute); });
  } else {
    rc = lasgd_comm_stream_wait(w->comm, w->seq, (void*)w->compute);
    if (rc) return rc;
    if (finalize_mode(w))
      rc = issue(w, K_FINALIZE, w->compute, [&] {
        return lasgd_finalize(w->x, w->snap[nxt], w->xbar, w->delta, w->n, w->dtype, w->nonfinite, (void*)w->compute);
      });
    else
      rc = issue(w, K_PULL, w->compute, [&] {
        return lasgd_elastic_pull(w->x, w->snap[nxt], w->snap[cur], w->xbar, w->n, w->dtype, w->cfg.alpha,
                                  w->nonfinite, (void*)w->compute);
      });
  }
  if (rc) return rc;
  close_round_bookkeeping(w, w->tau);
  if (w->world > 1) return submit_allreduce(w, w->snap_idx);
  return LASGD_OK;
}

static RoundAdv make_adv(const lasgd_worker* w, int close) {
  RoundAdv a;
  a.rd = w->rd;
  a.steps = 1;
  a.close = close;
  a.has_mom = w->m != nullptr;
  a.has_delta = w->delta != nullptr;
  a.seq_inc = 0;
  return a;
}

// Graph capture, one rank: the local step, with the next snapshot fused in when the
// step closes a round (K7 at P = 1, optimizer.py:168-169 — both pipelines).
static int dyn_step(lasgd_worker* w, const void* g, int close) {
  lasgd_sgd_params p = sgd_params(w, 0.0);  // lr, first_step, delta_reset come from rd
  void* snaps[2] = {w->snap[0], w->snap[1]};
  return issue(w, close ? K_FUSED : K_SGD, w->compute, [&] {
    return sgd_step_dyn(w->dtype, w->x, g, w->m, w->delta, close ? snaps : nullptr, w->n, &p, w->nonfinite,
                        (void*)w->compute, make_adv(w, close));
  });
}

static int fused_step(lasgd_worker* w, const void* g, double lr) {
  const int cur = w->snap_idx, nxt = 1 - cur;
  lasgd_sgd_params p = sgd_params(w, lr);
  const int mode = finalize_mode(w) ? 1 : 0;
  int rc;
  if (w->dyn && w->world == 1) {
    rc = dyn_step(w, g, 1);
  } else if (w->dyn) {
    unsigned long long s = 0;
    RoundAdv adv = make_adv(w, 1);
    adv.seq_inc = 1;
    rc = issue(w, K_FUSED, w->compute, [&] {
      return comm_fused_round_dyn(w->comm, cur, w->cfg.algo, w->x, g, w->m, w->delta, &p, w->cfg.alpha, mode,
                                  w->cfg.fused_nblocks, w->nonfinite, (void*)w->compute, adv, &s);
    });
    if (!rc) w->seq = s;
  } else if (w->world == 1) {
    void* xs[1] = {w->x};
    const void* gs[1] = {g};
    void* ms[1] = {w->m};
    void* ds[1] = {w->delta};
    const void* ss[1] = {w->snap[cur]};
    void* ns[1] = {w->snap[nxt]};
    rc = issue(w, K_FUSED, w->compute, [&] {
      return lasgd_fused_round_virtual(1, LASGD_ALGO_ONESHOT, xs, gs, w->m ? ms : nullptr, w->delta ? ds : nullptr,
                                       ss, nullptr, ns, w->n, w->dtype, &p, w->cfg.alpha, mode,
                                       w->cfg.fused_nblocks, w->nonfinite, (void*)w->compute);
    });
  } else {
    unsigned long long s = 0;
    rc = issue(w, K_FUSED, w->compute, [&] {
      return lasgd_comm_fused_round(w->comm, cur, w->cfg.algo, w->x, g, w->m, w->delta, &p, w->cfg.alpha, mode,
                                    w->cfg.fused_nblocks, w->nonfinite, (void*)w->compute, &s);
    });
    if (!rc) w->seq = s;
  }
  if (rc) return rc;
  w->mom_started = w->m != nullptr;
  w->local_clock++;
  close_round_bookkeeping(w, w->tau + 1);
  return 1;
}

// Round boundary of the deterministic overlap pipeline (P > 1): the previous round's
// mean has been on its way for a whole round, so the compute stream waits for it and
// applies the local step AND the pull / finalize in one pass (lasgd_sgd_pull, 8B instead
// of K5 5B + K4 5B), then hands the new snapshot to the side stream.
static int overlap_boundary(lasgd_worker* w, const void* g, double lr) {
  NvtxRange range("lasgd.close_round");
  const int cur = w->snap_idx, nxt = 1 - cur;
  lasgd_sgd_params p = sgd_params(w, lr);
  int rc = lasgd_comm_stream_wait(w->comm, w->seq, (void*)w->compute);
  if (rc) return rc;
  const int mode = finalize_mode(w) ? 1 : 0;
  rc = issue(w, K_SGD_PULL, w->compute, [&] {
    return lasgd_sgd_pull(w->x, g, w->m, w->delta, w->snap[nxt], w->snap[cur], w->xbar, w->n, w->dtype, &p,
                          w->cfg.alpha, mode, w->nonfinite, (void*)w->compute);
  });
  if (rc) return rc;
  w->mom_started = w->m != nullptr;
  w->local_clock++;
  close_round_bookkeeping(w, w->tau + 1);
  rc = submit_allreduce(w, w->snap_idx);
  return rc ? rc : 1;
}

extern "C" int lasgd_worker_create(lasgd_comm* comm, void* x, void* m, void* delta, void* snap0, void* snap1,
                                   size_t n, int dtype, const lasgd_worker_config* cfg, void* compute_stream,
                                   void* side_stream, unsigned long long* nonfinite, lasgd_worker** out) {
  if (!out || !cfg || !x) return fail(LASGD_ERR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  if (cfg->sync_period < 1) return fail(LASGD_ERR_INVALID_ARGUMENT, "sync_period must be >= 1");
  if (!(cfg->alpha > 0.0 && cfg->alpha <= 1.0)) return fail(LASGD_ERR_INVALID_ARGUMENT, "alpha must be in (0, 1]");
  if (cfg->mode != 0 && cfg->mode != 1) return fail(LASGD_ERR_INVALID_ARGUMENT, "mode must be 0 (pull) or 1 (delta)");
  if (cfg->mode == 1 && !delta) return fail(LASGD_ERR_INVALID_ARGUMENT, "delta mode needs the delta buffer");
  if (cfg->pipeline != 0 && cfg->pipeline != 1) return fail(LASGD_ERR_INVALID_ARGUMENT, "pipeline must be 0 or 1");
  if (cfg->pipeline == 1 && cfg->adaptive)
    return fail(LASGD_ERR_INVALID_ARGUMENT, "the fused pipeline implements the deterministic schedule only");
  if (cfg->momentum != 0.0 && !m) return fail(LASGD_ERR_INVALID_ARGUMENT, "momentum needs m");
  lasgd_worker* w = new lasgd_worker();
  w->comm = comm;
  w->x = x;
  w->m = m;
  w->delta = delta;
  w->n = n;
  w->dtype = dtype;
  w->cfg = *cfg;
  if (w->cfg.tau_max < 1) w->cfg.tau_max = w->cfg.sync_period;
  w->compute = reinterpret_cast<cudaStream_t>(compute_stream);
  w->side = reinterpret_cast<cudaStream_t>(side_stream);
  w->nonfinite = nonfinite;
  if (comm) {
    int wr = 0;
    if ((wr = lasgd_comm_info(comm, &w->rank, &w->world, &w->xbar)) != 0) {
      delete w;
      return wr;
    }
    // the kernels stream the caller's n over the communicator's buffers (and comm->n
    // over the caller's): a mismatch would read and write out of bounds, peers included
    size_t cn = 0;
    int cdt = -1;
    if ((wr = lasgd_comm_shape(comm, &cn, &cdt)) != 0) {
      delete w;
      return wr;
    }
    if (cn != n || cdt != dtype) {
      delete w;
      return fail(LASGD_ERR_DIMENSION, "communicator holds %zu elements of type %d, the worker %zu of type %d", cn,
                  cdt, n, dtype);
    }
    if (lasgd_comm_buffer(comm, 0, &w->snap[0]) || lasgd_comm_buffer(comm, 1, &w->snap[1])) {
      delete w;
      return LASGD_ERR_INVALID_ARGUMENT;
    }
  } else {
    if (!snap0 || !snap1) {
      delete w;
      return fail(LASGD_ERR_INVALID_ARGUMENT, "without a communicator two snapshot buffers are required");
    }
    w->snap[0] = snap0;
    w->snap[1] = snap1;
  }
  cudaError_t e = cudaEventCreateWithFlags(&w->ev_snap, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    delete w;
    return cuda_fail(e, "cudaEventCreate");
  }
  // Algorithm 1 lines 1-5: snapshot = x0, submit round 0 (overlap pipeline)
  int rc = issue(w, K_SNAPSHOT, w->compute,
                 [&] { return lasgd_snapshot(w->snap[0], w->x, w->n, w->dtype, (void*)w->compute); });
  if (!rc && comm) rc = lasgd_comm_invalidate_staging(comm);  // slot 0 rewritten: re-stage before a push round
  // side-stream all-reduces (overlap pipeline) wait for late peers in a one-warp gate
  // instead of a CTA per SM next to the compute stream's forward/backward
  if (!rc && comm) rc = lasgd_comm_set_gate(comm, w->cfg.pipeline == 0);
  if (!rc && w->world > 1 && w->cfg.sync && w->cfg.pipeline == 0) rc = submit_allreduce(w, 0);
  if (rc) {
    lasgd_worker_destroy(w);
    return rc;
  }
  *out = w;
  return LASGD_OK;
}

extern "C" int lasgd_worker_step(lasgd_worker* w, const void* g, double lr) {
  if (!w || !g) return fail(LASGD_ERR_INVALID_ARGUMENT, "null argument");
  NvtxRange range(w->dyn ? "lasgd.step (captured)" : "lasgd.step");
  if (!w->dyn) w->rd_dirty = true;
  const bool closes = w->cfg.sync && !w->cfg.adaptive && w->tau + 1 == w->cfg.sync_period;
  // deterministic round boundary: one pass — the fused round (fused pipeline, and P = 1
  // where the boundary is the local step with the snapshot fused in), or the local step
  // fused with the pull of the mean the side stream delivered (overlap pipeline)
  if ((w->cfg.pipeline == 1 || w->world == 1) && closes) return fused_step(w, g, lr);
  if (closes && !w->dyn) return overlap_boundary(w, g, lr);
  lasgd_sgd_params p = sgd_params(w, lr);
  int rc = w->dyn ? dyn_step(w, g, 0) : issue(w, K_SGD, w->compute, [&] {
    return lasgd_sgd_step(w->x, g, w->m, w->delta, w->n, w->dtype, &p, w->nonfinite, (void*)w->compute);
  });
  if (rc) return rc;
  w->mom_started = w->m != nullptr;
  w->delta_fresh = false;
  w->tau++;
  w->local_clock++;
  if (!w->cfg.sync) return 0;
  if (w->cfg.adaptive) {
    if (w->cfg.max_host_lead > 0) {
      if (w->lead.empty()) {
        w->lead.resize(w->cfg.max_host_lead);
        for (auto& ev : w->lead) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
      }
      cudaEvent_t& slot = w->lead[w->lead_pos];
      if (w->lead_count >= w->cfg.max_host_lead) {
        // Bounded wait: if the compute stream is stalled on a peer's next launch (a
        // rank that closed more rounds than its peers, e.g. at the end of a run), an
        // unbounded host wait would deadlock against the peer's drain.
        struct timespec t0, t;
        clock_gettime(CLOCK_MONOTONIC, &t0);
        const double cap = w->cfg.max_host_wait_us > 0 ? w->cfg.max_host_wait_us * 1e-6 : 0.25;
        while (cudaEventQuery(slot) == cudaErrorNotReady) {
          clock_gettime(CLOCK_MONOTONIC, &t);
          if ((t.tv_sec - t0.tv_sec) + 1e-9 * (t.tv_nsec - t0.tv_nsec) > cap) break;
          struct timespec ns = {0, 20000};
          nanosleep(&ns, nullptr);
        }
      }
      cudaEventRecord(slot, w->compute);
      w->lead_pos = (w->lead_pos + 1) % w->lead.size();
      w->lead_count++;
    }
    int done = 1;
    if (w->world > 1) {
      done = lasgd_comm_query(w->comm, w->seq);
      if (done < 0) return done;
      // The host runs ahead of its GPU, so the completion flag alone is stale: a rank
      // whose peers already entered a later launch is the round's laggard — its launch
      // is done or about to be, and the peers wait for its next one.  Close now.
      if (done == 0 && w->tau < w->cfg.tau_max) {
        const int ahead = lasgd_comm_peers_ahead(w->comm, w->seq);
        if (ahead < 0) return ahead;
        done = ahead;
      }
    }
    if (done == 1 || w->tau >= w->cfg.tau_max) {
      rc = close_round(w);
      return rc ? rc : 1;
    }
    return 0;
  }
  if (w->tau == w->cfg.sync_period) {
    rc = close_round(w);
    return rc ? rc : 1;
  }
  return 0;
}

extern "C" int lasgd_worker_drain(lasgd_worker* w) {
  if (!w) return fail(LASGD_ERR_INVALID_ARGUMENT, "null worker");
  if (w->world > 1 && w->seq && w->cfg.pipeline == 0) return lasgd_comm_stream_wait(w->comm, w->seq, (void*)w->compute);
  return LASGD_OK;
}

extern "C" int lasgd_worker_get_state(lasgd_worker* w, lasgd_worker_state* s) {
  if (!w || !s) return fail(LASGD_ERR_INVALID_ARGUMENT, "null argument");
  s->tau_i = w->tau;
  s->snap_idx = w->snap_idx;
  s->local_clock = w->local_clock;
  s->global_clock = w->global_clock;
  s->seq = w->seq;
  s->momentum_started = w->mom_started;
  s->delta_fresh = w->delta_fresh;
  for (int k = 0; k < LASGD_KERNEL_KINDS; ++k) s->launches[k] = w->launches[k];
  for (int t = 0; t < LASGD_TAU_HIST; ++t) s->tau_hist[t] = w->tau_hist[t];
  return LASGD_OK;
}

extern "C" int lasgd_worker_set_timing(lasgd_worker* w, int on) {
  if (!w) return fail(LASGD_ERR_INVALID_ARGUMENT, "null worker");
  w->timed = on != 0;
  return LASGD_OK;
}

// Durations (ms) of the timed launches of `kind` since the last reset, oldest first.
// The caller synchronises first.  Returns the number written.
extern "C" int lasgd_worker_timings(lasgd_worker* w, int kind, float* out, int max) {
  if (!w || !out) return fail(LASGD_ERR_INVALID_ARGUMENT, "null argument");
  int k = 0;
  for (const auto& r : w->recs) {
    if (r.kind != kind) continue;
    if (k >= max) break;
    float ms = 0.f;
    LASGD_CUDA_TRY(cudaEventElapsedTime(&ms, r.e0, r.e1));
    out[k++] = ms;
  }
  return k;
}

extern "C" int lasgd_worker_reset_stats(lasgd_worker* w) {
  if (!w) return fail(LASGD_ERR_INVALID_ARGUMENT, "null worker");
  for (auto& r : w->recs) {
    w->pool.push_back(r.e0);
    w->pool.push_back(r.e1);
  }
  w->recs.clear();
  memset(w->launches, 0, sizeof(w->launches));
  memset(w->tau_hist, 0, sizeof(w->tau_hist));
  return LASGD_OK;
}

// ---------------------------------------------------------------- graph replay
// Host mirror of the protocol state, saved at capture begin and put back at the end:
// the captured launches advance it as they are issued; a replay applies that advance.
struct lasgd_graph_saved {
  int tau, snap_idx;
  long long clock, gclock;
  bool mom, dfresh;
  unsigned long long seq;
  CommMirror comm;  // communicator bookkeeping (world > 1)
  long long launches[K_KINDS], hist[LASGD_TAU_HIST];
};

struct lasgd_graph {
  lasgd_worker* w = nullptr;
  cudaGraphExec_t exec = nullptr;
  int steps = 0, tau0 = 0;
  lasgd_graph_saved saved;
  CommMirror comm_after;  // the communicator bookkeeping after the captured launches
  int snap_after = 0;     // the worker's snapshot slot after the captured steps
  // what one replay does to the host mirror of the protocol state
  long long d_clock = 0, d_rounds = 0;
  bool mom_after = false, delta_fresh_after = false;
  long long d_launches[K_KINDS] = {0};
  long long d_tau_hist[LASGD_TAU_HIST] = {0};
};

namespace lasgd {
__global__ void k_round_set(DevRound* r, unsigned long long clock, unsigned long long seq, const double* lr,
                            unsigned long long lr_len, int snap_idx, int mom_started, int delta_fresh) {
  r->clock = clock;
  r->seq = seq;
  r->lr = lr;
  r->lr_len = lr_len;
  r->lr_now = lr[clock < lr_len ? clock : lr_len - 1];
  r->snap_idx = snap_idx;
  r->mom_started = mom_started;
  r->delta_fresh = delta_fresh;
  r->arrive = 0u;
}
}  // namespace lasgd

extern "C" int lasgd_worker_set_lr_table(lasgd_worker* w, const double* lr, size_t len) {
  if (!w || !lr || len == 0) return fail(LASGD_ERR_INVALID_ARGUMENT, "null or empty learning-rate table");
  for (size_t i = 0; i < len; ++i)
    if (!(lr[i] > 0.0)) return fail(LASGD_ERR_INVALID_ARGUMENT, "learning rate %zu is %g, must be positive", i, lr[i]);
  // the old table may still be read by queued replays
  LASGD_CUDA_TRY(cudaStreamSynchronize(w->compute));
  if (w->lr_dev) cudaFree(w->lr_dev);
  w->lr_dev = nullptr;
  w->lr_len = 0;
  if (!w->rd) LASGD_CUDA_TRY(cudaMalloc(&w->rd, sizeof(DevRound)));  // (no allocation may happen inside a capture)
  LASGD_CUDA_TRY(cudaMalloc(&w->lr_dev, len * sizeof(double)));
  LASGD_CUDA_TRY(cudaMemcpy(w->lr_dev, lr, len * sizeof(double), cudaMemcpyHostToDevice));
  w->lr_len = len;
  w->rd_dirty = true;
  return LASGD_OK;
}

static int capture_check(lasgd_worker* w) {
  if (w->cfg.adaptive) return fail(LASGD_ERR_UNSUPPORTED, "graph replay needs the deterministic schedule");
  if (w->world > 1 && w->cfg.sync && w->cfg.pipeline != 1)
    return fail(LASGD_ERR_UNSUPPORTED, "multi-rank graph replay needs the fused pipeline");
  if (w->timed) return fail(LASGD_ERR_STATE, "per-launch timing cannot be captured");
  if (w->dyn) return fail(LASGD_ERR_STATE, "a capture is already open on this worker");
  if (!w->lr_dev || !w->rd)
    return fail(LASGD_ERR_STATE, "set the learning-rate table first (lasgd_worker_set_lr_table)");
  return LASGD_OK;
}

static void capture_open(lasgd_worker* w, lasgd_graph* gr) {
  lasgd_graph_saved& v = gr->saved;
  gr->w = w;
  gr->tau0 = w->tau;
  v.tau = w->tau;
  v.snap_idx = w->snap_idx;
  v.clock = w->local_clock;
  v.gclock = w->global_clock;
  v.mom = w->mom_started;
  v.dfresh = w->delta_fresh;
  v.seq = w->seq;
  if (w->comm) comm_mirror_get(w->comm, &v.comm);
  memcpy(v.launches, w->launches, sizeof(v.launches));
  memcpy(v.hist, w->tau_hist, sizeof(v.hist));
  w->dyn = true;
}

// Close the capture: record what the captured steps did, put the mirror back.
static int capture_close(lasgd_worker* w, lasgd_graph* gr) {
  const lasgd_graph_saved& v = gr->saved;
  w->dyn = false;
  gr->steps = (int)(w->local_clock - v.clock);
  gr->d_clock = w->local_clock - v.clock;
  gr->d_rounds = w->global_clock - v.gclock;
  gr->mom_after = w->mom_started;
  gr->delta_fresh_after = w->delta_fresh;
  const int tau_end = w->tau;
  gr->snap_after = w->snap_idx;
  for (int k = 0; k < K_KINDS; ++k) gr->d_launches[k] = w->launches[k] - v.launches[k];
  for (int t = 0; t < LASGD_TAU_HIST; ++t) gr->d_tau_hist[t] = w->tau_hist[t] - v.hist[t];
  w->tau = v.tau;
  w->snap_idx = v.snap_idx;
  w->local_clock = v.clock;
  w->global_clock = v.gclock;
  w->mom_started = v.mom;
  w->delta_fresh = v.dfresh;
  w->seq = v.seq;
  if (w->comm) {
    comm_mirror_get(w->comm, &gr->comm_after);
    comm_mirror_set(w->comm, v.comm);
  }
  memcpy(w->launches, v.launches, sizeof(v.launches));
  memcpy(w->tau_hist, v.hist, sizeof(v.hist));
  if (w->cfg.sync && tau_end != gr->tau0)
    return fail(LASGD_ERR_INVALID_ARGUMENT, "a graph holds whole rounds: %d steps, sync period %d", gr->steps,
                w->cfg.sync_period);
  return LASGD_OK;
}

extern "C" int lasgd_worker_graph_capture(lasgd_worker* w, int steps, const void* const* g, lasgd_graph** out) {
  if (!w || !g || !out) return fail(LASGD_ERR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  if (steps < 1) return fail(LASGD_ERR_INVALID_ARGUMENT, "steps must be >= 1");
  for (int t = 0; t < steps; ++t)
    if (!g[t]) return fail(LASGD_ERR_INVALID_ARGUMENT, "gradient %d is null", t);
  if (w->cfg.sync && steps % w->cfg.sync_period)
    return fail(LASGD_ERR_INVALID_ARGUMENT, "a graph holds whole rounds: %d steps, sync period %d", steps,
                w->cfg.sync_period);
  int rc = capture_check(w);
  if (rc) return rc;
  // capture on a private stream (the compute stream may be the legacy default stream,
  // which cannot be captured); the graph is launched on the compute stream
  if (!w->cap_stream) LASGD_CUDA_TRY(cudaStreamCreateWithFlags(&w->cap_stream, cudaStreamNonBlocking));
  lasgd_graph* gr = new lasgd_graph();
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaStreamBeginCapture(w->cap_stream, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) {
    delete gr;
    return cuda_fail(e, "cudaStreamBeginCapture");
  }
  cudaStream_t compute = w->compute;
  w->compute = w->cap_stream;
  capture_open(w, gr);
  for (int t = 0; t < steps && rc >= 0; ++t) rc = lasgd_worker_step(w, g[t], 0.0);
  const int rc_close = capture_close(w, gr);
  w->compute = compute;
  e = cudaStreamEndCapture(w->cap_stream, &graph);
  if (rc >= 0) rc = rc_close;
  if (rc >= 0 && e != cudaSuccess) rc = cuda_fail(e, "cudaStreamEndCapture");
  if (rc >= 0) {
    e = cudaGraphInstantiate(&gr->exec, graph, 0);
    if (e != cudaSuccess) rc = cuda_fail(e, "cudaGraphInstantiate");
  }
  if (graph) cudaGraphDestroy(graph);
  if (rc < 0) {
    if (gr->exec) cudaGraphExecDestroy(gr->exec);
    delete gr;
    return rc;
  }
  *out = gr;
  return LASGD_OK;
}

extern "C" int lasgd_worker_capture_begin(lasgd_worker* w, lasgd_graph** out) {
  if (!w || !out) return fail(LASGD_ERR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  LASGD_CUDA_TRY(cudaStreamIsCapturing(w->compute, &st));
  if (st != cudaStreamCaptureStatusActive)
    return fail(LASGD_ERR_STATE, "the worker's compute stream is not being captured");
  int rc = capture_check(w);
  if (rc) return rc;
  lasgd_graph* gr = new lasgd_graph();
  capture_open(w, gr);
  *out = gr;
  return LASGD_OK;
}

extern "C" int lasgd_worker_capture_end(lasgd_graph* gr) {
  if (!gr || !gr->w || !gr->w->dyn) return fail(LASGD_ERR_STATE, "no capture open");
  return capture_close(gr->w, gr);
}

extern "C" int lasgd_graph_launch(lasgd_graph* gr) {
  if (!gr) return fail(LASGD_ERR_INVALID_ARGUMENT, "null graph");
  NvtxRange range("lasgd.graph_launch");
  lasgd_worker* w = gr->w;
  if (w->tau != gr->tau0)
    return fail(LASGD_ERR_STATE, "graph captured at local step %d of a round, worker is at step %d", gr->tau0, w->tau);
  if (w->lr_len > 1 && (unsigned long long)(w->local_clock + gr->d_clock) > w->lr_len)
    return fail(LASGD_ERR_STATE, "learning-rate table holds %zu clocks, the replay needs %lld", w->lr_len,
                w->local_clock + gr->d_clock);
  CommMirror cm = {0, 0, 0, -1};
  if (w->comm) {
    // the replayed rounds enter on the end signals of the launch before them: the
    // communicator must be where it was at capture (relative to its latest launch)
    comm_mirror_get(w->comm, &cm);
    const CommMirror& pre = gr->saved.comm;
    auto lag = [](unsigned long long seq, unsigned long long v) { return v ? (long long)(seq - v) : -1LL; };
    // staging parity relative to the snapshot slot (the graph itself is parity-agnostic)
    auto staged = [](int push_slot, int snap) { return push_slot < 0 ? -1 : (push_slot == snap ? 1 : 0); };
    if (staged(cm.push_slot, w->snap_idx) != staged(pre.push_slot, gr->saved.snap_idx) ||
        lag(cm.seq, cm.last_push) != lag(pre.seq, pre.last_push) || lag(cm.seq, cm.end_seq) != lag(pre.seq, pre.end_seq))
      return fail(LASGD_ERR_STATE, "the communicator's last launch differs from the capture's; run one eager round");
    if (cm.seq != w->rd_seq) w->rd_dirty = true;  // launches the descriptor has not seen
  }
  if (w->rd_dirty) {
    k_round_set<<<1, 1, 0, w->compute>>>(w->rd, (unsigned long long)w->local_clock, cm.seq, w->lr_dev,
                                         (unsigned long long)w->lr_len, w->snap_idx, w->mom_started ? 1 : 0,
                                         w->delta_fresh ? 1 : 0);
    LASGD_CUDA_TRY(cudaGetLastError());
    w->rd_dirty = false;
  }
  if (gr->exec) LASGD_CUDA_TRY(cudaGraphLaunch(gr->exec, w->compute));  // else the caller replays its own graph next
  w->local_clock += gr->d_clock;
  w->global_clock += gr->d_rounds;
  if (gr->d_rounds & 1) w->snap_idx ^= 1;
  if (gr->d_clock) {
    w->mom_started = gr->mom_after;
    w->delta_fresh = gr->delta_fresh_after;
  }
  for (int k = 0; k < K_KINDS; ++k) w->launches[k] += gr->d_launches[k];
  for (int t = 0; t < LASGD_TAU_HIST; ++t) w->tau_hist[t] += gr->d_tau_hist[t];
  if (w->comm) {
    const CommMirror& pre = gr->saved.comm;
    const CommMirror& post = gr->comm_after;
    const unsigned long long d = post.seq - pre.seq;
    CommMirror now;
    now.seq = cm.seq + d;
    now.last_push = post.last_push ? now.seq - (post.seq - post.last_push) : 0;
    now.end_seq = post.end_seq ? now.seq - (post.seq - post.end_seq) : 0;
    // w->snap_idx has advanced by the replay already; map the capture's final staging
    // parity (relative to its final slot) onto it
    now.push_slot = post.push_slot < 0 ? -1 : (post.push_slot == gr->snap_after ? w->snap_idx : 1 - w->snap_idx);
    comm_mirror_set(w->comm, now);
    if (d) {
      w->seq = now.seq;
      int rc = comm_record_last(w->comm, (void*)w->compute);
      if (rc) return rc;
    }
    w->rd_seq = now.seq;
  }
  return LASGD_OK;
}

extern "C" int lasgd_graph_destroy(lasgd_graph* gr) {
  if (!gr) return LASGD_OK;
  if (gr->exec) {
    cudaStreamSynchronize(gr->w->compute);
    cudaGraphExecDestroy(gr->exec);
  }
  delete gr;
  return LASGD_OK;
}

extern "C" int lasgd_worker_destroy(lasgd_worker* w) {
  if (!w) return LASGD_OK;
  cudaStreamSynchronize(w->compute);
  if (w->side) cudaStreamSynchronize(w->side);
  if (w->rd) cudaFree(w->rd);
  if (w->lr_dev) cudaFree(w->lr_dev);
  if (w->cap_stream) cudaStreamDestroy(w->cap_stream);
  for (auto& r : w->recs) {
    cudaEventDestroy(r.e0);
    cudaEventDestroy(r.e1);
  }
  for (auto e : w->pool) cudaEventDestroy(e);
  for (auto e : w->lead) cudaEventDestroy(e);
  if (w->ev_snap) cudaEventDestroy(w->ev_snap);
  delete w;
  return LASGD_OK;
}
