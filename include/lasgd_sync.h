/*
 * lasgd_sync.h — C ABI of the B200-native LASGD parameter-synchronisation path.
 *
 * Drop-in boundary for the reference's Python plug-in points
 * (/root/reference/pkg/src/lasgd; the reference has no FFI, its boundary is
 * duck-typed Python — SURVEY.md §8(b)).  Every entry point below names the
 * reference function it replaces.  Plain pointers and sizes only: device
 * pointers are raw CUDA device addresses, `stream` is a cudaStream_t passed as
 * void* (NULL = legacy default stream).  All kernel entry points are
 * stream-ordered and non-blocking.
 *
 * Return value: 0 on success, a negative LASGD_ERR_* code otherwise; the
 * Python layer maps codes to the reference exception types (see
 * paper_2203_13085_b200/_native.py).  lasgd_last_error() returns a
 * thread-local diagnostic for the most recent failure on the calling thread.
 *
 * Element type: LASGD_F32 (the product path, bit-exact against the fp32
 * restatement) or LASGD_F64 (bit-exact against the f64 reference itself).
 * Arithmetic contract: every product and sum is separately rounded (no FMA),
 * scalars are rounded to the element type first, exactly like the
 * reference's numpy expressions (params.py:87).
 */
#ifndef LASGD_SYNC_H
#define LASGD_SYNC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LASGD_ABI_VERSION 1

/* error codes (→ Python exception in _native.py) */
#define LASGD_OK 0
#define LASGD_ERR_INVALID_ARGUMENT (-1) /* ValueError                       */
#define LASGD_ERR_DIMENSION (-2)        /* DimensionMismatchError, params.py:15 */
#define LASGD_ERR_NONFINITE (-3)        /* NonFiniteError, params.py:19       */
#define LASGD_ERR_CUDA (-4)             /* RuntimeError (CUDA runtime)        */
#define LASGD_ERR_COLLECTIVE (-5)       /* CollectiveFailure, collective.py:26 */
#define LASGD_ERR_TIMEOUT (-6)          /* TimeoutError (host wait)           */
#define LASGD_ERR_STATE (-7)            /* RuntimeError (protocol misuse)     */
#define LASGD_ERR_UNSUPPORTED (-8)      /* e.g. world size > LASGD_MAX_RANKS  */

/* element types */
#define LASGD_F32 0
#define LASGD_F64 1

/* all-reduce algorithms */
#define LASGD_ALGO_AUTO 0
#define LASGD_ALGO_ONESHOT 1
#define LASGD_ALGO_TWOSHOT 2
#define LASGD_ALGO_NVLS 4 /* all-reduce only, NVLS communicators: reduced inside the NVSwitch
                            (tolerance mode, see lasgd_comm_nvls_bind) */
#define LASGD_ALGO_PUSH 3 /* data moved by remote stores.  Fused round: P = 2 mirrors the peer's
                             snapshot; P >= 3 owners reduce locally staged chunks, means pushed.
                             All-reduce: the push mean (scatter to owners' staging, owner reduces,
                             means stored into every rank), bit-identical to the two-shot */
#define LASGD_ALGO_CE 5 /* all-reduce only: the two-shot mean with the NVLink traffic moved by the
                           copy engines (SMs reduce the own chunk and flip flags); bit-identical to
                           LASGD_ALGO_TWOSHOT */

#define LASGD_MAX_RANKS 8
#define LASGD_MAX_BLOCKS 512
#define LASGD_IPC_HANDLE_BYTES 64

int lasgd_abi_version(void);
const char* lasgd_strerror(int code);
const char* lasgd_last_error(void);

/* ---- rank-local streaming kernels (HBM-bound) -------------------------- */

/* Occupancy of the streaming kernels (CTAs of 256 threads per SM, default 2).
 * Lower values leave room for the side-stream all-reduce to run concurrently. */
int lasgd_set_stream_ctas_per_sm(int ctas_per_sm);

/* K0: out = a*u + b*v.  Replaces params.py:80-89 `blend` (out-of-place). */
int lasgd_blend(void* out, double a, const void* u, double b, const void* v, size_t n, int dtype,
                unsigned long long* nonfinite, void* stream);

/* K1: snap = x.  Replaces the snapshot of optimizer.py:172-173 (the reference
 * aliases an immutable vector; the flat fp32 buffer needs a real copy). */
int lasgd_snapshot(void* snap, const void* x, size_t n, int dtype, void* stream);

typedef struct {
  double lr;           /* eta_t (problems.py:355 lr_at); kernel uses (T)(-lr)      */
  double momentum;     /* 0 = reference sgd_local_step                            */
  double dampening;
  double weight_decay;
  int nesterov;
  int first_step;      /* momentum buffer := direction (torch semantics)          */
  int delta_reset;     /* delta := 0 + (-lr)*d  (fresh accumulator, optimizer.py:174) */
} lasgd_sgd_params;

/* K5: fused local step on the flat buffer.
 *   d = g (+ wd*x);  m = first ? d : mu*m + (1-damp)*d;  d = nesterov ? d + mu*m : m;
 *   x = x + (-lr)*d;  delta = (reset ? 0 : delta) + (-lr)*d   (delta nullable)
 * With momentum = wd = 0 this is exactly optimizer.py:145-146 (`sgd_local_step`).
 * m may be NULL when momentum == 0. */
int lasgd_sgd_step(void* x, const void* g, void* m, void* delta, size_t n, int dtype,
                   const lasgd_sgd_params* p, unsigned long long* nonfinite, void* stream);

/* K4a: elastic pull x -= alpha*(snap - xbar), in blend order
 *   diff = 1*snap + (-1)*xbar;  x = 1*x + (-alpha)*diff;  snap_next = x (nullable).
 * Replaces Algorithm 1 line 9a for alpha = 1 and the
 * elastic pull rule of optimizer.py:256-257 for alpha in (0,1]. */
int lasgd_elastic_pull(void* x, void* snap_next, const void* snap, const void* xbar, size_t n, int dtype,
                       double alpha, unsigned long long* nonfinite, void* stream);

/* K5 + K4 in one pass — the round boundary of the deterministic overlap pipeline, once
 * the (previous round's) mean has landed: the local step of lasgd_sgd_step, then mode 0
 * the pull x -= alpha*(snap - xbar) or mode 1 the finalize x = xbar + delta'; snap_next =
 * x.  Bit-identical to lasgd_sgd_step followed by lasgd_elastic_pull / lasgd_finalize.
 * Replaces optimizer.py:145-146 + 170-174 (Algorithm 1 lines 8-9a). */
int lasgd_sgd_pull(void* x, const void* g, void* m, void* delta, void* snap_next, const void* snap, const void* xbar,
                   size_t n, int dtype, const lasgd_sgd_params* p, double alpha, int mode,
                   unsigned long long* nonfinite, void* stream);

/* K4b: reference finalize new = 1*z + 1*delta; x = new; snap_next = new (nullable).
 * delta may be NULL: the accumulator is zero (no local step since the previous
 * finalize reset it, optimizer.py:174), so new = z + 0.
 * Replaces optimizer.py:170-174 (`lasgd_finalize_round`, P > 1 branch). */
int lasgd_finalize(void* x, void* snap_next, const void* z, const void* delta, size_t n, int dtype,
                   unsigned long long* nonfinite, void* stream);

/* ---- mean all-reduce over ranks emulated on ONE device ------------------ */

/* Replaces collective.py:154-203 (`execute_allreduce`) for P virtual ranks
 * whose contributions all live on the calling device — the GPU analogue of
 * LoopbackTransport (collective.py:229-287).  srcs / outs are HOST arrays of
 * device pointers.  algo ONESHOT computes outs[0..n_out) directly from all P
 * sources; TWOSHOT runs the reduce-scatter of every virtual rank into outs[r]
 * (n_out must equal P) and then the all-gather, exercising exactly the
 * slicing of the multi-GPU two-shot kernel without its barriers.
 * Results are bit-identical to the reference ring order. */
int lasgd_mean_virtual(void* const* outs, int n_out, const void* const* srcs, int P, size_t n, int dtype,
                       int algo, int nblocks, unsigned long long* nonfinite, void* stream);

/* K8 (push round) over P virtual ranks on ONE device — test path.  snaps = every
 * rank's current snapshot (parity `cur`), stages = every rank's staging area of
 * 2 * P * lasgd_push_stage_elems(n, P, dtype) elements; init = 1 stages the current
 * snapshots first (the communicator does this on its first push round). */
int lasgd_fused_push_virtual(int P, void* const* x, const void* const* g, void* const* m, void* const* delta,
                             const void* const* snaps, void* const* snap_next, void* const* xbars,
                             void* const* stages, int cur, int init, size_t n, int dtype,
                             const lasgd_sgd_params* sgd, double alpha, int mode, int nblocks,
                             unsigned long long* nonfinite, void* stream);
size_t lasgd_push_stage_elems(size_t n, int P, int dtype);

/* ---- multi-GPU communicator (NVLink P2P through NVSwitch) -------------- */

typedef struct lasgd_comm lasgd_comm;

typedef struct {
  int nblocks;          /* SM budget: CTAs of the all-reduce kernel (<= LASGD_MAX_BLOCKS)     */
  int threads;          /* threads per CTA (multiple of 32 in [64, 256]; <= 128 regs each)     */
  double timeout_s;     /* watchdog for a peer flag (→ CollectiveFailure), e.g. 30.0          */
  long long fault_seq;  /* TEST KNOB: skip this rank's flag writes in launch #fault_seq (-1 off) */
  int fault_phase;      /* 0 entry barrier, 1 mid barrier, 2 end-of-round signal              */
} lasgd_comm_config;

/* Allocates this rank's IPC-exportable region: signal pad + snapshot slot 0/1
 * + mean buffer (n elements each, 256-B aligned) + a host-mapped status block. */
int lasgd_comm_create(int rank, int world, int device, size_t n, int dtype, const lasgd_comm_config* cfg,
                      lasgd_comm** out);
/* Export this rank's region handle (LASGD_IPC_HANDLE_BYTES bytes into `out`). */
int lasgd_comm_ipc_handle(lasgd_comm* c, void* out);
/* Map every peer's region; `handles` = world * LASGD_IPC_HANDLE_BYTES bytes in rank order. */
int lasgd_comm_open(lasgd_comm* c, const void* handles);
/* which: 0 = snapshot slot 0, 1 = snapshot slot 1, 2 = mean (xbar). */
int lasgd_comm_buffer(lasgd_comm* c, int which, void** ptr);

/* K2/K3 (+K6 flags): xbar = mean over ranks of snapshot slot `snap_slot`, in the
 * reference ring's per-chunk rotated order (bit-identical on every rank).
 * Replaces LoopbackTransport.submit / execute_allreduce (collective.py:248-260,
 * 154-203).  Every rank must issue the same sequence of calls.  *seq receives
 * this launch's sequence number for query/wait. */
int lasgd_comm_allreduce(lasgd_comm* c, int snap_slot, int algo, void* stream, unsigned long long* seq);

/* K7: the fused round boundary of the deterministic schedule, one pass per element:
 *   K5 local step on (x, g, m[, delta]);  xbar = ring-order mean of every rank's
 *   snapshot slot `snap_slot`, read from the peers over NVLink;
 *   mode 0 (pull):     x = x + (-alpha)*(snap_own + (-1)*xbar)
 *   mode 1 (finalize): x = xbar + delta            (optimizer.py:171; delta then resets)
 *   snapshot slot 1-snap_slot = x.
 *   mode 2 (SGD-AR, optimizer.py:214-242): the slots hold gradients; x = K5(x, mean of
 *   every rank's slot `snap_slot`) with the rate/momentum of `sgd` — g and delta unused,
 *   no slot written; one-shot or two-shot only (AUTO as for the all-reduce).
 * Bit-identical to lasgd_sgd_step -> lasgd_comm_allreduce -> lasgd_elastic_pull /
 * lasgd_finalize under the same schedule; launched on `stream` with `nblocks` CTAs
 * (<= 0: the communicator's budget), `algo` one-shot (every peer's whole snapshot) or
 * two-shot (reduce-scatter of the own chunk, per-CTA mid barrier, then the pull reads
 * each chunk's mean from its owner) or PUSH (K8: each owner reduces contributions
 * staged in its own HBM by the previous round and pushes the chunk mean to every
 * peer; the next snapshot's chunks are pushed to their owners; the first push round
 * after any other use of the slots adds one staging launch); AUTO = see
 * lasgd_comm_resolve_fused_algo.  A launch like lasgd_comm_allreduce (same
 * sequence numbers, query / wait / stream_wait apply).  The rounds own the snapshot
 * slots: a caller that writes a slot between rounds must call
 * lasgd_comm_invalidate_staging first (consecutive rounds enter on the previous round's
 * end-of-round signals, which only certify what the rounds themselves wrote). */
int lasgd_comm_fused_round(lasgd_comm* c, int snap_slot, int algo, void* x, const void* g, void* m, void* delta,
                           const lasgd_sgd_params* sgd, double alpha, int mode, int nblocks,
                           unsigned long long* nonfinite, void* stream, unsigned long long* seq);
/* K7 over P virtual ranks on ONE device (host arrays of P device pointers each;
 * m / delta / xbars arrays may be NULL; two-shot needs per-rank xbars scratch).
 * Test path for the fused arithmetic and slicing. */
int lasgd_fused_round_virtual(int P, int algo, void* const* x, const void* const* g, void* const* m,
                              void* const* delta, const void* const* snaps, void* const* xbars,
                              void* const* snap_next, size_t n, int dtype, const lasgd_sgd_params* sgd,
                              double alpha, int mode, int nblocks, unsigned long long* nonfinite, void* stream);
/* Non-blocking completion poll of launch `seq` (collective.py:142-144 `poll`):
 * 1 complete, 0 in flight, LASGD_ERR_COLLECTIVE failed (diagnostic via
 * lasgd_comm_diagnostic).  Reads a host-mapped flag: no CUDA call. */
int lasgd_comm_query(lasgd_comm* c, unsigned long long seq);
/* Make `stream` wait for launch `seq` (cudaStreamWaitEvent; no host block). */
int lasgd_comm_stream_wait(lasgd_comm* c, unsigned long long seq, void* stream);
/* Host wait (collective.py:138-139 `wait`): 1 complete, LASGD_ERR_TIMEOUT, or failure. */
int lasgd_comm_wait(lasgd_comm* c, unsigned long long seq, double timeout_s);
int lasgd_comm_diagnostic(lasgd_comm* c, char* buf, size_t len);
/* NVLink bytes this rank's peers read from it in one launch (collective.py:206-226 analogue). */
unsigned long long lasgd_comm_bytes_per_node(lasgd_comm* c, int algo);
int lasgd_comm_resolve_algo(lasgd_comm* c, int algo);
/* Bucketed SGD-AR (optimizer.py:214-242; the all-reduce split into buckets that a
 * trainer launches as backward completes them): the mean over NVLink of every rank's
 * gradient in slot `snap_slot` over elements [off, off + len) and the local step of
 * x[off, off + len) (and m) with it — one-shot, or two-shot (`algo`; AUTO picks by the
 * bucket's size like the all-reduce).  Each element is summed in the ring order of its
 * chunk of the WHOLE vector (collective.py:183-200), so the result is bit-identical to
 * one lasgd_comm_fused_round(mode 2) for any bucketing.  off must be 16-byte aligned in
 * elements.  A launch like lasgd_comm_allreduce (sequence numbers, query / wait). */
int lasgd_comm_sgd_ar_range(lasgd_comm* c, int snap_slot, size_t off, size_t len, int algo, void* x, void* m,
                            const lasgd_sgd_params* sgd, int nblocks, unsigned long long* nonfinite, void* stream,
                            unsigned long long* seq);
/* The algorithm lasgd_comm_fused_round runs for `algo`: AUTO resolves to PUSH (the
 * mirror form) at P = 2 for buffers >= 32 MiB, otherwise to one-shot where the all-reduce
 * would be one-shot and to PUSH where it would be two-shot. */
int lasgd_comm_resolve_fused_algo(lasgd_comm* c, int algo);
/* What ALGO_AUTO resolves to for a fused round of `bytes` per rank at `world` ranks
 * (host only, no device needed). */
int lasgd_resolve_fused_algo_for(int world, size_t bytes);
/* What ALGO_AUTO resolves to for a standalone all-reduce (lasgd_comm_allreduce, no NVLS)
 * of `bytes` per rank at `world` ranks.  Host only, no device needed. */
int lasgd_resolve_allreduce_algo_for(int world, size_t bytes);
/* Change the SM budget (CTAs per launch) for subsequent launches; every rank must
 * make the same call between the same two launches. */
int lasgd_comm_set_nblocks(lasgd_comm* c, int nblocks);
/* Tracing: when on, every CTA of each launch records %globaltimer stamps (start,
 * entry barrier passed, mid barrier passed, end) — the timeline of the last launch
 * is read back (synchronising) with lasgd_comm_read_trace into out[ctas][4]. */
int lasgd_comm_set_trace(lasgd_comm* c, int on);
int lasgd_comm_read_trace(lasgd_comm* c, unsigned long long* out, int max_ctas);
int lasgd_comm_destroy(lasgd_comm* c);

/* Highest launch sequence number any peer has started (from the entry flags peers
 * wrote into this rank's signal pad); used to drain adaptive runs without a host
 * collective.  Never waits behind the caller's streams. */
int lasgd_comm_peer_max_seq(lasgd_comm* c, unsigned long long* out);
/* 1 if some peer has already entered an all-reduce launch later than `seq` (this rank
 * is the laggard of that round: its launch `seq` is complete or about to be), else 0.
 * Reads the peers' entry flags of CTA 0 (32 bytes) on a private non-blocking stream.
 * Used by the adaptive schedule to close a round without another local step. */
int lasgd_comm_peers_ahead(lasgd_comm* c, unsigned long long seq);
/* on = 1: every lasgd_comm_allreduce launch is preceded (same stream) by a one-warp
 * gate kernel that waits until every peer reached the same launch, so a side-stream
 * all-reduce never holds a CTA per SM while a late peer catches up (which would
 * starve the compute stream).  Collective setting: every rank must use the same. */
int lasgd_comm_set_gate(lasgd_comm* c, int on);
/* Stream-ordered device barrier across the ranks (one warp, its own epoch counter and
 * flag slots: takes no launch sequence number and leaves the round chain and the push
 * staging untouched).  Collective: every rank calls it the same number of times.  The
 * benchmark starts its timed region behind it so every rank's clock starts together. */
int lasgd_comm_barrier(lasgd_comm* c, void* stream);
/* The caller rewrote a snapshot slot outside the fused rounds (also resets the chain of
 * end-of-round signals the next K7 would otherwise enter on).  The next push round
 * re-stages the current snapshot first. */
int lasgd_comm_invalidate_staging(lasgd_comm* c);
/* Number of launches this rank has issued on the communicator (its current sequence number). */
int lasgd_comm_launches(lasgd_comm* c, unsigned long long* out);
/* rank, world size and the mean buffer of a communicator (any pointer may be NULL). */
int lasgd_comm_info(lasgd_comm* c, int* rank, int* world, void** xbar);
/* ---- NVLink SHARP (tolerance mode) -----------------------------------------
 * The mean reduced inside the NVSwitch: multimem.ld_reduce of the rank's chunk over the
 * multicast view of the snapshot slot, multimem.st of the mean into every rank's mean
 * buffer — (P+1)/P*B per link direction instead of 2(P-1)/P*B.  The switch's summation
 * order is not the reference ring's (collective.py:183-200): the mean matches it to
 * rounding (the north star's 1e-6 relative); every rank receives the same bits.
 * Setup, collectively: rank 0 lasgd_comm_nvls_create (exports the multicast object as a
 * POSIX fd, which the caller passes to the other ranks, e.g. SCM_RIGHTS), the others
 * lasgd_comm_nvls_import; every rank lasgd_comm_nvls_add_device; after ALL have added,
 * lasgd_comm_nvls_bind.  From then on the snapshot slots and the mean buffer
 * (lasgd_comm_buffer / lasgd_comm_info) live in the multicast-bound allocation and
 * lasgd_comm_allreduce runs the in-switch mean (AUTO or NVLS); fused rounds are refused.
 * fp32 only. */
int lasgd_comm_nvls_supported(lasgd_comm* c);
int lasgd_comm_nvls_create(lasgd_comm* c, int* fd_out);
int lasgd_comm_nvls_import(lasgd_comm* c, int fd);
int lasgd_comm_nvls_add_device(lasgd_comm* c);
int lasgd_comm_nvls_bind(lasgd_comm* c);
/* Element count and element type of the communicator's buffers (either pointer may be NULL). */
int lasgd_comm_shape(lasgd_comm* c, size_t* n, int* dtype);

/* ---- native per-rank worker: the round protocol (optimizer.py:181-207) ---- */

typedef struct lasgd_worker lasgd_worker;

#define LASGD_TAU_HIST 64
#define LASGD_KERNEL_KINDS 7 /* sgd_step, snapshot, pull, finalize, allreduce, fused_round, sgd_pull */

typedef struct {
  int sync_period;     /* deterministic schedule: local steps per round (tau)                    */
  double alpha;        /* elastic coefficient, (0, 1]                                            */
  int mode;            /* 0 pull x -= alpha*(snap - xbar); 1 reference finalize z + delta (alpha 1) */
  int pipeline;        /* 0 overlap (K5 | K4 | K2/K3 on the side stream); 1 fused (K7)           */
  int algo;            /* LASGD_ALGO_*                                                           */
  int fused_nblocks;   /* CTAs of K7 (<= 0: 2 per SM)                                            */
  double momentum, dampening, weight_decay;
  int nesterov;
  int sync;            /* 0: local steps only (the no-sync ceiling)                              */
  int adaptive;        /* 1: close a round as soon as the mean landed (overlap pipeline only)    */
  int tau_max;         /* adaptive budget (optimizer.py:141-144); <= 0: sync_period              */
  int max_host_lead;   /* adaptive: host may run at most this many steps ahead of the GPU        */
  int max_host_wait_us; /* adaptive: cap on one run-ahead wait (<= 0: 250 ms); a stream stalled on
                           a peer's future launch must not block the host                        */
} lasgd_worker_config;

typedef struct {
  int tau_i, snap_idx;
  long long local_clock, global_clock;
  unsigned long long seq;
  int momentum_started, delta_fresh;
  long long launches[LASGD_KERNEL_KINDS];
  long long tau_hist[LASGD_TAU_HIST]; /* rounds closed after t local steps */
} lasgd_worker_state;

/* comm NULL = single rank (snap0/snap1 required); with a communicator the snapshot
 * slots and the mean buffer are the communicator's.  x, m (momentum != 0), delta
 * (mode 1) are caller-owned device buffers of n elements.  Issues the initial
 * snapshot (and, overlap pipeline, the round-0 launch) on compute_stream. */
int lasgd_worker_create(lasgd_comm* comm, void* x, void* m, void* delta, void* snap0, void* snap1, size_t n,
                        int dtype, const lasgd_worker_config* cfg, void* compute_stream, void* side_stream,
                        unsigned long long* nonfinite, lasgd_worker** out);
/* One local step from gradient g at rate lr (lr_at of the local clock, problems.py:355);
 * returns 1 when the step closed a round, 0 otherwise, < 0 on error. */
int lasgd_worker_step(lasgd_worker* w, const void* g, double lr);
/* Order the compute stream after the in-flight mean (overlap pipeline). */
int lasgd_worker_drain(lasgd_worker* w);
int lasgd_worker_get_state(lasgd_worker* w, lasgd_worker_state* s);
int lasgd_worker_set_timing(lasgd_worker* w, int on);
int lasgd_worker_timings(lasgd_worker* w, int kind, float* out_ms, int max);
int lasgd_worker_reset_stats(lasgd_worker* w);
int lasgd_worker_destroy(lasgd_worker* w);

/* ---- graph replay of the deterministic schedule (optimizer.py:181-207 with
 * collective_complete = (tau_i == k)) ------------------------------------------
 * The per-launch scalars of a worker step (learning rate, first_step, delta reset,
 * snapshot slot) live in a device round descriptor that every captured launch reads
 * at entry and its last CTA advances, so `steps` worker steps captured once replay as
 * ONE CUDA graph launch, any number of times, with results bit-identical to the same
 * steps issued one by one.  Single rank (comm NULL) for now; both pipelines (a round
 * boundary is the local step with the next snapshot fused in). */
typedef struct lasgd_graph lasgd_graph;
/* Learning rate per local clock (lr_at of problems.py:355 for clocks 0..len-1); len 1 =
 * a constant rate.  A replay that would read past a longer table fails with
 * LASGD_ERR_STATE.  Synchronises the compute stream. */
int lasgd_worker_set_lr_table(lasgd_worker* w, const double* lr, size_t len);
/* Capture `steps` steps (a whole number of rounds) reading gradient g[t] at step t.  Nothing
 * runs and the worker's state is unchanged until lasgd_graph_launch. */
int lasgd_worker_graph_capture(lasgd_worker* w, int steps, const void* const* g, lasgd_graph** out);
/* Capture worker steps into the caller's own stream capture (e.g. forward + backward +
 * step in one graph): call with the compute stream capturing, issue the steps, then
 * lasgd_worker_capture_end.  The returned lasgd_graph holds no executable: before each
 * replay of the caller's graph on the compute stream, call lasgd_graph_launch (it
 * refreshes the device descriptor when needed and advances the worker's state). */
int lasgd_worker_capture_begin(lasgd_worker* w, lasgd_graph** out);
int lasgd_worker_capture_end(lasgd_graph* gr);
/* Replay on the worker's compute stream and advance the worker's state by the captured
 * steps; LASGD_ERR_STATE if the worker is not at the round position of the capture. */
int lasgd_graph_launch(lasgd_graph* gr);
/* Destroy every graph of a worker before the worker itself. */
int lasgd_graph_destroy(lasgd_graph* gr);

/* ---- measurement aid ------------------------------------------------------ */
/* One thread that holds `stream` until lasgd_hold_release (or `timeout_s` passes): the
 * host enqueues a whole timed region behind it, then releases it, so host-side jitter
 * cannot open gaps in the region.  Destroy only after the stream has drained. */
/* Write the device's %globaltimer (ns) to *out (device memory) in stream order: the
 * clock of the communicator's per-CTA trace (lasgd_comm_read_trace). */
int lasgd_stamp(unsigned long long* out, void* stream);
typedef struct lasgd_hold lasgd_hold;
int lasgd_hold_create(lasgd_hold** out);
int lasgd_hold_enqueue(lasgd_hold* h, void* stream, double timeout_s);
int lasgd_hold_release(lasgd_hold* h);
int lasgd_hold_destroy(lasgd_hold* h);

/* ---- host utilities ------------------------------------------------------ */

/* partition_chunks (params.py:130-147): writes num_chunks+1 boundaries. */
int lasgd_partition_chunks(size_t d, int num_chunks, size_t* bounds);
/* bytes_per_node (collective.py:206-226); rank < 0 = max over ranks. */
unsigned long long lasgd_bytes_per_node(size_t d, int num_ranks, int bytes_per_element, int rank);

#ifdef __cplusplus
}
#endif
#endif /* LASGD_SYNC_H */
