// NVLink P2P communicator of the LASGD sync path: the C-ABI entry points, launch
// dispatch, virtual-rank test paths and the communicator lifecycle (IPC region,
// signal pad, work queues, host-mapped status).  The kernels live in headers:
//   comm_device.cuh    CommArgs, system-scope flags, per-CTA / rank-level barriers,
//                      launch gate (K9), completion word, tile work queues
//   comm_allreduce.cuh K2 one-shot and K3 two-shot mean all-reduce
//   comm_fused.cuh     K7 fused round (local step + mean + pull + next snapshot;
//                      mode 2 = one SGD-AR round)
//   comm_push.cuh      K8 push round (staged chunks for P >= 3, mirror for P = 2)
//   comm_launch.cuh    launch helpers and the dispatcher declarations
// and are instantiated in their own translation units (comm_launch_allreduce.cu,
// comm_launch_fused.cu, comm_launch_push.cu), compiled in parallel.
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

#include "comm_ce.h"
#include "comm_launch.cuh"
#include "comm_nvls.h"
#include "lasgd_common.cuh"

namespace lasgd {

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
  if (mode < 0 || mode > 2) return fail(LASGD_ERR_INVALID_ARGUMENT, "mode %d (0 pull, 1 finalize, 2 SGD-AR)", mode);
  if (mode == 2 && delta && delta[0]) return fail(LASGD_ERR_INVALID_ARGUMENT, "the SGD-AR round has no delta");
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
  // P <= 4: one-shot still wins at 4 MB (42 vs 53 us all-reduce, 43 vs 48 us fused),
  // two-shot / push from 16 MB (profiles/allreduce_sweep_r01_v2_p4.jsonl)
  const size_t cutoff = P <= 4 ? (size_t)8 << 20 : (size_t)1 << 20;
  return bytes <= cutoff ? LASGD_ALGO_ONESHOT : LASGD_ALGO_TWOSHOT;
}

// Fused round (K7/K8): where the all-reduce would be two-shot, the push round moves
// the same NVLink bytes with stores only and no entry wait on peers' snapshots
// (measured 3-5% faster per round at P=3/4, profiles/bench_r01_algo_*.json).
// At P = 2 the push round is the mirror form: same bytes as the one-shot, moved as
// posted stores: ~6% faster per round at ResNet-50 size (profiles/k8_mirror_ab_r01_p2.jsonl)
// and at ResNet-18 size (90 vs 96 us), 4% slower at MobileNetV2 size (48 vs 46 us), so the
// crossover sits between 14 and 45 MB (profiles/small_models_r01.jsonl).
int resolve_fused_algo(int algo, int P, size_t bytes) {
  if (P <= 1) return LASGD_ALGO_ONESHOT;
  if (algo != LASGD_ALGO_AUTO) return algo;
  if (P == 2) return bytes >= ((size_t)32 << 20) ? LASGD_ALGO_PUSH : LASGD_ALGO_ONESHOT;
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
  if (mode == 2 && P < 2) return fail(LASGD_ERR_INVALID_ARGUMENT, "the SGD-AR round needs P >= 2");
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
  if (mode == 2) return fail(LASGD_ERR_INVALID_ARGUMENT, "no push form of the SGD-AR round");
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
  unsigned int* aux_ctr = nullptr;   // [kDoneSlots] push mean: second-half scatter counters
  char* peer_base[kMaxR] = {nullptr};
  bool opened = false;
  bool poisoned = false;
  uint32_t* status_host = nullptr;  // ST_WORDS uint32 + u64 done_seq (host-mapped)
  uint32_t* status_dev = nullptr;
  unsigned long long* done_host = nullptr;
  unsigned long long* done_dev = nullptr;
  unsigned int* done_ctr = nullptr;
  unsigned long long* tile_ctr = nullptr;  // [kDoneSlots][kTileQ] work queues
  unsigned int* mid_ctr = nullptr;         // [kDoneSlots] rank-level barrier counters
  unsigned long long* trace_buf = nullptr;  // [kMaxB][4] globaltimer stamps of the last traced launch
  bool trace_on = false;
  bool gate = false;           // launch k_gate ahead of every all-reduce (side-stream use)
  unsigned long long seq = 0;  // launches issued
  uint32_t bar_epoch = 0;      // lasgd_comm_barrier calls (own flag slots, no sequence number)
  // NVLink SHARP (tolerance mode): once bound, the snapshot slots and the mean buffer live
  // in a multicast-bound allocation: nvls_uc (this rank's view) / nvls_mc (the switch's)
  NvlsState* nvls = nullptr;
  char* nvls_uc = nullptr;
  char* nvls_mc = nullptr;
  size_t nvls_off[3] = {0, 0, 0};
  uint32_t* epoch_host = nullptr;      // pinned readback of the peers' entry flags (read_peer_epochs)
  cudaStream_t epoch_stream = nullptr;  // on this communicator's device
  cudaEvent_t ev[kEvents];
  int nev = 0;
};

static size_t round_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// phases bit 8 for the staged push round (P >= 3): phase A signals its first half before
// the second, so phase B starts on the first half while the second half's means drain
static int push_split(const lasgd_comm* c) {
  return (c->world >= 3 && c->n * c->elem >= ((size_t)32 << 20)) ? 8 : 0;
}

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
  if (e == cudaSuccess) e = cudaMalloc(&c->tile_ctr, kTileQ * kDoneSlots * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(c->tile_ctr, 0, kTileQ * kDoneSlots * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMalloc(&c->aux_ctr, kDoneSlots * sizeof(unsigned int));
  if (e == cudaSuccess) e = cudaMemset(c->aux_ctr, 0, kDoneSlots * sizeof(unsigned int));
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
  if (c->nvls_uc && which >= 0 && which <= 2) *ptr = c->nvls_uc + c->nvls_off[which];
  else if (which == 0 || which == 1) *ptr = c->base + c->off_snap[which];
  else if (which == 2) *ptr = c->base + c->off_xbar;
  else return fail(LASGD_ERR_INVALID_ARGUMENT, "buffer index %d", which);
  return LASGD_OK;
}

// The all-reduce's AUTO at P = 3-4 (measured; profiles/r02/pm{2,3}_sweep_p{3,4}.jsonl):
// where resolve_algo picks the two-shot (and at P=4 from 4 MB), the push mean (every byte
// moved by stores) is faster at every size (P=4: 16 MB 0.065 vs 0.079 ms, 102 MB 0.276
// vs 0.301, 256 MB 0.617 vs 0.708; P=3 102 MB 0.248 vs 0.276), and at 1 GB the
// copy-engine mean is faster still (P=4 2.328 vs 2.372, P=3 2.130 vs 2.247).  Otherwise
// (P = 2: one-shot; P >= 5, unmeasured on hardware) resolve_algo.  Not for SGD-AR buckets
// or fused rounds: they have their own.
static int resolve_allreduce_bytes(int algo, int world, size_t bytes) {
  const int a = resolve_algo(algo, world, bytes);
  if (algo != LASGD_ALGO_AUTO || world < 3 || world > 4) return a;
  if (bytes >= ((size_t)512 << 20)) return LASGD_ALGO_CE;
  if (a == LASGD_ALGO_TWOSHOT) return LASGD_ALGO_PUSH;
  if (world == 4 && bytes >= ((size_t)3 << 20)) return LASGD_ALGO_PUSH;  // 4 MB: 0.0347 vs 0.0372 one-shot
  return a;
}

static int resolve_allreduce_algo(const lasgd_comm* c, int algo) {
  if (c->nvls_uc) return resolve_algo(algo, c->world, c->n * c->elem);
  return resolve_allreduce_bytes(algo, c->world, c->n * c->elem);
}

extern "C" int lasgd_resolve_allreduce_algo_for(int world, size_t bytes) {
  if (world < 1 || world > kMaxR) return fail(LASGD_ERR_UNSUPPORTED, "world size %d outside [1, %d]", world, kMaxR);
  return resolve_allreduce_bytes(LASGD_ALGO_AUTO, world, bytes);
}

int lasgd::comm_side_algo(lasgd_comm* c, int algo) {
  // under forward/backward the CE mean's NVLink traffic costs no SM time: ResNet-50 at
  // N=4 exposes 0.241-0.246 ms/step on it against 0.282-0.304 on the SM two-shot (three
  // runs), at N=3 0.231 against 0.264; at N=2 the SM one-shot exposes less (0.19-0.21 vs
  // 0.22) (profiles/r02/ce_train_n*.json)
  if (algo == LASGD_ALGO_AUTO && !c->nvls_uc && c->world >= 3 && c->world <= 4 && c->n * c->elem >= ((size_t)64 << 20))
    return LASGD_ALGO_CE;
  return algo;
}

extern "C" int lasgd_comm_resolve_algo(lasgd_comm* c, int algo) {
  if (!c) return fail(LASGD_ERR_INVALID_ARGUMENT, "null comm");
  return resolve_allreduce_algo(c, algo);
}

extern "C" int lasgd_resolve_fused_algo_for(int world, size_t bytes) {
  return resolve_fused_algo(LASGD_ALGO_AUTO, world, bytes);
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
  // per-communicator pinned buffer and stream, created on c->device (the caller holds a
  // DeviceGuard) and freed by lasgd_comm_destroy
  const size_t entry_words = (size_t)kMaxB * kMaxR;
  // rank-level rows carrying launch epochs: 0 mid, 1 end, 2 gate, 3-4 copy-engine signals
  // (the push and CE means have no per-CTA entry flags; row 5, the device barrier, counts
  // barriers, not launches)
  constexpr int kRankRows = 5;
  if (!c->epoch_host)
    LASGD_CUDA_TRY(cudaHostAlloc((void**)&c->epoch_host, (entry_words + kRankRows * kMaxR) * sizeof(uint32_t),
                                 cudaHostAllocDefault));
  if (!c->epoch_stream) LASGD_CUDA_TRY(cudaStreamCreateWithFlags(&c->epoch_stream, cudaStreamNonBlocking));
  uint32_t* host = c->epoch_host;
  cudaStream_t s = c->epoch_stream;
  const size_t rank_word = (size_t)2 * kMaxB * kMaxR;  // first rank-level slot row
  LASGD_CUDA_TRY(cudaMemcpyAsync(host, c->base, (size_t)rows * kMaxR * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  LASGD_CUDA_TRY(cudaMemcpyAsync(host + entry_words, c->base + rank_word * sizeof(uint32_t),
                                 (size_t)kRankRows * kMaxR * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  LASGD_CUDA_TRY(cudaStreamSynchronize(s));
  for (int q = 0; q < kMaxR; ++q) {
    uint32_t best = host[entry_words + q];
    for (int k = 1; k < kRankRows; ++k) {
      const uint32_t v = host[entry_words + (size_t)k * kMaxR + q];
      if ((int32_t)(v - best) > 0) best = v;
    }
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
  // epochs are the low 32 bits of the sequence numbers: wrapping compare, like peers_ahead
  uint32_t best = (uint32_t)c->seq;
  for (int q = 0; q < c->world; ++q)
    if (q != c->rank && (int32_t)(ep[q] - best) > 0) best = ep[q];
  // extend to 64 bits around this rank's own sequence number
  *out = c->seq + (unsigned long long)(int64_t)(int32_t)(best - (uint32_t)c->seq);
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
  // the rank-level rows: gate, end, CE signals) holds each peer's latest launch
  uint32_t ep[kMaxR];
  int rc = read_peer_epochs(c, 1, ep);
  if (rc) return rc;
  for (int q = 0; q < c->world; ++q)
    if (q != c->rank && (int32_t)(ep[q] - (uint32_t)seq) > 0) return 1;
  return 0;
}

extern "C" int lasgd_comm_barrier(lasgd_comm* c, void* stream) {
  if (!c) return fail(LASGD_ERR_INVALID_ARGUMENT, "null comm");
  if (c->world < 2) return LASGD_OK;
  if (!c->opened) return fail(LASGD_ERR_STATE, "lasgd_comm_open has not been called");
  if (c->poisoned || c->status_host[ST_ERR] != ERR_NONE) {
    c->poisoned = true;
    return fail(LASGD_ERR_COLLECTIVE, "communicator failed earlier; re-create it");
  }
  DeviceGuard g(c->device);
  CommArgs a;
  memset(&a, 0, sizeof(a));
  for (int r = 0; r < c->world; ++r) a.pad[r] = reinterpret_cast<uint32_t*>(c->peer_base[r]);
  a.rank = c->rank;
  a.epoch = ++c->bar_epoch;
  a.seq = c->seq;  // diagnostics only
  a.timeout_ns = c->timeout_ns;
  a.skip_signal_phase = -1;
  a.status = c->status_dev;
  return launch_rank_barrier(c->world, a, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int lasgd_comm_invalidate_staging(lasgd_comm* c) {
  if (!c) return fail(LASGD_ERR_INVALID_ARGUMENT, "null comm");
  c->push_slot = -1;
  c->end_seq = 0;  // a slot was rewritten outside the rounds: the next K7 uses the entry barrier
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
  if (xbar) *xbar = c->nvls_uc ? c->nvls_uc + c->nvls_off[2] : c->base + c->off_xbar;
  return LASGD_OK;
}

// ---------------------------------------------------------------- NVLink SHARP setup
extern "C" int lasgd_comm_nvls_supported(lasgd_comm* c) {
  if (!c) return fail(LASGD_ERR_INVALID_ARGUMENT, "null comm");
  DeviceGuard g(c->device);
  return c->dtype == LASGD_F32 && c->world >= 2 ? nvls_supported(c->device) : 0;
}

static size_t nvls_payload(lasgd_comm* c, size_t off[3]) {
  const size_t slot = round_up(c->n * c->elem, 256);
  off[0] = 0;
  off[1] = slot;
  off[2] = 2 * slot;
  return 3 * slot;
}

extern "C" int lasgd_comm_nvls_create(lasgd_comm* c, int* fd_out) {
  if (!c) return fail(LASGD_ERR_INVALID_ARGUMENT, "null comm");
  if (c->nvls) return fail(LASGD_ERR_STATE, "NVLS already set up");
  if (c->dtype != LASGD_F32) return fail(LASGD_ERR_UNSUPPORTED, "the in-switch mean is fp32 only");
  DeviceGuard g(c->device);
  return nvls_create(&c->nvls, c->device, c->world, nvls_payload(c, c->nvls_off), fd_out);
}

extern "C" int lasgd_comm_nvls_import(lasgd_comm* c, int fd) {
  if (!c) return fail(LASGD_ERR_INVALID_ARGUMENT, "null comm");
  DeviceGuard g(c->device);
  if (!c->nvls) {
    int rc = nvls_create(&c->nvls, c->device, c->world, nvls_payload(c, c->nvls_off), nullptr);
    if (rc) return rc;
  }
  return nvls_import(c->nvls, fd);
}

extern "C" int lasgd_comm_nvls_add_device(lasgd_comm* c) {
  if (!c || !c->nvls) return fail(LASGD_ERR_STATE, "create or import the multicast object first");
  DeviceGuard g(c->device);
  return nvls_add_device(c->nvls);
}

extern "C" int lasgd_comm_nvls_bind(lasgd_comm* c) {
  if (!c || !c->nvls) return fail(LASGD_ERR_STATE, "create or import the multicast object first");
  DeviceGuard g(c->device);
  void *uc = nullptr, *mc = nullptr;
  int rc = nvls_bind(c->nvls, &uc, &mc);
  if (rc) return rc;
  c->nvls_uc = reinterpret_cast<char*>(uc);
  c->nvls_mc = reinterpret_cast<char*>(mc);
  c->push_slot = -1;
  c->end_seq = 0;
  return LASGD_OK;
}

extern "C" int lasgd_comm_shape(lasgd_comm* c, size_t* n, int* dtype) {
  if (!c) return fail(LASGD_ERR_INVALID_ARGUMENT, "null comm");
  if (n) *n = c->n;
  if (dtype) *dtype = c->dtype;
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
    __atomic_store_n(&st[ST_CLAIM], 1u, __ATOMIC_SEQ_CST);
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
  a.tile_ctr = c->tile_ctr + kTileQ * (s % kDoneSlots);
  a.mid_ctr = c->mid_ctr + (s % kDoneSlots);
  a.end_ctr = c->end_ctr + (s % kDoneSlots);
  a.aux_ctr = c->aux_ctr + (s % kDoneSlots);
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
  if (c->nvls_uc) {  // NVLS communicator: the data lives in the multicast region
    if (algo != LASGD_ALGO_AUTO && algo != LASGD_ALGO_NVLS)
      return fail(LASGD_ERR_UNSUPPORTED, "an NVLS communicator runs the in-switch mean only (algo %d)", algo);
    DeviceGuard g(c->device);
    CommArgs a;
    unsigned long long s = 0;
    int rc = prepare_launch(c, snap_slot, a, s);
    if (rc) return rc;
    cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
    c->push_slot = -1;
    c->end_seq = 0;
    if (c->gate && (rc = launch_gate(c->world, a, cs))) return rc;
    // the switch, not the SMs, bounds this kernel: half the SMs issue enough loads
    // (profiles/r02/allreduce_sweep_p4_nvls.jsonl: 37-74 CTAs at least as fast as 148-512)
    const int nb = c->nblocks < num_sms() / 2 ? c->nblocks : num_sms() / 2;
    a.nblocks = nb;
    rc = launch_nvls_mean(c->world, a, c->nvls_mc + c->nvls_off[snap_slot], c->nvls_mc + c->nvls_off[2], nb, cs);
    if (rc) return rc;
    LASGD_CUDA_TRY(cudaEventRecord(c->ev[s % kEvents], cs));
    if (seq) *seq = s;
    return LASGD_OK;
  }
  if (algo == LASGD_ALGO_NVLS) return fail(LASGD_ERR_STATE, "the NVLS mean needs lasgd_comm_nvls_bind first");
  algo = resolve_allreduce_algo(c, algo);
  if (algo == LASGD_ALGO_CE && c->world > 1) {  // copy-engine two-shot (comm_ce.cu)
    DeviceGuard g(c->device);
    CommArgs a;
    unsigned long long s = 0;
    int rc = prepare_launch(c, snap_slot, a, s);
    if (rc) return rc;
    cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
    c->push_slot = -1;  // the contributions overwrite the push round's staging
    c->end_seq = 0;
    CeRound r;
    memset(&r, 0, sizeof(r));
    r.snap_local = c->base + c->off_snap[snap_slot];
    r.xbar_local = c->base + c->off_xbar;
    r.stage_local = c->base + c->off_stage;
    r.stage_elems = c->stage_elems;
    for (int q = 0; q < c->world; ++q) {
      r.stage_peer[q] = c->peer_base[q] + c->off_stage;
      r.xbar_peer[q] = c->peer_base[q] + c->off_xbar;
    }
    rc = launch_ce_mean(c->dtype, c->world, a, r, cs);  // its own entry gate
    if (rc) return rc;
    LASGD_CUDA_TRY(cudaEventRecord(c->ev[s % kEvents], cs));
    if (seq) *seq = s;
    return LASGD_OK;
  }
  if (algo == LASGD_ALGO_PUSH && c->world > 1) {  // the mean by remote stores (comm_push.cuh)
    DeviceGuard g(c->device);
    CommArgs a;
    unsigned long long s = 0;
    int rc = prepare_launch(c, snap_slot, a, s);
    if (rc) return rc;
    cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
    c->push_slot = -1;  // the staging now holds this mean's contributions, not a round's
    c->end_seq = 0;
    if (c->gate && (rc = launch_gate(c->world, a, cs))) return rc;
    // halves pipelined from 32 MB (P=4: 64 MB 0.1725 vs 0.1849 ms, 256 MB 0.617 vs 0.667;
    // at 4-16 MB the second signal costs more than it hides; profiles/r02/pm3_sweep_p*.jsonl)
    if (c->n * c->elem >= ((size_t)32 << 20)) a.phases |= 8;
    rc = c->dtype == LASGD_F64 ? launch_push_mean<double>(c->world, a, dim3(c->nblocks), c->threads, cs)
                               : launch_push_mean<float>(c->world, a, dim3(c->nblocks), c->threads, cs);
    if (rc) return rc;
    LASGD_CUDA_TRY(cudaEventRecord(c->ev[s % kEvents], cs));
    if (seq) *seq = s;
    return LASGD_OK;
  }
  if (algo == LASGD_ALGO_CE || algo == LASGD_ALGO_PUSH) algo = LASGD_ALGO_ONESHOT;  // P = 1: the copy
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
  if (c->nvls_uc) return fail(LASGD_ERR_UNSUPPORTED, "an NVLS communicator runs the side-stream mean only");
  // SGD-AR (mode 2) averages gradients that backward wrote into the slots, so there is
  // nothing to push ahead: one-shot or two-shot, chosen like the all-reduce
  if (mode == 2 && c->world < 2) return fail(LASGD_ERR_INVALID_ARGUMENT, "the SGD-AR round needs P >= 2");
  if (mode == 2 && algo == LASGD_ALGO_PUSH) return fail(LASGD_ERR_INVALID_ARGUMENT, "no push form of the SGD-AR round");
  if (algo == LASGD_ALGO_CE) return fail(LASGD_ERR_UNSUPPORTED, "the copy-engine mean is a side-stream all-reduce only");
  algo = mode == 2 ? resolve_algo(algo, c->world, c->n * c->elem) : resolve_fused_algo(algo, c->world, c->n * c->elem);
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
    a.phases = 3 | push_split(c);
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
  // (not for SGD-AR: its inputs are written by backward after the previous round ended)
  if (algo == LASGD_ALGO_ONESHOT && mode != 2 && c->end_seq != 0 && c->end_seq + 1 == s)
    a.prev_end = (uint32_t)c->end_seq;
  c->push_slot = -1;  // this round writes the next snapshot without staging it
  if (c->dtype == LASGD_F32)
    rc = launch_fused<float, false>(c->world, a, make_fused<float>(1, xs, gs, m ? ms : nullptr, delta ? ds : nullptr, ns, sgd, alpha, mode), dim3(nblocks, 1), c->threads, cs, algo);
  else
    rc = launch_fused<double, false>(c->world, a, make_fused<double>(1, xs, gs, m ? ms : nullptr, delta ? ds : nullptr, ns, sgd, alpha, mode), dim3(nblocks, 1), c->threads, cs, algo);
  if (rc) return rc;
  // the one-shot K7 raises end signals that certify its next snapshot; SGD-AR writes none
  c->end_seq = (algo == LASGD_ALGO_ONESHOT && mode != 2) ? s : 0;
  LASGD_CUDA_TRY(cudaEventRecord(c->ev[s % kEvents], cs));
  if (seq) *seq = s;
  return LASGD_OK;
}

namespace lasgd {

int comm_mirror_get(lasgd_comm* c, CommMirror* m) {
  if (!c || !m) return fail(LASGD_ERR_INVALID_ARGUMENT, "null argument");
  m->seq = c->seq;
  m->last_push = c->last_push;
  m->end_seq = c->end_seq;
  m->push_slot = c->push_slot;
  return LASGD_OK;
}

int comm_mirror_set(lasgd_comm* c, const CommMirror& m) {
  if (!c) return fail(LASGD_ERR_INVALID_ARGUMENT, "null comm");
  c->seq = m.seq;
  c->last_push = m.last_push;
  c->end_seq = m.end_seq;
  c->push_slot = m.push_slot;
  return LASGD_OK;
}

int comm_record_last(lasgd_comm* c, void* stream) {
  if (!c) return fail(LASGD_ERR_INVALID_ARGUMENT, "null comm");
  if (c->seq == 0) return LASGD_OK;
  DeviceGuard g(c->device);
  LASGD_CUDA_TRY(cudaEventRecord(c->ev[c->seq % kEvents], reinterpret_cast<cudaStream_t>(stream)));
  return LASGD_OK;
}

int comm_fused_round_dyn(lasgd_comm* c, int snap_slot, int algo, void* x, const void* g, void* m, void* delta,
                         const lasgd_sgd_params* sgd, double alpha, int mode, int nblocks,
                         unsigned long long* nonfinite, void* stream, const RoundAdv& adv, unsigned long long* seq) {
  if (!c || !adv.rd) return fail(LASGD_ERR_INVALID_ARGUMENT, "null comm or round descriptor");
  if (c->nvls_uc) return fail(LASGD_ERR_UNSUPPORTED, "an NVLS communicator runs the side-stream mean only");
  if (mode == 2) return fail(LASGD_ERR_UNSUPPORTED, "graph replay of SGD-AR rounds is not built");
  if (snap_slot != 0 && snap_slot != 1) return fail(LASGD_ERR_INVALID_ARGUMENT, "snapshot slot %d", snap_slot);
  algo = resolve_fused_algo(algo, c->world, c->n * c->elem);
  const bool push = algo == LASGD_ALGO_PUSH;
  if (!push && algo != LASGD_ALGO_ONESHOT)
    return fail(LASGD_ERR_UNSUPPORTED, "graph replay covers the one-shot and push rounds (algo %d)", algo);
  void* xs[1] = {x};
  const void* gs[1] = {g};
  void* ms[1] = {m};
  void* ds[1] = {delta};
  void* ns[1] = {c->base + c->off_snap[1 - snap_slot]};  // checked here; the kernel picks the slot itself
  int rc = check_fused_args(1, xs, gs, m ? ms : nullptr, delta ? ds : nullptr, ns, sgd, alpha, mode);
  if (rc) return rc;
  // steady state: this round enters on the previous launch's end signals
  if (push ? (c->seq == 0 || c->push_slot != snap_slot || c->last_push != c->seq)
           : (c->seq == 0 || c->end_seq != c->seq))
    return fail(LASGD_ERR_STATE, "capture a round only after an eager round of the same kind (launch %llu)", c->seq);
  if (nblocks <= 0) nblocks = 2 * num_sms() <= kMaxB ? 2 * num_sms() : kMaxB;
  if (nblocks > kMaxB) return fail(LASGD_ERR_INVALID_ARGUMENT, "nblocks=%d > %d", nblocks, kMaxB);
  DeviceGuard dg(c->device);
  CommArgs a;
  unsigned long long s = 0;
  rc = prepare_launch(c, 0, a, s);  // slot-0 pointers; the kernel offsets by the slot in rd
  if (rc) return rc;
  a.adv = adv;
  a.slot_stride = c->off_snap[1] - c->off_snap[0];
  a.dyn_chain = 1;
  a.tile_ctr = c->tile_ctr;  // slot-0 entries: the kernel indexes them by its dynamic sequence number
  a.mid_ctr = c->mid_ctr;
  a.end_ctr = c->end_ctr;
  a.aux_ctr = c->aux_ctr;
  a.skip_signal_phase = -1;
  a.nblocks = nblocks;
  a.nonfinite = nonfinite;
  a.phases = 3 | (push ? push_split(c) : 0);
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  if (push) {
    rc = c->dtype == LASGD_F32
             ? launch_push<float, false>(c->world, a, make_fused<float>(1, xs, gs, m ? ms : nullptr, delta ? ds : nullptr, ns, sgd, alpha, mode), dim3(nblocks, 1), c->threads, cs)
             : launch_push<double, false>(c->world, a, make_fused<double>(1, xs, gs, m ? ms : nullptr, delta ? ds : nullptr, ns, sgd, alpha, mode), dim3(nblocks, 1), c->threads, cs);
    if (rc) return rc;
    c->last_push = s;
    c->end_seq = s;
    c->push_slot = 1 - snap_slot;
  } else {
    rc = c->dtype == LASGD_F32
             ? launch_fused<float, false>(c->world, a, make_fused<float>(1, xs, gs, m ? ms : nullptr, delta ? ds : nullptr, ns, sgd, alpha, mode), dim3(nblocks, 1), c->threads, cs, LASGD_ALGO_ONESHOT)
             : launch_fused<double, false>(c->world, a, make_fused<double>(1, xs, gs, m ? ms : nullptr, delta ? ds : nullptr, ns, sgd, alpha, mode), dim3(nblocks, 1), c->threads, cs, LASGD_ALGO_ONESHOT);
    if (rc) return rc;
    c->end_seq = s;
    c->push_slot = -1;
  }
  if (seq) *seq = s;
  return LASGD_OK;
}

}  // namespace lasgd

// Bucketed SGD-AR (optimizer.py:214-242 with the gradient all-reduce split into
// buckets, as a data-parallel trainer overlaps it with backward): one-shot K7 mode 2 over
// the sub-range [off, off + len) of slot `snap_slot` — the ring-order mean of every
// rank's gradient over NVLink and the local step of x[off, off + len) with it.  Every
// element is summed in the rotation of its chunk of the whole vector, so any bucketing
// gives the bits of the one-launch round.
extern "C" int lasgd_comm_sgd_ar_range(lasgd_comm* c, int snap_slot, size_t off, size_t len, int algo, void* x,
                                       void* m, const lasgd_sgd_params* sgd, int nblocks,
                                       unsigned long long* nonfinite, void* stream, unsigned long long* seq) {
  if (!c) return fail(LASGD_ERR_INVALID_ARGUMENT, "null comm");
  if (c->nvls_uc) return fail(LASGD_ERR_UNSUPPORTED, "an NVLS communicator runs the side-stream mean only");
  if (c->world < 2) return fail(LASGD_ERR_INVALID_ARGUMENT, "the SGD-AR round needs P >= 2");
  if (snap_slot != 0 && snap_slot != 1) return fail(LASGD_ERR_INVALID_ARGUMENT, "snapshot slot %d", snap_slot);
  if (len == 0 || off > c->n || len > c->n - off)
    return fail(LASGD_ERR_INVALID_ARGUMENT, "range [%zu, %zu) outside the %zu-element vector", off, off + len, c->n);
  const size_t W = 16 / c->elem;
  if (off % W) return fail(LASGD_ERR_INVALID_ARGUMENT, "range offset %zu not a multiple of %zu elements", off, W);
  char* xo = reinterpret_cast<char*>(x) + off * c->elem;
  char* mo = m ? reinterpret_cast<char*>(m) + off * c->elem : nullptr;
  void* xs[1] = {xo};
  const void* gs[1] = {xo};  // unused by mode 2
  void* ms[1] = {mo};
  void* ns[1] = {xo};        // unused by mode 2
  int rc = check_fused_args(1, xs, gs, m ? ms : nullptr, nullptr, ns, sgd, 1.0, 2);
  if (rc) return rc;
  if (nblocks <= 0) nblocks = 2 * num_sms() <= kMaxB ? 2 * num_sms() : kMaxB;
  if (nblocks > kMaxB) return fail(LASGD_ERR_INVALID_ARGUMENT, "nblocks=%d > %d", nblocks, kMaxB);
  // one-shot, or two-shot for large buckets at P >= 3 (the bucket's own partition decides
  // who reduces what; the summation order stays the whole vector's).  Validated before
  // prepare_launch takes a sequence number: a refused call must not desynchronise ranks.
  algo = resolve_algo(algo == LASGD_ALGO_PUSH ? LASGD_ALGO_AUTO : algo, c->world, len * c->elem);
  if (algo != LASGD_ALGO_ONESHOT && algo != LASGD_ALGO_TWOSHOT)
    return fail(LASGD_ERR_INVALID_ARGUMENT, "algo %d: bucketed SGD-AR rounds are one-shot or two-shot", algo);
  DeviceGuard dg(c->device);
  CommArgs a;
  unsigned long long s = 0;
  rc = prepare_launch(c, snap_slot, a, s);
  if (rc) return rc;
  for (int r = 0; r < c->world; ++r) {
    a.snap[r] += off * c->elem;
    a.xbar[r] += off * c->elem;
  }
  a.n = len;
  a.range_off = off;
  a.n_glob = c->n;
  a.nblocks = nblocks;
  a.nonfinite = nonfinite;
  c->push_slot = -1;
  c->end_seq = 0;
  a.phases = 3;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  if (c->dtype == LASGD_F32)
    rc = launch_fused<float, false>(c->world, a, make_fused<float>(1, xs, gs, m ? ms : nullptr, nullptr, ns, sgd, 1.0, 2),
                                    dim3(nblocks, 1), c->threads, cs, algo);
  else
    rc = launch_fused<double, false>(c->world, a, make_fused<double>(1, xs, gs, m ? ms : nullptr, nullptr, ns, sgd, 1.0, 2),
                                     dim3(nblocks, 1), c->threads, cs, algo);
  if (rc) return rc;
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
  static const char* const kPhaseName[] = {"entry", "mid", "end-of-round", "launch gate",
                                           "copy-engine contributions", "copy-engine means", "device",
                                           "second half (push)"};
  const char* phase = st[ST_PHASE] < 8 ? kPhaseName[st[ST_PHASE]] : "unknown";
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
  if (c->aux_ctr) cudaFree(c->aux_ctr);
  if (c->trace_buf) cudaFree(c->trace_buf);
  if (c->status_host) cudaFreeHost(c->status_host);
  if (c->nvls) nvls_destroy(c->nvls);
  if (c->epoch_host) cudaFreeHost(c->epoch_host);
  if (c->epoch_stream) cudaStreamDestroy(c->epoch_stream);
  if (c->base) cudaFree(c->base);
  delete c;
  return LASGD_OK;
}
