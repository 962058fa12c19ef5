// Runtime helpers of the C ABI: thread-local diagnostics, error strings, device
// properties, and the host-side partition / byte-accounting utilities.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <mutex>

#include "lasgd_common.cuh"

namespace lasgd {

static thread_local char g_last_error[512] = "";

void set_last_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(LASGD_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
}

int num_sms() {
  static std::mutex mu;
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  std::lock_guard<std::mutex> lk(mu);
  if (cache[dev] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    cache[dev] = v;
  }
  return cache[dev];
}

static int g_stream_ctas_per_sm = 2;
int stream_ctas_per_sm() { return g_stream_ctas_per_sm; }

}  // namespace lasgd

using namespace lasgd;

extern "C" int lasgd_set_stream_ctas_per_sm(int v) {
  if (v < 1 || v > 32) return fail(LASGD_ERR_INVALID_ARGUMENT, "ctas per SM %d outside [1, 32]", v);
  g_stream_ctas_per_sm = v;
  return LASGD_OK;
}

extern "C" int lasgd_abi_version(void) { return LASGD_ABI_VERSION; }

extern "C" const char* lasgd_last_error(void) { return g_last_error; }

extern "C" const char* lasgd_strerror(int code) {
  switch (code) {
    case LASGD_OK: return "ok";
    case LASGD_ERR_INVALID_ARGUMENT: return "invalid argument";
    case LASGD_ERR_DIMENSION: return "dimension mismatch";
    case LASGD_ERR_NONFINITE: return "non-finite values";
    case LASGD_ERR_CUDA: return "CUDA runtime error";
    case LASGD_ERR_COLLECTIVE: return "collective failed";
    case LASGD_ERR_TIMEOUT: return "timed out";
    case LASGD_ERR_STATE: return "invalid state";
    case LASGD_ERR_UNSUPPORTED: return "unsupported";
    default: return "unknown error";
  }
}

// params.py:130-147
extern "C" int lasgd_partition_chunks(size_t d, int num_chunks, size_t* bounds) {
  if (d < 1) return fail(LASGD_ERR_INVALID_ARGUMENT, "d must be positive");
  if (num_chunks < 1) return fail(LASGD_ERR_INVALID_ARGUMENT, "num_chunks must be positive");
  if (!bounds) return fail(LASGD_ERR_INVALID_ARGUMENT, "null bounds");
  const size_t base = d / (size_t)num_chunks, rem = d % (size_t)num_chunks;
  size_t cur = 0;
  bounds[0] = 0;
  for (int i = 0; i < num_chunks; ++i) {
    cur += base + ((size_t)i < rem ? 1 : 0);
    bounds[i + 1] = cur;
  }
  return LASGD_OK;
}

// collective.py:206-226: replay of the ring schedule (send chunk (r-s)%P in reduce
// step s, (r+1-k)%P in gather step k) against the balanced partition.
extern "C" unsigned long long lasgd_bytes_per_node(size_t d, int P, int bpe, int rank) {
  if (P <= 1 || bpe < 1 || d < 1) return 0;
  const size_t base = d / (size_t)P, rem = d % (size_t)P;
  auto size = [&](int c) { return (unsigned long long)(base + ((size_t)c < rem ? 1 : 0)); };
  unsigned long long best = 0;
  for (int r = 0; r < P; ++r) {
    unsigned long long tot = 0;
    for (int s = 0; s < P - 1; ++s) tot += size(((r - s) % P + P) % P) * (unsigned long long)bpe;
    for (int k = 0; k < P - 1; ++k) tot += size(((r + 1 - k) % P + P) % P) * (unsigned long long)bpe;
    if (r == rank) return tot;
    if (tot > best) best = tot;
  }
  return best;
}

// ---------------------------------------------------------------- stream hold
// Measurement aid (the "blocking kernel" of GPU benchmarking practice): one thread
// spins on a host-mapped flag so that the host can enqueue a whole timed region behind
// it and release it at once — the device then runs the region back to back and host
// jitter before or during enqueueing (driver locks taken by NVML queries, the GIL)
// cannot open gaps in it.  Bounded: the kernel exits by itself after `timeout_ns`.
struct lasgd_hold {
  volatile unsigned int* host = nullptr;
  unsigned int* dev = nullptr;
};

namespace lasgd {
__global__ void k_hold(const volatile unsigned int* flag, long long timeout_ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (*flag == 0u) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if ((long long)(t - t0) > timeout_ns) break;
    __nanosleep(1000);
  }
}
}  // namespace lasgd

extern "C" int lasgd_hold_create(lasgd_hold** out) {
  if (!out) return fail(LASGD_ERR_INVALID_ARGUMENT, "null out");
  lasgd_hold* h = new lasgd_hold();
  unsigned int* p = nullptr;
  cudaError_t e = cudaHostAlloc((void**)&p, sizeof(unsigned int), cudaHostAllocMapped);
  if (e == cudaSuccess) e = cudaHostGetDevicePointer((void**)&h->dev, p, 0);
  if (e != cudaSuccess) {
    if (p) cudaFreeHost(p);
    delete h;
    return cuda_fail(e, "cudaHostAlloc(hold flag)");
  }
  h->host = p;
  *h->host = 0u;
  *out = h;
  return LASGD_OK;
}

extern "C" int lasgd_hold_enqueue(lasgd_hold* h, void* stream, double timeout_s) {
  if (!h) return fail(LASGD_ERR_INVALID_ARGUMENT, "null hold");
  *h->host = 0u;
  __sync_synchronize();
  k_hold<<<1, 1, 0, reinterpret_cast<cudaStream_t>(stream)>>>(h->dev, (long long)(timeout_s * 1e9));
  LASGD_CUDA_TRY(cudaGetLastError());
  return LASGD_OK;
}

extern "C" int lasgd_hold_release(lasgd_hold* h) {
  if (!h) return fail(LASGD_ERR_INVALID_ARGUMENT, "null hold");
  __sync_synchronize();
  *h->host = 1u;
  __sync_synchronize();
  return LASGD_OK;
}

extern "C" int lasgd_hold_destroy(lasgd_hold* h) {
  if (!h) return LASGD_OK;
  *h->host = 1u;
  cudaFreeHost((void*)h->host);
  delete h;
  return LASGD_OK;
}

// ---------------------------------------------------------------- device timestamps
// %globaltimer (ns, the clock the communicator's per-CTA trace uses) written in stream
// order: puts compute-stream events (forward start, backward end) on the same timeline
// as the side-stream all-reduce CTAs.
namespace lasgd {
__global__ void k_stamp(unsigned long long* out) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *out = t;
}
}  // namespace lasgd

extern "C" int lasgd_stamp(unsigned long long* out, void* stream) {
  if (!out) return fail(LASGD_ERR_INVALID_ARGUMENT, "null output");
  k_stamp<<<1, 1, 0, reinterpret_cast<cudaStream_t>(stream)>>>(out);
  LASGD_CUDA_TRY(cudaGetLastError());
  return LASGD_OK;
}
