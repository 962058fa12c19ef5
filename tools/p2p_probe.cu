// NVLink peer-access probe (one process, 2 GPUs with peer access): bandwidth of
//   ldg  : kernel on GPU a reads GPU b's buffer (LDG.128), writes local
//   stg  : kernel on GPU a reads local, writes GPU b's buffer (STG.128)
//   tma  : kernel on GPU a bulk-copies (cp.async.bulk) GPU b's buffer into smem, then
//          bulk-stores smem into a local buffer
//   ce   : cudaMemcpyPeerAsync (copy engine)
// each unidirectional (only GPU0 active) and bidirectional (both GPUs at once).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o p2p_probe p2p_probe.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s failed: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_ldg(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n16) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i + 7 * st < n16; i += 8 * st) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcg(src + i + u * st);
#pragma unroll
    for (int u = 0; u < 8; ++u) __stcs(dst + i + u * st, v[u]);
  }
  for (; i < n16; i += st) __stcs(dst + i, __ldcg(src + i));
}

__global__ void k_stg(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n16) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i + 7 * st < n16; i += 8 * st) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcs(src + i + u * st);
#pragma unroll
    for (int u = 0; u < 8; ++u) dst[i + u * st] = v[u];
  }
  for (; i < n16; i += st) dst[i] = __ldcs(src + i);
}

// TMA bulk: per CTA, STAGES buffers of TILE bytes; thread 0 drives the pipeline.
template <int TILE, int STAGES>
__global__ void __launch_bounds__(32) k_tma(const char* __restrict__ src, char* __restrict__ dst, size_t bytes) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t bar[STAGES];
  const size_t ntiles = bytes / TILE;
  if (threadIdx.x != 0) return;
  for (int s = 0; s < STAGES; ++s) {
    uint32_t a = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a));
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint32_t phase[STAGES] = {0};
  size_t t = blockIdx.x;
  int issued = 0;
  // prologue
  size_t tt = t;
  for (int s = 0; s < STAGES && tt < ntiles; ++s, tt += gridDim.x) {
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    uint32_t d = (uint32_t)__cvta_generic_to_shared(smem + s * TILE);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(TILE) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(d), "l"(src + tt * TILE), "r"(TILE), "r"(b) : "memory");
    issued++;
  }
  int s = 0;
  for (; t < ntiles; t += gridDim.x) {
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    uint32_t d = (uint32_t)__cvta_generic_to_shared(smem + s * TILE);
    // wait tile
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }"
                 ::"r"(b), "r"(phase[s]) : "memory");
    phase[s] ^= 1;
    // store tile to local global
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + t * TILE), "r"(d), "r"(TILE) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    // refill this stage
    size_t nt = t + (size_t)STAGES * gridDim.x;
    if (nt < ntiles) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(TILE) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(d), "l"(src + nt * TILE), "r"(TILE), "r"(b) : "memory");
    }
    s = (s + 1) % STAGES;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

struct Bufs { char* loc[2]; char* rem[2]; };

int main() {
  int nd = 0;
  cudaGetDeviceCount(&nd);
  if (nd < 2) { printf("need 2 GPUs\n"); return 0; }
  const size_t bytes = (size_t)1 << 30;
  char *a[2], *b[2];
  cudaStream_t st[2];
  cudaEvent_t e0[2], e1[2];
  int sms = 148;
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceEnablePeerAccess(1 - d, 0));
    CK(cudaMalloc(&a[d], bytes));
    CK(cudaMalloc(&b[d], bytes));
    CK(cudaMemset(a[d], 1, bytes));
    CK(cudaMemset(b[d], 2, bytes));
    CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
    CK(cudaFuncSetAttribute(k_tma<16384, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 * 8));
    CK(cudaFuncSetAttribute(k_tma<32768, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 * 6));
  }
  const char* names[] = {"ldg", "stg", "tma16k", "tma32k", "ce"};
  for (int m = 0; m < 5; ++m) {
    for (int bidir = 0; bidir < 2; ++bidir) {
      for (int ctas : {32, 64, 148, 296}) {
        if (m == 4 && ctas != 32) continue;
        float best = 1e9;
        for (int rep = 0; rep < 4; ++rep) {
          for (int d = 0; d <= bidir; ++d) {
            CK(cudaSetDevice(d));
            CK(cudaEventRecord(e0[d], st[d]));
            const int o = 1 - d;
            if (m == 0) k_ldg<<<ctas, 512, 0, st[d]>>>((const uint4*)a[o], (uint4*)b[d], bytes / 16);
            if (m == 1) k_stg<<<ctas, 512, 0, st[d]>>>((const uint4*)a[d], (uint4*)b[o], bytes / 16);
            if (m == 2) k_tma<16384, 8><<<ctas, 32, 16384 * 8, st[d]>>>(a[o], b[d], bytes);
            if (m == 3) k_tma<32768, 6><<<ctas, 32, 32768 * 6, st[d]>>>(a[o], b[d], bytes);
            if (m == 4) CK(cudaMemcpyPeerAsync(b[d], d, a[o], o, bytes, st[d]));
            CK(cudaEventRecord(e1[d], st[d]));
          }
          float ms = 0;
          for (int d = 0; d <= bidir; ++d) {
            CK(cudaSetDevice(d));
            CK(cudaEventSynchronize(e1[d]));
            float t;
            CK(cudaEventElapsedTime(&t, e0[d], e1[d]));
            ms = t > ms ? t : ms;
          }
          if (rep > 0 && ms < best) best = ms;
        }
        printf("{\"method\": \"%s\", \"bidir\": %d, \"ctas\": %d, \"GBps_per_direction\": %.1f}\n", names[m], bidir,
               m == 4 ? 0 : ctas, bytes / (best * 1e-3) / 1e9);
        fflush(stdout);
      }
    }
  }
  return 0;
}
