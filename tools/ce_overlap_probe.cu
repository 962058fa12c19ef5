// Copy-engine peer traffic next to an HBM-bound kernel (design probe for a CE-fed
// fused round).  Two GPUs, peer access on: each GPU's copy stream pulls the other
// GPU's 102 MB buffer with cudaMemcpyPeerAsync (bidirectional NVLink through the copy
// engines, whole or in chunks) while its compute stream runs a streaming kernel that
// moves 7 x 102 MB of HBM (the fused round's local traffic).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ce_overlap_probe tools/ce_overlap_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));        \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

// 4 streams read, 3 written (x, g, m, snap -> x, m, snap'): 7 x n4 x 16 bytes
__global__ void __launch_bounds__(256) k_stream(const uint4* __restrict__ a, const uint4* __restrict__ b,
                                                uint4* __restrict__ c, uint4* __restrict__ d, uint4* __restrict__ e,
                                                size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    uint4 va = __ldcs(a + i), vb = __ldcs(b + i), vc = __ldcs(c + i), vd = __ldcs(d + i);
    uint4 r;
    r.x = va.x ^ vb.x ^ vc.x;
    r.y = va.y ^ vb.y ^ vd.y;
    r.z = va.z + vb.z;
    r.w = vc.w + vd.w;
    __stcs(c + i, r);
    __stcs(d + i, va);
    __stcs(e + i, vb);
  }
}

int main() {
  int nd = 0;
  cudaGetDeviceCount(&nd);
  if (nd < 2) {
    printf("need 2 GPUs\n");
    return 0;
  }
  const size_t bytes = 102228128;
  const size_t n4 = bytes / 16;
  char *src[2], *dst[2], *buf[2][5];
  cudaStream_t cs[2], ks[2];
  cudaEvent_t ev[2][4];
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceEnablePeerAccess(1 - d, 0));
    CK(cudaMalloc(&src[d], bytes));
    CK(cudaMalloc(&dst[d], bytes));
    for (int k = 0; k < 5; ++k) {
      CK(cudaMalloc(&buf[d][k], bytes));
      CK(cudaMemset(buf[d][k], k, bytes));
    }
    CK(cudaMemset(src[d], 1, bytes));
    CK(cudaStreamCreateWithFlags(&cs[d], cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&ks[d], cudaStreamNonBlocking));
    for (int k = 0; k < 4; ++k) CK(cudaEventCreate(&ev[d][k]));
  }
  const char* names[] = {"copy_only", "kernel_only", "both"};
  for (int chunks : {1, 16}) {
    for (int mode = 0; mode < 3; ++mode) {
      float best_c = 1e9, best_k = 1e9, best_span = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        for (int d = 0; d < 2; ++d) {
          CK(cudaSetDevice(d));
          CK(cudaDeviceSynchronize());
        }
        for (int d = 0; d < 2; ++d) {
          CK(cudaSetDevice(d));
          CK(cudaEventRecord(ev[d][0], cs[d]));
          CK(cudaEventRecord(ev[d][2], ks[d]));
          if (mode != 1) {
            const size_t cb = (bytes / chunks + 255) / 256 * 256;
            for (size_t off = 0; off < bytes; off += cb) {
              const size_t len = off + cb <= bytes ? cb : bytes - off;
              CK(cudaMemcpyPeerAsync(dst[d] + off, d, src[1 - d] + off, 1 - d, len, cs[d]));
            }
          }
          if (mode != 0)
            k_stream<<<296, 256, 0, ks[d]>>>((const uint4*)buf[d][0], (const uint4*)buf[d][1], (uint4*)buf[d][2],
                                             (uint4*)buf[d][3], (uint4*)buf[d][4], n4);
          CK(cudaEventRecord(ev[d][1], cs[d]));
          CK(cudaEventRecord(ev[d][3], ks[d]));
        }
        float tc = 0, tk = 0, span = 0;
        for (int d = 0; d < 2; ++d) {
          CK(cudaSetDevice(d));
          CK(cudaDeviceSynchronize());
          float a, b, s1, s2;
          CK(cudaEventElapsedTime(&a, ev[d][0], ev[d][1]));
          CK(cudaEventElapsedTime(&b, ev[d][2], ev[d][3]));
          CK(cudaEventElapsedTime(&s1, ev[d][0], ev[d][3]));
          CK(cudaEventElapsedTime(&s2, ev[d][2], ev[d][1]));
          tc = a > tc ? a : tc;
          tk = b > tk ? b : tk;
          const float sp = (a > b ? a : b);
          span = sp > span ? sp : span;
          (void)s1;
          (void)s2;
        }
        if (rep > 0) {
          best_c = tc < best_c ? tc : best_c;
          best_k = tk < best_k ? tk : best_k;
          best_span = span < best_span ? span : best_span;
        }
      }
      printf("{\"case\": \"%s\", \"chunks\": %d, \"copy_us\": %.1f, \"copy_GBps\": %.1f, \"kernel_us\": %.1f, "
             "\"kernel_hbm_GBps\": %.1f, \"span_us\": %.1f}\n",
             names[mode], chunks, mode != 1 ? best_c * 1e3 : 0.0, mode != 1 ? bytes / (best_c * 1e-3) / 1e9 : 0.0,
             mode != 0 ? best_k * 1e3 : 0.0, mode != 0 ? 7.0 * bytes / (best_k * 1e-3) / 1e9 : 0.0, best_span * 1e3);
      fflush(stdout);
    }
  }
  return 0;
}
