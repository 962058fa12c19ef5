// NVLink fan-out stores mixed with local HBM streaming (design probe for the P >= 3 push
// round).  Per GPU, the push round's work at P = 4: 153 MB of remote stores (a 51 MB
// source fanned out to 3 peers) and ~1 GB of local HBM traffic (4 streams read,
// 3 written).  Variants:
//   push_only / hbm_only      each half alone
//   interleaved               one kernel, every thread does both (the current design)
//   concurrent                two kernels on two streams, disjoint CTA counts (a stand-in
//                             for warp/CTA specialisation)
// All GPUs run the same variant at once (all-to-all traffic).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mix_probe tools/mix_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));        \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

struct Args {
  const uint4* push_src;
  uint4* push_dst[8];
  int npeers;
  size_t push_n;        // packs in the push source
  const uint4* r[4];    // local read streams
  uint4* w[3];          // local write streams
  size_t hbm_n;         // packs per local stream
};

__device__ __forceinline__ void push_range(const Args& a, size_t i) {
  const uint4 v = __ldcs(a.push_src + i);
  for (int k = 0; k < a.npeers; ++k) a.push_dst[k][i] = v;
}
__device__ __forceinline__ void hbm_range(const Args& a, size_t i) {
  uint4 v0 = __ldcs(a.r[0] + i), v1 = __ldcs(a.r[1] + i), v2 = __ldcs(a.r[2] + i), v3 = __ldcs(a.r[3] + i);
  uint4 o;
  o.x = v0.x ^ v1.x;
  o.y = v1.y ^ v2.y;
  o.z = v2.z ^ v3.z;
  o.w = v3.w ^ v0.w;
  __stcs(a.w[0] + i, o);
  __stcs(a.w[1] + i, v0);
  __stcs(a.w[2] + i, v3);
}

__global__ void __launch_bounds__(256) k_push(Args a) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < a.push_n; i += (size_t)gridDim.x * blockDim.x)
    push_range(a, i);
}
__global__ void __launch_bounds__(256) k_hbm(Args a) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < a.hbm_n; i += (size_t)gridDim.x * blockDim.x)
    hbm_range(a, i);
}
// interleaved: the index space of the larger job; push work spread uniformly over it
__global__ void __launch_bounds__(256) k_mixed(Args a) {
  const size_t ratio = (a.hbm_n + a.push_n - 1) / a.push_n;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < a.hbm_n; i += (size_t)gridDim.x * blockDim.x) {
    hbm_range(a, i);
    if (i % ratio == 0 && i / ratio < a.push_n) push_range(a, i / ratio);
  }
}

int main(int argc, char** argv) {
  int P = 0;
  cudaGetDeviceCount(&P);
  if (P < 2) {
    printf("need >= 2 GPUs\n");
    return 0;
  }
  // defaults: the P = 4 staged push round; argv: push source MB, MB per local stream
  const size_t push_bytes = (argc > 1 ? (size_t)atoi(argv[1]) : 51ull) << 20;
  const size_t hbm_bytes = (argc > 2 ? (size_t)atoi(argv[2]) : 146ull) << 20;
  Args args[8];
  cudaStream_t s0[8], s1[8];
  cudaEvent_t e0[8], e1[8];
  char* recv[8];
  for (int d = 0; d < P; ++d) {
    CK(cudaSetDevice(d));
    for (int q = 0; q < P; ++q)
      if (q != d) CK(cudaDeviceEnablePeerAccess(q, 0));
    CK(cudaMalloc(&recv[d], push_bytes * P));
    char* src;
    CK(cudaMalloc(&src, push_bytes));
    CK(cudaMemset(src, 1, push_bytes));
    args[d].push_src = (const uint4*)src;
    args[d].push_n = push_bytes / 16;
    for (int k = 0; k < 4; ++k) {
      char* b;
      CK(cudaMalloc(&b, hbm_bytes));
      CK(cudaMemset(b, k, hbm_bytes));
      args[d].r[k] = (const uint4*)b;
    }
    for (int k = 0; k < 3; ++k) {
      char* b;
      CK(cudaMalloc(&b, hbm_bytes));
      args[d].w[k] = (uint4*)b;
    }
    args[d].hbm_n = hbm_bytes / 16;
    CK(cudaStreamCreateWithFlags(&s0[d], cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s1[d], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
  }
  for (int d = 0; d < P; ++d) {
    int k = 0;
    for (int q = 0; q < P; ++q)
      if (q != d) args[d].push_dst[k++] = (uint4*)(recv[q] + push_bytes * d);
    args[d].npeers = k;
  }
  const char* names[] = {"push_only", "hbm_only", "interleaved", "concurrent_74_222", "concurrent_148_148"};
  for (int v = 0; v < 5; ++v) {
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      for (int d = 0; d < P; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaDeviceSynchronize());
      }
      for (int d = 0; d < P; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaEventRecord(e0[d], s0[d]));
        CK(cudaStreamWaitEvent(s1[d], e0[d], 0));
        if (v == 0) k_push<<<296, 256, 0, s0[d]>>>(args[d]);
        if (v == 1) k_hbm<<<296, 256, 0, s0[d]>>>(args[d]);
        if (v == 2) k_mixed<<<296, 256, 0, s0[d]>>>(args[d]);
        if (v == 3) {
          k_push<<<74, 256, 0, s1[d]>>>(args[d]);
          k_hbm<<<222, 256, 0, s0[d]>>>(args[d]);
        }
        if (v == 4) {
          k_push<<<148, 256, 0, s1[d]>>>(args[d]);
          k_hbm<<<148, 256, 0, s0[d]>>>(args[d]);
        }
        cudaEvent_t done;
        CK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
        CK(cudaEventRecord(done, s1[d]));
        CK(cudaStreamWaitEvent(s0[d], done, 0));
        CK(cudaEventRecord(e1[d], s0[d]));
        CK(cudaEventDestroy(done));
      }
      float ms = 0;
      for (int d = 0; d < P; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaEventSynchronize(e1[d]));
        float t;
        CK(cudaEventElapsedTime(&t, e0[d], e1[d]));
        ms = t > ms ? t : ms;
      }
      if (rep > 0 && ms < best) best = ms;
    }
    const double pb = (double)push_bytes * (P - 1), hb = 7.0 * hbm_bytes;
    printf("{\"P\": %d, \"variant\": \"%s\", \"us\": %.1f, \"push_GBps\": %.1f, \"hbm_GBps\": %.1f}\n", P, names[v],
           best * 1e3, v == 1 ? 0.0 : pb / (best * 1e-3) / 1e9, v == 0 ? 0.0 : hb / (best * 1e-3) / 1e9);
    fflush(stdout);
  }
  return 0;
}
