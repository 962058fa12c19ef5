// NVLink SHARP probe: mean all-reduce of a 102 MB fp32 buffer through a multicast object
// (one process, all GPUs).  Each GPU reduces its 1/P chunk in the switch with
// multimem.ld_reduce (sum over every GPU's copy) and multicasts the mean with
// multimem.st.  Compared with the P2P kernels this moves (P+1)/P*B per GPU link
// direction instead of 2(P-1)/P*B, and the SMs issue only B/P of loads + B/P of stores.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvls_probe tools/nvls_probe.cu -lcuda
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

#define CU(x)                                                                              \
  do {                                                                                     \
    CUresult r_ = (x);                                                                     \
    if (r_ != CUDA_SUCCESS) {                                                              \
      const char* s_ = nullptr;                                                            \
      cuGetErrorString(r_, &s_);                                                           \
      printf("%s:%d %s -> %s\n", __FILE__, __LINE__, #x, s_ ? s_ : "?");                   \
      return 1;                                                                            \
    }                                                                                      \
  } while (0)
#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));                   \
      return 1;                                                                            \
    }                                                                                      \
  } while (0)

__device__ __forceinline__ float4 mm_ld_reduce_add(const float* p) {
  float4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ void mm_st(float* p, float4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}

// chunk [c0, c1) in float4 units: sum over all GPUs in the switch, scale, multicast back.
// U independent multimem loads in flight per thread (the switch round trip is long:
// one load per thread leaves the reduction latency-bound).
template <int U>
__global__ void __launch_bounds__(256) k_nvls_mean(float* mc_src, float* mc_dst, size_t c0, size_t c1, float inv) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = c0 + blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < c1; i += U * stride) {
    float4 s[U];
#pragma unroll
    for (int u = 0; u < U; ++u) s[u] = mm_ld_reduce_add(mc_src + 4 * (i + u * stride));
#pragma unroll
    for (int u = 0; u < U; ++u) {
      s[u].x *= inv;
      s[u].y *= inv;
      s[u].z *= inv;
      s[u].w *= inv;
      mm_st(mc_dst + 4 * (i + u * stride), s[u]);
    }
  }
  for (; i < c1; i += stride) {
    float4 s = mm_ld_reduce_add(mc_src + 4 * i);
    s.x *= inv;
    s.y *= inv;
    s.z *= inv;
    s.w *= inv;
    mm_st(mc_dst + 4 * i, s);
  }
}

// multicast fan-out only: this GPU's chunk (plain local loads) stored once through the
// switch into every GPU's copy of the destination
template <int U>
__global__ void __launch_bounds__(256) k_nvls_bcast(const float* src, float* mc_dst, size_t c0, size_t c1) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = c0 + blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < c1; i += U * stride) {
    float4 s[U];
#pragma unroll
    for (int u = 0; u < U; ++u) s[u] = __ldcs(reinterpret_cast<const float4*>(src) + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) mm_st(mc_dst + 4 * (i + u * stride), s[u]);
  }
  for (; i < c1; i += stride) mm_st(mc_dst + 4 * i, __ldcs(reinterpret_cast<const float4*>(src) + i));
}

template <int U>
void launch_mean(int ctas, cudaStream_t s, float* src, float* dst, size_t c0, size_t c1, float inv) {
  k_nvls_mean<U><<<ctas, 256, 0, s>>>(src, dst, c0, c1, inv);
}

int main() {
  CU(cuInit(0));
  int P = 0;
  CK(cudaGetDeviceCount(&P));
  if (P < 2) {
    printf("need >= 2 GPUs\n");
    return 0;
  }
  const size_t bytes = 102228128;
  CUmulticastObjectProp mp = {};
  mp.numDevices = P;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_NONE;
  size_t gran = 0;
  mp.size = bytes;
  CU(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  const size_t S = (bytes + gran - 1) / gran * gran;
  mp.size = 2 * S;  // src and dst regions
  CUmemGenericAllocationHandle mc;
  CU(cuMulticastCreate(&mc, &mp));
  CUdevice devs[8];
  for (int d = 0; d < P; ++d) {
    CU(cuDeviceGet(&devs[d], d));
    CU(cuMulticastAddDevice(mc, devs[d]));
  }
  float* uc[8];
  float* mcp[8];
  cudaStream_t st[8];
  cudaEvent_t e0[8], e1[8];
  for (int d = 0; d < P; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaFree(0));
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = d;
    CUmemGenericAllocationHandle h;
    CU(cuMemCreate(&h, 2 * S, &ap, 0));
    CU(cuMulticastBindMem(mc, 0, h, 0, 2 * S, 0));
    CUdeviceptr va, mva;
    CUmemAccessDesc acc = {};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = d;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CU(cuMemAddressReserve(&va, 2 * S, gran, 0, 0));
    CU(cuMemMap(va, 2 * S, 0, h, 0));
    CU(cuMemSetAccess(va, 2 * S, &acc, 1));
    CU(cuMemAddressReserve(&mva, 2 * S, gran, 0, 0));
    CU(cuMemMap(mva, 2 * S, 0, mc, 0));
    CU(cuMemSetAccess(mva, 2 * S, &acc, 1));
    uc[d] = (float*)va;
    mcp[d] = (float*)mva;
    CK(cudaMemset(uc[d], 0, 2 * S));
    CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
  }
  // contributions: rank d holds value d+1 everywhere -> mean = (P+1)/2
  const size_t n = bytes / 4, n4 = n / 4;
  for (int d = 0; d < P; ++d) {
    CK(cudaSetDevice(d));
    float* h = new float[1024];
    for (int i = 0; i < 1024; ++i) h[i] = (float)(d + 1);
    for (size_t off = 0; off < n; off += 1024)
      CK(cudaMemcpy(uc[d] + off, h, sizeof(float) * (off + 1024 <= n ? 1024 : n - off), cudaMemcpyHostToDevice));
    delete[] h;
  }
  for (int mode = 0; mode < 2; ++mode)
  for (int U : {1, 4}) {
  for (int ctas : {148, 296, 592}) {
    float best = 1e9;
    for (int rep = 0; rep < 6; ++rep) {
      for (int d = 0; d < P; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaDeviceSynchronize());
      }
      for (int d = 0; d < P; ++d) {
        CK(cudaSetDevice(d));
        const size_t c0 = n4 * d / P, c1 = n4 * (d + 1) / P;
        CK(cudaEventRecord(e0[d], st[d]));
        if (mode == 1) {
          if (U == 1) k_nvls_bcast<1><<<ctas, 256, 0, st[d]>>>(uc[d], mcp[d] + S / 4, c0, c1);
          else k_nvls_bcast<4><<<ctas, 256, 0, st[d]>>>(uc[d], mcp[d] + S / 4, c0, c1);
        } else if (U == 1) launch_mean<1>(ctas, st[d], mcp[d], mcp[d] + S / 4, c0, c1, 1.0f / P);
        else launch_mean<4>(ctas, st[d], mcp[d], mcp[d] + S / 4, c0, c1, 1.0f / P);
        CK(cudaEventRecord(e1[d], st[d]));
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
    float check = 0;
    CK(cudaSetDevice(P - 1));
    CK(cudaMemcpy(&check, uc[P - 1] + S / 4 + 12345, 4, cudaMemcpyDeviceToHost));
    printf("{\"mode\": \"%s\", \"P\": %d, \"U\": %d, \"ctas\": %d, \"us\": %.1f, \"algbw_GBps\": %.1f, \"check\": %.3f, \"expect\": %.3f}\n", mode ? "bcast" : "mean", P, U, ctas,
           best * 1e3, bytes / (best * 1e-3) / 1e9, check, mode ? (double)P : (P + 1) / 2.0);
    fflush(stdout);
  }
  }
  return 0;
}
