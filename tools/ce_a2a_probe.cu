// Copy-engine all-to-all at P GPUs (design probe for a CE-driven two-shot mean): every
// GPU sends its B/P chunk q to GPU q's staging buffer (the reduce-scatter's data
// movement), all GPUs at once, with cudaMemcpyPeerAsync.  Modes:
//   seq    one stream per GPU, the P-1 copies back to back (push: issued by the sender)
//   par    P-1 streams per GPU, one copy each, concurrently
//   pull   one stream per GPU, the receiver issues the copies (dst local, src remote)
//   round  seq scatter + a reduce kernel (ring-order sum of the P staged chunks) + seq
//          all-gather of the mean chunk: the whole two-shot mean on copy engines
// Prints the max-over-GPUs device time and GB/s per direction (bytes each GPU sends).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ce_a2a_probe tools/ce_a2a_probe.cu
//   tools/ce_a2a_probe [P] [MB]
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));        \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

// mean of P staged chunks (the own one included), fixed order, plain fp32
__global__ void k_reduce(const float* __restrict__ stage, float* __restrict__ out, size_t m, int P) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < m; i += (size_t)gridDim.x * blockDim.x) {
    float s = stage[i];
    for (int q = 1; q < P; ++q) s = __fadd_rn(s, stage[q * m + i]);
    out[i] = __fdiv_rn(s, (float)P);
  }
}

int main(int argc, char** argv) {
  int nd = 0;
  CK(cudaGetDeviceCount(&nd));
  int P = argc > 1 ? atoi(argv[1]) : nd;
  double mb = argc > 2 ? atof(argv[2]) : 102.228128;
  if (P < 2 || P > nd) {
    printf("{\"error\": \"need %d GPUs, have %d\"}\n", P, nd);
    return 0;
  }
  const size_t bytes = ((size_t)(mb * 1e6) / (16 * P)) * 16 * P;
  const size_t chunk = bytes / P;
  std::vector<char*> src(P), stage(P), mean(P);
  std::vector<cudaStream_t> st(P * P);
  std::vector<cudaEvent_t> e0(P), e1(P);
  for (int d = 0; d < P; ++d) {
    CK(cudaSetDevice(d));
    for (int p = 0; p < P; ++p)
      if (p != d) CK(cudaDeviceEnablePeerAccess(p, 0));
    CK(cudaMalloc(&src[d], bytes));
    CK(cudaMalloc(&stage[d], bytes));  // P slots of one chunk
    CK(cudaMalloc(&mean[d], bytes));   // the gathered mean
    CK(cudaMemset(src[d], 0, bytes));
    for (int k = 0; k < P; ++k) CK(cudaStreamCreateWithFlags(&st[d * P + k], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
  }
  const char* modes[] = {"seq", "par", "pull", "round"};
  for (int mode = 0; mode < 4; ++mode) {
    float best = 1e30f;
    for (int it = 0; it < 12; ++it) {
      for (int d = 0; d < P; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaDeviceSynchronize());
      }
      for (int d = 0; d < P; ++d) {
        CK(cudaSetDevice(d));
        cudaStream_t s = st[d * P];
        CK(cudaEventRecord(e0[d], s));
        if (mode == 1)
          for (int k = 1; k < P; ++k) CK(cudaStreamWaitEvent(st[d * P + k], e0[d], 0));
        for (int j = 1; j < P; ++j) {
          int q = (d + j) % P;
          if (mode == 2) {  // receiver d pulls chunk d of GPU q into its slot q
            CK(cudaMemcpyPeerAsync(stage[d] + q * chunk, d, src[q] + d * chunk, q, chunk, s));
          } else {  // sender d pushes its chunk q into GPU q's slot d
            CK(cudaMemcpyPeerAsync(stage[q] + d * chunk, q, src[d] + q * chunk, d, chunk, mode == 1 ? st[d * P + j] : s));
          }
        }
        if (mode == 1)
          for (int k = 1; k < P; ++k) {
            cudaEvent_t ev;
            CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            CK(cudaEventRecord(ev, st[d * P + k]));
            CK(cudaStreamWaitEvent(s, ev, 0));
            CK(cudaEventDestroy(ev));
          }
      }
      if (mode == 3) {
        // (a real round needs a cross-GPU barrier here; the probe synchronises the host)
        for (int d = 0; d < P; ++d) {
          CK(cudaSetDevice(d));
          CK(cudaStreamSynchronize(st[d * P]));
        }
        for (int d = 0; d < P; ++d) {
          CK(cudaSetDevice(d));
          k_reduce<<<296, 256, 0, st[d * P]>>>((const float*)stage[d], (float*)(mean[d] + d * chunk), chunk / 4, P);
          CK(cudaStreamSynchronize(st[d * P]));
        }
        for (int d = 0; d < P; ++d) {
          CK(cudaSetDevice(d));
          for (int j = 1; j < P; ++j) {
            int q = (d + j) % P;
            CK(cudaMemcpyPeerAsync(mean[q] + d * chunk, q, mean[d] + d * chunk, d, chunk, st[d * P]));
          }
        }
      }
      float worst = 0;
      for (int d = 0; d < P; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaEventRecord(e1[d], st[d * P]));
      }
      for (int d = 0; d < P; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaEventSynchronize(e1[d]));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
        worst = ms > worst ? ms : worst;
      }
      if (it >= 2 && worst < best) best = worst;
    }
    double out = (double)(P - 1) * chunk * (mode == 3 ? 2 : 1);
    printf("{\"probe\": \"ce_a2a\", \"P\": %d, \"bytes\": %zu, \"mode\": \"%s\", \"ms\": %.4f, "
           "\"gbs_per_direction\": %.1f%s}\n",
           P, bytes, modes[mode], best, out / best / 1e6,
           mode == 3 ? ", \"note\": \"host-synchronised phases: upper bound of a device-signalled round\"" : "");
  }
  return 0;
}
