// Launch plumbing of the communicator kernels: plain / cooperative launch, cached
// cooperative capacity, and the dispatchers over (element type, world size, algorithm).
// The dispatchers are defined and explicitly instantiated in comm_launch_*.cu so the
// kernel families compile as separate translation units.
#ifndef LASGD_COMM_LAUNCH_CUH
#define LASGD_COMM_LAUNCH_CUH

#include <map>
#include <mutex>
#include <utility>

#include "comm_fused.cuh"

namespace lasgd {

template <typename... Args>
int launch_kernel(bool coop, void (*kernel)(Args...), dim3 grid, int threads, cudaStream_t s, Args... args) {
  if (!coop) {  // programmatic dependent launch: the kernels start with pdl_entry()
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(threads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    LASGD_CUDA_TRY(cudaLaunchKernelEx(&cfg, kernel, args...));
    return LASGD_OK;
  }
  void* kargs[] = {(void*)&args...};
  LASGD_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)kernel, grid, dim3(threads), kargs, 0, s));
  return LASGD_OK;
}

template <typename... Args>
int coop_capacity(void (*kernel)(Args...), int threads) {
  // cached per (kernel, threads): an occupancy query per launch costs host time every step
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> cache;
  const auto key = std::make_pair(reinterpret_cast<const void*>(kernel), threads);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  const int cap = per_sm * num_sms();
  std::lock_guard<std::mutex> lk(mu);
  cache[key] = cap;
  return cap;
}

// Launch `kernel` normally, or cooperatively (all CTAs co-resident, required by the
// rank-level barrier of the P2P two-shot and push kernels).  A cooperative grid is
// clamped to what fits on the device — every rank computes the same clamp on the same
// GPU type, so the per-CTA flag slots still line up.
template <typename T, bool VIRTUAL>
int launch_allreduce(int algo, int P, const CommArgs& a, dim3 grid, int threads, cudaStream_t s);
template <typename T, bool VIRTUAL>
int launch_fused(int P, const CommArgs& a, const FusedRound<T>& f, dim3 grid, int threads, cudaStream_t s,
                 int algo = LASGD_ALGO_ONESHOT);
template <typename T, bool VIRTUAL>
int launch_push(int P, const CommArgs& a, const FusedRound<T>& f, dim3 grid, int threads, cudaStream_t s);

// the all-reduce with every byte moved by remote stores (ALGO_PUSH through lasgd_comm_allreduce)
template <typename T>
int launch_push_mean(int P, const CommArgs& a, dim3 grid, int threads, cudaStream_t s);
extern template int launch_push_mean<float>(int, const CommArgs&, dim3, int, cudaStream_t);
extern template int launch_push_mean<double>(int, const CommArgs&, dim3, int, cudaStream_t);

#define LASGD_EXTERN_LAUNCHERS(T, V)                                                                          \
  extern template int launch_allreduce<T, V>(int, int, const CommArgs&, dim3, int, cudaStream_t);            \
  extern template int launch_fused<T, V>(int, const CommArgs&, const FusedRound<T>&, dim3, int, cudaStream_t, \
                                         int);                                                                \
  extern template int launch_push<T, V>(int, const CommArgs&, const FusedRound<T>&, dim3, int, cudaStream_t);
LASGD_EXTERN_LAUNCHERS(float, false)
LASGD_EXTERN_LAUNCHERS(float, true)
LASGD_EXTERN_LAUNCHERS(double, false)
LASGD_EXTERN_LAUNCHERS(double, true)
#undef LASGD_EXTERN_LAUNCHERS

}  // namespace lasgd

#endif  // LASGD_COMM_LAUNCH_CUH
