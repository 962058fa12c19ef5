// Dispatch of the mean all-reduce kernels (K2 one-shot, K3 two-shot).
// Separate translation unit: see comm_launch.cuh.
#include "comm_allreduce.cuh"
#include "comm_launch.cuh"

namespace lasgd {

// packs in flight per thread of the two-shot reduce-scatter / all-gather, sized so the
// loaded data fits the 128 registers of __launch_bounds__(256, 2) without spills
template <typename T, int P>
constexpr int unroll_for() { return (P <= 2 ? 8 : (P <= 4 ? 4 : 2)) / (sizeof(T) == 8 && P <= 4 ? 2 : 1); }
template <typename T, int P>
constexpr int ag_unroll() { return (sizeof(T) == 8 || P >= 5) ? 4 : 8; }
template <int P>
constexpr int oneshot_unroll() { return P <= 2 ? 4 : (P <= 4 ? 2 : 1); }  // <= 128 regs, no spills

template <typename T, bool VIRTUAL>
int launch_allreduce(int algo, int P, const CommArgs& a, dim3 grid, int threads, cudaStream_t s) {
#define LASGD_CASE(PP)                                                                                    \
  case PP:                                                                                                \
    if (algo == LASGD_ALGO_ONESHOT) return launch_kernel(false, k_oneshot<T, PP, VIRTUAL, oneshot_unroll<PP>()>, \
                                                         grid, threads, s, a);                            \
    {                                                                                                     \
      auto kern = k_twoshot<T, PP, VIRTUAL, unroll_for<T, PP>(), ag_unroll<T, PP>()>;                                         \
      CommArgs aa = a;                                                                                    \
      if (!VIRTUAL) {                                                                                     \
        const int cap = coop_capacity(kern, threads);                                                     \
        if ((int)grid.x > cap) grid.x = cap;                                                              \
        aa.nblocks = grid.x;                                                                              \
      }                                                                                                   \
      return launch_kernel(!VIRTUAL, kern, grid, threads, s, aa);                                         \
    }
  switch (P) {
    LASGD_CASE(1)
    LASGD_CASE(2)
    LASGD_CASE(3)
    LASGD_CASE(4)
    LASGD_CASE(5)
    LASGD_CASE(6)
    LASGD_CASE(7)
    LASGD_CASE(8)
    default: return fail(LASGD_ERR_UNSUPPORTED, "world size %d > %d", P, kMaxR);
  }
#undef LASGD_CASE
  LASGD_CUDA_TRY(cudaGetLastError());
  return LASGD_OK;
}

template int launch_allreduce<float, false>(int, int, const CommArgs&, dim3, int, cudaStream_t);
template int launch_allreduce<float, true>(int, int, const CommArgs&, dim3, int, cudaStream_t);
template int launch_allreduce<double, false>(int, int, const CommArgs&, dim3, int, cudaStream_t);
template int launch_allreduce<double, true>(int, int, const CommArgs&, dim3, int, cudaStream_t);

}  // namespace lasgd
