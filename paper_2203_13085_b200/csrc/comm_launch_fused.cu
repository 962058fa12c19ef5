// Dispatch of the fused round kernels (K7 one-shot / two-shot).
// Separate translation unit: see comm_launch.cuh.
#include "comm_fused.cuh"
#include "comm_launch.cuh"

namespace lasgd {

template <typename T, bool VIRTUAL>
int launch_fused(int P, const CommArgs& a, const FusedRound<T>& f, dim3 grid, int threads, cudaStream_t s,
                 int algo) {
  static_assert(sizeof(CommArgs) + sizeof(FusedRound<T>) < 4000, "kernel parameters");
#define LASGD_FCASE(PP)                                                                             \
  case PP:                                                                                          \
    if (algo == LASGD_ALGO_TWOSHOT && PP > 1) {                                                     \
      auto kern = k_fused_twoshot<T, PP, VIRTUAL, (PP <= 4 && sizeof(T) == 4 ? 2 : 1)>;                               \
      CommArgs aa = a;                                                                              \
      if (!VIRTUAL) {                                                                               \
        const int cap = coop_capacity(kern, threads);                                               \
        if ((int)grid.x > cap) grid.x = cap;                                                        \
        aa.nblocks = grid.x;                                                                        \
      }                                                                                             \
      return launch_kernel(!VIRTUAL, kern, grid, threads, s, aa, f);                                \
    }                                                                                               \
    return launch_kernel(false, k_fused_round<T, PP, VIRTUAL, (PP <= 2 && sizeof(T) == 4 ? 2 : 1)>, grid, threads, s, \
                         a, f);
  switch (P) {
    LASGD_FCASE(1)
    LASGD_FCASE(2)
    LASGD_FCASE(3)
    LASGD_FCASE(4)
    LASGD_FCASE(5)
    LASGD_FCASE(6)
    LASGD_FCASE(7)
    LASGD_FCASE(8)
    default: return fail(LASGD_ERR_UNSUPPORTED, "world size %d > %d", P, kMaxR);
  }
#undef LASGD_FCASE
  LASGD_CUDA_TRY(cudaGetLastError());
  return LASGD_OK;
}

template int launch_fused<float, false>(int, const CommArgs&, const FusedRound<float>&, dim3, int, cudaStream_t, int);
template int launch_fused<float, true>(int, const CommArgs&, const FusedRound<float>&, dim3, int, cudaStream_t, int);
template int launch_fused<double, false>(int, const CommArgs&, const FusedRound<double>&, dim3, int, cudaStream_t, int);
template int launch_fused<double, true>(int, const CommArgs&, const FusedRound<double>&, dim3, int, cudaStream_t, int);

}  // namespace lasgd
