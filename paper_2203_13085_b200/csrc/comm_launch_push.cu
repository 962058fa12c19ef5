// Dispatch of the push round kernels (K8: mirror form at P = 2, staged form at P >= 3).
// Separate translation unit: see comm_launch.cuh.
#include "comm_push.cuh"
#include "comm_launch.cuh"

namespace lasgd {

template <typename T, bool VIRTUAL>
int launch_push(int P, const CommArgs& a, const FusedRound<T>& f, dim3 grid, int threads, cudaStream_t s) {
#define LASGD_PCASE(PP)                                                                             \
  case PP: {                                                                                        \
    auto kern = k_push_round<T, PP, VIRTUAL, (PP <= 4 && sizeof(T) == 4 ? 2 : 1)>;                                    \
    CommArgs aa = a;                                                                                \
    if (!VIRTUAL) {                                                                                 \
      const int cap = coop_capacity(kern, threads);                                                 \
      if ((int)grid.x > cap) grid.x = cap;                                                          \
      aa.nblocks = grid.x;                                                                          \
    }                                                                                               \
    return launch_kernel(!VIRTUAL, kern, grid, threads, s, aa, f);                                  \
  }
  if (P == 2) {  // mirror form: one phase, no barrier inside the launch, so no cooperative launch
    auto kern = k_push_mirror<T, VIRTUAL, sizeof(T) == 4 ? 2 : 1>;
    CommArgs aa = a;
    if (!VIRTUAL) {
      const int cap = coop_capacity(kern, threads);
      if ((int)grid.x > cap) grid.x = cap;
      aa.nblocks = grid.x;
    }
    return launch_kernel(false, kern, grid, threads, s, aa, f);
  }
  switch (P) {
    LASGD_PCASE(3)
    LASGD_PCASE(4)
    LASGD_PCASE(5)
    LASGD_PCASE(6)
    LASGD_PCASE(7)
    LASGD_PCASE(8)
    default: return fail(LASGD_ERR_UNSUPPORTED, "push round needs 2 <= P <= %d, got %d", kMaxR, P);
  }
#undef LASGD_PCASE
}

// packs in flight per thread, sized so the P loaded packs fit 128 registers without spills
template <typename T, int P>
constexpr int push_mean_unroll() { return sizeof(T) == 4 ? (P <= 3 ? 4 : (P <= 6 ? 2 : 1)) : (P <= 3 ? 2 : 1); }

template <typename T>
int launch_push_mean(int P, const CommArgs& a, dim3 grid, int threads, cudaStream_t s) {
#define LASGD_MCASE(PP)                                                       \
  case PP: {                                                                  \
    auto kern = k_push_mean<T, PP, push_mean_unroll<T, PP>()>;                \
    CommArgs aa = a;                                                          \
    const int cap = coop_capacity(kern, threads);                             \
    if ((int)grid.x > cap) grid.x = cap;                                      \
    aa.nblocks = grid.x;                                                      \
    return launch_kernel(true, kern, grid, threads, s, aa);                   \
  }
  switch (P) {
    LASGD_MCASE(2)
    LASGD_MCASE(3)
    LASGD_MCASE(4)
    LASGD_MCASE(5)
    LASGD_MCASE(6)
    LASGD_MCASE(7)
    LASGD_MCASE(8)
    default: return fail(LASGD_ERR_UNSUPPORTED, "push mean needs 2 <= P <= %d, got %d", kMaxR, P);
  }
#undef LASGD_MCASE
}

template int launch_push_mean<float>(int, const CommArgs&, dim3, int, cudaStream_t);
template int launch_push_mean<double>(int, const CommArgs&, dim3, int, cudaStream_t);

template int launch_push<float, false>(int, const CommArgs&, const FusedRound<float>&, dim3, int, cudaStream_t);
template int launch_push<float, true>(int, const CommArgs&, const FusedRound<float>&, dim3, int, cudaStream_t);
template int launch_push<double, false>(int, const CommArgs&, const FusedRound<double>&, dim3, int, cudaStream_t);
template int launch_push<double, true>(int, const CommArgs&, const FusedRound<double>&, dim3, int, cudaStream_t);

}  // namespace lasgd
