/*
 * CPU ORACLE (C restatement) of the LASGD parameter-synchronisation path.
 * TEST INFRASTRUCTURE ONLY: pinned by tests/test_c_oracle.py (reference goldens in f64,
 * the Python oracle bit for bit in f32); used by bench.py
 * as the timed CPU baseline ("kind": "port") / the `--impl reference` arm.
 * The product path never links or loads this library.
 *
 * Same arithmetic contract as oracle/lasgd_oracle.py (which is pinned to the
 * reference by tests/golden/): every product and sum separately rounded
 * (compiled with -ffp-contract=off, no -ffast-math), scalars rounded to the
 * element type first, ring mean summed per chunk in rotated rank order.
 * Elementwise loops are split across OpenMP threads (static schedule); the
 * arithmetic per element is independent of the thread count.
 *
 * Reference anchors (/root/reference/pkg/src/lasgd):
 *   blend                params.py:80-89       -> *_blend
 *   _check_finite        params.py:23-26       -> fused non-finite counts
 *   partition_chunks     params.py:130-147     -> chunk bounds in *_ring_mean
 *   execute_allreduce    collective.py:154-203 -> *_ring_mean
 *   sgd_local_step       optimizer.py:136-149  -> *_sgd_delta
 *   lasgd_finalize_round optimizer.py:152-178  -> *_finalize
 *   elastic pull (blend order of optimizer.py:256-257) -> *_pull
 */
#include <stddef.h>
#include <stdint.h>
#include <math.h>
#include <string.h>
#include <omp.h>

#define EXPORT __attribute__((visibility("default")))

EXPORT void oracle_set_threads(int n) { if (n > 0) omp_set_num_threads(n); }
EXPORT int oracle_get_threads(void) { return omp_get_max_threads(); }

#define DEFINE_OPS(T, SFX)                                                                    \
  /* out = a*u + b*v (params.py:87) ; returns number of non-finite outputs (params.py:88) */ \
  EXPORT int64_t oracle_blend_##SFX(T* out, double a, const T* u, double b, const T* v,      \
                                    int64_t n) {                                              \
    const T ta = (T)a, tb = (T)b;                                                             \
    int64_t bad = 0;                                                                          \
    _Pragma("omp parallel for schedule(static) reduction(+:bad)")                             \
    for (int64_t i = 0; i < n; ++i) {                                                         \
      T p = ta * u[i];                                                                        \
      T q = tb * v[i];                                                                        \
      T r = p + q;                                                                            \
      out[i] = r;                                                                             \
      bad += !isfinite(r);                                                                    \
    }                                                                                         \
    return bad;                                                                               \
  }                                                                                           \
  /* sgd_local_step: x' = 1*x + (-eta)*g ; delta' = 1*delta + (-eta)*g (optimizer.py:145-146) \
     out-of-place like the reference; delta_reset models the fresh zeros of :174 */          \
  EXPORT int64_t oracle_sgd_delta_##SFX(T* x_out, T* d_out, const T* x, const T* d,         \
                                        const T* g, int64_t n, double eta, int delta_reset) { \
    const T ne = (T)(-eta), one = (T)1.0;                                                     \
    int64_t bad = 0;                                                                          \
    _Pragma("omp parallel for schedule(static) reduction(+:bad)")                             \
    for (int64_t i = 0; i < n; ++i) {                                                         \
      T step = ne * g[i];                                                                     \
      T xn = one * x[i] + step;                                                               \
      T d0 = delta_reset ? (T)0 : d[i];                                                       \
      T dn = one * d0 + step;                                                                 \
      x_out[i] = xn;                                                                          \
      d_out[i] = dn;                                                                          \
      bad += !isfinite(xn) + !isfinite(dn);                                                   \
    }                                                                                         \
    return bad;                                                                               \
  }                                                                                           \
  /* momentum / weight decay step, torch.optim.SGD order, each op rounded (see oracle .py) */ \
  EXPORT int64_t oracle_sgd_momentum_##SFX(T* x, const T* g, T* m, int64_t n, double lr,     \
                                           double mu, double damp, double wd, int nesterov,  \
                                           int first) {                                       \
    const T nlr = (T)(-lr), tmu = (T)mu, tdp = (T)(1.0 - damp), twd = (T)wd;                  \
    int64_t bad = 0;                                                                          \
    _Pragma("omp parallel for schedule(static) reduction(+:bad)")                             \
    for (int64_t i = 0; i < n; ++i) {                                                         \
      T xi = x[i];                                                                            \
      T d = g[i];                                                                             \
      if (wd != 0.0) { T t = twd * xi; d = d + t; }                                           \
      if (mu != 0.0) {                                                                        \
        T mi;                                                                                 \
        if (first) mi = d; else { T p = tmu * m[i]; T q = tdp * d; mi = p + q; }              \
        m[i] = mi;                                                                            \
        if (nesterov) { T t = tmu * mi; d = d + t; } else d = mi;                             \
      }                                                                                       \
      T s = nlr * d;                                                                          \
      T xn = xi + s;                                                                          \
      x[i] = xn;                                                                              \
      bad += !isfinite(xn);                                                                   \
    }                                                                                         \
    return bad;                                                                               \
  }                                                                                           \
  /* lasgd_finalize_round (P>1): new = 1*z + 1*delta (optimizer.py:171) */                    \
  EXPORT int64_t oracle_finalize_##SFX(T* out, const T* z, const T* d, int64_t n) {          \
    int64_t bad = 0;                                                                          \
    _Pragma("omp parallel for schedule(static) reduction(+:bad)")                             \
    for (int64_t i = 0; i < n; ++i) {                                                         \
      T r = z[i] + d[i];                                                                      \
      out[i] = r;                                                                             \
      bad += !isfinite(r);                                                                    \
    }                                                                                         \
    return bad;                                                                               \
  }                                                                                           \
  /* pull: diff = 1*snap + (-1)*xbar ; x = 1*x + (-alpha)*diff ; snap_next = x */            \
  EXPORT int64_t oracle_pull_##SFX(T* x, T* snap_next, const T* snap, const T* xbar,         \
                                   int64_t n, double alpha) {                                 \
    const T na = (T)(-alpha), m1 = (T)(-1.0);                                                 \
    int64_t bad = 0;                                                                          \
    _Pragma("omp parallel for schedule(static) reduction(+:bad)")                             \
    for (int64_t i = 0; i < n; ++i) {                                                         \
      T diff = snap[i] + m1 * xbar[i];                                                        \
      T s = na * diff;                                                                        \
      T xn = x[i] + s;                                                                        \
      x[i] = xn;                                                                              \
      if (snap_next) snap_next[i] = xn;                                                       \
      bad += !isfinite(diff) + !isfinite(xn);                                                 \
    }                                                                                         \
    return bad;                                                                               \
  }                                                                                           \
  /* execute_allreduce: chunk c summed x_c, x_{c+1}, ..., x_{c-1}; then / P.                  \
     Writes the mean to each of the n_out output vectors (one per rank, like per_rank). */    \
  EXPORT int64_t oracle_ring_mean_##SFX(T* const* outs, int n_out, const T* const* srcs,     \
                                        int P, int64_t n) {                                   \
    int64_t bad = 0;                                                                          \
    if (P == 1) {                                                                             \
      for (int o = 0; o < n_out; ++o)                                                         \
        if (outs[o] != srcs[0]) memcpy(outs[o], srcs[0], (size_t)n * sizeof(T));              \
      return 0;                                                                               \
    }                                                                                         \
    const int64_t base = n / P, rem = n % P;                                                  \
    const T tP = (T)P;                                                                        \
    _Pragma("omp parallel for schedule(static) reduction(+:bad)")                             \
    for (int64_t i = 0; i < n; ++i) {                                                         \
      int64_t big = rem * (base + 1);                                                         \
      int c = (int)(base == 0 ? i : (i < big ? i / (base + 1) : rem + (i - big) / base));     \
      T acc = srcs[c][i];                                                                     \
      for (int k = 1; k < P; ++k) acc = acc + srcs[(c + k) % P][i];                           \
      T r = acc / tP;                                                                         \
      for (int o = 0; o < n_out; ++o) outs[o][i] = r;                                         \
      bad += !isfinite(r);                                                                    \
    }                                                                                         \
    return bad;                                                                               \
  }                                                                                           \
  EXPORT void oracle_copy_##SFX(T* dst, const T* src, int64_t n) {                            \
    _Pragma("omp parallel for schedule(static)")                                              \
    for (int64_t i = 0; i < n; ++i) dst[i] = src[i];                                          \
  }

DEFINE_OPS(float, f32)
DEFINE_OPS(double, f64)
