/* Plain-C consumer of the C ABI (include/lasgd_sync.h): no Python, no torch.
 * Runs K5 (momentum + Nesterov + weight decay local step, optimizer.py:136-149 plus the
 * torch-SGD extensions) and K0 (blend, params.py:80-89) on the device and checks them
 * bit for bit against scalar C loops with the same rounding contract (every product
 * and sum separately rounded: build with -ffp-contract=off).
 *
 *   gcc -std=c11 -O2 -ffp-contract=off -I include -I $CUDA/include tests/c_abi/abi_smoke.c \
 *       -L paper_2203_13085_b200/_lib -llasgd_sync -L $CUDA/lib64 -lcudart -o abi_smoke
 */
#include <cuda_runtime_api.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "lasgd_sync.h"

#define CHECK(x)                                                                  \
  do {                                                                            \
    int rc_ = (x);                                                                \
    if (rc_ != 0) {                                                               \
      fprintf(stderr, "%s failed: %d (%s)\n", #x, rc_, lasgd_last_error());       \
      return 1;                                                                   \
    }                                                                             \
  } while (0)
#define CUDA(x)                                                                   \
  do {                                                                            \
    cudaError_t e_ = (x);                                                         \
    if (e_ != cudaSuccess) {                                                      \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));                    \
      return 1;                                                                   \
    }                                                                             \
  } while (0)

static unsigned bits(float f) {
  unsigned u;
  memcpy(&u, &f, sizeof u);
  return u;
}

int main(void) {
  const size_t n = 4099; /* ragged on purpose: vector body + scalar tail */
  const size_t bytes = n * sizeof(float);
  float *hx = malloc(bytes), *hg = malloc(bytes), *hm = malloc(bytes), *out = malloc(bytes);
  float *rx = malloc(bytes), *rm = malloc(bytes);
  unsigned seed = 12345u;
  for (size_t i = 0; i < n; ++i) {
    seed = seed * 1664525u + 1013904223u;
    hx[i] = (float)((int)(seed >> 8) % 20001 - 10000) / 7919.0f;
    seed = seed * 1664525u + 1013904223u;
    hg[i] = (float)((int)(seed >> 8) % 20001 - 10000) / 104729.0f;
    hm[i] = 0.0f;
  }
  if (lasgd_abi_version() != LASGD_ABI_VERSION) {
    fprintf(stderr, "ABI version mismatch\n");
    return 1;
  }
  float *dx, *dg, *dm, *dout;
  CUDA(cudaMalloc((void**)&dx, bytes));
  CUDA(cudaMalloc((void**)&dg, bytes));
  CUDA(cudaMalloc((void**)&dm, bytes));
  CUDA(cudaMalloc((void**)&dout, bytes));
  CUDA(cudaMemcpy(dx, hx, bytes, cudaMemcpyHostToDevice));
  CUDA(cudaMemcpy(dg, hg, bytes, cudaMemcpyHostToDevice));
  CUDA(cudaMemcpy(dm, hm, bytes, cudaMemcpyHostToDevice));
  memcpy(rx, hx, bytes);
  memcpy(rm, hm, bytes);

  /* three K5 steps: d = g + wd*x; m = d (first) | mu*m + (1-damp)*d; d = d + mu*m; x = x + (-lr)*d */
  const float mu = 0.9f, wd = 1e-4f;
  for (int step = 0; step < 3; ++step) {
    lasgd_sgd_params p = {0.05, 0.9, 0.0, 1e-4, 1, step == 0, 0};
    CHECK(lasgd_sgd_step(dx, dg, dm, NULL, n, LASGD_F32, &p, NULL, NULL));
    const float nlr = (float)(-0.05);
    for (size_t i = 0; i < n; ++i) {
      float d = hg[i] + wd * rx[i];
      rm[i] = step == 0 ? d : mu * rm[i] + (float)(1.0 - 0.0) * d;
      d = d + mu * rm[i];
      rx[i] = rx[i] + nlr * d;
    }
  }
  CUDA(cudaDeviceSynchronize());
  CUDA(cudaMemcpy(out, dx, bytes, cudaMemcpyDeviceToHost));
  for (size_t i = 0; i < n; ++i)
    if (bits(out[i]) != bits(rx[i])) {
      fprintf(stderr, "K5 mismatch at %zu: %.9g vs %.9g\n", i, out[i], rx[i]);
      return 1;
    }

  /* K0: out = 0.25*x + (-1.5)*g */
  CHECK(lasgd_blend(dout, 0.25, dx, -1.5, dg, n, LASGD_F32, NULL, NULL));
  CUDA(cudaDeviceSynchronize());
  CUDA(cudaMemcpy(out, dout, bytes, cudaMemcpyDeviceToHost));
  for (size_t i = 0; i < n; ++i) {
    const float want = 0.25f * rx[i] + (-1.5f) * hg[i];
    if (bits(out[i]) != bits(want)) {
      fprintf(stderr, "K0 mismatch at %zu\n", i);
      return 1;
    }
  }

  /* error path: a dimension/argument error comes back as a negative code with a message */
  if (lasgd_sgd_step(NULL, dg, dm, NULL, n, LASGD_F32, NULL, NULL, NULL) >= 0) {
    fprintf(stderr, "expected an error for null arguments\n");
    return 1;
  }
  size_t bounds[3 + 1]; /* num_chunks + 1 boundaries */
  CHECK(lasgd_partition_chunks(10, 3, bounds));
  if (bounds[0] != 0 || bounds[1] != 4 || bounds[2] != 7 || bounds[3] != 10) {
    fprintf(stderr, "partition_chunks(10, 3) wrong\n");
    return 1;
  }
  printf("c abi ok: K5 x3 and K0 bit-exact vs scalar C (n=%zu), errors and partition via the C ABI\n", n);
  cudaFree(dx);
  cudaFree(dg);
  cudaFree(dm);
  cudaFree(dout);
  free(hx), free(hg), free(hm), free(out), free(rx), free(rm);
  return 0;
}
