/* A C host driving an l1-Cox fit through the solver-level C ABI alone (no Python):
 * X (m x n, float32, column-major) = Generator(Philox(key)).random stream drawn on the
 * device, delta from a host array, then bs_cox_run.  Prints one objective per line.
 *
 *   gcc -O2 -I include examples/cox_host.c -o cox_host \
 *       -L paper_2010_16114_b200 -lbsb200 -L/usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_2010_16114_b200 -Wl,-rpath,/usr/local/cuda/lib64
 *   ./cox_host KEY0 KEY1 [iters]        (keys: numpy's Philox(seed).state key words) */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "bsb200.h"

#define CHECK(call)                                                               \
  do {                                                                            \
    int rc_ = (call);                                                             \
    if (rc_) {                                                                    \
      fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, bs_last_error());       \
      return 1;                                                                   \
    }                                                                             \
  } while (0)

int main(int argc, char** argv) {
  const int64_t m = 4096, n = 256;
  if (argc < 3) {
    fprintf(stderr, "usage: %s KEY0 KEY1 [iters]\n", argv[0]);
    return 2;
  }
  const uint64_t k0 = strtoull(argv[1], NULL, 10), k1 = strtoull(argv[2], NULL, 10);
  const int iters = argc > 3 ? atoi(argv[3]) : 10;
  float *X, *beta, *grad, *delta;
  if (cudaMalloc((void**)&X, sizeof(float) * m * n) || cudaMalloc((void**)&beta, sizeof(float) * n) ||
      cudaMalloc((void**)&grad, sizeof(float) * n) || cudaMalloc((void**)&delta, sizeof(float) * m)) {
    fprintf(stderr, "cudaMalloc failed\n");
    return 1;
  }
  CHECK(bs_philox_uniform(X, BS_F32, m * n, 0, k0, k1, NULL));  /* rand_fill(common_init=True) */
  cudaMemset(beta, 0, sizeof(float) * n);
  float* hd = (float*)malloc(sizeof(float) * m);
  for (int64_t i = 0; i < m; ++i) hd[i] = (float)((i * 7919) % 10 < 6);  /* 60% events */
  cudaMemcpy(delta, hd, sizeof(float) * m, cudaMemcpyHostToDevice);
  bs_ctx_t ctx;
  bs_cox_t st;
  CHECK(bs_ctx_create(0, 1, 0, NULL, NULL, &ctx));
  CHECK(bs_cox_state_create(ctx, X, BS_F32, BS_F32, m, n, delta, NULL, 1e-4, 1e-5, beta, grad, &st));
  double* trace = (double*)malloc(sizeof(double) * (size_t)iters);
  int nt = 0, ran = 0, flags = 0;
  CHECK(bs_cox_run(st, iters, 1, 0, 0.0, trace, &nt, &ran, &flags));
  for (int i = 0; i < nt; ++i) printf("%.17g\n", trace[i]);
  CHECK(bs_cox_state_destroy(st));
  CHECK(bs_ctx_destroy(ctx));
  free(trace);
  free(hd);
  cudaFree(X);
  cudaFree(beta);
  cudaFree(grad);
  cudaFree(delta);
  return 0;
}
