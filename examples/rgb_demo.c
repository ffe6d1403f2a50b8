/* rgb_demo.c -- the drop-in boundary used from plain C (no Python, no torch):
 * solve_batch of a small rank-deficient system through librgb.so's C ABI
 * (include/rgb.h), the way a C/C++ or other-FFI host would call it.
 *
 *   nvcc -o rgb_demo examples/rgb_demo.c -Iinclude -Lpaper_2106_11594_b200 -lrgb -lcudart \
 *        -Xlinker -rpath=$PWD/paper_2106_11594_b200
 *   ./rgb_demo            # prints rank, branch sequence and the residual of x
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime.h>

#include "rgb.h"

#define CHECK(x)                                                          \
  do {                                                                    \
    int rc_ = (x);                                                        \
    if (rc_ != RGB_OK) {                                                  \
      fprintf(stderr, "%s failed (%d): %s\n", #x, rc_, rgb_last_error()); \
      return 1;                                                           \
    }                                                                     \
  } while (0)

int main(void) {
  enum { N = 12, M = 6, R = 3 };
  double A[N][M], y[N], x[M];
  /* A = G1 G2 with integer factors (rank 3, exact), y consistent with x0 = (1..6) */
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < M; ++j) {
      double s = 0.0;
      for (int t = 0; t < R; ++t) s += (double)((i + 2 * t) % 5 - 2) * (double)((j * (t + 1)) % 4 - 1);
      A[i][j] = s;
    }
  for (int i = 0; i < N; ++i) {
    y[i] = 0.0;
    for (int j = 0; j < M; ++j) y[i] += A[i][j] * (double)(j + 1);
  }
  rgb_config cfg = {1, M, 1, M, RGB_F64, RGB_GENERAL, RGB_EPS_AUTO, 0.0, 1.0};
  double *C, *D, *P, *X, *rows, *tg;
  int32_t *rank, *status;
  int64_t *nobs;
  uint8_t *branch;
  cudaMalloc((void**)&C, sizeof(double) * M * M);
  cudaMalloc((void**)&D, sizeof(double) * M * M);
  cudaMalloc((void**)&P, sizeof(double) * M * M);
  cudaMalloc((void**)&X, sizeof(double) * M);
  cudaMalloc((void**)&rows, sizeof(A));
  cudaMalloc((void**)&tg, sizeof(y));
  cudaMalloc((void**)&rank, sizeof(int32_t));
  cudaMalloc((void**)&status, sizeof(int32_t));
  cudaMalloc((void**)&nobs, sizeof(int64_t));
  cudaMalloc((void**)&branch, N);
  rgb_state st = {C, D, P, X, rank, nobs, status};
  rgb_logs logs = {branch, NULL, NULL, NULL};
  cudaMemcpy(rows, A, sizeof(A), cudaMemcpyHostToDevice);
  cudaMemcpy(tg, y, sizeof(y), cudaMemcpyHostToDevice);
  CHECK(rgb_state_reset(&cfg, &st, NULL));
  CHECK(rgb_ingest(&cfg, &st, rows, 0, tg, 0, N, &logs, NULL));
  int32_t r = 0, stat = 0;
  uint8_t br[N];
  cudaMemcpy(x, X, sizeof(x), cudaMemcpyDeviceToHost);
  cudaMemcpy(&r, rank, sizeof(r), cudaMemcpyDeviceToHost);
  cudaMemcpy(&stat, status, sizeof(stat), cudaMemcpyDeviceToHost);
  cudaMemcpy(br, branch, N, cudaMemcpyDeviceToHost);
  double res = 0.0;
  for (int i = 0; i < N; ++i) {
    double ax = 0.0;
    for (int j = 0; j < M; ++j) ax += A[i][j] * x[j];
    res = fmax(res, fabs(ax - y[i]));
  }
  printf("abi %d rank %d status %d branches ", rgb_abi_version(), r, stat);
  for (int i = 0; i < N; ++i) printf("%d", br[i]);
  printf(" max|Ax-y| %.3e\n", res);
  return (r == R && stat == 0 && res < 1e-9) ? 0 : 2;
}
