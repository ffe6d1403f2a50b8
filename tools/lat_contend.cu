// fp64 CUDA-core chain latency on one warp while other warps stream independent
// DMMAs: on the same SM sub-partition (warp slot mod 4) vs another one.
#include <cstdio>
#include <cuda_runtime.h>

#define N 2048
__global__ void k(double* out, long long* cyc, int mode, double seed) {
  unsigned wid;
  asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
  double a = seed + threadIdx.x, b = 1.0000001, c = 1e-9;
  __shared__ volatile int done;
  if (threadIdx.x == 0) done = 0;
  __syncthreads();
  if (wid == 0) {
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) { a = fma(a, b, c); a = fma(a, b, c); a = a * b; a = a * b; }
    long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) { cyc[0] = (t1 - t0) / (4 * N); done = 1; }
  } else {
    bool stream = (mode == 1 && (wid & 3) == 0) || (mode == 2 && (wid & 3) == 1) || (mode == 3);
    if (stream) {
      double d[8][2] = {};
      while (!done) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(d[j][0]), "+d"(d[j][1]) : "d"(a), "d"(b));
      }
      double s = 0; for (int j = 0; j < 8; ++j) s += d[j][0] + d[j][1];
      a += s;
    }
  }
  out[threadIdx.x] = a;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMallocManaged(&c, 16 * 8);
  const char* nm[] = {"alone", "DMMA streams on the same sub-partition", "DMMA streams on another sub-partition", "DMMA streams on every warp"};
  for (int mode = 0; mode < 4; ++mode) {
    k<<<1, 256>>>(o, c, mode, 1.0); cudaDeviceSynchronize();
    k<<<1, 256>>>(o, c, mode, 1.0); cudaDeviceSynchronize();
    printf("fp64 chain op latency, %-40s %lld cycles\n", nm[mode], c[0]);
  }
  return 0;
}
