// fp64_mix.cu -- do DMMA (fp64 tensor) and DFMA (fp64 CUDA-core) issue from
// different warps of one SM overlap, or share one pipe?  Times a DMMA-only,
// a DFMA-only and a mixed kernel (even warps DMMA, odd warps DFMA, the same
// per-warp work as the single-kind runs) and prints the three times.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma_work(int iters, double* out) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double d[4][2] = {{0, 1}, {2, 3}, {4, 5}, {6, 7}};
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int c = 0; c < 4; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a), "d"(b));
  double s = 0;
  for (int c = 0; c < 4; ++c) s += d[c][0] + d[c][1];
  if (s == 12345.678) out[0] = s;
}
__device__ __forceinline__ void dfma_work(int iters, double* out) {
  double acc[8];
  for (int c = 0; c < 8; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] = fma(acc[c], 1.0000001, 1e-9);
  double s = 0;
  for (int c = 0; c < 8; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}
// mode 0: all warps DMMA; 1: all warps DFMA; 2: even DMMA / odd DFMA;
// 3: even DMMA, odd idle; 4: even idle, odd DFMA
__global__ void mix(int mode, int it_mma, int it_fma, double* out) {
  const int w = threadIdx.x >> 5;
  const bool even = (w & 1) == 0;
  if (mode == 0 || ((mode == 2 || mode == 3) && even)) dmma_work(it_mma, out);
  else if (mode == 1 || ((mode == 2 || mode == 4) && !even)) dfma_work(it_fma, out);
}
int main() {
  double* out;
  cudaMalloc(&out, 64);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int it_mma = 4096, it_fma = 8192;
  const char* names[] = {"dmma-all", "dfma-all", "mixed", "dmma-half", "dfma-half"};
  for (int mode = 0; mode < 5; ++mode) {
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      mix<<<sms * 2, 256>>>(mode, it_mma, it_fma, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("%-10s %.3f ms\n", names[mode], best);
  }
  return 0;
}
