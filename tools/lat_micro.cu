// Dependent-chain latencies on one warp (cycles per op): DFMA, DMUL, DADD,
// shfl of a double, MUFU rcp.approx.f64, DMMA m8n8k4, FFMA -- the building
// blocks of the LDL^T / row-mode chains.  Single CTA, single warp.
#include <cstdio>
#include <cuda_runtime.h>

#define N 256
__global__ void lat(double* out, long long* cyc, double seed) {
  double a = seed + threadIdx.x, b = 1.0000001, c = 1e-9;
  float fa = (float)a;
  long long t0, t1;
  // DFMA
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) { a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); }
  t1 = clock64(); cyc[0] = (t1 - t0) / (4 * N);
  // DMUL
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) { a = a * b; a = a * b; a = a * b; a = a * b; }
  t1 = clock64(); cyc[1] = (t1 - t0) / (4 * N);
  // DADD
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) { a = a + c; a = a + c; a = a + c; a = a + c; }
  t1 = clock64(); cyc[2] = (t1 - t0) / (4 * N);
  // shfl double
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) { a = __shfl_sync(0xffffffffu, a, (threadIdx.x + 1) & 31); a = __shfl_sync(0xffffffffu, a, (threadIdx.x + 3) & 31); }
  t1 = clock64(); cyc[3] = (t1 - t0) / (2 * N);
  // rcp.approx.f64
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a)); asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(a) : "d"(r)); }
  t1 = clock64(); cyc[4] = (t1 - t0) / (2 * N);
  // DMMA chain
  double d0 = 0, d1 = 0;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
  }
  t1 = clock64(); cyc[5] = (t1 - t0) / (2 * N);
  // FFMA
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) { fa = fmaf(fa, 1.0001f, 1e-7f); fa = fmaf(fa, 1.0001f, 1e-7f); fa = fmaf(fa, 1.0001f, 1e-7f); fa = fmaf(fa, 1.0001f, 1e-7f); }
  t1 = clock64(); cyc[6] = (t1 - t0) / (4 * N);
  // shared load chain (pointer chasing through a double index)
  __shared__ int sidx[64];
  if (threadIdx.x < 32) { sidx[threadIdx.x] = (threadIdx.x + 1) & 31; }
  __syncwarp();
  int j = threadIdx.x;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) { j = sidx[j]; j = sidx[j]; }
  t1 = clock64(); cyc[7] = (t1 - t0) / (2 * N);
  out[threadIdx.x] = a + d0 + d1 + fa + j;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 64 * 8); cudaMallocManaged(&c, 16 * 8);
  lat<<<1, 32>>>(o, c, 1.0); cudaDeviceSynchronize();
  lat<<<1, 32>>>(o, c, 1.0); cudaDeviceSynchronize();
  const char* nm[] = {"DFMA", "DMUL", "DADD", "SHFL.f64", "MUFU.RCP64", "DMMA", "FFMA", "LDS"};
  for (int i = 0; i < 8; ++i) printf("%-10s %lld cycles\n", nm[i], c[i]);
  return 0;
}
