// DMMA m8n8k4 latency / per-warp throughput vs independent accumulator chains.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void chain(long long* out, double* dout, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double d[CH][2];
#pragma unroll
  for (int c = 0; c < CH; ++c) { d[c][0] = c; d[c][1] = -c; }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
  dout[threadIdx.x + blockIdx.x * blockDim.x] = s;
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}
template <int CH> void run(int warps) {
  long long* o; double* d; cudaMalloc(&o, 8 * 64); cudaMalloc(&d, 8 * 4096);
  int it = 2000;
  chain<CH><<<1, 32 * warps>>>(o, d, it); cudaDeviceSynchronize();
  chain<CH><<<1, 32 * warps>>>(o, d, it); cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
  printf("{\"chains\": %d, \"warps_per_sm\": %d, \"cycles_per_mma_per_warp\": %.2f, \"sm_mma_per_cycle\": %.4f}\n",
         CH, warps, (double)h / (it * CH), (double)it * CH * warps / h);
  cudaFree(o); cudaFree(d);
}
int main() {
  run<1>(1); run<2>(1); run<4>(1); run<8>(1); run<16>(1);
  run<1>(4); run<2>(4); run<4>(4); run<8>(4);
  run<1>(8); run<2>(8); run<4>(8);
  run<1>(16); run<2>(16);
  return 0;
}
