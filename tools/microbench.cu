// Microbenchmarks for the B200 numbers the rank-Greville kernels depend on:
// fp64 FMA throughput (vector pipe), fp64 mma.sync (DMMA) throughput,
// fp64 warp-shuffle throughput and latencies.  Built and run by hand:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dfma_tput(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void ffma_tput(float* out, int iters, float a, float b) {
  float acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-3f + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fmaf(acc[c], a, b);
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678f) out[0] = s;
}

template <int CHAINS>
__global__ void dmma_tput(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double d[CHAINS][2];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) { d[c][0] = c; d[c][1] = -c; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += d[c][0] + d[c][1];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void shfl_tput(double* out, int iters) {
  double v[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) v[c] = threadIdx.x + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) v[c] = __shfl_xor_sync(0xffffffffu, v[c], (c & 15) + 1);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += v[c];
  if (s == 12345.678) out[0] = s;
}

__global__ void lat_kernel(long long* out, double* dout, int iters) {
  double x = threadIdx.x * 1e-9 + 1.0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, 1.0000001, 1e-9);
  long long t1 = clock64();
  for (int i = 0; i < iters; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1);
  long long t2 = clock64();
  for (int i = 0; i < iters; ++i) x = 1.0 / (x + 0.5);
  long long t3 = clock64();
  __shared__ double sm[64];
  sm[threadIdx.x] = x; __syncwarp();
  int idx = threadIdx.x;
  for (int i = 0; i < iters; ++i) { double y = sm[idx]; idx = (int)(y * 0.0) + ((idx + 1) & 31); x += y; }
  long long t4 = clock64();
  for (int i = 0; i < iters; ++i) x = x + 1e-9;
  long long t5 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3; out[4] = t5 - t4; }
  dout[threadIdx.x] = x;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("{\"device\": \"%s\", \"sms\": %d, \"clock_khz\": %d, \"l2_bytes\": %d, \"smem_per_sm\": %zu, \"regs_per_sm\": %d}\n",
         p.name, p.multiProcessorCount, clk, p.l2CacheSize, p.sharedMemPerMultiprocessor, p.regsPerMultiprocessor);
  double* dbuf; CK(cudaMalloc(&dbuf, 1 << 20)); float* fbuf = (float*)dbuf; long long* lbuf; CK(cudaMalloc(&lbuf, 1024));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  auto timeit = [&](auto launch) { launch(); cudaDeviceSynchronize(); float best = 1e30f;
    for (int r = 0; r < 5; ++r) { cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
    return best; };
  const int it = 4096;
  for (int bpsm : {1, 2, 4}) {
    int blocks = sms * bpsm, threads = 256;
    float ms = timeit([&] { dfma_tput<8><<<blocks, threads>>>(dbuf, it, 1.0000001, 1e-9); });
    double fl = 2.0 * 8 * it * (double)blocks * threads;
    printf("{\"test\": \"dfma\", \"blocks_per_sm\": %d, \"tflops\": %.3f}\n", bpsm, fl / ms / 1e9);
    ms = timeit([&] { ffma_tput<8><<<blocks, threads>>>(fbuf, it, 1.0000001f, 1e-9f); });
    printf("{\"test\": \"ffma\", \"blocks_per_sm\": %d, \"tflops\": %.3f}\n", bpsm, fl / ms / 1e9);
    ms = timeit([&] { dmma_tput<4><<<blocks, threads>>>(dbuf, it / 4); });
    fl = 2.0 * 256 * 4 * (it / 4) * (double)blocks * (threads / 32);
    printf("{\"test\": \"dmma_m8n8k4\", \"blocks_per_sm\": %d, \"tflops\": %.3f}\n", bpsm, fl / ms / 1e9);
    ms = timeit([&] { shfl_tput<8><<<blocks, threads>>>(dbuf, it); });
    double shfl = 8.0 * it * (double)blocks * (threads / 32);  // fp64 warp-shuffles
    printf("{\"test\": \"shfl_f64\", \"blocks_per_sm\": %d, \"warp_shfl_f64_per_clk_per_sm\": %.3f}\n", bpsm,
           shfl / (ms * 1e-3) / sms / (clk * 1e3));
  }
  lat_kernel<<<1, 32>>>(lbuf, dbuf, 1000); cudaDeviceSynchronize();
  long long h[5]; cudaMemcpy(h, lbuf, sizeof(h), cudaMemcpyDeviceToHost);
  printf("{\"test\": \"latency_cycles\", \"dfma\": %.1f, \"shfl_f64\": %.1f, \"ddiv_chain\": %.1f, \"lds_chain\": %.1f, \"dadd\": %.1f}\n",
         h[0] / 1000.0, h[1] / 1000.0, h[2] / 1000.0, h[3] / 1000.0, h[4] / 1000.0);
  CK(cudaGetLastError());
  return 0;
}
