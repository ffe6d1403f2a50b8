// fp64_peak.cu -- live fp64 peak probe for bench.py's roofline denominator.
// MEASURED_PEAKS.json carries HBM and bf16 peaks only; this measures, on the
// same box and in the same process as the bench, the fp64 throughput of
//   which = 0: DFMA (CUDA-core fp64 pipe)
//   which = 1: DMMA m8n8k4 (fp64 tensor path, mma.sync)
//   which = 2: FFMA (CUDA-core fp32 pipe; the fp32-state roofline)
//   which = 3: mma.sync m16n8k8 tf32 (warp-level tf32 tensor path, for reference)
// as TFLOP/s (best of 5 launches, CUDA events).  Not part of librgb.so.
#include <cuda_runtime.h>

template <int CH>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

template <int CH>
__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double d[CH][2];
#pragma unroll
  for (int c = 0; c < CH; ++c) { d[c][0] = c; d[c][1] = -c; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
  if (s == 12345.678) out[0] = s;
}

template <int CH>
__global__ void ffma_loop(float* out, int iters, float a, float b) {
  float acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-3f + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fmaf(acc[c], a, b);
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 12345.678f) out[0] = s;
}

template <int CH>
__global__ void tf32mma_loop(float* out, int iters) {
  unsigned a[4], b[2];
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = __float_as_uint(threadIdx.x * 1e-3f + i);
  b[0] = __float_as_uint(1.0f);
  b[1] = __float_as_uint(0.5f);
  float d[CH][4];
#pragma unroll
  for (int c = 0; c < CH; ++c)
#pragma unroll
    for (int i = 0; i < 4; ++i) d[c][i] = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};\n"
          : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  if (s == 12345.678f) out[0] = s;
}

extern "C" double rgb_probe_fp64_peak(int which) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* buf = nullptr;
  if (cudaMalloc(&buf, 64) != cudaSuccess) return -1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 4, threads = 256, it = 8192;
  const double warps = (double)blocks * (threads / 32);
  double flops = (which == 0 || which == 2) ? 2.0 * 8 * it * (double)blocks * threads
                 : which == 1              ? 2.0 * 256 * 4 * (it / 4) * warps
                                           : 2.0 * 16 * 8 * 8 * 4 * (it / 4) * warps;
  float best = 1e30f;
  for (int r = 0; r < 6; ++r) {
    cudaEventRecord(e0);
    if (which == 0) dfma_loop<8><<<blocks, threads>>>(buf, it, 1.0000001, 1e-9);
    else if (which == 1) dmma_loop<4><<<blocks, threads>>>(buf, it / 4);
    else if (which == 2) ffma_loop<8><<<blocks, threads>>>((float*)buf, it, 1.0000001f, 1e-9f);
    else tf32mma_loop<4><<<blocks, threads>>>((float*)buf, it / 4);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r > 0 && ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(buf);
  if (cudaGetLastError() != cudaSuccess) return -1;
  return flops / (best * 1e-3) / 1e12;
}
