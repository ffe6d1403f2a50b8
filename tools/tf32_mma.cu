// Throughput of legacy warp-level mma.sync on sm_100a for tf32 and f16 inputs.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void tf32_loop(float* out, int iters) {
  unsigned a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = __float_as_uint(1.0f + threadIdx.x * 1e-3f + i);
  for (int i = 0; i < 2; ++i) b[i] = __float_as_uint(1.0f - threadIdx.x * 1e-4f + i);
  float d[CH][4];
  for (int c = 0; c < CH; ++c) for (int i = 0; i < 4; ++i) d[c][i] = c + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0;
  for (int c = 0; c < CH; ++c) for (int i = 0; i < 4; ++i) s += d[c][i];
  if (s == 1234.5f) out[0] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* buf; cudaMalloc(&buf, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int wpb : {4, 8, 16}) {
    int blocks = sms * 2, threads = 32 * wpb, it = 4096;
    tf32_loop<4><<<blocks, threads>>>(buf, it); cudaDeviceSynchronize();
    cudaEventRecord(e0); tf32_loop<4><<<blocks, threads>>>(buf, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 16 * 8 * 8 * 4.0 * it * blocks * wpb;
    printf("{\"test\": \"tf32_mma_sync_m16n8k8\", \"warps_per_block\": %d, \"tflops\": %.1f}\n", wpb, fl / ms / 1e9);
  }
  return 0;
}
