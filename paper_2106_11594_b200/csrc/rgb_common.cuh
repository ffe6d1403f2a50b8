// rgb_common.cuh -- shared helpers for the rank-Greville CUDA kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/rgb.h"

namespace rgb {

template <typename REAL>
struct Num;
template <>
struct Num<double> {
  // float64 machine epsilon, scalars.py:141-147
  static __device__ __forceinline__ double eps_m() { return 2.220446049250313e-16; }
};
template <>
struct Num<float> {
  static __device__ __forceinline__ float eps_m() { return 1.1920928955078125e-07f; }
};

// Threshold of EpsPolicy (solver.py:66-72, inline copy solver.py:292-295):
// auto -> (m^2 r + m r + m) eps_M with r the CURRENT rank; fixed -> value.
// The operation count is an exact integer; eps_M is a power of two, so the
// product is exact and eps^2 is rounded once, as in the reference.
template <typename REAL>
__device__ __forceinline__ REAL eps_sq(const rgb_config& cfg, int r) {
  REAL e;
  if (cfg.eps_mode == RGB_EPS_FIXED) {
    e = (REAL)cfg.eps_value;
  } else {
    long long m = cfg.m;
    e = (REAL)(double)(m * m * r + m * r + m) * Num<REAL>::eps_m();
  }
  return e * e;
}

// Rank test of solver.py:296 / is_dependent (solver.py:221-229).
template <typename REAL>
__device__ __forceinline__ bool is_dependent(REAL rej_sq, REAL row_sq, REAL esq) {
  return (rej_sq < esq) || (rej_sq < esq * row_sq);
}

// Opt a kernel into more than 48 KB of dynamic shared memory, once per device
// (the attribute belongs to the device's context, so a per-process flag would
// skip every device after the first).  Setting it twice from racing host
// threads is harmless.
template <typename K>
inline void smem_attr_once(K kern, size_t smem, bool (&done)[64]) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    return;
  }
  if (!done[dev]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    done[dev] = true;
  }
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace rgb
