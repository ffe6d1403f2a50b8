// rgb_mma.cuh -- fp64 tensor-core, cp.async and reciprocal helpers shared by
// the blocked kernels (rgb_blocked.cu, rgb_blocked_wg.cu).
#pragma once

#include "rgb_common.cuh"

namespace rgb {
namespace blk {

constexpr unsigned FULL = 0xffffffffu;
constexpr int TT = 8;  // rows per tile

__device__ __forceinline__ void mma(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}


__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, int bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
// one lane slot of the staged input: 2 consecutive values (fp64 or fp32 input),
// widened exactly to double
template <typename TI>
__device__ __forceinline__ void cp_async_pair(TI* smem, const TI* gmem, bool ok) {
  if constexpr (sizeof(TI) == 8) cp_async16(smem, gmem, ok ? 16 : 0);
  else cp_async8(smem, gmem, ok ? 8 : 0);
}
template <typename TI>
__device__ __forceinline__ void cp_async_one(TI* smem, const TI* gmem, bool ok) {
  if constexpr (sizeof(TI) == 8) cp_async8(smem, gmem, ok ? 8 : 0);
  else cp_async4(smem, gmem, ok ? 4 : 0);
}
// lane slot i (a pair of values) of a staged tile, widened to double
__device__ __forceinline__ double2 slot(const double* base, int i) { return reinterpret_cast<const double2*>(base)[i]; }
__device__ __forceinline__ double2 slot(const float* base, int i) {
  const float2 f = reinterpret_cast<const float2*>(base)[i];
  return make_double2((double)f.x, (double)f.y);
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ int sigma(int kt, int q) { return 8 * (kt >> 1) + 2 * q + (kt & 1); }

// 1/x to within an ulp without branches: MUFU.RCP64H seed (rcp.approx.ftz.f64)
// and two Newton steps.  Only used for LDL^T pivots of I + G P G^T (>= 1).
__device__ __forceinline__ double rcp64(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// 8x8 LDL^T of the SPD matrix M (accumulator layout mi[e] = M[p][2q+e]):
// ev[e] = E[p][2q+e] with E = L^-1, rd0 / rd1 = 1/d at t = 2q, 2q+1.
__device__ __forceinline__ void ldl8(double (&mi)[2], double (&ev)[2], double& rd0, double& rd1, int p, int q) {
  // Gaussian elimination in registers, the same steps as the other blocked
  // kernels (a fraction-free variant without the reciprocal on the chain and a
  // one-Newton-step reciprocal were both measured slower here).
  ev[0] = p == 2 * q ? 1.0 : 0.0;
  ev[1] = p == 2 * q + 1 ? 1.0 : 0.0;
#pragma unroll
  for (int kk = 0; kk < TT - 1; ++kk) {
    const double v = (kk & 1) ? mi[1] : mi[0];
    const double piv = __shfl_sync(FULL, v, 4 * kk + (kk >> 1));
    const double mps = __shfl_sync(FULL, v, 4 * p + (kk >> 1));
    const double m0 = __shfl_sync(FULL, mi[0], 4 * kk + q);
    const double m1 = __shfl_sync(FULL, mi[1], 4 * kk + q);
    const double e0 = __shfl_sync(FULL, ev[0], 4 * kk + q);
    const double e1 = __shfl_sync(FULL, ev[1], 4 * kk + q);
    const double f = (p > kk) ? mps * rcp64(piv) : 0.0;
    mi[0] = fma(-f, m0, mi[0]);
    mi[1] = fma(-f, m1, mi[1]);
    ev[0] = fma(-f, e0, ev[0]);
    ev[1] = fma(-f, e1, ev[1]);
  }
  const double dsel0 = (p & 1) ? mi[1] : mi[0];
  const double rd_ = rcp64(__shfl_sync(FULL, dsel0, 4 * p + (p >> 1)));
  rd0 = __shfl_sync(FULL, rd_, 8 * q);
  rd1 = __shfl_sync(FULL, rd_, 8 * q + 4);
}

}  // namespace blk
}  // namespace rgb
