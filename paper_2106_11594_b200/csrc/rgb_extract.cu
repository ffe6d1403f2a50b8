// rgb_extract.cu -- read-side kernels: projection, pseudoinverse, covariance.
//
// project    : RecursiveSolver.project + is_dependent (solver.py:210-229)
// pinv       : A+ = C~^T P^-1 B^T, the closed form the
//              reference pins against its incremental tracker
//              (test_tracking.py:87-98); replaces the Theta(mn)-per-row column
//              update of PseudoinverseTracker (tracking.py:76-85) by one
//              m x r x n contraction at read time.
// covariance : V = A+ A+^T = C~^T P^-1 C~ (test_tracking.py:188-198); replaces
//              CovarianceTracker's per-row O(m^2) update (tracking.py:103-119).
#include "rgb_common.cuh"

namespace rgb {

constexpr int PJ_NT = 128;

template <typename REAL>
__global__ void __launch_bounds__(PJ_NT) project_kernel(rgb_config cfg, rgb_state st,
                                                        const REAL* __restrict__ rows, REAL* coords,
                                                        REAL* rejection, REAL* rej_sq_out,
                                                        uint8_t* dependent) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int m = cfg.m, rc = cfg.r_cap;
  REAL* a_s = reinterpret_cast<REAL*>(smem_raw);
  REAL* gam = a_s + m;
  REAL* red = gam + rc;  // 2 x 4 warps
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t b = blockIdx.x;
  const REAL* C = reinterpret_cast<const REAL*>(st.basis) + b * (int64_t)rc * m;
  const REAL* D = reinterpret_cast<const REAL*>(st.dual) + b * (int64_t)rc * m;
  const int r = st.rank[b];
  const REAL* a = rows + b * m;
  for (int j = tid; j < m; j += PJ_NT) a_s[j] = a[j];
  __syncthreads();
  for (int i = w; i < r; i += PJ_NT / 32) {
    REAL s = 0;
    for (int j = lane; j < m; j += 32) s = fma(D[(int64_t)i * m + j], a_s[j], s);
    s = warp_sum(s);
    if (lane == 0) gam[i] = s;
  }
  __syncthreads();
  REAL pr = 0, pa = 0;
  for (int j = tid; j < m; j += PJ_NT) {
    REAL s = 0;
    for (int i = 0; i < r; ++i) s = fma(gam[i], C[(int64_t)i * m + j], s);
    REAL v = a_s[j] - s;
    if (rejection) rejection[b * m + j] = v;
    pr = fma(v, v, pr);
    pa = fma(a_s[j], a_s[j], pa);
  }
  pr = warp_sum(pr);
  pa = warp_sum(pa);
  if (lane == 0) { red[w] = pr; red[4 + w] = pa; }
  if (coords)
    for (int i = tid; i < rc; i += PJ_NT) coords[b * rc + i] = i < r ? gam[i] : (REAL)0;
  __syncthreads();
  if (tid == 0) {
    REAL rs = red[0] + red[1] + red[2] + red[3];
    REAL as = red[4] + red[5] + red[6] + red[7];
    if (rej_sq_out) rej_sq_out[b] = rs;
    if (dependent) dependent[b] = is_dependent<REAL>(rs, as, eps_sq<REAL>(cfg, r)) ? 1 : 0;
  }
}

// out[b][j][t] = sum_i D[i][j] * w[i][t],  w[i][t] = sum_l P[i][l] * F(t, l)
// F(t, l) = coords[b][t][l] (pinv) or D[l][t] (covariance).  Lanes run over t
// (coalesced stores), warps over j; w for 32 columns t is staged in smem.
template <typename REAL, bool COV>
__global__ void __launch_bounds__(256) dual_gram_kernel(rgb_config cfg, rgb_state st,
                                                        const REAL* __restrict__ coords, int64_t n,
                                                        REAL* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  REAL* wsm = reinterpret_cast<REAL*>(smem_raw);  // [r][32]
  const int m = cfg.m, rc = cfg.r_cap;
  const int64_t b = blockIdx.y;
  const int64_t t0 = (int64_t)blockIdx.x * 32;
  const REAL* D = reinterpret_cast<const REAL*>(st.dual) + b * (int64_t)rc * m;
  const REAL* P = reinterpret_cast<const REAL*>(st.gram_inv) + b * (int64_t)rc * rc;
  const int r = st.rank[b];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int idx = tid; idx < r * 32; idx += 256) {
    int i = idx >> 5, tl = idx & 31;
    int64_t t = t0 + tl;
    REAL s = 0;
    if (t < n) {
      for (int l = 0; l < r; ++l) {
        REAL f = COV ? D[(int64_t)l * m + t] : coords[(b * n + t) * rc + l];
        s = fma(P[(int64_t)i * rc + l], f, s);
      }
    }
    wsm[i * 32 + tl] = s;
  }
  __syncthreads();
  const int64_t t = t0 + lane;
  if (t >= n) return;
  for (int j = w; j < m; j += 8) {
    REAL s = 0;
    for (int i = 0; i < r; ++i) s = fma(D[(int64_t)i * m + j], wsm[i * 32 + lane], s);
    out[(b * m + j) * n + t] = s;
  }
}

int launch_project(const rgb_config& cfg, const rgb_state& st, const void* rows, void* coords,
                   void* rejection, void* rej_sq, uint8_t* dependent, cudaStream_t stream) {
  size_t es = cfg.dtype == RGB_F32 ? 4 : 8;
  size_t smem = ((size_t)cfg.m + cfg.r_cap + 8) * es;
  if (smem > 200 * 1024) return RGB_E_UNSUPPORTED;
  dim3 grid((unsigned)cfg.num_streams);
  if (cfg.dtype == RGB_F64) {
    auto k = project_kernel<double>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<grid, PJ_NT, smem, stream>>>(cfg, st, (const double*)rows, (double*)coords, (double*)rejection,
                                     (double*)rej_sq, dependent);
  } else {
    auto k = project_kernel<float>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<grid, PJ_NT, smem, stream>>>(cfg, st, (const float*)rows, (float*)coords, (float*)rejection,
                                     (float*)rej_sq, dependent);
  }
  return cudaGetLastError() == cudaSuccess ? RGB_OK : RGB_E_CUDA;
}

template <bool COV>
static int launch_dual_gram(const rgb_config& cfg, const rgb_state& st, const void* coords, int64_t n,
                            void* out, cudaStream_t stream) {
  size_t es = cfg.dtype == RGB_F32 ? 4 : 8;
  size_t smem = (size_t)cfg.r_cap * 32 * es;
  if (smem > 200 * 1024) return RGB_E_UNSUPPORTED;
  if (cfg.num_streams > 65535) return RGB_E_UNSUPPORTED;
  dim3 grid((unsigned)((n + 31) / 32), (unsigned)cfg.num_streams);
  if (cfg.dtype == RGB_F64) {
    auto k = dual_gram_kernel<double, COV>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<grid, 256, smem, stream>>>(cfg, st, (const double*)coords, n, (double*)out);
  } else {
    auto k = dual_gram_kernel<float, COV>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<grid, 256, smem, stream>>>(cfg, st, (const float*)coords, n, (float*)out);
  }
  return cudaGetLastError() == cudaSuccess ? RGB_OK : RGB_E_CUDA;
}

int launch_pinv(const rgb_config& cfg, const rgb_state& st, const void* coords, int64_t n, void* out,
                cudaStream_t stream) {
  return launch_dual_gram<false>(cfg, st, coords, n, out, stream);
}

int launch_covariance(const rgb_config& cfg, const rgb_state& st, void* out, cudaStream_t stream) {
  return launch_dual_gram<true>(cfg, st, nullptr, cfg.m, out, stream);
}

}  // namespace rgb
