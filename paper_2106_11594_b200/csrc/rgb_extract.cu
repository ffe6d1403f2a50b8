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
#include "rgb_mma.cuh"

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

// ---- fp64 batched tensor-core contraction for A+ and the covariance -----------
//
// out[b][mm][nn] = sum_{k < K_b} X[b][k][mm] * Y(b, k, nn),  K_b = rank[b],
// Y(b, k, nn) = Y[b][nn][k] (YKN false) or Y[b][k][nn] (YKN true).
// A+ = C~^T (P^-1 B^T) runs as two of these (rgb_pinv): V = P^-1 C~ (X = P^-1,
// Y = C~, r_cap x m), then out = V^T B^T (X = V, Y = the coords log B, m x n);
// the covariance C~^T P^-1 C~ is V^T C~ (Y = C~).  A CTA of 4 warps computes a
// 64 x 64 output tile on mma.sync.m8n8k4.f64 (DMMA), each warp 32 x 32 (4 x 4
// fragments); K streams through shared memory 16 at a time, double-buffered
// with cp.async, both operands stored k-major with a row pitch of 72 doubles
// (== 8 mod 16), so the A/B fragment reads are conflict-free.  Global loads are
// 16-byte and coalesced along the contiguous dimension of each operand
// (a coords row of B is r_cap contiguous values; rows of P and C~ are
// contiguous).  Rows of X / Y at or beyond K_b are zero-filled in shared
// memory, so stale values past the rank never enter the sum.
namespace ext {

constexpr int BM = 64, BN = 64, KC = 16, PIT = 72, NT = 128;

struct GemmArgs {
  const double* X;
  int64_t ldx, sx;
  const double* Y;
  int64_t ldy, sy;
  double* out;
  int64_t ldo, so;
  int64_t M, N;
  const int32_t* rank;
  int32_t k_cap;  // K_b = min(rank[b], k_cap)
};

__device__ __forceinline__ void cp16(double* s, const double* g, bool ok) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(g), "r"(ok ? 16 : 0));
}
__device__ __forceinline__ void cp8(double* s, const double* g, bool ok) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(g), "r"(ok ? 8 : 0));
}

// stage a KC x 64 k-major tile: rows k of a row-major [k][col] operand (ld), cols c0..c0+63
template <bool VEC>
__device__ __forceinline__ void stage_kmajor(double* sm, const double* g, int64_t ld, int k0, int K, int64_t c0,
                                             int64_t ncol, int tid) {
  if (VEC) {  // 16-byte copies
    const int kk = tid >> 3, c = (tid & 7) * 8;  // 16 rows x 8 threads x 8 values
#pragma unroll
    for (int q = 0; q < 8; q += 2) {
      const int64_t col = c0 + c + q;
      const bool ok = (k0 + kk < K) && (col + 1 < ncol);
      if (ok || !((k0 + kk < K) && col < ncol)) {
        cp16(sm + kk * PIT + c + q, ok ? g + (int64_t)(k0 + kk) * ld + col : g, ok);
      } else {  // the last column of an odd-width operand
        cp8(sm + kk * PIT + c + q, g + (int64_t)(k0 + kk) * ld + col, true);
        sm[kk * PIT + c + q + 1] = 0.0;
      }
    }
  } else {
    for (int idx = tid; idx < KC * BM; idx += NT) {
      const int kk = idx >> 6, c = idx & 63;
      const int64_t col = c0 + c;
      const bool ok = (k0 + kk < K) && col < ncol;
      cp8(sm + kk * PIT + c, ok ? g + (int64_t)(k0 + kk) * ld + col : g, ok);
    }
  }
}

// stage a KC x 64 k-major tile from an operand stored [col][k] (ld): 64 rows of
// KC contiguous values; written transposed into shared memory
__device__ __forceinline__ void stage_colmajor(double* sm, const double* g, int64_t ld, int k0, int K, int64_t c0,
                                               int64_t ncol, int tid) {
  for (int idx = tid; idx < KC * BN; idx += NT) {
    const int c = idx >> 4, kk = idx & 15;  // 16 consecutive lanes read one contiguous 128-byte run
    const int64_t col = c0 + c;
    const bool ok = (k0 + kk < K) && col < ncol;
    cp8(sm + kk * PIT + c, ok ? g + col * ld + k0 + kk : g, ok);
  }
}

template <bool YKN, bool XVEC, bool YVEC>
__global__ void __launch_bounds__(NT) xt_gemm_kernel(GemmArgs a) {
  __shared__ __align__(16) double Xs[2][KC * PIT];
  __shared__ __align__(16) double Ys[2][KC * PIT];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t b = blockIdx.y;
  const int64_t tiles_n = (a.N + BN - 1) / BN;
  const int64_t m0 = (blockIdx.x / tiles_n) * BM, n0 = (blockIdx.x % tiles_n) * BN;
  int K = a.rank[b];
  if (K > a.k_cap) K = a.k_cap;
  const double* X = a.X + b * a.sx;
  const double* Y = a.Y + b * a.sy;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int wm = (w >> 1) * 32, wn = (w & 1) * 32;
  const int fr = lane >> 2, fk = lane & 3;
  auto stage = [&](int buf, int k0) {
    stage_kmajor<XVEC>(Xs[buf], X, a.ldx, k0, K, m0, a.M, tid);
    if (YKN) stage_kmajor<YVEC>(Ys[buf], Y, a.ldy, k0, K, n0, a.N, tid);
    else stage_colmajor(Ys[buf], Y, a.ldy, k0, K, n0, a.N, tid);
    asm volatile("cp.async.commit_group;\n" ::);
  };
  const int nk = (K + KC - 1) / KC;
  if (nk > 0) stage(0, 0);
  for (int kc = 0; kc < nk; ++kc) {
    if (kc + 1 < nk) {
      stage((kc + 1) & 1, (kc + 1) * KC);
      asm volatile("cp.async.wait_group 1;\n" ::);
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::);
    }
    __syncthreads();
    const double* xs = Xs[kc & 1];
    const double* ys = Ys[kc & 1];
#pragma unroll
    for (int ks = 0; ks < KC; ks += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = xs[(ks + fk) * PIT + wm + 8 * i + fr];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = ys[(ks + fk) * PIT + wn + 8 * j + fr];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) blk::mma(acc[i][j], af[i], bf[j]);
    }
    __syncthreads();
  }
  double* out = a.out + b * a.so;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t row = m0 + wm + 8 * i + fr;
    if (row >= a.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t col = n0 + wn + 8 * j + 2 * fk;
      double* o = out + row * a.ldo + col;
      if (col + 1 < a.N && ((a.ldo | col) & 1) == 0) {
        *reinterpret_cast<double2*>(o) = make_double2(acc[i][j][0], acc[i][j][1]);
      } else {
        if (col < a.N) o[0] = acc[i][j][0];
        if (col + 1 < a.N) o[1] = acc[i][j][1];
      }
    }
  }
}

// 16-byte staging needs even leading dimensions and an even base address
inline bool vec_ok(const double* p, int64_t ld, int64_t stride) {
  return ((reinterpret_cast<uintptr_t>(p) & 15) == 0) && (ld % 2 == 0) && (stride % 2 == 0);
}

template <bool YKN>
int launch_xt(const GemmArgs& a, int64_t B, cudaStream_t stream) {
  const int64_t tiles = ((a.M + BM - 1) / BM) * ((a.N + BN - 1) / BN);
  if (tiles > 0x7fffffff) return RGB_E_UNSUPPORTED;
  const bool xv = vec_ok(a.X, a.ldx, a.sx), yv = YKN && vec_ok(a.Y, a.ldy, a.sy);
  for (int64_t b0 = 0; b0 < B; b0 += 65535) {  // grid.y limit: launch stream chunks
    const int64_t nb = B - b0 < 65535 ? B - b0 : 65535;
    GemmArgs c = a;
    c.X += b0 * a.sx;
    c.Y += b0 * a.sy;
    c.out += b0 * a.so;
    c.rank += b0;
    dim3 grid((unsigned)tiles, (unsigned)nb);
    if (xv && yv) xt_gemm_kernel<YKN, true, true><<<grid, NT, 0, stream>>>(c);
    else if (xv) xt_gemm_kernel<YKN, true, false><<<grid, NT, 0, stream>>>(c);
    else xt_gemm_kernel<YKN, false, false><<<grid, NT, 0, stream>>>(c);
  }
  return cudaGetLastError() == cudaSuccess ? RGB_OK : RGB_E_CUDA;
}

}  // namespace ext

cudaMemPool_t workspace_pool();  // rgb_grid.cu

// fp64: V = P^-1 C~ into a workspace from the library pool (per chunk of
// streams, so the workspace stays under 256 MB), then out = V^T F with F the
// coords log (pinv) or C~ (covariance).
static int extract_f64(const rgb_config& cfg, const rgb_state& st, const double* coords, int64_t n, double* out,
                       bool cov, cudaStream_t stream) {
  const int64_t m = cfg.m, rc = cfg.r_cap, B = cfg.num_streams;
  const int64_t per = rc * m;  // V per stream
  int64_t chunk = (int64_t)(256ll << 20) / (8 * per);
  if (chunk < 1) chunk = 1;
  if (chunk > B) chunk = B;
  cudaMemPool_t pool = workspace_pool();
  void* ws = nullptr;
  if (!pool || cudaMallocFromPoolAsync(&ws, (size_t)(chunk * per * 8), pool, stream) != cudaSuccess) return RGB_E_CUDA;
  double* V = static_cast<double*>(ws);
  const double* P = static_cast<const double*>(st.gram_inv);
  const double* D = static_cast<const double*>(st.dual);
  int rc_ = RGB_OK;
  for (int64_t b0 = 0; b0 < B && rc_ == RGB_OK; b0 += chunk) {
    const int64_t nb = B - b0 < chunk ? B - b0 : chunk;
    // V[i][j] = sum_l P[l][i] C~[l][j]   (P^-1 is symmetric)
    ext::GemmArgs v{P + b0 * rc * rc, rc, rc * rc, D + b0 * per, m, per, V, m, per, rc, m, st.rank + b0, (int32_t)rc};
    rc_ = ext::launch_xt<true>(v, nb, stream);
    if (rc_ != RGB_OK) break;
    if (cov) {  // out[j][t] = sum_i V[i][j] C~[i][t]
      ext::GemmArgs o{V, m, per, D + b0 * per, m, per, out + b0 * m * m, m, m * m, m, m, st.rank + b0, (int32_t)rc};
      rc_ = ext::launch_xt<true>(o, nb, stream);
    } else {    // out[j][t] = sum_i V[i][j] B[t][i]
      ext::GemmArgs o{V, m, per, coords + b0 * n * rc, rc, n * rc, out + b0 * m * n, n, m * n, m, n, st.rank + b0,
                      (int32_t)rc};
      rc_ = ext::launch_xt<false>(o, nb, stream);
    }
  }
  cudaFreeAsync(ws, stream);
  return rc_;
}

// fp32 state (generic-kernel streams): CUDA cores.
// out[b][j][t] = sum_i D[i][j] * w[i][t],  w[i][t] = sum_l P[i][l] * F(t, l)
// F(t, l) = coords[b][t][l] (pinv) or D[l][t] (covariance).  Lanes run over t
// (coalesced stores), warps over j; w for 32 columns t is staged in smem.
template <typename REAL, bool COV>
__global__ void __launch_bounds__(256) dual_gram_kernel(rgb_config cfg, rgb_state st,
                                                        const REAL* __restrict__ coords, int64_t n,
                                                        REAL* __restrict__ out, int64_t b_off) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  REAL* wsm = reinterpret_cast<REAL*>(smem_raw);  // [r][32]
  const int m = cfg.m, rc = cfg.r_cap;
  const int64_t b = b_off + blockIdx.y;
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
  if (cfg.dtype == RGB_F64)
    return extract_f64(cfg, st, (const double*)coords, n, (double*)out, COV, stream);
  const size_t smem = (size_t)cfg.r_cap * 32 * sizeof(float);
  if (smem > 200 * 1024) return RGB_E_UNSUPPORTED;
  auto k = dual_gram_kernel<float, COV>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int64_t b0 = 0; b0 < cfg.num_streams; b0 += 65535) {  // grid.y limit
    const int64_t nb = cfg.num_streams - b0 < 65535 ? cfg.num_streams - b0 : 65535;
    dim3 grid((unsigned)((n + 31) / 32), (unsigned)nb);
    k<<<grid, 256, smem, stream>>>(cfg, st, (const float*)coords, n, (float*)out, b0);
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
