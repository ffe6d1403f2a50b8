// rgb_generic.cu -- shape-generic rank-Greville update kernel.
//
// One CTA per stream (grid-stride over streams), NT threads.  The factors
// live in the caller's global buffers (L2 resident for the single-stream
// configs), threads own strided columns j of C, C~, x; warps own rows i of
// C~ and P^-1 for the reductions over m and r.  This kernel covers every
// (m, r_cap, k, variant, dtype) the ABI accepts; the shapes the tensor-core
// kernels serve (rgb_blocked*.cu, rgb_cluster.cu, rgb_grid.cu) run there.
//
// Per row it restates RecursiveSolver.ingest (solver.py:276-319):
//   coords  = C~ a                       solver.py:286
//   rej     = a - C^T coords, |rej|^2    solver.py:287-291
//   test    rej^2 < eps^2 (1 + |a|^2)    solver.py:292-296
//   dependent:   z = P coords, zs = z/(1+coords.z), P -= z zs^T,
//                K = zs^T C~             solver.py:297-304
//   independent: K = rej/|rej|^2 and _grow (solver.py:368-397)
//   x += K (y - a.x)                     solver.py:303-304, 316-318
#include "rgb_common.cuh"

namespace rgb {

constexpr int GEN_NT = 256;

// phase timing (debug builds only: -DRGB_GEN_PROBE): %globaltimer ns summed per
// phase by thread 0 of CTA 0, read back with rgb_generic_probe()
#ifdef RGB_GEN_PROBE
__device__ unsigned long long g_genprobe[16];
__device__ __forceinline__ unsigned long long gen_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define GENPROBE(i)                                             \
  do {                                                          \
    if (threadIdx.x == 0 && blockIdx.x == 0) {                  \
      const unsigned long long now_ = gen_now();                \
      g_genprobe[i] += now_ - probe_t;                          \
      probe_t = now_;                                           \
    }                                                           \
  } while (0)
#else
#define GENPROBE(i) \
  do {              \
  } while (0)
#endif
constexpr int GEN_NW = GEN_NT / 32;
constexpr int GEN_MAX_K = 64;

// Reduce `nv` per-thread partial sums held in smem-free fashion: each warp
// reduces its lanes, lane 0 parks the result, then threads v < nv add the
// per-warp partials.  `part(v)` returns this thread's partial for value v.
template <typename REAL, typename F>
__device__ __forceinline__ void block_reduce(int nv, REAL* red, REAL* out, F part) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int v = 0; v < nv; ++v) {
    REAL s = warp_sum(part(v));
    if (lane == 0) red[w * (GEN_MAX_K + 2) + v] = s;
  }
  __syncthreads();
  for (int v = threadIdx.x; v < nv; v += GEN_NT) {
    REAL s = 0;
    for (int q = 0; q < GEN_NW; ++q) s += red[q * (GEN_MAX_K + 2) + v];
    out[v] = s;
  }
  __syncthreads();
}

__device__ __forceinline__ void cp_async_n(void* smem, const void* gmem, int bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  if (bytes == 16) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
  else if (bytes == 8) asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
  else asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem));
}

// Asynchronous global -> shared copy of n contiguous elements (16-byte pieces
// when both ends are 16-byte aligned); the caller commits and waits.
template <typename REAL>
__device__ __forceinline__ void stage_async(REAL* dst, const REAL* src, int64_t n, int tid) {
  constexpr int V = 16 / sizeof(REAL);
  if ((((uintptr_t)dst | (uintptr_t)src) & 15) == 0) {
    const int64_t nv = n / V;
    for (int64_t e = tid; e < nv; e += GEN_NT) cp_async_n(dst + e * V, src + e * V, 16);
    for (int64_t e = nv * V + tid; e < n; e += GEN_NT) cp_async_n(dst + e, src + e, sizeof(REAL));
  } else {
    for (int64_t e = tid; e < n; e += GEN_NT) cp_async_n(dst + e, src + e, sizeof(REAL));
  }
}

// Row pipe (rgb_rowpipe.cu): the counters, then the sequence word, into the
// caller's mapped host block; a barrier plus one system-scope release order
// every thread's report writes before the sequence word the host spins on.
__device__ __forceinline__ void publish_row_report(unsigned char* mirror, unsigned long long* dseq, int64_t nobs,
                                                   int r, int status, int tid) {
  __syncthreads();  // every thread's report writes happen before thread 0's release below
  if (tid == 0) {
    *reinterpret_cast<volatile int64_t*>(mirror + RGB_ROWPIPE_OFF_NOBS) = nobs;
    *reinterpret_cast<volatile int32_t*>(mirror + RGB_ROWPIPE_OFF_RANK) = r;
    *reinterpret_cast<volatile int32_t*>(mirror + RGB_ROWPIPE_OFF_STATUS) = status;
    const unsigned long long sq = *dseq + 1;
    *dseq = sq;
    // one system-scope release (cumulative over the barrier): the report and
    // the counters are visible to the host before the sequence word
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(mirror + RGB_ROWPIPE_OFF_SEQ), "l"(sq) : "memory");
  }
}

// TI: input element type (REAL, or float widened exactly into a double state)
template <typename REAL, typename TI>
__global__ void __launch_bounds__(GEN_NT) generic_ingest_kernel(
    rgb_config cfg, rgb_state st, const TI* __restrict__ rows, int64_t rows_stride,
    const TI* __restrict__ targets, int64_t tg_stride, int64_t T, rgb_logs logs, int cached,
    unsigned char* __restrict__ mirror, unsigned long long* __restrict__ dseq, REAL* __restrict__ hx) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int m = cfg.m, k = cfg.k, rc = cfg.r_cap, var = cfg.variant;
  REAL* a_s = reinterpret_cast<REAL*>(smem_raw);        // m
  REAL* rej_s = a_s + m;                                 // m
  REAL* gam = rej_s + m;                                 // rc
  REAL* z_s = gam + rc;                                  // rc
  REAL* zs_s = z_s + rc;                                 // rc
  REAL* y_s = zs_s + rc;                                 // k
  REAL* sums = y_s + GEN_MAX_K;                          // k + 2: rej_sq, row_sq, a.x_c
  REAL* red = sums + GEN_MAX_K + 2;                      // GEN_NW x (GEN_MAX_K + 2)
  REAL* scal = red + GEN_NW * (GEN_MAX_K + 2);           // denom etc.
  REAL* cache = scal + 8;  // cached: the stream's C, C~, P^-1, x (generic_cache_elems)
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
#ifdef RGB_GEN_PROBE
  unsigned long long probe_t = gen_now();
  if (tid == 0 && blockIdx.x == 0) g_genprobe[15] += 1;
#endif

  for (int64_t b = blockIdx.x; b < cfg.num_streams; b += gridDim.x) {
    REAL* Cg = reinterpret_cast<REAL*>(st.basis) + b * (int64_t)rc * m;
    REAL* Dg = (var == RGB_ORTHONORMAL) ? Cg : reinterpret_cast<REAL*>(st.dual) + b * (int64_t)rc * m;
    REAL* Pg = reinterpret_cast<REAL*>(st.gram_inv) + b * (int64_t)rc * rc;
    REAL* Xg = reinterpret_cast<REAL*>(st.x) + b * (int64_t)k * m;
    const TI* R = rows + b * rows_stride;
    const TI* Y = targets + b * tg_stride;
    int r = st.rank[b];
    int status = st.status[b];
    int64_t nobs = st.nobs[b];
    if (status) {  // frozen: nothing to fold (a row pipe still publishes its counters)
      if (mirror) publish_row_report(mirror, dseq, nobs, r, status, tid);
      continue;
    }
    const int r0 = r;
    REAL *C = Cg, *D = Dg, *P = Pg, *X = Xg;
    if (cached) {
      // a state that fits in shared memory is read once, with every load in
      // flight, instead of one dependent L2 round trip per step of every row
      // (a one-row update() is a chain of such steps)
      C = cache;
      D = (var == RGB_ORTHONORMAL) ? C : C + (size_t)rc * m;
      P = C + (size_t)(var == RGB_ORTHONORMAL ? 1 : 2) * rc * m;
      X = P + (size_t)rc * rc;
      // every copy in flight at once (cp.async), one wait: a single L2 round
      // trip instead of one per unrolled batch of loads
      stage_async(C, Cg, (int64_t)r0 * m, tid);
      if (var != RGB_ORTHONORMAL) stage_async(D, Dg, (int64_t)r0 * m, tid);
      for (int e = tid; e < r0 * r0; e += GEN_NT) {
        const int i = e / r0, l = e - i * r0;
        cp_async_n(P + (size_t)i * rc + l, Pg + (size_t)i * rc + l, sizeof(REAL));
      }
      stage_async(X, Xg, (int64_t)k * m, tid);
      if constexpr (sizeof(TI) == sizeof(REAL)) {
        // the first row rides with the state: its latency (an L2 or, for a row
        // pipe, a host-memory round trip) overlaps the state's
        if (T > 0) {
          for (int j = tid; j < m; j += GEN_NT) cp_async_n(a_s + j, R + j, sizeof(REAL));
          for (int c = tid; c < k; c += GEN_NT) cp_async_n(y_s + c, Y + c, sizeof(REAL));
        }
      }
      asm volatile("cp.async.commit_group;\n" ::);
      asm volatile("cp.async.wait_group 0;\n" ::);
      __syncthreads();
    }
    GENPROBE(0);
    for (int64_t t = 0; t < T; ++t) {
      if (!(cached && t == 0 && sizeof(TI) == sizeof(REAL))) {
        const TI* a = R + t * m;
        for (int j = tid; j < m; j += GEN_NT) a_s[j] = (REAL)a[j];
        for (int c = tid; c < k; c += GEN_NT) y_s[c] = (REAL)Y[t * k + c];
        __syncthreads();
      }
      GENPROBE(1);
      // coords = C~ a (solver.py:286): warp per dual row, lanes over columns
      for (int i = w; i < r; i += GEN_NW) {
        const REAL* d = D + (int64_t)i * m;
        REAL s = 0;
        for (int j = lane; j < m; j += 32) s = fma(d[j], a_s[j], s);
        s = warp_sum(s);
        if (lane == 0) gam[i] = s;
      }
      __syncthreads();
      GENPROBE(2);
      // rej = a - C^T coords (solver.py:287-288), kept for the independent branch
      for (int j = tid; j < m; j += GEN_NT) {
        REAL s = 0;
        for (int i = 0; i < r; ++i) s = fma(gam[i], C[(int64_t)i * m + j], s);
        rej_s[j] = a_s[j] - s;
      }
      __syncthreads();
      // |rej|^2, |a|^2 and the k a-priori dot products a.x_c in one reduction
      block_reduce<REAL>(2 + k, red, sums, [&](int v) {
        REAL s = 0;
        if (v == 0) {
          for (int j = tid; j < m; j += GEN_NT) s = fma(rej_s[j], rej_s[j], s);
        } else if (v == 1) {
          for (int j = tid; j < m; j += GEN_NT) s = fma(a_s[j], a_s[j], s);
        } else {
          const REAL* xc = X + (int64_t)(v - 2) * m;
          for (int j = tid; j < m; j += GEN_NT) s = fma(a_s[j], xc[j], s);
        }
        return s;
      });
      GENPROBE(3);
      const REAL rej_sq = sums[0], row_sq = sums[1];
      bool bad = !isfinite(row_sq);
      for (int c = 0; c < k; ++c) bad |= !isfinite(y_s[c]);
      if (bad) { status |= RGB_ST_NONFINITE; break; }
      const bool dep = is_dependent<REAL>(rej_sq, row_sq, eps_sq<REAL>(cfg, r));
      if (!dep && r >= rc) { status |= RGB_ST_RANK_CAP; break; }
      if (logs.branch && tid == 0) logs.branch[b * T + t] = dep ? 0 : 1;
      if (logs.resid)
        for (int c = tid; c < k; c += GEN_NT)
          reinterpret_cast<REAL*>(logs.resid)[(b * T + t) * k + c] = y_s[c] - sums[2 + c];
      // z = P coords and denom = 1 + coords.z: dependent rows, and independent
      // rows of the orthogonal/orthonormal variants (solver.py:298-299, 307-310)
      const bool need_z = r > 0 && (dep || var != RGB_GENERAL);
      if (need_z) {
        for (int i = w; i < r; i += GEN_NW) {
          const REAL* p = P + (int64_t)i * rc;
          REAL s = 0;
          for (int l = lane; l < r; l += 32) s = fma(p[l], gam[l], s);
          s = warp_sum(s);
          if (lane == 0) z_s[i] = s;
        }
        __syncthreads();
        if (w == 0) {
          REAL s = 0;
          for (int i = lane; i < r; i += 32) s = fma(gam[i], z_s[i], s);
          s = warp_sum(s);
          if (lane == 0) scal[0] = (REAL)1 + s;
        }
        __syncthreads();
      }
      GENPROBE(4);
      // rescaling of the stored rejection (orthogonal / orthonormal, solver.py:354-366, 383)
      REAL alpha = 1, last = 1;
      if (!dep && var != RGB_GENERAL) {
        REAL resc;
        if (var == RGB_ORTHONORMAL) resc = (REAL)1 / sqrt(rej_sq);          // solver.py:359-361
        else resc = (REAL)cfg.alpha;                                          // solver.py:362-366
        if (resc == (REAL)0) { status |= RGB_ST_BAD_ALPHA; break; }
        last = (REAL)1 / resc;    // coords_row[r], solver.py:354
        alpha = (REAL)1 / last;   // solver.py:383
      }
      if (logs.coords) {  // coords_row of _UpdateStep (solver.py:331, 344-355)
        REAL* cl = reinterpret_cast<REAL*>(logs.coords) + (b * T + t) * rc;
        for (int i = tid; i < rc; i += GEN_NT) {
          REAL v = i < r ? gam[i] : (REAL)0;
          if (!dep && var == RGB_GENERAL) v = (i == r) ? (REAL)1 : (REAL)0;
          if (!dep && var != RGB_GENERAL && i == r) v = last;
          cl[i] = v;
        }
      }
      if (dep) {
        if (r > 0) {
          const REAL denom = scal[0];
          for (int i = tid; i < r; i += GEN_NT) zs_s[i] = z_s[i] / denom;
          __syncthreads();
          for (int idx = tid; idx < r * r; idx += GEN_NT) {
            int i = idx / r, l = idx - i * r;
            P[(int64_t)i * rc + l] -= z_s[i] * zs_s[l];
          }
          for (int j = tid; j < m; j += GEN_NT) {
            REAL g = 0;
            for (int i = 0; i < r; ++i) g = fma(zs_s[i], D[(int64_t)i * m + j], g);
            for (int c = 0; c < k; ++c) X[(int64_t)c * m + j] += g * (y_s[c] - sums[2 + c]);
            if (logs.gain && t == T - 1) reinterpret_cast<REAL*>(logs.gain)[b * m + j] = g;
          }
        } else if (logs.gain && t == T - 1) {
          for (int j = tid; j < m; j += GEN_NT) reinterpret_cast<REAL*>(logs.gain)[b * m + j] = 0;
        }
      } else {
        // independent branch: gain = rej / |rej|^2 (solver.py:336) and _grow
        for (int j = tid; j < m; j += GEN_NT) {
          const REAL g = rej_s[j] / rej_sq;
          if (var == RGB_GENERAL) {
            for (int i = 0; i < r; ++i) D[(int64_t)i * m + j] -= gam[i] * g;   // solver.py:378
            D[(int64_t)r * m + j] = g;                                          // solver.py:379
            C[(int64_t)r * m + j] = a_s[j];                                     // solver.py:376
          } else {
            C[(int64_t)r * m + j] = alpha * rej_s[j];                           // solver.py:384
            if (var == RGB_ORTHOGONAL) D[(int64_t)r * m + j] = rej_s[j] / (alpha * rej_sq);
          }
          for (int c = 0; c < k; ++c) X[(int64_t)c * m + j] += g * (y_s[c] - sums[2 + c]);
          if (logs.gain && t == T - 1) reinterpret_cast<REAL*>(logs.gain)[b * m + j] = g;
        }
        for (int i = tid; i <= r; i += GEN_NT) {
          REAL edge = 0, corner = 1;
          if (var != RGB_GENERAL) {
            if (i < r) edge = -(alpha * z_s[i]);
            corner = alpha * alpha * (r > 0 ? scal[0] : (REAL)1);
          }
          if (i < r) {
            P[(int64_t)i * rc + r] = edge;
            P[(int64_t)r * rc + i] = edge;
          } else {
            P[(int64_t)r * rc + r] = corner;
          }
        }
        r += 1;
      }
      nobs += 1;
      __syncthreads();
      GENPROBE(5);
    }
    __syncthreads();
    if (cached) {  // write back what the rows changed (rows >= r0 are new; C~ and P^-1 change in place)
      for (int e = tid; e < r * m; e += GEN_NT) {
        if (e >= r0 * m) Cg[e] = C[e];
        if (var != RGB_ORTHONORMAL) Dg[e] = D[e];
      }
      for (int e = tid; e < r * r; e += GEN_NT) Pg[(e / r) * rc + e % r] = P[(e / r) * rc + e % r];
      for (int e = tid; e < k * m; e += GEN_NT) Xg[e] = X[e];
      __syncthreads();
    }
    if (tid == 0) {
      st.rank[b] = r;
      st.nobs[b] = nobs;
      st.status[b] = status;
    }
    GENPROBE(6);
    if (hx)  // row pipe: the solution (first right-hand side) into the caller's host mirror
      for (int j = tid; j < m; j += GEN_NT) hx[j] = X[j];
    if (mirror) publish_row_report(mirror, dseq, nobs, r, status, tid);
    GENPROBE(7);
  }
}

#ifdef RGB_GEN_PROBE
}  // namespace rgb
extern "C" int rgb_generic_probe(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, rgb::g_genprobe, sizeof(rgb::g_genprobe));
  if (reset) {
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(rgb::g_genprobe, z, sizeof(z));
  }
  return 0;
}
namespace rgb {
#endif

size_t generic_smem_bytes(const rgb_config& cfg) {
  size_t s = cfg.dtype == RGB_F32 ? 4 : 8;
  size_t n = 2 * (size_t)cfg.m + 3 * (size_t)cfg.r_cap + GEN_MAX_K + (GEN_MAX_K + 2) +
             GEN_NW * (GEN_MAX_K + 2) + 8;
  return n * s;
}

// elements of the shared-memory copy of one stream's state
static size_t generic_cache_elems(const rgb_config& cfg) {
  const size_t m = cfg.m, rc = cfg.r_cap, k = cfg.k;
  return (cfg.variant == RGB_ORTHONORMAL ? 1 : 2) * rc * m + rc * rc + k * m;
}

// the state is cached in shared memory when it fits in 96 KB (two CTAs per SM
// stay resident for multi-stream calls)
static constexpr size_t GEN_CACHE_MAX = 96 * 1024;

int launch_generic(const rgb_config& cfg, rgb_state& st, const void* rows, int64_t rows_stride,
                   const void* targets, int64_t tg_stride, int64_t T, const rgb_logs& logs,
                   cudaStream_t stream, int num_sms, bool f32in, unsigned char* mirror,
                   unsigned long long* dseq, void* hx) {
  if (cfg.k > GEN_MAX_K) return RGB_E_UNSUPPORTED;
  size_t smem = generic_smem_bytes(cfg);
  if (smem > 200 * 1024) return RGB_E_UNSUPPORTED;
  const size_t esz = cfg.dtype == RGB_F32 ? 4 : 8;
  const int cached = smem + esz * generic_cache_elems(cfg) <= GEN_CACHE_MAX ? 1 : 0;
  if (cached) smem += esz * generic_cache_elems(cfg);
  int64_t grid = cfg.num_streams < (int64_t)num_sms * 8 ? cfg.num_streams : (int64_t)num_sms * 8;
  if (grid < 1) return RGB_OK;
  if (cfg.dtype == RGB_F64 && f32in) {
    auto kern = generic_ingest_kernel<double, float>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<(unsigned)grid, GEN_NT, smem, stream>>>(cfg, st, (const float*)rows, rows_stride, (const float*)targets,
                                                   tg_stride, T, logs, cached, mirror, dseq, (double*)hx);
  } else if (cfg.dtype == RGB_F64) {
    auto kern = generic_ingest_kernel<double, double>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<(unsigned)grid, GEN_NT, smem, stream>>>(cfg, st, (const double*)rows, rows_stride, (const double*)targets,
                                                   tg_stride, T, logs, cached, mirror, dseq, (double*)hx);
  } else {
    auto kern = generic_ingest_kernel<float, float>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<(unsigned)grid, GEN_NT, smem, stream>>>(cfg, st, (const float*)rows, rows_stride, (const float*)targets,
                                                  tg_stride, T, logs, cached, mirror, dseq, (float*)hx);
  }
  return cudaGetLastError() == cudaSuccess ? RGB_OK : RGB_E_CUDA;
}

}  // namespace rgb
