// rgb_rowpipe.cu -- low-latency one-row fold for the drop-in per-row API.
//
// RecursiveSolver.update (solver.py:231-250) is one row per call, so its cost is
// latency, not throughput.  A row pipe is a CUDA graph captured once per solver
// layout: row1_kernel (or, for states too large for shared memory, the
// shape-generic kernel) reads the row and its targets straight from
// a pinned, device-mapped host block (no copy node) and writes the report
// (branch, a-priori residuals, gain) back into it, then mirrors the counters
// (nobs, rank, status) and bumps a sequence word behind system-scope fences.  rgb_rowpipe_run launches the graph on the caller's
// stream and spins on the sequence word instead of synchronising the stream,
// so a call costs one graph launch plus the kernel's own latency.
#include <immintrin.h>
#include <sched.h>
#include <stdlib.h>
#include <string.h>

#include <chrono>

#include "rgb_common.cuh"

namespace rgb {
int launch_generic(const rgb_config& cfg, rgb_state& st, const void* rows, int64_t rows_stride,
                   const void* targets, int64_t tg_stride, int64_t T, const rgb_logs& logs,
                   cudaStream_t stream, int num_sms, bool f32in, unsigned char* mirror = nullptr,
                   unsigned long long* dseq = nullptr, void* hx = nullptr);


// The row pipe's kernel: one row of one stream, the shape-generic kernel's
// arithmetic in the same order (bit-identical results) with its phases merged
// for latency -- the state and the row are staged with one round of cp.async
// (the row's host-memory read overlaps the state's), the coords, |a|^2 and
// a.x partials share a phase, z = P^-1 coords runs beside the rejection, and
// the updated factors go straight to global memory: three barriers per row
// instead of about ten plus a write-back pass.
constexpr int R1_NT = 256, R1_NW = 8, R1_MK = 64;

__device__ __forceinline__ void r1_cp(void* smem, const void* gmem, int bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  if (bytes == 8) asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
  else asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem));
}

template <typename REAL>
__device__ __forceinline__ void r1_publish(unsigned char* mirror, unsigned long long* dseq, int64_t nobs, int r,
                                           int status, int tid) {
  __syncthreads();
  if (tid == 0) {
    *reinterpret_cast<volatile int64_t*>(mirror + RGB_ROWPIPE_OFF_NOBS) = nobs;
    *reinterpret_cast<volatile int32_t*>(mirror + RGB_ROWPIPE_OFF_RANK) = r;
    *reinterpret_cast<volatile int32_t*>(mirror + RGB_ROWPIPE_OFF_STATUS) = status;
    const unsigned long long sq = *dseq + 1;
    *dseq = sq;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(mirror + RGB_ROWPIPE_OFF_SEQ), "l"(sq) : "memory");
  }
}

// (Measured alternative: a plain launch carrying the row in a 3 KB kernel
// parameter instead of the graph plus the host-memory read: 17.5 vs 14.6 us
// per call at m = 128.)
template <typename REAL>
__global__ void __launch_bounds__(R1_NT) row1_kernel(rgb_config cfg, rgb_state st, const REAL* __restrict__ a_g,
                                                     const REAL* __restrict__ y_g, rgb_logs logs,
                                                     unsigned char* __restrict__ mirror,
                                                     unsigned long long* __restrict__ dseq, REAL* __restrict__ hx) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int m = cfg.m, k = cfg.k, rc = cfg.r_cap, var = cfg.variant;
  const bool onorm = var == RGB_ORTHONORMAL;
  REAL* a_s = reinterpret_cast<REAL*>(smem_raw);
  REAL* rej_s = a_s + m;
  REAL* gam = rej_s + m;
  REAL* z_s = gam + rc;
  REAL* y_s = z_s + rc;
  REAL* red = y_s + R1_MK;                     // [NW][MK + 2]
  REAL* Cg = reinterpret_cast<REAL*>(st.basis);
  REAL* Dg = onorm ? Cg : reinterpret_cast<REAL*>(st.dual);
  REAL* D = red + R1_NW * (R1_MK + 2);         // C~ rows < r
  REAL* C = onorm ? D : D + (size_t)rc * m;    // C rows < r
  REAL* P = C + (size_t)rc * m;                // P^-1 [r][r] at stride rc
  REAL* X = P + (size_t)rc * rc;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  REAL* Pg = reinterpret_cast<REAL*>(st.gram_inv);
  REAL* Xg = reinterpret_cast<REAL*>(st.x);
  int r = st.rank[0];
  int status = st.status[0];
  int64_t nobs = st.nobs[0];
  if (status) {
    r1_publish<REAL>(mirror, dseq, nobs, r, status, tid);
    return;
  }
  // ---- stage: the row and targets (host memory) first, then the state ------------
  for (int j = tid; j < m; j += R1_NT) r1_cp(a_s + j, a_g + j, sizeof(REAL));
  for (int c = tid; c < k; c += R1_NT) r1_cp(y_s + c, y_g + c, sizeof(REAL));
  for (int e = tid; e < r * m; e += R1_NT) r1_cp(D + e, Dg + e, sizeof(REAL));
  if (!onorm)
    for (int e = tid; e < r * m; e += R1_NT) r1_cp(C + e, Cg + e, sizeof(REAL));
  for (int e = tid; e < r * r; e += R1_NT) {
    const int i = e / r, l = e - i * r;
    r1_cp(P + (size_t)i * rc + l, Pg + (size_t)i * rc + l, sizeof(REAL));
  }
  for (int e = tid; e < k * m; e += R1_NT) r1_cp(X + e, Xg + e, sizeof(REAL));
  asm volatile("cp.async.commit_group;\n" ::);
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();
  // ---- A: coords (warp per dual row) and the |a|^2, a.x_c block partials ---------
  for (int i = w; i < r; i += R1_NW) {
    const REAL* d = D + (size_t)i * m;
    REAL s = 0;
    for (int j = lane; j < m; j += 32) s = fma(d[j], a_s[j], s);
    s = warp_sum(s);
    if (lane == 0) gam[i] = s;
  }
  for (int v = 1; v < 2 + k; ++v) {
    REAL s = 0;
    if (v == 1) {
      for (int j = tid; j < m; j += R1_NT) s = fma(a_s[j], a_s[j], s);
    } else {
      const REAL* xc = X + (size_t)(v - 2) * m;
      for (int j = tid; j < m; j += R1_NT) s = fma(a_s[j], xc[j], s);
    }
    s = warp_sum(s);
    if (lane == 0) red[w * (R1_MK + 2) + v] = s;
  }
  __syncthreads();
  // ---- B: rejection (thread per column) with its |rej|^2 partial; z = P^-1 coords
  {
    REAL s2 = 0;
    for (int j = tid; j < m; j += R1_NT) {
      REAL s = 0;
      for (int i = 0; i < r; ++i) s = fma(gam[i], C[(size_t)i * m + j], s);
      const REAL v = a_s[j] - s;
      rej_s[j] = v;
      s2 = fma(v, v, s2);
    }
    s2 = warp_sum(s2);
    if (lane == 0) red[w * (R1_MK + 2)] = s2;
  }
  for (int i = w; i < r; i += R1_NW) {
    const REAL* pr = P + (size_t)i * rc;
    REAL s = 0;
    for (int l = lane; l < r; l += 32) s = fma(pr[l], gam[l], s);
    s = warp_sum(s);
    if (lane == 0) z_s[i] = s;
  }
  __syncthreads();
  // ---- C: the sums (warp order), denom = 1 + coords.z, the rank test ---------------
  auto total = [&](int v) {
    REAL s = 0;
    for (int q = 0; q < R1_NW; ++q) s += red[q * (R1_MK + 2) + v];
    return s;
  };
  const REAL rej_sq = total(0), row_sq = total(1);
  REAL denom = 1;
  if (r > 0) {
    REAL s = 0;
    for (int i = lane; i < r; i += 32) s = fma(gam[i], z_s[i], s);
    s = warp_sum(s);
    denom = (REAL)1 + s;
  }
  bool bad = !isfinite(row_sq);
  for (int c = 0; c < k; ++c) bad |= !isfinite(y_s[c]);
  const bool dep = is_dependent<REAL>(rej_sq, row_sq, eps_sq<REAL>(cfg, r));
  REAL alpha = 1, last = 1;
  if (!bad && !dep && var != RGB_GENERAL) {
    const REAL resc = onorm ? (REAL)1 / sqrt(rej_sq) : (REAL)cfg.alpha;  // solver.py:359-366
    if (resc == (REAL)0) status |= RGB_ST_BAD_ALPHA;
    else {
      last = (REAL)1 / resc;
      alpha = (REAL)1 / last;
    }
  }
  if (bad) status |= RGB_ST_NONFINITE;
  else if (!dep && r >= rc) status |= RGB_ST_RANK_CAP;
  if (!status) {
    // a-priori residual y_c - a.x_c (recomputed where used: same bits, no local array)
    auto dy = [&](int c) { return y_s[c] - total(2 + c); };
    if (tid == 0 && logs.branch) logs.branch[0] = dep ? 0 : 1;
    if (logs.resid)
      for (int c = tid; c < k; c += R1_NT) reinterpret_cast<REAL*>(logs.resid)[c] = dy(c);
    REAL* gl = reinterpret_cast<REAL*>(logs.gain);
    // ---- D: the update, straight to global memory --------------------------------
    if (dep) {
      if (r > 0) {
        for (int idx = tid; idx < r * r; idx += R1_NT) {
          const int i = idx / r, l = idx - i * r;
          const REAL zs = z_s[l] / denom;
          REAL pv = P[(size_t)i * rc + l];
          pv -= z_s[i] * zs;
          Pg[(size_t)i * rc + l] = pv;
        }
        for (int j = tid; j < m; j += R1_NT) {
          REAL g = 0;
          for (int i = 0; i < r; ++i) g = fma(z_s[i] / denom, D[(size_t)i * m + j], g);
          for (int c = 0; c < k; ++c) {
            REAL xv = X[(size_t)c * m + j];
            xv += g * dy(c);
            Xg[(size_t)c * m + j] = xv;
            if (c == 0 && hx) hx[j] = xv;
          }
          if (gl) gl[j] = g;
        }
      } else if (gl) {
        for (int j = tid; j < m; j += R1_NT) gl[j] = 0;
      }
    } else {
      for (int j = tid; j < m; j += R1_NT) {
        const REAL g = rej_s[j] / rej_sq;
        if (var == RGB_GENERAL) {
          for (int i = 0; i < r; ++i) {
            REAL dv = D[(size_t)i * m + j];
            dv -= gam[i] * g;                        // solver.py:378
            Dg[(size_t)i * m + j] = dv;
          }
          Dg[(size_t)r * m + j] = g;                 // solver.py:379
          Cg[(size_t)r * m + j] = a_s[j];            // solver.py:376
        } else {
          Cg[(size_t)r * m + j] = alpha * rej_s[j];  // solver.py:384
          if (var == RGB_ORTHOGONAL) Dg[(size_t)r * m + j] = rej_s[j] / (alpha * rej_sq);
        }
        for (int c = 0; c < k; ++c) {
          REAL xv = X[(size_t)c * m + j];
          xv += g * dy(c);
          Xg[(size_t)c * m + j] = xv;
          if (c == 0 && hx) hx[j] = xv;
        }
        if (gl) gl[j] = g;
      }
      for (int i = tid; i <= r; i += R1_NT) {
        REAL edge = 0, corner = 1;
        if (var != RGB_GENERAL) {
          if (i < r) edge = -(alpha * z_s[i]);
          corner = alpha * alpha * (r > 0 ? denom : (REAL)1);
        }
        if (i < r) {
          Pg[(size_t)i * rc + r] = edge;
          Pg[(size_t)r * rc + i] = edge;
        } else {
          Pg[(size_t)r * rc + r] = corner;
        }
      }
      r += 1;
    }
    nobs += 1;
  }
  if (tid == 0) {
    st.rank[0] = r;
    st.nobs[0] = nobs;
    st.status[0] = status;
  }
  r1_publish<REAL>(mirror, dseq, nobs, r, status, tid);
}

static size_t row1_smem(const rgb_config& cfg) {
  const size_t es = cfg.dtype == RGB_F32 ? 4 : 8;
  const size_t m = cfg.m, rc = cfg.r_cap, k = cfg.k;
  const size_t n = 2 * m + 2 * rc + R1_MK + R1_NW * (R1_MK + 2) +
                   (cfg.variant == RGB_ORTHONORMAL ? 1 : 2) * rc * m + rc * rc + k * m;
  return n * es;
}
constexpr size_t R1_MAXS = 200 * 1024;

template <typename REAL>
static int launch_row1(const rgb_config& cfg, const rgb_state& st, const void* rows, const void* tgts,
                       const rgb_logs& logs, unsigned char* mirror, unsigned long long* dseq, void* hx,
                       cudaStream_t cs) {
  const size_t smem = row1_smem(cfg);
  if (smem > R1_MAXS) return RGB_E_UNSUPPORTED;
  auto kern = row1_kernel<REAL>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<1, R1_NT, smem, cs>>>(cfg, st, (const REAL*)rows, (const REAL*)tgts, logs, mirror, dseq, (REAL*)hx);
  return cudaGetLastError() == cudaSuccess ? RGB_OK : RGB_E_CUDA;
}
}  // namespace rgb

struct rgb_rowpipe {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  unsigned char* host = nullptr;      // pinned, mapped
  unsigned char* host_dev = nullptr;  // its device alias
  unsigned long long* dseq = nullptr;
  unsigned long long seq = 0;
  void* hx_dev = nullptr;  // caller's host x mirror (device alias), or null
  rgb_config cfg;
  rgb_state st;
  rgb_logs logs;
  int64_t off_in = 0;
};

static size_t align64(size_t v) { return (v + 63) & ~(size_t)63; }

extern "C" {

int64_t rgb_rowpipe_layout(const rgb_config* cfg, int f32in, int64_t* off_in, int64_t* off_resid,
                           int64_t* off_gain) {
  if (!cfg || cfg->m < 1 || cfg->k < 1) return RGB_E_INVALID;
  const size_t es = cfg->dtype == RGB_F32 ? 4 : 8, ies = (f32in || cfg->dtype == RGB_F32) ? 4 : 8;
  const size_t in = RGB_ROWPIPE_HEADER;
  const size_t resid = align64(in + ies * ((size_t)cfg->m + cfg->k));
  const size_t gain = align64(resid + es * (size_t)cfg->k);
  if (off_in) *off_in = (int64_t)in;
  if (off_resid) *off_resid = (int64_t)resid;
  if (off_gain) *off_gain = (int64_t)gain;
  return (int64_t)align64(gain + es * (size_t)cfg->m);
}

void rgb_rowpipe_destroy(rgb_rowpipe* p) {
  if (!p) return;
  if (p->exec) cudaGraphExecDestroy(p->exec);
  if (p->graph) cudaGraphDestroy(p->graph);
  if (p->dseq) cudaFree(p->dseq);
  if (p->host) cudaFreeHost(p->host);
  delete p;
}

int rgb_rowpipe_create(const rgb_config* cfg, const rgb_state* st, int want_report, int f32in, void* host_x,
                       rgb_rowpipe** out, void** host_block) {
  if (!cfg || !st || !out || !host_block) return RGB_E_INVALID;
  if (cfg->num_streams != 1) return RGB_E_INVALID;  // one stream (the drop-in solver)
  *out = nullptr;
  *host_block = nullptr;
  int64_t off_in, off_resid, off_gain;
  const int64_t bytes = rgb_rowpipe_layout(cfg, f32in, &off_in, &off_resid, &off_gain);
  if (bytes < 0) return (int)bytes;
  rgb_rowpipe* p = new rgb_rowpipe();
  p->cfg = *cfg;
  p->st = *st;
  if (cfg->variant == RGB_ORTHONORMAL) p->st.dual = p->st.basis;
  cudaError_t e = cudaHostAlloc(&p->host, (size_t)bytes, cudaHostAllocMapped | cudaHostAllocPortable);
  if (e == cudaSuccess) e = cudaHostGetDevicePointer((void**)&p->host_dev, p->host, 0);
  if (e == cudaSuccess && host_x) e = cudaHostGetDevicePointer(&p->hx_dev, host_x, 0);
  if (e == cudaSuccess) e = cudaMalloc(&p->dseq, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(p->dseq, 0, sizeof(unsigned long long));
  if (e != cudaSuccess) {
    rgb_rowpipe_destroy(p);
    return RGB_E_CUDA;
  }
  memset(p->host, 0, (size_t)bytes);
  memset(&p->logs, 0, sizeof(p->logs));
  if (want_report) {
    p->logs.branch = p->host_dev + RGB_ROWPIPE_OFF_BRANCH;
    p->logs.resid = p->host_dev + off_resid;
    p->logs.gain = p->host_dev + off_gain;
  }
  p->off_in = off_in;
  int nsm = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaStream_t cs;
  if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) {
    rgb_rowpipe_destroy(p);
    return RGB_E_CUDA;
  }
  const size_t ies = (f32in || cfg->dtype == RGB_F32) ? 4 : 8;
  const void* rows = p->host_dev + off_in;
  const void* tgts = p->host_dev + off_in + ies * cfg->m;
  int rc = RGB_OK;
  e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
  if (e == cudaSuccess) {
    rc = RGB_E_UNSUPPORTED;
    if (!f32in && cfg->k <= rgb::R1_MK)
      rc = cfg->dtype == RGB_F64
               ? rgb::launch_row1<double>(p->cfg, p->st, rows, tgts, p->logs, p->host_dev, p->dseq, p->hx_dev, cs)
               : rgb::launch_row1<float>(p->cfg, p->st, rows, tgts, p->logs, p->host_dev, p->dseq, p->hx_dev, cs);
    if (rc == RGB_E_UNSUPPORTED)  // float rows into a double state, k > 64, states beyond shared memory
      rc = rgb::launch_generic(p->cfg, p->st, rows, cfg->m, tgts, cfg->k, 1, p->logs, cs, nsm,
                               f32in && cfg->dtype == RGB_F64, p->host_dev, p->dseq, p->hx_dev);
    e = cudaStreamEndCapture(cs, &p->graph);
  }
  if (e == cudaSuccess && rc == RGB_OK) e = cudaGraphInstantiate(&p->exec, p->graph, 0);
  cudaStreamDestroy(cs);
  if (e != cudaSuccess || rc != RGB_OK) {
    cudaGetLastError();
    rgb_rowpipe_destroy(p);
    return rc != RGB_OK ? rc : RGB_E_CUDA;
  }
  *out = p;
  *host_block = p->host;
  return RGB_OK;
}

int rgb_rowpipe_run(rgb_rowpipe* p, void* stream) {
  if (!p) return RGB_E_INVALID;
  const unsigned long long want = p->seq + 1;
  const cudaError_t e = cudaGraphLaunch(p->exec, (cudaStream_t)stream);
  if (e != cudaSuccess) return RGB_E_CUDA;
  volatile unsigned long long* s = reinterpret_cast<volatile unsigned long long*>(p->host + RGB_ROWPIPE_OFF_SEQ);
  // spin on the sequence word; after a while also poll the stream (a kernel
  // fault never writes it) and yield the core
  for (long it = 0;; ++it) {
    if (*s == want) break;
    if (it < 20000) {
      _mm_pause();
      continue;
    }
    const cudaError_t q = cudaStreamQuery((cudaStream_t)stream);
    if (q != cudaSuccess && q != cudaErrorNotReady) return RGB_E_CUDA;
    if (q == cudaSuccess && *s != want) return RGB_E_CUDA;  // finished without the tail
    sched_yield();
  }
  p->seq = want;
  return RGB_OK;
}

}  // extern "C"
