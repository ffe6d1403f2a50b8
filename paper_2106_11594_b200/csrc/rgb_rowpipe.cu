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
// the global-state kernels (states beyond shared memory) run 1 024 threads: their
// phases stream the factors from L2, and more warps keep more loads in flight
constexpr int R1_NT_GS = 1024;
__host__ __device__ constexpr int r1_threads(bool gs) { return gs ? R1_NT_GS : R1_NT; }

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
// shared-memory layout of the row kernels: the row and its scratch, then the state
template <typename REAL>
struct R1Smem {
  REAL *a_s, *rej_s, *gam, *z_s, *y_s, *red, *zd, *dyv, *D, *C, *P, *X;
  // gst: the state stays in global memory (states beyond shared memory; L2-resident)
  __device__ R1Smem(unsigned char* raw, const rgb_config& cfg, const rgb_state* gst = nullptr, int nw = R1_NW) {
    const int m = cfg.m, rc = cfg.r_cap;
    a_s = reinterpret_cast<REAL*>(raw);
    rej_s = a_s + m;
    gam = rej_s + m;
    z_s = gam + rc;
    y_s = z_s + rc;
    red = y_s + R1_MK;                                       // [NW][MK + 2]
    zd = red + nw * (R1_MK + 2);                             // z / denom
    dyv = zd + rc;                                           // y - a.x (a-priori residuals)
    if (gst) {
      C = reinterpret_cast<REAL*>(gst->basis);
      D = cfg.variant == RGB_ORTHONORMAL ? C : reinterpret_cast<REAL*>(gst->dual);
      P = reinterpret_cast<REAL*>(gst->gram_inv);
      X = reinterpret_cast<REAL*>(gst->x);
      return;
    }
    D = dyv + R1_MK;                                         // C~ rows < r
    C = cfg.variant == RGB_ORTHONORMAL ? D : D + (size_t)rc * m;  // C rows < r
    P = C + (size_t)rc * m;                                  // P^-1 [r][r] at stride rc
    X = P + (size_t)rc * rc;
  }
};

// the state into shared memory (cp.async; the caller commits and waits)
template <typename REAL>
__device__ __forceinline__ void r1_stage_state(const rgb_config& cfg, const REAL* Cg, const REAL* Dg, const REAL* Pg,
                                               const REAL* Xg, const R1Smem<REAL>& S_, int r) {
  const int m = cfg.m, k = cfg.k, rc = cfg.r_cap, tid = threadIdx.x;
  for (int e = tid; e < r * m; e += R1_NT) r1_cp(S_.D + e, Dg + e, sizeof(REAL));
  if (cfg.variant != RGB_ORTHONORMAL)
    for (int e = tid; e < r * m; e += R1_NT) r1_cp(S_.C + e, Cg + e, sizeof(REAL));
  for (int e = tid; e < r * r; e += R1_NT) {
    const int i = e / r, l = e - i * r;
    r1_cp(S_.P + (size_t)i * rc + l, Pg + (size_t)i * rc + l, sizeof(REAL));
  }
  for (int e = tid; e < k * m; e += R1_NT) r1_cp(S_.X + e, Xg + e, sizeof(REAL));
}

#ifdef RGB_SERVE_PROBE
__device__ unsigned long long g_sprobe[16];  // ns summed: poll, row read, fold, publish; rows; fold phases A-D at 8..11
__device__ __forceinline__ unsigned long long sp_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define SPROBE(i)                                    \
  do {                                               \
    if (threadIdx.x == 0) {                          \
      const unsigned long long n_ = sp_now();        \
      atomicAdd(&g_sprobe[i], n_ - sp_t);            \
      sp_t = n_;                                     \
    }                                                \
  } while (0)
#else
#define SPROBE(i) \
  do {            \
  } while (0)
#endif

// The fold of the staged row (a_s, y_s) on the staged state, phases A-D: results
// straight to global memory (and, for the row server, SERVE, into the staged
// state too, which it keeps between rows).  r, status, nobs are updated.
// Phases A and B of the fold -- the projection of the staged row a_s on the staged
// basis (solver.py:286-291): coords gam (warp per dual row), the rejection rej_s
// (thread per column) and per-warp partials of |rej|^2 (red[w][0]), |a|^2 (red[w][1])
// and a.x_c (red[w][2 + c]); z = P^-1 coords (z_s).  Ends with a CTA barrier.
template <typename REAL, int NT>
__device__ __forceinline__ void row1_ab(const rgb_config& cfg, const R1Smem<REAL>& S_, int r) {
  const int m = cfg.m, k = cfg.k, rc = cfg.r_cap;
  const REAL *a_s = S_.a_s, *D = S_.D, *C = S_.C, *P = S_.P, *X = S_.X;
  REAL *rej_s = S_.rej_s, *gam = S_.gam, *z_s = S_.z_s, *red = S_.red;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  // ---- A: coords (warp per dual row) and the |a|^2, a.x_c block partials ---------
  for (int i = w; i < r; i += (NT / 32)) {
    const REAL* d = D + (size_t)i * m;
    REAL s = 0;
    for (int j = lane; j < m; j += 32) s = fma(d[j], a_s[j], s);
    s = warp_sum(s);
    if (lane == 0) gam[i] = s;
  }
  for (int v = 1; v < 2 + k; ++v) {
    REAL s = 0;
    if (v == 1) {
      for (int j = tid; j < m; j += NT) s = fma(a_s[j], a_s[j], s);
    } else {
      const REAL* xc = X + (size_t)(v - 2) * m;
      for (int j = tid; j < m; j += NT) s = fma(a_s[j], xc[j], s);
    }
    s = warp_sum(s);
    if (lane == 0) red[w * (R1_MK + 2) + v] = s;
  }
  __syncthreads();
  // ---- B: rejection (thread per column) with its |rej|^2 partial; z = P^-1 coords
  {
    REAL s2 = 0;
    for (int j = tid; j < m; j += NT) {
      REAL s = 0;
      for (int i = 0; i < r; ++i) s = fma(gam[i], C[(size_t)i * m + j], s);
      const REAL v = a_s[j] - s;
      rej_s[j] = v;
      s2 = fma(v, v, s2);
    }
    s2 = warp_sum(s2);
    if (lane == 0) red[w * (R1_MK + 2)] = s2;
  }
  for (int i = w; i < r; i += (NT / 32)) {
    const REAL* pr = P + (size_t)i * rc;
    REAL s = 0;
    for (int l = lane; l < r; l += 32) s = fma(pr[l], gam[l], s);
    s = warp_sum(s);
    if (lane == 0) z_s[i] = s;
  }
  __syncthreads();
}

template <typename REAL, bool SERVE, int NT>
__device__ __forceinline__ void row1_fold(const rgb_config& cfg, const rgb_state& st, const rgb_logs& logs,
                                          const R1Smem<REAL>& S_, int& r, int& status, int64_t& nobs, REAL* hx) {
  const int m = cfg.m, k = cfg.k, rc = cfg.r_cap, var = cfg.variant;
  const bool onorm = var == RGB_ORTHONORMAL;
  REAL *a_s = S_.a_s, *rej_s = S_.rej_s, *gam = S_.gam, *z_s = S_.z_s, *y_s = S_.y_s, *red = S_.red;
  REAL *zd = S_.zd, *dyv = S_.dyv;
  REAL *D = S_.D, *C = S_.C, *P = S_.P, *X = S_.X;
  REAL* Cg = reinterpret_cast<REAL*>(st.basis);
  REAL* Dg = onorm ? Cg : reinterpret_cast<REAL*>(st.dual);
  REAL* Pg = reinterpret_cast<REAL*>(st.gram_inv);
  REAL* Xg = reinterpret_cast<REAL*>(st.x);
  const int tid = threadIdx.x, lane = tid & 31;
#ifdef RGB_SERVE_PROBE
  unsigned long long sp_t = sp_now();
#endif
  row1_ab<REAL, NT>(cfg, S_, r);
  SPROBE(9);
  // ---- C: the sums (warp order), denom = 1 + coords.z, the rank test ---------------
  auto total = [&](int v) {
    REAL s = 0;
    for (int q = 0; q < (NT / 32); ++q) s += red[q * (R1_MK + 2) + v];
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
    // a-priori residuals y_c - a.x_c and z / denom, once (the same bits as forming
    // them where used)
    for (int c = tid; c < k; c += NT) dyv[c] = y_s[c] - total(2 + c);
    if (dep)
      for (int i = tid; i < r; i += NT) zd[i] = z_s[i] / denom;
    __syncthreads();
    SPROBE(10);
    auto dy = [&](int c) { return dyv[c]; };
    if (tid == 0 && logs.branch) logs.branch[0] = dep ? 0 : 1;
    if (logs.resid)
      for (int c = tid; c < k; c += NT) reinterpret_cast<REAL*>(logs.resid)[c] = dy(c);
    REAL* gl = reinterpret_cast<REAL*>(logs.gain);
    // ---- D: the update, straight to global memory --------------------------------
    if (dep) {
      if (r > 0) {
        for (int idx = tid; idx < r * r; idx += NT) {
          const int i = idx / r, l = idx - i * r;
          const REAL zs = zd[l];
          REAL pv = P[(size_t)i * rc + l];
          pv -= z_s[i] * zs;
          Pg[(size_t)i * rc + l] = pv;
          if constexpr (SERVE) P[(size_t)i * rc + l] = pv;
        }
        for (int j = tid; j < m; j += NT) {
          REAL g = 0;
          for (int i = 0; i < r; ++i) g = fma(zd[i], D[(size_t)i * m + j], g);
          for (int c = 0; c < k; ++c) {
            REAL xv = X[(size_t)c * m + j];
            xv += g * dy(c);
            Xg[(size_t)c * m + j] = xv;
            if constexpr (SERVE) X[(size_t)c * m + j] = xv;
            if (c == 0 && hx) hx[j] = xv;
          }
          if (gl) gl[j] = g;
        }
      } else if (gl) {
        for (int j = tid; j < m; j += NT) gl[j] = 0;
      }
    } else {
      for (int j = tid; j < m; j += NT) {
        const REAL g = rej_s[j] / rej_sq;
        if (var == RGB_GENERAL) {
          for (int i = 0; i < r; ++i) {
            REAL dv = D[(size_t)i * m + j];
            dv -= gam[i] * g;                        // solver.py:378
            Dg[(size_t)i * m + j] = dv;
            if constexpr (SERVE) D[(size_t)i * m + j] = dv;
          }
          Dg[(size_t)r * m + j] = g;                 // solver.py:379
          Cg[(size_t)r * m + j] = a_s[j];            // solver.py:376
          if constexpr (SERVE) {
            D[(size_t)r * m + j] = g;
            C[(size_t)r * m + j] = a_s[j];
          }
        } else {
          Cg[(size_t)r * m + j] = alpha * rej_s[j];  // solver.py:384
          if (var == RGB_ORTHOGONAL) Dg[(size_t)r * m + j] = rej_s[j] / (alpha * rej_sq);
          if constexpr (SERVE) {
            C[(size_t)r * m + j] = alpha * rej_s[j];  // (orthonormal: D aliases C)
            if (var == RGB_ORTHOGONAL) D[(size_t)r * m + j] = rej_s[j] / (alpha * rej_sq);
          }
        }
        for (int c = 0; c < k; ++c) {
          REAL xv = X[(size_t)c * m + j];
          xv += g * dy(c);
          Xg[(size_t)c * m + j] = xv;
          if constexpr (SERVE) X[(size_t)c * m + j] = xv;
          if (c == 0 && hx) hx[j] = xv;
        }
        if (gl) gl[j] = g;
      }
      for (int i = tid; i <= r; i += NT) {
        REAL edge = 0, corner = 1;
        if (var != RGB_GENERAL) {
          if (i < r) edge = -(alpha * z_s[i]);
          corner = alpha * alpha * (r > 0 ? denom : (REAL)1);
        }
        if (i < r) {
          Pg[(size_t)i * rc + r] = edge;
          Pg[(size_t)r * rc + i] = edge;
          if constexpr (SERVE) P[(size_t)i * rc + r] = P[(size_t)r * rc + i] = edge;
        } else {
          Pg[(size_t)r * rc + r] = corner;
          if constexpr (SERVE) P[(size_t)r * rc + r] = corner;
        }
      }
      r += 1;
    }
    nobs += 1;
#ifdef RGB_SERVE_PROBE
    __syncthreads();
#endif
    SPROBE(11);
  }
}

// GS: the state stays in global memory (no staging; the fold reads and writes it there)
template <typename REAL, bool GS>
__global__ void __launch_bounds__(r1_threads(GS), 1) row1_kernel(rgb_config cfg, rgb_state st, const REAL* __restrict__ a_g,
                                                     const REAL* __restrict__ y_g, rgb_logs logs,
                                                     unsigned char* __restrict__ mirror,
                                                     unsigned long long* __restrict__ dseq, REAL* __restrict__ hx) {
  constexpr int NT = r1_threads(GS);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const R1Smem<REAL> S_(smem_raw, cfg, GS ? &st : nullptr, NT / 32);
  const int m = cfg.m, k = cfg.k;
  const bool onorm = cfg.variant == RGB_ORTHONORMAL;
  const REAL* Cg = reinterpret_cast<const REAL*>(st.basis);
  const REAL* Dg = onorm ? Cg : reinterpret_cast<const REAL*>(st.dual);
  const REAL* Pg = reinterpret_cast<const REAL*>(st.gram_inv);
  const REAL* Xg = reinterpret_cast<const REAL*>(st.x);
  const int tid = threadIdx.x;
  int r = st.rank[0];
  int status = st.status[0];
  int64_t nobs = st.nobs[0];
  if (status) {
    r1_publish<REAL>(mirror, dseq, nobs, r, status, tid);
    return;
  }
  // ---- stage: the row and targets (host memory) first, then the state ------------
  for (int j = tid; j < m; j += NT) r1_cp(S_.a_s + j, a_g + j, sizeof(REAL));
  for (int c = tid; c < k; c += NT) r1_cp(S_.y_s + c, y_g + c, sizeof(REAL));
  if (!GS) r1_stage_state<REAL>(cfg, Cg, Dg, Pg, Xg, S_, r);
  asm volatile("cp.async.commit_group;\n" ::);
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();
  row1_fold<REAL, false, NT>(cfg, st, logs, S_, r, status, nobs, hx);
  if (tid == 0) {
    st.rank[0] = r;
    st.nobs[0] = nobs;
    st.status[0] = status;
  }
  r1_publish<REAL>(mirror, dseq, nobs, r, status, tid);
}


// The row SERVER (rgb_rowpipe_run with a positive idle time): one persistent CTA
// that stages the state once and then folds row after row.  Thread 0 polls the
// request word of the mapped host block (acquire, system scope); a request is
// the number of the row to fold (one more than the rows served, dseq); the row
// and its targets are then read from the block with volatile loads (never from a
// cache line of an earlier row), folded with row1_fold<SERVE> -- the same
// arithmetic as row1_kernel, so results are bit-identical -- and published as
// row1_kernel does.  The server exits on the stop word, after a stop status, or
// after idle_ns without a request (the host relaunches it on demand).
template <typename REAL, bool GS>
__global__ void __launch_bounds__(r1_threads(GS), 1) row1_serve_kernel(rgb_config cfg, rgb_state st,
                                                           const REAL* __restrict__ a_g,
                                                           const REAL* __restrict__ y_g, rgb_logs logs,
                                                           unsigned char* __restrict__ mirror,
                                                           unsigned long long* __restrict__ dseq,
                                                           REAL* __restrict__ hx, REAL* __restrict__ proj,
                                                           unsigned long long idle_ns) {
  constexpr int NT = r1_threads(GS);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int s_cmd;
  const R1Smem<REAL> S_(smem_raw, cfg, GS ? &st : nullptr, NT / 32);
  const int m = cfg.m, k = cfg.k;
  const bool onorm = cfg.variant == RGB_ORTHONORMAL;
  const REAL* Cg = reinterpret_cast<const REAL*>(st.basis);
  const REAL* Dg = onorm ? Cg : reinterpret_cast<const REAL*>(st.dual);
  const REAL* Pg = reinterpret_cast<const REAL*>(st.gram_inv);
  const REAL* Xg = reinterpret_cast<const REAL*>(st.x);
  const int tid = threadIdx.x;
  int r = st.rank[0];
  int status = st.status[0];
  int64_t nobs = st.nobs[0];
  if (!GS) r1_stage_state<REAL>(cfg, Cg, Dg, Pg, Xg, S_, r);  // (a stopped state still projects)
  asm volatile("cp.async.commit_group;\n" ::);
  asm volatile("cp.async.wait_group 0;\n" ::);
  const unsigned long long* req = reinterpret_cast<const unsigned long long*>(mirror + RGB_ROWPIPE_OFF_REQ);
  const unsigned long long* preq = reinterpret_cast<const unsigned long long*>(mirror + RGB_ROWPIPE_OFF_PREQ);
  __shared__ unsigned long long s_preq;
  const volatile unsigned* stop = reinterpret_cast<const volatile unsigned*>(mirror + RGB_ROWPIPE_OFF_STOP);
  const volatile REAL* av = a_g;
  const volatile REAL* yv = y_g;
#ifdef RGB_SERVE_PROBE
  unsigned long long sp_t = sp_now();
#endif
  while (true) {
    if (tid == 0) {
      const unsigned long long want = *dseq + 1;
      unsigned long long t0, now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      // the projection served last is the one whose number the block's PSEQ word holds
      const unsigned long long pdone =
          *reinterpret_cast<volatile const unsigned long long*>(mirror + RGB_ROWPIPE_OFF_PSEQ);
      int cmd = 0;
      while (true) {
        unsigned long long v;
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(req) : "memory");
        if (v == want) {
          cmd = 1;
          break;
        }
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(preq) : "memory");
        if (v != pdone) {
          cmd = 2;
          s_preq = v;
          break;
        }
        if (*stop) break;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        if (now - t0 > idle_ns) break;
      }
      s_cmd = cmd;
    }
    __syncthreads();
    if (s_cmd == 2) {
      // project() (solver.py:210-219): coords, rejection and |rej|^2 of the staged row on
      // the current basis -- phases A and B of the fold, nothing written to the state
      for (int j = tid; j < m; j += NT) S_.a_s[j] = av[j];
      __syncthreads();
      row1_ab<REAL, NT>(cfg, S_, r);
      for (int i = tid; i < cfg.r_cap; i += NT) proj[i] = i < r ? S_.gam[i] : (REAL)0;
      for (int j = tid; j < m; j += NT) proj[cfg.r_cap + j] = S_.rej_s[j];
      if (tid == 0) {
        REAL s = 0;
        for (int q = 0; q < NT / 32; ++q) s += S_.red[q * (R1_MK + 2)];  // warp order, as the fold
        proj[cfg.r_cap + m] = s;
      }
      __syncthreads();
      if (tid == 0)
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(mirror + RGB_ROWPIPE_OFF_PSEQ), "l"(s_preq)
                     : "memory");
      __syncthreads();
      continue;
    }
    if (s_cmd != 1) return;
    SPROBE(0);
    if (!status) {  // (a state stopped earlier only publishes its counters, as row1_kernel)
      for (int j = tid; j < m; j += NT) S_.a_s[j] = av[j];
      for (int c = tid; c < k; c += NT) S_.y_s[c] = yv[c];
      __syncthreads();
      SPROBE(1);
      row1_fold<REAL, true, NT>(cfg, st, logs, S_, r, status, nobs, hx);
      __syncthreads();
      SPROBE(2);
      if (tid == 0) {
        st.rank[0] = r;
        st.nobs[0] = nobs;
        st.status[0] = status;
      }
    }
    r1_publish<REAL>(mirror, dseq, nobs, r, status, tid);
    SPROBE(3);
#ifdef RGB_SERVE_PROBE
    if (tid == 0) atomicAdd(&g_sprobe[4], 1ull);
#endif
    if (status) return;  // a stop: the host grows the capacity or reports it
    __syncthreads();     // the request word is re-read only after every thread's publish path
  }
}

// shared memory of the row kernels: the scratch, plus the staged state unless gs
static size_t row1_smem(const rgb_config& cfg, bool gs = false) {
  const size_t es = cfg.dtype == RGB_F32 ? 4 : 8;
  const size_t m = cfg.m, rc = cfg.r_cap, k = cfg.k;
  size_t n = 2 * m + 3 * rc + 2 * R1_MK + (r1_threads(gs) / 32) * (R1_MK + 2);
  if (!gs) n += (cfg.variant == RGB_ORTHONORMAL ? 1 : 2) * rc * m + rc * rc + k * m;
  return n * es;
}
constexpr size_t R1_MAXS = 200 * 1024;

template <typename REAL>
static int launch_row1(const rgb_config& cfg, const rgb_state& st, const void* rows, const void* tgts,
                       const rgb_logs& logs, unsigned char* mirror, unsigned long long* dseq, void* hx,
                       cudaStream_t cs) {
  // states beyond shared memory stay in global memory (L2-resident)
  const bool gs = row1_smem(cfg) > R1_MAXS;
  const size_t smem = row1_smem(cfg, gs);
  if (smem > R1_MAXS) return RGB_E_UNSUPPORTED;
  auto kern = gs ? row1_kernel<REAL, true> : row1_kernel<REAL, false>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<1, r1_threads(gs), smem, cs>>>(cfg, st, (const REAL*)rows, (const REAL*)tgts, logs, mirror, dseq, (REAL*)hx);
  return cudaGetLastError() == cudaSuccess ? RGB_OK : RGB_E_CUDA;
}

template <typename REAL>
static int launch_row1_serve(const rgb_config& cfg, const rgb_state& st, const void* rows, const void* tgts,
                             const rgb_logs& logs, unsigned char* mirror, unsigned long long* dseq, void* hx,
                             void* proj, unsigned long long idle_ns, cudaStream_t cs) {
  const bool gs = row1_smem(cfg) > R1_MAXS;
  const size_t smem = row1_smem(cfg, gs);
  if (smem > R1_MAXS) return RGB_E_UNSUPPORTED;
  auto kern = gs ? row1_serve_kernel<REAL, true> : row1_serve_kernel<REAL, false>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<1, r1_threads(gs), smem, cs>>>(cfg, st, (const REAL*)rows, (const REAL*)tgts, logs, mirror, dseq, (REAL*)hx,
                                       (REAL*)proj, idle_ns);
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
  int64_t off_in = 0, off_proj = 0;
  // row server (rgb_rowpipe_run with RGB_ROWSERVE_IDLE_US > 0): a persistent
  // kernel on its own stream, launched on demand, that exits after idle_ns
  bool serve_ok = false, serving = false;
  unsigned long long idle_ns = 0;
  cudaStream_t sstream = nullptr;
  cudaEvent_t ev = nullptr;
  std::chrono::steady_clock::time_point last;
  const void* rows = nullptr;
  const void* tgts = nullptr;
  unsigned long long pseq = 0;  // projections requested so far
};

// Stop the row server (if it runs) and wait for it: the state in global memory is
// then final and the caller may run other kernels on it.
static int serve_stop(rgb_rowpipe* p) {
  if (!p->serving) return RGB_OK;
  __atomic_store_n(reinterpret_cast<unsigned*>(p->host + RGB_ROWPIPE_OFF_STOP), 1u, __ATOMIC_RELEASE);
  const cudaError_t e = cudaStreamSynchronize(p->sstream);
  __atomic_store_n(reinterpret_cast<unsigned*>(p->host + RGB_ROWPIPE_OFF_STOP), 0u, __ATOMIC_RELEASE);
  p->serving = false;
  return e == cudaSuccess ? RGB_OK : RGB_E_CUDA;
}

static int serve_launch(rgb_rowpipe* p, cudaStream_t caller) {
  // ordered after the caller's earlier work on the state
  if (cudaEventRecord(p->ev, caller) != cudaSuccess || cudaStreamWaitEvent(p->sstream, p->ev, 0) != cudaSuccess)
    return RGB_E_CUDA;
  const int rc = p->cfg.dtype == RGB_F64
                     ? rgb::launch_row1_serve<double>(p->cfg, p->st, p->rows, p->tgts, p->logs, p->host_dev, p->dseq,
                                                      p->hx_dev, p->host_dev + p->off_proj, p->idle_ns, p->sstream)
                     : rgb::launch_row1_serve<float>(p->cfg, p->st, p->rows, p->tgts, p->logs, p->host_dev, p->dseq,
                                                     p->hx_dev, p->host_dev + p->off_proj, p->idle_ns, p->sstream);
  if (rc == RGB_OK) p->serving = true;
  return rc;
}

static size_t align64(size_t v) { return (v + 63) & ~(size_t)63; }

extern "C" {

int64_t rgb_rowpipe_layout(const rgb_config* cfg, int f32in, int64_t* off_in, int64_t* off_resid,
                           int64_t* off_gain) {
  if (!cfg || cfg->m < 1 || cfg->k < 1) return RGB_E_INVALID;
  const size_t es = cfg->dtype == RGB_F32 ? 4 : 8, ies = (f32in || cfg->dtype == RGB_F32) ? 4 : 8;
  const size_t in = RGB_ROWPIPE_HEADER;
  const size_t resid = align64(in + ies * ((size_t)cfg->m + cfg->k));
  const size_t gain = align64(resid + es * (size_t)cfg->k);
  const size_t proj = align64(gain + es * (size_t)cfg->m);  // rgb_rowpipe_proj_offset
  if (off_in) *off_in = (int64_t)in;
  if (off_resid) *off_resid = (int64_t)resid;
  if (off_gain) *off_gain = (int64_t)gain;
  return (int64_t)align64(proj + es * ((size_t)cfg->r_cap + cfg->m + 1));
}

int64_t rgb_rowpipe_proj_offset(const rgb_config* cfg, int f32in) {
  int64_t off_gain = 0;
  const int64_t bytes = rgb_rowpipe_layout(cfg, f32in, nullptr, nullptr, &off_gain);
  if (bytes < 0) return bytes;
  const size_t es = cfg->dtype == RGB_F32 ? 4 : 8;
  return (int64_t)align64((size_t)off_gain + es * (size_t)cfg->m);
}

void rgb_rowpipe_destroy(rgb_rowpipe* p) {
  if (!p) return;
  serve_stop(p);
  if (p->sstream) cudaStreamDestroy(p->sstream);
  if (p->ev) cudaEventDestroy(p->ev);
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
  p->off_proj = rgb_rowpipe_proj_offset(cfg, f32in);
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
    if (rc == RGB_E_UNSUPPORTED)  // float rows into a double state, k > 64, scratch beyond shared memory
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
  // the row server: where the one-row kernel applies (same-type inputs, k <= 64; the
  // state in shared memory when it fits, else in global memory)
  p->rows = rows;
  p->tgts = tgts;
  const char* idle = getenv("RGB_ROWSERVE_IDLE_US");
  const long idle_us = idle && idle[0] ? atol(idle) : 500;
  if (idle_us > 0 && !f32in && cfg->k <= rgb::R1_MK && rgb::row1_smem(*cfg, true) <= rgb::R1_MAXS &&
      cudaStreamCreateWithFlags(&p->sstream, cudaStreamNonBlocking) == cudaSuccess &&
      cudaEventCreateWithFlags(&p->ev, cudaEventDisableTiming) == cudaSuccess) {
    p->serve_ok = true;
    p->idle_ns = (unsigned long long)idle_us * 1000ull;
  }
  cudaGetLastError();
  *out = p;
  *host_block = p->host;
  return RGB_OK;
}

int rgb_rowpipe_quiesce(rgb_rowpipe* p) {
  if (!p) return RGB_E_INVALID;
  return serve_stop(p);
}

// a server that is surely still polling, or a new one (ordered after `caller`)
static int serve_ensure(rgb_rowpipe* p, cudaStream_t caller) {
  using clk = std::chrono::steady_clock;
  if (p->serving) {
    // surely still polling when the last request was served well within its idle time
    // (its idle clock started before that request's publish was seen here)
    const auto idle = std::chrono::nanoseconds((long long)p->idle_ns);
    if (clk::now() - p->last > idle - std::chrono::microseconds(100)) {
      const cudaError_t q = cudaStreamQuery(p->sstream);
      if (q == cudaSuccess) p->serving = false;
      else if (q != cudaErrorNotReady) return RGB_E_CUDA;
    }
  }
  return p->serving ? RGB_OK : serve_launch(p, caller);
}

// post request `want` at the block's word `off_req` and spin until the server
// publishes it at `off_done`
static int serve_request(rgb_rowpipe* p, cudaStream_t caller, size_t off_req, size_t off_done,
                         unsigned long long want) {
  int rc = serve_ensure(p, caller);
  if (rc != RGB_OK) return rc;
  __atomic_store_n(reinterpret_cast<unsigned long long*>(p->host + off_req), want, __ATOMIC_RELEASE);
  volatile unsigned long long* s = reinterpret_cast<volatile unsigned long long*>(p->host + off_done);
  for (long it = 0;; ++it) {
    if (*s == want) break;
    if (it < 4000) {
      _mm_pause();
      continue;
    }
    // the server may have timed out just before the request: relaunch it (it
    // serves the pending request: a row whose number is one more than the rows
    // served, a projection whose number differs from the last one published)
    const cudaError_t q = cudaStreamQuery(p->sstream);
    if (q == cudaSuccess && *s != want) {
      p->serving = false;
      rc = serve_launch(p, caller);
      if (rc != RGB_OK) return rc;
      it = 0;
      continue;
    }
    if (q != cudaSuccess && q != cudaErrorNotReady) return RGB_E_CUDA;
    sched_yield();
  }
  p->last = std::chrono::steady_clock::now();
  return RGB_OK;
}

static int serve_run(rgb_rowpipe* p, cudaStream_t caller) {
  const unsigned long long want = p->seq + 1;
  const int rc = serve_request(p, caller, RGB_ROWPIPE_OFF_REQ, RGB_ROWPIPE_OFF_SEQ, want);
  if (rc == RGB_OK) p->seq = want;
  return rc;
}

int rgb_rowpipe_project(rgb_rowpipe* p, void* stream) {
  if (!p) return RGB_E_INVALID;
  if (!p->serve_ok) return RGB_E_UNSUPPORTED;
  const unsigned long long want = p->pseq + 1;
  const int rc = serve_request(p, (cudaStream_t)stream, RGB_ROWPIPE_OFF_PREQ, RGB_ROWPIPE_OFF_PSEQ, want);
  if (rc == RGB_OK) p->pseq = want;
  return rc;
}

int rgb_rowpipe_run(rgb_rowpipe* p, void* stream) {
  if (!p) return RGB_E_INVALID;
  if (p->serve_ok) return serve_run(p, (cudaStream_t)stream);
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

#ifdef RGB_SERVE_PROBE
extern "C" int rgb_serve_probe(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, rgb::g_sprobe, sizeof(rgb::g_sprobe));
  if (reset) {
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(rgb::g_sprobe, z, sizeof(z));
  }
  return 0;
}
#endif
