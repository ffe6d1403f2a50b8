// rgb_abi.cu -- extern "C" entry points of librgb.so (declared in include/rgb.h).
//
// Validation mirrors the reference's constructor and input checks
// (solver.py:142-158, scalars.py:108-138) as return codes.  Dispatch, first
// match wins: the one-warp tensor-core kernel (m 64, r_cap 16, k <= 8), the
// panel kernel (general variant: m 128 with r_cap 16 / 32, m 256 with r_cap 16;
// RGB_NO_PANEL=1 in the environment turns it off, for A/B runs and tests;
// RGB_BLOCKED_SEQ=1 / RGB_PANEL_SEQ=1 / RGB_CLUSTER_SEQ=1 make these kernels and the cluster
// kernel fold every stream with the sequential chain instead of the deferred fold, see
// rgb_blocked.cu), the
// warp-group kernel (m 128 / 256 with r_cap 16 / 32, every variant), the cluster kernel
// (r_cap 64, m <= 1 080) and the grid kernel (a few large streams, m <= 2 368,
// r_cap <= 512) -- the last two for calls of 8+ rows -- and the shape-generic
// kernel for everything else, for fp32 state and for per-row residual logs.
// No host allocation and no per-call state (the grid kernel's workspace is
// stream-ordered, from a library-owned device memory pool that is kept
// between calls).
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "rgb_common.cuh"

namespace rgb {
int launch_generic(const rgb_config& cfg, rgb_state& st, const void* rows, int64_t rows_stride,
                   const void* targets, int64_t tg_stride, int64_t T, const rgb_logs& logs,
                   cudaStream_t stream, int num_sms, bool f32in, unsigned char* mirror = nullptr,
                   unsigned long long* dseq = nullptr, void* hx = nullptr);
bool blocked_supports(const rgb_config& cfg);
bool blocked_wg_supports(const rgb_config& cfg);
bool panel_supports(const rgb_config& cfg);
int launch_panel(const rgb_config& cfg, rgb_state& st, const void* rows, int64_t rows_stride, const void* targets,
                 int64_t tg_stride, int64_t T, const rgb_logs& logs, cudaStream_t stream, int num_sms, bool f32in);
bool grid_supports(const rgb_config& cfg);
bool f32_supports(const rgb_config& cfg);
int launch_f32(const rgb_config& cfg, rgb_state& st, const void* rows, int64_t rows_stride, const void* targets,
               int64_t tg_stride, int64_t T, const rgb_logs& logs, cudaStream_t stream, int num_sms);
bool cluster_supports(const rgb_config& cfg);
int launch_cluster(const rgb_config& cfg, rgb_state& st, const void* rows, int64_t rows_stride, const void* targets,
                   int64_t tg_stride, int64_t T, const rgb_logs& logs, cudaStream_t stream, int num_sms,
                   bool f32in);
int launch_grid(const rgb_config& cfg, rgb_state& st, const void* rows, int64_t rows_stride, const void* targets,
                int64_t tg_stride, int64_t T, const rgb_logs& logs, cudaStream_t stream, int num_sms,
                bool f32in);
int launch_blocked_wg(const rgb_config& cfg, rgb_state& st, const void* rows, int64_t rows_stride,
                      const void* targets, int64_t tg_stride, int64_t T, const rgb_logs& logs,
                      cudaStream_t stream, int num_sms, bool f32in);
int launch_blocked(const rgb_config& cfg, rgb_state& st, const void* rows, int64_t rows_stride,
                   const void* targets, int64_t tg_stride, int64_t T, const rgb_logs& logs,
                   cudaStream_t stream, int num_sms, bool f32in);
int launch_project(const rgb_config& cfg, const rgb_state& st, const void* rows, void* coords,
                   void* rejection, void* rej_sq, uint8_t* dependent, cudaStream_t stream);
int launch_pinv(const rgb_config& cfg, const rgb_state& st, const void* coords, int64_t n,
                void* out, cudaStream_t stream);
int launch_covariance(const rgb_config& cfg, const rgb_state& st, void* out, cudaStream_t stream);
}  // namespace rgb

static thread_local char g_err[512] = "";

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof(g_err), "%s", msg);
  return code;
}

static int cuda_fail(cudaError_t e, const char* where) {
  snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
  return RGB_E_CUDA;
}

static int check_cfg(const rgb_config* cfg) {
  if (!cfg) return fail(RGB_E_INVALID, "null config");
  if (cfg->num_streams < 0) return fail(RGB_E_INVALID, "num_streams must be >= 0");
  if (cfg->m < 1) return fail(RGB_E_INVALID, "num_regressors must be a positive integer");
  if (cfg->k < 1) return fail(RGB_E_INVALID, "k (right-hand sides) must be >= 1");
  if (cfg->r_cap < 1) return fail(RGB_E_INVALID, "r_cap must be >= 1");
  if (cfg->dtype != RGB_F64 && cfg->dtype != RGB_F32) return fail(RGB_E_INVALID, "unknown dtype");
  if (cfg->variant < RGB_GENERAL || cfg->variant > RGB_ORTHONORMAL)
    return fail(RGB_E_INVALID, "unknown variant; expected general, orthogonal or orthonormal");
  if (cfg->eps_mode != RGB_EPS_AUTO && cfg->eps_mode != RGB_EPS_FIXED)
    return fail(RGB_E_INVALID, "unknown eps mode (exact-zero is rational-only)");
  if (cfg->eps_mode == RGB_EPS_FIXED && !(cfg->eps_value >= 0))
    return fail(RGB_E_INVALID, "fixed eps requires a nonnegative value");
  return RGB_OK;
}

static int check_state(const rgb_config* cfg, const rgb_state* st) {
  if (!st) return fail(RGB_E_INVALID, "null state");
  if (!st->basis || !st->gram_inv || !st->x || !st->rank || !st->nobs || !st->status)
    return fail(RGB_E_INVALID, "null state buffer");
  if (cfg->variant != RGB_ORTHONORMAL && !st->dual) return fail(RGB_E_INVALID, "null dual buffer");
  return RGB_OK;
}

static bool env_flag(const char* name) {
  const char* v = getenv(name);
  return v && v[0] && strcmp(v, "0") != 0;
}

static int sm_count() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (!cache[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 148;
  }
  return cache[dev];
}

extern "C" {

int rgb_abi_version(void) { return RGB_ABI_VERSION; }

const char* rgb_last_error(void) { return g_err; }

int rgb_state_reset(const rgb_config* cfg, rgb_state* st, void* stream) {
  int rc = check_cfg(cfg);
  if (rc) return rc;
  if ((rc = check_state(cfg, st))) return rc;
  g_err[0] = 0;
  cudaStream_t s = (cudaStream_t)stream;
  size_t es = cfg->dtype == RGB_F32 ? 4 : 8;
  size_t B = (size_t)cfg->num_streams;
  size_t fac = B * cfg->r_cap * cfg->m * es;
  cudaError_t e = cudaMemsetAsync(st->basis, 0, fac, s);
  if (e == cudaSuccess && st->dual && st->dual != st->basis) e = cudaMemsetAsync(st->dual, 0, fac, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(st->gram_inv, 0, B * cfg->r_cap * cfg->r_cap * es, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(st->x, 0, B * cfg->k * cfg->m * es, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(st->rank, 0, B * sizeof(int32_t), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(st->nobs, 0, B * sizeof(int64_t), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(st->status, 0, B * sizeof(int32_t), s);
  return e == cudaSuccess ? RGB_OK : cuda_fail(e, "rgb_state_reset");
}

static int ingest_impl(const rgb_config* cfg, rgb_state* st, const void* rows, int64_t rows_stride,
                       const void* targets, int64_t targets_stride, int64_t T, const rgb_logs* logs,
                       void* stream, bool f32in) {
  int rc = check_cfg(cfg);
  if (rc) return rc;
  if ((rc = check_state(cfg, st))) return rc;
  if (T < 0) return fail(RGB_E_INVALID, "negative row count");
  if (T == 0 || cfg->num_streams == 0) return RGB_OK;
  if (!rows || !targets) return fail(RGB_E_INVALID, "null rows or targets");
  if (rows_stride == 0) rows_stride = T * cfg->m;
  if (targets_stride == 0) targets_stride = T * cfg->k;
  if (rows_stride < T * cfg->m || targets_stride < T * cfg->k)
    return fail(RGB_E_INVALID, "stride smaller than one stream's block");
  g_err[0] = 0;
  rgb_logs lg;
  memset(&lg, 0, sizeof(lg));
  if (logs) lg = *logs;
  rgb_state s2 = *st;
  if (cfg->variant == RGB_ORTHONORMAL) s2.dual = s2.basis;  // C~ is C (solver.py:168, 386)
  cudaStream_t s = (cudaStream_t)stream;
  const int nsm = sm_count();
  if (cfg->dtype == RGB_F32) f32in = false;  // the inputs already have the state's type
  rc = RGB_E_UNSUPPORTED;
  if (rgb::f32_supports(*cfg) && !lg.resid && !lg.gain && !env_flag("RGB_NO_F32K"))
    rc = rgb::launch_f32(*cfg, s2, rows, rows_stride, targets, targets_stride, T, lg, s, nsm);
  if (rc != RGB_E_UNSUPPORTED) {
  } else if (rgb::blocked_supports(*cfg) && !lg.resid && !lg.gain)
    rc = rgb::launch_blocked(*cfg, s2, rows, rows_stride, targets, targets_stride, T, lg, s, nsm, f32in);
  else if (rgb::panel_supports(*cfg) && !lg.resid && !lg.gain && !env_flag("RGB_NO_PANEL"))
    rc = rgb::launch_panel(*cfg, s2, rows, rows_stride, targets, targets_stride, T, lg, s, nsm, f32in);
  else if (rgb::blocked_wg_supports(*cfg) && !lg.resid && !lg.gain)
    rc = rgb::launch_blocked_wg(*cfg, s2, rows, rows_stride, targets, targets_stride, T, lg, s, nsm, f32in);
  // the multi-SM kernels pay microseconds of setup and barriers per call: a
  // call of a few rows (a per-row update()) is faster on the generic kernel
  else if (rgb::cluster_supports(*cfg) && T >= 8 && !lg.resid && !lg.gain)
    rc = rgb::launch_cluster(*cfg, s2, rows, rows_stride, targets, targets_stride, T, lg, s, nsm, f32in);
  if (rc == RGB_E_UNSUPPORTED && rgb::grid_supports(*cfg) && T >= 8 && !lg.resid && !lg.gain)
    rc = rgb::launch_grid(*cfg, s2, rows, rows_stride, targets, targets_stride, T, lg, s, nsm, f32in);
  if (rc == RGB_E_UNSUPPORTED)
    rc = rgb::launch_generic(*cfg, s2, rows, rows_stride, targets, targets_stride, T, lg, s, nsm, f32in);
  if (rc == RGB_E_UNSUPPORTED) return fail(rc, "shape beyond kernel limits (k <= 64, smem)");
  if (rc == RGB_E_CUDA) return cuda_fail(cudaGetLastError(), "rgb_ingest launch");
  return rc;
}

int rgb_ingest(const rgb_config* cfg, rgb_state* st, const void* rows, int64_t rows_stride,
               const void* targets, int64_t targets_stride, int64_t T, const rgb_logs* logs,
               void* stream) {
  return ingest_impl(cfg, st, rows, rows_stride, targets, targets_stride, T, logs, stream, false);
}

int rgb_ingest_f32in(const rgb_config* cfg, rgb_state* st, const float* rows, int64_t rows_stride,
                     const float* targets, int64_t targets_stride, int64_t T, const rgb_logs* logs,
                     void* stream) {
  return ingest_impl(cfg, st, rows, rows_stride, targets, targets_stride, T, logs, stream, true);
}

int rgb_project(const rgb_config* cfg, const rgb_state* st, const void* rows, void* coords,
                void* rejection, void* rej_sq, uint8_t* dependent, void* stream) {
  int rc = check_cfg(cfg);
  if (rc) return rc;
  if ((rc = check_state(cfg, st))) return rc;
  if (!rows) return fail(RGB_E_INVALID, "null rows");
  g_err[0] = 0;
  rgb_state s2 = *st;
  if (cfg->variant == RGB_ORTHONORMAL) s2.dual = s2.basis;
  rc = rgb::launch_project(*cfg, s2, rows, coords, rejection, rej_sq, dependent, (cudaStream_t)stream);
  if (rc == RGB_E_CUDA) return cuda_fail(cudaGetLastError(), "rgb_project launch");
  if (rc) return fail(rc, "rgb_project: unsupported shape");
  return RGB_OK;
}

int rgb_pinv(const rgb_config* cfg, const rgb_state* st, const void* coords, int64_t n, void* out,
             void* stream) {
  int rc = check_cfg(cfg);
  if (rc) return rc;
  if ((rc = check_state(cfg, st))) return rc;
  if (n < 0) return fail(RGB_E_INVALID, "negative observation count");
  if (!out || (n > 0 && !coords)) return fail(RGB_E_INVALID, "null coords or output");
  if (n == 0 || cfg->num_streams == 0) return RGB_OK;
  g_err[0] = 0;
  rgb_state s2 = *st;
  if (cfg->variant == RGB_ORTHONORMAL) s2.dual = s2.basis;
  rc = rgb::launch_pinv(*cfg, s2, coords, n, out, (cudaStream_t)stream);
  if (rc == RGB_E_CUDA) return cuda_fail(cudaGetLastError(), "rgb_pinv launch");
  if (rc) return fail(rc, "rgb_pinv: unsupported shape");
  return RGB_OK;
}

int rgb_memcpy_async(void* dst, const void* src, int64_t bytes, void* stream) {
  if (bytes < 0 || (bytes > 0 && (!dst || !src))) return fail(RGB_E_INVALID, "rgb_memcpy_async: bad arguments");
  if (bytes == 0) return RGB_OK;
  const cudaError_t e = cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault, (cudaStream_t)stream);
  return e == cudaSuccess ? RGB_OK : cuda_fail(e, "rgb_memcpy_async");
}

int rgb_covariance(const rgb_config* cfg, const rgb_state* st, void* out, void* stream) {
  int rc = check_cfg(cfg);
  if (rc) return rc;
  if ((rc = check_state(cfg, st))) return rc;
  if (!out) return fail(RGB_E_INVALID, "null output");
  if (cfg->num_streams == 0) return RGB_OK;
  g_err[0] = 0;
  rgb_state s2 = *st;
  if (cfg->variant == RGB_ORTHONORMAL) s2.dual = s2.basis;
  rc = rgb::launch_covariance(*cfg, s2, out, (cudaStream_t)stream);
  if (rc == RGB_E_CUDA) return cuda_fail(cudaGetLastError(), "rgb_covariance launch");
  if (rc) return fail(rc, "rgb_covariance: unsupported shape");
  return RGB_OK;
}

}  // extern "C"
