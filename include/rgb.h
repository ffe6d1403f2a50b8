/*
 * rgb.h -- C ABI of the B200-native rank-Greville recursive least-squares
 * library (librgb.so).  arXiv 2106.11594, Algorithm 1.
 *
 * Plain C: raw device pointers, sizes and a cudaStream_t passed as void*.
 * The caller owns every state and input buffer (allocate with cudaMalloc,
 * torch, cupy ...); the library keeps no state between calls except a
 * thread-local error string, stream-ordered scratch from a library-owned
 * device memory pool (grid kernel, A+ / covariance), and the row pipes the
 * caller creates and destroys explicitly.  Every call is asynchronous on
 * `stream` except rgb_rowpipe_run, which returns with the row folded.
 * Calls on one state must be stream-ordered (single writer, as SPEC.md:197);
 * distinct states may run concurrently on different streams or GPUs.
 *
 * Each entry point names the reference interface it replaces
 * (/root/reference/pkg/src/rankrls/<file>:<line>); INTEGRATION.md shows the
 * ctypes binding a maintainer of the reference would add.
 */
#ifndef RGB_H_
#define RGB_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RGB_ABI_VERSION 4

/* scalar kinds: scalars.py:141-147 (FLOAT64); FLOAT32 is a new kind */
enum { RGB_F64 = 0, RGB_F32 = 1 };
/* basis flavours: solver.py:29 VARIANTS */
enum { RGB_GENERAL = 0, RGB_ORTHOGONAL = 1, RGB_ORTHONORMAL = 2 };
/* EpsPolicy modes usable with floats: solver.py:32-72 ("exact" is rational-only) */
enum { RGB_EPS_AUTO = 0, RGB_EPS_FIXED = 1 };

/* return codes */
enum {
  RGB_OK = 0,
  RGB_E_INVALID = -1,     /* bad argument: maps to ValueError (solver.py:142-158) */
  RGB_E_UNSUPPORTED = -2, /* shape beyond kernel limits */
  RGB_E_CUDA = -3         /* CUDA launch or runtime failure */
};

/* per-stream status bits (the stream is frozen once one is set) */
enum {
  RGB_ST_RANK_CAP = 1,  /* an independent row arrived with rank == r_cap */
  RGB_ST_NONFINITE = 2, /* NaN/Inf row or target (scalars.py:122-123 raises) */
  RGB_ST_BAD_ALPHA = 4  /* orthogonal rescaling factor zero (solver.py:364-365) */
};

/* Constructor arguments of RecursiveSolver (solver.py:140-141), batched:
 * num_streams independent solvers of m regressors sharing one shape, each
 * with k right-hand sides. */
typedef struct rgb_config {
  int64_t num_streams; /* B */
  int32_t m;           /* num_regressors */
  int32_t k;           /* right-hand sides per stream (reference: 1) */
  int32_t r_cap;       /* stored-rank capacity; the reference grows unbounded */
  int32_t dtype;       /* RGB_F64 / RGB_F32 */
  int32_t variant;     /* RGB_GENERAL / RGB_ORTHOGONAL / RGB_ORTHONORMAL */
  int32_t eps_mode;    /* RGB_EPS_AUTO / RGB_EPS_FIXED */
  double eps_value;    /* EpsPolicy.fixed(value) */
  double alpha;        /* orthogonal rescaling constant (solver.py:362) */
} rgb_config;

/* Solver state (solver.py:164-171), device pointers, row-major:
 *   basis    [B][r_cap][m]      C       (solver._basis)
 *   dual     [B][r_cap][m]      C~      (solver._dual; == basis for orthonormal)
 *   gram_inv [B][r_cap][r_cap]  P^-1    (solver._gram_inv)
 *   x        [B][k][m]          one solution per right-hand side (solver._x)
 *   rank [B] int32, nobs [B] int64, status [B] int32
 * Rows/columns beyond the current rank must be zero (rgb_state_reset). */
typedef struct rgb_state {
  void *basis;
  void *dual;
  void *gram_inv;
  void *x;
  int32_t *rank;
  int64_t *nobs;
  int32_t *status;
} rgb_state;

/* Optional per-row outputs of rgb_ingest; NULL members are not written. */
typedef struct rgb_logs {
  uint8_t *branch; /* [B][T]: 1 independent, 0 dependent (UpdateReport.branch, solver.py:84-91) */
  void *coords;    /* [B][T][r_cap]: coordinate-factor row (_UpdateStep.coords_row, solver.py:94-109,
                      the rows of B in A = B C, tracking.py:54-74), zero padded */
  void *resid;     /* [B][T][k]: a-priori residual y - a.x (UpdateReport.predicted_residual) */
  void *gain;      /* [B][m]: gain of the last ingested row (UpdateReport.gain) */
} rgb_logs;

/* Library ABI version (RGB_ABI_VERSION). */
int rgb_abi_version(void);

/* Message of the last failing call on this thread ("" if none). */
const char *rgb_last_error(void);

/* Empty solver state: RecursiveSolver.__init__ (solver.py:160-171) for all B
 * streams -- zero factors and solutions, rank 0, nobs 0, status 0. */
int rgb_state_reset(const rgb_config *cfg, rgb_state *state, void *stream);

/* Fold T rows into every stream:
 *   rows    : stream b's rows start at rows + b * rows_stride (elements),
 *             T rows of m contiguous values (rows_stride 0 means T*m);
 *   targets : stream b's targets at targets + b * targets_stride, T x k
 *             (targets_stride 0 means T*k).
 * Replaces RecursiveSolver.ingest (solver.py:252-319) and, with T = 1,
 * RecursiveSolver.update (solver.py:231-250); solve_batch (solver.py:406-422)
 * is reset + ingest.  Branch decisions use the reference's rank test
 * (solver.py:292-296).  Streams whose status is nonzero are skipped.  The kernel
 * is chosen from the shape (rgb_abi.cu); the environment variable RGB_NO_PANEL=1
 * turns off the panel kernel (m 128 / 256; A/B runs and tests; results agree within
 * the fp64 parity bar, not bitwise, since the summation orders differ). */
int rgb_ingest(const rgb_config *cfg, rgb_state *state, const void *rows, int64_t rows_stride,
               const void *targets, int64_t targets_stride, int64_t T, const rgb_logs *logs,
               void *stream);

/* rgb_ingest with single-precision rows and targets (same layout and strides,
 * in float elements) folded into a state of cfg->dtype.  Every input value is
 * widened exactly on load, so with an RGB_F64 state the result is identical to
 * rgb_ingest on the widened inputs -- fp64 state and arithmetic, fp64 parity --
 * while the input stream (HBM reads, host-link copies) halves.  With an RGB_F32
 * state it is rgb_ingest.  No reference counterpart (the reference has no fp32
 * kind, scalars.py:121); it serves the fp32 inputs of config 5. */
int rgb_ingest_f32in(const rgb_config *cfg, rgb_state *state, const float *rows, int64_t rows_stride,
                     const float *targets, int64_t targets_stride, int64_t T, const rgb_logs *logs,
                     void *stream);

/* RecursiveSolver.project + is_dependent (solver.py:210-229) for one row per
 * stream: coords [B][r_cap] (zero padded), rejection [B][m], rej_sq [B],
 * dependent [B] (uint8).  Any output pointer may be NULL. */
int rgb_project(const rgb_config *cfg, const rgb_state *state, const void *rows, void *coords,
                void *rejection, void *rej_sq, uint8_t *dependent, void *stream);

/* Pseudoinverse from the factors (PseudoinverseTracker.pinv, tracking.py:19-85;
 * closed form A+ = C~^T P^-1 B^T):
 *   coords : [B][n][r_cap] coordinate-factor log written by rgb_ingest,
 *   out    : [B][m][n].  Uses the current rank of each stream. */
int rgb_pinv(const rgb_config *cfg, const rgb_state *state, const void *coords, int64_t n,
             void *out, void *stream);

/* Asynchronous copy of `bytes` between host (pinned) and device memory on the
 * stream (direction inferred from the unified address space), for FFI callers
 * that stage rows and read results without a CUDA runtime binding of their own
 * -- the drop-in solver's per-row update() path uses it. */
int rgb_memcpy_async(void *dst, const void *src, int64_t bytes, void *stream);

/* Covariance V = A+ A+^T = C~^T P^-1 C~ (CovarianceTracker.covariance,
 * tracking.py:88-119; identity of test_tracking.py:188-198): out [B][m][m]. */
int rgb_covariance(const rgb_config *cfg, const rgb_state *state, void *out, void *stream);

/* ---- low-latency one-row pipe (the drop-in per-row API) -------------------
 * RecursiveSolver.update (solver.py:231-250) and a one-row ingest are latency
 * bound.  A row pipe belongs to ONE stream's state (num_streams == 1) and owns
 * a pinned, device-mapped host block and a CUDA graph: the shape-generic
 * kernel reads the row (m values) and targets (k values) from the block's
 * input area and writes the report into it; the counters follow, then a
 * sequence word.  rgb_rowpipe_run launches the graph on `stream` and returns
 * once the report is visible (it spins on the sequence word; no stream
 * synchronisation).  Recreate the pipe when the state buffers move (capacity
 * growth).  Block layout (bytes): header of RGB_ROWPIPE_HEADER -- sequence
 * u64 @0, nobs i64 @8, rank i32 @16, status i32 @20, branch u8 @24 (1 =
 * independent) -- then the areas whose offsets rgb_rowpipe_layout returns:
 * input (row then targets, float when f32in or an RGB_F32 state, else
 * double), a-priori residuals [k] and gain [m] (the state's type). */
#define RGB_ROWPIPE_HEADER 64
#define RGB_ROWPIPE_OFF_SEQ 0
#define RGB_ROWPIPE_OFF_NOBS 8
#define RGB_ROWPIPE_OFF_RANK 16
#define RGB_ROWPIPE_OFF_STATUS 20
#define RGB_ROWPIPE_OFF_BRANCH 24
#define RGB_ROWPIPE_OFF_REQ 32  /* u64: row server request (the row number), written by rgb_rowpipe_run */
#define RGB_ROWPIPE_OFF_STOP 40 /* u32: row server stop word, written by rgb_rowpipe_quiesce */
#define RGB_ROWPIPE_OFF_PREQ 48 /* u64: projection request number, written by rgb_rowpipe_project */
#define RGB_ROWPIPE_OFF_PSEQ 56 /* u64: the projection last served (written by the server) */
typedef struct rgb_rowpipe rgb_rowpipe;

/* Size of a row pipe's host block (bytes) and the offsets of its areas. */
int64_t rgb_rowpipe_layout(const rgb_config *cfg, int f32in, int64_t *off_in, int64_t *off_resid,
                           int64_t *off_gain);
/* Capture the pipe for `state` (report logs when want_report); *host_block
 * receives the block the caller fills and reads.  host_x (optional, pinned
 * host memory of m values of the state's type, cudaHostAlloc) receives the
 * solution of the first right-hand side after every run -- the drop-in's
 * live `solution` view (solver.py:200-202). */
int rgb_rowpipe_create(const rgb_config *cfg, const rgb_state *state, int want_report, int f32in,
                       void *host_x, rgb_rowpipe **pipe, void **host_block);
/* Fold the row staged in the block; blocks until its report is visible.
 * Where the one-row kernel applies (the state fits its shared memory) the row
 * goes to a ROW SERVER: a one-CTA persistent kernel on the pipe's own stream
 * that keeps the state in shared memory, polls the block for requests and
 * exits after RGB_ROWSERVE_IDLE_US microseconds without one (environment, read
 * at create; default 500, 0 = one graph launch per row).  It is launched on
 * demand, ordered after the work already on `stream`. */
int rgb_rowpipe_run(rgb_rowpipe *pipe, void *stream);
/* Project the row staged in the block's input area on the current basis
 * (RecursiveSolver.project, solver.py:210-219) through the row server, without
 * touching the state: coords [r_cap] (zero past the rank), rejection [m] and
 * |rejection|^2 (the state's type) at rgb_rowpipe_proj_offset.  Blocks until they
 * are visible; RGB_E_UNSUPPORTED when the pipe has no row server. */
int rgb_rowpipe_project(rgb_rowpipe *pipe, void *stream);
int64_t rgb_rowpipe_proj_offset(const rgb_config *cfg, int f32in);
/* Stop the pipe's row server (if it runs) and wait for it: call before any
 * other kernel writes the state (an ingest of several rows, a reset).
 * rgb_rowpipe_destroy stops it too. */
int rgb_rowpipe_quiesce(rgb_rowpipe *pipe);
void rgb_rowpipe_destroy(rgb_rowpipe *pipe);

#ifdef __cplusplus
}
#endif

#endif /* RGB_H_ */
