/*
 * rgb_oracle.c -- CPU restatement of the rank-Greville recursive least-squares
 * update of rankrls 0.1.0 (arXiv 2106.11594, Algorithm 1).
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path and the CPU baseline timed by bench.py (`cpu_baseline`, `--impl
 * reference`).  Nothing under paper_2106_11594_b200/ links or calls it.
 *
 * Every function follows the reference's operation sequence, citing
 * /root/reference/pkg/src/rankrls/<file>:<line>:
 *   - the per-row loop of RecursiveSolver.ingest            solver.py:276-319
 *   - the auto threshold (m^2 r + m r + m) eps_M            solver.py:66-72, 292-296
 *   - the dependent branch (Sherman-Morrison on P^-1)       solver.py:297-304
 *   - the independent branch, _grow for all three variants  solver.py:305-318, 347-397
 *   - the a-priori residual and solution update             solver.py:303-304, 316-318
 * Arithmetic is IEEE float64 (or float32 for the fp32 mode, which the
 * reference does not have), compiled with -ffp-contract=off so that every
 * product and sum is rounded separately, as numpy does.  Dot products run in
 * index order; OpenBLAS sums in a different order, so the restatement matches
 * the reference to rounding (pinned in tests/test_oracle.py against golden
 * vectors produced by the reference itself), not bit for bit.
 *
 * State layout (identical to the CUDA library, include/rgb.h):
 *   C  [r_cap][m]       basis rows (solver._basis)
 *   D  [r_cap][m]       dual basis rows (solver._dual); for the orthonormal
 *                       variant D aliases C exactly as solver.py:168,386
 *   P  [r_cap][r_cap]   inverse Gram factor (solver._gram_inv)
 *   X  [k][m]           one solution column per right-hand side (solver._x)
 * Multi-RHS: the k targets share every factor update; only x differs
 * (targets never influence C, D, P -- solver.py:247-248).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_GENERAL 0
#define ORC_ORTHOGONAL 1
#define ORC_ORTHONORMAL 2
#define ORC_EPS_AUTO 0
#define ORC_EPS_FIXED 1

#define ORC_ST_RANK_CAP 1
#define ORC_ST_NONFINITE 2
#define ORC_ST_BAD_ALPHA 4

typedef struct {
  int32_t m, k, r_cap, variant, eps_mode;
  int32_t pad;
  double eps_value, alpha;
} orc_cfg;

#define DEFINE_INGEST(NAME, REAL, EPS_M, SQRT)                                   \
  long long NAME(const orc_cfg *cfg, REAL *C, REAL *D, REAL *P, REAL *X,         \
                 int32_t *rank, int64_t *nobs, int32_t *status, const REAL *rows, \
                 const REAL *targets, long long T, uint8_t *branch_log,          \
                 REAL *coords_log, REAL *resid_log, double *rho_log) {           \
    const int m = cfg->m, k = cfg->k, rc = cfg->r_cap, var = cfg->variant;       \
    REAL *coords = (REAL *)malloc(sizeof(REAL) * (rc + 1));                      \
    REAL *z = (REAL *)malloc(sizeof(REAL) * (rc + 1));                           \
    REAL *zs = (REAL *)malloc(sizeof(REAL) * (rc + 1));                          \
    REAL *rej = (REAL *)malloc(sizeof(REAL) * m);                                \
    REAL *gain = (REAL *)malloc(sizeof(REAL) * m);                               \
    REAL *dy = (REAL *)malloc(sizeof(REAL) * (k > 0 ? k : 1));                   \
    if (var == ORC_ORTHONORMAL) D = C;                                           \
    long long t;                                                                 \
    for (t = 0; t < T; ++t) {                                                    \
      const REAL *a = rows + (size_t)t * m;                                      \
      const REAL *y = targets + (size_t)t * k;                                   \
      int r = *rank;                                                             \
      /* solver.py:267 -- squared row norm */                                    \
      REAL row_sq = 0;                                                           \
      for (int j = 0; j < m; ++j) row_sq = row_sq + a[j] * a[j];                 \
      /* solver.py:285-291 -- coords = D a, rej = a - C^T coords */              \
      for (int i = 0; i < r; ++i) {                                              \
        REAL s = 0;                                                              \
        const REAL *d = D + (size_t)i * m;                                       \
        for (int j = 0; j < m; ++j) s = s + d[j] * a[j];                         \
        coords[i] = s;                                                           \
      }                                                                          \
      for (int j = 0; j < m; ++j) {                                              \
        REAL s = 0;                                                              \
        for (int i = 0; i < r; ++i) s = s + coords[i] * C[(size_t)i * m + j];    \
        rej[j] = r ? a[j] - s : a[j];                                            \
      }                                                                          \
      REAL rej_sq = 0;                                                           \
      for (int j = 0; j < m; ++j) rej_sq = rej_sq + rej[j] * rej[j];             \
      /* solver.py:292-296 -- threshold test */                                  \
      REAL eps;                                                                  \
      if (cfg->eps_mode == ORC_EPS_FIXED)                                        \
        eps = (REAL)cfg->eps_value;                                              \
      else                                                                       \
        eps = (REAL)((double)((long long)m * m * r + (long long)m * r + m)) *    \
              (REAL)(EPS_M);                                                     \
      REAL eps_sq = eps * eps;                                                   \
      int dependent = (rej_sq < eps_sq) || (rej_sq < eps_sq * row_sq);           \
      if (rho_log) {                                                             \
        REAL thr = eps_sq > eps_sq * row_sq ? eps_sq : eps_sq * row_sq;          \
        rho_log[t] = thr > 0 ? sqrt((double)rej_sq / (double)thr) : INFINITY;    \
      }                                                                          \
      /* solver.py:303 -- a priori residual, computed before x moves */          \
      for (int c = 0; c < k; ++c) {                                              \
        REAL s = 0;                                                              \
        const REAL *xc = X + (size_t)c * m;                                      \
        for (int j = 0; j < m; ++j) s = s + a[j] * xc[j];                        \
        dy[c] = y[c] - s;                                                        \
      }                                                                          \
      if (coords_log) {                                                          \
        REAL *cl = coords_log + (size_t)t * rc;                                  \
        for (int i = 0; i < rc; ++i) cl[i] = i < r ? coords[i] : (REAL)0;        \
      }                                                                          \
      if (resid_log)                                                             \
        for (int c = 0; c < k; ++c) resid_log[(size_t)t * k + c] = dy[c];        \
      if (dependent) {                                                           \
        if (branch_log) branch_log[t] = 0;                                       \
        if (r) {                                                                 \
          /* solver.py:298-304 -- Sherman-Morrison and gain = zs^T D */          \
          for (int i = 0; i < r; ++i) {                                          \
            REAL s = 0;                                                          \
            for (int l = 0; l < r; ++l) s = s + P[(size_t)i * rc + l] * coords[l]; \
            z[i] = s;                                                            \
          }                                                                      \
          REAL cz = 0;                                                           \
          for (int i = 0; i < r; ++i) cz = cz + coords[i] * z[i];                \
          REAL denom = (REAL)1.0 + cz;                                           \
          for (int i = 0; i < r; ++i) zs[i] = z[i] / denom;                      \
          for (int i = 0; i < r; ++i)                                            \
            for (int l = 0; l < r; ++l)                                          \
              P[(size_t)i * rc + l] = P[(size_t)i * rc + l] - z[i] * zs[l];      \
          for (int j = 0; j < m; ++j) {                                          \
            REAL s = 0;                                                          \
            for (int i = 0; i < r; ++i) s = s + zs[i] * D[(size_t)i * m + j];    \
            gain[j] = s;                                                         \
          }                                                                      \
          for (int c = 0; c < k; ++c) {                                          \
            REAL *xc = X + (size_t)c * m;                                        \
            for (int j = 0; j < m; ++j) {                                        \
              REAL g = gain[j] * dy[c];                                          \
              xc[j] = xc[j] + g;                                                 \
            }                                                                    \
          }                                                                      \
        }                                                                        \
      } else {                                                                   \
        if (branch_log) branch_log[t] = 1;                                       \
        if (r >= rc) { /* capacity: the CUDA path flags and freezes the stream */ \
          *status |= ORC_ST_RANK_CAP;                                            \
          break;                                                                 \
        }                                                                        \
        /* solver.py:334-345, 368-397 -- grow the factorization */               \
        for (int j = 0; j < m; ++j) gain[j] = rej[j] / rej_sq;                   \
        if (var == ORC_GENERAL) {                                                \
          for (int i = 0; i < r; ++i)                                            \
            for (int j = 0; j < m; ++j)                                          \
              D[(size_t)i * m + j] = D[(size_t)i * m + j] - coords[i] * gain[j]; \
          for (int j = 0; j < m; ++j) {                                          \
            D[(size_t)r * m + j] = gain[j];                                      \
            C[(size_t)r * m + j] = a[j];                                         \
          }                                                                      \
          for (int i = 0; i < r; ++i) {                                          \
            P[(size_t)i * rc + r] = 0;                                           \
            P[(size_t)r * rc + i] = 0;                                           \
          }                                                                      \
          P[(size_t)r * rc + r] = 1;                                             \
        } else {                                                                 \
          REAL denom = 1;                                                        \
          if (r) {                                                               \
            for (int i = 0; i < r; ++i) {                                        \
              REAL s = 0;                                                        \
              for (int l = 0; l < r; ++l) s = s + P[(size_t)i * rc + l] * coords[l]; \
              z[i] = s;                                                          \
            }                                                                    \
            REAL cz = 0;                                                         \
            for (int i = 0; i < r; ++i) cz = cz + coords[i] * z[i];              \
            denom = (REAL)1.0 + cz;                                              \
          }                                                                      \
          REAL rescale;                                                          \
          if (var == ORC_ORTHONORMAL) {                                          \
            REAL norm = SQRT(rej_sq);                                            \
            rescale = (REAL)1.0 / norm;                                          \
          } else {                                                               \
            rescale = (REAL)cfg->alpha;                                          \
            if (rescale == 0) { *status |= ORC_ST_BAD_ALPHA; break; }            \
          }                                                                      \
          REAL last = (REAL)1.0 / rescale;   /* coords_row[r], solver.py:354 */  \
          REAL alpha = (REAL)1.0 / last;     /* solver.py:383 */                 \
          for (int j = 0; j < m; ++j) C[(size_t)r * m + j] = alpha * rej[j];     \
          if (var == ORC_ORTHOGONAL) {                                           \
            REAL sc = alpha * rej_sq;                                            \
            for (int j = 0; j < m; ++j) D[(size_t)r * m + j] = rej[j] / sc;      \
          }                                                                      \
          for (int i = 0; i < r; ++i) {                                          \
            REAL edge = -(alpha * z[i]);                                         \
            P[(size_t)i * rc + r] = edge;                                        \
            P[(size_t)r * rc + i] = edge;                                        \
          }                                                                      \
          P[(size_t)r * rc + r] = alpha * alpha * denom;                         \
          if (coords_log) coords_log[(size_t)t * rc + r] = last;                 \
        }                                                                        \
        if (var == ORC_GENERAL && coords_log) {                                  \
          REAL *cl = coords_log + (size_t)t * rc;                                \
          for (int i = 0; i < rc; ++i) cl[i] = 0;                                \
          cl[r] = 1;                                                             \
        }                                                                        \
        *rank = r + 1;                                                           \
        /* solver.py:316-318 */                                                  \
        for (int c = 0; c < k; ++c) {                                            \
          REAL *xc = X + (size_t)c * m;                                          \
          for (int j = 0; j < m; ++j) {                                          \
            REAL g = gain[j] * dy[c];                                            \
            xc[j] = xc[j] + g;                                                   \
          }                                                                      \
        }                                                                        \
      }                                                                          \
      *nobs += 1;                                                                \
    }                                                                            \
    free(coords); free(z); free(zs); free(rej); free(gain); free(dy);            \
    return t;                                                                    \
  }

DEFINE_INGEST(orc_ingest_f64, double, 2.220446049250313e-16, sqrt)
DEFINE_INGEST(orc_ingest_f32, float, 1.1920928955078125e-07f, sqrtf)

/* ---- batched driver: B independent streams over a pthread pool ------------- */

typedef struct {
  const orc_cfg *cfg;
  int is_f32;
  long long b0, b1;
  char *C, *D, *P, *X;
  int32_t *rank;
  int64_t *nobs;
  int32_t *status;
  const char *rows, *targets;
  long long T;
  uint8_t *branch_log;
  char *coords_log;
  char *resid_log;
  double *rho_log;
} orc_job;

static void *orc_worker(void *arg) {
  orc_job *j = (orc_job *)arg;
  const orc_cfg *c = j->cfg;
  size_t s = j->is_f32 ? 4 : 8;
  size_t fm = (size_t)c->r_cap * c->m, pm = (size_t)c->r_cap * c->r_cap, xm = (size_t)c->k * c->m;
  for (long long b = j->b0; b < j->b1; ++b) {
    char *Cb = j->C + b * fm * s, *Db = j->D + b * fm * s;
    char *Pb = j->P + b * pm * s, *Xb = j->X + b * xm * s;
    const char *Rb = j->rows + (size_t)b * j->T * c->m * s;
    const char *Yb = j->targets + (size_t)b * j->T * c->k * s;
    uint8_t *bl = j->branch_log ? j->branch_log + (size_t)b * j->T : NULL;
    char *cl = j->coords_log ? j->coords_log + (size_t)b * j->T * c->r_cap * s : NULL;
    char *rl = j->resid_log ? j->resid_log + (size_t)b * j->T * c->k * s : NULL;
    double *hl = j->rho_log ? j->rho_log + (size_t)b * j->T : NULL;
    if (j->is_f32)
      orc_ingest_f32(c, (float *)Cb, (float *)Db, (float *)Pb, (float *)Xb, j->rank + b, j->nobs + b,
                     j->status + b, (const float *)Rb, (const float *)Yb, j->T, bl, (float *)cl,
                     (float *)rl, hl);
    else
      orc_ingest_f64(c, (double *)Cb, (double *)Db, (double *)Pb, (double *)Xb, j->rank + b,
                     j->nobs + b, j->status + b, (const double *)Rb, (const double *)Yb, j->T, bl,
                     (double *)cl, (double *)rl, hl);
  }
  return NULL;
}

/* Streams b in [0, B): state arrays are [B][...] in the layout above, rows are
 * [B][T][m], targets [B][T][k]; optional logs are [B][T], [B][T][r_cap],
 * [B][T][k], [B][T].  Returns 0. */
int orc_ingest_batch(const orc_cfg *cfg, int is_f32, long long B, void *C, void *D, void *P, void *X,
                     int32_t *rank, int64_t *nobs, int32_t *status, const void *rows,
                     const void *targets, long long T, uint8_t *branch_log, void *coords_log,
                     void *resid_log, double *rho_log, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > B) nthreads = (int)(B > 0 ? B : 1);
  pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * nthreads);
  orc_job *jobs = (orc_job *)malloc(sizeof(orc_job) * nthreads);
  for (int w = 0; w < nthreads; ++w) {
    orc_job *j = jobs + w;
    j->cfg = cfg; j->is_f32 = is_f32;
    j->b0 = B * w / nthreads; j->b1 = B * (w + 1) / nthreads;
    j->C = (char *)C; j->D = (char *)D; j->P = (char *)P; j->X = (char *)X;
    j->rank = rank; j->nobs = nobs; j->status = status;
    j->rows = (const char *)rows; j->targets = (const char *)targets; j->T = T;
    j->branch_log = branch_log; j->coords_log = (char *)coords_log;
    j->resid_log = (char *)resid_log; j->rho_log = rho_log;
    if (nthreads == 1) orc_worker(j);
    else pthread_create(th + w, NULL, orc_worker, j);
  }
  if (nthreads > 1)
    for (int w = 0; w < nthreads; ++w) pthread_join(th[w], NULL);
  free(th); free(jobs);
  return 0;
}
