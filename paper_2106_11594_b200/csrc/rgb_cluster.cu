// rgb_cluster.cu -- one large stream per thread-block cluster (sm_100a: DSMEM,
// hardware cluster barriers, fp64 tensor cores), in k-row panels.
//
// For a stream whose factors are too large for one SM but fit one cluster
// (config 2: m 1024, r 64 -- C~ and C are 1 MB) the stream's columns are split
// over NCL = m / 64 CTAs of one cluster (16 on config 2, the non-portable
// maximum).  CTA c holds columns [64c, 64c + 64) of C~ and C in shared memory
// (MMA fragment order); CTA 0 ("home") also holds P^-1 and W.  Per panel of TT
// rows (TT = 32: the north star's blocked k = 32-row variant):
//
//   P1  G_c = A[:, cols] C~[:, cols]^T (+ a.x0 as 8 extra rows of C~)    own smem
//   --- cluster barrier
//   P2  G = sum_c G_c: CTA c reduces a 1/NCL chunk from every CTA's smem
//       (DSMEM loads, fixed order) and stores it into every CTA's smem
//   --- cluster barrier
//   P3  R[:, cols] = A - G C[:, cols]; |R_t|^2, |a_t|^2 partials stored into
//       every CTA's smem
//   --- cluster barrier
//   P4  the rank test (every CTA, identical sums); home folds the dependent
//       rows into P^-1 and W (LDL^T-factored Sherman-Morrison, 8-row blocks,
//       solver.py:297-304) while the other CTAs go on to the next panel
//
// An independent row (solver.py:305-318, _grow solver.py:368-397) is applied
// by every CTA to its own columns -- gamma, the rejection and |rej|^2 are all
// local after P3 -- and by home to P^-1 and W; the rest of its panel is
// re-projected.  Three hardware cluster barriers per panel replace the five
// global-memory grid barriers per 8 rows of rgb_grid.cu.
#include <cooperative_groups.h>

#include "rgb_mma.cuh"

namespace cg = cooperative_groups;

namespace rgb {
namespace cls {

using blk::FULL;
using blk::mma;
using blk::rcp64;

constexpr int NT = 256;  // threads per CTA (8 warps)
constexpr int NW = NT / 32;
constexpr int CW = 64;     // columns per CTA
constexpr int MAXCL = 16;  // largest (non-portable) cluster

template <int R, int TT, typename TI>
struct Smem {
  static constexpr int NXT = (R + 8) / 8, GX = R + 8, GS = R + 12, PS = R + 4, AS = CW + 4;
  double Ds[NXT][CW / 4][32];   // C~ (+ x0^T as rows R..R+7) of my columns, B-fragment order
  double Cs[R / 4][CW / 8][32]; // -C of my columns, B-fragment order
  TI At[2][TT][AS];             // panel rows, my columns (2 stages, input type)
  TI Yv[2][TT][8];              // panel targets
  double Gp[TT * GX];           // my G partial [t][i] (read by the chunk reducers)
  double Gs[TT][GS];            // reduced G (+ a.x0), written by the chunk reducers
  double Rs[TT][CW];            // rejections of my columns
  double nrm[MAXCL][2][TT];     // |R_t|^2, |a_t|^2 partials of every CTA
  double scal[TT];              // |R_t|^2 totals
  // home only: P^-1, W and the 8-row update scratch
  double Ps[R][PS];
  double Wb[R][8];
  double Ub[R][8], Yb[R][8];
  double Eb[8][8], Dy[8][8];
  double rd[8];
  double zg[R + 8];             // non-general growth: z = P gamma, gamma^T W
  int flags[4];
};

// phase timing (debug builds only: -DRGB_CLUSTER_PROBE): ns per phase summed
// over the run, for CTA 0 (home) and CTA 1, read back with rgb_cluster_probe()
#ifdef RGB_CLUSTER_PROBE
__device__ unsigned long long g_probe[2][16];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define PROBE(i)                                                              \
  do {                                                                        \
    if (tid == 0 && c < 2) {                                                  \
      const unsigned long long now_ = gtime();                                \
      atomicAdd(&g_probe[c][i], now_ - probe_t);                              \
      probe_t = now_;                                                         \
    }                                                                         \
  } while (0)
#else
#define PROBE(i) \
  do {           \
  } while (0)
#endif

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// GEN: general variant only; !GEN: orthogonal / orthonormal (solver.py:382-395)
template <int R, int TT, bool GEN, typename TI>
__global__ void __launch_bounds__(NT, 1) cluster_kernel(rgb_config cfg, rgb_state st, const TI* __restrict__ rows,
                                                        int64_t rstride, const TI* __restrict__ tgts, int64_t tstride,
                                                        int64_t T, uint8_t* __restrict__ blog,
                                                        double* __restrict__ clog) {
  constexpr int IT = R / 8, NXT = (R + 8) / 8, GX = R + 8, MT = TT / 8;
  constexpr int NG = NW / MT;                 // warps per M tile
  constexpr int NJ1 = (NXT + NG - 1) / NG;    // P1 N tiles per warp
  constexpr int NJ3 = (CW / 8) / NG;          // P3 N tiles per warp
  static_assert(NW % MT == 0 && (CW / 8) % NG == 0, "warp tiling");
  using SM = Smem<R, TT, TI>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SM& S = *reinterpret_cast<SM*>(smem_raw);
  cg::cluster_group cluster = cg::this_cluster();
  const int ncl = (int)cluster.num_blocks();
  const int c = (int)cluster.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, p = lane >> 2, q = lane & 3;
  const int M = cfg.m, k = cfg.k, c0 = c * CW;
  const bool home = (c == 0);
  const int64_t cid = blockIdx.x / ncl, ncid = gridDim.x / ncl;
  auto rem = [&](int u) { return cluster.map_shared_rank(&S, u); };
#ifdef RGB_CLUSTER_PROBE
  unsigned long long probe_t = gtime();
#endif

  for (int64_t b = cid; b < cfg.num_streams; b += ncid) {
    int status = st.status[b];
    if (status) continue;  // uniform across the cluster
    int r = st.rank[b];
    const int64_t nobs0 = st.nobs[b];
    double* Cg = reinterpret_cast<double*>(st.basis) + b * (int64_t)R * M;
    double* Dg = reinterpret_cast<double*>(st.dual) + b * (int64_t)R * M;
    double* Pg = reinterpret_cast<double*>(st.gram_inv) + b * (int64_t)R * R;
    double* Xg = reinterpret_cast<double*>(st.x) + b * (int64_t)k * M;
    const TI* Rb = rows + b * rstride;
    const TI* Yb = tgts + b * tstride;

    // ---- my slices: C~ (+ x0^T), -C; home: P^-1, W = 0 ---------------------------
    for (int e = tid; e < NXT * (CW / 4) * 32; e += NT) {
      const int l = e & 31, kt = (e >> 5) % (CW / 4), nt = e / (32 * (CW / 4));
      const int i = 8 * nt + (l >> 2), col = c0 + 4 * kt + (l & 3);
      double v = 0.0;
      if (i < R) v = Dg[(int64_t)i * M + col];
      else if (i - R < k) v = Xg[(int64_t)(i - R) * M + col];
      S.Ds[nt][kt][l] = v;
    }
    for (int e = tid; e < (R / 4) * (CW / 8) * 32; e += NT) {
      const int l = e & 31, nt = (e >> 5) % (CW / 8), kt = e / (32 * (CW / 8));
      S.Cs[kt][nt][l] = -Cg[(int64_t)(4 * kt + (l & 3)) * M + c0 + 8 * nt + (l >> 2)];
    }
    if (home) {
      for (int e = tid; e < R * R; e += NT) S.Ps[e / R][e % R] = Pg[e];
      for (int e = tid; e < R * 8; e += NT) S.Wb[e >> 3][e & 7] = 0.0;
    }

    const int64_t npan = (T + TT - 1) / TT;
    auto prefetch = [&](int64_t pan, int s) {
      if (pan < npan) {
        const int64_t t0 = pan * TT;
        constexpr int CH = 16 / (int)sizeof(TI);  // values per 16-byte chunk
        for (int e = tid; e < TT * (CW / CH); e += NT) {
          const int t = e / (CW / CH), j = (e % (CW / CH)) * CH;
          const bool ok = t0 + t < T;
          blk::cp_async16(&S.At[s][t][j], ok ? Rb + (t0 + t) * M + c0 + j : Rb, ok ? 16 : 0);
        }
        for (int e = tid; e < TT * 8; e += NT) {
          const int t = e >> 3, cc = e & 7;
          const bool ok = t0 + t < T && cc < k;
          blk::cp_async_one<TI>(&S.Yv[s][t][cc], ok ? Yb + (t0 + t) * k + cc : Yb, ok);
        }
      }
      blk::cp_commit();
    };

    // ---- home: blocked Sherman-Morrison over dependent rows [rs, te) of the
    // 8-row block at panel row base (solver.py:297-304 applied to 8 rows at once,
    // M = I + G P G^T = L D L^T, E = L^-1; Y = P G^T E^T; P -= Y D^-1 Y^T;
    // W += Y D^-1 E dy0, dy0 = y - a.x0 - G W) ------------------------------------
    auto dep_block = [&](int s, int base, int rs, int te, int64_t t0) {
      const int kr = (r + 3) >> 2;  // K steps over the rank (rows beyond it are zero)
      const bool in_t = base + p >= rs && base + p < te;
      // U = P G^T (M = i, N = t, K = i'): warp w owns rows 8w..8w+7
      {
        double acc[2] = {0.0, 0.0}, acc2[2] = {0.0, 0.0};
        if (8 * w < r) {
          for (int kt = 0; kt < kr; kt += 2) {
            mma(acc, S.Ps[8 * w + p][4 * kt + q], in_t ? S.Gs[base + p][4 * kt + q] : 0.0);
            if (kt + 1 < kr) mma(acc2, S.Ps[8 * w + p][4 * kt + 4 + q], in_t ? S.Gs[base + p][4 * kt + 4 + q] : 0.0);
          }
        }
        S.Ub[8 * w + p][2 * q] = acc[0] + acc2[0];
        S.Ub[8 * w + p][2 * q + 1] = acc[1] + acc2[1];
      }
      __syncthreads();
      PROBE(10);
      if (w == 0) {
        // S = G U and G W (M = t, K = i), two chains each
        double s0[2] = {0.0, 0.0}, s1[2] = {0.0, 0.0}, g0[2] = {0.0, 0.0}, g1[2] = {0.0, 0.0};
        for (int kt = 0; kt < kr; kt += 2) {
          const double a0 = in_t ? S.Gs[base + p][4 * kt + q] : 0.0;
          mma(s0, a0, S.Ub[4 * kt + q][p]);
          mma(g0, a0, S.Wb[4 * kt + q][p]);
          if (kt + 1 < kr) {
            const double a1 = in_t ? S.Gs[base + p][4 * kt + 4 + q] : 0.0;
            mma(s1, a1, S.Ub[4 * kt + 4 + q][p]);
            mma(g1, a1, S.Wb[4 * kt + 4 + q][p]);
          }
        }
        double mi[2] = {s0[0] + s1[0], s0[1] + s1[1]};
        const double gws[2] = {g0[0] + g1[0], g0[1] + g1[1]};
        if (p == 2 * q) mi[0] += 1.0;
        if (p == 2 * q + 1) mi[1] += 1.0;
#pragma unroll
        for (int e = 0; e < 2; ++e)  // dy0[t = p][cc = 2q + e]
          S.Dy[p][2 * q + e] = in_t ? (double)S.Yv[s][base + p][2 * q + e] - S.Gs[base + p][R + 2 * q + e] - gws[e] : 0.0;
        // M = L D L^T by forward elimination; E = L^-1 (rows are t = p)
        double ev[2] = {p == 2 * q ? 1.0 : 0.0, p == 2 * q + 1 ? 1.0 : 0.0};
#pragma unroll
        for (int kk = 0; kk < 7; ++kk) {
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
        S.Eb[p][2 * q] = ev[0];
        S.Eb[p][2 * q + 1] = ev[1];
        if ((p >> 1) == q) S.rd[p] = rcp64((p & 1) ? mi[1] : mi[0]);
        __syncwarp();
        // dh = E dy0 / d (M = t, N = cc, K = t')
        double dh[2] = {0.0, 0.0};
#pragma unroll
        for (int kt = 0; kt < 2; ++kt) mma(dh, S.Eb[p][4 * kt + q], S.Dy[4 * kt + q][p]);
        __syncwarp();
        S.Dy[p][2 * q] = dh[0] * S.rd[p];
        S.Dy[p][2 * q + 1] = dh[1] * S.rd[p];
      }
      __syncthreads();
      PROBE(11);
      // Y = U E^T (M = i, N = t, K = t'), W += Y (D^-1 E dy0) (M = i, N = cc, K = t)
      if (8 * w < r) {
        double yb[2] = {0.0, 0.0};
#pragma unroll
        for (int kt = 0; kt < 2; ++kt) mma(yb, S.Ub[8 * w + p][4 * kt + q], S.Eb[p][4 * kt + q]);
        S.Yb[8 * w + p][2 * q] = yb[0];
        S.Yb[8 * w + p][2 * q + 1] = yb[1];
        __syncwarp();
        double wb[2] = {S.Wb[8 * w + p][2 * q], S.Wb[8 * w + p][2 * q + 1]};
#pragma unroll
        for (int kt = 0; kt < 2; ++kt) mma(wb, S.Yb[8 * w + p][4 * kt + q], S.Dy[4 * kt + q][p]);
        S.Wb[8 * w + p][2 * q] = wb[0];
        S.Wb[8 * w + p][2 * q + 1] = wb[1];
      }
      __syncthreads();
      PROBE(12);
      // P -= Y D^-1 Y^T (M = i, N = i', K = t): warp w owns row block w
      if (8 * w < r) {
        const double ys0 = -S.Yb[8 * w + p][q] * S.rd[q], ys1 = -S.Yb[8 * w + p][4 + q] * S.rd[4 + q];
#pragma unroll
        for (int nt = 0; nt < IT; ++nt) {
          if (8 * nt < r) {
            double acc[2] = {S.Ps[8 * w + p][8 * nt + 2 * q], S.Ps[8 * w + p][8 * nt + 2 * q + 1]};
            mma(acc, ys0, S.Yb[8 * nt + p][q]);
            mma(acc, ys1, S.Yb[8 * nt + p][4 + q]);
            S.Ps[8 * w + p][8 * nt + 2 * q] = acc[0];
            S.Ps[8 * w + p][8 * nt + 2 * q + 1] = acc[1];
          }
        }
      }
      // logs of the dependent rows
      if (tid < 8 && base + tid >= rs && base + tid < te) {
        const int64_t row = b * T + t0 + base + tid;
        if (blog) blog[row] = 0;
        if (clog)
          for (int i = 0; i < R; ++i) clog[row * R + i] = S.Gs[base + tid][i];
      }
      __syncthreads();
      PROBE(13);
    };

    int64_t consumed = 0;
    bool stopped = false;
    prefetch(0, 0);
    for (int64_t pan = 0; pan < npan && !stopped; ++pan) {
      const int s = (int)(pan & 1);
      const int64_t t0 = pan * TT;
      const int tv = (int)((T - t0) < TT ? (T - t0) : TT);
      prefetch(pan + 1, s ^ 1);
      blk::cp_wait<1>();
      __syncthreads();
      PROBE(9);
      int row_start = 0;
      while (true) {
        // ---- P1: G partial of my columns (M = t, N = i, K = my columns) ----------------
        // warp w: M tile w % MT, N tiles w / MT + NG j -- independent MMA chains
        // that share the A fragment of each K step
        {
          const int mt = w % MT, n0 = w / MT;
          double acc[NJ1][2];
#pragma unroll
          for (int j = 0; j < NJ1; ++j) acc[j][0] = acc[j][1] = 0.0;
          bool on[NJ1];
#pragma unroll
          for (int j = 0; j < NJ1; ++j) {
            const int nt = n0 + NG * j;
            on[j] = nt < NXT && (nt >= IT || 8 * nt < r);  // rows of C~ beyond the rank are zero
          }
#pragma unroll
          for (int kt = 0; kt < CW / 4; ++kt) {
            const double a = (double)S.At[s][8 * mt + p][4 * kt + q];
#pragma unroll
            for (int j = 0; j < NJ1; ++j)
              if (on[j]) mma(acc[j], a, S.Ds[n0 + NG * j][kt][lane]);
          }
#pragma unroll
          for (int j = 0; j < NJ1; ++j) {
            const int nt = n0 + NG * j;
            if (nt < NXT)
              *reinterpret_cast<double2*>(&S.Gp[(8 * mt + p) * GX + 8 * nt + 2 * q]) = make_double2(acc[j][0], acc[j][1]);
          }
        }
        PROBE(0);
        cluster_sync_all();
        PROBE(1);
        // ---- P2: G = sum of the partials; my chunk, stored into every CTA ---------------
        {
          constexpr int NE = TT * GX;
          const int chunk = (NE + ncl - 1) / ncl;
          const int e0 = c * chunk, e1 = (e0 + chunk < NE) ? e0 + chunk : NE;
          // (DSMEM-bandwidth bound: 2 x 15/16 of an 18 KB panel of partials per CTA)
          for (int e = e0 + tid; e < e1; e += NT) {
            double v = 0.0;
            for (int u = 0; u < ncl; ++u) v += rem(u)->Gp[e];
            const int t = e / GX, i = e % GX;
            for (int u = 0; u < ncl; ++u) rem(u)->Gs[t][i] = v;
          }
        }
        PROBE(2);
        cluster_sync_all();
        PROBE(3);
        // ---- P3: R = A - G C on my columns (M = t, N = my columns, K = i) ---------------
        {
          const int kmax = (r + 3) >> 2;
          const int mt = w % MT, n0 = w / MT;  // warp w: M tile w % MT, N tiles w / MT + NG j
          double acc[NJ3][2];
#pragma unroll
          for (int j = 0; j < NJ3; ++j) {
            const int nt = n0 + NG * j;
            acc[j][0] = (double)S.At[s][8 * mt + p][8 * nt + 2 * q];
            acc[j][1] = (double)S.At[s][8 * mt + p][8 * nt + 2 * q + 1];
          }
          for (int kt = 0; kt < kmax; ++kt) {
            const double a = S.Gs[8 * mt + p][4 * kt + q];
#pragma unroll
            for (int j = 0; j < NJ3; ++j) mma(acc[j], a, S.Cs[kt][n0 + NG * j][lane]);
          }
#pragma unroll
          for (int j = 0; j < NJ3; ++j)
            *reinterpret_cast<double2*>(&S.Rs[8 * mt + p][8 * (n0 + NG * j) + 2 * q]) = make_double2(acc[j][0], acc[j][1]);
          __syncthreads();
          // |R_t|^2 and |a_t|^2 of my columns -> every CTA's nrm[c]
          // NT / TT threads per row, each over every (NT / TT)-th column
          constexpr int TPR = NT / TT;
          static_assert(TPR >= 2 && (TPR & (TPR - 1)) == 0 && MAXCL <= 2 * TPR, "norm threads");
          {
            const int t = tid / TPR, part = tid % TPR;
            double rs2 = 0.0, as2 = 0.0;
#pragma unroll
            for (int j = part; j < CW; j += TPR) {
              const double rv = S.Rs[t][j], av = (double)S.At[s][t][j];
              rs2 = fma(rv, rv, rs2);
              as2 = fma(av, av, as2);
            }
#pragma unroll
            for (int o = 1; o < TPR; o <<= 1) {
              rs2 += __shfl_xor_sync(FULL, rs2, o);
              as2 += __shfl_xor_sync(FULL, as2, o);
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int u = part + h * TPR;
              if (u < ncl) {
                SM* d = rem(u);
                d->nrm[c][0][t] = rs2;
                d->nrm[c][1][t] = as2;
              }
            }
          }
        }
        PROBE(4);
        cluster_sync_all();
        PROBE(5);
        // ---- P4: the rank test (identical in every CTA) --------------------------------
        if (w == 0) {
          double rsq = 0.0, asq = 0.0;
          bool ybad = false;
          if (lane < TT) {
            for (int u = 0; u < ncl; ++u) {
              rsq += S.nrm[u][0][lane];
              asq += S.nrm[u][1][lane];
            }
            for (int cc = 0; cc < k; ++cc) ybad |= !isfinite((double)S.Yv[s][lane][cc]);
            S.scal[lane] = rsq;
          }
          const bool valid = lane >= row_start && lane < tv;
          const bool dep = is_dependent<double>(rsq, asq, eps_sq<double>(cfg, r));
          const bool bad = !isfinite(asq) || ybad;
          const unsigned stopm = __ballot_sync(FULL, valid && (!dep || bad));
          const unsigned badm = __ballot_sync(FULL, valid && bad);
          if (lane == 0) {
            S.flags[0] = stopm ? __ffs(stopm) - 1 : tv;
            S.flags[1] = (int)badm;
          }
        }
        __syncthreads();
        const int tstar = S.flags[0];
        const unsigned badm = (unsigned)S.flags[1];
        PROBE(6);
        if (home && tstar > row_start) {
          PROBE(14);
          for (int base = (row_start & ~7); base < tstar; base += 8) dep_block(s, base, row_start, tstar, t0);
        }
        PROBE(7);
        if (tstar >= tv) break;
        if ((badm >> tstar) & 1u) {
          status |= RGB_ST_NONFINITE;
          stopped = true;
          consumed = t0 + tstar;
          break;
        }
        if (r >= R) {
          status |= RGB_ST_RANK_CAP;
          stopped = true;
          consumed = t0 + tstar;
          break;
        }
        // ---- independent row tstar (solver.py:305-318, _grow solver.py:368-397) ---------
        const int ts = tstar;
        const double rsq = S.scal[ts];
        if (GEN || cfg.variant == RGB_GENERAL) {
          const double rinv = 1.0 / rsq;  // K = rej / |rej|^2 (one rounding more than a division)
          // C~[:r] -= gamma K^T, C~[r] = K on my columns; C[r] = a
          for (int e = tid; e < IT * (CW / 4) * 32; e += NT) {
            const int l = e & 31, kt = (e >> 5) % (CW / 4), nt = e / (32 * (CW / 4));
            const int i = 8 * nt + (l >> 2), jl = 4 * kt + (l & 3);
            if (i > r) continue;
            const double K = S.Rs[ts][jl] * rinv;
            S.Ds[nt][kt][l] = (i == r) ? K : fma(-S.Gs[ts][i], K, S.Ds[nt][kt][l]);
          }
          for (int e = tid; e < CW; e += NT) {
            const int kt = r >> 2, nt = e >> 3, l = 4 * (e & 7) + (r & 3);
            S.Cs[kt][nt][l] = -(double)S.At[s][ts][e];
          }
          if (home) {
            // P = diag(P, 1); W gains row r = y - a.x0 of row ts
            for (int i = tid; i < R; i += NT) {
              S.Ps[r][i] = (i == r) ? 1.0 : 0.0;
              S.Ps[i][r] = (i == r) ? 1.0 : 0.0;
            }
            if (tid < 8) S.Wb[r][tid] = tid < k ? (double)S.Yv[s][ts][tid] - S.Gs[ts][R + tid] : 0.0;
            if (tid == 0) {
              const int64_t row = b * T + t0 + ts;
              if (blog) blog[row] = 1;
              if (clog)
                for (int i = 0; i < R; ++i) clog[row * R + i] = (i == r) ? 1.0 : 0.0;
            }
          }
        } else {
          // orthogonal / orthonormal: C~[:r], C[:r] stay; P gains an edge -alpha z
          // and a corner alpha^2 (1 + gamma.z), z = P gamma (solver.py:307-310,
          // 382-395); W gains alpha (y - a.x), a.x = a.x0 + gamma^T W
          const double resc = (cfg.variant == RGB_ORTHONORMAL) ? 1.0 / sqrt(rsq) : cfg.alpha;
          const double last = 1.0 / resc;
          const double alpha = 1.0 / last;
          const double sc = alpha * rsq;
          for (int e = tid; e < CW; e += NT) {
            const double rj = S.Rs[ts][e];
            const int kt = e >> 2, l = 4 * (r & 7) + (e & 3);
            S.Ds[r >> 3][kt][l] = (cfg.variant == RGB_ORTHONORMAL) ? alpha * rj : rj / sc;
            S.Cs[r >> 2][e >> 3][4 * (e & 7) + (r & 3)] = -(alpha * rj);
          }
          if (home) {
            if (tid < R) {  // z_i = (P gamma)_i
              double z = 0.0;
              for (int i2 = 0; i2 < R; ++i2) z = fma(S.Ps[tid][i2], S.Gs[ts][i2], z);
              S.zg[tid] = z;
            } else if (tid < R + 8) {  // (gamma^T W)_c
              const int cc = tid - R;
              double g = 0.0;
              for (int i = 0; i < R; ++i) g = fma(S.Gs[ts][i], S.Wb[i][cc], g);
              S.zg[tid] = g;
            }
            __syncthreads();
            double dn = 0.0;
            for (int i = 0; i < R; ++i) dn = fma(S.Gs[ts][i], S.zg[i], dn);
            const double denom = 1.0 + dn;
            for (int i = tid; i < R; i += NT) {
              const double edge = (i < r) ? -(alpha * S.zg[i]) : 0.0;
              S.Ps[i][r] = (i == r) ? alpha * alpha * denom : edge;
              if (i != r) S.Ps[r][i] = edge;
            }
            if (tid < 8)
              S.Wb[r][tid] = tid < k ? alpha * (((double)S.Yv[s][ts][tid] - S.Gs[ts][R + tid]) - S.zg[R + tid]) : 0.0;
            if (tid == 0) {
              const int64_t row = b * T + t0 + ts;
              if (blog) blog[row] = 1;
              if (clog)
                for (int i = 0; i < R; ++i) clog[row * R + i] = i < r ? S.Gs[ts][i] : (i == r ? last : 0.0);
            }
          }
        }
        __syncthreads();
        PROBE(8);
        r += 1;
        row_start = tstar + 1;
        if (row_start >= tv) break;
      }
      if (!stopped) consumed = t0 + tv;
    }
    blk::cp_wait<0>();

    // ---- write back: C~, C (my columns), P (home); x = x0 + C~^T W ------------------------
    for (int e = tid; e < IT * (CW / 4) * 32; e += NT) {
      const int l = e & 31, kt = (e >> 5) % (CW / 4), nt = e / (32 * (CW / 4));
      Dg[(int64_t)(8 * nt + (l >> 2)) * M + c0 + 4 * kt + (l & 3)] = S.Ds[nt][kt][l];
    }
    for (int e = tid; e < (R / 4) * (CW / 8) * 32; e += NT) {
      const int l = e & 31, nt = (e >> 5) % (CW / 8), kt = e / (32 * (CW / 8));
      Cg[(int64_t)(4 * kt + (l & 3)) * M + c0 + 8 * nt + (l >> 2)] = -S.Cs[kt][nt][l];
    }
    if (home)
      for (int e = tid; e < R * R; e += NT) Pg[e] = S.Ps[e / R][e % R];
    cluster_sync_all();  // W final in home
    // W from home into my Yb scratch (unused outside home's updates), then x
    {
      SM* h = rem(0);
      double* Wl = &S.Ub[0][0];
      if (!home)
        for (int e = tid; e < R * 8; e += NT) Wl[e] = h->Wb[e >> 3][e & 7];
      __syncthreads();
      const double* Wr = home ? &S.Wb[0][0] : Wl;
      for (int e = tid; e < k * CW; e += NT) {
        const int cc = e / CW, jl = e % CW;
        double x = S.Ds[NXT - 1][jl >> 2][4 * cc + (jl & 3)];  // x0^T row cc (last N tile of Ds)
        for (int i = 0; i < r; ++i) x = fma(S.Ds[i >> 3][jl >> 2][4 * (i & 7) + (jl & 3)], Wr[i * 8 + cc], x);
        Xg[(int64_t)cc * M + c0 + jl] = x;
      }
    }
    if (home && tid == 0) {
      st.rank[b] = r;
      st.nobs[b] = nobs0 + consumed;
      st.status[b] = status;
    }
    cluster_sync_all();  // the next stream reuses every buffer
  }
}

}  // namespace cls

template <int R, int TT, typename TI>
static int launch_cluster_t(const rgb_config& cfg, rgb_state& st, const void* rows, int64_t rows_stride,
                            const void* targets, int64_t tg_stride, int64_t T, const rgb_logs& logs,
                            cudaStream_t stream, int num_sms) {
  const int ncl = cfg.m / cls::CW;
  const bool gen = cfg.variant == RGB_GENERAL;
  auto kern = gen ? cls::cluster_kernel<R, TT, true, TI> : cls::cluster_kernel<R, TT, false, TI>;
  const size_t smem = sizeof(cls::Smem<R, TT, TI>);
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
      cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
    cudaGetLastError();
    return RGB_E_UNSUPPORTED;
  }
  cudaLaunchConfig_t lc = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)ncl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.blockDim = dim3(cls::NT);
  lc.dynamicSmemBytes = smem;
  lc.stream = stream;
  lc.attrs = at;
  lc.numAttrs = 1;
  lc.gridDim = dim3((unsigned)ncl);
  int nclusters = 0;
  if (cudaOccupancyMaxActiveClusters(&nclusters, (const void*)kern, &lc) != cudaSuccess || nclusters < 1) {
    cudaGetLastError();
    return RGB_E_UNSUPPORTED;
  }
  (void)num_sms;
  if ((int64_t)nclusters > cfg.num_streams) nclusters = (int)cfg.num_streams;
  lc.gridDim = dim3((unsigned)(ncl * nclusters));
  const TI* rp = (const TI*)rows;
  const TI* tp = (const TI*)targets;
  cudaError_t e = cudaLaunchKernelEx(&lc, kern, cfg, st, rp, rows_stride, tp, tg_stride, T, logs.branch,
                                     (double*)logs.coords);
  return e == cudaSuccess ? RGB_OK : RGB_E_CUDA;
}

bool cluster_supports(const rgb_config& cfg) {
  const bool var_ok = cfg.variant == RGB_GENERAL || cfg.variant == RGB_ORTHONORMAL ||
                      (cfg.variant == RGB_ORTHOGONAL && cfg.alpha != 0.0);
  if (cfg.dtype != RGB_F64 || !var_ok || cfg.k < 1 || cfg.k > 8) return false;
  return cfg.r_cap == 64 && cfg.m % cls::CW == 0 && cfg.m / cls::CW >= 2 && cfg.m / cls::CW <= cls::MAXCL;
}

int launch_cluster(const rgb_config& cfg, rgb_state& st, const void* rows, int64_t rows_stride, const void* targets,
                   int64_t tg_stride, int64_t T, const rgb_logs& logs, cudaStream_t stream, int num_sms,
                   bool f32in) {
  if (logs.resid || logs.gain) return RGB_E_UNSUPPORTED;
  if (!cluster_supports(cfg)) return RGB_E_UNSUPPORTED;
  return f32in ? launch_cluster_t<64, 32, float>(cfg, st, rows, rows_stride, targets, tg_stride, T, logs, stream, num_sms)
               : launch_cluster_t<64, 32, double>(cfg, st, rows, rows_stride, targets, tg_stride, T, logs, stream, num_sms);
}

}  // namespace rgb

#ifdef RGB_CLUSTER_PROBE
extern "C" int rgb_cluster_probe(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, rgb::cls::g_probe, sizeof(rgb::cls::g_probe));
  if (reset) {
    unsigned long long z[2][16] = {};
    cudaMemcpyToSymbol(rgb::cls::g_probe, z, sizeof(z));
  }
  return 0;
}
#endif
