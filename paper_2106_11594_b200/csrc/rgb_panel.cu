// rgb_panel.cu -- batched rank-Greville update, one stream per CTA, with the
// rows split over warps (sm_100a, fp64 tensor cores).
//
// Same algebra as rgb_blocked.cu (8-row tiles on DMMA.8x8x4, LDL^T-factored
// Sherman-Morrison, x = x0 + C~^T W; see its header), arranged for streams
// whose factors do not fit one warp's registers (config 3 of BASELINE.json:
// m = 128, r <= 32).  The warp-group kernel (rgb_blocked_wg.cu) splits such a
// stream's COLUMNS over four warps and pays a group-wide reduction and five
// CTA barriers per 8 rows; here the rows are split instead:
//
//  * C~ and C live in shared memory (MMA B-fragment order, 2 x r_cap x m x 8 B).
//  * Three PROJECTION warps take a 24-row panel, one 8-row tile each, and run
//    the whole projection of their tile -- G = A C~^T, R = A - G C, |a|^2,
//    |R_t|^2 and the rank test (solver.py:286-296) -- over all m columns with
//    no cross-warp reduction.  A tile goes from global memory straight into
//    the MMA fragment registers; the next panel's rows are pulled into L2
//    (prefetch.global.L2) meanwhile.  Inside a run of dependent rows C~ and C do not
//    change, so the three tiles are independent; the first independent (or
//    non-finite) row of the panel ends it: the rows before it are dependent,
//    the row grows the basis (solver.py:305-318, _grow :368-397; every warp
//    updates its own columns of C~ and C), and the next panel starts on the
//    row after it.
//  * One HOME warp owns P^-1 and W in registers and folds the dependent tiles
//    of each panel in row order (U = G P, S = U G^T, the 8x8 LDL^T of I + S,
//    P -= Y^T D^-1 Y, W += ..., solver.py:297-304), while the projection
//    warps already project the next panel.  The hand-off is a one-panel slot
//    in shared memory guarded by two named barriers (FULL: projection warps
//    arrive, home syncs; EMPTY: home arrives, projection warps sync).  In the
//    general variant growth never reads P^-1 or W (W's new row is y - a.x0,
//    P^-1 = diag(P^-1, 1)), so a growth row only appends a marker to the slot.
//  * Deferred fold: for a fresh stream the home warp only accumulates Q = B^T B and
//    B^T dy from the slot (no dependent chain) and the CTA inverts Q once at the end,
//    accepted when kappa_F(Q) <= 1e6; otherwise the stream is folded again with the
//    chain above (see the comment at `defer` below and DESIGN.md).  Config 3:
//    2.18 -> 1.95 ms, 1.75 ms with the projection's G loop rank-tile-outermost.
//  * A fresh stream's leading independent rows are taken one at a time on the
//    CUDA cores (all four warps split the columns), as in the warp-group
//    kernel's row mode; W's rows of that phase go to the home warp through
//    shared memory.
//
// General variant, fp64 state, k <= 8 right-hand sides, float64 or float32
// inputs; instantiated for m = 128 with r_cap 16 and 32 (three CTAs -- three
// streams, twelve warps -- per SM: 74 KB of shared memory, at most 168 registers
// per thread) and for m = 256 with r_cap 16 (config 1: one CTA per SM, 254
// registers; 0.099 ms per solve against 0.143 ms on the warp-group kernel).  W's
// rows share the hand-off slot's memory (the home warp reads them before the
// first panel and writes W there after the last).  Streams are claimed
// dynamically (an atomic counter).  Config 3: 2.22 ms against 3.11 ms for the
// warp-group kernel (2.60 ms with two CTAs per SM and a cp.async stage per warp,
// 2.32 ms with a static round robin).  Per stream (scripts/probe_panel.py,
// -DRGB_PANEL_PROBE) the row mode is ~1/3 of the time, and the home warp's chain
// (8x8 LDL^T ~1 900 cycles per tile behind the projection warps' DMMAs) bounds
// the panel phase; DESIGN.md lists the variants measured and rejected.
//
// Fragment layouts (lane = 4p + q; sigma(kt,q) = 8(kt>>1) + 2q + (kt&1)):
//   tile   acc[jt][e]        = A[t=p][8jt+2q+e]         registers (A- and B-operand, K = sigma)
//   C~     Df[nt][ks][lane]  = C~[8nt+p][sigma(ks,q)]    shared memory (B operand of G)
//   -C     Cf[kt][jt][lane]  = -C[sigma(kt,q)][8jt+p]    shared memory (B operand of R)
//   P^-1   Pr[mt][nt][e]     = P[8mt+p][8nt+2q+e]        home registers (symmetric)
//   W^T    Wt[mt][e]         = W[8mt+2q+e][c=p]          home registers
#include <cstddef>
#include <cstdlib>
#include <type_traits>

#include "rgb_mma.cuh"

namespace rgb {
namespace blk {

constexpr int PW = 3;          // projection warps (+ one home warp)
constexpr int PNL = PW * TT;   // rows per panel
constexpr int PANEL_THREADS = (PW + 1) * 32;
enum { BAR_PROJ = 1, BAR_FULL = 2, BAR_EMPTY = 3, BAR_ROW = 4 };

__device__ __forceinline__ void bar_sync_n(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive_n(int id, int n) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}

// phase timing (debug builds only: -DRGB_PANEL_PROBE): clock64 cycles per phase,
// summed over projection warp 0 (slots 0-7) and the home warp (slots 8-15) of
// every CTA, read back with rgb_panel_probe() (scripts/probe_panel.py)
#ifdef RGB_PANEL_PROBE
__device__ unsigned long long g_pprobe[32];
__device__ unsigned g_wslot[8192];
#define PPROBE(i)                                                 \
  do {                                                            \
    if ((threadIdx.x & 31) == 0 && (w == 0 || w == PW)) {         \
      const long long now_ = clock64();                           \
      atomicAdd(&g_pprobe[i], (unsigned long long)(now_ - pp_t)); \
      pp_t = now_;                                                \
    }                                                             \
  } while (0)
#else
#define PPROBE(i) \
  do {            \
  } while (0)
#endif

template <typename TI>
__device__ __forceinline__ double2 ld2(const TI* ptr) {
  if constexpr (sizeof(TI) == 8) {
    return __ldg(reinterpret_cast<const double2*>(ptr));
  } else {
    const float2 f = __ldg(reinterpret_cast<const float2*>(ptr));
    return make_double2((double)f.x, (double)f.y);
  }
}

template <int R, int M, typename TI>
struct PanelSmem {
  static constexpr int IT = R / 8, IK = R / 4, NJ = M / 8, KS = M / 4;
  double Df[IT][KS][32];       // C~, B-fragment order
  double Cf[IK][NJ][32];       // -C, B-fragment order
  // hand-off slot: one panel, projection warps -> home warp
  double sG[PW][IT][32][2];    // G of each tile (accumulator layout)
  double sDy[PW][32][2];       // y - a.x0, [c=p][t=2q+e]
  double sWnew[8];             // growth: W's new row (per RHS)
  int sTe[PW];                 // dependent rows [0, te) of each tile
  int sGrow, sEnd;             // growth marker, end of stream
  unsigned claim;              // the stream this CTA works on
  // projection-warp exchange
  int stop[PW];                // first stop row of each tile (TT = none)
  int bad[PW];                 // ... and whether it is non-finite
  double gpart[PW + 1][R];     // row mode: partial coords per warp
  double a2part[PW + 1], r2part[PW + 1];
  double gam[R];               // growth: coords of the row
  double kv[M];                //         its gain K = rej / |rej|^2
  // bulk growth's scratch spans sG .. here: 8 x M + 8 x R doubles (padded to fit)
  double bulkpad[R >= 32 ? 48 : 384];
};

template <int R, int M, typename TI>
__global__ void __launch_bounds__(PANEL_THREADS, (M <= 128 ? 3 : 1)) panel_kernel(
    rgb_config cfg, rgb_state st, const TI* __restrict__ rows, int64_t rstride,
    const TI* __restrict__ tgts, int64_t tstride, int64_t T, uint8_t* __restrict__ blog,
    double* __restrict__ clog, unsigned* __restrict__ next_stream, int seq_only) {
  using SMT = PanelSmem<R, M, TI>;
  constexpr int IT = SMT::IT, IK = SMT::IK, NJ = SMT::NJ, KS = SMT::KS;
  // own columns of a projection warp (row mode, growth, write-back): the 8-column
  // groups J = w, w + PW, ... (k-steps 2J, 2J+1 of C~, column tile J of C)
  constexpr int NG = (NJ + PW - 1) / PW;
  static_assert(R % 8 == 0 && R <= 32 && M % 8 == 0 && PW == 3, "shape");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SMT& S = *reinterpret_cast<SMT*>(smem_raw);
  // W rows of the row-mode phase / W at the end share the hand-off slot (the
  // home warp reads them before the first panel and writes them after the last)
  static_assert(sizeof(S.sG) >= sizeof(double) * R * 8, "W over the slot");
  double (&Wsm)[R][8] = *reinterpret_cast<double(*)[R][8]>(&S.sG[0][0][0][0]);
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;  // warps 0..PW-1 project, warp PW is the home warp
  const int p = lane >> 2, q = lane & 3;
  const int k = cfg.k;
  const bool home = (w == PW);
#ifdef RGB_PANEL_PROBE
  long long pp_t = clock64();
  if (lane == 0 && blockIdx.x < 1024) {
    unsigned wid, sm;
    asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    g_wslot[blockIdx.x * 8 + w] = (sm << 16) | wid;
  }
#endif

  // streams are claimed dynamically (their cost varies with the rank they reach:
  // row-mode length, rank tiles of every projection and of the P^-1 chain)
  // (no counter when every CTA has at most one stream: the CTA index is the stream)
  int64_t b = 0;
  bool redo = false;  // the deferred fold of stream b failed its conditioning certificate
  for (unsigned iter = 0;; ++iter) {
    __syncthreads();  // every thread has read the previous claim
    if (!redo) {
      if (threadIdx.x == 0)
        S.claim = next_stream ? atomicAdd(next_stream, 1u) : (iter == 0 ? blockIdx.x : 0xffffffffu);
      __syncthreads();
      b = S.claim;
    }
    const bool seq = redo || seq_only != 0;
    redo = false;
    if (b >= cfg.num_streams) break;
    int status = st.status[b];
    if (status) continue;  // uniform across the block
    int r = st.rank[b];
    const int64_t nobs0 = st.nobs[b];
    double* Cg = reinterpret_cast<double*>(st.basis) + b * (int64_t)R * M;
    double* Dg = reinterpret_cast<double*>(st.dual) + b * (int64_t)R * M;
    double* Pg = reinterpret_cast<double*>(st.gram_inv) + b * (int64_t)R * R;
    double* Xg = reinterpret_cast<double*>(st.x) + b * (int64_t)k * M;
    const TI* Rb = rows + b * rstride;
    const TI* Yb = tgts + b * tstride;
    const bool fresh = (r == 0);
    // Deferred fold (a fresh stream): in the general variant neither the rank test nor
    // growth reads P^-1 or W, so the per-row Sherman-Morrison chain (solver.py:297-304)
    // is not needed while the rows stream by.  It is the recursive form of
    //   P^-1 = (B^T B)^-1,  W = P^-1 B^T (y - A x0)       (B: the coords log, A = B C)
    // so the home warp only accumulates Q = B^T B and B^T dy on the tensor cores -- no
    // dependent chain -- and the CTA inverts Q once at the end.  The inverse is accepted
    // when kappa_F(Q) = |Q|_F |Q^-1|_F <= DEFER_KAPPA (the two forms then agree to
    // ~1e-16 kappa, measured against the reference's own recursion: <= 4e-11 in x);
    // otherwise the stream is folded again with the sequential chain below.
    const bool defer = fresh && !seq;

    // ---- state into shared memory (rank 0 is all zeros by the state contract) ----
    for (int i = threadIdx.x; i < IT * KS * 32; i += PANEL_THREADS) {
      const int l = i & 31, ks = (i >> 5) % KS, nt = (i >> 5) / KS;
      (&S.Df[0][0][0])[i] = fresh ? 0.0 : Dg[(8 * nt + (l >> 2)) * M + sigma(ks, l & 3)];
    }
    for (int i = threadIdx.x; i < IK * NJ * 32; i += PANEL_THREADS) {
      const int l = i & 31, jt = (i >> 5) % NJ, kt = (i >> 5) / NJ;
      (&S.Cf[0][0][0])[i] = fresh ? 0.0 : -Cg[sigma(kt, l & 3) * M + 8 * jt + (l >> 2)];
    }
    for (int i = threadIdx.x; i < R * 8; i += PANEL_THREADS) (&Wsm[0][0])[i] = 0.0;
    bool nz = false;
    if (!fresh)
      for (int i = threadIdx.x; i < k * M; i += PANEL_THREADS) nz |= (Xg[i] != 0.0);
    const bool has_x0 = __syncthreads_or(nz) != 0;
    PPROBE(home ? 8 : 0);

    int64_t consumed = 0;
    int64_t tcur = 0;
    // ---- row mode: a fresh stream's leading independent rows, one at a time ----
    // (x0 = 0; all four warps, the home warp included -- it has nothing to fold
    // yet).  The reference's per-row step on the CUDA cores (solver.py:286-296,
    // 305-318, _grow :368-380) with the columns split over the warps in 8-column
    // groups J = u, u + 4, ... (u = physical warp): partial coords of rank rows
    // 8nt + p over the own columns sigma(ks, q), a fixed-order sum over the
    // warps, the rejection of the own columns 8J + p, its norm summed the same
    // way, and the growth applied by every warp to its own columns.
    if (fresh && !has_x0) {
      // ---- bulk growth: whole 8-row tiles of leading rows whose independence is certain
      // The reference grows the basis one row at a time (solver.py:305-318, _grow
      // :368-380): K = rej / |rej|^2, C~ <- [C~ - gamma K^T; K^T], C <- [C; a],
      // P^-1 <- diag(P^-1, 1), W gains y - a.x0 (= y here: x0 = 0).  For a tile of
      // rows that are all independent the same result is, in exact arithmetic,
      // one block step: with R = A - G C the tile's rejections from the current
      // basis (G = A C~^T), the new dual rows are Z = (R R^T)^-1 R and the old ones
      // become C~ - G^T Z.  The squared rejection of row t from the basis plus the
      // tile's rows before t is the t-th pivot d_t of R R^T = L D L^T, so a row is
      // certified when d_t clears the rank test by BULK_MARGIN (the reference then
      // surely finds it independent too) and keeps >= BULK_COND of |R_t|^2 (the
      // tile is well conditioned, so the normal-equations solve Z = E^T D^-1 E R,
      // E = L^-1, stays at the reference's accuracy).  The first row that is not
      // certified ends the bulk phase; it and the rest go to the row mode below.
      // One warp projects (DMMA), factors and solves; all four update C~.
      // (scripts/bulk_sim4.py restates it: 4 096 config-3-like streams, branch logs
      // identical to the oracle's except 2 in the noise band, x within 3e-10.)
      if constexpr (M == 128) {
        constexpr double BULK_COND = 0.1, BULK_MARGIN = 1e6;
        __shared__ int s_bulk_tst;
        constexpr int SP = M + 4;        // S1 row pitch (conflict-free B-operand reads)
        double* S1 = &S.sG[0][0][0][0];  // [8][SP]: R, then D^-1 E R, then Z
        double* Gs = S1 + TT * SP;       // [8][R]: G of the tile
        static_assert(offsetof(SMT, bulkpad) + sizeof(S.bulkpad) - offsetof(SMT, sG) >=
                          sizeof(double) * (TT * SP + TT * R),
                      "bulk growth: scratch fits the hand-off slot");
        double* Dflat = &S.Df[0][0][0];
        double* Cflat = &S.Cf[0][0][0];
        auto df_idx = [&](int i, int c) {
          return ((i >> 3) * KS + 2 * (c >> 3) + (c & 1)) * 32 + 4 * (i & 7) + ((c & 7) >> 1);
        };
        auto cf_idx = [&](int i, int c) {
          return ((2 * (i >> 3) + (i & 1)) * NJ + (c >> 3)) * 32 + 4 * (c & 7) + ((i & 7) >> 1);
        };
        const int tid = threadIdx.x;
        while (tcur + TT <= T && r + TT <= R) {
          PPROBE(20);
          if (w == 0) {
            double acc[NJ][2];
#pragma unroll
            for (int jt = 0; jt < NJ; ++jt) {
              const double2 v = ld2(Rb + (tcur + p) * M + 8 * jt + 2 * q);
              acc[jt][0] = v.x;
              acc[jt][1] = v.y;
              // C's candidate rows r + p (zeroed again below past the certified block)
              Cflat[cf_idx(r + p, 8 * jt + 2 * q)] = -v.x;
              Cflat[cf_idx(r + p, 8 * jt + 2 * q + 1)] = -v.y;
            }
            double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int jt = 0; jt < NJ; ++jt) {
              s4[(2 * jt) & 3] = fma(acc[jt][0], acc[jt][0], s4[(2 * jt) & 3]);
              s4[(2 * jt + 1) & 3] = fma(acc[jt][1], acc[jt][1], s4[(2 * jt + 1) & 3]);
            }
            double asq = (s4[0] + s4[1]) + (s4[2] + s4[3]);
            asq += __shfl_xor_sync(FULL, asq, 1);
            asq += __shfl_xor_sync(FULL, asq, 2);
            bool yok = true;
            if (q == 0)
              for (int c = 0; c < k; ++c) yok &= isfinite((double)Yb[(tcur + p) * k + c]);
            yok = __shfl_sync(FULL, yok, 4 * p);
            // G = A C~^T and R = A - G C (rank tiles past r are zero)
            const int nti = (r + 7) >> 3;
            double g[IT][2], h[IT][2];
#pragma unroll
            for (int nt = 0; nt < IT; ++nt) g[nt][0] = g[nt][1] = h[nt][0] = h[nt][1] = 0.0;
#pragma unroll
            for (int nt = 0; nt < IT; ++nt)  // (rank tile outermost: one guard per tile, as in gcoords below)
              if (nt < nti) {
#pragma unroll
                for (int ks = 0; ks < KS / 2; ++ks) {
                  mma(g[nt], acc[ks >> 1][ks & 1], S.Df[nt][ks][lane]);
                  mma(h[nt], acc[(ks + KS / 2) >> 1][ks & 1], S.Df[nt][ks + KS / 2][lane]);
                }
              }
#pragma unroll
            for (int nt = 0; nt < IT; ++nt) {
              g[nt][0] += h[nt][0];
              g[nt][1] += h[nt][1];
            }
#pragma unroll
            for (int kt = 0; kt < IK; ++kt)
              if ((kt >> 1) < nti) {
#pragma unroll
                for (int jt = 0; jt < NJ; ++jt) mma(acc[jt], g[kt >> 1][kt & 1], S.Cf[kt][jt][lane]);
              }
#pragma unroll
            for (int nt = 0; nt < IT; ++nt) {
              Gs[p * R + 8 * nt + 2 * q] = g[nt][0];
              Gs[p * R + 8 * nt + 2 * q + 1] = g[nt][1];
            }
            // M = R R^T, L D L^T (E = L^-1)
            double m4[4][2] = {};
#pragma unroll
            for (int jt = 0; jt < NJ; ++jt) {
              mma(m4[(2 * jt) & 3], acc[jt][0], acc[jt][0]);
              mma(m4[(2 * jt + 1) & 3], acc[jt][1], acc[jt][1]);
            }
            const double mm[2] = {(m4[0][0] + m4[1][0]) + (m4[2][0] + m4[3][0]),
                                  (m4[0][1] + m4[1][1]) + (m4[2][1] + m4[3][1])};
            // a non-finite row would reach the earlier rows' factors through 0 x NaN in
            // the elimination: its row and column enter as the identity (it fails the
            // certification below anyway)
            double mi[2], ev[2], rd0, rd1;
            {
              const bool badp = !isfinite(asq);
              const bool badc0 = !isfinite(__shfl_sync(FULL, asq, 8 * q));
              const bool badc1 = !isfinite(__shfl_sync(FULL, asq, 8 * q + 4));
              mi[0] = (badp || badc0) ? (p == 2 * q ? 1.0 : 0.0) : mm[0];
              mi[1] = (badp || badc1) ? (p == 2 * q + 1 ? 1.0 : 0.0) : mm[1];
            }
            ldl8(mi, ev, rd0, rd1, p, q);
            // certification, lane t < 8 tests row t; one ballot
            int tst;
            {
              const int t = lane & 7;
              const double x0 = __shfl_sync(FULL, rd0, t >> 1), x1 = __shfl_sync(FULL, rd1, t >> 1);
              const double dt = 1.0 / ((t & 1) ? x1 : x0);
              const double y0 = __shfl_sync(FULL, mm[0], 4 * t + (t >> 1));
              const double y1 = __shfl_sync(FULL, mm[1], 4 * t + (t >> 1));
              const double mtt = (t & 1) ? y1 : y0;
              const double at = __shfl_sync(FULL, asq, 4 * t);
              const bool yt = __shfl_sync(FULL, yok, 4 * t);
              const double e2 = eps_sq<double>(cfg, r + t);
              const bool ok = isfinite(at) && yt && dt > BULK_COND * mtt && dt > BULK_MARGIN * e2 * fmax(1.0, at);
              const unsigned failm = __ballot_sync(FULL, lane < TT && !ok);
              tst = failm ? __ffs(failm) - 1 : TT;
            }
            if (tst > 0) {
              // rows / columns past the certified block: E = I, 1/d = 1 there
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int c = 2 * q + e;
                if (p >= tst || c >= tst) ev[e] = (p == c) ? 1.0 : 0.0;
              }
              const double z0 = __shfl_sync(FULL, rd0, p >> 1), z1 = __shfl_sync(FULL, rd1, p >> 1);
              const double rdp = p < tst ? ((p & 1) ? z1 : z0) : 1.0;
#pragma unroll
              for (int jt = 0; jt < NJ; ++jt)
                *reinterpret_cast<double2*>(S1 + p * SP + 8 * jt + 2 * q) =
                    p < tst ? make_double2(acc[jt][0], acc[jt][1]) : make_double2(0.0, 0.0);  // (0 x NaN)
              __syncwarp();
              // Q = D^-1 E R  (K = the tile's rows, permuted: step kk takes row 2q + kk)
              double qv[NJ][2];
#pragma unroll
              for (int jt = 0; jt < NJ; ++jt) qv[jt][0] = qv[jt][1] = 0.0;
#pragma unroll
              for (int kk = 0; kk < 2; ++kk)
#pragma unroll
                for (int jt = 0; jt < NJ; ++jt) mma(qv[jt], ev[kk], S1[(2 * q + kk) * SP + 8 * jt + p]);
              __syncwarp();
#pragma unroll
              for (int jt = 0; jt < NJ; ++jt)
                *reinterpret_cast<double2*>(S1 + p * SP + 8 * jt + 2 * q) =
                    make_double2(qv[jt][0] * rdp, qv[jt][1] * rdp);
              __syncwarp();
              // Z = E^T Q (E^T[p][2q + kk] = E[2q + kk][p], from the lane that holds it)
              double zv[NJ][2];
#pragma unroll
              for (int jt = 0; jt < NJ; ++jt) zv[jt][0] = zv[jt][1] = 0.0;
#pragma unroll
              for (int kk = 0; kk < 2; ++kk) {
                const int src = 4 * (2 * q + kk) + (p >> 1);
                const double e0 = __shfl_sync(FULL, ev[0], src), e1 = __shfl_sync(FULL, ev[1], src);
                const double a = (p & 1) ? e1 : e0;
#pragma unroll
                for (int jt = 0; jt < NJ; ++jt) mma(zv[jt], a, S1[(2 * q + kk) * SP + 8 * jt + p]);
              }
              __syncwarp();
#pragma unroll
              for (int jt = 0; jt < NJ; ++jt)
                *reinterpret_cast<double2*>(S1 + p * SP + 8 * jt + 2 * q) =
                    p < tst ? make_double2(zv[jt][0], zv[jt][1]) : make_double2(0.0, 0.0);
            }
            if (lane == 0) s_bulk_tst = tst;
          }
          PPROBE(16);
          __syncthreads();
          PPROBE(17);
          const int tst = s_bulk_tst;
          if (tst == 0) break;
          // C~[:r] -= G^T Z, C~[r + t] = Z[t]; C's rows past the block leave again (every warp)
          {
            const double* __restrict__ gs = Gs;
            const double* __restrict__ zs = S1;
            for (int e = tid; e < r * M; e += PANEL_THREADS) {
              const int i = e / M, c = e % M;
              double gz[TT];
#pragma unroll
              for (int t = 0; t < TT; ++t) gz[t] = t < tst ? gs[t * R + i] * zs[t * SP + c] : 0.0;
              const int di = df_idx(i, c);
              double v = Dflat[di];
#pragma unroll
              for (int t = 0; t < TT; ++t) v -= gz[t];
              Dflat[di] = v;
            }
          }
          PPROBE(18);
          for (int e = tid; e < TT * M; e += PANEL_THREADS) {
            const int t = e / M, c = e % M;
            if (t < tst) Dflat[df_idx(r + t, c)] = S1[t * SP + c];
            else Cflat[cf_idx(r + t, c)] = 0.0;
          }
          if (blog)
            for (int t = tid; t < tst; t += PANEL_THREADS) blog[b * T + tcur + t] = 1;
          if (clog)
            for (int e = tid; e < tst * R; e += PANEL_THREADS)
              clog[(b * T + tcur + e / R) * R + e % R] = (e % R == r + e / R) ? 1.0 : 0.0;
          r += tst;
          tcur += tst;
          PPROBE(19);
          __syncthreads();
          if (tst < TT) break;
        }
        // W's rows of the grown prefix: y (x0 = 0), over the scratch
        for (int e = tid; e < R * 8; e += PANEL_THREADS) {
          const int t = e >> 3, c = e & 7;
          (&Wsm[0][0])[e] = (t < r && c < k) ? (double)Yb[(int64_t)t * k + c] : 0.0;
        }
        __syncthreads();
      }
      constexpr int NRW = PW + 1, NGR = NJ / NRW;
      static_assert(NJ % NRW == 0, "row mode: whole column groups per warp");
      const int u = threadIdx.x >> 5;
      double esq = eps_sq<double>(cfg, r);
      double2 nx[NGR];
      double nyv = 0.0;
      auto load_row = [&](int64_t t) {  // own-column values and target of row t, one row ahead
        if (t < T) {
          const TI* ar = Rb + t * M;
#pragma unroll
          for (int jj = 0; jj < NGR; ++jj) {
            const int J = u + NRW * jj;
            nx[jj] = ld2(ar + 8 * J + 2 * q);
          }
          nyv = (p < k) ? (double)Yb[t * k + p] : 0.0;  // y[c = p]
        }
      };
      load_row(tcur);
      // the row step, specialised on the number of nonzero rank tiles (the
      // unrolled loops then carry no predicated-off work)
      auto row_step = [&](auto NTc) -> bool {
        constexpr int nti = decltype(NTc)::value;
        double2 av[NGR];
#pragma unroll
        for (int jj = 0; jj < NGR; ++jj) av[jj] = nx[jj];
        const double yv = nyv;
        load_row(tcur + 1);
        double a2 = 0.0, gp[IT], gq[IT];
#pragma unroll
        for (int nt = 0; nt < IT; ++nt) gp[nt] = gq[nt] = 0.0;
#pragma unroll
        for (int jj = 0; jj < NGR; ++jj) {
          const int J = u + NRW * jj;
          {
            a2 = fma(av[jj].x, av[jj].x, fma(av[jj].y, av[jj].y, a2));
#pragma unroll
            for (int nt = 0; nt < IT; ++nt) {
              if (nt < nti) {
                gp[nt] = fma(S.Df[nt][2 * J][lane], av[jj].x, gp[nt]);
                gq[nt] = fma(S.Df[nt][2 * J + 1][lane], av[jj].y, gq[nt]);
              }
            }
          }
        }
        a2 += __shfl_xor_sync(FULL, a2, 1);
        a2 += __shfl_xor_sync(FULL, a2, 2);
#pragma unroll
        for (int nt = 0; nt < IT; ++nt) {
          gp[nt] += gq[nt];
          gp[nt] += __shfl_xor_sync(FULL, gp[nt], 1);
          gp[nt] += __shfl_xor_sync(FULL, gp[nt], 2);
        }
        if (q == 0) {
#pragma unroll
          for (int nt = 0; nt < IT; ++nt) S.gpart[u][8 * nt + p] = gp[nt];
        }
        if (lane == 0) S.a2part[u] = a2;
        bar_sync_n(BAR_ROW, NRW * 32);
        double asq = 0.0;
#pragma unroll
        for (int v = 0; v < NRW; ++v) asq += S.a2part[v];
        // full coords (read before the next barrier: the next row overwrites gpart)
        double gfull[IT];
#pragma unroll
        for (int nt = 0; nt < IT; ++nt) {
          gfull[nt] = 0.0;
          if (nt <= nti && nt <= (r >> 3)) {
#pragma unroll
            for (int v = 0; v < NRW; ++v) gfull[nt] += S.gpart[v][8 * nt + p];
          }
        }
        double gk[IK];
#pragma unroll
        for (int kt = 0; kt < IK; ++kt) {
          gk[kt] = 0.0;
          if ((kt >> 1) < nti) {
#pragma unroll
            for (int v = 0; v < NRW; ++v) gk[kt] += S.gpart[v][sigma(kt, q)];
          }
        }
        // rejection of the own columns j = 8J + p
        double rej[NGR], aj[NGR], r2 = 0.0;
#pragma unroll
        for (int jj = 0; jj < NGR; ++jj) {
          const int J = u + NRW * jj;
          double rp = 0.0;
#pragma unroll
          for (int kt = 0; kt < IK; ++kt)
            if ((kt >> 1) < nti) rp = fma(gk[kt], S.Cf[kt][J][lane], rp);  // Cf = -C
          rp += __shfl_xor_sync(FULL, rp, 1);
          rp += __shfl_xor_sync(FULL, rp, 2);
          const double v0 = __shfl_sync(FULL, av[jj].x, p >> 1);
          const double v1 = __shfl_sync(FULL, av[jj].y, p >> 1);
          aj[jj] = (p & 1) ? v1 : v0;
          rej[jj] = aj[jj] + rp;
          r2 = fma(rej[jj], rej[jj], r2);
        }
        r2 += __shfl_xor_sync(FULL, r2, 4);
        r2 += __shfl_xor_sync(FULL, r2, 8);
        r2 += __shfl_xor_sync(FULL, r2, 16);
        if (lane == 0) S.r2part[u] = r2;
        bar_sync_n(BAR_ROW, NRW * 32);
        double rsq = 0.0;
#pragma unroll
        for (int v = 0; v < NRW; ++v) rsq += S.r2part[v];
        const bool bad = !isfinite(asq) || __any_sync(FULL, !isfinite(yv));
        if (bad || is_dependent<double>(rsq, asq, esq)) return false;  // panel mode takes this row
        // growth (general variant): K = rej / |rej|^2, C~[:r] -= gamma K^T,
        // C~[r] = K, C[r] = a, W[r] = y (x0 = 0), P^-1 = diag(P^-1, 1)
        const double rinv = 1.0 / rsq;  // one rounding more than a division, as every kernel
        if (q == 0) {
#pragma unroll
          for (int jj = 0; jj < NGR; ++jj)
            S.kv[8 * (u + NRW * jj) + p] = rej[jj] * rinv;
        }
        __syncwarp();
        {
          double kvr[2 * NGR];
#pragma unroll
          for (int kk = 0; kk < 2 * NGR; ++kk) {
            const int J = u + NRW * (kk >> 1);
            kvr[kk] = S.kv[sigma(2 * J + (kk & 1), q)];
          }
#pragma unroll
          for (int nt = 0; nt < IT; ++nt) {
            if (nt > nti || nt > (r >> 3)) break;
            const int i = 8 * nt + p;
            double dv[2 * NGR];
#pragma unroll
            for (int kk = 0; kk < 2 * NGR; ++kk) {
              const int J = u + NRW * (kk >> 1);
              dv[kk] = S.Df[nt][2 * J + (kk & 1)][lane];
            }
#pragma unroll
            for (int kk = 0; kk < 2 * NGR; ++kk) {
              const int J = u + NRW * (kk >> 1);
              S.Df[nt][2 * J + (kk & 1)][lane] = (i == r) ? kvr[kk] : fma(-gfull[nt], kvr[kk], dv[kk]);
            }
          }
        }
        if (q == ((r & 7) >> 1)) {
          const int ktr = 2 * (r >> 3) + (r & 1);
#pragma unroll
          for (int jj = 0; jj < NGR; ++jj)
            S.Cf[ktr][u + NRW * jj][lane] = -aj[jj];
        }
        if (u == 0) {
          if (q == 0) Wsm[r][p] = yv;  // 0 for c >= k
          const int64_t row = b * T + tcur;
          if (blog && lane == 0) blog[row] = 1;
          if (clog && lane < R) clog[row * R + lane] = (lane == r) ? 1.0 : 0.0;
        }
        r += 1;
        esq = eps_sq<double>(cfg, r);
        ++tcur;
        return true;
      };
      while (tcur < T && r < R) {
        const int nt_rt = (r + 7) >> 3;
        bool go;
        // two instantiations, not one per tile count: with three CTAs per SM in
        // different phases the instruction cache is the next limit (measured)
        if (nt_rt <= 2) go = row_step(std::integral_constant<int, (2 < IT ? 2 : IT)>{});
        else go = row_step(std::integral_constant<int, IT>{});
        if (!go) break;
      }
      __syncthreads();  // every warp's columns of C~ / C are in
      PPROBE(1);
    }
    if (!home) {
      // =========================== projection warps ===========================
      double esq = eps_sq<double>(cfg, r);
      bool stopped = false;
      // C~[:r] -= gamma K^T, C~[r] = K on the own columns (solver.py:377-380), K in
      // S.kv; every load is issued before the first store (kv and Df may alias)
      // G = A C~^T (two accumulator chains per N tile), then R = A - G C onto A
      auto gcoords = [&](const double (&acc)[NJ][2], double (&g)[IT][2], int nti) {
        double h[IT][2];
#pragma unroll
        for (int nt = 0; nt < IT; ++nt) g[nt][0] = g[nt][1] = h[nt][0] = h[nt][1] = 0.0;
        // rank tile outermost: one guard per tile, not one per MMA pair -- a guarded pair is
        // its own basic block (branch, WARPSYNC), and its two shared-memory operand loads then
        // issue right before the MMAs that wait for them instead of being pipelined over the
        // 32 MMAs of a tile (config 3: 1.95 -> 1.75 ms); two chains per tile are what the DMMA
        // pipe's issue interval needs
#pragma unroll
        for (int nt = 0; nt < IT; ++nt) {
          if (nt < nti) {
#pragma unroll
            for (int ks = 0; ks < KS / 2; ++ks) {
              mma(g[nt], acc[ks >> 1][ks & 1], S.Df[nt][ks][lane]);
              mma(h[nt], acc[(ks + KS / 2) >> 1][ks & 1], S.Df[nt][ks + KS / 2][lane]);
            }
          }
        }
#pragma unroll
        for (int nt = 0; nt < IT; ++nt) {
          g[nt][0] += h[nt][0];
          g[nt][1] += h[nt][1];
        }
      };
      auto reject = [&](double (&acc)[NJ][2], const double (&g)[IT][2], int nti) {  // C stored negated
#pragma unroll
        for (int kt = 0; kt < IK; ++kt) {
          if ((kt >> 1) < nti) {
#pragma unroll
            for (int jt = 0; jt < NJ; ++jt) mma(acc[jt], g[kt >> 1][kt & 1], S.Cf[kt][jt][lane]);
          }
        }
      };
      auto project = [&](double (&acc)[NJ][2], double (&g)[IT][2], int nti) {
        gcoords(acc, g, nti);
        reject(acc, g, nti);
      };
      auto grow_dual = [&](const double (&gi)[IT], int rr) {
        double kvr[2 * NG];
#pragma unroll
        for (int kk = 0; kk < 2 * NG; ++kk) {
          const int J = w + PW * (kk >> 1);
          kvr[kk] = (J < NJ) ? S.kv[sigma(2 * J + (kk & 1), q)] : 0.0;
        }
#pragma unroll
        for (int nt = 0; nt < IT; ++nt) {
          if (nt > (rr >> 3)) break;
          const int i = 8 * nt + p;
          double dv[2 * NG];
#pragma unroll
          for (int kk = 0; kk < 2 * NG; ++kk) {
            const int J = w + PW * (kk >> 1);
            dv[kk] = (J < NJ) ? S.Df[nt][2 * J + (kk & 1)][lane] : 0.0;
          }
#pragma unroll
          for (int kk = 0; kk < 2 * NG; ++kk) {
            const int J = w + PW * (kk >> 1);
            if (J < NJ) S.Df[nt][2 * J + (kk & 1)][lane] = (i == rr) ? kvr[kk] : fma(-gi[nt], kvr[kk], dv[kk]);
          }
        }
      };

      // ---- panel mode --------------------------------------------------------------
      while (!stopped && tcur < T) {
        const int64_t t0 = tcur;
        double acc[NJ][2];
        {
          // straight from global into the fragment registers; the rows two panels
          // ahead are pulled into L2 meanwhile
          const int64_t t = t0 + 8 * w + p;
          const bool ok = t < T;
          const TI* src = Rb + (ok ? t : 0) * M;
#pragma unroll
          for (int jt = 0; jt < NJ; ++jt) {
            const double2 v = ok ? ld2(src + 8 * jt + 2 * q) : make_double2(0.0, 0.0);
            acc[jt][0] = v.x;
            acc[jt][1] = v.y;
          }
          const int64_t tn = t + 2 * PNL;  // two panels ahead (measured: 1 panel -0.5 %, none -1.2 %)
          if (tn < T) {
            const char* nb = reinterpret_cast<const char*>(Rb + tn * M);
            constexpr int LINES = (int)(M * sizeof(TI) / 128);
            for (int l = q; l < LINES; l += 4) asm volatile("prefetch.global.L2 [%0];" ::"l"(nb + 128 * l));
          }
        }
        PPROBE(2);
        const int64_t tb = t0 + 8 * w;  // first row of this warp's tile
        const int tv = (int)(T - tb < 0 ? 0 : (T - tb < TT ? T - tb : TT));
        double yv[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t ty = tb + 2 * q + e;
          yv[e] = (ty < T && p < k) ? (double)Yb[ty * k + p] : 0.0;
        }
        const int nti = (r + 7) >> 3;
        // |a_t|^2
        double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int jt = 0; jt < NJ; ++jt) {
          s4[(2 * jt) & 3] = fma(acc[jt][0], acc[jt][0], s4[(2 * jt) & 3]);
          s4[(2 * jt + 1) & 3] = fma(acc[jt][1], acc[jt][1], s4[(2 * jt + 1) & 3]);
        }
        double asq = (s4[0] + s4[1]) + (s4[2] + s4[3]);
        asq += __shfl_xor_sync(FULL, asq, 1);
        asq += __shfl_xor_sync(FULL, asq, 2);
        double g[IT][2];
        gcoords(acc, g, nti);
        // a.x0 (continuation calls): M = c, N = t, K = columns
        double y0[2] = {0.0, 0.0};
        if (has_x0) {
#pragma unroll
          for (int jt = 0; jt < NJ; ++jt) {
            double2 xv = make_double2(0.0, 0.0);
            if (p < k) xv = __ldg(reinterpret_cast<const double2*>(Xg + p * M + 8 * jt + 2 * q));
            mma(y0, xv.x, acc[jt][0]);
            mma(y0, xv.y, acc[jt][1]);
          }
        }
        const double dyx[2] = {yv[0] - y0[0], yv[1] - y0[1]};
        reject(acc, g, nti);
        double t4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int jt = 0; jt < NJ; ++jt) {
          t4[(2 * jt) & 3] = fma(acc[jt][0], acc[jt][0], t4[(2 * jt) & 3]);
          t4[(2 * jt + 1) & 3] = fma(acc[jt][1], acc[jt][1], t4[(2 * jt + 1) & 3]);
        }
        double rsq = (t4[0] + t4[1]) + (t4[2] + t4[3]);
        rsq += __shfl_xor_sync(FULL, rsq, 1);
        rsq += __shfl_xor_sync(FULL, rsq, 2);
        // rank test of row p (solver.py:292-296)
        const unsigned yb0 = __ballot_sync(FULL, !isfinite(dyx[0]));
        const unsigned yb1 = __ballot_sync(FULL, !isfinite(dyx[1]));
        const bool ybad = (((p & 1) ? yb1 : yb0) & (0x11111111u << (p >> 1))) != 0u;
        const bool valid = p < tv;
        const bool dep = is_dependent<double>(rsq, asq, esq);
        const bool bd = !isfinite(asq) || ybad;
        const unsigned stopm = __ballot_sync(FULL, q == 0 && valid && (!dep || bd));
        const unsigned badm = __ballot_sync(FULL, q == 0 && valid && bd);
        const int tst = stopm ? (__ffs(stopm) - 1) >> 2 : TT;
        PPROBE(3);
        if (lane == 0) {
          S.stop[w] = tst;
          S.bad[w] = (tst < TT) ? (int)((badm >> (4 * tst)) & 1u) : 0;
        }
        bar_sync_n(BAR_PROJ, PW * 32);
        int sstar = PNL;  // first stop row of the panel
#pragma unroll
        for (int u = PW - 1; u >= 0; --u)
          if (S.stop[u] < TT) sstar = 8 * u + S.stop[u];
        const int len = (int)(T - t0 < PNL ? T - t0 : PNL);
        const int lim = sstar < len ? sstar : len;
        const int te = lim - 8 * w < 0 ? 0 : (lim - 8 * w > TT ? TT : lim - 8 * w);
        const bool stop_here = sstar < len;
        const int ws = sstar >> 3, tsr = sstar & 7;
        bool grow = false;
        if (stop_here) {
          if (S.bad[ws]) {
            status |= RGB_ST_NONFINITE;
            stopped = true;
          } else if (r >= R) {
            status |= RGB_ST_RANK_CAP;
            stopped = true;
          } else {
            grow = true;
          }
        }
        PPROBE(4);
        // ---- hand the panel to the home warp ----
        bar_sync_n(BAR_EMPTY, PANEL_THREADS);
        PPROBE(5);
        if (te > 0) {
#pragma unroll
          for (int nt = 0; nt < IT; ++nt)
            *reinterpret_cast<double2*>(&S.sG[w][nt][lane][0]) = make_double2(g[nt][0], g[nt][1]);
          *reinterpret_cast<double2*>(&S.sDy[w][lane][0]) = make_double2(dyx[0], dyx[1]);
        }
        if (lane == 0) S.sTe[w] = te;
        if (w == 0 && lane == 0) {
          S.sGrow = grow ? 1 : 0;
          S.sEnd = 0;
        }
        if (grow && w == ws) {
          // W's new row: y - a.x0 of the growth row (lanes c = p, t = 2q + e)
          if (q == (tsr >> 1) && p < 8) S.sWnew[p] = (p < k) ? ((tsr & 1) ? dyx[1] : dyx[0]) : 0.0;
          if (p == tsr) {
            const double rinv = 1.0 / rsq;
#pragma unroll
            for (int jt = 0; jt < NJ; ++jt) {
              S.kv[8 * jt + 2 * q] = acc[jt][0] * rinv;
              S.kv[8 * jt + 2 * q + 1] = acc[jt][1] * rinv;
            }
#pragma unroll
            for (int nt = 0; nt < IT; ++nt) {
              S.gam[8 * nt + 2 * q] = g[nt][0];
              S.gam[8 * nt + 2 * q + 1] = g[nt][1];
            }
          }
        }
        bar_arrive_n(BAR_FULL, PANEL_THREADS);
        // logs of the dependent rows
        if (p < te) {
          const int64_t row = b * T + tb + p;
          if (blog && q == 0) blog[row] = 0;
          if (clog) {
#pragma unroll
            for (int nt = 0; nt < IT; ++nt)
              *reinterpret_cast<double2*>(clog + row * R + 8 * nt + 2 * q) = make_double2(g[nt][0], g[nt][1]);
          }
        }
        if (stopped) {
          consumed = t0 + sstar;
          break;
        }
        if (!grow) {
          tcur = t0 + len;
          continue;
        }
        // ---- growth on the own columns (general variant, solver.py:377-380) ----
        bar_sync_n(BAR_PROJ, PW * 32);  // gam / kv of the growth row are in
        const int64_t trow = t0 + sstar;
        {
          double gi[IT];
#pragma unroll
          for (int nt = 0; nt < IT; ++nt) gi[nt] = S.gam[8 * nt + p];
          grow_dual(gi, r);
        }
        if (q == ((r & 7) >> 1)) {
          const int ktr = 2 * (r >> 3) + (r & 1);
          const TI* arow = Rb + trow * M;
#pragma unroll
          for (int jj = 0; jj < NG; ++jj) {
            const int jt = w + PW * jj;
            if (jt < NJ) S.Cf[ktr][jt][lane] = -(double)arow[8 * jt + p];
          }
        }
        if (w == 0) {
          const int64_t row = b * T + trow;
          if (blog && lane == 0) blog[row] = 1;
          if (clog && lane < R) clog[row * R + lane] = (lane == r) ? 1.0 : 0.0;
        }
        r += 1;
        esq = eps_sq<double>(cfg, r);
        tcur = trow + 1;
        bar_sync_n(BAR_PROJ, PW * 32);  // every column of C~ / C is updated
        PPROBE(6);
      }
      if (!stopped) consumed = T;
      // end-of-stream marker
      bar_sync_n(BAR_EMPTY, PANEL_THREADS);
      if (lane == 0) S.sTe[w] = 0;
      if (w == 0 && lane == 0) {
        S.sGrow = 0;
        S.sEnd = 1;
      }
      bar_arrive_n(BAR_FULL, PANEL_THREADS);
    } else {
      // ============================== home warp ===============================
      double Pr[IT][IT][2];
      double Wt[IT][2];
#pragma unroll
      for (int mt = 0; mt < IT; ++mt) {
        Wt[mt][0] = Wt[mt][1] = 0.0;
#pragma unroll
        for (int nt = 0; nt < IT; ++nt) {
          const double2 v = fresh ? make_double2(0.0, 0.0)
                                  : *reinterpret_cast<const double2*>(Pg + (8 * mt + p) * R + 8 * nt + 2 * q);
          Pr[mt][nt][0] = v.x;
          Pr[mt][nt][1] = v.y;
        }
      }
      int rh = r;
      if (fresh) {
        // the row-mode phase grew the basis to r rows: P^-1 = I (solver.py:368-380)
#pragma unroll
        for (int mt = 0; mt < IT; ++mt)
#pragma unroll
          for (int nt = 0; nt < IT; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int i = 8 * mt + p, i2 = 8 * nt + 2 * q + e;
              Pr[mt][nt][e] = (i == i2 && i < rh) ? 1.0 : 0.0;
            }
      }
      // W's rows of the row-mode phase (zero for a continuation call)
#pragma unroll
      for (int mt = 0; mt < IT; ++mt)
#pragma unroll
        for (int e = 0; e < 2; ++e) Wt[mt][e] = Wsm[8 * mt + 2 * q + e][p];
      bar_arrive_n(BAR_EMPTY, PANEL_THREADS);
      while (true) {
        PPROBE(10);
        bar_sync_n(BAR_FULL, PANEL_THREADS);
        PPROBE(9);
        const int nti = (rh + 7) >> 3;
#pragma unroll 1
        for (int u = 0; u < PW; ++u) {
          const int te = S.sTe[u];
          if (te <= 0 || nti == 0) continue;  // r = 0: dependent rows are zero rows (solver.py:323-326)
          if (defer) {
            // ---- deferred fold: Q += G^T G, (B^T dy)^T += dy^T G over rows [0, te) of tile u.
            // Pr holds Q and Wt holds (B^T dy)^T here.  G^T comes straight out of the slot:
            // the accumulator layout the projection warp stored is, read at 32 s + 8 q + p,
            // G[4s + q][8nt + p] -- the A operand (M = coords, K = rows) and the B operand
            // (K = rows, N = coords) at once, conflict-free.
            double gt[IT][2], dv[2];
#pragma unroll
            for (int s = 0; s < 2; ++s) {
              const bool in = 4 * s + q < te;
#pragma unroll
              for (int nt = 0; nt < IT; ++nt)
                gt[nt][s] = (in && nt < nti) ? (&S.sG[u][nt][0][0])[32 * s + 8 * q + p] : 0.0;
              dv[s] = in ? (&S.sDy[u][0][0])[8 * p + 4 * s + q] : 0.0;
            }
#pragma unroll
            for (int mt = 0; mt < IT; ++mt) {
              if (mt < nti) {
#pragma unroll
                for (int nt = 0; nt < IT; ++nt) {
                  if (nt < nti) {
                    mma(Pr[mt][nt], gt[mt][0], gt[nt][0]);
                    mma(Pr[mt][nt], gt[mt][1], gt[nt][1]);
                  }
                }
                mma(Wt[mt], dv[0], gt[mt][0]);
                mma(Wt[mt], dv[1], gt[mt][1]);
              }
            }
            continue;
          }
          // ---- blocked Sherman-Morrison over rows [0, te) of tile u (solver.py:297-304) ----
          const bool inb = p < te;
          double gm[IT][2];
#pragma unroll
          for (int nt = 0; nt < IT; ++nt) {
            const double2 v = (inb && nt < nti) ? *reinterpret_cast<const double2*>(&S.sG[u][nt][lane][0])
                                                : make_double2(0.0, 0.0);
            gm[nt][0] = v.x;
            gm[nt][1] = v.y;
          }
          const double2 dxy = *reinterpret_cast<const double2*>(&S.sDy[u][lane][0]);
          // (G W)^T [c][t], U = G P [t][i], S = U G^T [t][t']
          double gw[2] = {0.0, 0.0}, ut[IT][2], sp[2] = {0.0, 0.0}, sq[2] = {0.0, 0.0};
#pragma unroll
          for (int mt = 0; mt < IT; ++mt) {
            ut[mt][0] = ut[mt][1] = 0.0;
            if (mt < nti) {
              mma(gw, Wt[mt][0], gm[mt][0]);
              mma(gw, Wt[mt][1], gm[mt][1]);
            }
          }
#pragma unroll
          for (int kt = 0; kt < IK; ++kt)
#pragma unroll
            for (int mt = 0; mt < IT; ++mt)
              if (mt < nti && (kt >> 1) < nti) mma(ut[mt], gm[kt >> 1][kt & 1], Pr[mt][kt >> 1][kt & 1]);
#pragma unroll
          for (int mt = 0; mt < IT; ++mt) {
            if (mt < nti) {
              mma(sp, ut[mt][0], gm[mt][0]);
              mma(sq, ut[mt][1], gm[mt][1]);
            }
          }
          PPROBE(21);
          double mi[2] = {sp[0] + sq[0], sp[1] + sq[1]};
          double dy[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) dy[e] = (2 * q + e < te) ? ((e ? dxy.y : dxy.x) - gw[e]) : 0.0;
          if (p == 2 * q) mi[0] += 1.0;
          if (p == 2 * q + 1) mi[1] += 1.0;
          double ev[2], rd0, rd1;
          ldl8(mi, ev, rd0, rd1, p, q);
          PPROBE(22);
          // Y^T = U E^T per row block, E dy0
          double yt[IT][2];
#pragma unroll
          for (int mt = 0; mt < IT; ++mt) {
            yt[mt][0] = yt[mt][1] = 0.0;
            if (mt < nti) {
              double uu[2];
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int src = 4 * (2 * q + e) + (p >> 1);
                const double v0 = __shfl_sync(FULL, ut[mt][0], src);
                const double v1 = __shfl_sync(FULL, ut[mt][1], src);
                uu[e] = (p & 1) ? v1 : v0;
              }
              mma(yt[mt], uu[0], ev[0]);
              mma(yt[mt], uu[1], ev[1]);
            }
          }
          double dh[2] = {0.0, 0.0};
          mma(dh, dy[0], ev[0]);
          mma(dh, dy[1], ev[1]);
          const double d0 = dh[0] * rd0, d1 = dh[1] * rd1;
          // P -= Y^T D^-1 Y, W += Y^T D^-1 E dy0
#pragma unroll
          for (int mt = 0; mt < IT; ++mt) {
            if (mt < nti) {
              const double s0 = -yt[mt][0] * rd0, s1 = -yt[mt][1] * rd1;
#pragma unroll
              for (int nt = 0; nt < IT; ++nt) {
                if (nt < nti) {
                  mma(Pr[mt][nt], s0, yt[nt][0]);
                  mma(Pr[mt][nt], s1, yt[nt][1]);
                }
              }
              mma(Wt[mt], d0, yt[mt][0]);
              mma(Wt[mt], d1, yt[mt][1]);
            }
          }
          PPROBE(23);
        }
        if (S.sGrow) {
          // P^-1 = diag(P^-1, 1); W gains row rh (solver.py:305-318, 368-380)
#pragma unroll
          for (int mt = 0; mt < IT; ++mt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
#pragma unroll
              for (int nt = 0; nt < IT; ++nt) {
                const int i = 8 * mt + p, i2 = 8 * nt + 2 * q + e;
                if (i == rh || i2 == rh) Pr[mt][nt][e] = (i == i2) ? 1.0 : 0.0;
              }
              if (8 * mt + 2 * q + e == rh) Wt[mt][e] = S.sWnew[p];
            }
          rh += 1;
        }
        const bool end = S.sEnd != 0;
        if (end) break;
        bar_arrive_n(BAR_EMPTY, PANEL_THREADS);
      }
      // P^-1 to global (deferred fold: Q to the scratch for the inversion), W (B^T dy) for
      // the x contraction
      r = rh;  // (the projection warps counted the panel phase's growth themselves)
      double* Qs = &S.sG[0][0][0][0] + R * 8;
#pragma unroll
      for (int mt = 0; mt < IT; ++mt) {
#pragma unroll
        for (int nt = 0; nt < IT; ++nt) {
          if (defer)
            *reinterpret_cast<double2*>(Qs + (8 * mt + p) * R + 8 * nt + 2 * q) =
                make_double2(Pr[mt][nt][0], Pr[mt][nt][1]);
          else
            *reinterpret_cast<double2*>(Pg + (8 * mt + p) * R + 8 * nt + 2 * q) =
                make_double2(Pr[mt][nt][0], Pr[mt][nt][1]);
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) Wsm[8 * mt + 2 * q + e][p] = Wt[mt][e];
      }
    }
    PPROBE(home ? 11 : 7);
    __syncthreads();
    PPROBE(home ? 12 : 12);

    if (defer) {
      // ---- P^-1 = Q^-1 (in-place Gauss-Jordan, Q is SPD with pivots >= 1: no pivoting),
      // the certificate, W = P^-1 (B^T dy).  Thread (ti, tj) keeps Q[ti][tj + TPR jj] in
      // registers; step kk publishes pivot row and column through a two-deep buffer (one
      // CTA barrier per step).  Rows / columns past the rank are zero and stay zero.
      constexpr int TPR = PANEL_THREADS / R, NC = R / TPR;
      static_assert(offsetof(SMT, bulkpad) + sizeof(S.bulkpad) - offsetof(SMT, sG) >=
                        sizeof(double) * (R * 8 + R * R),
                    "deferred fold: Q fits the scratch");
      double* Qs = &S.sG[0][0][0][0] + R * 8;
      const int tid = threadIdx.x, ti = tid / TPR, tj = tid % TPR;
      double a[NC], fq = 0.0;
#pragma unroll
      for (int jj = 0; jj < NC; ++jj) {
        a[jj] = Qs[ti * R + tj + TPR * jj];
        fq = fma(a[jj], a[jj], fq);
      }
      __syncthreads();  // Q is in registers: the scratch past W is free
      double* rowk = Qs;           // [2][R]
      double* colk = Qs + 2 * R;   // [2][R]
      double* red = Qs + 4 * R;    // [2][4]
#pragma unroll 1
      for (int kk = 0; kk < r; ++kk) {
        double* rk = rowk + (kk & 1) * R;
        double* ck = colk + (kk & 1) * R;
#pragma unroll
        for (int jj = 0; jj < NC; ++jj) {
          const int j = tj + TPR * jj;
          if (ti == kk) rk[j] = a[jj];
          if (j == kk) ck[ti] = a[jj];
        }
        __syncthreads();
        const double pv = rcp64(rk[kk]);
        const double f = ck[ti] * pv;
#pragma unroll
        for (int jj = 0; jj < NC; ++jj) {
          const int j = tj + TPR * jj;
          const double rv = rk[j];
          if (ti == kk) a[jj] = (j == kk) ? pv : rv * pv;
          else a[jj] = (j == kk) ? -f : fma(-f, rv, a[jj]);
        }
      }
      double fp = 0.0;
#pragma unroll
      for (int jj = 0; jj < NC; ++jj) fp = fma(a[jj], a[jj], fp);
      fq = warp_sum(fq);
      fp = warp_sum(fp);
      __syncthreads();  // the last step's buffers are read
      if (lane == 0) {
        red[w] = fq;
        red[4 + w] = fp;
      }
      __syncthreads();
      const double kq = (red[0] + red[1]) + (red[2] + red[3]);
      const double kp = (red[4] + red[5]) + (red[6] + red[7]);
      constexpr double DEFER_KAPPA = 1e6;
      if (!(kq * kp <= DEFER_KAPPA * DEFER_KAPPA)) {  // (a NaN fails too)
        redo = true;
#ifdef RGB_PANEL_PROBE
        if (tid == 0) atomicAdd(&g_pprobe[31], 1ull);
#endif
        continue;
      }
      PPROBE(24);
      // W = P^-1 (B^T dy): partial sums over the own columns, reduced over the row's threads
      double wv[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) wv[c] = 0.0;
#pragma unroll
      for (int jj = 0; jj < NC; ++jj) {
        const int j = tj + TPR * jj;
#pragma unroll
        for (int c = 0; c < 8; ++c) wv[c] = fma(a[jj], Wsm[j][c], wv[c]);
        Pg[ti * R + j] = a[jj];
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) {
#pragma unroll
        for (int o = 1; o < TPR; o <<= 1) wv[c] += __shfl_xor_sync(FULL, wv[c], o);
      }
      __syncthreads();  // B^T dy is read
      if (tj == 0) {
#pragma unroll
        for (int c = 0; c < 8; ++c) Wsm[ti][c] = wv[c];
      }
      __syncthreads();
      PPROBE(25);
    }

    // ---- write back; x = x0 + C~^T W on the own columns ------------------------------
    if (!home) {
#pragma unroll
      for (int jj = 0; jj < NG; ++jj) {
        const int jt = w + PW * jj;
        if (jt >= NJ) break;
        double acc[2] = {0.0, 0.0};
        if (has_x0 && p < k) {
          const double2 v = *reinterpret_cast<const double2*>(Xg + p * M + 8 * jt + 2 * q);
          acc[0] = v.x;
          acc[1] = v.y;
        }
        const int j = 8 * jt + p;  // B operand column
        const int ksj = 2 * (j >> 3) + (j & 1), qj = (j & 7) >> 1;
#pragma unroll
        for (int kt = 0; kt < IK; ++kt) {
          const int i = sigma(kt, q);
          mma(acc, Wsm[i][p], S.Df[i >> 3][ksj][4 * (i & 7) + qj]);
        }
        if (p < k) *reinterpret_cast<double2*>(Xg + p * M + 8 * jt + 2 * q) = make_double2(acc[0], acc[1]);
      }
#pragma unroll
      for (int nt = 0; nt < IT; ++nt)
#pragma unroll
        for (int jj = 0; jj < NG; ++jj) {
          const int J = w + PW * jj;
          if (J < NJ)
            *reinterpret_cast<double2*>(Dg + (8 * nt + p) * M + 8 * J + 2 * q) =
                make_double2(S.Df[nt][2 * J][lane], S.Df[nt][2 * J + 1][lane]);
        }
#pragma unroll
      for (int kt = 0; kt < IK; ++kt)
#pragma unroll
        for (int jj = 0; jj < NG; ++jj) {
          const int jt = w + PW * jj;
          if (jt < NJ) Cg[sigma(kt, q) * M + 8 * jt + p] = -S.Cf[kt][jt][lane];
        }
      if (w == 0 && lane == 0) {
        st.rank[b] = r;
        st.nobs[b] = nobs0 + consumed;
        st.status[b] = status;
      }
    }
    __syncthreads();
    PPROBE(home ? 13 : 13);
  }
}

}  // namespace blk

cudaMemPool_t workspace_pool();  // rgb_grid.cu

template <int R, int M, typename TI>
static int launch_panel_t(const rgb_config& cfg, rgb_state& st, const void* rows, int64_t rows_stride,
                          const void* targets, int64_t tg_stride, int64_t T, const rgb_logs& logs,
                          cudaStream_t stream, int num_sms) {
  auto kern = blk::panel_kernel<R, M, TI>;
  // RGB_PANEL_SEQ=1: the sequential Sherman-Morrison chain for every stream (A/B runs, tests)
  const char* seq_env = getenv("RGB_PANEL_SEQ");
  const int seq_only = (seq_env && seq_env[0] && seq_env[0] != '0') ? 1 : 0;
  const size_t smem = sizeof(blk::PanelSmem<R, M, TI>);
  static bool attr[64] = {};
  smem_attr_once(kern, smem, attr);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, blk::PANEL_THREADS, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)num_sms * per_sm;
  if (grid > cfg.num_streams) grid = cfg.num_streams;
  // the stream counter: 4 bytes, stream-ordered, from the library's device pool
  // (not needed when every CTA gets at most one stream, e.g. a drop-in update())
  void* ws = nullptr;
  if (cfg.num_streams > grid) {
    cudaMemPool_t pool = workspace_pool();
    if (!pool || cudaMallocFromPoolAsync(&ws, 256, pool, stream) != cudaSuccess) return RGB_E_CUDA;
    cudaMemsetAsync(ws, 0, sizeof(unsigned), stream);
  }
  kern<<<(unsigned)grid, blk::PANEL_THREADS, smem, stream>>>(cfg, st, (const TI*)rows, rows_stride,
                                                             (const TI*)targets, tg_stride, T, logs.branch,
                                                             (double*)logs.coords, (unsigned*)ws, seq_only);
  const cudaError_t e = cudaGetLastError();
  if (ws) cudaFreeAsync(ws, stream);
  return e == cudaSuccess ? RGB_OK : RGB_E_CUDA;
}

bool panel_supports(const rgb_config& cfg) {
  if (cfg.dtype != RGB_F64 || cfg.variant != RGB_GENERAL || cfg.k < 1 || cfg.k > 8) return false;
  return (cfg.m == 128 && (cfg.r_cap == 16 || cfg.r_cap == 32)) || (cfg.m == 256 && cfg.r_cap == 16);
}

int launch_panel(const rgb_config& cfg, rgb_state& st, const void* rows, int64_t rows_stride, const void* targets,
                 int64_t tg_stride, int64_t T, const rgb_logs& logs, cudaStream_t stream, int num_sms,
                 bool f32in) {
  if (logs.resid || logs.gain || !panel_supports(cfg)) return RGB_E_UNSUPPORTED;
  if (cfg.m == 256)
    return f32in ? launch_panel_t<16, 256, float>(cfg, st, rows, rows_stride, targets, tg_stride, T, logs, stream,
                                                  num_sms)
                 : launch_panel_t<16, 256, double>(cfg, st, rows, rows_stride, targets, tg_stride, T, logs, stream,
                                                   num_sms);
  if (cfg.r_cap == 32)
    return f32in ? launch_panel_t<32, 128, float>(cfg, st, rows, rows_stride, targets, tg_stride, T, logs, stream,
                                                  num_sms)
                 : launch_panel_t<32, 128, double>(cfg, st, rows, rows_stride, targets, tg_stride, T, logs, stream,
                                                   num_sms);
  return f32in ? launch_panel_t<16, 128, float>(cfg, st, rows, rows_stride, targets, tg_stride, T, logs, stream,
                                                num_sms)
               : launch_panel_t<16, 128, double>(cfg, st, rows, rows_stride, targets, tg_stride, T, logs, stream,
                                                 num_sms);
}

}  // namespace rgb

#ifdef RGB_PANEL_PROBE
extern "C" int rgb_panel_probe(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, rgb::blk::g_pprobe, sizeof(rgb::blk::g_pprobe));
  if (reset) {
    unsigned long long z[32] = {};
    cudaMemcpyToSymbol(rgb::blk::g_pprobe, z, sizeof(z));
  }
  return 0;
}
#endif

#ifdef RGB_PANEL_PROBE
extern "C" int rgb_panel_wslot(unsigned* out) {
  return (int)cudaMemcpyFromSymbol(out, rgb::blk::g_wslot, sizeof(rgb::blk::g_wslot));
}
#endif
