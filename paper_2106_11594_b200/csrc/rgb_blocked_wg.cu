// rgb_blocked_wg.cu -- batched rank-Greville update for wider streams: one
// warp GROUP per stream (sm_100a, fp64 tensor cores).
//
// Same algorithm as rgb_blocked.cu (8-row tiles, tensor-core projections,
// LDL^T-factored Sherman-Morrison, x = x0 + C~^T W; see its header), for
// shapes whose factors do not fit one warp: the 32*WG columns of a stream are
// split over WG warps (warp w owns columns [32w, 32w+32)), and the r_cap rows
// of P^-1 and W over the same warps by 8-row tiles.  Contractions over the
// columns (G = A C~^T, |a|^2, |rej|^2, a.x0) are reduced across the group
// through shared memory in a fixed order (deterministic); the 8x8 LDL^T is
// computed redundantly by every warp.  Built for config 3 of BASELINE.json
// (m = 128, r <= 32, k = 1): WG = 4, r_cap = 32.
//
// Per warp w, lane = 4p + q (fragment layouts of mma.m8n8k4.f64):
//   tile   As[nt][l]   = A[t=p][32w + 8nt + 2q + e]
//   C~^T   Dt[nt][kt]  = C~[8nt + p][32w + sigma(kt,q)]        registers
//   -C     Cs[kt][jt][l] = -C[sigma(kt,q)][32w + 8jt + p]     shared memory
//   P^-1   Pr[nt][e]   = P[8w + p][8nt + 2q + e]   (row block w, symmetric)
//   W^T    Wt[e]       = W[8w + 2q + e][c = p]     (row block w)
#include "rgb_mma.cuh"

namespace rgb {
namespace blk {
// phase timing (debug builds only: -DRGB_WG_PROBE): clock64 cycles per phase,
// summed over warp 0 of every CTA, read back with rgb_wg_probe()
// (scripts/probe_wg.py)
#ifdef RGB_WG_PROBE
__device__ unsigned long long g_wprobe[16];
#define WPROBE(i)                                                 \
  do {                                                            \
    if ((threadIdx.x & 31) == 0 && (threadIdx.x >> 5) == 0) {     \
      const long long now_ = clock64();                           \
      atomicAdd(&g_wprobe[i], (unsigned long long)(now_ - wp_t)); \
      wp_t = now_;                                                \
    }                                                             \
  } while (0)
#else
#define WPROBE(i) \
  do {            \
  } while (0)
#endif

template <int R, int WG, typename TI>
struct GroupSmem {
  static constexpr int M = 32 * WG, IT = R / 8, IK = R / 4;
  double Cs[WG][IK][4][32];          // -C, per warp column slice
  TI At[WG][2][4][32][2];        // row tiles, per warp column slice, 2 stages
  TI Yt[WG][2][32][2];           // targets y[t=2q+e][c=p], per warp copy
  double Gp[WG][IT][32][2];          // partial G of each warp
  double red[3][WG][32][2];          // asq / rsq / dyx partials
  double Sp[WG][32][2];              // partial S (and G W)
  double Yb[IT][32][2];              // Y^T tiles exchanged for the P update
  double gam[R];                     // independent row: coords
  double kv[M];                      //                  gain K
  double av[M];                      //                  the row
};

// GEN: general variant only; !GEN: orthogonal / orthonormal (solver.py:382-395)
template <int R, int WG, bool GEN, typename TI>
__global__ void __launch_bounds__(WG * 32, (WG <= 4 ? 3 : 1)) blocked_wg_kernel(
    rgb_config cfg, rgb_state st, const TI* __restrict__ rows, int64_t rstride,
    const TI* __restrict__ tgts, int64_t tstride, int64_t T, uint8_t* __restrict__ blog,
    double* __restrict__ clog) {
  constexpr int M = 32 * WG, IT = R / 8, IK = R / 4;
  static_assert(R % 8 == 0 && R <= 32 && IT <= WG, "shape");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  GroupSmem<R, WG, TI>& S = *reinterpret_cast<GroupSmem<R, WG, TI>*>(smem_raw);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int p = lane >> 2, q = lane & 3;
  const int k = cfg.k;
  const int j0 = 32 * w;

#ifdef RGB_WG_PROBE
  long long wp_t = clock64();
#endif
  for (int64_t b = blockIdx.x; b < cfg.num_streams; b += gridDim.x) {
    int status = st.status[b];
    if (status) continue;  // uniform across the block
    int r = st.rank[b];
    double esq = eps_sq<double>(cfg, r);  // rank-test threshold, refreshed when r grows
    const int64_t nobs0 = st.nobs[b];
    double* Cg = reinterpret_cast<double*>(st.basis) + b * (int64_t)R * M;
    double* Dg = reinterpret_cast<double*>(st.dual) + b * (int64_t)R * M;
    double* Pg = reinterpret_cast<double*>(st.gram_inv) + b * (int64_t)R * R;
    double* Xg = reinterpret_cast<double*>(st.x) + b * (int64_t)k * M;
    const TI* Rb = rows + b * rstride;
    const TI* Yb = tgts + b * tstride;

    // ---- state (rank 0 is all zeros by the state contract) ------------------------
    const bool fresh = (r == 0);
    double Dt[IT][8];
    double Pr[IT][2];
    double Wt[2] = {0.0, 0.0};
#pragma unroll
    for (int nt = 0; nt < IT; ++nt) {
#pragma unroll
      for (int J = 0; J < 4; ++J) {
        const double2 v = fresh ? make_double2(0.0, 0.0)
                                : *reinterpret_cast<const double2*>(Dg + (8 * nt + p) * M + j0 + 8 * J + 2 * q);
        Dt[nt][2 * J] = v.x;
        Dt[nt][2 * J + 1] = v.y;
      }
      const double2 v = (fresh || w >= IT) ? make_double2(0.0, 0.0)
                                           : *reinterpret_cast<const double2*>(Pg + (8 * w + p) * R + 8 * nt + 2 * q);
      Pr[nt][0] = v.x;
      Pr[nt][1] = v.y;
    }
#pragma unroll
    for (int kt = 0; kt < IK; ++kt)
#pragma unroll
      for (int jt = 0; jt < 4; ++jt) S.Cs[w][kt][jt][lane] = fresh ? 0.0 : -Cg[sigma(kt, q) * M + j0 + 8 * jt + p];
    bool nz = false;
    if (!fresh && p < k) {
#pragma unroll
      for (int J = 0; J < 4; ++J) {
        const double2 v = *reinterpret_cast<const double2*>(Xg + p * M + j0 + 8 * J + 2 * q);
        nz |= (v.x != 0.0) || (v.y != 0.0);
      }
    }
    const bool has_x0 = __syncthreads_or(nz) != 0;

    const int64_t ntiles = (T + TT - 1) / TT;
    auto prefetch = [&](int64_t tile, int s) {
      if (tile < ntiles) {
        const int64_t t0 = tile * TT;
        const int64_t t = t0 + p;
        const bool ok = t < T;
        const TI* src = ok ? Rb + t * M + j0 : Rb;
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) cp_async_pair<TI>(&S.At[w][s][nt][lane][0], src + 8 * nt + 2 * q, ok);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t ty = t0 + 2 * q + e;
          const bool oky = ty < T && p < k;
          cp_async_one<TI>(&S.Yt[w][s][lane][e], oky ? Yb + ty * k + p : Yb, oky);
        }
      }
      cp_commit();
    };

    struct Front {
      double g[IT][2];   // G[t=p][8nt+2q+e] (full, identical in every warp)
      double acc[4][2];  // rejection of the own columns: A - G C
      double rsq, asq;   // |rej_t|^2, |a_t|^2 for t = p
      double dyx[2];     // y - a.x0 for (c = p, t = 2q+e)
      unsigned badm;
      int tstar, tv;
      int64_t t0;
    };

    // projection of one tile and the rank test (solver.py:286-296)
    auto front = [&](int64_t tile, int s, int row_start, Front& F) {
      WPROBE(0);
      const TI* As = &S.At[w][s][0][lane][0];
      F.t0 = tile * TT;
      F.tv = (int)((T - F.t0) < TT ? (T - F.t0) : TT);
      const double2 yy = slot(&S.Yt[w][s][lane][0], 0);
      const int nti = (r + 7) >> 3;  // N tiles of G that can be nonzero
      double s4[4] = {0.0, 0.0, 0.0, 0.0};
      double g[IT][2], g2[IT][2];
#pragma unroll
      for (int nt = 0; nt < IT; ++nt) g[nt][0] = g[nt][1] = g2[nt][0] = g2[nt][1] = 0.0;
#pragma unroll
      for (int J = 0; J < 4; ++J) {
        const double2 v = slot(As, J * 32);
        s4[(2 * J) & 3] = fma(v.x, v.x, s4[(2 * J) & 3]);
        s4[(2 * J + 1) & 3] = fma(v.y, v.y, s4[(2 * J + 1) & 3]);
#pragma unroll
        for (int nt = 0; nt < IT; ++nt) {
          if (nt < nti) {
            mma(g[nt], v.x, Dt[nt][2 * J]);
            mma(g2[nt], v.y, Dt[nt][2 * J + 1]);
          }
        }
      }
      double asq = (s4[0] + s4[1]) + (s4[2] + s4[3]);
      asq += __shfl_xor_sync(FULL, asq, 1);
      asq += __shfl_xor_sync(FULL, asq, 2);
      // a.x0 of the own columns (M = c, N = t, K = j) when x0 != 0
      double y0[2] = {0.0, 0.0};
      if (has_x0) {
#pragma unroll
        for (int J = 0; J < 4; ++J) {
          double2 xv = make_double2(0.0, 0.0);
          if (p < k) xv = __ldg(reinterpret_cast<const double2*>(Xg + p * M + j0 + 8 * J + 2 * q));
          const double2 v = slot(As, J * 32);
          mma(y0, xv.x, v.x);
          mma(y0, xv.y, v.y);
        }
      }
      // cross-warp sums: G partials, |a|^2, a.x0
#pragma unroll
      for (int nt = 0; nt < IT; ++nt)
        *reinterpret_cast<double2*>(&S.Gp[w][nt][lane][0]) = make_double2(g[nt][0] + g2[nt][0], g[nt][1] + g2[nt][1]);
      *reinterpret_cast<double2*>(&S.red[0][w][lane][0]) = make_double2(asq, 0.0);
      *reinterpret_cast<double2*>(&S.red[2][w][lane][0]) = make_double2(y0[0], y0[1]);
      WPROBE(1);
      __syncthreads();
      WPROBE(2);
#pragma unroll
      for (int nt = 0; nt < IT; ++nt) {
        double2 sum = make_double2(0.0, 0.0);
#pragma unroll
        for (int u = 0; u < WG; ++u) {
          const double2 v = *reinterpret_cast<const double2*>(&S.Gp[u][nt][lane][0]);
          sum.x += v.x;
          sum.y += v.y;
        }
        F.g[nt][0] = sum.x;
        F.g[nt][1] = sum.y;
      }
      asq = 0.0;
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int u = 0; u < WG; ++u) {
        asq += S.red[0][u][lane][0];
        a0 += S.red[2][u][lane][0];
        a1 += S.red[2][u][lane][1];
      }
      F.asq = asq;
      F.dyx[0] = yy.x - a0;
      F.dyx[1] = yy.y - a1;
      // R = A - G C on the own columns (C stored negated, accumulated onto A)
#pragma unroll
      for (int jt = 0; jt < 4; ++jt) {
        const double2 v = slot(As, jt * 32);
        F.acc[jt][0] = v.x;
        F.acc[jt][1] = v.y;
      }
#pragma unroll
      for (int kt = 0; kt < IK; ++kt) {
        if (8 * (kt >> 1) < r) {  // rows of C beyond the rank are zero
#pragma unroll
          for (int jt = 0; jt < 4; ++jt) mma(F.acc[jt], F.g[kt >> 1][kt & 1], S.Cs[w][kt][jt][lane]);
        }
      }
      double t4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int jt = 0; jt < 4; ++jt) {
        t4[(2 * jt) & 3] = fma(F.acc[jt][0], F.acc[jt][0], t4[(2 * jt) & 3]);
        t4[(2 * jt + 1) & 3] = fma(F.acc[jt][1], F.acc[jt][1], t4[(2 * jt + 1) & 3]);
      }
      double rsq = (t4[0] + t4[1]) + (t4[2] + t4[3]);
      rsq += __shfl_xor_sync(FULL, rsq, 1);
      rsq += __shfl_xor_sync(FULL, rsq, 2);
      S.red[1][w][lane][0] = rsq;
      WPROBE(3);
      __syncthreads();
      WPROBE(4);
      rsq = 0.0;
#pragma unroll
      for (int u = 0; u < WG; ++u) rsq += S.red[1][u][lane][0];
      F.rsq = rsq;
      const unsigned yb0 = __ballot_sync(FULL, !isfinite(F.dyx[0]));
      const unsigned yb1 = __ballot_sync(FULL, !isfinite(F.dyx[1]));
      const bool ybad = (((p & 1) ? yb1 : yb0) & (0x11111111u << (p >> 1))) != 0u;
      const bool valid = p >= row_start && p < F.tv;
      const bool dep = is_dependent<double>(rsq, asq, esq);
      const bool bad = !isfinite(asq) || ybad;
      const unsigned stopm = __ballot_sync(FULL, q == 0 && valid && (!dep || bad));
      F.badm = __ballot_sync(FULL, q == 0 && valid && bad);
      F.tstar = stopm ? (__ffs(stopm) - 1) >> 2 : F.tv;
    };

    // blocked Sherman-Morrison over the dependent rows [rs, te) (solver.py:297-304)
    auto scan = [&](const Front& F, int rs, int te) {
      WPROBE(6);
      const bool inb = p >= rs && p < te;
      double gm[IT][2];
#pragma unroll
      for (int nt = 0; nt < IT; ++nt) {
        gm[nt][0] = inb ? F.g[nt][0] : 0.0;
        gm[nt][1] = inb ? F.g[nt][1] : 0.0;
      }
      const bool own = w < IT;  // warps beyond the P / W row blocks only help the front
      // (G W)^T over the own row block of W, and U^T = G P[:, own block]
      double gw[2] = {0.0, 0.0}, ut[2] = {0.0, 0.0};
      if (own) {
        mma(gw, Wt[0], gm[w][0]);
        mma(gw, Wt[1], gm[w][1]);
#pragma unroll
        for (int kt = 0; kt < IK; ++kt) mma(ut, gm[kt >> 1][kt & 1], Pr[kt >> 1][kt & 1]);
      }
      // S partial = U^T[:, own] G[:, own]^T
      double sp[2] = {0.0, 0.0};
      if (own) {
        mma(sp, ut[0], gm[w][0]);
        mma(sp, ut[1], gm[w][1]);
      }
      *reinterpret_cast<double2*>(&S.Sp[w][lane][0]) = make_double2(sp[0], sp[1]);
      *reinterpret_cast<double2*>(&S.red[2][w][lane][0]) = make_double2(gw[0], gw[1]);
      WPROBE(7);
      __syncthreads();
      WPROBE(8);
      double mi[2] = {0.0, 0.0}, gws[2] = {0.0, 0.0};
#pragma unroll
      for (int u = 0; u < WG; ++u) {
        mi[0] += S.Sp[u][lane][0];
        mi[1] += S.Sp[u][lane][1];
        gws[0] += S.red[2][u][lane][0];
        gws[1] += S.red[2][u][lane][1];
      }
      double dy[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int t = 2 * q + e;
        dy[e] = (t >= rs && t < te) ? F.dyx[e] - gws[e] : 0.0;
      }
      if (p == 2 * q) mi[0] += 1.0;
      if (p == 2 * q + 1) mi[1] += 1.0;
      // M = L diag(d) L^T, E = L^-1 (every warp, identical)
      double ev[2] = {p == 2 * q ? 1.0 : 0.0, p == 2 * q + 1 ? 1.0 : 0.0};
#pragma unroll
      for (int kk = 0; kk < TT - 1; ++kk) {
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
      const double dsel = (p & 1) ? mi[1] : mi[0];
      const double rd = rcp64(__shfl_sync(FULL, dsel, 4 * p + (p >> 1)));
      const double rd0 = __shfl_sync(FULL, rd, 8 * q);
      const double rd1 = __shfl_sync(FULL, rd, 8 * q + 4);
      // U = (U^T)^T on the own block, Y^T = U E^T (rows of the own block)
      double yt[2] = {0.0, 0.0};
      if (own) {
        double u[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int src = 4 * (2 * q + e) + (p >> 1);
          const double v0 = __shfl_sync(FULL, ut[0], src);
          const double v1 = __shfl_sync(FULL, ut[1], src);
          u[e] = (p & 1) ? v1 : v0;
        }
        mma(yt, u[0], ev[0]);
        mma(yt, u[1], ev[1]);
        *reinterpret_cast<double2*>(&S.Yb[w][lane][0]) = make_double2(yt[0], yt[1]);
      }
      WPROBE(9);
      __syncthreads();
      WPROBE(10);
      if (own) {
        // E dy0 (every RHS), then P[own rows] -= Y^T D^-1 Y and W[own] += ...
        double dh[2] = {0.0, 0.0};
        mma(dh, dy[0], ev[0]);
        mma(dh, dy[1], ev[1]);
        const double d0 = dh[0] * rd0, d1 = dh[1] * rd1;
        const double s0 = -yt[0] * rd0, s1 = -yt[1] * rd1;
#pragma unroll
        for (int nt = 0; nt < IT; ++nt) {
          const double2 yb = *reinterpret_cast<const double2*>(&S.Yb[nt][lane][0]);
          mma(Pr[nt], s0, yb.x);
          mma(Pr[nt], s1, yb.y);
        }
        mma(Wt, d0, yt[0]);
        mma(Wt, d1, yt[1]);
      }
      if (inb && w == 0) {
        const int64_t row = b * T + F.t0 + p;
        if (blog && q == 0) blog[row] = 0;
        if (clog) {
#pragma unroll
          for (int nt = 0; nt < IT; ++nt)
            *reinterpret_cast<double2*>(clog + row * R + 8 * nt + 2 * q) = make_double2(F.g[nt][0], F.g[nt][1]);
        }
      }
    };

    // the update itself, from the scratch rows (gam, kv, av)
    auto grow_core = [&](double wnew, double rsq, int64_t t0, int ts) {
      const int var = GEN ? RGB_GENERAL : cfg.variant;
      double last = 1.0;  // coords_row[r] of the orthogonal / orthonormal variants
      if (var == RGB_GENERAL) {
        if (w == (r >> 3)) {
#pragma unroll
          for (int e = 0; e < 2; ++e)
            if (8 * w + 2 * q + e == r) Wt[e] = wnew;
        }
        // C~[:r] -= gamma K^T, C~[r] = K on the own columns (solver.py:377-380)
#pragma unroll
        for (int nt = 0; nt < IT; ++nt) {
          const int i = 8 * nt + p;
          const double gi = S.gam[i];
#pragma unroll
          for (int J = 0; J < 4; ++J) {
            const double2 kv = *reinterpret_cast<const double2*>(&S.kv[j0 + 8 * J + 2 * q]);
            Dt[nt][2 * J] = (i == r) ? kv.x : fma(-gi, kv.x, Dt[nt][2 * J]);
            Dt[nt][2 * J + 1] = (i == r) ? kv.y : fma(-gi, kv.y, Dt[nt][2 * J + 1]);
          }
        }
        // C[r] = a
        if (q == ((r & 7) >> 1)) {
          const int ktr = 2 * (r >> 3) + (r & 1);
#pragma unroll
          for (int jt = 0; jt < 4; ++jt) S.Cs[w][ktr][jt][lane] = -S.av[j0 + 8 * jt + p];
        }
        // P = diag(P, 1)
        if (w < IT) {
#pragma unroll
          for (int nt = 0; nt < IT; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int i = 8 * w + p, i2 = 8 * nt + 2 * q + e;
              if (i == r || i2 == r) Pr[nt][e] = (i == i2) ? 1.0 : 0.0;
            }
        }
      } else {
        // orthogonal / orthonormal _grow (solver.py:382-395); av holds the rejection.
        // z = P gamma (rows 8w + p), gamma^T W (column p) partials of warp w
        double z = 0.0, gw = 0.0;
        if (w < IT) {
#pragma unroll
          for (int nt = 0; nt < IT; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) z = fma(Pr[nt][e], S.gam[8 * nt + 2 * q + e], z);
#pragma unroll
          for (int e = 0; e < 2; ++e) gw = fma(S.gam[8 * w + 2 * q + e], Wt[e], gw);
          z += __shfl_xor_sync(FULL, z, 1);
          z += __shfl_xor_sync(FULL, z, 2);
          gw += __shfl_xor_sync(FULL, gw, 1);
          gw += __shfl_xor_sync(FULL, gw, 2);
          if (q == 0) {
            S.kv[8 * w + p] = z;  // kv is free: C~[:r] is unchanged
            S.red[2][w][p][0] = gw;
          }
        }
        __syncthreads();
        double dn = 0.0, gws = 0.0;
#pragma unroll
        for (int i = 0; i < R; ++i) dn = fma(S.gam[i], S.kv[i], dn);
#pragma unroll
        for (int u = 0; u < IT; ++u) gws += S.red[2][u][p][0];
        const double denom = 1.0 + dn;  // solver.py:307-310
        const double resc = (var == RGB_ORTHONORMAL) ? 1.0 / sqrt(rsq) : cfg.alpha;
        last = 1.0 / resc;
        const double alpha = 1.0 / last;
        // W gains row r: alpha (y - a.x), the new dual row being K / alpha
        if (w == (r >> 3)) {
          const double wr = alpha * (wnew - gws);
#pragma unroll
          for (int e = 0; e < 2; ++e)
            if (8 * w + 2 * q + e == r) Wt[e] = wr;
        }
        // C[r] = alpha rej;  C~[r] = rej / (alpha |rej|^2)  (orthonormal: C~ is C)
        if (q == ((r & 7) >> 1)) {
          const int ktr = 2 * (r >> 3) + (r & 1);
#pragma unroll
          for (int jt = 0; jt < 4; ++jt) S.Cs[w][ktr][jt][lane] = -(alpha * S.av[j0 + 8 * jt + p]);
        }
        const double sc = alpha * rsq;
#pragma unroll
        for (int nt = 0; nt < IT; ++nt) {
          if (8 * nt + p == r) {
#pragma unroll
            for (int J = 0; J < 4; ++J)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const double rj = S.av[j0 + 8 * J + 2 * q + e];
                Dt[nt][2 * J + e] = (var == RGB_ORTHONORMAL) ? alpha * rj : rj / sc;
              }
          }
        }
        // P gains edge -alpha z and corner alpha^2 denom
        if (w < IT) {
#pragma unroll
          for (int nt = 0; nt < IT; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int i = 8 * w + p, i2 = 8 * nt + 2 * q + e;
              if (i == r && i2 == r) Pr[nt][e] = alpha * alpha * denom;
              else if (i2 == r) Pr[nt][e] = (i < r) ? -(alpha * S.kv[i]) : 0.0;
              else if (i == r) Pr[nt][e] = (i2 < r) ? -(alpha * S.kv[i2]) : 0.0;
            }
        }
      }
      const int64_t row = b * T + t0 + ts;
      if (w == 0) {
        if (blog && lane == 0) blog[row] = 1;
        if (clog && lane < R) {
          double v = (lane == r) ? 1.0 : 0.0;
          if (var != RGB_GENERAL) v = (lane < r) ? S.gam[lane] : (lane == r ? last : 0.0);
          clog[row * R + lane] = v;
        }
      }
      __syncthreads();
      r += 1;
      esq = eps_sq<double>(cfg, r);
    };
    // independent row ts (solver.py:305-318, _grow solver.py:368-397)
    auto grow = [&](const Front& F, int s, int ts) {
      if (p == ts) {
        const TI* As = &S.At[w][s][0][lane][0];
        const double rinv = 1.0 / F.rsq;  // K = rej / |rej|^2, one rounding more than a division
#pragma unroll
        for (int jt = 0; jt < 4; ++jt) {
          *reinterpret_cast<double2*>(&S.kv[j0 + 8 * jt + 2 * q]) =
              make_double2(F.acc[jt][0] * rinv, F.acc[jt][1] * rinv);
          // the row itself (general: C[r] = a) or its rejection (other variants)
          *reinterpret_cast<double2*>(&S.av[j0 + 8 * jt + 2 * q]) =
              GEN ? slot(As, jt * 32) : make_double2(F.acc[jt][0], F.acc[jt][1]);
        }
        if (w == 0) {
#pragma unroll
          for (int nt = 0; nt < IT; ++nt)
            *reinterpret_cast<double2*>(&S.gam[8 * nt + 2 * q]) = make_double2(F.g[nt][0], F.g[nt][1]);
        }
      }
      __syncthreads();
      // W gains row r: y - a.x0 of row ts (x = x0 + C~^T W stays exact)
      const double dv = (ts & 1) ? F.dyx[1] : F.dyx[0];
      grow_core(__shfl_sync(FULL, dv, 4 * p + (ts >> 1)), GEN ? 0.0 : __shfl_sync(FULL, F.rsq, 4 * ts), F.t0, ts);
    };

    // Single-row projection of row ts of stage s across the group on the CUDA
    // cores (solver.py:286-291), for a fresh stream's leading independent rows
    // (re-projecting the whole tile after each growth costs 64 MMAs per warp).
    // Leaves gamma, K and the row in the scratch rows; returns |rej|^2, |a|^2.
    auto project_row = [&](int s, int ts, double& rsq_o, double& asq_o) {
      const TI* Ar = &S.At[w][s][0][4 * ts + q][0];
      double gp[IT], a2 = 0.0;
#pragma unroll
      for (int nt = 0; nt < IT; ++nt) gp[nt] = 0.0;
#pragma unroll
      for (int J = 0; J < 4; ++J) {  // my columns j0 + sigma(kt, q) = j0 + 8J + 2q + e
        const double2 v = slot(Ar, J * 32);
        a2 = fma(v.x, v.x, fma(v.y, v.y, a2));
#pragma unroll
        for (int nt = 0; nt < IT; ++nt) gp[nt] = fma(Dt[nt][2 * J], v.x, fma(Dt[nt][2 * J + 1], v.y, gp[nt]));
      }
      a2 += __shfl_xor_sync(FULL, a2, 1);
      a2 += __shfl_xor_sync(FULL, a2, 2);
#pragma unroll
      for (int nt = 0; nt < IT; ++nt) {
        gp[nt] += __shfl_xor_sync(FULL, gp[nt], 1);
        gp[nt] += __shfl_xor_sync(FULL, gp[nt], 2);
      }
      // group sums of gamma (per i) and |a|^2 (fixed order)
      if (q == 0) {
#pragma unroll
        for (int nt = 0; nt < IT; ++nt) S.Gp[w][nt][p][0] = gp[nt];
        S.red[0][w][p][0] = a2;
      }
      __syncthreads();
      double asq = 0.0;
#pragma unroll
      for (int u = 0; u < WG; ++u) asq += S.red[0][u][p][0];
      // rej_j = a_j - sum_i gamma_i C_ij, j = j0 + 8jt + p, over my rows i = sigma(kt, q)
      double rp[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int kt = 0; kt < IK; ++kt) {
        const int i = sigma(kt, q);
        double gi = 0.0;
#pragma unroll
        for (int u = 0; u < WG; ++u) gi += S.Gp[u][i >> 3][i & 7][0];
#pragma unroll
        for (int jt = 0; jt < 4; ++jt) rp[jt] = fma(gi, S.Cs[w][kt][jt][lane], rp[jt]);  // Cs = -C
      }
      double rej[4], r2 = 0.0;
#pragma unroll
      for (int jt = 0; jt < 4; ++jt) {
        rp[jt] += __shfl_xor_sync(FULL, rp[jt], 1);
        rp[jt] += __shfl_xor_sync(FULL, rp[jt], 2);
        rej[jt] = (double)S.At[w][s][jt][4 * ts + (p >> 1)][p & 1] + rp[jt];
        r2 = fma(rej[jt], rej[jt], r2);
      }
      r2 += __shfl_xor_sync(FULL, r2, 4);
      r2 += __shfl_xor_sync(FULL, r2, 8);
      r2 += __shfl_xor_sync(FULL, r2, 16);
      if (lane == 0) S.red[1][w][0][0] = r2;
      __syncthreads();
      double rsq = 0.0;
#pragma unroll
      for (int u = 0; u < WG; ++u) rsq += S.red[1][u][0][0];
      if (q == 0) {
        const double rinv = 1.0 / rsq;
#pragma unroll
        for (int jt = 0; jt < 4; ++jt) {
          S.kv[j0 + 8 * jt + p] = rej[jt] * rinv;
          S.av[j0 + 8 * jt + p] = GEN ? (double)S.At[w][s][jt][4 * ts + (p >> 1)][p & 1] : rej[jt];
        }
        if (w == 0) {
#pragma unroll
          for (int nt = 0; nt < IT; ++nt) {
            double g = 0.0;
#pragma unroll
            for (int u = 0; u < WG; ++u) g += S.Gp[u][nt][p][0];
            S.gam[8 * nt + p] = g;
          }
        }
      }
      __syncthreads();
      rsq_o = rsq;
      asq_o = asq;
    };

    bool stopped = false;
    int64_t consumed = 0;
    Front F;
    int64_t tile = 0;
    int first_row = 0;
    if (ntiles > 0) {
      prefetch(0, 0);
      prefetch(1, 1);
      cp_wait<1>();
      __syncthreads();
      // row mode: a fresh stream's leading independent rows, one at a time
      if (fresh && !has_x0) {
        while (tile < ntiles) {
          const int s = (int)(tile & 1);
          const int64_t t0 = tile * TT;
          const int tv = (int)((T - t0) < TT ? (T - t0) : TT);
          int ts = 0;
          for (; ts < tv; ++ts) {
            double rsq, asq;
            project_row(s, ts, rsq, asq);
            const double yv = (double)S.Yt[w][s][4 * p + (ts >> 1)][ts & 1];  // y[ts][c = p] (0 for c >= k)
            const bool bad = !isfinite(asq) || __any_sync(FULL, !isfinite(yv));
            if (bad || r >= R || is_dependent<double>(rsq, asq, esq)) break;
            grow_core(yv, rsq, t0, ts);
          }
          if (ts < tv) {
            first_row = ts;
            break;
          }
          consumed = t0 + tv;
          ++tile;
          __syncthreads();
          prefetch(tile + 1, s);
          cp_wait<1>();
          __syncthreads();
        }
      }
    }
    for (; tile < ntiles; ++tile) {
      const int s = (int)(tile & 1);
      int row_start = first_row;
      front(tile, s, first_row, F);
      first_row = 0;
      while (true) {
        if (F.tstar > row_start) scan(F, row_start, F.tstar);
        if (F.tstar >= F.tv) break;
        if ((F.badm >> (4 * F.tstar)) & 1u) {
          status |= RGB_ST_NONFINITE;
          stopped = true;
          break;
        }
        if (r >= R) {
          status |= RGB_ST_RANK_CAP;
          stopped = true;
          break;
        }
        grow(F, s, F.tstar);
        row_start = F.tstar + 1;
        if (row_start >= F.tv) break;
        front(tile, s, row_start, F);
      }
      if (stopped) {
        consumed = F.t0 + F.tstar;
        break;
      }
      consumed = F.t0 + F.tv;
      WPROBE(12);
      __syncthreads();  // every warp is done with stage s before it is refilled
      WPROBE(13);
      prefetch(tile + 2, s);
      cp_wait<1>();
      __syncwarp();
    }
    cp_wait<0>();
    __syncthreads();

    // ---- write back; x = x0 + C~^T W ------------------------------------------------
#pragma unroll
    for (int kt = 0; kt < IK; ++kt)
#pragma unroll
      for (int jt = 0; jt < 4; ++jt) Cg[sigma(kt, q) * M + j0 + 8 * jt + p] = -S.Cs[w][kt][jt][lane];
    // W of every row block, for the x contraction of the own columns
    if (w < IT) *reinterpret_cast<double2*>(&S.Yb[w][lane][0]) = make_double2(Wt[0], Wt[1]);
    __syncwarp();
    // C~ of the own columns, staged row-major over the own Cs slice
    double* Dm = &S.Cs[w][0][0][0];
    constexpr int DS = 32;
    static_assert(sizeof(S.Cs[0]) >= sizeof(double) * R * DS, "staging");
#pragma unroll
    for (int nt = 0; nt < IT; ++nt)
#pragma unroll
      for (int J = 0; J < 4; ++J) {
        const double2 v = make_double2(Dt[nt][2 * J], Dt[nt][2 * J + 1]);
        *reinterpret_cast<double2*>(Dg + (8 * nt + p) * M + j0 + 8 * J + 2 * q) = v;
        *reinterpret_cast<double2*>(Dm + (8 * nt + p) * DS + 8 * J + 2 * q) = v;
      }
    __syncthreads();
    // x^T = x0^T + W^T C~ : M = c, N = j (own), K = i
#pragma unroll
    for (int jt = 0; jt < 4; ++jt) {
      double acc[2] = {0.0, 0.0};
      if (has_x0 && p < k) {
        const double2 v = *reinterpret_cast<const double2*>(Xg + p * M + j0 + 8 * jt + 2 * q);
        acc[0] = v.x;
        acc[1] = v.y;
      }
#pragma unroll
      for (int kt = 0; kt < IK; ++kt) {
        const double a = S.Yb[kt >> 1][lane][kt & 1];
        mma(acc, a, Dm[sigma(kt, q) * DS + 8 * jt + p]);
      }
      if (p < k) *reinterpret_cast<double2*>(Xg + p * M + j0 + 8 * jt + 2 * q) = make_double2(acc[0], acc[1]);
    }
    if (w < IT) {
#pragma unroll
      for (int nt = 0; nt < IT; ++nt)
        *reinterpret_cast<double2*>(Pg + (8 * w + p) * R + 8 * nt + 2 * q) = make_double2(Pr[nt][0], Pr[nt][1]);
    }
    if (threadIdx.x == 0) {
      st.rank[b] = r;
      st.nobs[b] = nobs0 + consumed;
      st.status[b] = status;
    }
    __syncthreads();
  }
}

}  // namespace blk

// Instantiations: (r_cap, warps) with m = 32 * warps, r_cap 16 or 32 -- config 3
// (m 128, r_cap 32), config 1 (m 256, r_cap 16, one stream: 8 warps share its
// work), and m 128 / r_cap 16, m 256 / r_cap 32.
template <int R, int WG, typename TI>
static int launch_wg(const rgb_config& cfg, rgb_state& st, const void* rows, int64_t rows_stride,
                     const void* targets, int64_t tg_stride, int64_t T, const rgb_logs& logs,
                     cudaStream_t stream, int num_sms) {
  const bool gen = cfg.variant == RGB_GENERAL;
  auto kern = gen ? blk::blocked_wg_kernel<R, WG, true, TI> : blk::blocked_wg_kernel<R, WG, false, TI>;
  const size_t smem = sizeof(blk::GroupSmem<R, WG, TI>);
  static bool attr[2][64] = {};
  smem_attr_once(kern, smem, attr[gen]);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WG * 32, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)num_sms * per_sm;
  if (grid > cfg.num_streams) grid = cfg.num_streams;
  kern<<<(unsigned)grid, WG * 32, smem, stream>>>(cfg, st, (const TI*)rows, rows_stride, (const TI*)targets,
                                                  tg_stride, T, logs.branch, (double*)logs.coords);
  return cudaGetLastError() == cudaSuccess ? RGB_OK : RGB_E_CUDA;
}

bool blocked_wg_supports(const rgb_config& cfg) {
  const bool var_ok = cfg.variant == RGB_GENERAL || cfg.variant == RGB_ORTHONORMAL ||
                      (cfg.variant == RGB_ORTHOGONAL && cfg.alpha != 0.0);
  if (cfg.dtype != RGB_F64 || !var_ok || cfg.k < 1 || cfg.k > 8) return false;
  return (cfg.m == 128 || cfg.m == 256) && (cfg.r_cap == 16 || cfg.r_cap == 32);
}

int launch_blocked_wg(const rgb_config& cfg, rgb_state& st, const void* rows, int64_t rows_stride,
                      const void* targets, int64_t tg_stride, int64_t T, const rgb_logs& logs,
                      cudaStream_t stream, int num_sms, bool f32in) {
  if (logs.resid || logs.gain) return RGB_E_UNSUPPORTED;
  if (cfg.m == 128 && cfg.r_cap == 32)
    return f32in ? launch_wg<32, 4, float>(cfg, st, rows, rows_stride, targets, tg_stride, T, logs, stream, num_sms)
                 : launch_wg<32, 4, double>(cfg, st, rows, rows_stride, targets, tg_stride, T, logs, stream, num_sms);
  if (cfg.m == 256 && cfg.r_cap == 16)
    return f32in ? launch_wg<16, 8, float>(cfg, st, rows, rows_stride, targets, tg_stride, T, logs, stream, num_sms)
                 : launch_wg<16, 8, double>(cfg, st, rows, rows_stride, targets, tg_stride, T, logs, stream, num_sms);
  if (cfg.m == 128 && cfg.r_cap == 16)
    return f32in ? launch_wg<16, 4, float>(cfg, st, rows, rows_stride, targets, tg_stride, T, logs, stream, num_sms)
                 : launch_wg<16, 4, double>(cfg, st, rows, rows_stride, targets, tg_stride, T, logs, stream, num_sms);
  if (cfg.m == 256 && cfg.r_cap == 32)
    return f32in ? launch_wg<32, 8, float>(cfg, st, rows, rows_stride, targets, tg_stride, T, logs, stream, num_sms)
                 : launch_wg<32, 8, double>(cfg, st, rows, rows_stride, targets, tg_stride, T, logs, stream, num_sms);
  return RGB_E_UNSUPPORTED;
}

}  // namespace rgb

#ifdef RGB_WG_PROBE
extern "C" int rgb_wg_probe(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, rgb::blk::g_wprobe, sizeof(rgb::blk::g_wprobe));
  if (reset) {
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(rgb::blk::g_wprobe, z, sizeof(z));
  }
  return 0;
}
#endif
