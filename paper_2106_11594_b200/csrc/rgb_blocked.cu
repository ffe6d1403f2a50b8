// rgb_blocked.cu -- batched rank-Greville update on fp64 tensor cores (sm_100a).
//
// One warp owns one stream at a time (persistent grid, streams claimed dynamically)
// and consumes its rows in tiles of 8.  Inside a run of dependent
// rows the basis C and dual C~ do not change (solver.py:297-304 touch only
// P^-1 and x), so the per-row GEMVs of the reference become 8-row contractions
// on DMMA.8x8x4 (mma.sync m8n8k4 f64), with every reduction inside the tensor
// core instead of in warp shuffles:
//
//   G   = A C~^T                 coords of the 8 rows      (solver.py:286)
//   R   = A - G C, |R_t|^2       rejections and the test   (solver.py:287-296)
//   U   = P G^T,  S = G P G^T    Sherman-Morrison inputs   (solver.py:298-299)
//   M   = I + S = L diag(d) L^T  8x8 LDL^T by elimination in registers, E = L^-1
//   Y^T = U E^T                  columns = the z_t of the 8 sequential steps
//   P  -= Y^T D^-1 Y             = 8 sequential rank-1 updates of solver.py:300-301
//   W  += Y^T D^-1 E dy0         the 8 solution updates of solver.py:302-304
//
// This is the reference's 8 sequential Sherman-Morrison steps in factored
// (LDL^T) form -- identical algebra, the same accuracy as the
// sequential recursion (an explicit M^-1 / Woodbury update is not; see
// DESIGN.md), and every contraction on the tensor cores (the blocked variant
// of SURVEY.md section 7, hard part 5).  The solution is carried as
// x = x0 + C~^T W (W is r x k): a dependent row changes only W, an independent
// row appends W's row r = y - a.x0 (exact algebra for x' = x + K dy with
// C~' = [C~ - gamma K^T; K^T]), and x is materialised once at the end of the
// call.  dy0 = y - a.x0 - gamma^T W is the reference's a-priori residual.
//
// Deferred fold (general variant, a fresh stream): the chain above is the recursive form
// of P^-1 = (B^T B)^-1, W = P^-1 B^T dy, and neither the rank test nor growth reads
// P^-1 or W -- so the tiles only accumulate Q = B^T B and B^T dy (12 MMAs, no chain) and
// Q is inverted once per call, accepted when kappa_F(Q) <= 1e6; a stream that fails is
// folded again with the chain (see `defer` below and DESIGN.md).  18.96 -> 14.15 ms.
//
// Independent rows (solver.py:305-318, _grow solver.py:368-397) split the tile:
// the dependent prefix is folded, the row grows the basis (K = rej/|rej|^2,
// C~[:r] -= gamma K^T, C~[r] = K, C[r] = a, P = diag(P, 1)), and the rest of
// the tile is re-projected on the new basis.  Rank tests use the reference's
// threshold with the CURRENT rank for every row (solver.py:292-296).
//
// Fragment layouts (m8n8k4 f64; lane = 4p + q): A[m=p][k=q], B[k=q][n=p],
// C/D[m=p][n=2q+e].  K slots are permuted, sigma(kt,q) = 8(kt>>1)+2q+(kt&1),
// so that every accumulator is directly the next MMA's operand:
//   tile   a[nt][e]      = A[t=p][8nt+2q+e]            (A- and B-operand, K=sigma)
//   C~^T   Dt[nt][kt]    = C~[8nt+p][sigma(kt,q)]       registers
//   -C     Cs[kt][jt][l] = -C[sigma(kt,q)][8jt+p]       shared memory (R accumulates onto A)
//   P^-1   Pr[mt][nt][e] = P[8mt+p][8nt+2q+e]           registers (symmetric)
//   W^T    Wt[nt][e]     = W[8nt+2q+e][c=p]             registers
//
// Instantiated for the batched configuration m = 64, r_cap = 16, k <= 8
// right-hand sides (unused RHS lanes masked), fp64 state, all three variants
// (the orthogonal / orthonormal growth in its own instantiation), float64 or
// float32 inputs; other shapes run on the warp-group, cluster, grid or
// generic kernels.
#include <cstdlib>

#include "rgb_mma.cuh"

namespace rgb {
namespace blk {

template <int M, int R, int KC, typename TI>
struct WarpSmem {
  double Cs[R / 4][M / 8][32];   // -C, the B operand of R = A + G (-C) accumulated onto A
  TI At[2][M / 8][32][2];        // double-buffered row tile, lane-slot layout (input type)
  TI Yt[2][32][2];               // targets y[t=2q+e][c=p]
  union {
    struct {
      double gam[R];             // coords of an independent row
      double kv[M];              // its gain K = rej / |rej|^2
      double av[M];              // the row itself
    } ind;
  } u;
  // at the end of a call C~ is staged row-major with stride M + 2 over Cs and At
  static_assert(sizeof(Cs) + sizeof(At) >= sizeof(double) * R * (M + 2), "staging");
};

// In-place Gauss-Jordan inverse of the SPD matrix A (fragment layout A[mt][nt][e] =
// A[8mt+p][8nt+2q+e], pivots >= 1: no pivoting); rows / columns past the rank r are zero
// and stay zero.  Returns |A|_F^2 |A^-1|_F^2.  Not inlined: it runs once or twice per
// stream, and its 8 IT unrolled steps would otherwise sit in the tile loop's code.
template <int IT>
__device__ __noinline__ double gj_invert(double (&A)[IT][IT][2], int r, int p, int q) {
  double fq = 0.0, fp = 0.0;
#pragma unroll
  for (int mt = 0; mt < IT; ++mt)
#pragma unroll
    for (int nt = 0; nt < IT; ++nt) fq = fma(A[mt][nt][0], A[mt][nt][0], fma(A[mt][nt][1], A[mt][nt][1], fq));
#pragma unroll
  for (int kk = 0; kk < 8 * IT; ++kk) {
    if (kk < r) {  // (uniform)
      const int mk = kk >> 3, pk = kk & 7, qk = (kk & 7) >> 1, ek = kk & 1;
      const double pv = rcp64(__shfl_sync(FULL, A[mk][mk][ek], 4 * pk + qk));
      double rowv[IT][2], f[IT];
#pragma unroll
      for (int nt = 0; nt < IT; ++nt) {
        rowv[nt][0] = __shfl_sync(FULL, A[mk][nt][0], 4 * pk + q);
        rowv[nt][1] = __shfl_sync(FULL, A[mk][nt][1], 4 * pk + q);
      }
#pragma unroll
      for (int mt = 0; mt < IT; ++mt) f[mt] = __shfl_sync(FULL, A[mt][mk][ek], 4 * p + qk) * pv;
#pragma unroll
      for (int mt = 0; mt < IT; ++mt)
#pragma unroll
        for (int nt = 0; nt < IT; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const bool ir = (mt == mk) && (p == pk);
            const bool jc = (nt == mk) && (2 * q + e == (kk & 7));
            double v = fma(-f[mt], rowv[nt][e], A[mt][nt][e]);
            if (ir) v = rowv[nt][e] * pv;
            if (jc) v = ir ? pv : -f[mt];
            A[mt][nt][e] = v;
          }
    }
  }
#pragma unroll
  for (int mt = 0; mt < IT; ++mt)
#pragma unroll
    for (int nt = 0; nt < IT; ++nt) fp = fma(A[mt][nt][0], A[mt][nt][0], fma(A[mt][nt][1], A[mt][nt][1], fp));
  return warp_sum(fq) * warp_sum(fp);
}

#ifndef RGB_BLOCKED_MINB
#define RGB_BLOCKED_MINB 6  // x 2 warps: 12 warps per SM (same-box A/B: 4 x 3 +0.8 %, 12 x 1 +2.6 %, 1 x 12 +2.0 %)
#endif

// GEN: general variant only (the headline instantiation); !GEN: orthogonal /
// orthonormal, whose grow step differs (solver.py:382-395)
// TI: input element type (double, or float widened exactly on load)
// KM: k < KC right-hand sides (RHS lanes p >= k masked; KM = false is k = KC)
template <int M, int R, int KC, int WARPS, bool GEN, typename TI, bool KM = false>
__global__ void __launch_bounds__(WARPS * 32, RGB_BLOCKED_MINB) blocked_kernel(
    rgb_config cfg, rgb_state st, const TI* __restrict__ rows, int64_t rstride,
    const TI* __restrict__ tgts, int64_t tstride, int64_t T, uint8_t* __restrict__ blog,
    double* __restrict__ clog, int seq_only, unsigned* __restrict__ next_stream) {
  static_assert(M % 8 == 0 && R % 8 == 0 && KC == 8, "shape");
  constexpr int JT = M / 8, JK = M / 4, IT = R / 8, IK = R / 4;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int p = lane >> 2, q = lane & 3;
  WarpSmem<M, R, KC, TI>& S = reinterpret_cast<WarpSmem<M, R, KC, TI>*>(smem_raw)[wid];

  // Streams are claimed dynamically, one atomicAdd per warp and stream (a stream whose deferred
  // fold is folded again costs twice the others: a static round robin left the busiest warp
  // ~10 % behind the mean); without a counter every warp has at most one stream.
  bool redo = false;  // the deferred fold of the stream failed its conditioning certificate
  int64_t b = (int64_t)blockIdx.x * WARPS + wid;
  for (unsigned iter = 0;; ++iter) {
    if (!redo) {
      if (next_stream) {
        unsigned c = 0;
        if (lane == 0) c = atomicAdd(next_stream, 1u);
        b = __shfl_sync(FULL, c, 0);
      } else if (iter > 0) {
        break;
      }
    }
    if (b >= cfg.num_streams) break;
    const bool seq = redo || seq_only != 0;
    redo = false;
    int status = st.status[b];
    if (status) continue;
    int r = st.rank[b];
    const int64_t nobs0 = st.nobs[b];
    double* Cg = reinterpret_cast<double*>(st.basis) + b * (int64_t)R * M;
    double* Dg = reinterpret_cast<double*>(st.dual) + b * (int64_t)R * M;
    double* Pg = reinterpret_cast<double*>(st.gram_inv) + b * (int64_t)R * R;
    const int kk_ = KM ? cfg.k : KC;  // right-hand sides (targets stride, X rows)
    double* Xg = reinterpret_cast<double*>(st.x) + b * (int64_t)kk_ * M;
    const TI* Rb = rows + b * rstride;
    const TI* Yb = tgts + b * tstride;

    // ---- load the stream's state into fragment layouts -------------------------
    // A rank-0 stream is all zeros by the state contract (include/rgb.h: rows
    // beyond the rank are zero, and the minimum-norm solution of rank 0 is 0),
    // so a fresh solve reads nothing.
    const bool fresh = (r == 0);
    // Deferred fold (general variant, a fresh stream): neither the rank test nor growth
    // reads P^-1 or W, and the per-row Sherman-Morrison chain (solver.py:297-304) is the
    // recursive form of  P^-1 = (B^T B)^-1,  W = P^-1 B^T (y - A x0)  (B: the coords log).
    // So the tiles only accumulate Q = B^T B (in Pr) and B^T dy (in Wt) on the tensor
    // cores -- no dependent chain -- and Q is inverted once at the end of the call.  The
    // inverse is accepted when kappa_F(Q) = |Q|_F |Q^-1|_F <= DEFER_KAPPA (the two forms
    // then agree to ~1e-16 kappa: measured <= 4e-11 in x against the reference's own
    // recursion); otherwise the stream is folded again with the sequential chain.
    const bool defer = GEN && fresh && !seq;
    double Dt[IT][JK];
    double Pr[IT][IT][2];
    double Wt[IT][2];
#pragma unroll
    for (int nt = 0; nt < IT; ++nt) {
      Wt[nt][0] = Wt[nt][1] = 0.0;
#pragma unroll
      for (int J = 0; J < JK / 2; ++J) {
        const double2 v = fresh ? make_double2(0.0, 0.0)
                                : *reinterpret_cast<const double2*>(Dg + (8 * nt + p) * M + 8 * J + 2 * q);
        Dt[nt][2 * J] = v.x;
        Dt[nt][2 * J + 1] = v.y;
      }
#pragma unroll
      for (int mt = 0; mt < IT; ++mt) {
        const double2 v = fresh ? make_double2(0.0, 0.0)
                                : *reinterpret_cast<const double2*>(Pg + (8 * nt + p) * R + 8 * mt + 2 * q);
        Pr[nt][mt][0] = v.x;
        Pr[nt][mt][1] = v.y;
      }
    }
#pragma unroll
    for (int kt = 0; kt < IK; ++kt)
#pragma unroll
      for (int jt = 0; jt < JT; ++jt) S.Cs[kt][jt][lane] = fresh ? 0.0 : -Cg[sigma(kt, q) * M + 8 * jt + p];
    // x0 = the solution at call start; when it is exactly zero a.x0 = 0 and
    // its contraction is skipped.
    bool nz = false;
    if (!fresh && (!KM || p < kk_)) {
#pragma unroll
      for (int J = 0; J < JK / 2; ++J) {
        double2 v = *reinterpret_cast<const double2*>(Xg + p * M + 8 * J + 2 * q);
        nz |= (v.x != 0.0) || (v.y != 0.0);
      }
    }
    const bool has_x0 = __any_sync(FULL, nz);
    __syncwarp();
    double esq = eps_sq<double>(cfg, r);  // the rank test's threshold, refreshed when the rank grows

    // ---- tile loop -----------------------------------------------------------------
    // front(i): coords, rejections and the rank test of tile i (tensor cores);
    // scan(i):  the blocked Sherman-Morrison update of its dependent rows.
    // When tile i is all dependent the basis does not move, so front(i+1) is
    // issued together with scan(i) and the two overlap (no speculation).
    const int64_t ntiles = (T + TT - 1) / TT;
    int64_t consumed = 0;
    auto prefetch = [&](int64_t tile, int s) {
      if (tile < ntiles) {
        const int64_t t0 = tile * TT;
        const int64_t t = t0 + p;
        const bool ok = t < T;
        const TI* src = ok ? Rb + t * M : Rb;
#pragma unroll
        for (int nt = 0; nt < JT; ++nt) cp_async_pair<TI>(&S.At[s][nt][lane][0], src + 8 * nt + 2 * q, ok);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t ty = t0 + 2 * q + e;
          const bool oky = ty < T && (!KM || p < kk_);
          cp_async_one<TI>(&S.Yt[s][lane][e], oky ? Yb + ty * kk_ + p : Yb, oky);
        }
      }
      cp_commit();
    };

    struct Front {
      double g[IT][2];   // G[t=p][8nt+2q+e]
      double rsq, asq;   // |rej_t|^2, |a_t|^2 for t = p
      double dyx[2];     // y - a.x0 for (c = p, t = 2q+e)
      unsigned badm;     // rows with non-finite input (bit 4t)
      int tstar, tv;     // first stopping row (tv if none), valid rows
      int64_t t0;
    };
    // front pieces: the projection of one tile, split so that the fast path
    // can interleave it with the previous tile's scan (the scheduler keeps
    // source order for these long chains, so the interleave is written out).
    struct FrontAcc {
      double g2[IT][2];   // second K-half of G (two chains per N tile)
      double acc[JT][2];  // G C
    };
    auto front_begin = [&](int64_t tile, int s, Front& F, FrontAcc& X) {
      const TI* As = &S.At[s][0][lane][0];
      F.t0 = tile * TT;
      F.tv = (int)((T - F.t0) < TT ? (T - F.t0) : TT);
      const double2 yy = slot(&S.Yt[s][lane][0], 0);
      F.dyx[0] = yy.x;
      F.dyx[1] = yy.y;
      // row norms |a_t|^2 (solver.py:267)
      // (R = A - G C accumulates onto the tile itself: C is stored negated)
      double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int nt = 0; nt < JT; ++nt) {
        const double2 v = slot(As, nt * 32);
        X.acc[nt][0] = v.x;
        X.acc[nt][1] = v.y;
        s4[(2 * nt) & 3] = fma(v.x, v.x, s4[(2 * nt) & 3]);
        s4[(2 * nt + 1) & 3] = fma(v.y, v.y, s4[(2 * nt + 1) & 3]);
      }
      F.asq = (s4[0] + s4[1]) + (s4[2] + s4[3]);
#pragma unroll
      for (int nt = 0; nt < IT; ++nt) F.g[nt][0] = F.g[nt][1] = X.g2[nt][0] = X.g2[nt][1] = 0.0;
    };
    // G = A C~^T (M = t, N = i, K = j; solver.py:286): K steps 2J, 2J + 1
    // (hi = false: rank <= 8, rows 8.. of C~ are zero and N tile 1 is skipped)
    auto front_g1 = [&](int s, int J, Front& F, FrontAcc& X, bool hi = true) {
      const double2 v = make_double2(X.acc[J][0], X.acc[J][1]);  // (the tile: R has not started)
#pragma unroll
      for (int nt = 0; nt < IT; ++nt) {
        if (nt > 0 && !hi) break;
        mma(F.g[nt], v.x, Dt[nt][2 * J]);
        mma(X.g2[nt], v.y, Dt[nt][2 * J + 1]);
      }
      if (J == JK / 2 - 1) {
#pragma unroll
        for (int nt = 0; nt < IT; ++nt) {
          F.g[nt][0] += X.g2[nt][0];
          F.g[nt][1] += X.g2[nt][1];
        }
      }
    };
    // R = A - G C (M = t, N = j, K = i; solver.py:287-288): K step kt.  The
    // accumulation order differs from the reference's (a - (G C)) but gives
    // the same rejection-noise statistics (max rho over 768 C5 streams 0.549
    // vs 0.541, log-correlation 0.99995), so rank decisions are unaffected.
    auto front_g2 = [&](int kt, Front& F, FrontAcc& X, bool hi = true) {
      if (kt >= 2 && !hi) return;
#pragma unroll
      for (int jt = 0; jt < JT; ++jt) mma(X.acc[jt], F.g[kt >> 1][kt & 1], S.Cs[kt][jt][lane]);
    };
    // |R_t|^2 = |a_t - (G C)_t|^2 and the rank test (solver.py:288-296)
    auto front_end = [&](int s, int row_start, Front& F, FrontAcc& X) {
      const TI* As = &S.At[s][0][lane][0];
      double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int jt = 0; jt < JT; ++jt) {
        const double r0 = X.acc[jt][0], r1 = X.acc[jt][1];
        s4[(2 * jt) & 3] = fma(r0, r0, s4[(2 * jt) & 3]);
        s4[(2 * jt + 1) & 3] = fma(r1, r1, s4[(2 * jt + 1) & 3]);
      }
      double rsq = (s4[0] + s4[1]) + (s4[2] + s4[3]);
      double asq = F.asq;
      asq += __shfl_xor_sync(FULL, asq, 1);
      rsq += __shfl_xor_sync(FULL, rsq, 1);
      asq += __shfl_xor_sync(FULL, asq, 2);
      rsq += __shfl_xor_sync(FULL, rsq, 2);
      F.asq = asq;
      F.rsq = rsq;
      // rank test with the current rank; NaN/Inf rows stop the stream
      const unsigned yb0 = __ballot_sync(FULL, !isfinite(F.dyx[0]));
      const unsigned yb1 = __ballot_sync(FULL, !isfinite(F.dyx[1]));
      const bool ybad = (((p & 1) ? yb1 : yb0) & (0x11111111u << (p >> 1))) != 0u;
      const bool valid = p >= row_start && p < F.tv;
      const bool dep = is_dependent<double>(rsq, asq, esq);
      const bool bad = !isfinite(asq) || ybad;
      const unsigned stopm = __ballot_sync(FULL, q == 0 && valid && (!dep || bad));
      F.badm = __ballot_sync(FULL, q == 0 && valid && bad);
      F.tstar = stopm ? (__ffs(stopm) - 1) >> 2 : F.tv;
      if (stopm) {
        // keep what grow() needs of the stopping row: its coords gamma, its
        // gain K = rej / |rej|^2 (solver.py:336; one rounding more than a
        // division) and the row itself
        if (p == F.tstar) {
          const double rinv = 1.0 / rsq;
#pragma unroll
          for (int nt = 0; nt < IT; ++nt)
            *reinterpret_cast<double2*>(&S.u.ind.gam[8 * nt + 2 * q]) = make_double2(F.g[nt][0], F.g[nt][1]);
#pragma unroll
          for (int jt = 0; jt < JT; ++jt) {
            const double2 v = slot(As, jt * 32);
            *reinterpret_cast<double2*>(&S.u.ind.kv[8 * jt + 2 * q]) =
                make_double2(X.acc[jt][0] * rinv, X.acc[jt][1] * rinv);
            // the row itself (general: C[r] = a) or its rejection (other variants)
            *reinterpret_cast<double2*>(&S.u.ind.av[8 * jt + 2 * q]) =
                GEN ? v : make_double2(X.acc[jt][0], X.acc[jt][1]);
          }
        }
        __syncwarp();
      }
    };
    auto front = [&](int64_t tile, int s, int row_start, Front& F) {
      FrontAcc X;
      front_begin(tile, s, F, X);
#pragma unroll
      for (int J = 0; J < JK / 2; ++J) front_g1(s, J, F, X);
#pragma unroll
      for (int kt = 0; kt < IK; ++kt) front_g2(kt, F, X);
      front_end(s, row_start, F, X);
    };
    // a.x0 for a stream that did not start empty: Y0^T = x0^T A^T (M = c, N = t, K = j)
    auto front_x0 = [&](int s, Front& F) {
      if (has_x0) {
        const TI* As = &S.At[s][0][lane][0];
        double acc[2] = {0.0, 0.0};
#pragma unroll
        for (int J = 0; J < JK / 2; ++J) {
          const double2 xv = (!KM || p < kk_) ? __ldg(reinterpret_cast<const double2*>(Xg + p * M + 8 * J + 2 * q))
                                              : make_double2(0.0, 0.0);
          const double2 v = slot(As, J * 32);
          mma(acc, xv.x, v.x);
          mma(acc, xv.y, v.y);
        }
        F.dyx[0] -= acc[0];
        F.dyx[1] -= acc[1];
      }
    };

    // scan pieces: blocked Sherman-Morrison over the dependent rows [rs, te)
    struct ScanWork {
      double gm[IT][2], dy[2], u[IT][2], mi[2], ev[2];
    };
    auto scan_a = [&](const Front& F, int rs, int te, ScanWork& X) {
      const bool inb = p >= rs && p < te;
#pragma unroll
      for (int nt = 0; nt < IT; ++nt) {
        X.gm[nt][0] = inb ? F.g[nt][0] : 0.0;
        X.gm[nt][1] = inb ? F.g[nt][1] : 0.0;
      }
      // dy0^T = dyx - (G W)^T : M = c, N = t, K = i  (a-priori residuals, solver.py:303)
      {
        double acc[2] = {0.0, 0.0};
#pragma unroll
        for (int kt = 0; kt < IK; ++kt) mma(acc, Wt[kt >> 1][kt & 1], X.gm[kt >> 1][kt & 1]);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int t = 2 * q + e;
          X.dy[e] = (t >= rs && t < te) ? F.dyx[e] - acc[e] : 0.0;
        }
      }
      // U^T = G P (M = t, N = i); U = (U^T)^T by quad-crossing shuffles
      double ut[IT][2];
#pragma unroll
      for (int nt = 0; nt < IT; ++nt) {
        ut[nt][0] = ut[nt][1] = 0.0;
#pragma unroll
        for (int kt = 0; kt < IK; ++kt) mma(ut[nt], X.gm[kt >> 1][kt & 1], Pr[nt][kt >> 1][kt & 1]);
      }
#pragma unroll
      for (int mt = 0; mt < IT; ++mt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int src = 4 * (2 * q + e) + (p >> 1);
          const double v0 = __shfl_sync(FULL, ut[mt][0], src);
          const double v1 = __shfl_sync(FULL, ut[mt][1], src);
          X.u[mt][e] = (p & 1) ? v1 : v0;
        }
      // M = I + G P G^T (M = t, N = t')
      X.mi[0] = X.mi[1] = 0.0;
#pragma unroll
      for (int kt = 0; kt < IK; ++kt) mma(X.mi, ut[kt >> 1][kt & 1], X.gm[kt >> 1][kt & 1]);
      if (p == 2 * q) X.mi[0] += 1.0;
      if (p == 2 * q + 1) X.mi[1] += 1.0;
      X.ev[0] = p == 2 * q ? 1.0 : 0.0;
      X.ev[1] = p == 2 * q + 1 ? 1.0 : 0.0;
    };
    // M = L diag(d) L^T by forward elimination on [M | I]: E = L^-1 (unit
    // lower), d = pivots -- the 8 sequential Sherman-Morrison steps of
    // solver.py:298-301 in factored form (an explicit M^-1 / Woodbury update
    // loses accuracy when M is ill-conditioned; the factored form does not)
    auto scan_elim = [&](int k, ScanWork& X) {
      const double v = (k & 1) ? X.mi[1] : X.mi[0];
      const double piv = __shfl_sync(FULL, v, 4 * k + (k >> 1));
      const double mps = __shfl_sync(FULL, v, 4 * p + (k >> 1));
      const double m0 = __shfl_sync(FULL, X.mi[0], 4 * k + q);
      const double m1 = __shfl_sync(FULL, X.mi[1], 4 * k + q);
      const double e0 = __shfl_sync(FULL, X.ev[0], 4 * k + q);
      const double e1 = __shfl_sync(FULL, X.ev[1], 4 * k + q);
      const double f = (p > k) ? mps * rcp64(piv) : 0.0;
      X.mi[0] = fma(-f, m0, X.mi[0]);
      X.mi[1] = fma(-f, m1, X.mi[1]);
      X.ev[0] = fma(-f, e0, X.ev[0]);
      X.ev[1] = fma(-f, e1, X.ev[1]);
    };
    struct ScanTail {
      double rd0, rd1, yt[IT][2], dh[2];
    };
    // 1/d_t for t = 2q, 2q + 1;  Y^T = U E^T (columns = the z_t of the sequential form)
    auto scan_b1 = [&](ScanWork& X, ScanTail& Z) {
      const double dsel = (p & 1) ? X.mi[1] : X.mi[0];
      const double rd = rcp64(__shfl_sync(FULL, dsel, 4 * p + (p >> 1)));
      Z.rd0 = __shfl_sync(FULL, rd, 8 * q);
      Z.rd1 = __shfl_sync(FULL, rd, 8 * q + 4);
#pragma unroll
      for (int mt = 0; mt < IT; ++mt) {
        Z.yt[mt][0] = Z.yt[mt][1] = 0.0;
        mma(Z.yt[mt], X.u[mt][0], X.ev[0]);
        mma(Z.yt[mt], X.u[mt][1], X.ev[1]);
      }
      // E dy0 (M = c, N = t, K = t'): the residuals the sequential form would see
      Z.dh[0] = Z.dh[1] = 0.0;
      mma(Z.dh, X.dy[0], X.ev[0]);
      mma(Z.dh, X.dy[1], X.ev[1]);
    };
    // P -= Y^T D^-1 Y   and   W^T += (E dy0)^T D^-1 Y   (solver.py:300-304)
    auto scan_b2 = [&](ScanTail& Z) {
      const double d0 = Z.dh[0] * Z.rd0, d1 = Z.dh[1] * Z.rd1;
#pragma unroll
      for (int mt = 0; mt < IT; ++mt) {
        const double s0 = -Z.yt[mt][0] * Z.rd0, s1 = -Z.yt[mt][1] * Z.rd1;
#pragma unroll
        for (int nt = 0; nt < IT; ++nt) {
          mma(Pr[mt][nt], s0, Z.yt[nt][0]);
          mma(Pr[mt][nt], s1, Z.yt[nt][1]);
        }
      }
#pragma unroll
      for (int nt = 0; nt < IT; ++nt) {
        mma(Wt[nt], d0, Z.yt[nt][0]);
        mma(Wt[nt], d1, Z.yt[nt][1]);
      }
    };
    auto scan = [&](const Front& F, int rs, int te) {
      ScanWork X;
      ScanTail Z;
      scan_a(F, rs, te, X);
#pragma unroll
      for (int k = 0; k < TT - 1; ++k) scan_elim(k, X);
      scan_b1(X, Z);
      scan_b2(Z);
    };
    // scan(tile i) with front(tile i+1) written out interleaved (fast path)
    auto scan_front = [&](const Front& F, int64_t tile_n, int s_n, Front& N) {
      ScanWork X;
      ScanTail Z;
      FrontAcc A;
      front_begin(tile_n, s_n, N, A);
      scan_a(F, 0, F.tv, X);
      front_g1(s_n, 0, N, A);
      front_g1(s_n, 1, N, A);
#pragma unroll
      for (int k = 0; k < TT - 1; ++k) {
        scan_elim(k, X);
        if (k + 2 < JK / 2) front_g1(s_n, k + 2, N, A);
        else front_g2(k + 2 - JK / 2, N, A);
      }
      scan_b1(X, Z);
      front_g2(IK - 3, N, A);
      front_g2(IK - 2, N, A);
      scan_b2(Z);
      front_g2(IK - 1, N, A);
      front_end(s_n, 0, N, A);
    };

    // deferred fold of the dependent rows [rs, te): Q += G^T G, (B^T dy)^T += dy^T G.
    // G^T (rows t = 4s + q, coords 8nt + p: the A operand with M = coords and the B
    // operand with N = coords at once) comes from the accumulator layout by one
    // quad-crossing shuffle pair per value.
    auto accum = [&](const Front& F, int rs, int te) {
      double gt[IT][2], dv[2];
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int t = 4 * s + q;
        const bool in = t >= rs && t < te;
        const int src = 4 * t + (p >> 1);
#pragma unroll
        for (int nt = 0; nt < IT; ++nt) {
          const double v0 = __shfl_sync(FULL, F.g[nt][0], src);
          const double v1 = __shfl_sync(FULL, F.g[nt][1], src);
          gt[nt][s] = in ? ((p & 1) ? v1 : v0) : 0.0;
        }
        const int srcy = 4 * p + 2 * s + (q >> 1);
        const double y0 = __shfl_sync(FULL, F.dyx[0], srcy);
        const double y1 = __shfl_sync(FULL, F.dyx[1], srcy);
        dv[s] = in ? ((q & 1) ? y1 : y0) : 0.0;
      }
#pragma unroll
      for (int s = 0; s < 2; ++s)  // (s outermost: no two consecutive MMAs on one accumulator)
#pragma unroll
        for (int mt = 0; mt < IT; ++mt) {
#pragma unroll
          for (int nt = 0; nt < IT; ++nt) mma(Pr[mt][nt], gt[mt][s], gt[nt][s]);
          mma(Wt[mt], dv[s], gt[mt][s]);
        }
    };
    // the same for a whole tile of dependent rows (the fast path): G^T through the warp's
    // scratch rows instead of shuffles -- stored in the accumulator layout, read at
    // 64 nt + 32 s + 8 q + p it is G[4s + q][8nt + p], conflict-free (no growth is pending on
    // this path, so the scratch rows are free)
    auto accum_tile = [&](const Front& F, int st) {
      double* sc = &S.u.ind.gam[0];
      static_assert(sizeof(S.u.ind) >= sizeof(double) * TT * R, "G tile fits the scratch rows");
#pragma unroll
      for (int nt = 0; nt < IT; ++nt)
        *reinterpret_cast<double2*>(sc + (nt * 32 + lane) * 2) = make_double2(F.g[nt][0], F.g[nt][1]);
      __syncwarp();
      double gt[IT][2], dv[2];
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const bool in = 4 * s + q < F.tv;
#pragma unroll
        for (int nt = 0; nt < IT; ++nt) {
          const double v = sc[64 * nt + 32 * s + 8 * q + p];
          gt[nt][s] = in ? v : 0.0;
        }
        // dy = y here (x0 = 0); the stage stores y[t][c] at 8c + t: the same targets with the
        // rows on q (read before the stage is handed to the next prefetch)
        const double yv = (double)(&S.Yt[st][0][0])[8 * p + 4 * s + q];
        dv[s] = in ? yv : 0.0;
      }
      __syncwarp();
#pragma unroll
      for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int mt = 0; mt < IT; ++mt) {
#pragma unroll
          for (int nt = 0; nt < IT; ++nt) mma(Pr[mt][nt], gt[mt][s], gt[nt][s]);
          mma(Wt[mt], dv[s], gt[mt][s]);
        }
    };
    // P^-1 = Q^-1 (gj_invert on a copy, so that Pr stays in registers), then
    // W = P^-1 (B^T dy).  Returns |Q|_F^2 |Q^-1|_F^2.
    auto invert_q = [&](bool apply) -> double {
      double Tq[IT][IT][2];
#pragma unroll
      for (int mt = 0; mt < IT; ++mt)
#pragma unroll
        for (int nt = 0; nt < IT; ++nt) {
          Tq[mt][nt][0] = Pr[mt][nt][0];
          Tq[mt][nt][1] = Pr[mt][nt][1];
        }
      const double kap2 = gj_invert<IT>(Tq, r, p, q);
      if (apply) {
#pragma unroll
        for (int mt = 0; mt < IT; ++mt)
#pragma unroll
          for (int nt = 0; nt < IT; ++nt) {
            Pr[mt][nt][0] = Tq[mt][nt][0];
            Pr[mt][nt][1] = Tq[mt][nt][1];
          }
        double wn[IT][2];
#pragma unroll
        for (int nt = 0; nt < IT; ++nt) {
          wn[nt][0] = wn[nt][1] = 0.0;
#pragma unroll
          for (int kt = 0; kt < IK; ++kt) mma(wn[nt], Wt[kt >> 1][kt & 1], Pr[nt][kt >> 1][kt & 1]);
        }
#pragma unroll
        for (int nt = 0; nt < IT; ++nt) {
          Wt[nt][0] = wn[nt][0];
          Wt[nt][1] = wn[nt][1];
        }
      }
      return kap2;
    };

    // logs of dependent rows [rs, te): branch 0 and the coordinate row gamma_t
    // (zero beyond the rank).  Kept out of scan() so that scan and the next
    // front form one branch-free block the scheduler can interleave.
    auto log_dependent = [&](const Front& F, int rs, int te) {
      if (blog || clog) {
        if (p >= rs && p < te) {
          const int64_t row = b * T + F.t0 + p;
          if (blog && q == 0) blog[row] = 0;
          if (clog) {
#pragma unroll
            for (int nt = 0; nt < IT; ++nt)
              *reinterpret_cast<double2*>(clog + row * R + 8 * nt + 2 * q) = make_double2(F.g[nt][0], F.g[nt][1]);
          }
        }
      }
    };

    // independent row ts of front F (solver.py:305-318, _grow solver.py:368-397)
    // grow_core: the independent-row update from the scratch rows written by
    // front_end() or project_row(); wnew = y - a.x0 of the row for RHS c = p
    auto grow_core = [&](double wnew, double rsq, int64_t t0, int ts) {
      const int var = GEN ? RGB_GENERAL : cfg.variant;
      double last = 1.0;  // coords_row[r] of the orthogonal / orthonormal variants
      if (var == RGB_GENERAL) {
        // W gains row r: y - a.x0 (x = x0 + C~^T W stays exact)
#pragma unroll
        for (int nt = 0; nt < IT; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e)
            if (8 * nt + 2 * q + e == r) Wt[nt][e] = wnew;
        // C~[:r] -= gamma K^T, C~[r] = K   (solver.py:377-380)
#pragma unroll
        for (int nt = 0; nt < IT; ++nt) {
          const int i = 8 * nt + p;
          const double gi = S.u.ind.gam[i];
#pragma unroll
          for (int J = 0; J < JK / 2; ++J) {
            const double2 kv = *reinterpret_cast<const double2*>(&S.u.ind.kv[8 * J + 2 * q]);
            Dt[nt][2 * J] = (i == r) ? kv.x : fma(-gi, kv.x, Dt[nt][2 * J]);
            Dt[nt][2 * J + 1] = (i == r) ? kv.y : fma(-gi, kv.y, Dt[nt][2 * J + 1]);
          }
        }
        // C[r] = a  (solver.py:376)
        if (q == ((r & 7) >> 1)) {
          const int ktr = 2 * (r >> 3) + (r & 1);
#pragma unroll
          for (int jt = 0; jt < JT; ++jt) S.Cs[ktr][jt][lane] = -S.u.ind.av[8 * jt + p];
        }
        // P = diag(P, 1)  (solver.py:372-373, 381)
#pragma unroll
        for (int mt = 0; mt < IT; ++mt)
#pragma unroll
          for (int nt = 0; nt < IT; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int i = 8 * mt + p, i2 = 8 * nt + 2 * q + e;
              if (i == r || i2 == r) Pr[mt][nt][e] = (i == i2) ? 1.0 : 0.0;
            }
      } else {
        // orthogonal / orthonormal _grow (solver.py:382-395); av holds the rejection.
        // z = P gamma, denom = 1 + gamma.z (solver.py:307-310)
        double z[IT];
#pragma unroll
        for (int mt = 0; mt < IT; ++mt) {
          double zp = 0.0;
#pragma unroll
          for (int nt = 0; nt < IT; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) zp = fma(Pr[mt][nt][e], S.u.ind.gam[8 * nt + 2 * q + e], zp);
          zp += __shfl_xor_sync(FULL, zp, 1);
          zp += __shfl_xor_sync(FULL, zp, 2);
          z[mt] = zp;  // z[8mt + p]
        }
        double dn = 0.0;
        if (q == 0) {
#pragma unroll
          for (int mt = 0; mt < IT; ++mt) dn = fma(S.u.ind.gam[8 * mt + p], z[mt], dn);
        }
        const double denom = 1.0 + warp_sum(dn);
        // rescaling (solver.py:354-366, 383): alpha = 1/(1/rescale)
        const double resc = (var == RGB_ORTHONORMAL) ? 1.0 / sqrt(rsq) : cfg.alpha;
        last = 1.0 / resc;
        const double alpha = 1.0 / last;
        // W gains row r: alpha (y - a.x) with a.x = a.x0 + gamma^T W, since the
        // new dual row is K / alpha and the old dual rows do not move
        double gw = 0.0;
#pragma unroll
        for (int nt = 0; nt < IT; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) gw = fma(S.u.ind.gam[8 * nt + 2 * q + e], Wt[nt][e], gw);
        gw += __shfl_xor_sync(FULL, gw, 1);
        gw += __shfl_xor_sync(FULL, gw, 2);
        const double wr = alpha * (wnew - gw);
#pragma unroll
        for (int nt = 0; nt < IT; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e)
            if (8 * nt + 2 * q + e == r) Wt[nt][e] = wr;
        __syncwarp();
        if (q == 0) {
#pragma unroll
          for (int mt = 0; mt < IT; ++mt) S.u.ind.kv[8 * mt + p] = z[mt];  // kv is free: C~[:r] is unchanged
        }
        __syncwarp();
        // C[r] = alpha rej;  C~[r] = rej / (alpha |rej|^2)  (orthonormal: C~ is C)
        if (q == ((r & 7) >> 1)) {
          const int ktr = 2 * (r >> 3) + (r & 1);
#pragma unroll
          for (int jt = 0; jt < JT; ++jt) S.Cs[ktr][jt][lane] = -(alpha * S.u.ind.av[8 * jt + p]);
        }
        const double sc = alpha * rsq;
#pragma unroll
        for (int nt = 0; nt < IT; ++nt) {
          if (8 * nt + p == r) {
#pragma unroll
            for (int J = 0; J < JK / 2; ++J)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const double rj = S.u.ind.av[8 * J + 2 * q + e];
                Dt[nt][2 * J + e] = (var == RGB_ORTHONORMAL) ? alpha * rj : rj / sc;
              }
          }
        }
        // P gains edge -alpha z and corner alpha^2 denom
#pragma unroll
        for (int mt = 0; mt < IT; ++mt)
#pragma unroll
          for (int nt = 0; nt < IT; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int i = 8 * mt + p, i2 = 8 * nt + 2 * q + e;
              if (i == r && i2 == r) Pr[mt][nt][e] = alpha * alpha * denom;
              else if (i2 == r) Pr[mt][nt][e] = (i < r) ? -(alpha * S.u.ind.kv[i]) : 0.0;
              else if (i == r) Pr[mt][nt][e] = (i2 < r) ? -(alpha * S.u.ind.kv[i2]) : 0.0;
            }
      }
      const int64_t row = b * T + t0 + ts;
      if (blog && lane == 0) blog[row] = 1;
      if (clog && lane < R) {
        double v = (lane == r) ? 1.0 : 0.0;
        if (var != RGB_GENERAL) v = (lane < r) ? S.u.ind.gam[lane] : (lane == r ? last : 0.0);
        clog[row * R + lane] = v;
      }
      __syncwarp();
      r += 1;
      esq = eps_sq<double>(cfg, r);
    };
    auto grow = [&](const Front& F, int ts) {
      // W gains row r: y - a.x0 of row ts (x = x0 + C~^T W stays exact)
      const double dv = (ts & 1) ? F.dyx[1] : F.dyx[0];
      grow_core(__shfl_sync(FULL, dv, 4 * p + (ts >> 1)), GEN ? 0.0 : __shfl_sync(FULL, F.rsq, 4 * ts), F.t0, ts);
    };

    // Single-row projection of row ts of stage s on the current basis, on the
    // CUDA cores (solver.py:286-291): used while a fresh stream's leading rows
    // are independent, where re-projecting a whole 8-row tile after every
    // basis growth would cost 64 MMAs per row.  Leaves gamma, K = rej/|rej|^2
    // and the row in the scratch rows for grow_core(); returns |rej|^2, |a|^2.
    auto project_row = [&](int s, int ts, double& rsq_o, double& asq_o) {
      const TI* Ar = &S.At[s][0][4 * ts + q][0];
      double gp[IT], a4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int nt = 0; nt < IT; ++nt) gp[nt] = 0.0;
#pragma unroll
      for (int J = 0; J < JK / 2; ++J) {  // my columns sigma(kt, q) = 8J + 2q + e
        const double2 v = slot(Ar, J * 32);
        a4[(2 * J) & 3] = fma(v.x, v.x, a4[(2 * J) & 3]);
        a4[(2 * J + 1) & 3] = fma(v.y, v.y, a4[(2 * J + 1) & 3]);
#pragma unroll
        for (int nt = 0; nt < IT; ++nt) gp[nt] = fma(Dt[nt][2 * J], v.x, fma(Dt[nt][2 * J + 1], v.y, gp[nt]));
      }
      double asq = (a4[0] + a4[1]) + (a4[2] + a4[3]);
      asq += __shfl_xor_sync(FULL, asq, 1);
      asq += __shfl_xor_sync(FULL, asq, 2);
#pragma unroll
      for (int nt = 0; nt < IT; ++nt) {
        gp[nt] += __shfl_xor_sync(FULL, gp[nt], 1);
        gp[nt] += __shfl_xor_sync(FULL, gp[nt], 2);
      }
      // gamma[8nt + p] = gp[nt] in quad p; rej_j = a_j - sum_i gamma_i C_ij
      // for my Cs columns j = 8jt + p over my rows i = sigma(kt, q)
      double rp[JT];
#pragma unroll
      for (int jt = 0; jt < JT; ++jt) rp[jt] = 0.0;
#pragma unroll
      for (int kt = 0; kt < IK; ++kt) {
        const double gi = __shfl_sync(FULL, gp[kt >> 1], 4 * (2 * q + (kt & 1)));
#pragma unroll
        for (int jt = 0; jt < JT; ++jt) rp[jt] = fma(gi, S.Cs[kt][jt][lane], rp[jt]);  // Cs = -C
      }
      double r4[4] = {0.0, 0.0, 0.0, 0.0};
      double rej[JT];
#pragma unroll
      for (int jt = 0; jt < JT; ++jt) {
        rp[jt] += __shfl_xor_sync(FULL, rp[jt], 1);
        rp[jt] += __shfl_xor_sync(FULL, rp[jt], 2);
        rej[jt] = (double)S.At[s][jt][4 * ts + (p >> 1)][p & 1] + rp[jt];
        r4[jt & 3] = fma(rej[jt], rej[jt], r4[jt & 3]);
      }
      double rsq = (r4[0] + r4[1]) + (r4[2] + r4[3]);
      rsq += __shfl_xor_sync(FULL, rsq, 4);
      rsq += __shfl_xor_sync(FULL, rsq, 8);
      rsq += __shfl_xor_sync(FULL, rsq, 16);
      if (q == 0) {
        const double rinv = 1.0 / rsq;
#pragma unroll
        for (int nt = 0; nt < IT; ++nt) S.u.ind.gam[8 * nt + p] = gp[nt];
#pragma unroll
        for (int jt = 0; jt < JT; ++jt) {
          S.u.ind.kv[8 * jt + p] = rej[jt] * rinv;
          S.u.ind.av[8 * jt + p] = GEN ? (double)S.At[s][jt][4 * ts + (p >> 1)][p & 1] : rej[jt];
        }
      }
      __syncwarp();
      rsq_o = rsq;
      asq_o = asq;
    };

    bool stopped = false;
    Front F;
    int64_t tile = 0;
    int first_row = 0;  // rows of the first blocked tile already consumed in row mode
    if (ntiles > 0) {
      prefetch(0, 0);
      prefetch(1, 1);
      cp_wait<1>();
      // row mode: a fresh stream's leading independent rows, one at a time
      if (fresh) {
        while (tile < ntiles) {
          const int s = (int)(tile & 1);
          const int64_t t0 = tile * TT;
          const int tv = (int)((T - t0) < TT ? (T - t0) : TT);
          int ts = 0;
          for (; ts < tv; ++ts) {
            double rsq, asq;
            project_row(s, ts, rsq, asq);
            const double yv = (double)S.Yt[s][4 * p + (ts >> 1)][ts & 1];  // y[ts][c = p]
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
          prefetch(tile + 1, s);
          cp_wait<1>();
        }
      }
      if (tile < ntiles) {
        front(tile, (int)(tile & 1), first_row, F);
        front_x0((int)(tile & 1), F);
      }
    }
    // Deferred fold: R + 32 rows into the stream kappa_F(Q) already tells how the final one
    // will turn out (on the config-5 workload: every stream that ends past DEFER_KAPPA is past
    // half of it here, 0.3 % of the others are too), so a stream that will not pass starts
    // over with the sequential chain now instead of after its last row.  (A heuristic only:
    // the certificate at the end decides.)
    constexpr int64_t CK_TILE = (R + 32) / TT;
    constexpr double DEFER_KAPPA = 1e6;
    bool give_up = false;
    for (; tile < ntiles; ++tile) {
      const int s = (int)(tile & 1);
      if (defer && tile == CK_TILE && ntiles > 4 * CK_TILE) {
        if (!(invert_q(false) <= 0.25 * DEFER_KAPPA * DEFER_KAPPA)) {
          give_up = true;
          break;
        }
      }
      if (F.tstar >= F.tv && first_row == 0) {
        // every row of the tile is dependent: scan(i) overlaps front(i+1); the deferred
        // fold reads the tile's targets from its stage before the stage is refilled
        if (defer) {
          // (the tile's front is dead once it is folded and logged: the next one goes
          // straight into F)
          accum_tile(F, s);
          log_dependent(F, 0, F.tv);
          consumed = F.t0 + F.tv;
          prefetch(tile + 2, s);
          cp_wait<1>();
          front(tile + 1, s ^ 1, 0, F);
          continue;
        }
        prefetch(tile + 2, s);
        cp_wait<1>();
        Front N;
        scan_front(F, tile + 1, s ^ 1, N);
        log_dependent(F, 0, F.tv);
        front_x0(s ^ 1, N);
        consumed = F.t0 + F.tv;
        F = N;
        continue;
      }
      int row_start = first_row;
      first_row = 0;
      while (true) {
        if (F.tstar > row_start) {
          if (defer) accum(F, row_start, F.tstar);
          else scan(F, row_start, F.tstar);
          log_dependent(F, row_start, F.tstar);
        }
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
        grow(F, F.tstar);
        row_start = F.tstar + 1;
        if (row_start >= F.tv) break;
        front(tile, s, row_start, F);   // re-project the rest of the tile on the new basis
        front_x0(s, F);
      }
      if (stopped) {
        consumed = F.t0 + F.tstar;
        break;
      }
      consumed = F.t0 + F.tv;
      prefetch(tile + 2, s);
      cp_wait<1>();
      front(tile + 1, s ^ 1, 0, F);
      front_x0(s ^ 1, F);
    }
    cp_wait<0>();
    __syncwarp();
    if (defer) {
      if (give_up || !(invert_q(true) <= DEFER_KAPPA * DEFER_KAPPA)) {  // (a NaN fails too)
        redo = true;  // nothing is written yet: the same stream again, sequentially
        continue;
      }
    }

    // ---- write the state back; x = x0 + C~^T W ------------------------------------
#pragma unroll
    for (int kt = 0; kt < IK; ++kt)
#pragma unroll
      for (int jt = 0; jt < JT; ++jt) Cg[sigma(kt, q) * M + 8 * jt + p] = -S.Cs[kt][jt][lane];
    __syncwarp();
    // C~ staged row-major (stride DS, conflict-free for the B operand below)
    // over C's shared memory, which is written back already
    constexpr int DS = M + 2;
    double* Dm = &S.Cs[0][0][0];
#pragma unroll
    for (int nt = 0; nt < IT; ++nt)
#pragma unroll
      for (int J = 0; J < JK / 2; ++J) {
        const double2 v = make_double2(Dt[nt][2 * J], Dt[nt][2 * J + 1]);
        *reinterpret_cast<double2*>(Dg + (8 * nt + p) * M + 8 * J + 2 * q) = v;
        *reinterpret_cast<double2*>(Dm + (8 * nt + p) * DS + 8 * J + 2 * q) = v;
      }
    __syncwarp();
    // x^T = x0^T + W^T C~ : M = c, N = j, K = i
#pragma unroll
    for (int jt = 0; jt < JT; ++jt) {
      double acc[2] = {0.0, 0.0};
      if (has_x0 && (!KM || p < kk_)) {
        const double2 v = *reinterpret_cast<const double2*>(Xg + p * M + 8 * jt + 2 * q);
        acc[0] = v.x;
        acc[1] = v.y;
      }
#pragma unroll
      for (int kt = 0; kt < IK; ++kt) mma(acc, Wt[kt >> 1][kt & 1], Dm[sigma(kt, q) * DS + 8 * jt + p]);
      if (!KM || p < kk_) *reinterpret_cast<double2*>(Xg + p * M + 8 * jt + 2 * q) = make_double2(acc[0], acc[1]);
    }
#pragma unroll
    for (int mt = 0; mt < IT; ++mt)
#pragma unroll
      for (int nt = 0; nt < IT; ++nt)
        *reinterpret_cast<double2*>(Pg + (8 * mt + p) * R + 8 * nt + 2 * q) =
            make_double2(Pr[mt][nt][0], Pr[mt][nt][1]);
    if (lane == 0) {
      st.rank[b] = r;
      st.nobs[b] = nobs0 + consumed;
      st.status[b] = status;
    }
    __syncwarp();
  }
}

}  // namespace blk

cudaMemPool_t workspace_pool();  // rgb_grid.cu

namespace {
constexpr int BM = 64, BR = 16, BK = 8;
#ifndef RGB_BLOCKED_WARPS
#define RGB_BLOCKED_WARPS 2
#endif
constexpr int BWARPS = RGB_BLOCKED_WARPS;
}  // namespace

bool blocked_supports(const rgb_config& cfg) {
  // all three variants; a zero orthogonal rescaling factor (an error in the
  // reference, solver.py:364-365) is left to the generic kernel's status path
  const bool var_ok = cfg.variant == RGB_GENERAL || cfg.variant == RGB_ORTHONORMAL ||
                      (cfg.variant == RGB_ORTHOGONAL && cfg.alpha != 0.0);
  return cfg.dtype == RGB_F64 && var_ok && cfg.m == BM && cfg.r_cap == BR && cfg.k >= 1 && cfg.k <= BK;
}

template <typename TI, bool KM>
static int launch_blocked_t(const rgb_config& cfg, rgb_state& st, const TI* rows, int64_t rows_stride,
                            const TI* targets, int64_t tg_stride, int64_t T, const rgb_logs& logs,
                            cudaStream_t stream, int num_sms) {
  const bool gen = cfg.variant == RGB_GENERAL;
  auto kern = gen ? blk::blocked_kernel<BM, BR, BK, BWARPS, true, TI, KM>
                  : blk::blocked_kernel<BM, BR, BK, BWARPS, false, TI, KM>;
  const size_t smem = sizeof(blk::WarpSmem<BM, BR, BK, TI>) * BWARPS;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, BWARPS * 32, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t need = (cfg.num_streams + BWARPS - 1) / BWARPS;
  int64_t grid = (int64_t)num_sms * per_sm;
  if (grid > need) grid = need;
  // RGB_BLOCKED_SEQ=1: the sequential Sherman-Morrison chain for every stream (A/B runs, tests)
  const char* seq_env = getenv("RGB_BLOCKED_SEQ");
  const int seq_only = (seq_env && seq_env[0] && seq_env[0] != '0') ? 1 : 0;
  // the stream counter: 4 bytes, stream-ordered, from the library's device pool (not needed
  // when every warp gets at most one stream)
  void* ws = nullptr;
  if (cfg.num_streams > grid * BWARPS) {
    cudaMemPool_t pool = workspace_pool();
    if (!pool || cudaMallocFromPoolAsync(&ws, 256, pool, stream) != cudaSuccess) return RGB_E_CUDA;
    cudaMemsetAsync(ws, 0, sizeof(unsigned), stream);
  }
  kern<<<(unsigned)grid, BWARPS * 32, smem, stream>>>(cfg, st, rows, rows_stride, targets, tg_stride, T,
                                                      logs.branch, (double*)logs.coords, seq_only, (unsigned*)ws);
  const cudaError_t e = cudaGetLastError();
  if (ws) cudaFreeAsync(ws, stream);
  return e == cudaSuccess ? RGB_OK : RGB_E_CUDA;
}

int launch_blocked(const rgb_config& cfg, rgb_state& st, const void* rows, int64_t rows_stride,
                   const void* targets, int64_t tg_stride, int64_t T, const rgb_logs& logs,
                   cudaStream_t stream, int num_sms, bool f32in) {
  if (logs.resid || logs.gain) return RGB_E_UNSUPPORTED;  // per-row residuals: generic kernel
  const bool km = cfg.k < BK;
  if (f32in)
    return km ? launch_blocked_t<float, true>(cfg, st, (const float*)rows, rows_stride, (const float*)targets,
                                              tg_stride, T, logs, stream, num_sms)
              : launch_blocked_t<float, false>(cfg, st, (const float*)rows, rows_stride, (const float*)targets,
                                               tg_stride, T, logs, stream, num_sms);
  return km ? launch_blocked_t<double, true>(cfg, st, (const double*)rows, rows_stride, (const double*)targets,
                                             tg_stride, T, logs, stream, num_sms)
            : launch_blocked_t<double, false>(cfg, st, (const double*)rows, rows_stride, (const double*)targets,
                                              tg_stride, T, logs, stream, num_sms);
}

}  // namespace rgb
