// rgb_cluster.cu -- one large stream per thread-block cluster (sm_100a: DSMEM,
// mbarriers across the cluster, fp64 tensor cores), in 32-row panels.
//
// For a stream whose factors are too large for one SM but fit one cluster
// (config 2: m 1024, r 64 -- C~ and C are 1 MB) the stream runs on one cluster
// of NCOL + 1 CTAs:
//
//   column CTAs c < NCOL hold columns [c CW, (c + 1) CW) of C~ and C in shared
//     memory (MMA fragment order; CW = 64 or 72, columns past m masked) and run
//     the projection chain of every panel of TT = 32 rows (the north star's
//     blocked k = 32-row variant):
//       P1  G_c = A[:, cols] C~[:, cols]^T (+ a.x0 as 8 extra rows of C~)
//       --- column barrier
//       P2  G = sum_c G_c: CTA c reduces a 1/NCOL chunk from every column CTA's
//           shared memory (DSMEM, fixed order) and stores it into every column
//           CTA and into home's ring slot
//       --- column barrier
//       P3  R[:, cols] = A - G C[:, cols]; |R_t|^2, |a_t|^2 partials stored into
//           every column CTA and home's slot
//       --- column barrier; the slot is handed to home
//       P4  the rank test (identical sums everywhere); an independent row grows
//           C~ and C on the own columns (gamma, the rejection and |rej|^2 are all
//           local), the rest of its panel is re-projected;
//   the home CTA (rank NCOL) holds P^-1 and W and folds each projection's
//     dependent rows (LDL^T-factored Sherman-Morrison, 8-row blocks,
//     solver.py:297-304) and growth into them, reading G and the norm partials
//     from a 2-slot ring.
//
// The column barriers are mbarriers that only the column CTAs arrive on, and
// the ring is guarded by full/free mbarriers, so home's sequential P^-1 chain
// runs concurrently with the next panels' projections instead of stalling
// them; the hardware cluster barrier is used only at the end of a stream,
// where the column CTAs read W to form x = x0 + C~^T W.
//
// Deferred fold (general variant, a fresh stream): home only accumulates Q = B^T B and
// B^T dy per block (no LDL^T, no barrier inside a block) and inverts Q once at the end,
// accepted when kappa_F(Q) <= 1e6; otherwise the whole cluster folds the stream again with
// the chain (rgb_blocked.cu has the derivation; RGB_CLUSTER_SEQ=1 forces the chain).
// Config 2: 2.01 -> 1.78 ms.
#include <cooperative_groups.h>

#include <cstdlib>

#include "rgb_mma.cuh"

namespace cg = cooperative_groups;

namespace rgb {
namespace cls {

using blk::FULL;
using blk::mma;
using blk::rcp64;

constexpr int NT = 256;  // threads per CTA (8 warps)
constexpr int NW = NT / 32;
constexpr int MAXCL = 16;  // largest (non-portable) cluster: 15 column CTAs + home

template <int R, int TT, int CW, typename TI>
struct ColSmem {
  static constexpr int NXT = (R + 8) / 8, GX = R + 8, GS = R + 12, AS = CW + 4;
  double Ds[NXT][CW / 4][32];    // C~ (+ x0^T as rows R..R+7) of my columns, B-fragment order
  double Cs[R / 4][CW / 8][32];  // -C of my columns, B-fragment order
  TI At[2][TT][AS];              // panel rows, my columns (2 stages, input type)
  TI Yv[2][TT][8];               // panel targets (non-finite check)
  double Gp[TT * GX];            // my G partial [t][i] (read by the chunk reducers)
  double Gs[TT][GS];             // reduced G (+ a.x0), written by the chunk reducers
  double Rs[TT][CW];             // rejections of my columns
  double nrm[MAXCL][2][TT];      // |R_t|^2, |a_t|^2 partials of every column CTA
  double scal[TT];               // |R_t|^2 totals
  double Wl[R][8];               // W, copied from home at the end of a stream
  int flags[4];
};

template <int R, int TT, typename TI>
struct HomeSmem {
  static constexpr int GS = R + 12, PS = R + 2;
  double slotG[2][TT][GS];       // ring: reduced G of a projection
  double slotN[2][MAXCL][2][TT]; //       its norm partials
  double Ps[R][PS];              // P^-1
  double Wb[R][8];               // W (x = x0 + C~^T W)
  double Ub[2][R][8];            // U of the block, double-buffered (no barrier between blocks)
  double Eb[8][8], Dy[8][8];
  double rd[8];
  double zg[R + 8];              // |rej_t|^2 of the rank test; non-general growth: z = P gamma, gamma^T W
  double Sp[NW][32][4];          // per-warp partials of S = G U and G W
  TI Yv[2][TT][8];               // panel targets
  int flags[4];
};

template <int R, int TT, int CW, typename TI>
struct Smem {
  unsigned long long colbar;        // column barrier: NCOL arrivals per phase
  unsigned long long slot_free[2];  // column CTAs: home released slot j (1 arrival)
  unsigned long long slot_full[2];  // home: slot j filled (NCOL arrivals)
  unsigned long long pad_;
  union {
    ColSmem<R, TT, CW, TI> col;
    HomeSmem<R, TT, TI> home;
  } u;
};

__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

// arrive (release, cluster scope) on the barrier at the same offset in CTA `rank`
__device__ __forceinline__ void mbar_arrive_at(unsigned long long* bar, unsigned rank) {
  unsigned a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_addr(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
}

// wait (acquire, cluster scope) for the completion of the phase with this parity
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred done;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 done, [%0], %1;\n"
      " @!done bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// phase timing (debug builds only: -DRGB_CLUSTER_PROBE): ns per phase summed
// over the run, for column CTA 0 (row 0) and home (row 1), read back with
// rgb_cluster_probe()
#ifdef RGB_CLUSTER_PROBE
__device__ unsigned long long g_probe[2][16];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define PROBE(i)                                                          \
  do {                                                                    \
    if (tid == 0 && (c == 0 || home)) {                                   \
      const unsigned long long now_ = gtime();                            \
      atomicAdd(&g_probe[home ? 1 : 0][i], now_ - probe_t);               \
      probe_t = now_;                                                     \
    }                                                                     \
  } while (0)
#else
#define PROBE(i) \
  do {           \
  } while (0)
#endif

// GEN: general variant only; !GEN: orthogonal / orthonormal (solver.py:382-395)
template <int R, int TT, int CW, bool GEN, typename TI>
__global__ void __launch_bounds__(NT, 1) cluster_kernel(rgb_config cfg, rgb_state st, const TI* __restrict__ rows,
                                                        int64_t rstride, const TI* __restrict__ tgts, int64_t tstride,
                                                        int64_t T, uint8_t* __restrict__ blog,
    double* __restrict__ clog, int seq_only) {
  constexpr int IT = R / 8, IK = R / 4, NXT = (R + 8) / 8, GX = R + 8, MT = TT / 8;
  constexpr int NG = NW / MT;                       // warps per M tile
  constexpr int NJ1 = (NXT + NG - 1) / NG;          // P1 N tiles per warp
  constexpr int NJ3 = (CW / 8 + NG - 1) / NG;       // P3 N tiles per warp
  constexpr int TPR = NT / TT;                      // norm threads per row
  constexpr int HGS = HomeSmem<R, TT, TI>::GS;
  static_assert(NW % MT == 0 && TPR >= 2 && (TPR & (TPR - 1)) == 0 && MAXCL <= 2 * TPR, "tiling");
  using SM = Smem<R, TT, CW, TI>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SM& S = *reinterpret_cast<SM*>(smem_raw);
  cg::cluster_group cluster = cg::this_cluster();
  const int ncl = (int)cluster.num_blocks();
  const int ncol = ncl - 1;
  const int c = (int)cluster.block_rank();
  const bool home = (c == ncol);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, p = lane >> 2, q = lane & 3;
  const int M = cfg.m, k = cfg.k, c0 = c * CW;
  const int64_t cid = blockIdx.x / ncl, ncid = gridDim.x / ncl;
  auto rem = [&](int u) { return cluster.map_shared_rank(&S, u); };
#ifdef RGB_CLUSTER_PROBE
  unsigned long long probe_t = gtime();
#endif

  if (tid == 0) {
    mbar_init(&S.colbar, (unsigned)ncol);
    mbar_init(&S.slot_free[0], 1u);
    mbar_init(&S.slot_free[1], 1u);
    mbar_init(&S.slot_full[0], (unsigned)ncol);
    mbar_init(&S.slot_full[1], (unsigned)ncol);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster_sync_all();

  unsigned nsync = 0;  // column barriers passed (phase parity)
  unsigned proj = 0;   // projections so far (ring slot = proj & 1), the same count in every CTA
  // column barrier: the CTA's writes are ordered before its arrivals by the CTA
  // barrier, and one thread per column CTA carries the release to that CTA
  auto colsync = [&]() {
    __syncthreads();
    if (tid < ncol) mbar_arrive_at(&S.colbar, (unsigned)tid);
    mbar_wait(&S.colbar, nsync & 1u);
    nsync += 1;
  };

  bool redo = false;  // the stream's deferred fold failed its conditioning certificate
  for (int64_t b = cid; b < cfg.num_streams; b += ncid) {
    const bool seq = redo || seq_only != 0;
    redo = false;
    int status = st.status[b];
    if (status) continue;  // uniform across the cluster
    int r = st.rank[b];
    // Deferred fold (general variant, a fresh stream; rgb_blocked.cu has the derivation): the
    // home CTA only accumulates Q = B^T B and B^T dy from each projection's G -- no LDL^T
    // chain, no barrier inside a block -- and inverts Q once at the end of the call; the
    // result is accepted when kappa_F(Q) <= 1e6, otherwise the whole cluster folds the
    // stream again with the sequential chain (a fresh stream's factors are never read, so
    // the column CTAs' early write-back of C~ and C does not matter).
    const bool fresh = (r == 0);
    const bool defer = GEN && fresh && !seq;
    const int64_t nobs0 = st.nobs[b];
    const int rc = cfg.r_cap;  // stored capacity (<= R): global row stride; rows past it are zero
    double* Cg = reinterpret_cast<double*>(st.basis) + b * (int64_t)rc * M;
    double* Dg = reinterpret_cast<double*>(st.dual) + b * (int64_t)rc * M;
    double* Pg = reinterpret_cast<double*>(st.gram_inv) + b * (int64_t)rc * rc;
    double* Xg = reinterpret_cast<double*>(st.x) + b * (int64_t)k * M;
    const TI* Rb = rows + b * rstride;
    const TI* Yb = tgts + b * tstride;
    const int64_t npan = (T + TT - 1) / TT;
    int64_t consumed = 0;
    bool stopped = false;

    if (!home) {
      // ======================= column CTA ==========================================
      auto& C = S.u.col;
      for (int e = tid; e < NXT * (CW / 4) * 32; e += NT) {
        const int l = e & 31, kt = (e >> 5) % (CW / 4), nt = e / (32 * (CW / 4));
        const int i = 8 * nt + (l >> 2), col = c0 + 4 * kt + (l & 3);
        double v = 0.0;
        if (col < M) {
          if (i < rc) v = fresh ? 0.0 : Dg[(int64_t)i * M + col];
          else if (i >= R && i - R < k) v = Xg[(int64_t)(i - R) * M + col];
        }
        C.Ds[nt][kt][l] = v;
      }
      for (int e = tid; e < (R / 4) * (CW / 8) * 32; e += NT) {
        const int l = e & 31, nt = (e >> 5) % (CW / 8), kt = e / (32 * (CW / 8));
        const int col = c0 + 8 * nt + (l >> 2);
        const int i = 4 * kt + (l & 3);
        C.Cs[kt][nt][l] = (col < M && i < rc && !fresh) ? -Cg[(int64_t)i * M + col] : 0.0;
      }
      auto prefetch = [&](int64_t pan, int s) {
        if (pan < npan) {
          const int64_t t0 = pan * TT;
          constexpr int CH = 16 / (int)sizeof(TI);  // values per 16-byte chunk (m % 4 == 0)
          for (int e = tid; e < TT * (CW / CH); e += NT) {
            const int t = e / (CW / CH), jc = (e % (CW / CH)) * CH;
            const bool ok = t0 + t < T && c0 + jc < M;
            blk::cp_async16(&C.At[s][t][jc], ok ? Rb + (t0 + t) * M + c0 + jc : Rb, ok ? 16 : 0);
          }
          for (int e = tid; e < TT * 8; e += NT) {
            const int t = e >> 3, cc = e & 7;
            const bool ok = t0 + t < T && cc < k;
            blk::cp_async_one<TI>(&C.Yv[s][t][cc], ok ? Yb + (t0 + t) * k + cc : Yb, ok);
          }
        }
        blk::cp_commit();
      };
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
          const int j = (int)(proj & 1u);
          // ---- P1: G partial of my columns (M = t, N = i, K = my columns) ------------
          {
            const int mt = w % MT, n0 = w / MT;
            double acc[NJ1][2];
            bool on[NJ1];
#pragma unroll
            for (int jj = 0; jj < NJ1; ++jj) {
              const int nt = n0 + NG * jj;
              acc[jj][0] = acc[jj][1] = 0.0;
              on[jj] = nt < NXT && (nt >= IT || 8 * nt < r);  // rows of C~ beyond the rank are zero
            }
#pragma unroll
            for (int kt = 0; kt < CW / 4; ++kt) {
              const double a = (double)C.At[s][8 * mt + p][4 * kt + q];
#pragma unroll
              for (int jj = 0; jj < NJ1; ++jj)
                if (on[jj]) mma(acc[jj], a, C.Ds[n0 + NG * jj][kt][lane]);
            }
#pragma unroll
            for (int jj = 0; jj < NJ1; ++jj) {
              const int nt = n0 + NG * jj;
              if (nt < NXT)
                *reinterpret_cast<double2*>(&C.Gp[(8 * mt + p) * GX + 8 * nt + 2 * q]) =
                    make_double2(acc[jj][0], acc[jj][1]);
            }
          }
          PROBE(0);
          colsync();
          PROBE(1);
          // ---- P2: G = sum of the partials: my chunk, into every column CTA and home --
          if (proj >= 2) mbar_wait(&S.slot_free[j], ((proj >> 1) - 1) & 1u);  // home done with slot j
          {
            constexpr int NE = TT * GX;
            const int chunk = (NE + ncol - 1) / ncol;
            const int e0 = c * chunk, e1 = (e0 + chunk < NE) ? e0 + chunk : NE;
            double(*hg)[HGS] = rem(ncol)->u.home.slotG[j];
            for (int e = e0 + tid; e < e1; e += NT) {
              // every remote load in flight before the fixed-order sum
              double pv[MAXCL];
#pragma unroll
              for (int u = 0; u < MAXCL; ++u) pv[u] = (u < ncol) ? rem(u)->u.col.Gp[e] : 0.0;
              double v = 0.0;
#pragma unroll
              for (int u = 0; u < MAXCL; ++u)
                if (u < ncol) v += pv[u];
              const int t = e / GX, i = e % GX;
              for (int u = 0; u < ncol; ++u) rem(u)->u.col.Gs[t][i] = v;
              hg[t][i] = v;
            }
          }
          PROBE(2);
          colsync();
          PROBE(3);
          // ---- P3: R = A - G C on my columns (M = t, N = my columns, K = i) -----------
          {
            const int kmax = (r + 3) >> 2;
            const int mt = w % MT, n0 = w / MT;
            double acc[NJ3][2];
#pragma unroll
            for (int jj = 0; jj < NJ3; ++jj) {
              const int nt = n0 + NG * jj;
              acc[jj][0] = nt < CW / 8 ? (double)C.At[s][8 * mt + p][8 * nt + 2 * q] : 0.0;
              acc[jj][1] = nt < CW / 8 ? (double)C.At[s][8 * mt + p][8 * nt + 2 * q + 1] : 0.0;
            }
            for (int kt = 0; kt < kmax; ++kt) {
              const double a = C.Gs[8 * mt + p][4 * kt + q];
#pragma unroll
              for (int jj = 0; jj < NJ3; ++jj)
                if (n0 + NG * jj < CW / 8) mma(acc[jj], a, C.Cs[kt][n0 + NG * jj][lane]);
            }
#pragma unroll
            for (int jj = 0; jj < NJ3; ++jj) {
              const int nt = n0 + NG * jj;
              if (nt < CW / 8)
                *reinterpret_cast<double2*>(&C.Rs[8 * mt + p][8 * nt + 2 * q]) = make_double2(acc[jj][0], acc[jj][1]);
            }
          }
          __syncthreads();
          {  // |R_t|^2 and |a_t|^2 of my columns -> every column CTA's nrm[c] and home's slot
            const int t = tid / TPR, part = tid % TPR;
            double rs2 = 0.0, as2 = 0.0;
#pragma unroll
            for (int jc = part; jc < CW; jc += TPR) {
              const double rv = C.Rs[t][jc], av = (double)C.At[s][t][jc];
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
              if (u < ncol) {
                SM* d = rem(u);
                d->u.col.nrm[c][0][t] = rs2;
                d->u.col.nrm[c][1][t] = as2;
              } else if (u == ncol) {
                SM* d = rem(ncol);
                d->u.home.slotN[j][c][0][t] = rs2;
                d->u.home.slotN[j][c][1][t] = as2;
              }
            }
          }
          PROBE(4);
          colsync();
          if (tid == 0) mbar_arrive_at(&S.slot_full[j], (unsigned)ncol);  // my part of slot j is in
          PROBE(5);
          // ---- P4: the rank test (identical in every CTA, home included) --------------
          if (w == 0) {
            double rsq = 0.0, asq = 0.0;
            bool ybad = false;
            if (lane < TT) {
              for (int u = 0; u < ncol; ++u) {
                rsq += C.nrm[u][0][lane];
                asq += C.nrm[u][1][lane];
              }
              for (int cc = 0; cc < k; ++cc) ybad |= !isfinite((double)C.Yv[s][lane][cc]);
              C.scal[lane] = rsq;
            }
            const bool valid = lane >= row_start && lane < tv;
            const bool dep = is_dependent<double>(rsq, asq, eps_sq<double>(cfg, r));
            const bool bad = !isfinite(asq) || ybad;
            const unsigned stopm = __ballot_sync(FULL, valid && (!dep || bad));
            const unsigned badm = __ballot_sync(FULL, valid && bad);
            if (lane == 0) {
              C.flags[0] = stopm ? __ffs(stopm) - 1 : tv;
              C.flags[1] = (int)badm;
            }
          }
          __syncthreads();
          const int tstar = C.flags[0];
          const unsigned badm = (unsigned)C.flags[1];
          proj += 1;
          PROBE(6);
          if (tstar >= tv) break;
          if (((badm >> tstar) & 1u) || r >= rc) {
            status |= ((badm >> tstar) & 1u) ? RGB_ST_NONFINITE : RGB_ST_RANK_CAP;
            stopped = true;
            consumed = t0 + tstar;
            break;
          }
          // ---- independent row tstar: grow C~ and C on my columns (solver.py:368-397) --
          const int ts = tstar;
          const double rsq = C.scal[ts];
          if (GEN || cfg.variant == RGB_GENERAL) {
            const double rinv = 1.0 / rsq;  // K = rej / |rej|^2 (one rounding more than a division)
            for (int e = tid; e < IT * (CW / 4) * 32; e += NT) {
              const int l = e & 31, kt = (e >> 5) % (CW / 4), nt = e / (32 * (CW / 4));
              const int i = 8 * nt + (l >> 2), jl = 4 * kt + (l & 3);
              if (i > r) continue;
              const double K = C.Rs[ts][jl] * rinv;
              C.Ds[nt][kt][l] = (i == r) ? K : fma(-C.Gs[ts][i], K, C.Ds[nt][kt][l]);
            }
            for (int e = tid; e < CW; e += NT) {
              const int kt = r >> 2, nt = e >> 3, l = 4 * (e & 7) + (r & 3);
              C.Cs[kt][nt][l] = -(double)C.At[s][ts][e];
            }
          } else {
            const double resc = (cfg.variant == RGB_ORTHONORMAL) ? 1.0 / sqrt(rsq) : cfg.alpha;
            const double alpha = 1.0 / (1.0 / resc);
            const double sc = alpha * rsq;
            for (int e = tid; e < CW; e += NT) {
              const double rj = C.Rs[ts][e];
              const int kt = e >> 2, l = 4 * (r & 7) + (e & 3);
              C.Ds[r >> 3][kt][l] = (cfg.variant == RGB_ORTHONORMAL) ? alpha * rj : rj / sc;
              C.Cs[r >> 2][e >> 3][4 * (e & 7) + (r & 3)] = -(alpha * rj);
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
      // ---- write back C~, C of my columns; then x = x0 + C~^T W with W from home ----
      for (int e = tid; e < IT * (CW / 4) * 32; e += NT) {
        const int l = e & 31, kt = (e >> 5) % (CW / 4), nt = e / (32 * (CW / 4));
        const int col = c0 + 4 * kt + (l & 3);
        const int i = 8 * nt + (l >> 2);
        if (col < M && i < rc) Dg[(int64_t)i * M + col] = C.Ds[nt][kt][l];
      }
      for (int e = tid; e < (R / 4) * (CW / 8) * 32; e += NT) {
        const int l = e & 31, nt = (e >> 5) % (CW / 8), kt = e / (32 * (CW / 8));
        const int col = c0 + 8 * nt + (l >> 2);
        const int i = 4 * kt + (l & 3);
        if (col < M && i < rc) Cg[(int64_t)i * M + col] = -C.Cs[kt][nt][l];
      }
      cluster_sync_all();  // home has folded every projection: W is final
      redo = defer && rem(ncol)->u.home.flags[2] != 0;  // (the same value in every CTA)
      if (!redo) {
        SM* h = rem(ncol);
        for (int e = tid; e < R * 8; e += NT) C.Wl[e >> 3][e & 7] = h->u.home.Wb[e >> 3][e & 7];
        __syncthreads();
        for (int e = tid; e < k * CW; e += NT) {
          const int cc = e / CW, jl = e % CW;
          double x = C.Ds[NXT - 1][jl >> 2][4 * cc + (jl & 3)];  // x0^T row cc (last N tile of Ds)
          for (int i = 0; i < r; ++i) x = fma(C.Ds[i >> 3][jl >> 2][4 * (i & 7) + (jl & 3)], C.Wl[i][cc], x);
          if (c0 + jl < M) Xg[(int64_t)cc * M + c0 + jl] = x;
        }
      }
      if (!redo && c == 0 && tid == 0) {
        st.rank[b] = r;
        st.nobs[b] = nobs0 + consumed;
        st.status[b] = status;
      }
      cluster_sync_all();  // the next stream reuses every buffer
    } else {
      // ======================= home CTA: P^-1 and W ===================================
      auto& H = S.u.home;
      for (int e = tid; e < R * R; e += NT) {
        const int i = e / R, i2 = e % R;
        H.Ps[i][i2] = (i < rc && i2 < rc && !fresh) ? Pg[(int64_t)i * rc + i2] : 0.0;
      }
      for (int e = tid; e < R * 8; e += NT) H.Wb[e >> 3][e & 7] = 0.0;
      auto prefetch = [&](int64_t pan, int s) {
        if (pan < npan) {
          const int64_t t0 = pan * TT;
          for (int e = tid; e < TT * 8; e += NT) {
            const int t = e >> 3, cc = e & 7;
            const bool ok = t0 + t < T && cc < k;
            blk::cp_async_one<TI>(&H.Yv[s][t][cc], ok ? Yb + (t0 + t) * k + cc : Yb, ok);
          }
        }
        blk::cp_commit();
      };
      // blocked Sherman-Morrison over dependent rows [rs, te) of the 8-row block at
      // panel row base (M = I + G P G^T = L D L^T, E = L^-1; Y = P G^T E^T;
      // P -= Y D^-1 Y^T; W += Y D^-1 E dy0, dy0 = y - a.x0 - G W)
      unsigned nblk = 0;  // dependent blocks folded (selects the U buffer)
      auto dep_log = [&](const double (*Gs)[HGS], int base, int rs, int te, int64_t t0) {
        if (tid < 8 && base + tid >= rs && base + tid < te) {  // logs of the dependent rows
          const int64_t row = b * T + t0 + base + tid;
          if (blog) blog[row] = 0;
          if (clog)
            for (int i = 0; i < rc; ++i) clog[row * rc + i] = Gs[base + tid][i];
        }
      };
      // deferred fold of rows [rs, te) of the block at panel row base: warp w owns rows
      // 8w..8w+7 of Q (in Ps) and of B^T dy (in Wb); A = G^T (M = i, K = t), B = G (K = t,
      // N = i') or dy (N = cc), both straight from the slot; no barrier
      auto dep_block_deferred = [&](int s, const double (*Gs)[HGS], int base, int rs, int te, int64_t t0) {
        if (8 * w < r) {
          double a[2];
#pragma unroll
          for (int kt = 0; kt < 2; ++kt) {
            const int t = base + 4 * kt + q;
            a[kt] = (t >= rs && t < te) ? Gs[t][8 * w + p] : 0.0;
          }
#pragma unroll
          for (int nt = 0; nt < IT; ++nt) {
            if (8 * nt < r) {
              const double2 v = *reinterpret_cast<const double2*>(&H.Ps[8 * w + p][8 * nt + 2 * q]);
              double acc[2] = {v.x, v.y};
#pragma unroll
              for (int kt = 0; kt < 2; ++kt) {
                const int t = base + 4 * kt + q;
                mma(acc, a[kt], (t >= rs && t < te) ? Gs[t][8 * nt + p] : 0.0);
              }
              *reinterpret_cast<double2*>(&H.Ps[8 * w + p][8 * nt + 2 * q]) = make_double2(acc[0], acc[1]);
            }
          }
          double wb[2] = {H.Wb[8 * w + p][2 * q], H.Wb[8 * w + p][2 * q + 1]};
#pragma unroll
          for (int kt = 0; kt < 2; ++kt) {
            const int t = base + 4 * kt + q;
            const double dy = (t >= rs && t < te) ? (double)H.Yv[s][t][p] - Gs[t][R + p] : 0.0;
            mma(wb, a[kt], dy);
          }
          H.Wb[8 * w + p][2 * q] = wb[0];
          H.Wb[8 * w + p][2 * q + 1] = wb[1];
        }
        dep_log(Gs, base, rs, te, t0);
      };
      auto dep_block = [&](int s, const double (*Gs)[HGS], int base, int rs, int te, int64_t t0) {
        if (defer) {
          dep_block_deferred(s, Gs, base, rs, te, t0);
          return;
        }
        const int ub = (int)(nblk++ & 1u);
        const int kr = (r + 3) >> 2;  // K steps over the rank (rows beyond it are zero)
        const bool in_t = base + p >= rs && base + p < te;
        {  // U = P G^T (M = i, N = t, K = i'): warp w owns rows 8w..8w+7
          double acc[4][2] = {};
          if (8 * w < r) {
            double a[IK], g[IK];
#pragma unroll
            for (int kt = 0; kt < IK; ++kt) {
              a[kt] = kt < kr ? H.Ps[8 * w + p][4 * kt + q] : 0.0;
              g[kt] = (kt < kr && in_t) ? Gs[base + p][4 * kt + q] : 0.0;
            }
#pragma unroll
            for (int kt = 0; kt < IK; ++kt)
              if (kt < kr) mma(acc[kt & 3], a[kt], g[kt]);
          }
          H.Ub[ub][8 * w + p][2 * q] = (acc[0][0] + acc[1][0]) + (acc[2][0] + acc[3][0]);
          H.Ub[ub][8 * w + p][2 * q + 1] = (acc[0][1] + acc[1][1]) + (acc[2][1] + acc[3][1]);
          __syncwarp();
          // this warp's share of S = G U and G W: K = its own rows i = 8w..8w+7
          double sp[2] = {0.0, 0.0}, gp[2] = {0.0, 0.0};
          if (8 * w < r) {
#pragma unroll
            for (int kt = 0; kt < 2; ++kt) {
              const double a0 = in_t ? Gs[base + p][8 * w + 4 * kt + q] : 0.0;
              mma(sp, a0, H.Ub[ub][8 * w + 4 * kt + q][p]);
              mma(gp, a0, H.Wb[8 * w + 4 * kt + q][p]);
            }
          }
          H.Sp[w][lane][0] = sp[0];
          H.Sp[w][lane][1] = sp[1];
          H.Sp[w][lane][2] = gp[0];
          H.Sp[w][lane][3] = gp[1];
        }
        __syncthreads();
        PROBE(10);
        if (w == 0) {
          double mi[2] = {0.0, 0.0}, gws[2] = {0.0, 0.0};
#pragma unroll
          for (int u = 0; u < NW; ++u) {  // fixed order
            const double2 v = *reinterpret_cast<const double2*>(&H.Sp[u][lane][0]);
            const double2 g = *reinterpret_cast<const double2*>(&H.Sp[u][lane][2]);
            mi[0] += v.x;
            mi[1] += v.y;
            gws[0] += g.x;
            gws[1] += g.y;
          }
          if (p == 2 * q) mi[0] += 1.0;
          if (p == 2 * q + 1) mi[1] += 1.0;
#pragma unroll
          for (int e = 0; e < 2; ++e)  // dy0[t = p][cc = 2q + e]
            H.Dy[p][2 * q + e] = in_t ? (double)H.Yv[s][base + p][2 * q + e] - Gs[base + p][R + 2 * q + e] - gws[e] : 0.0;
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
          H.Eb[p][2 * q] = ev[0];
          H.Eb[p][2 * q + 1] = ev[1];
          if ((p >> 1) == q) H.rd[p] = rcp64((p & 1) ? mi[1] : mi[0]);
          __syncwarp();
          double dh[2] = {0.0, 0.0};  // dh = E dy0 / d (M = t, N = cc, K = t')
#pragma unroll
          for (int kt = 0; kt < 2; ++kt) mma(dh, H.Eb[p][4 * kt + q], H.Dy[4 * kt + q][p]);
          __syncwarp();
          H.Dy[p][2 * q] = dh[0] * H.rd[p];
          H.Dy[p][2 * q + 1] = dh[1] * H.rd[p];
        }
        __syncthreads();
        PROBE(11);
        // Y = U E^T: every warp forms all the Y rows its P update needs, directly in
        // the B-operand layout (the N index of the MMA permuted, n -> t = (n >> 1) +
        // 4 (n & 1)), so Y needs no exchange through shared memory and no barrier;
        // then W += Y (D^-1 E dy0) and P -= Y D^-1 Y^T on the own row block
        if (8 * w < r) {
          const int pe = (p >> 1) + 4 * (p & 1);
          double ya[IT][2], yo[2] = {0.0, 0.0};
#pragma unroll
          for (int nt = 0; nt < IT; ++nt) {
            ya[nt][0] = ya[nt][1] = 0.0;
            if (8 * nt < r) {
#pragma unroll
              for (int kt = 0; kt < 2; ++kt) mma(ya[nt], H.Ub[ub][8 * nt + p][4 * kt + q], H.Eb[pe][4 * kt + q]);
            }
          }
#pragma unroll
          for (int kt = 0; kt < 2; ++kt) mma(yo, H.Ub[ub][8 * w + p][4 * kt + q], H.Eb[pe][4 * kt + q]);
          // yo[e] = Y[8w + p][q + 4e]: W's own rows (M = i, N = cc, K = t)
          double wb[2] = {H.Wb[8 * w + p][2 * q], H.Wb[8 * w + p][2 * q + 1]};
#pragma unroll
          for (int kt = 0; kt < 2; ++kt) mma(wb, yo[kt], H.Dy[4 * kt + q][p]);
          H.Wb[8 * w + p][2 * q] = wb[0];
          H.Wb[8 * w + p][2 * q + 1] = wb[1];
          // P -= Y D^-1 Y^T (M = i, N = i', K = t): warp w owns row block w
          const double ys0 = -yo[0] * H.rd[q], ys1 = -yo[1] * H.rd[4 + q];
          double acc[IT][2];
#pragma unroll
          for (int nt = 0; nt < IT; ++nt) {
            const double2 v = *reinterpret_cast<const double2*>(&H.Ps[8 * w + p][8 * nt + 2 * q]);
            acc[nt][0] = v.x;
            acc[nt][1] = v.y;
          }
#pragma unroll
          for (int nt = 0; nt < IT; ++nt) {
            if (8 * nt < r) {
              mma(acc[nt], ys0, ya[nt][0]);
              mma(acc[nt], ys1, ya[nt][1]);
            }
          }
#pragma unroll
          for (int nt = 0; nt < IT; ++nt)
            if (8 * nt < r)
              *reinterpret_cast<double2*>(&H.Ps[8 * w + p][8 * nt + 2 * q]) = make_double2(acc[nt][0], acc[nt][1]);
        }
        PROBE(12);
        dep_log(Gs, base, rs, te, t0);
        // no barrier: the next block reads only its own rows of P^-1 and W, writes
        // the other U buffer, and its first barrier orders the rest
        PROBE(13);
      };

      prefetch(0, 0);
      for (int64_t pan = 0; pan < npan && !stopped; ++pan) {
        const int s = (int)(pan & 1);
        const int64_t t0 = pan * TT;
        const int tv = (int)((T - t0) < TT ? (T - t0) : TT);
        prefetch(pan + 1, s ^ 1);
        blk::cp_wait<1>();
        __syncthreads();
        int row_start = 0;
        while (true) {
          const int j = (int)(proj & 1u);
          mbar_wait(&S.slot_full[j], (proj >> 1) & 1u);  // G and the norms of this projection
          PROBE(14);
          const double(*Gs)[HGS] = H.slotG[j];
          if (w == 0) {  // the rank test, exactly as the column CTAs compute it
            double rsq = 0.0, asq = 0.0;
            bool ybad = false;
            if (lane < TT) {
              for (int u = 0; u < ncol; ++u) {
                rsq += H.slotN[j][u][0][lane];
                asq += H.slotN[j][u][1][lane];
              }
              for (int cc = 0; cc < k; ++cc) ybad |= !isfinite((double)H.Yv[s][lane][cc]);
              H.zg[lane] = rsq;
            }
            const bool valid = lane >= row_start && lane < tv;
            const bool dep = is_dependent<double>(rsq, asq, eps_sq<double>(cfg, r));
            const bool bad = !isfinite(asq) || ybad;
            const unsigned stopm = __ballot_sync(FULL, valid && (!dep || bad));
            const unsigned badm = __ballot_sync(FULL, valid && bad);
            if (lane == 0) {
              H.flags[0] = stopm ? __ffs(stopm) - 1 : tv;
              H.flags[1] = (int)badm;
            }
          }
          __syncthreads();
          const int tstar = H.flags[0];
          const unsigned badm = (unsigned)H.flags[1];
          const double rsq_ts = tstar < tv ? H.zg[tstar] : 0.0;
          __syncthreads();
          for (int base = (row_start & ~7); base < tstar; base += 8) dep_block(s, Gs, base, row_start, tstar, t0);
          __syncthreads();  // every warp's P^-1 / W rows are folded (growth below writes across blocks)
          bool done = tstar >= tv;
          if (!done && (((badm >> tstar) & 1u) || r >= rc)) {
            status |= ((badm >> tstar) & 1u) ? RGB_ST_NONFINITE : RGB_ST_RANK_CAP;
            stopped = true;
            consumed = t0 + tstar;
            done = true;
          }
          if (!done) {
            // growth of P^-1 and W for the independent row tstar (solver.py:368-397)
            const int ts = tstar;
            if (GEN || cfg.variant == RGB_GENERAL) {
              for (int i = tid; i < R; i += NT) {  // P = diag(P, 1)
                H.Ps[r][i] = (i == r) ? 1.0 : 0.0;
                H.Ps[i][r] = (i == r) ? 1.0 : 0.0;
              }
              if (tid < 8) H.Wb[r][tid] = tid < k ? (double)H.Yv[s][ts][tid] - Gs[ts][R + tid] : 0.0;
              if (tid == 0) {
                const int64_t row = b * T + t0 + ts;
                if (blog) blog[row] = 1;
                if (clog)
                  for (int i = 0; i < rc; ++i) clog[row * rc + i] = (i == r) ? 1.0 : 0.0;
              }
            } else {
              const double resc = (cfg.variant == RGB_ORTHONORMAL) ? 1.0 / sqrt(rsq_ts) : cfg.alpha;
              const double last = 1.0 / resc;
              const double alpha = 1.0 / last;
              if (tid < R) {  // z_i = (P gamma)_i
                double z = 0.0;
                for (int i2 = 0; i2 < R; ++i2) z = fma(H.Ps[tid][i2], Gs[ts][i2], z);
                H.zg[tid] = z;
              } else if (tid < R + 8) {  // (gamma^T W)_c
                const int cc = tid - R;
                double g = 0.0;
                for (int i = 0; i < R; ++i) g = fma(Gs[ts][i], H.Wb[i][cc], g);
                H.zg[tid] = g;
              }
              __syncthreads();
              double dn = 0.0;
              for (int i = 0; i < R; ++i) dn = fma(Gs[ts][i], H.zg[i], dn);
              const double denom = 1.0 + dn;
              for (int i = tid; i < R; i += NT) {
                const double edge = (i < r) ? -(alpha * H.zg[i]) : 0.0;
                H.Ps[i][r] = (i == r) ? alpha * alpha * denom : edge;
                if (i != r) H.Ps[r][i] = edge;
              }
              if (tid < 8)
                H.Wb[r][tid] = tid < k ? alpha * (((double)H.Yv[s][ts][tid] - Gs[ts][R + tid]) - H.zg[R + tid]) : 0.0;
              if (tid == 0) {
                const int64_t row = b * T + t0 + ts;
                if (blog) blog[row] = 1;
                if (clog)
                  for (int i = 0; i < rc; ++i) clog[row * rc + i] = i < r ? Gs[ts][i] : (i == r ? last : 0.0);
              }
            }
          }
          // release the slot to the column CTAs
          __syncthreads();
          if (tid < ncol) mbar_arrive_at(&S.slot_free[j], (unsigned)tid);
          proj += 1;
          if (done) break;
          r += 1;
          row_start = tstar + 1;
          if (row_start >= tv) break;
        }
        if (!stopped) consumed = t0 + tv;
      }
      blk::cp_wait<0>();
      __syncthreads();
      if (defer) {
        // P^-1 = Q^-1 in place (Gauss-Jordan, Q is SPD with pivots >= 1: no pivoting; the
        // pivot row and column of a step go through the U buffers), the certificate
        // kappa_F(Q) = |Q|_F |Q^-1|_F <= 1e6, then W = P^-1 (B^T dy)
        double* rowk = &H.Ub[0][0][0];
        double* colk = rowk + R;
        double* red = colk + R;  // [2][NW]
        double fq = 0.0, fp = 0.0;
        for (int e = tid; e < r * r; e += NT) {
          const double v = H.Ps[e / r][e % r];
          fq = fma(v, v, fq);
        }
#pragma unroll 1
        for (int kk = 0; kk < r; ++kk) {
          if (tid < r) {
            rowk[tid] = H.Ps[kk][tid];
            colk[tid] = H.Ps[tid][kk];
          }
          __syncthreads();
          const double pv = blk::rcp64(rowk[kk]);
          for (int e = tid; e < r * r; e += NT) {
            const int i = e / r, j = e % r;
            const double f = colk[i] * pv, rv = rowk[j];
            double v = fma(-f, rv, H.Ps[i][j]);
            if (i == kk) v = rv * pv;
            if (j == kk) v = (i == kk) ? pv : -f;
            H.Ps[i][j] = v;
          }
          __syncthreads();
        }
        for (int e = tid; e < r * r; e += NT) {
          const double v = H.Ps[e / r][e % r];
          fp = fma(v, v, fp);
        }
        fq = warp_sum(fq);
        fp = warp_sum(fp);
        if (lane == 0) {
          red[w] = fq;
          red[NW + w] = fp;
        }
        __syncthreads();
        double kq = 0.0, kp = 0.0;
        for (int u = 0; u < NW; ++u) {
          kq += red[u];
          kp += red[NW + u];
        }
        const bool bad = !(kq * kp <= 1e12);  // (a NaN fails too)
        if (tid == 0) H.flags[2] = bad ? 1 : 0;
        redo = bad;
        if (!bad) {
          double wv = 0.0;
          const int i = tid >> 3, cc = tid & 7;  // NT = 8 R at most: one (i, cc) per thread and pass
          for (int i0 = 0; i0 < R; i0 += NT / 8) {
            wv = 0.0;
            if (i0 + i < r)
              for (int j = 0; j < r; ++j) wv = fma(H.Ps[i0 + i][j], H.Wb[j][cc], wv);
            rowk[(i0 + i) * 8 + cc] = wv;  // (R * 8 doubles: the U buffers hold 2 R * 8)
          }
          __syncthreads();
          for (int e = tid; e < R * 8; e += NT) H.Wb[e >> 3][e & 7] = (e >> 3) < r ? rowk[e] : 0.0;
          __syncthreads();
        }
      } else if (tid == 0) {
        H.flags[2] = 0;
      }
      if (!redo)
        for (int e = tid; e < rc * rc; e += NT) Pg[e] = H.Ps[e / rc][e % rc];
      cluster_sync_all();  // W final for the column CTAs
      cluster_sync_all();  // they have read it
    }
    if (redo) b -= ncid;  // nothing of the state's rank / counters / x is written: the same stream again
  }
}

}  // namespace cls

template <int R, int TT, int CW, typename TI>
static int launch_cluster_t(const rgb_config& cfg, rgb_state& st, const void* rows, int64_t rows_stride,
                            const void* targets, int64_t tg_stride, int64_t T, const rgb_logs& logs,
                            cudaStream_t stream) {
  const int ncl = (cfg.m + CW - 1) / CW + 1;  // column CTAs + home
  const bool gen = cfg.variant == RGB_GENERAL;
  auto kern = gen ? cls::cluster_kernel<R, TT, CW, true, TI> : cls::cluster_kernel<R, TT, CW, false, TI>;
  const size_t smem = sizeof(cls::Smem<R, TT, CW, TI>);
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
  if ((int64_t)nclusters > cfg.num_streams) nclusters = (int)cfg.num_streams;
  lc.gridDim = dim3((unsigned)(ncl * nclusters));
  const TI* rp = (const TI*)rows;
  const TI* tp = (const TI*)targets;
  // RGB_CLUSTER_SEQ=1: the sequential Sherman-Morrison chain for every stream (A/B runs, tests)
  const char* seq_env = getenv("RGB_CLUSTER_SEQ");
  const int seq_only = (seq_env && seq_env[0] && seq_env[0] != '0') ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&lc, kern, cfg, st, rp, rows_stride, tp, tg_stride, T, logs.branch,
                                     (double*)logs.coords, seq_only);
  return e == cudaSuccess ? RGB_OK : RGB_E_CUDA;
}

// r_cap 16..64 (rows past r_cap masked) and m up to 15 x 72 = 1 080 (a
// multiple of 4): 15 column CTAs at most
bool cluster_supports(const rgb_config& cfg) {
  const bool var_ok = cfg.variant == RGB_GENERAL || cfg.variant == RGB_ORTHONORMAL ||
                      (cfg.variant == RGB_ORTHOGONAL && cfg.alpha != 0.0);
  if (cfg.dtype != RGB_F64 || !var_ok || cfg.k < 1 || cfg.k > 8) return false;
  return cfg.r_cap >= 16 && cfg.r_cap <= 64 && cfg.m % 4 == 0 && cfg.m >= 128 &&
         cfg.m <= (cls::MAXCL - 1) * 72;
}

int launch_cluster(const rgb_config& cfg, rgb_state& st, const void* rows, int64_t rows_stride, const void* targets,
                   int64_t tg_stride, int64_t T, const rgb_logs& logs, cudaStream_t stream, int num_sms,
                   bool f32in) {
  (void)num_sms;
  if (logs.resid || logs.gain) return RGB_E_UNSUPPORTED;
  if (!cluster_supports(cfg)) return RGB_E_UNSUPPORTED;
  if (cfg.m <= (cls::MAXCL - 1) * 64)
    return f32in ? launch_cluster_t<64, 32, 64, float>(cfg, st, rows, rows_stride, targets, tg_stride, T, logs, stream)
                 : launch_cluster_t<64, 32, 64, double>(cfg, st, rows, rows_stride, targets, tg_stride, T, logs, stream);
  return f32in ? launch_cluster_t<64, 32, 72, float>(cfg, st, rows, rows_stride, targets, tg_stride, T, logs, stream)
               : launch_cluster_t<64, 32, 72, double>(cfg, st, rows, rows_stride, targets, tg_stride, T, logs, stream);
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
