// rgb_grid.cu -- one large stream on the whole GPU (sm_100a, fp64 tensor cores).
//
// For a few single streams whose factors are too large for one SM (config 4:
// m 2048, r 512; any m <= 2 368 with r_cap <= 512, columns past m and factor
// rows past r_cap masked; config 2 runs on rgb_cluster.cu) the same 8-row tile algebra as
// rgb_blocked.cu runs on NC cooperative CTAs (one per SM) separated by grid
// barriers:
//
//   CTA c owns columns [c*CW, (c+1)*CW) of C~ and C (shared memory, MMA
//   fragment order) and, for c < R/8, the 8-row block c of P^-1 and of W.
//
//   P1  G_c = A[:, cols] C~[:, cols]^T (+ a.x0 as 8 extra rows of C~)  -> ws
//   P2  G   = sum_c G_c (a grid-wide reduction, fixed order)             -> ws
//   P3  R[:, cols] = A - G C[:, cols]; |R_t|^2 partial                   -> ws
//   P4  rank test (every CTA, identical); for the dependent rows of the
//       tile the owners of P compute U_b = P_b G^T and the partials of
//       S = G P G^T and of G W                                           -> ws
//   P5  M = I + S = L D L^T, E = L^-1 (every owner, identical);
//       Y_b = U_b E^T -> ws; W_b += Y_b D^-1 E dy0
//   P6  P_b -= Y_b D^-1 Y^T  (overlaps P1 of the next tile)
//
// three grid barriers per 8 rows (U_b and the S / G W partials of P4 are formed
// in P3 for every row of the tile and masked after the rank test, which leaves
// the values of the masked computation unchanged; P6 waits for the next
// projection's second barrier, its L2 loads beside the reduced G's) instead of
// three-plus per row for a per-row multi-SM scheme -- and two for a tile of
// dependent rows: when a projection ends, the next tile is staged (its rows come
// into registers one tile ahead) and its P1 issued before the rank-test barrier,
// which is then also the next tile's first barrier; a growth in between (the
// basis moved) discards it.  An independent row (solver.py:305-318) is applied by
// every CTA to its own columns / row block, and the rest of its tile is
// re-projected.  The workspace (partials, barrier counter) is allocated per
// call, stream-ordered on the caller's stream, so calls stay reentrant; it
// comes from a library-owned pool per device whose memory is kept between
// calls (the default pool hands it back to the driver at every
// synchronisation, and re-mapping cost 3.8 ms per call at m = 2048).
#include <cooperative_groups.h>

#include <cstdint>
#include <mutex>

#include "rgb_mma.cuh"

namespace rgb {
namespace grd {

using blk::FULL;
using blk::TT;
using blk::mma;
using blk::rcp64;

constexpr int NT = 256;  // threads per CTA (8 warps)
constexpr int NW = NT / 32;

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// phase timing (debug builds only: -DRGB_GRID_PROBE): ns summed per phase for
// CTA 0 and CTA 1, read back with rgb_grid_probe()
#ifdef RGB_GRID_PROBE
__device__ unsigned long long g_gprobe[2][16];
__device__ __forceinline__ unsigned long long ggtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define GPROBE(i)                                              \
  do {                                                         \
    if (threadIdx.x == 0 && blockIdx.x < 2) {                  \
      const unsigned long long now_ = ggtime();                \
      atomicAdd(&g_gprobe[blockIdx.x][i], now_ - probe_t);     \
      probe_t = now_;                                          \
    }                                                          \
  } while (0)
#else
#define GPROBE(i) \
  do {            \
  } while (0)
#endif

// all CTAs of the (cooperative) grid; counter zeroed before the launch
__device__ __forceinline__ void grid_sync(unsigned* ctr, unsigned& epoch) {
  __syncthreads();
  epoch += 1;
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    const unsigned target = epoch * gridDim.x;
    while (ld_acquire(ctr) < target) __nanosleep(20);
  }
  __syncthreads();
}

template <int R, int CW>
struct Ws {  // global workspace layout (doubles), per launch
  static constexpr int GX = R + 8;  // G columns plus 8 for a.x0
  __host__ __device__ static size_t gpart(int nc) { return (size_t)nc * TT * GX; }
  static size_t bytes(int nc) {
    return 256 + sizeof(double) * (gpart(nc) + TT * GX + (size_t)nc * 4 * TT + (size_t)(R / 8) * 2 * 64 +
                                   (size_t)R * TT + (size_t)R * 8 + (size_t)R + (size_t)(R / 8) * 16 +
                                   (size_t)nc * 64);
  }
};

template <int R, int CW>
struct GridSmem {
  static constexpr int IT = R / 8, GX = R + 8, GS = R + 20, PS = R + 4, AS = CW + 4;
  double Ds[(R + 8) / 8][CW / 4][32];  // C~ (and x0^T) of my columns, B-fragment order
  double Cs[R / 4][CW / 8][32];        // -C of my columns, B-fragment order
  double Gs[TT][GS];                   // full G of the tile (+ a.x0)
  double Ps[8][PS];                    // my row block of P^-1
  double Wb[8][8];                     // my row block of W (c = column)
  double At[2][TT][AS];                // the tile's rows, my columns (two tiles: the next
  double Yv[2][TT][8];                 // one is staged for the speculative projection); targets
  double Rs[TT][CW];                   // rejections of my columns
  double red[NW][TT * CW > 128 ? TT * CW : 128];  // per-warp partials
  double Ub[8][8], Eb[8][8], Dy[8][8], Yb[8][8];
  double rd[8];
  double scal[8];
  int flags[8];
};

// GEN: general variant only; !GEN: orthogonal / orthonormal (solver.py:382-395)
template <int R, int CW, bool GEN, typename TI>
__global__ void __launch_bounds__(NT, 1) grid_kernel(rgb_config cfg, rgb_state st, const TI* __restrict__ rows,
                                                     int64_t rstride, const TI* __restrict__ tgts, int64_t tstride,
                                                     int64_t T, uint8_t* __restrict__ blog, double* __restrict__ clog,
                                                     double* __restrict__ ws, unsigned* __restrict__ ctr) {
  constexpr int IT = R / 8, GX = R + 8, NXT = (R + 8) / 8;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  GridSmem<R, CW>& S = *reinterpret_cast<GridSmem<R, CW>*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, p = lane >> 2, q = lane & 3;
  const int nc = gridDim.x, c = blockIdx.x, c0 = c * CW;
  const int M = cfg.m, k = cfg.k;
  const int rc = cfg.r_cap;   // stored rank capacity (<= R): global row stride of the factors
  const bool owner = c < IT;  // owns row block c of P and W
  double* ws_g = ws + 32;                          // [nc][TT][GX]
  double* ws_gf = ws_g + Ws<R, CW>::gpart(nc);     // [TT][GX]
  double* ws_r0 = ws_gf + TT * GX;                 // [2][2][TT][nc]: |R|^2, |a|^2 partials,
                                                   // double-buffered by projection parity
  double* ws_s = ws_r0 + (size_t)nc * 4 * TT;      // [IT][2][64]: S and G W partials
  double* ws_y = ws_s + (size_t)IT * 2 * 64;       // [R][TT]
  double* ws_w = ws_y + (size_t)R * TT;            // [R][8]
  double* ws_z = ws_w + (size_t)R * 8;             // [R]: z = P gamma (non-general growth)
  double* ws_d = ws_z + R;                         // [IT][16]: gamma.z, gamma^T W partials
  double* ws_m = ws_d + (size_t)IT * 16;           // [nc][64]: R R^T partials (block growth)
  unsigned epoch = 0;
#ifdef RGB_GRID_PROBE
  unsigned long long probe_t = ggtime();
  const unsigned long long probe_t0 = probe_t;
#endif
  unsigned nproj = 0;  // projections so far (selects the ws_r buffer)

  for (int64_t b = 0; b < cfg.num_streams; ++b) {
    int status = st.status[b];
    if (status) continue;
    int r = st.rank[b];
    // P_b -= Y_b D^-1 Y^T of the last dependent block, deferred to the next grid
    // barrier (the next projection's P1 barrier, or one of its own before a
    // non-general growth / the write-back): P is next read by the next tile's U_b,
    // and a general growth only resets row / column r, which Y leaves untouched
    bool pending_p6 = false;
    auto apply_p6 = [&]() {
        if (owner) {
          // P_b -= Y_b D^-1 Y^T (M = i in my block, N = i', K = t)
          const double ys0 = -S.Yb[p][q] * S.rd[q], ys1 = -S.Yb[p][4 + q] * S.rd[4 + q];
          const int nlive = (r + 7) >> 3;  // row blocks of Y past the rank are zero
          constexpr int NPW = (IT + NW - 1) / NW;
          double y0[NPW], y1[NPW];  // every L2 load in flight first
#pragma unroll
          for (int i = 0; i < NPW; ++i) {
            const int nt = w + NW * i;
            const bool on = nt < nlive;
            y0[i] = on ? __ldcg(ws_y + (size_t)(8 * nt + p) * TT + q) : 0.0;
            y1[i] = on ? __ldcg(ws_y + (size_t)(8 * nt + p) * TT + 4 + q) : 0.0;
          }
#pragma unroll
          for (int i = 0; i < NPW; ++i) {
            const int nt = w + NW * i;
            if (nt < nlive) {
              double acc[2] = {S.Ps[p][8 * nt + 2 * q], S.Ps[p][8 * nt + 2 * q + 1]};
              mma(acc, ys0, y0[i]);
              mma(acc, ys1, y1[i]);
              S.Ps[p][8 * nt + 2 * q] = acc[0];
              S.Ps[p][8 * nt + 2 * q + 1] = acc[1];
            }
          }
        }
      __syncthreads();
      pending_p6 = false;
    };
    const int64_t nobs0 = st.nobs[b];
    // certified block growth of a fresh stream's leading rows (general variant,
    // x0 = 0): on until the first tile with a row it cannot certify
    bool bulk = (GEN || cfg.variant == RGB_GENERAL) && r == 0 && nobs0 == 0;
    double* Cg = reinterpret_cast<double*>(st.basis) + b * (int64_t)rc * M;
    double* Dg = reinterpret_cast<double*>(st.dual) + b * (int64_t)rc * M;
    double* Pg = reinterpret_cast<double*>(st.gram_inv) + b * (int64_t)rc * rc;
    double* Xg = reinterpret_cast<double*>(st.x) + b * (int64_t)k * M;
    const TI* Rb = rows + b * rstride;
    const TI* Yb = tgts + b * tstride;

    // ---- load my slices: C~ (+ x0^T as rows R..R+7), -C, my P / W blocks ---------
    for (int e = tid; e < NXT * (CW / 4) * 32; e += NT) {
      const int l = e & 31, kt = (e >> 5) % (CW / 4), nt = e / (32 * (CW / 4));
      const int i = 8 * nt + (l >> 2), col = c0 + 4 * kt + (l & 3);
      double v = 0.0;  // rows past the capacity and columns past m are zero
      if (col < M) {
        if (i < rc) v = Dg[(int64_t)i * M + col];
        else if (i >= R && i - R < k) v = Xg[(int64_t)(i - R) * M + col];
      }
      S.Ds[nt][kt][l] = v;
    }
    for (int e = tid; e < (R / 4) * (CW / 8) * 32; e += NT) {
      const int l = e & 31, nt = (e >> 5) % (CW / 8), kt = e / (32 * (CW / 8));
      const int i = 4 * kt + (l & 3), col = c0 + 8 * nt + (l >> 2);
      S.Cs[kt][nt][l] = (i < rc && col < M) ? -Cg[(int64_t)i * M + col] : 0.0;
    }
    if (owner) {
      for (int e = tid; e < 8 * R; e += NT) {
        const int i = 8 * c + e / R, i2 = e % R;
        S.Ps[e / R][i2] = (i < rc && i2 < rc) ? Pg[(int64_t)i * rc + i2] : 0.0;
      }
      for (int e = tid; e < 64; e += NT) S.Wb[e >> 3][e & 7] = 0.0;
    }
    __syncthreads();

    const int64_t ntiles = (T + TT - 1) / TT;
    int64_t consumed = 0;
    bool stopped = false;
    // the next tile's rows of my columns and its targets are loaded into registers
    // one tile ahead (their HBM latency overlaps the current tile's phases)
    constexpr int PA = (TT * CW + NT - 1) / NT;
    double na[PA], ny = 0.0;
    auto load_next = [&](int64_t tile) {
      const int64_t t0 = tile * TT;
#pragma unroll
      for (int i = 0; i < PA; ++i) {
        const int e = tid + NT * i, t = e / CW, j = e % CW;
        na[i] = (e < TT * CW && tile < ntiles && t0 + t < T && c0 + j < M) ? (double)__ldg(Rb + (t0 + t) * M + c0 + j)
                                                                         : 0.0;
      }
      const int t = tid >> 3, cc = tid & 7;
      ny = (tid < 64 && tile < ntiles && t0 + t < T && cc < k) ? (double)__ldg(Yb + (t0 + t) * k + cc) : 0.0;
    };
    // stage the registers (the next tile) into At / Yv buffer s
    auto stage = [&](int s) {
#pragma unroll
      for (int i = 0; i < PA; ++i) {
        const int e = tid + NT * i;
        if (e < TT * CW) S.At[s][e / CW][e % CW] = na[i];
      }
      if (tid < 64) S.Yv[s][tid >> 3][tid & 7] = ny;
    };
    // P1: G partial of my columns for the tile in At buffer s (M = t, N = i, K = my
    // columns) -> ws_g, and its |a_t|^2 partials -> ws_rp (N tiles past the rank are
    // zero: skipped here, zeroed by the reducers)
    auto p1 = [&](int s, double* ws_rp) {
      const int nlive = (r + 7) >> 3;
      for (int n0 = w; n0 < NXT; n0 += 4 * NW) {
        double acc[4][2] = {};
        bool on[4];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int nt = n0 + NW * jj;
          on[jj] = nt < NXT && (nt >= IT || nt < nlive);
        }
#pragma unroll
        for (int kt = 0; kt < CW / 4; ++kt) {
          const double a = S.At[s][p][4 * kt + q];
#pragma unroll
          for (int jj = 0; jj < 4; ++jj)
            if (on[jj]) mma(acc[jj], a, S.Ds[n0 + NW * jj][kt][lane]);
        }
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
          if (on[jj])
            *reinterpret_cast<double2*>(ws_g + ((size_t)c * TT + p) * GX + 8 * (n0 + NW * jj) + 2 * q) =
                make_double2(acc[jj][0], acc[jj][1]);
      }
      if (tid < TT) {  // |a_t|^2 of my columns
        double sa = 0.0;
        for (int j = 0; j < CW; ++j) sa = fma(S.At[s][tid][j], S.At[s][tid][j], sa);
        ws_rp[((size_t)1 * TT + tid) * nc + c] = sa;
      }
    };
    // speculation: when the projection of a tile ends, the next tile is staged and
    // its P1 issued before the rank-test barrier (C~ does not change unless the
    // test finds an independent row); the next tile then starts at its second
    // barrier -- two grid barriers per dependent tile instead of three
    int cur = 0;
    bool staged = false, spec_valid = false;
    load_next(0);
    for (int64_t tile = 0; tile < ntiles && !stopped; ++tile) {
      const int64_t t0 = tile * TT;
      const int tv = (int)((T - t0) < TT ? (T - t0) : TT);
#ifdef RGB_GRID_PROBE
      // elapsed time until the stream's rank first reaches its final value's tile
      if (threadIdx.x == 0 && blockIdx.x < 2 && tile == (int64_t)(R / 8)) g_gprobe[blockIdx.x][12] = ggtime() - probe_t0;
#endif
      // tile rows of my columns and the targets (loaded one tile ahead); a tile
      // staged already by the previous tile's speculative projection is used as
      // it is, and its projection too when no growth came in between
      bool skip_p1 = false;
      if (staged) {
        cur ^= 1;
        staged = false;
        skip_p1 = spec_valid;
      } else {
        stage(cur);
        load_next(tile + 1);
        __syncthreads();
      }
      spec_valid = false;
      int row_start = 0;
      while (true) {
        // a tile whose rows are all independent runs no barrier between the
        // test's reads of ws_r and the next projection's writes: alternate buffers
        double* ws_r = ws_r0 + (size_t)(nproj++ & 1u) * nc * 2 * TT;
        const bool bulk_try = bulk && row_start == 0 && tv == TT && r + TT <= rc;
        const int nlive = (r + 7) >> 3;
        if (!skip_p1) {  // (else issued by the previous tile's speculation)
          p1(cur, ws_r);
          GPROBE(0);
          grid_sync(ctr, epoch);
          GPROBE(1);
        }
        skip_p1 = false;
        // ---- P2: G = sum of the partials.  CTA c reduces a contiguous chunk of
        // elements: warp w reads partials u = w, w+8, ... (coalesced rows of
        // 32 elements), then the 8 warp sums are added in a fixed order.
        {
          constexpr int NE = TT * GX;
          const int chunk = (NE + nc - 1) / nc;
          const int e0 = c * chunk, e1 = (e0 + chunk < NE) ? e0 + chunk : NE;
          constexpr int MAXU = (148 + NW - 1) / NW;  // partials per warp (one CTA per SM)
          // two elements per lane per round: a chunk of up to 64 elements (nc >= 66) is
          // one round of loads, all in flight before the (fixed-order) sums
          for (int eb = e0; eb < e1; eb += 64) {
            double v[2][MAXU];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int e = eb + 32 * h + lane;
              const int col = e % GX;  // G column: coordinate i < R, or R + c for a.x0
              const bool live = e < e1 && (col >= R || col < 8 * nlive);
#pragma unroll
              for (int i = 0; i < MAXU; ++i) {
                const int u = w + NW * i;
                v[h][i] = (live && u < nc) ? __ldcg(ws_g + (size_t)u * NE + e) : 0.0;
              }
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              double sum = 0.0;
#pragma unroll
              for (int i = 0; i < MAXU; ++i) sum += v[h][i];
              S.red[w][32 * h + lane] = sum;
            }
            __syncthreads();
            if (w < 2 && eb + 32 * w + lane < e1) {
              double v = 0.0;
#pragma unroll
              for (int u = 0; u < NW; ++u) v += S.red[u][32 * w + lane];
              ws_gf[eb + 32 * w + lane] = v;
            }
            __syncthreads();
          }
        }
        GPROBE(2);
        grid_sync(ctr, epoch);
        GPROBE(3);
        {  // the reduced G into shared memory: all of a thread's L2 loads in flight first
          constexpr int PER = (TT * GX + NT - 1) / NT;
          double v[PER];
#pragma unroll
          for (int i = 0; i < PER; ++i) {
            const int e = tid + NT * i;
            v[i] = e < TT * GX ? __ldcg(ws_gf + e) : 0.0;
          }
          // meanwhile P_b -= Y_b D^-1 Y^T of the last fold: every owner's Y rows are in
          // (written before this barrier) and P_b is next read by U_b below
          if (pending_p6) apply_p6();
#pragma unroll
          for (int i = 0; i < PER; ++i) {
            const int e = tid + NT * i;
            if (e < TT * GX) S.Gs[e / GX][e % GX] = v[i];
          }
        }
        __syncthreads();
        // ---- P3: R = A - G C on my columns (M = t, N = my columns, K = i split over warps)
        {
          double acc[CW / 8][2], acc2[CW / 8][2];
#pragma unroll
          for (int nt = 0; nt < CW / 8; ++nt) acc[nt][0] = acc[nt][1] = acc2[nt][0] = acc2[nt][1] = 0.0;
          const int kmax = (r + 3) >> 2;  // rows of C beyond the rank are zero
          int kt = w;
          for (; kt + NW < kmax; kt += 2 * NW) {  // two independent chains
            const double a = S.Gs[p][4 * kt + q], a2 = S.Gs[p][4 * (kt + NW) + q];
#pragma unroll
            for (int nt = 0; nt < CW / 8; ++nt) {
              mma(acc[nt], a, S.Cs[kt][nt][lane]);
              mma(acc2[nt], a2, S.Cs[kt + NW][nt][lane]);
            }
          }
          if (kt < kmax) {
            const double a = S.Gs[p][4 * kt + q];
#pragma unroll
            for (int nt = 0; nt < CW / 8; ++nt) mma(acc[nt], a, S.Cs[kt][nt][lane]);
          }
#pragma unroll
          for (int nt = 0; nt < CW / 8; ++nt) {
            acc[nt][0] += acc2[nt][0];
            acc[nt][1] += acc2[nt][1];
          }
#pragma unroll
          for (int nt = 0; nt < CW / 8; ++nt) {
            S.red[w][p * CW + 8 * nt + 2 * q] = acc[nt][0];
            S.red[w][p * CW + 8 * nt + 2 * q + 1] = acc[nt][1];
          }
          __syncthreads();
          for (int e = tid; e < TT * CW; e += NT) {
            double v = S.At[cur][e / CW][e % CW];
#pragma unroll
            for (int u = 0; u < NW; ++u) v += S.red[u][e];
            S.Rs[e / CW][e % CW] = v;
          }
          __syncthreads();
          if (tid < TT) {
            double s = 0.0;
            for (int j = 0; j < CW; ++j) s = fma(S.Rs[tid][j], S.Rs[tid][j], s);
            ws_r[((size_t)0 * TT + tid) * nc + c] = s;
          }
          if (bulk_try && w == 1) {
            // R R^T over my columns (M = t, N = t', K = j): the same fragment is both operands
            double acc[2] = {0.0, 0.0};
#pragma unroll
            for (int kt = 0; kt < CW / 4; ++kt) {
              const double v = S.Rs[p][4 * kt + q];
              mma(acc, v, v);
            }
            *reinterpret_cast<double2*>(ws_m + (size_t)c * 64 + p * 8 + 2 * q) = make_double2(acc[0], acc[1]);
          }
        }
        // U_b = P_b G^T and the S / G W partials of every row of the tile, before the
        // rank test is known: the rows the test leaves out are masked afterwards
        // (zeroing the rows / columns of S and the columns of U_b gives the values of
        // the masked computation exactly), which saves the grid barrier that used to
        // separate the test from these partials
        if (owner) {
          // U_b = P_b G^T (M = i in my block, N = t, K = i' split over warps)
          double acc[2] = {0.0, 0.0};
          for (int kt = w; kt < R / 4; kt += NW) mma(acc, S.Ps[p][4 * kt + q], S.Gs[p][4 * kt + q]);
          __syncthreads();  // S.red is free again (the R reduction above is done)
          S.red[w][p * 8 + 2 * q] = acc[0];
          S.red[w][p * 8 + 2 * q + 1] = acc[1];
          __syncthreads();
          if (tid < 64) {
            double v = 0.0;
#pragma unroll
            for (int u = 0; u < NW; ++u) v += S.red[u][tid];
            S.Ub[tid >> 3][tid & 7] = v;
          }
          __syncthreads();
          if (w == 0) {
            // S_b = G[:, b] U_b and (G W)_b = G[:, b] W_b (M = t, K = i in my block)
            double sp[2] = {0.0, 0.0}, gw[2] = {0.0, 0.0};
#pragma unroll
            for (int kt = 0; kt < 2; ++kt) {
              const double a = S.Gs[p][8 * c + 4 * kt + q];
              mma(sp, a, S.Ub[4 * kt + q][p]);
              mma(gw, a, S.Wb[4 * kt + q][p]);
            }
            *reinterpret_cast<double2*>(ws_s + ((size_t)c * 2) * 64 + p * 8 + 2 * q) = make_double2(sp[0], sp[1]);
            *reinterpret_cast<double2*>(ws_s + ((size_t)c * 2 + 1) * 64 + p * 8 + 2 * q) = make_double2(gw[0], gw[1]);
          }
        }
        if (!bulk && tile + 1 < ntiles) {
          if (!staged) {
            stage(cur ^ 1);
            load_next(tile + 2);
            staged = true;
          }
          __syncthreads();
          p1(cur ^ 1, ws_r0 + (size_t)(nproj & 1u) * nc * 2 * TT);
          spec_valid = true;
        }
        GPROBE(4);
        grid_sync(ctr, epoch);
        GPROBE(5);
        // ---- P4: the rank test (identical in every CTA).  Warp t sums row t's
        // partials (lane l: CTAs l, l+32, ...; then a fixed butterfly).  The owners'
        // S and G W partials are loaded in the same round (used if rows are dependent).
        constexpr int SPER = (IT + NW - 1) / NW;
        double2 s2[SPER], g2[SPER];
        if (owner) {
#pragma unroll
          for (int i = 0; i < SPER; ++i) {
            const int u = w + NW * i;
            s2[i] = u < IT ? __ldcg(reinterpret_cast<const double2*>(ws_s + ((size_t)u * 2) * 64 + p * 8 + 2 * q))
                           : make_double2(0.0, 0.0);
            g2[i] = u < IT ? __ldcg(reinterpret_cast<const double2*>(ws_s + ((size_t)u * 2 + 1) * 64 + p * 8 + 2 * q))
                           : make_double2(0.0, 0.0);
          }
        }
        {
          constexpr int PER = (148 + 31) / 32;  // one CTA per SM
          double rv[PER], av[PER];
#pragma unroll
          for (int i = 0; i < PER; ++i) {  // [2][TT][nc]: coalesced, all in flight
            const int u = lane + 32 * i;
            rv[i] = u < nc ? __ldcg(ws_r + ((size_t)0 * TT + w) * nc + u) : 0.0;
            av[i] = u < nc ? __ldcg(ws_r + ((size_t)1 * TT + w) * nc + u) : 0.0;
          }
          double rs_ = 0.0, as_ = 0.0;
#pragma unroll
          for (int i = 0; i < PER; ++i) {
            rs_ += rv[i];
            as_ += av[i];
          }
          rs_ = warp_sum(rs_);
          as_ = warp_sum(as_);
          if (lane == 0) {
            S.red[0][w] = rs_;
            S.red[0][TT + w] = as_;
          }
        }
        __syncthreads();
        if (bulk_try) {
          // ---- certified block growth (general variant, x0 = 0; the panel kernel's
          // algebra, rgb_panel.cu): for a tile of independent rows the reference's
          // row-by-row growth (solver.py:305-318, _grow :368-380) is one block step
          // -- Z = (R R^T)^-1 R are the new dual rows, C~ - G^T Z the old ones, C
          // gains the rows, P^-1 = diag(P^-1, I), W gains y.  The pivot d_t of
          // R R^T = L D L^T is row t's squared rejection from the basis plus the
          // tile's rows before it; a row is certified when d_t clears the rank test
          // by BULK_MARGIN and keeps >= BULK_COND of |R_t|^2.  The certified prefix
          // is grown here (3 grid barriers per 8 rows instead of per row); the
          // first uncertified row ends the bulk phase and goes to the exact test.
          constexpr double BULK_COND = 0.1, BULK_MARGIN = 1e6;
          {
            // R R^T = the CTAs' partials summed in a fixed order (identical in every CTA)
            const int e = tid & 63, g = tid >> 6;
            constexpr int PER = (148 + NT / 64 - 1) / (NT / 64);
            double v[PER];
#pragma unroll
            for (int i = 0; i < PER; ++i) {
              const int u = g + (NT / 64) * i;
              v[i] = u < nc ? __ldcg(ws_m + (size_t)u * 64 + e) : 0.0;
            }
            double sum = 0.0;
#pragma unroll
            for (int i = 0; i < PER; ++i) sum += v[i];
            S.red[4 + g][e] = sum;
          }
          __syncthreads();
          if (w == 0) {
            double mm[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int idx = p * 8 + 2 * q + e;
              mm[e] = ((S.red[4][idx] + S.red[5][idx]) + S.red[6][idx]) + S.red[7][idx];
            }
            // a non-finite row enters as the identity (0 x NaN in the elimination
            // would reach the earlier rows); it fails the certification anyway
            double mi[2], ev[2], rd0, rd1;
            {
              const bool badp = !isfinite(S.red[0][TT + p]);
              const bool badc0 = !isfinite(S.red[0][TT + 2 * q]);
              const bool badc1 = !isfinite(S.red[0][TT + 2 * q + 1]);
              mi[0] = (badp || badc0) ? (p == 2 * q ? 1.0 : 0.0) : mm[0];
              mi[1] = (badp || badc1) ? (p == 2 * q + 1 ? 1.0 : 0.0) : mm[1];
            }
            blk::ldl8(mi, ev, rd0, rd1, p, q);
            const int t = lane & 7;
            const double x0 = __shfl_sync(FULL, rd0, t >> 1), x1 = __shfl_sync(FULL, rd1, t >> 1);
            const double rdt = (t & 1) ? x1 : x0;
            const double y0 = __shfl_sync(FULL, mm[0], 4 * t + (t >> 1));
            const double y1 = __shfl_sync(FULL, mm[1], 4 * t + (t >> 1));
            const double mtt = (t & 1) ? y1 : y0;
            const double at = S.red[0][TT + t];
            bool yok = true;
            for (int cc = 0; cc < k; ++cc) yok &= isfinite(S.Yv[cur][t][cc]);
            const double dt = 1.0 / rdt;
            const double e2 = eps_sq<double>(cfg, r + t);
            const bool ok = isfinite(at) && yok && dt > BULK_COND * mtt && dt > BULK_MARGIN * e2 * fmax(1.0, at);
            const unsigned failm = __ballot_sync(FULL, lane < TT && !ok);
            const int tst = failm ? __ffs(failm) - 1 : TT;
            S.Eb[p][2 * q] = ev[0];
            S.Eb[p][2 * q + 1] = ev[1];
            if (lane < TT) S.rd[lane] = rdt;
            if (lane == 0) S.flags[2] = tst;
          }
          __syncthreads();
          const int tst = S.flags[2];
          if (tst < TT) bulk = false;
          if (tst > 0) {
            // Q = D^-1 E R, then Z = E^T Q on my columns (rows t < tst)
            double* Qs = &S.red[1][0];
            double* Zs = &S.red[2][0];
            for (int e = tid; e < TT * CW; e += NT) {
              const int t = e / CW, j = e % CW;
              double v = 0.0;
              for (int t2 = 0; t2 <= t && t2 < tst; ++t2) v = fma(S.Eb[t][t2], S.Rs[t2][j], v);
              Qs[e] = t < tst ? v * S.rd[t] : 0.0;
            }
            __syncthreads();
            for (int e = tid; e < TT * CW; e += NT) {
              const int t = e / CW, j = e % CW;
              double v = 0.0;
              for (int t2 = tst - 1; t2 >= t; --t2) v = fma(S.Eb[t2][t], Qs[t2 * CW + j], v);
              Zs[e] = t < tst ? v : 0.0;
            }
            __syncthreads();
            // C~[:r] -= G^T Z, C~[r + t] = Z[t] on my columns; C[r + t] = a_t
            for (int e = tid; e < IT * (CW / 4) * 32; e += NT) {
              const int l = e & 31, kt = (e >> 5) % (CW / 4), nt = e / (32 * (CW / 4));
              const int i = 8 * nt + (l >> 2), jl = 4 * kt + (l & 3);
              if (i < r) {
                double v = S.Ds[nt][kt][l];
                for (int t = 0; t < tst; ++t) v -= S.Gs[t][i] * Zs[t * CW + jl];
                S.Ds[nt][kt][l] = v;
              } else if (i < r + tst) {
                S.Ds[nt][kt][l] = Zs[(i - r) * CW + jl];
              }
            }
            for (int e = tid; e < tst * CW; e += NT) {
              const int t = e / CW, jl = e % CW, i = r + t;
              S.Cs[i >> 2][jl >> 3][4 * (jl & 7) + (i & 3)] = -S.At[cur][t][jl];
            }
            if (owner) {
              // P = diag(P, I); W gains rows y_t - a_t.x0 (a.x0 = 0 here)
              for (int e = tid; e < 8 * R; e += NT) {
                const int i = 8 * c + e / R, i2 = e % R;
                const bool ni = i >= r && i < r + tst, ni2 = i2 >= r && i2 < r + tst;
                if (ni || ni2) S.Ps[e / R][i2] = (i == i2) ? 1.0 : 0.0;
              }
              if (tid < 64) {
                const int i = 8 * c + (tid >> 3), cc = tid & 7;
                if (i >= r && i < r + tst) S.Wb[tid >> 3][cc] = cc < k ? S.Yv[cur][i - r][cc] - S.Gs[i - r][R + cc] : 0.0;
              }
            }
            if (c == 0) {
              for (int t = tid; t < tst; t += NT)
                if (blog) blog[b * T + t0 + t] = 1;
              if (clog)
                for (int e = tid; e < tst * rc; e += NT)
                  clog[(b * T + t0 + e / rc) * rc + e % rc] = (e % rc == r + e / rc) ? 1.0 : 0.0;
            }
            __syncthreads();
            r += tst;
            spec_valid = false;  // the basis moved: a speculative next-tile projection is stale
            if (tst >= tv) break;    // the whole tile grew
            row_start = tst;         // the rest of the tile: re-projected on the new basis
            continue;
          }
          // nothing certified: the exact rank test below, on this projection
        }
        if (w == 0) {
          const double rsq = lane < TT ? S.red[0][lane] : 0.0;
          const double asq = lane < TT ? S.red[0][TT + lane] : 0.0;
          bool ybad = false;
          if (lane < TT)
            for (int cc = 0; cc < k; ++cc) ybad |= !isfinite(S.Yv[cur][lane][cc]);
          const bool valid = lane >= row_start && lane < tv;
          const bool dep = is_dependent<double>(rsq, asq, eps_sq<double>(cfg, r));
          const bool bad = !isfinite(asq) || ybad;
          const unsigned stopm = __ballot_sync(FULL, lane < TT && valid && (!dep || bad));
          const unsigned badm = __ballot_sync(FULL, lane < TT && valid && bad);
          if (lane < TT) S.scal[lane] = rsq;
          if (lane == 0) {
            S.flags[0] = stopm ? __ffs(stopm) - 1 : tv;
            S.flags[1] = (int)badm;
          }
        }
        __syncthreads();
        const int tstar = S.flags[0];
        const unsigned badm = (unsigned)S.flags[1];
        if (tstar > row_start) {
          // ---- dependent rows [row_start, tstar): blocked Sherman-Morrison
          const int rs = row_start, te = tstar;
          if (owner) {
            {
              // sums of the S and G W partials: warp w takes owners w, w+8, ...
              double a4[4] = {0.0, 0.0, 0.0, 0.0};  // loaded with the rank test, summed in owner order
#pragma unroll
              for (int i = 0; i < SPER; ++i) {
                a4[0] += s2[i].x;
                a4[1] += s2[i].y;
                a4[2] += g2[i].x;
                a4[3] += g2[i].y;
              }
#pragma unroll
              for (int i = 0; i < 4; ++i) S.red[w][4 * lane + i] = a4[i];
            }
            __syncthreads();
            if (w == 0) {
              // M = I + S, dy0 = y - a.x0 - G W (acc layout t = p, t' / c = 2q + e)
              double mi[2] = {0.0, 0.0}, gws[2] = {0.0, 0.0};
#pragma unroll
              for (int u = 0; u < NW; ++u) {
                mi[0] += S.red[u][4 * lane];
                mi[1] += S.red[u][4 * lane + 1];
                gws[0] += S.red[u][4 * lane + 2];
                gws[1] += S.red[u][4 * lane + 3];
              }
              const bool in_r = p >= rs && p < te;
              // rows / columns outside the dependent rows [rs, te) drop out of S
#pragma unroll
              for (int e = 0; e < 2; ++e)
                if (!in_r || 2 * q + e < rs || 2 * q + e >= te) mi[e] = 0.0;
              if (p == 2 * q) mi[0] += 1.0;
              if (p == 2 * q + 1) mi[1] += 1.0;
#pragma unroll
              for (int e = 0; e < 2; ++e)  // dy0[t = p][cc = 2q + e]
                S.Dy[p][2 * q + e] = in_r ? S.Yv[cur][p][2 * q + e] - S.Gs[p][R + 2 * q + e] - gws[e] : 0.0;
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
              S.Eb[p][2 * q] = ev[0];
              S.Eb[p][2 * q + 1] = ev[1];
              if ((p >> 1) == q) S.rd[p] = rcp64((p & 1) ? mi[1] : mi[0]);
              __syncwarp();
              // ... and the columns of U_b
#pragma unroll
              for (int kt = 0; kt < 2; ++kt)
                if (4 * kt + q < rs || 4 * kt + q >= te) S.Ub[p][4 * kt + q] = 0.0;
              __syncwarp();
              // Y_b = U_b E^T (M = i, N = t, K = t')
              double yb[2] = {0.0, 0.0};
#pragma unroll
              for (int kt = 0; kt < 2; ++kt) mma(yb, S.Ub[p][4 * kt + q], S.Eb[p][4 * kt + q]);
              S.Yb[p][2 * q] = yb[0];
              S.Yb[p][2 * q + 1] = yb[1];
              *reinterpret_cast<double2*>(ws_y + (size_t)(8 * c + p) * TT + 2 * q) = make_double2(yb[0], yb[1]);
              __syncwarp();
              // dh = E dy0 (M = t, N = cc, K = t'), scaled by 1/d_t
              double dh[2] = {0.0, 0.0};
#pragma unroll
              for (int kt = 0; kt < 2; ++kt) mma(dh, S.Eb[p][4 * kt + q], S.Dy[4 * kt + q][p]);
              S.Dy[p][2 * q] = dh[0] * S.rd[p];
              S.Dy[p][2 * q + 1] = dh[1] * S.rd[p];
              __syncwarp();
              // W_b += Y_b D^-1 E dy0 (M = i, N = cc, K = t)
              double wb[2] = {S.Wb[p][2 * q], S.Wb[p][2 * q + 1]};
#pragma unroll
              for (int kt = 0; kt < 2; ++kt) mma(wb, S.Yb[p][4 * kt + q], S.Dy[4 * kt + q][p]);
              S.Wb[p][2 * q] = wb[0];
              S.Wb[p][2 * q + 1] = wb[1];
            }
          }
          if (c == 0 && tid < TT && tid >= rs && tid < te) {
            const int64_t row = b * T + t0 + tid;
            if (blog) blog[row] = 0;
            if (clog)
              for (int i = 0; i < rc; ++i) clog[row * rc + i] = S.Gs[tid][i];
          }
          pending_p6 = true;  // applied after the next grid barrier (see apply_p6)
          __syncthreads();
        }
        if (tstar >= tv) break;
        if ((badm >> tstar) & 1u) {
          status |= RGB_ST_NONFINITE;
          stopped = true;
          consumed = t0 + tstar;
          break;
        }
        if (r >= rc) {
          status |= RGB_ST_RANK_CAP;
          stopped = true;
          consumed = t0 + tstar;
          break;
        }
        // ---- independent row tstar (solver.py:305-318, _grow solver.py:368-397)
        if (GEN || cfg.variant == RGB_GENERAL) {
          const int ts = tstar;
          const double rinv = 1.0 / S.scal[ts];  // K = rej / |rej|^2 (one rounding more than a division)
          // C~[:r] -= gamma K^T, C~[r] = K on my columns; C[r] = a
          for (int e = tid; e < IT * (CW / 4) * 32; e += NT) {
            const int l = e & 31, kt = (e >> 5) % (CW / 4), nt = e / (32 * (CW / 4));
            const int i = 8 * nt + (l >> 2), jl = 4 * kt + (l & 3);
            const double K = S.Rs[ts][jl] * rinv;
            S.Ds[nt][kt][l] = (i == r) ? K : fma(-S.Gs[ts][i], K, S.Ds[nt][kt][l]);
          }
          for (int e = tid; e < CW; e += NT) {
            const int kt = r >> 2, nt = e >> 3, l = 4 * (e & 7) + (r & 3);
            S.Cs[kt][nt][l] = -S.At[cur][ts][e];
          }
          if (owner) {
            // P = diag(P, 1); W gains row r = y - a.x0 of row ts
            for (int e = tid; e < 8 * R; e += NT) {
              const int i = 8 * c + e / R, i2 = e % R;
              if (i == r || i2 == r) S.Ps[e / R][i2] = (i == i2) ? 1.0 : 0.0;
            }
            if ((r >> 3) == c && tid < 8)
              S.Wb[r & 7][tid] = tid < k ? S.Yv[cur][ts][tid] - S.Gs[ts][R + tid] : 0.0;
          }
          if (c == 0 && tid == 0) {
            const int64_t row = b * T + t0 + ts;
            if (blog) blog[row] = 1;
            if (clog)
              for (int i = 0; i < rc; ++i) clog[row * rc + i] = (i == r) ? 1.0 : 0.0;
          }
          __syncthreads();
          r += 1;
          spec_valid = false;  // the basis moved: a speculative next-tile projection is stale
        } else {
          if (pending_p6) {  // z = P gamma needs the folded P
            grid_sync(ctr, epoch);
            apply_p6();
          }
          // orthogonal / orthonormal growth: C~[:r] and C[:r] stay, P gains an
          // edge -alpha z and a corner alpha^2 (1 + gamma.z), z = P gamma
          // (solver.py:307-310, 382-395); W gains alpha (y - a.x), a.x = a.x0 + gamma^T W
          const int ts = tstar;
          const double rsq = S.scal[ts];
          if (owner) {
            // z and the gamma.z / gamma^T W partials of my row block
            if (tid < 8) {
              const int i = 8 * c + tid;
              double z = 0.0;
              for (int i2 = 0; i2 < R; ++i2) z = fma(S.Ps[tid][i2], S.Gs[ts][i2], z);
              ws_z[i] = z;
              S.rd[tid] = z;
            }
            __syncthreads();
            if (tid < 9) {
              double v = 0.0;
              for (int u = 0; u < 8; ++u)
                v = fma(S.Gs[ts][8 * c + u], tid == 0 ? S.rd[u] : S.Wb[u][tid - 1], v);
              ws_d[(size_t)c * 16 + tid] = v;
            }
          }
          GPROBE(10);
          grid_sync(ctr, epoch);
          GPROBE(11);
          const double resc = (cfg.variant == RGB_ORTHONORMAL) ? 1.0 / sqrt(rsq) : cfg.alpha;
          const double last = 1.0 / resc;
          const double alpha = 1.0 / last;
          const double sc = alpha * rsq;
          for (int e = tid; e < (CW / 4) * 4; e += NT) {  // C~[r] on my columns
            const int kt = e >> 2, l = 4 * (r & 7) + (e & 3), jl = e;
            const double rj = S.Rs[ts][jl];
            S.Ds[r >> 3][kt][l] = (cfg.variant == RGB_ORTHONORMAL) ? alpha * rj : rj / sc;
          }
          for (int e = tid; e < CW; e += NT) {  // C[r] = alpha rej
            const int kt = r >> 2, nt = e >> 3, l = 4 * (e & 7) + (r & 3);
            S.Cs[kt][nt][l] = -(alpha * S.Rs[ts][e]);
          }
          if (owner) {
            const bool rown = (r >> 3) == c;
            double denom = 0.0;
            if (rown) {
              double dn = 0.0;
              for (int u = 0; u < IT; ++u) dn += __ldcg(ws_d + (size_t)u * 16);
              denom = 1.0 + dn;
            }
            for (int e = tid; e < 8 * R; e += NT) {
              const int i = 8 * c + e / R, i2 = e % R;
              double& P = S.Ps[e / R][i2];
              if (i == r && i2 == r) P = alpha * alpha * denom;
              else if (i2 == r) P = (i < r) ? -(alpha * S.rd[e / R]) : 0.0;
              else if (i == r) P = (i2 < r) ? -(alpha * __ldcg(ws_z + i2)) : 0.0;
            }
            if (rown && tid < 8) {
              double gw = 0.0;
              for (int u = 0; u < IT; ++u) gw += __ldcg(ws_d + (size_t)u * 16 + 1 + tid);
              S.Wb[r & 7][tid] = tid < k ? alpha * ((S.Yv[cur][ts][tid] - S.Gs[ts][R + tid]) - gw) : 0.0;
            }
          }
          if (c == 0 && tid == 0) {
            const int64_t row = b * T + t0 + ts;
            if (blog) blog[row] = 1;
            if (clog)
              for (int i = 0; i < rc; ++i) clog[row * rc + i] = i < r ? S.Gs[ts][i] : (i == r ? last : 0.0);
          }
          __syncthreads();
          r += 1;
          spec_valid = false;  // the basis moved: a speculative next-tile projection is stale
        }
        row_start = tstar + 1;
        if (row_start >= tv) break;
      }
      if (!stopped) consumed = t0 + tv;
    }

    if (pending_p6) {
      grid_sync(ctr, epoch);
      apply_p6();
    }
    // ---- write back: C~, C, P, W -> ws, then x = x0 + C~^T W on my columns ------------
    for (int e = tid; e < IT * (CW / 4) * 32; e += NT) {
      const int l = e & 31, kt = (e >> 5) % (CW / 4), nt = e / (32 * (CW / 4));
      const int i = 8 * nt + (l >> 2), col = c0 + 4 * kt + (l & 3);
      if (i < rc && col < M) Dg[(int64_t)i * M + col] = S.Ds[nt][kt][l];
    }
    for (int e = tid; e < (R / 4) * (CW / 8) * 32; e += NT) {
      const int l = e & 31, nt = (e >> 5) % (CW / 8), kt = e / (32 * (CW / 8));
      const int i = 4 * kt + (l & 3), col = c0 + 8 * nt + (l >> 2);
      if (i < rc && col < M) Cg[(int64_t)i * M + col] = -S.Cs[kt][nt][l];
    }
    if (owner) {
      for (int e = tid; e < 8 * R; e += NT) {
        const int i = 8 * c + e / R, i2 = e % R;
        if (i < rc && i2 < rc) Pg[(int64_t)i * rc + i2] = S.Ps[e / R][i2];
      }
      for (int e = tid; e < 64; e += NT) ws_w[(size_t)(8 * c + (e >> 3)) * 8 + (e & 7)] = S.Wb[e >> 3][e & 7];
    }
    grid_sync(ctr, epoch);
    for (int e = tid; e < k * CW; e += NT) {
      const int cc = e / CW, jl = e % CW;
      double x = S.Ds[NXT - 1][jl >> 2][4 * (cc) + (jl & 3)];  // x0^T row cc sits in the last N tile
      // the last N tile of Ds holds x0^T rows R..R+7: lane = 4 * (i - R) + (jl & 3)
      for (int i = 0; i < r; ++i) x = fma(S.Ds[i >> 3][jl >> 2][4 * (i & 7) + (jl & 3)], __ldcg(ws_w + (size_t)i * 8 + cc), x);
      if (c0 + jl < M) Xg[(int64_t)cc * M + c0 + jl] = x;
    }
    if (c == 0 && tid == 0) {
      st.rank[b] = r;
      st.nobs[b] = nobs0 + consumed;
      st.status[b] = status;
    }
    grid_sync(ctr, epoch);  // the next stream reuses the workspace
  }
}

}  // namespace grd

// Workspace pool of the current device: created once, never trimmed (the grid
// kernel's workspace, the panel kernel's stream counter).
cudaMemPool_t workspace_pool() {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!pools[dev]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t p = nullptr;
    if (cudaMemPoolCreate(&p, &props) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &keep);
    pools[dev] = p;
  }
  return pools[dev];
}

template <int R, int CW, typename TI>
static int launch_grid_t(const rgb_config& cfg, rgb_state& st, const void* rows, int64_t rows_stride,
                         const void* targets, int64_t tg_stride, int64_t T, const rgb_logs& logs,
                         cudaStream_t stream, int num_sms) {
  // CTA c owns columns [c CW, (c + 1) CW) (masked past m) and, for c < R / 8, a
  // row block of P^-1 and W: enough CTAs for both, all co-resident (one per SM)
  int nc = (cfg.m + CW - 1) / CW;
  if (nc < R / 8) nc = R / 8;
  if (nc > num_sms || cfg.r_cap > R) return RGB_E_UNSUPPORTED;
  auto kern = cfg.variant == RGB_GENERAL ? grd::grid_kernel<R, CW, true, TI> : grd::grid_kernel<R, CW, false, TI>;
  const size_t smem = sizeof(grd::GridSmem<R, CW>);
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    cudaGetLastError();
    return RGB_E_UNSUPPORTED;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, grd::NT, smem);
  if (per_sm < 1) return RGB_E_UNSUPPORTED;
  const size_t wsb = grd::Ws<R, CW>::bytes(nc);
  void* ws = nullptr;
  cudaMemPool_t pool = workspace_pool();
  if (!pool || cudaMallocFromPoolAsync(&ws, wsb, pool, stream) != cudaSuccess) return RGB_E_CUDA;
  cudaMemsetAsync(ws, 0, 256, stream);
  double* wsd = reinterpret_cast<double*>(ws);
  unsigned* ctr = reinterpret_cast<unsigned*>(ws);
  const TI* rp = (const TI*)rows;
  const TI* tp = (const TI*)targets;
  uint8_t* bl = logs.branch;
  double* cl = (double*)logs.coords;
  rgb_config c2 = cfg;
  rgb_state s2 = st;
  void* args[] = {&c2, &s2, (void*)&rp, &rows_stride, (void*)&tp, &tg_stride, &T, &bl, &cl, &wsd, &ctr};
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)kern, dim3(nc), dim3(grd::NT), args, smem, stream);
  cudaFreeAsync(ws, stream);
  return e == cudaSuccess ? RGB_OK : RGB_E_CUDA;
}

// Single large streams of any width up to 148 x 16 columns with capacity up
// to 512, or up to 148 x 32 columns with capacity up to 256: the smallest
// instantiated R >= r_cap.  (Small problems stay on the
// generic kernel: a grid step costs a few microseconds of barriers.)
bool grid_supports(const rgb_config& cfg) {
  const bool var_ok = cfg.variant == RGB_GENERAL || cfg.variant == RGB_ORTHONORMAL ||
                      (cfg.variant == RGB_ORTHOGONAL && cfg.alpha != 0.0);
  if (cfg.dtype != RGB_F64 || !var_ok || cfg.k < 1 || cfg.k > 8) return false;
  if (cfg.num_streams > 4) return false;  // a handful of large streams, one after the other
  if (cfg.r_cap > 512 || cfg.m > 148 * 32) return false;
  if (cfg.m > 148 * 16 && cfg.r_cap > 256) return false;  // 32-column slices: R <= 256 fits shared memory
  return (int64_t)cfg.m * cfg.r_cap >= 32768;
}

template <typename TI>
static int launch_grid_r(const rgb_config& cfg, rgb_state& st, const void* rows, int64_t rows_stride,
                         const void* targets, int64_t tg_stride, int64_t T, const rgb_logs& logs,
                         cudaStream_t stream, int num_sms) {
  if (cfg.m > 148 * 16) {  // wide streams: 32 columns per CTA
    if (cfg.r_cap <= 64)
      return launch_grid_t<64, 32, TI>(cfg, st, rows, rows_stride, targets, tg_stride, T, logs, stream, num_sms);
    if (cfg.r_cap <= 128)
      return launch_grid_t<128, 32, TI>(cfg, st, rows, rows_stride, targets, tg_stride, T, logs, stream, num_sms);
    return launch_grid_t<256, 32, TI>(cfg, st, rows, rows_stride, targets, tg_stride, T, logs, stream, num_sms);
  }
  if (cfg.r_cap <= 64 && cfg.m <= 148 * 8)
    return launch_grid_t<64, 8, TI>(cfg, st, rows, rows_stride, targets, tg_stride, T, logs, stream, num_sms);
  if (cfg.r_cap <= 64)
    return launch_grid_t<64, 16, TI>(cfg, st, rows, rows_stride, targets, tg_stride, T, logs, stream, num_sms);
  if (cfg.r_cap <= 128)
    return launch_grid_t<128, 16, TI>(cfg, st, rows, rows_stride, targets, tg_stride, T, logs, stream, num_sms);
  if (cfg.r_cap <= 256)
    return launch_grid_t<256, 16, TI>(cfg, st, rows, rows_stride, targets, tg_stride, T, logs, stream, num_sms);
  return launch_grid_t<512, 16, TI>(cfg, st, rows, rows_stride, targets, tg_stride, T, logs, stream, num_sms);
}

int launch_grid(const rgb_config& cfg, rgb_state& st, const void* rows, int64_t rows_stride, const void* targets,
                int64_t tg_stride, int64_t T, const rgb_logs& logs, cudaStream_t stream, int num_sms, bool f32in) {
  if (logs.resid || logs.gain) return RGB_E_UNSUPPORTED;
  if (!grid_supports(cfg)) return RGB_E_UNSUPPORTED;
  return f32in ? launch_grid_r<float>(cfg, st, rows, rows_stride, targets, tg_stride, T, logs, stream, num_sms)
               : launch_grid_r<double>(cfg, st, rows, rows_stride, targets, tg_stride, T, logs, stream, num_sms);
}

}  // namespace rgb

#ifdef RGB_GRID_PROBE
extern "C" int rgb_grid_probe(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, rgb::grd::g_gprobe, sizeof(rgb::grd::g_gprobe));
  if (reset) {
    unsigned long long z[2][16] = {};
    cudaMemcpyToSymbol(rgb::grd::g_gprobe, z, sizeof(z));
  }
  return 0;
}
#endif
