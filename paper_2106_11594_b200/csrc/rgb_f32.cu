// rgb_f32.cu -- config-5 streams with a float32 state on the fp32 CUDA cores.
//
// BASELINE.json's config 5 asks for fp32 as well as fp64.  tcgen05 and the
// warp-level tensor paths have no fp32-exact kind (tf32 keeps 10 mantissa
// bits), so fp32 arithmetic runs on the FFMA pipe (70.9 TF/s measured here,
// tools/fp64_peak.cu, against 36.6 TF/s for the fp64 DMMA path).  One warp owns
// one stream (m 64, rank capacity 16, k <= 8, general variant) and consumes
// 8-row tiles with the blocked algebra of rgb_blocked.cu restated for FFMA:
//
//   G  = A C~^T (+ A x0 for continuation calls)   lane-local partials over the
//        lane's two columns, then a warp reduce-scatter (5 shuffle stages)
//   R  = A - G C, |R_t|^2, |a_t|^2                 lane-local, one reduce-scatter
//   rank test per row (solver.py:292-296, float32 eps policy)
//   dependent rows [rs, te): U = G P, M = I + U G^T = L D L^T, E = L^-1,
//        Y = U^T E^T, P -= Y D^-1 Y^T, W += Y D^-1 E dy0   (solver.py:297-304
//        folded over the tile: the sequential Sherman-Morrison steps in LDL^T form)
//   independent row (solver.py:305-318, general _grow 368-379): C~ -= gamma K^T,
//        C~[r] = K, C[r] = a, P = diag(P, 1), W[r] = y - a.x0; the rest of the
//        tile is re-projected on the new basis
//   x = x0 + C~^T W once per call.
//
// Lane l owns columns l and l + 32 of C~ and C in registers (32 + 32 floats);
// P^-1, W, G and the small tile matrices live in the warp's shared memory.
#include "rgb_common.cuh"

#ifndef RGB_F32_MINB
#define RGB_F32_MINB 3  // CTAs of 4 warps per SM (168 registers; 4 spills, measured slower/faster below)
#endif

namespace rgb {
namespace f32k {

constexpr unsigned FULL = 0xffffffffu;
constexpr int M = 64, R = 16, KX = 8, TT = 8, WARPS = 4, NT = WARPS * 32;
constexpr int PS = 20;  // padded row pitch of P^-1 (conflict-light row reads)
constexpr int AP = M + 4;  // row pitch of the tile ring: conflict-free 8-byte MMA fragment reads
constexpr int GS = 28;  // row pitch of G: 16 coordinates + 8 a.x0 columns + pad

struct __align__(16) WarpSmem {
  float A[2][TT][AP];   // tile ring (cp.async)
  float Y[2][TT][KX];   // targets ring
  float G[TT][GS];      // G | a.x0
  float P[R][PS];       // P^-1
  float Wt[KX][PS];     // W^T (W: R x k)
  float Us[TT][PS];     // U = G P (t x i)
  float Em[TT][TT];     // E = L^-1
  float Yy[R][TT];      // Y = U^T E^T (i x t)
  float Dy[TT][KX];     // dy0
  float DhT[KX][TT];    // (D^-1 E dy0)^T
  float rd[TT];         // 1 / d_t (16-byte aligned: float4 reads)
  float sums[2][TT];    // |R_t|^2, |a_t|^2
  float X0[KX][M];      // x0^T (continuation calls)
  float Kv[M];          // K = rej / |rej|^2 of a growing row
};

// 1/x to ~1 ulp (MUFU.RCP): LDL^T pivots of I + G P G^T (>= 1)
__device__ __forceinline__ float rcpf(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// 3xTF32: x = big + small with big = x rounded to tf32 (cvt.rna) and small = x - big
// (exact; the tensor core reads its top 10 mantissa bits), so that
// big_a big_b + big_a small_b + small_a big_b carries fp32-level accuracy
__device__ __forceinline__ void tf32_split(float x, uint32_t& big, uint32_t& small) {
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(big) : "f"(x));
  small = __float_as_uint(x - __uint_as_float(big));
}
// D += A B on mma.sync m16n8k8 (tf32 in, fp32 accumulate)
__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

__device__ __forceinline__ void cp4(void* smem, const void* gmem, bool ok) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(gmem), "r"(ok ? 4 : 0));
}
__device__ __forceinline__ void cp16(void* smem, const void* gmem, bool ok) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(ok ? 16 : 0));
}

// 8x8 L D L^T of the SPD matrix M in registers (lane = 4p + q holds M[p][2q + e]):
// ev[e] = E[p][2q + e] with E = L^-1; rd0 / rd1 = 1/d at t = 2q, 2q + 1.  The
// float32 restatement of rgb_mma.cuh's ldl8 (Gaussian elimination by shuffles).
__device__ __forceinline__ void ldl8f(float (&mi)[2], float (&ev)[2], float& rd0, float& rd1, int p, int q) {
  ev[0] = p == 2 * q ? 1.f : 0.f;
  ev[1] = p == 2 * q + 1 ? 1.f : 0.f;
#pragma unroll
  for (int kk = 0; kk < TT - 1; ++kk) {
    const float v = (kk & 1) ? mi[1] : mi[0];
    const float piv = __shfl_sync(FULL, v, 4 * kk + (kk >> 1));
    const float mps = __shfl_sync(FULL, v, 4 * p + (kk >> 1));
    const float m0 = __shfl_sync(FULL, mi[0], 4 * kk + q);
    const float m1 = __shfl_sync(FULL, mi[1], 4 * kk + q);
    const float e0 = __shfl_sync(FULL, ev[0], 4 * kk + q);
    const float e1 = __shfl_sync(FULL, ev[1], 4 * kk + q);
    const float f = (p > kk) ? mps * rcpf(piv) : 0.f;
    mi[0] = fmaf(-f, m0, mi[0]);
    mi[1] = fmaf(-f, m1, mi[1]);
    ev[0] = fmaf(-f, e0, ev[0]);
    ev[1] = fmaf(-f, e1, ev[1]);
  }
  const float dsel = (p & 1) ? mi[1] : mi[0];
  const float rdp = rcpf(__shfl_sync(FULL, dsel, 4 * p + (p >> 1)));
  rd0 = __shfl_sync(FULL, rdp, 8 * q);
  rd1 = __shfl_sync(FULL, rdp, 8 * q + 4);
}

// Reduce-scatter of N values (N = 32 or 16 per half-warp) across the lanes:
// lane l returns the sum over the participating lanes of value index l (mod N).
// Fixed shuffle order: deterministic.
template <int N>
__device__ __forceinline__ float reduce_scatter(float (&v)[N], int lane) {
#pragma unroll
  for (int half = N / 2; half >= 1; half >>= 1) {
    const bool up = lane & half;
#pragma unroll
    for (int j = 0; j < half; ++j) {
      const float send = up ? v[j] : v[j + half];
      const float keep = up ? v[j + half] : v[j];
      v[j] = keep + __shfl_xor_sync(FULL, send, half);
    }
  }
  return v[0];
}

// stage tile `tile` (8 rows and targets) of one stream into ring slot s
__device__ __forceinline__ void stage_tile(WarpSmem& S, int s, const float* rows, const float* tg, int64_t T,
                                           int k, int64_t tile, int lane) {
  const int64_t t0 = tile * TT;
  // rows: 8 x 64 floats = 128 16-byte pieces, 4 per lane (rows are contiguous per stream)
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int e = lane + 32 * q, t = e >> 4, c4 = (e & 15) * 4;
    const bool ok = t0 + t < T;
    cp16(&S.A[s][t][c4], ok ? rows + (t0 + t) * M + c4 : rows, ok);
  }
  if (k == KX && ((reinterpret_cast<uintptr_t>(tg) & 15) == 0)) {
    // 8 targets per row = two 16-byte pieces, 16 pieces per tile
    if (lane < 2 * TT) {
      const int t = lane >> 1, c4 = (lane & 1) * 4;
      const bool ok = t0 + t < T;
      cp16(&S.Y[s][t][c4], ok ? tg + (t0 + t) * KX + c4 : tg, ok);
    }
  } else {
    for (int e = lane; e < TT * KX; e += 32) {
      const int t = e >> 3, c = e & 7;
      const bool ok = t0 + t < T && c < k;
      cp4(&S.Y[s][t][c], ok ? tg + (t0 + t) * k + c : tg, ok);
    }
  }
  asm volatile("cp.async.commit_group;\n" ::);
}

template <bool LOGC>
__global__ void __launch_bounds__(NT, RGB_F32_MINB) f32_kernel(rgb_config cfg, rgb_state st, const float* __restrict__ rows,
                                                 int64_t rstride, const float* __restrict__ tgts, int64_t tstride,
                                                 int64_t T, uint8_t* __restrict__ blog, float* __restrict__ clog) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  WarpSmem& S = reinterpret_cast<WarpSmem*>(smem_raw)[wib];
  const int k = cfg.k, rc = cfg.r_cap;
  const int64_t gw = (int64_t)blockIdx.x * WARPS + wib, nw = (int64_t)gridDim.x * WARPS;
  const int j0 = lane, j1 = lane + 32;  // my columns
  const int pi = lane & 15, ph = lane >> 4;  // my (row, half) in the 16 x 16 / 16 x 8 matrices
  const int fg = lane >> 2, fq = lane & 3;    // my MMA fragment coordinates

  for (int64_t b = gw; b < cfg.num_streams; b += nw) {
    int status = st.status[b];
    if (status) continue;
    int r = st.rank[b];
    const int64_t nobs0 = st.nobs[b];
    float* Cg = reinterpret_cast<float*>(st.basis) + b * (int64_t)rc * M;
    float* Dg = reinterpret_cast<float*>(st.dual) + b * (int64_t)rc * M;
    float* Pg = reinterpret_cast<float*>(st.gram_inv) + b * (int64_t)rc * rc;
    float* Xg = reinterpret_cast<float*>(st.x) + b * (int64_t)k * M;
    const float* Rb = rows + b * rstride;
    const float* Yb = tgts + b * tstride;
    const int64_t ntiles = (T + TT - 1) / TT;
    if (ntiles > 0) stage_tile(S, 0, Rb, Yb, T, k, 0, lane);

    // ---- load the state: C~, C (my columns), x0 (my columns), P^-1; W = 0 ----
    // C~: the A fragments of G^T = C~ A^T on mma.sync m16n8k8 (M = rank, K = column):
    // lane (fg, fq) holds rows fg and fg + 8 at columns 8kk + 2fq + {0, 1}, kk < 8
    // (logical K slots fq and fq + 4 of k-step kk); C: lane l holds columns l and
    // l + 32 of every row (R is lane-local)
    float Dm[8][4], Ct[R][2];
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const float2 v0 = fg < r ? *reinterpret_cast<const float2*>(Dg + fg * M + 8 * kk + 2 * fq) : make_float2(0, 0);
      const float2 v1 =
          fg + 8 < r ? *reinterpret_cast<const float2*>(Dg + (fg + 8) * M + 8 * kk + 2 * fq) : make_float2(0, 0);
      Dm[kk][0] = v0.x;
      Dm[kk][1] = v1.x;
      Dm[kk][2] = v0.y;
      Dm[kk][3] = v1.y;
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const bool on = i < r;
      Ct[i][0] = on ? Cg[i * M + j0] : 0.f;
      Ct[i][1] = on ? Cg[i * M + j1] : 0.f;
    }
    const bool has_x0 = nobs0 > 0;  // a fresh stream has x0 = 0 exactly
#pragma unroll
    for (int c = 0; c < KX; ++c) {
      S.X0[c][j0] = (has_x0 && c < k) ? Xg[c * M + j0] : 0.f;
      S.X0[c][j1] = (has_x0 && c < k) ? Xg[c * M + j1] : 0.f;
    }
    for (int e = lane; e < R * R; e += 32) {
      const int i = e >> 4, l = e & 15;
      S.P[i][l] = (i < r && l < r) ? Pg[i * rc + l] : 0.f;
    }
    for (int e = lane; e < KX * R; e += 32) S.Wt[e >> 4][e & 15] = 0.f;
    __syncwarp();

    int64_t consumed = 0;
    bool stopped = false;
    for (int64_t tile = 0; tile < ntiles && !stopped; ++tile) {
      const int s = (int)(tile & 1);
      if (tile + 1 < ntiles) {
        stage_tile(S, s ^ 1, Rb, Yb, T, k, tile + 1, lane);
        asm volatile("cp.async.wait_group 1;\n" ::);
      } else {
        asm volatile("cp.async.wait_group 0;\n" ::);
      }
      __syncwarp();
      const int64_t t0 = tile * TT;
      const int tv = (int)((T - t0) < TT ? (T - t0) : TT);
      float a[TT][2];
#pragma unroll
      for (int t = 0; t < TT; ++t) {
        a[t][0] = S.A[s][t][j0];
        a[t][1] = S.A[s][t][j1];
      }
      // rows whose targets are not finite (scalars.py:122-123): two ballots per tile
      unsigned ybad = 0;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int idx = lane + 32 * e, t = idx >> 3, c = idx & 7;
        const unsigned bm = __ballot_sync(FULL, c < k && !isfinite(S.Y[s][t][c]));
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if ((bm >> (8 * u)) & 0xFFu) ybad |= 1u << (4 * e + u);
      }
      int row_start = 0;
      while (true) {
        // ---- G = A C~^T on the tensor cores: G^T = C~ A^T (M = rank, N = the tile's
        // rows, K = columns), tf32 in three passes (big x big, then big x small and
        // small x big into a second accumulator), fp32 accumulation
        {
          float gb[4] = {0.f, 0.f, 0.f, 0.f}, gsm[4] = {0.f, 0.f, 0.f, 0.f};
          const float* arow = &S.A[s][fg][2 * fq];
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const float2 bv = *reinterpret_cast<const float2*>(arow + 8 * kk);
            uint32_t bb[2], bs[2], ab[4], as[4];
            tf32_split(bv.x, bb[0], bs[0]);
            tf32_split(bv.y, bb[1], bs[1]);
#pragma unroll
            for (int e = 0; e < 4; ++e) tf32_split(Dm[kk][e], ab[e], as[e]);
            mma_tf32(gb, ab, bb);
            mma_tf32(gsm, ab, bs);
            mma_tf32(gsm, as, bb);
          }
          // G^T[fg][2fq], G^T[fg][2fq + 1], G^T[fg + 8][2fq], G^T[fg + 8][2fq + 1]
          S.G[2 * fq][fg] = gb[0] + gsm[0];
          S.G[2 * fq + 1][fg] = gb[1] + gsm[1];
          S.G[2 * fq][fg + 8] = gb[2] + gsm[2];
          S.G[2 * fq + 1][fg + 8] = gb[3] + gsm[3];
        }
        if (has_x0) {  // a.x0_c (continuation calls): 2 more reduce-scatters
#pragma unroll
          for (int g = 0; g < 2; ++g) {
            float v[32];
#pragma unroll
            for (int q = 0; q < 32; ++q) {
              const int t = 4 * g + (q >> 3), c = q & 7;
              v[q] = fmaf(a[t][1], S.X0[c][j1], a[t][0] * S.X0[c][j0]);
            }
            S.G[4 * g + (lane >> 3)][16 + (lane & 7)] = reduce_scatter<32>(v, lane);
          }
        } else if (lane < TT * KX / 8) {
          // (a.x0 = 0: zero the 8 x 8 block, 8 floats per lane for 8 lanes)
#pragma unroll
          for (int c = 0; c < KX; ++c) S.G[lane][16 + c] = 0.f;
        }
        __syncwarp();
        // ---- R = A - G C on my columns, |R_t|^2 and |a_t|^2 ----------------------
        // (the rejection itself is not kept: a growth recomputes its row's)
        {
          float v[16];
#pragma unroll
          for (int t = 0; t < TT; ++t) {
            float s0 = 0.f, s1 = 0.f;
#pragma unroll
            for (int i4 = 0; i4 < R; i4 += 4) {
              const float4 gq = *reinterpret_cast<const float4*>(&S.G[t][i4]);
              s0 = fmaf(gq.x, Ct[i4][0], s0);
              s1 = fmaf(gq.x, Ct[i4][1], s1);
              s0 = fmaf(gq.y, Ct[i4 + 1][0], s0);
              s1 = fmaf(gq.y, Ct[i4 + 1][1], s1);
              s0 = fmaf(gq.z, Ct[i4 + 2][0], s0);
              s1 = fmaf(gq.z, Ct[i4 + 2][1], s1);
              s0 = fmaf(gq.w, Ct[i4 + 3][0], s0);
              s1 = fmaf(gq.w, Ct[i4 + 3][1], s1);
            }
            const float r0 = a[t][0] - s0, r1 = a[t][1] - s1;
            v[t] = fmaf(r1, r1, r0 * r0);
            v[TT + t] = fmaf(a[t][1], a[t][1], a[t][0] * a[t][0]);
          }
          // reduce-scatter inside each half-warp, then add the two halves
          float part = reduce_scatter<16>(v, lane);
          part += __shfl_xor_sync(FULL, part, 16);
          if (lane < 16) S.sums[lane >> 3][lane & 7] = part;
        }
        __syncwarp();
        // ---- rank test: lane t tests row t, one ballot (identical result in every lane)
        const float esq = eps_sq<float>(cfg, r);
        unsigned badm, stopm;
        {
          const int t = lane & 7;
          const float rsq = S.sums[0][t], asq = S.sums[1][t];
          const bool bad = !isfinite(asq) || ((ybad >> t) & 1u);
          const bool valid = lane < TT && t >= row_start && t < tv;
          badm = __ballot_sync(FULL, valid && bad);
          stopm = __ballot_sync(FULL, valid && (bad || !is_dependent<float>(rsq, asq, esq)));
        }
        const int tstar = stopm ? __ffs(stopm) - 1 : tv;
        const int rs = row_start, te = tstar;
        if (te > rs) {
          // ---- dependent rows [rs, te): blocked Sherman-Morrison in LDL^T form -------
          const bool full_fold = r > 0;
          if (full_fold) {
            // U = G P (t x i): lane (i = pi, t = 4 ph .. 4 ph + 3); P's row pi read once
            float pr[R];
#pragma unroll
            for (int l4 = 0; l4 < R; l4 += 4) {
              const float4 pq = *reinterpret_cast<const float4*>(&S.P[pi][l4]);
              pr[l4] = pq.x;
              pr[l4 + 1] = pq.y;
              pr[l4 + 2] = pq.z;
              pr[l4 + 3] = pq.w;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int t = 4 * ph + u;
              float acc = 0.f;
#pragma unroll
              for (int l4 = 0; l4 < R; l4 += 4) {
                const float4 gq = *reinterpret_cast<const float4*>(&S.G[t][l4]);
                acc = fmaf(gq.x, pr[l4], acc);
                acc = fmaf(gq.y, pr[l4 + 1], acc);
                acc = fmaf(gq.z, pr[l4 + 2], acc);
                acc = fmaf(gq.w, pr[l4 + 3], acc);
              }
              S.Us[t][pi] = (t >= rs && t < te) ? acc : 0.f;  // rows outside the run drop out
            }
          }
          __syncwarp();
          // M = I + U G^T (masked, in registers: lane (t = l / 4, t' = 2 (l % 4) + e)),
          // dy0 = y - a.x0 - G W (same lanes, c = t'), then M = L D L^T by shuffles
          {
            const int t = lane >> 2, q2 = 2 * (lane & 3);
            const bool in_t = t >= rs && t < te;
            float ur[R], gr[R];
#pragma unroll
            for (int i4 = 0; i4 < R; i4 += 4) {
              const float4 u = *reinterpret_cast<const float4*>(&S.Us[t][i4]);
              const float4 g1 = *reinterpret_cast<const float4*>(&S.G[t][i4]);
              ur[i4] = u.x; ur[i4 + 1] = u.y; ur[i4 + 2] = u.z; ur[i4 + 3] = u.w;
              gr[i4] = g1.x; gr[i4 + 1] = g1.y; gr[i4 + 2] = g1.z; gr[i4 + 3] = g1.w;
            }
            float mi[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int t2 = q2 + e;
              float sv = 0.f, gwv = 0.f;
              if (full_fold) {
#pragma unroll
                for (int i4 = 0; i4 < R; i4 += 4) {
                  const float4 g2 = *reinterpret_cast<const float4*>(&S.G[t2][i4]);
                  const float4 w = *reinterpret_cast<const float4*>(&S.Wt[t2][i4]);
                  sv = fmaf(ur[i4], g2.x, sv);
                  gwv = fmaf(gr[i4], w.x, gwv);
                  sv = fmaf(ur[i4 + 1], g2.y, sv);
                  gwv = fmaf(gr[i4 + 1], w.y, gwv);
                  sv = fmaf(ur[i4 + 2], g2.z, sv);
                  gwv = fmaf(gr[i4 + 2], w.z, gwv);
                  sv = fmaf(ur[i4 + 3], g2.w, sv);
                  gwv = fmaf(gr[i4 + 3], w.w, gwv);
                }
              }
              const bool in2 = t2 >= rs && t2 < te;
              mi[e] = (in_t && in2 ? sv : 0.f) + (t == t2 ? 1.f : 0.f);
              S.Dy[t][t2] = in_t && t2 < k ? (S.Y[s][t][t2] - S.G[t][16 + t2]) - gwv : 0.f;
            }
            if (full_fold) {
              float ev[2], rd0, rd1;
              ldl8f(mi, ev, rd0, rd1, t, lane & 3);
              S.Em[t][q2] = ev[0];
              S.Em[t][q2 + 1] = ev[1];
              if (t == 0) {
                S.rd[q2] = rd0;
                S.rd[q2 + 1] = rd1;
              }
            }
          }
          __syncwarp();
          if (full_fold) {
            const int t = lane >> 2, q2 = 2 * (lane & 3);
            // Y = U^T E^T (i x t): lane (i = pi, t = 4 ph + u); U's column pi read once
            float uc[TT];
#pragma unroll
            for (int t2 = 0; t2 < TT; ++t2) uc[t2] = S.Us[t2][pi];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int tt = 4 * ph + u;
              const float4 e0 = *reinterpret_cast<const float4*>(&S.Em[tt][0]);
              const float4 e1 = *reinterpret_cast<const float4*>(&S.Em[tt][4]);
              float acc = uc[0] * e0.x;
              acc = fmaf(uc[1], e0.y, acc);
              acc = fmaf(uc[2], e0.z, acc);
              acc = fmaf(uc[3], e0.w, acc);
              acc = fmaf(uc[4], e1.x, acc);
              acc = fmaf(uc[5], e1.y, acc);
              acc = fmaf(uc[6], e1.z, acc);
              acc = fmaf(uc[7], e1.w, acc);
              S.Yy[pi][tt] = acc;
            }
            // dh = D^-1 E dy0 (t x c): lane (t = l / 4, c = 2 (l % 4) + e); E's row t read once
            float er[TT];
            {
              const float4 e0 = *reinterpret_cast<const float4*>(&S.Em[t][0]);
              const float4 e1 = *reinterpret_cast<const float4*>(&S.Em[t][4]);
              er[0] = e0.x; er[1] = e0.y; er[2] = e0.z; er[3] = e0.w;
              er[4] = e1.x; er[5] = e1.y; er[6] = e1.z; er[7] = e1.w;
            }
            const float rdt = S.rd[t];
            float dh[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int c = q2 + e;
              float acc = 0.f;
#pragma unroll
              for (int t2 = 0; t2 < TT; ++t2) acc = fmaf(er[t2], S.Dy[t2][c], acc);
              dh[e] = acc * rdt;
            }
            S.DhT[q2][t] = dh[0];
            S.DhT[q2 + 1][t] = dh[1];
            __syncwarp();
            // P -= Y D^-1 Y^T: lane (i = pi, l = 8 ph .. 8 ph + 7);  W += Y dh: lane (i = pi, c = 4 ph + u)
            float yi[TT], ys[TT];
            {
              const float4 y0 = *reinterpret_cast<const float4*>(&S.Yy[pi][0]);
              const float4 y1 = *reinterpret_cast<const float4*>(&S.Yy[pi][4]);
              const float4 d0 = *reinterpret_cast<const float4*>(&S.rd[0]);
              const float4 d1 = *reinterpret_cast<const float4*>(&S.rd[4]);
              yi[0] = y0.x; yi[1] = y0.y; yi[2] = y0.z; yi[3] = y0.w;
              yi[4] = y1.x; yi[5] = y1.y; yi[6] = y1.z; yi[7] = y1.w;
              ys[0] = y0.x * d0.x; ys[1] = y0.y * d0.y; ys[2] = y0.z * d0.z; ys[3] = y0.w * d0.w;
              ys[4] = y1.x * d1.x; ys[5] = y1.y * d1.y; ys[6] = y1.z * d1.z; ys[7] = y1.w * d1.w;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int l = 8 * ph + u;
              const float4 a0 = *reinterpret_cast<const float4*>(&S.Yy[l][0]);
              const float4 a1 = *reinterpret_cast<const float4*>(&S.Yy[l][4]);
              float acc = S.P[pi][l];
              acc = fmaf(-ys[0], a0.x, acc);
              acc = fmaf(-ys[1], a0.y, acc);
              acc = fmaf(-ys[2], a0.z, acc);
              acc = fmaf(-ys[3], a0.w, acc);
              acc = fmaf(-ys[4], a1.x, acc);
              acc = fmaf(-ys[5], a1.y, acc);
              acc = fmaf(-ys[6], a1.z, acc);
              acc = fmaf(-ys[7], a1.w, acc);
              S.P[pi][l] = acc;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int c = 4 * ph + u;
              const float4 h0 = *reinterpret_cast<const float4*>(&S.DhT[c][0]);
              const float4 h1 = *reinterpret_cast<const float4*>(&S.DhT[c][4]);
              float acc = S.Wt[c][pi];
              acc = fmaf(yi[0], h0.x, acc);
              acc = fmaf(yi[1], h0.y, acc);
              acc = fmaf(yi[2], h0.z, acc);
              acc = fmaf(yi[3], h0.w, acc);
              acc = fmaf(yi[4], h1.x, acc);
              acc = fmaf(yi[5], h1.y, acc);
              acc = fmaf(yi[6], h1.z, acc);
              acc = fmaf(yi[7], h1.w, acc);
              S.Wt[c][pi] = acc;
            }
          }
          if (lane < TT && lane >= rs && lane < te) {
            const int64_t row = b * T + t0 + lane;
            if (blog) blog[row] = 0;
            if (LOGC)
              for (int i = 0; i < rc; ++i) clog[row * rc + i] = i < R && i < r ? S.G[lane][i] : 0.f;
          }
          __syncwarp();
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
        // ---- independent row tstar: general _grow (solver.py:368-379) ------------------
        {
          const int ts = tstar;
          const float rsq = S.sums[0][ts];
          float ats0 = 0.f, ats1 = 0.f;
#pragma unroll
          for (int t = 0; t < TT; ++t)
            if (t == ts) {
              ats0 = a[t][0];
              ats1 = a[t][1];
            }
          // its rejection on my columns, exactly as in the R pass above
          float s0 = 0.f, s1 = 0.f;
#pragma unroll
          for (int i4 = 0; i4 < R; i4 += 4) {
            const float4 gq = *reinterpret_cast<const float4*>(&S.G[ts][i4]);
            s0 = fmaf(gq.x, Ct[i4][0], s0);
            s1 = fmaf(gq.x, Ct[i4][1], s1);
            s0 = fmaf(gq.y, Ct[i4 + 1][0], s0);
            s1 = fmaf(gq.y, Ct[i4 + 1][1], s1);
            s0 = fmaf(gq.z, Ct[i4 + 2][0], s0);
            s1 = fmaf(gq.z, Ct[i4 + 2][1], s1);
            s0 = fmaf(gq.w, Ct[i4 + 3][0], s0);
            s1 = fmaf(gq.w, Ct[i4 + 3][1], s1);
          }
          const float K0 = (ats0 - s0) / rsq, K1 = (ats1 - s1) / rsq;  // K = rej / |rej|^2
          S.Kv[j0] = K0;
          S.Kv[j1] = K1;
#pragma unroll
          for (int i = 0; i < R; ++i)
            if (i == r) {
              Ct[i][0] = ats0;  // C[r] = a
              Ct[i][1] = ats1;
            }
          __syncwarp();
          {  // C~[:r] -= gamma K^T, C~[r] = K on my fragment rows fg, fg + 8
            const float gi0 = S.G[ts][fg], gi1 = S.G[ts][fg + 8];
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
              const float2 kq = *reinterpret_cast<const float2*>(&S.Kv[8 * kk + 2 * fq]);
              if (fg < r) {
                Dm[kk][0] = fmaf(-gi0, kq.x, Dm[kk][0]);
                Dm[kk][2] = fmaf(-gi0, kq.y, Dm[kk][2]);
              } else if (fg == r) {
                Dm[kk][0] = kq.x;
                Dm[kk][2] = kq.y;
              }
              if (fg + 8 < r) {
                Dm[kk][1] = fmaf(-gi1, kq.x, Dm[kk][1]);
                Dm[kk][3] = fmaf(-gi1, kq.y, Dm[kk][3]);
              } else if (fg + 8 == r) {
                Dm[kk][1] = kq.x;
                Dm[kk][3] = kq.y;
              }
            }
          }
          __syncwarp();
          if (lane == 0) S.P[r][r] = 1.f;  // P = diag(P, 1): row / column r were zero
          if (lane < k) S.Wt[lane][r] = S.Y[s][ts][lane] - S.G[ts][16 + lane];  // W[r] = y - a.x0
          if (lane == 0) {
            const int64_t row = b * T + t0 + ts;
            if (blog) blog[row] = 1;
            if (LOGC)
              for (int i = 0; i < rc; ++i) clog[row * rc + i] = i == r ? 1.f : 0.f;
          }
          __syncwarp();
          r += 1;
        }
        row_start = tstar + 1;
        if (row_start >= tv) break;
      }
      if (!stopped) consumed = t0 + tv;
      __syncwarp();
    }
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncwarp();

    // ---- write back C~, C, P^-1; x = x0 + C~^T W ---------------------------------------
    // (C~ is staged in the tile ring so that column owners can form x)
    float* Dsm = &S.A[0][0][0];  // 16 x 64 floats within the two tile slots
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const float2 v0 = make_float2(Dm[kk][0], Dm[kk][2]), v1 = make_float2(Dm[kk][1], Dm[kk][3]);
      *reinterpret_cast<float2*>(Dsm + fg * M + 8 * kk + 2 * fq) = v0;
      *reinterpret_cast<float2*>(Dsm + (fg + 8) * M + 8 * kk + 2 * fq) = v1;
      if (fg < rc) *reinterpret_cast<float2*>(Dg + fg * M + 8 * kk + 2 * fq) = v0;
      if (fg + 8 < rc) *reinterpret_cast<float2*>(Dg + (fg + 8) * M + 8 * kk + 2 * fq) = v1;
    }
#pragma unroll
    for (int i = 0; i < R; ++i)
      if (i < rc) {
        Cg[i * M + j0] = Ct[i][0];
        Cg[i * M + j1] = Ct[i][1];
      }
    for (int e = lane; e < R * R; e += 32) {
      const int i = e >> 4, l = e & 15;
      if (i < rc && l < rc) Pg[i * rc + l] = S.P[i][l];
    }
    __syncwarp();
#pragma unroll
    for (int c = 0; c < KX; ++c) {
      if (c >= k) break;
      float x0 = S.X0[c][j0], x1 = S.X0[c][j1];
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const float w = S.Wt[c][i];
        x0 = fmaf(Dsm[i * M + j0], w, x0);
        x1 = fmaf(Dsm[i * M + j1], w, x1);
      }
      Xg[c * M + j0] = x0;
      Xg[c * M + j1] = x1;
    }
    if (lane == 0) {
      st.rank[b] = r;
      st.nobs[b] = nobs0 + consumed;
      st.status[b] = status;
    }
    __syncwarp();
  }
}

}  // namespace f32k

// m 64, rank capacity 16, k <= 8, general variant, float32 state and inputs,
// no residual / gain logs (those run on the shape-generic kernel)
bool f32_supports(const rgb_config& cfg) {
  return cfg.dtype == RGB_F32 && cfg.variant == RGB_GENERAL && cfg.m == f32k::M && cfg.r_cap == f32k::R &&
         cfg.k >= 1 && cfg.k <= f32k::KX;
}

int launch_f32(const rgb_config& cfg, rgb_state& st, const void* rows, int64_t rows_stride, const void* targets,
               int64_t tg_stride, int64_t T, const rgb_logs& logs, cudaStream_t stream, int num_sms) {
  // 16-byte tile copies: every stream's rows must start 16-byte aligned
  if ((reinterpret_cast<uintptr_t>(rows) & 15) || (rows_stride & 3)) return RGB_E_UNSUPPORTED;
  const size_t smem = sizeof(f32k::WarpSmem) * f32k::WARPS;
  auto kern = logs.coords ? f32k::f32_kernel<true> : f32k::f32_kernel<false>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, f32k::NT, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t need = (cfg.num_streams + f32k::WARPS - 1) / f32k::WARPS;
  int64_t grid = (int64_t)num_sms * per_sm;
  if (grid > need) grid = need;
  if (grid < 1) return RGB_OK;
  kern<<<(unsigned)grid, f32k::NT, smem, stream>>>(cfg, st, (const float*)rows, rows_stride, (const float*)targets,
                                                    tg_stride, T, logs.branch, (float*)logs.coords);
  return cudaGetLastError() == cudaSuccess ? RGB_OK : RGB_E_CUDA;
}

}  // namespace rgb
