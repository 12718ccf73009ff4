// Fused full-resolution guided filter forward (gf/guided.py:198-233) for fp32
// NCHW on sm_100a: ONE kernel reads guide and src once and writes out once.
//
// Work item = (plane, column strip of TX output columns, row segment of TY
// output rows).  A CTA streams its segment top to bottom in batches of R
// coefficient rows.  Two kinds of work alternate, separated by the only two
// CTA barriers of a batch:
//
//   column phase X(k)   one thread per column, every thread busy
//     V1(k)    vertical running window sums of g, g^2, s, g*s for batch k
//              (entering rows from the TMA-staged rows, leaving rows re-read
//              from L2)                                          -> smem vs
//     V2(k-1)  vertical running sums of the coefficient rows A, b of batch
//              k-1 (entering rows and the leaving rows of batch k are read
//              from the coefficient ring before H1(k) overwrites them) -> vs2
//   run phase Y(k)      one thread per (row, run of K columns)
//     H1(k)    horizontal window sums of the 4 fields streamed over a run of
//              K=16 columns, A = cov/(var+eps), b = mean_s - A mean_g
//                                                        -> coefficient ring
//     H2(k-1)  horizontal sums of A, b streamed over a run, out = Ah*G + bh,
//              128-bit loads of G and stores of out
//
// The TMA load of the next batch's entering rows (cp.async.bulk.tensor,
// zero-filled outside the image) is issued at the start of Y(k) and lands
// while Y(k) computes.  Run-phase reads are 128-bit and conflict free: the 8
// lanes of a quarter warp are 8 rows of one run and every row pitch is 4 mod
// 32 words; column-phase accesses are consecutive words.
//
// Windows are clamped to the image and normalised by the true count
// N = ny*nx (gf/filters.py:82-103): out-of-image rows/columns contribute 0.
// g and s are shifted by a per-CTA constant (var/cov are shift invariant) to
// keep the fp32 sums small; running sums restart for every segment, so their
// rounding error is bounded by the segment length, not the image size.
#include <cuda_runtime.h>

#include "gf_common.cuh"
#include "gf_internal.h"
#include "gf_tma.cuh"

namespace gfb {
namespace hrf {

constexpr int R = 8;     // coefficient rows per batch (= lanes per run group)
constexpr int TX = 256;  // output columns per work item
constexpr int K = 16;    // run length of H1 and H2
constexpr int kMaxRadius = 16;

__host__ __device__ constexpr int up4(int n) { return (n + 3) / 4 * 4; }
// smallest p >= n with p = 4 (mod 32)
__host__ __device__ constexpr int pitch4(int n) { return n + ((36 - n % 32) % 32); }
__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }
__host__ __device__ constexpr int cdiv(int a, int b) { return (a + b - 1) / b; }

template <int RAD>
struct Geo {
  static constexpr int W2 = TX + 2 * RAD;  // coefficient columns
  static constexpr int nq1 = cdiv(W2, K);  // H1 runs per row
  static constexpr int nq2 = TX / K;       // H2 runs per row
  static constexpr int RW = nq1 * K;       // ring row width (>= W2)
  // vs column c <-> image column x0 - PADL + c (16-byte aligned TMA boxes); the
  // window of coefficient column a starts at vs column a + off
  static constexpr int PADL = up4(2 * RAD);
  static constexpr int off = PADL - 2 * RAD;  // 0 or 2
  static constexpr int VW = up4(cmax(TX + 2 * PADL, RW + PADL));  // V1 columns
  static constexpr int P1 = pitch4(VW);
  static constexpr int ringN = cmax(2 * RAD + 1, R);
  static constexpr int Pr = pitch4(RW);
  static constexpr int P2 = pitch4(W2);
  static constexpr int h1w = cdiv(nq1, 4);  // warps of H1 (4 runs x 8 rows each)
  static constexpr int h2w = nq2 / 4;       // warps of H2
  static constexpr int nt = 32 * cmax(cdiv(cmax(VW, W2), 32), h1w + h2w);
  // TMA boxes of the staged rows: NB boxes of BX columns (box dims <= 256)
  static constexpr int NB = cdiv(VW, 256);
  static constexpr int BX = up4(cdiv(VW, NB));
  static constexpr int SWF = NB * BX;  // staged columns per field (>= VW)
  static constexpr size_t smem_floats = (size_t)2 * R * SWF + (size_t)4 * R * P1 +
                                        (size_t)2 * ringN * Pr + (size_t)2 * R * P2 + 4;
  static constexpr size_t smem_bytes = smem_floats * sizeof(float);
  static constexpr uint32_t tx_bytes = 2u * NB * R * BX * 4u;
  static constexpr int min_blocks = smem_bytes <= 112 * 1024 ? 2 : 1;
  // float4 window chunks at offset 2r from an aligned run start are aligned
  // when 2r = 0 mod 4 (else two 8-byte halves)
  static constexpr bool A4 = (2 * RAD) % 4 == 0;
};

__device__ __forceinline__ float4 lds4(const float* p) {
  return *reinterpret_cast<const float4*>(p);
}
template <bool A4>
__device__ __forceinline__ float4 lds4u(const float* p) {
  if constexpr (A4) {
    return *reinterpret_cast<const float4*>(p);
  } else {  // 8-byte aligned
    const float2 a = *reinterpret_cast<const float2*>(p);
    const float2 b = *reinterpret_cast<const float2*>(p + 2);
    return make_float4(a.x, a.y, b.x, b.y);
  }
}
__device__ __forceinline__ void sts4(float* p, float a, float b, float c, float d) {
  *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
}

// sum of p[0 .. N-1], N even; p 16-byte aligned, or 8-byte aligned with
// (N - 2) = 0 mod 4 when HEAD2
template <int N, bool HEAD2 = false>
__device__ __forceinline__ float window_sum(const float* p) {
  float acc = 0.f;
  if constexpr (HEAD2) {
    const float2 v = *reinterpret_cast<const float2*>(p);
    acc += v.x;
    acc += v.y;
#pragma unroll
    for (int c = 2; c + 4 <= N; c += 4) {
      const float4 w = lds4(p + c);
      acc += w.x;
      acc += w.y;
      acc += w.z;
      acc += w.w;
    }
    return acc;
  }
#pragma unroll
  for (int c = 0; c + 4 <= N; c += 4) {
    const float4 v = lds4(p + c);
    acc += v.x;
    acc += v.y;
    acc += v.z;
    acc += v.w;
  }
  if constexpr (N % 4 == 2) {
    const float2 v = *reinterpret_cast<const float2*>(p + (N / 4) * 4);
    acc += v.x;
    acc += v.y;
  }
  return acc;
}

struct Args {
  const float* guide;
  const float* src;
  float* out;
  int64_t C, Cg, H, W;
  int TY, strips, segs;
  float eps;
  uint32_t* status;
};

__device__ __forceinline__ int wlen(int i, int n, int r) {
  int a = i - r < 0 ? 0 : i - r;
  int b = i + r > n - 1 ? n - 1 : i + r;
  return b - a + 1;
}

template <int RAD>
__global__ void __launch_bounds__(Geo<RAD>::nt, Geo<RAD>::min_blocks)
    k_highres_fused(const __grid_constant__ CUtensorMap tmG,
                    const __grid_constant__ CUtensorMap tmS, Args a) {
  using GG = Geo<RAD>;
  constexpr int r = RAD;
  constexpr int ringN = GG::ringN;
  extern __shared__ __align__(128) float4 smem4[];
  float* stg = reinterpret_cast<float*>(smem4);  // [2 fields][NB][R][BX] (TMA boxes)
  float* vs = stg + 2 * R * GG::SWF;             // [4 fields][R][P1]
  float* ring = vs + 4 * R * GG::P1;             // [2 fields][ringN][Pr]
  float* vs2 = ring + 2 * ringN * GG::Pr;        // [2 fields][R][P2]
  uint64_t* bar = reinterpret_cast<uint64_t*>(vs2 + 2 * R * GG::P2);
  const int H = (int)a.H, W = (int)a.W;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // work item: plane fastest (the C planes sharing a guide run together)
  int64_t item = blockIdx.x;
  const int c = (int)(item % a.C);
  item /= a.C;
  const int strip = (int)(item % a.strips);
  item /= a.strips;
  const int seg = (int)(item % a.segs);
  const int64_t b = item / a.segs;
  const int x0 = strip * TX;
  const int y0 = seg * a.TY;
  if (y0 >= H) return;
  const int yend = min(y0 + a.TY, H);
  const int64_t plane = (int64_t)H * W;
  const int64_t gplane = a.Cg == a.C ? b * a.C + c : b * a.Cg;
  const float* __restrict__ G = a.guide + gplane * plane;
  const float* __restrict__ S = a.src + (b * a.C + c) * plane;
  float* __restrict__ O = a.out + (b * a.C + c) * plane;
  const float sG = __ldg(G + (int64_t)y0 * W + x0);
  const float sS = __ldg(S + (int64_t)y0 * W + x0);
  const float eps = a.eps;
  constexpr float inv_full = 1.0f / (float)(2 * r + 1);

  const int ya0 = y0 - r;                 // image row of coefficient row 0
  const int nrows = (yend - y0) + 2 * r;  // coefficient rows of this item
  const int nb = (nrows + R - 1) / R;     // batches
  const int first_add = y0 - 2 * r;       // first input row ever added
  const int xs0 = x0 - GG::PADL;          // image column of vs / stg column 0

  if (tid == 0) tma::mbar_init(bar, 1);
  __syncthreads();
  uint32_t phase = 0;
  // TMA of the R entering input rows of batch k (image rows ya0 + kR + r ...)
  auto prefetch = [&](int k) {
    if (tid == 0) {
      tma::fence_proxy_async();
      tma::mbar_arrive_expect_tx(bar, GG::tx_bytes);
      const int e0 = ya0 + k * R + r;
#pragma unroll
      for (int box = 0; box < GG::NB; ++box) {
        tma::load_3d(stg + (0 * GG::NB + box) * R * GG::BX, &tmG, xs0 + box * GG::BX, e0,
                     (int)gplane, bar);
        tma::load_3d(stg + (1 * GG::NB + box) * R * GG::BX, &tmS, xs0 + box * GG::BX, e0,
                     (int)(b * a.C + c), bar);
      }
    }
  };
  prefetch(0);

  // ---- column-phase state: thread owns vs column `tid` (V1) and
  //      coefficient column `tid` (V2)
  const bool v1 = tid < GG::VW;
  const int gx = xs0 + tid;
  const bool col_ok = v1 && gx >= 0 && gx < W;
  const int sbox = tid / GG::BX;
  const float* st_g = stg + sbox * R * GG::BX + (tid - sbox * GG::BX);
  const float* st_s = st_g + GG::NB * R * GG::BX;
  float sI = 0.f, sII = 0.f, sP = 0.f, sIP = 0.f;
  if (col_ok) {
    for (int y = max(first_add, 0); y < y0; ++y) {
      const float gv = __ldg(G + (int64_t)y * W + gx) - sG;
      const float pv = __ldg(S + (int64_t)y * W + gx) - sS;
      sI += gv;
      sII = fmaf(gv, gv, sII);
      sP += pv;
      sIP = fmaf(gv, pv, sIP);
    }
  }
  const bool v2 = tid < GG::W2;
  float cA = 0.f, cB = 0.f;  // level-2 sums at the end of the last finished batch
  float pA[R], pB[R];        // running sums minus the leaving rows (pre-subtracted)
#pragma unroll
  for (int j = 0; j < R; ++j) pA[j] = pB[j] = 0.f;
  int s_cur = 0;                                      // ring slot of coefficient row kR
  int s_prev = ringN - (R % ringN);                   // ... of row (k-1)R
  if (s_prev == ringN) s_prev = 0;
  int s_old = ringN - ((2 * r + 1) % ringN);          // ... of row kR - 2r - 1
  if (s_old == ringN) s_old = 0;
  bool bad = false, degen = false;

  for (int k = 0; k <= nb; ++k) {
    const int base = k * R;
    if (k < nb) {
      tma::mbar_wait(bar, phase);  // batch k's entering rows landed in stg
      phase ^= 1u;
    }

    // ================= column phase X(k) =================================
    if (k < nb && v1) {
      float* o = vs + tid;
      const int l0 = ya0 + base - r - 1;  // leaving image row of row 0
      const bool rows_fast = base + R <= nrows && l0 >= max(first_add, 0) &&
                             ya0 + base + R - 1 + r < H;
      if (rows_fast) {
        if (col_ok) {
          float lg[R], ls[R];
          const float* gl = G + (int64_t)l0 * W + gx;
          const float* sl = S + (int64_t)l0 * W + gx;
#pragma unroll
          for (int j = 0; j < R; ++j) {
            lg[j] = __ldg(gl + (int64_t)j * W);
            ls[j] = __ldg(sl + (int64_t)j * W);
          }
#pragma unroll
          for (int j = 0; j < R; ++j) {
            const float eg = st_g[j * GG::BX] - sG, es = st_s[j * GG::BX] - sS;
            const float qg = lg[j] - sG, qs = ls[j] - sS;
            sI += eg - qg;
            sII = fmaf(eg, eg, sII);
            sII = fmaf(-qg, qg, sII);
            sP += es - qs;
            sIP = fmaf(eg, es, sIP);
            sIP = fmaf(-qg, qs, sIP);
            o[(0 * R + j) * GG::P1] = sI;
            o[(1 * R + j) * GG::P1] = sII;
            o[(2 * R + j) * GG::P1] = sP;
            o[(3 * R + j) * GG::P1] = sIP;
          }
        } else {
#pragma unroll
          for (int j = 0; j < R; ++j) {
            o[(0 * R + j) * GG::P1] = 0.f;
            o[(1 * R + j) * GG::P1] = 0.f;
            o[(2 * R + j) * GG::P1] = 0.f;
            o[(3 * R + j) * GG::P1] = 0.f;
          }
        }
      } else {  // top / bottom batches: per-row predicates
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const int i = base + j;
          const int e = ya0 + i + r, l = e - 2 * r - 1;
          const bool in_i = i < nrows;
          const bool e_ok = col_ok && in_i && e >= 0 && e < H;
          const bool l_ok = col_ok && in_i && l >= first_add && l >= 0 && l < H;
          float eg = 0.f, es = 0.f, qg = 0.f, qs = 0.f;
          if (e_ok) {
            eg = st_g[j * GG::BX] - sG;
            es = st_s[j * GG::BX] - sS;
          }
          if (l_ok) {
            qg = __ldg(G + (int64_t)l * W + gx) - sG;
            qs = __ldg(S + (int64_t)l * W + gx) - sS;
          }
          sI += eg - qg;
          sII = fmaf(eg, eg, sII);
          sII = fmaf(-qg, qg, sII);
          sP += es - qs;
          sIP = fmaf(eg, es, sIP);
          sIP = fmaf(-qg, qs, sIP);
          o[(0 * R + j) * GG::P1] = sI;
          o[(1 * R + j) * GG::P1] = sII;
          o[(2 * R + j) * GG::P1] = sP;
          o[(3 * R + j) * GG::P1] = sIP;
        }
      }
    }
    if (v2) {
      const float* rA = ring + tid;
      const float* rB = ring + ringN * GG::Pr + tid;
      if (k >= 1) {  // V2(k-1): add batch k-1's coefficient rows -> vs2
        const int bb = base - R;
        float nA = 0.f, nB = 0.f;
#pragma unroll
        for (int j = 0; j < R; ++j) {
          if (bb + j < nrows) {
            int s = s_prev + j;
            if (s >= ringN) s -= ringN;
            nA += rA[s * GG::Pr];
            nB += rB[s * GG::Pr];
            if (j >= 2 * r + 1) {  // leaving row inside this batch (small r)
              int so = s - (2 * r + 1);
              if (so < 0) so += ringN;
              nA -= rA[so * GG::Pr];
              nB -= rB[so * GG::Pr];
            }
          }
          vs2[j * GG::P2 + tid] = pA[j] + nA;
          vs2[(R + j) * GG::P2 + tid] = pB[j] + nB;
        }
        cA = pA[R - 1] + nA;
        cB = pB[R - 1] + nB;
      }
      if (k < nb) {  // pre-subtract batch k's leaving rows before H1(k) overwrites them
        float qa = cA, qb = cB;
#pragma unroll
        for (int j = 0; j < R; ++j) {
          if (j < 2 * r + 1 && base + j - 2 * r - 1 >= 0) {
            int so = s_old + j;
            if (so >= ringN) so -= ringN;
            qa -= rA[so * GG::Pr];
            qb -= rB[so * GG::Pr];
          }
          pA[j] = qa;
          pB[j] = qb;
        }
      }
    }
    __syncthreads();  // vs, vs2 complete; stg and the leaving ring rows consumed

    // ================= run phase Y(k) ====================================
    if (k + 1 < nb) prefetch(k + 1);
    const int j = lane & 7;
    if (warp < GG::h1w) {
      // ---- H1(k): coefficient row base+j, columns [qK, qK+K) ---------------
      const int q = warp * 4 + (lane >> 3);
      const int i = base + j;
      if (k < nb && q < GG::nq1 && i < nrows) {
        const int ya = ya0 + i;
        int s = s_cur + j;
        if (s >= ringN) s -= ringN;
        float* ra = ring + s * GG::Pr + q * K;
        float* rb = ring + (ringN + s) * GG::Pr + q * K;
        if (ya < 0 || ya >= H) {
#pragma unroll
          for (int m = 0; m < K / 4; ++m) {
            sts4(ra + 4 * m, 0.f, 0.f, 0.f, 0.f);
            sts4(rb + 4 * m, 0.f, 0.f, 0.f, 0.f);
          }
        } else {
          const float* v = vs + j * GG::P1 + q * K + GG::off;  // field f at + f*R*P1
          float acc[4];
#pragma unroll
          for (int f = 0; f < 4; ++f)
            acc[f] = window_sum<2 * r, GG::off != 0>(v + f * R * GG::P1);
          const float iny = fast_rcp((float)wlen(ya, H, r));
          const int gxa0 = x0 - r + q * K;  // image column of the run's first coefficient
          const bool interior = gxa0 >= r && gxa0 + K - 1 + r <= W - 1 && q * K + K <= GG::W2;
          const float inv_i = iny * inv_full;
#pragma unroll
          for (int m = 0; m < K / 4; ++m) {
            float h[4][4];
#pragma unroll
            for (int f = 0; f < 4; ++f) {
              const float* vf = v + f * R * GG::P1 + 4 * m;
              const float4 e = lds4(vf + 2 * r);            // vs column q*K + PADL + 4m
              const float4 l = lds4u<GG::off == 0>(vf);
              acc[f] += e.x; h[f][0] = acc[f]; acc[f] -= l.x;
              acc[f] += e.y; h[f][1] = acc[f]; acc[f] -= l.y;
              acc[f] += e.z; h[f][2] = acc[f]; acc[f] -= l.z;
              acc[f] += e.w; h[f][3] = acc[f]; acc[f] -= l.w;
            }
            float A[4], B[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const int gxa = gxa0 + 4 * m + t;
              const bool ok = interior || (q * K + 4 * m + t < GG::W2 && gxa >= 0 && gxa < W);
              const float inv = interior ? inv_i : iny * fast_rcp((float)wlen(gxa, W, r));
              const float mg = h[0][t] * inv, ms = h[2][t] * inv;
              const float var = fmaf(h[1][t], inv, -mg * mg);
              const float cov = fmaf(h[3][t], inv, -mg * ms);
              if (ok && eps == 0.f && !(var > 0.f)) degen = true;
              const float At = cov * fast_rcp(var + eps);
              A[t] = ok ? At : 0.f;
              B[t] = ok ? fmaf(-At, mg + sG, ms + sS) : 0.f;
            }
            sts4(ra + 4 * m, A[0], A[1], A[2], A[3]);
            sts4(rb + 4 * m, B[0], B[1], B[2], B[3]);
          }
        }
      }
    } else if (warp < GG::h1w + GG::h2w) {
      // ---- H2(k-1): output row of coefficient row base-R+j, columns [qK, qK+K)
      const int q = (warp - GG::h1w) * 4 + (lane >> 3);
      const int yo = y0 - 2 * r + base - R + j;
      const int gxo0 = x0 + q * K;
      if (k >= 1 && yo >= y0 && yo < yend && gxo0 < W) {
        const float* vA = vs2 + j * GG::P2 + q * K;
        const float* vB = vs2 + (R + j) * GG::P2 + q * K;
        float accA = window_sum<2 * r>(vA), accB = window_sum<2 * r>(vB);
        const float iny = fast_rcp((float)wlen(yo, H, r));
        const bool interior = gxo0 >= r && gxo0 + K - 1 + r <= W - 1;
        const float inv_i = iny * inv_full;
        const float* grow = G + (int64_t)yo * W + gxo0;
        float* orow = O + (int64_t)yo * W + gxo0;
#pragma unroll
        for (int m = 0; m < K / 4; ++m) {
          if (gxo0 + 4 * m >= W) break;  // W % 4 == 0: a float4 is all in or all out
          const float4 g4 = __ldg(reinterpret_cast<const float4*>(grow + 4 * m));
          const float4 eA = lds4u<GG::A4>(vA + 4 * m + 2 * r), lA = lds4(vA + 4 * m);
          const float4 eB = lds4u<GG::A4>(vB + 4 * m + 2 * r), lB = lds4(vB + 4 * m);
          float hA[4], hB[4];
          accA += eA.x; hA[0] = accA; accA -= lA.x;
          accA += eA.y; hA[1] = accA; accA -= lA.y;
          accA += eA.z; hA[2] = accA; accA -= lA.z;
          accA += eA.w; hA[3] = accA; accA -= lA.w;
          accB += eB.x; hB[0] = accB; accB -= lB.x;
          accB += eB.y; hB[1] = accB; accB -= lB.y;
          accB += eB.z; hB[2] = accB; accB -= lB.z;
          accB += eB.w; hB[3] = accB; accB -= lB.w;
          const float gv[4] = {g4.x, g4.y, g4.z, g4.w};
          float ov[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const float inv =
                interior ? inv_i : iny * fast_rcp((float)wlen(gxo0 + 4 * m + t, W, r));
            ov[t] = fmaf(hA[t], gv[t], hB[t]) * inv;
            if (!isfinite(ov[t])) bad = true;
          }
          *reinterpret_cast<float4*>(orow + 4 * m) = make_float4(ov[0], ov[1], ov[2], ov[3]);
        }
      }
    }
    s_prev = s_cur;
    s_cur += R;
    if (s_cur >= ringN) s_cur -= ringN;
    s_old += R;
    if (s_old >= ringN) s_old -= ringN;
    __syncthreads();  // ring rows of batch k and the outputs of batch k-1 done
  }
  // Non-finite inputs are not tested per element here: they always poison
  // the output at their own pixel, so the host (gf_check_finite) classifies
  // an OUTPUT flag as an input error when the inputs are non-finite.
  if (degen) flag(a.status, GF_STATUS_DEGENERATE);
  if (bad) flag(a.status, GF_STATUS_NONFINITE_OUTPUT);
}

struct Launch {
  const void* fn;
  int nt;
  size_t smem;
  int box_w;  // TMA box width of the staged rows
};

template <int RAD>
Launch launch_info() {
  return {(const void*)k_highres_fused<RAD>, Geo<RAD>::nt, Geo<RAD>::smem_bytes, Geo<RAD>::BX};
}

Launch pick(int r) {
  switch (r) {
    case 1: return launch_info<1>();
    case 2: return launch_info<2>();
    case 3: return launch_info<3>();
    case 4: return launch_info<4>();
    case 5: return launch_info<5>();
    case 6: return launch_info<6>();
    case 7: return launch_info<7>();
    case 8: return launch_info<8>();
    case 9: return launch_info<9>();
    case 10: return launch_info<10>();
    case 11: return launch_info<11>();
    case 12: return launch_info<12>();
    case 13: return launch_info<13>();
    case 14: return launch_info<14>();
    case 15: return launch_info<15>();
    case 16: return launch_info<16>();
    default: return {nullptr, 0, 0, 0};
  }
}

}  // namespace hrf

bool fused_highres_fwd_ok(int64_t B, int64_t Cg, int64_t C, int64_t H, int64_t W, int r) {
  if (r < 1 || r > hrf::kMaxRadius) return false;
  if (W % 4 != 0 || W < 4 || H < 1) return false;
  if (H > (1 << 30) || W > (1 << 30) || H * W > ((int64_t)1 << 40)) return false;
  if (B * C > (1 << 30)) return false;  // TMA plane coordinate is a 32-bit int
  if (Cg != 1 && Cg != C) return false;
  if (hrf::pick(r).smem > 227 * 1024) return false;
  return B >= 1 && C >= 1;
}

void fused_highres_fwd(const float* guide, const float* src, float* out, int64_t B, int64_t Cg,
                       int64_t C, int64_t H, int64_t W, int r, float eps, uint32_t* status,
                       cudaStream_t s) {
  const hrf::Launch L = hrf::pick(r);
  // per-radius launch configuration, cached (the queries cost microseconds)
  static int per_sm_cache[hrf::kMaxRadius + 1] = {0};
  static int sms = 0;
  if (per_sm_cache[r] == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(L.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, L.fn, L.nt, L.smem);
    per_sm_cache[r] = per_sm < 1 ? 1 : per_sm;
  }
  const int64_t strips = (W + hrf::TX - 1) / hrf::TX;
  const int64_t planes = B * C;
  const int64_t slots = (int64_t)sms * per_sm_cache[r];
  // choose the row segmentation: minimise waves x (rows per item incl. the
  // 4r warm-up rows), with segments of at most 1024 rows (bounded rounding)
  int64_t best_segs = 1;
  double best_cost = 1e300;
  const int64_t max_segs = H / (2 * r + 1) > 0 ? H / (2 * r + 1) : 1;
  for (int64_t sg = (H + 1023) / 1024; sg <= max_segs && sg <= 4096; ++sg) {
    const int64_t ty = (H + sg - 1) / sg;
    const int64_t items = planes * strips * ((H + ty - 1) / ty);
    const int64_t waves = (items + slots - 1) / slots;
    const double cost = (double)waves * (double)(ty + 4 * r);
    if (cost < best_cost * 0.999) {
      best_cost = cost;
      best_segs = sg;
    }
  }
  const int64_t TY = (H + best_segs - 1) / best_segs;
  const int64_t segs = (H + TY - 1) / TY;
  hrf::Args a{guide, src, out, C, Cg, H, W, (int)TY, (int)strips, (int)segs, eps, status};
  const int64_t grid = planes * strips * segs;
  CUtensorMap tmG, tmS;
  if (!tma::make_plane_map(&tmG, guide, W, H, B * Cg, L.box_w, hrf::R) ||
      !tma::make_plane_map(&tmS, src, W, H, B * C, L.box_w, hrf::R)) {
    // surfaces as a launch error through the C ABI's cudaGetLastError check
    cudaLaunchKernel(L.fn, dim3(0), dim3(0), nullptr, 0, s);
    return;
  }
  void* args[] = {&tmG, &tmS, &a};
  cudaLaunchKernel(L.fn, dim3((unsigned)grid), dim3(L.nt), args, L.smem, s);
}

}  // namespace gfb
