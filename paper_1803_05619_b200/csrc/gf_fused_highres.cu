// Fused full-resolution guided filter forward (gf/guided.py:198-233) for fp32
// NCHW on sm_100a: ONE kernel reads guide and src once and writes out once.
//
// Work item = (plane, column strip of TX output columns, row segment of TY
// output rows).  A CTA walks its segment top to bottom in batches of R rows
// and keeps every intermediate on chip:
//
//   stage  the batch's R entering input rows stream into shared memory with
//          cp.async one batch ahead (zero-filled outside the image)
//   V1     vertical running window sums of g, g^2, s, g*s, four columns per
//          thread (the rows leaving the window are re-read from L2 with
//          128-bit loads)                                         -> smem vs
//   H1     horizontal window sums (runs of 8 columns), window means, var,
//          cov, A = cov/(var+eps), b = mean_s - A*mean_g           -> smem ring
//   V2     vertical running sums of A and b over the ring of the last
//          max(2r+1, R) coefficient rows, four columns per thread; the
//          leaving rows are subtracted before H1 overwrites them  -> smem vs2
//   H2     horizontal sums (runs of 8), Ah = M(A), bh = M(b), out = Ah*G + bh
//          with 128-bit loads of G and 128-bit stores of out.
//
// Every shared row is 16-byte aligned with a pitch = 4 (mod 32) words: the
// 8 lanes of a quarter warp (8 rows of one run) then read 8 distinct bank
// quads with 128-bit loads.  The radius is a template parameter (1..16) so
// every window loop is unrolled; runs that lie inside the image use the
// constant 1/(2r+1) column normaliser.
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

constexpr int R = 8;     // rows per batch
constexpr int TX = 256;  // output columns per work item
constexpr int KR = 8;    // run length of H1 and H2
constexpr int kMaxRadius = 16;

__host__ __device__ constexpr int up4(int n) { return (n + 3) / 4 * 4; }
// smallest p >= n with p = 4 (mod 32)
__host__ __device__ constexpr int pitch4(int n) { return n + ((36 - n % 32) % 32); }
__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }

template <int RAD>
struct Geo {
  static constexpr int W2 = TX + 2 * RAD;                 // coefficient columns
  static constexpr int nq1 = (W2 + KR - 1) / KR;          // H1 runs per row
  static constexpr int PADL = up4(2 * RAD);               // staged columns left of x0
  static constexpr int off = PADL - 2 * RAD;              // vs col of a window start
  static constexpr int nv1 = (off + 2 * RAD + KR + 3) / 4;  // float4s per H1 run window
  static constexpr int VW = up4(cmax(TX + 2 * PADL, (nq1 - 1) * KR + 4 * nv1));  // V1 columns
  static constexpr int P1 = pitch4(VW);
  static constexpr int ringN = cmax(2 * RAD + 1, R);
  static constexpr int ringw = nq1 * KR;                  // >= W2
  static constexpr int Pr = pitch4(ringw);
  static constexpr int nv2 = (2 * RAD + KR + 3) / 4;      // float4s per H2 run window
  static constexpr int v2w = up4(cmax(ringw, TX - KR + 4 * nv2));
  static constexpr int P2 = pitch4(v2w);
  static constexpr int nt = 32 * cmax(cmax((nq1 + 3) / 4, TX / KR / 4),
                                      cmax((VW / 2 + 31) / 32, (v2w / 2 + 31) / 32));
  // TMA boxes of the staged rows: NB boxes of BX columns (box dims <= 256)
  static constexpr int NB = (VW + 255) / 256;
  static constexpr int BX = up4((VW + NB - 1) / NB);
  static constexpr int SWF = NB * BX;  // staged columns per field (>= VW)
  static constexpr size_t smem_floats = (size_t)2 * R * SWF + (size_t)4 * R * P1 +
                                        (size_t)2 * ringN * Pr + (size_t)2 * R * P2 + 4;
  static constexpr size_t smem_bytes = smem_floats * sizeof(float);
  static constexpr uint32_t tx_bytes = 2u * NB * R * BX * 4u;
};

__device__ __forceinline__ void cp_async16(float* dst, const float* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const int n = valid ? 16 : 0;  // 0 -> zero fill, nothing read
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n"); }

__device__ __forceinline__ float4 lds4(const float* p) {
  return *reinterpret_cast<const float4*>(p);
}
__device__ __forceinline__ void sts4(float* p, float a, float b, float c, float d) {
  *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
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

// staged column c of row j of field f: boxes of BX columns, dense rows
template <typename GG>
__device__ __forceinline__ int stg_idx(int f, int j, int c) {
  const int box = c / GG::BX;
  return ((f * GG::NB + box) * R + j) * GG::BX + (c - box * GG::BX);
}

template <int RAD>
__global__ void __launch_bounds__(320, 2)
    k_highres_fused(const __grid_constant__ CUtensorMap tmG,
                    const __grid_constant__ CUtensorMap tmS, Args a) {
  using GG = Geo<RAD>;
  constexpr int r = RAD;
  constexpr int nt = GG::nt;
  extern __shared__ __align__(128) float4 smem4[];
  float* stg = reinterpret_cast<float*>(smem4);  // [2 fields][NB][R][BX] (TMA boxes)
  float* vs = stg + 2 * R * GG::SWF;             // [4 fields][R][P1]
  float* ring = vs + 4 * R * GG::P1;             // [2 fields][ringN][Pr]
  float* vs2 = ring + 2 * GG::ringN * GG::Pr;    // [2 fields][R][P2]
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
  const float* __restrict__ G = a.guide + (a.Cg == a.C ? b * a.C + c : b * a.Cg) * plane;
  const float* __restrict__ S = a.src + (b * a.C + c) * plane;
  float* __restrict__ O = a.out + (b * a.C + c) * plane;
  const float sG = __ldg(G + (int64_t)y0 * W + x0);
  const float sS = __ldg(S + (int64_t)y0 * W + x0);
  const float eps = a.eps;
  constexpr float inv_full = 1.0f / (float)(2 * r + 1);

  for (int i = tid; i < 2 * GG::ringN * GG::Pr; i += nt) ring[i] = 0.f;

  const int ya0 = y0 - r;                 // first coefficient row
  const int nrows = (yend - y0) + 2 * r;  // coefficient rows of this item
  const int first_add = y0 - 2 * r;       // first input row ever added
  const int xs0 = x0 - GG::PADL;          // global column of vs/stg column 0

  // TMA of the R entering input rows of the batch at bb (rows ya0+bb+r ...);
  // out-of-image box elements are zero-filled by the hardware
  const int zG = (int)(a.Cg == a.C ? b * a.C + c : b * a.Cg);
  const int zS = (int)(b * a.C + c);
  if (tid == 0) tma::mbar_init(bar, 1);
  __syncthreads();
  uint32_t phase = 0;
  auto prefetch = [&](int bb) {
    if (tid == 0) {
      tma::fence_proxy_async();
      tma::mbar_arrive_expect_tx(bar, GG::tx_bytes);
      const int e0 = ya0 + bb + r;
#pragma unroll
      for (int box = 0; box < GG::NB; ++box) {
        tma::load_3d(stg + (0 * GG::NB + box) * R * GG::BX, &tmG, xs0 + box * GG::BX, e0, zG, bar);
        tma::load_3d(stg + (1 * GG::NB + box) * R * GG::BX, &tmS, xs0 + box * GG::BX, e0, zS, bar);
      }
    }
  };
  prefetch(0);

  // ---- level-1 state: V1T threads per field group; group 0 keeps the guide
  //      sums (g, g^2), group 1 the source sums (s, g*s); thread owns vs
  //      columns 4t..4t+3 of its group
  constexpr int V1T = GG::VW / 4;
  const int grp = tid < V1T ? 0 : 1;
  const int t4 = tid - grp * V1T;
  const bool v1 = tid < 2 * V1T;
  const int gx4 = xs0 + 4 * t4;
  const bool col_ok = v1 && gx4 >= 0 && gx4 < W;  // W % 4 == 0: all 4 or none
  const bool cols_in = xs0 >= 0 && xs0 + GG::VW <= W;  // CTA-uniform
  float sA[4] = {0.f, 0.f, 0.f, 0.f}, sB[4] = {0.f, 0.f, 0.f, 0.f};
  if (col_ok) {
    for (int y = max(first_add, 0); y < min(y0, H); ++y) {
      const float4 g4 = __ldg(reinterpret_cast<const float4*>(G + (int64_t)y * W + gx4));
      const float gg[4] = {g4.x - sG, g4.y - sG, g4.z - sG, g4.w - sG};
      if (grp == 0) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          sA[k] += gg[k];
          sB[k] += gg[k] * gg[k];
        }
      } else {
        const float4 v4 = __ldg(reinterpret_cast<const float4*>(S + (int64_t)y * W + gx4));
        const float ss[4] = {v4.x - sS, v4.y - sS, v4.z - sS, v4.w - sS};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          sA[k] += ss[k];
          sB[k] += gg[k] * ss[k];
        }
      }
    }
  }
  // ---- level-2 state: V2T threads per coefficient field (A, then b); a
  //      thread owns coefficient columns 4u..4u+3 of its field
  constexpr int V2T = GG::v2w / 4;
  const int fld = tid < V2T ? 0 : 1;
  const int u4 = tid - fld * V2T;
  const bool v2 = tid < 2 * V2T;
  const bool v2ring = v2 && u4 < GG::ringw / 4;
  float c_sum[4] = {0.f, 0.f, 0.f, 0.f};
  bool bad = false, degen = false;
  int ring_new = 0;                                   // slot of coefficient row `base`
  int ring_old = GG::ringN - (2 * r + 1) % GG::ringN;  // slot of row base - 2r - 1
  if (ring_old == GG::ringN) ring_old = 0;
  const int jl = lane & 7;   // run mapping of H1/H2: row
  const int ql = lane >> 3;  //                       run within the warp's chunk

  for (int base = 0; base < nrows; base += R) {
    tma::mbar_wait(bar, phase);  // this batch's rows landed in stg
    phase ^= 1u;
    __syncthreads();  // ... and the previous batch's H2 is done with vs2

    // ---- V2 (part 1): subtract the leaving coefficient rows while their
    //      ring slots still hold them: vs2[j] = sum - sum_{i<=j} old_i
    if (v2) {
      float pc[4] = {c_sum[0], c_sum[1], c_sum[2], c_sum[3]};
      const float* rf = ring + fld * GG::ringN * GG::Pr + 4 * u4;
      float* vf = vs2 + fld * R * GG::P2 + 4 * u4;
#pragma unroll
      for (int j = 0; j < R; ++j) {
        // rows leaving for j >= 2r+1 belong to this batch: part 2 handles them
        if (j < 2 * r + 1 && v2ring && base + j - 2 * r - 1 >= 0) {
          int so = ring_old + j;
          if (so >= GG::ringN) so -= GG::ringN;
          const float4 o = lds4(rf + so * GG::Pr);
          pc[0] -= o.x; pc[1] -= o.y; pc[2] -= o.z; pc[3] -= o.w;
        }
        sts4(vf + j * GG::P2, pc[0], pc[1], pc[2], pc[3]);
      }
    }

    // ---- V1 -----------------------------------------------------------
    // uniform fast path: every row and column of the batch inside the image
    const bool fast = cols_in && base + R <= nrows && ya0 + base - r - 1 >= max(first_add, 0) &&
                      ya0 + base + R - 1 + r < H;
    if (v1 && fast) {
      // no predicates: leaving rows straight from L2, entering rows from stg
      float* out0 = vs + (2 * grp + 0) * R * GG::P1 + 4 * t4;
      float* out1 = vs + (2 * grp + 1) * R * GG::P1 + 4 * t4;
      const float* gl_p = G + (int64_t)(ya0 + base - r - 1) * W + gx4;
      const float* sl_p = S + (int64_t)(ya0 + base - r - 1) * W + gx4;
      const float* ge_p = stg + stg_idx<GG>(0, 0, 4 * t4);
      const float* se_p = stg + stg_idx<GG>(1, 0, 4 * t4);
      float4 gl[R], sl[R];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        gl[j] = __ldg(reinterpret_cast<const float4*>(gl_p + (int64_t)j * W));
        if (grp) sl[j] = __ldg(reinterpret_cast<const float4*>(sl_p + (int64_t)j * W));
      }
      if (grp == 0) {
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const float4 e = lds4(ge_p + j * GG::BX);
          const float gn[4] = {e.x - sG, e.y - sG, e.z - sG, e.w - sG};
          const float gq[4] = {gl[j].x - sG, gl[j].y - sG, gl[j].z - sG, gl[j].w - sG};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            sA[k] += gn[k] - gq[k];
            sB[k] += fmaf(gn[k], gn[k], -gq[k] * gq[k]);
          }
          sts4(out0 + j * GG::P1, sA[0], sA[1], sA[2], sA[3]);
          sts4(out1 + j * GG::P1, sB[0], sB[1], sB[2], sB[3]);
        }
      } else {
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const float4 e = lds4(ge_p + j * GG::BX);
          const float4 f = lds4(se_p + j * GG::BX);
          const float gn[4] = {e.x - sG, e.y - sG, e.z - sG, e.w - sG};
          const float sn[4] = {f.x - sS, f.y - sS, f.z - sS, f.w - sS};
          const float gq[4] = {gl[j].x - sG, gl[j].y - sG, gl[j].z - sG, gl[j].w - sG};
          const float sq[4] = {sl[j].x - sS, sl[j].y - sS, sl[j].z - sS, sl[j].w - sS};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            sA[k] += sn[k] - sq[k];
            sB[k] += fmaf(gn[k], sn[k], -gq[k] * sq[k]);
          }
          sts4(out0 + j * GG::P1, sA[0], sA[1], sA[2], sA[3]);
          sts4(out1 + j * GG::P1, sB[0], sB[1], sB[2], sB[3]);
        }
      }
    } else if (v1) {
      float* out0 = vs + (2 * grp + 0) * R * GG::P1 + 4 * t4;
      float* out1 = vs + (2 * grp + 1) * R * GG::P1 + 4 * t4;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        float4 gl[R / 2], sl[R / 2];
#pragma unroll
        for (int jj = 0; jj < R / 2; ++jj) {
          const int j = half * (R / 2) + jj;
          const int l = ya0 + base + j - r - 1;
          const bool l_ok = fast || (col_ok && base + j < nrows && l >= first_add && l >= 0 && l < H);
          gl[jj] = sl[jj] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (l_ok) {
            gl[jj] = __ldg(reinterpret_cast<const float4*>(G + (int64_t)l * W + gx4));
            if (grp) sl[jj] = __ldg(reinterpret_cast<const float4*>(S + (int64_t)l * W + gx4));
          }
        }
#pragma unroll
        for (int jj = 0; jj < R / 2; ++jj) {
          const int j = half * (R / 2) + jj;
          const float4 ge4 = lds4(stg + stg_idx<GG>(0, j, 4 * t4));
          float gn[4] = {ge4.x - sG, ge4.y - sG, ge4.z - sG, ge4.w - sG};
          float gq[4] = {gl[jj].x - sG, gl[jj].y - sG, gl[jj].z - sG, gl[jj].w - sG};
          float sn[4] = {0.f, 0.f, 0.f, 0.f}, sq[4] = {0.f, 0.f, 0.f, 0.f};
          if (grp) {
            const float4 se4 = lds4(stg + stg_idx<GG>(1, j, 4 * t4));
            sn[0] = se4.x - sS; sn[1] = se4.y - sS; sn[2] = se4.z - sS; sn[3] = se4.w - sS;
            sq[0] = sl[jj].x - sS; sq[1] = sl[jj].y - sS;
            sq[2] = sl[jj].z - sS; sq[3] = sl[jj].w - sS;
          }
          if (!fast) {  // edge batch: zero the out-of-image contributions
            const int e = ya0 + base + j + r;
            const int l = ya0 + base + j - r - 1;
            const bool e_ok = col_ok && base + j < nrows && e >= 0 && e < H;
            const bool l_ok = col_ok && base + j < nrows && l >= first_add && l >= 0 && l < H;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              gn[k] = e_ok ? gn[k] : 0.f;
              sn[k] = e_ok ? sn[k] : 0.f;
              gq[k] = l_ok ? gq[k] : 0.f;
              sq[k] = l_ok ? sq[k] : 0.f;
            }
          }
          if (grp == 0) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              sA[k] += gn[k] - gq[k];
              sB[k] += gn[k] * gn[k] - gq[k] * gq[k];
            }
          } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              sA[k] += sn[k] - sq[k];
              sB[k] += gn[k] * sn[k] - gq[k] * sq[k];
            }
          }
          const float m = col_ok ? 1.f : 0.f;
          sts4(out0 + j * GG::P1, m * sA[0], m * sA[1], m * sA[2], m * sA[3]);
          sts4(out1 + j * GG::P1, m * sB[0], m * sB[1], m * sB[2], m * sB[3]);
        }
      }
    }
    __syncthreads();  // vs complete; stg consumed

    // the next batch's entering rows stream in while H1/V2/H2 compute
    if (base + R < nrows) prefetch(base + R);

    // ---- H1 -----------------------------------------------------------
    for (int ch = warp; ch * 4 < GG::nq1; ch += nt / 32) {
      const int j = jl, q = ch * 4 + ql;
      if (q >= GG::nq1 || base + j >= nrows) continue;
      const int ya = ya0 + base + j;
      const int xa0 = q * KR;
      int slot = ring_new + j;
      if (slot >= GG::ringN) slot -= GG::ringN;
      float* ra = ring + slot * GG::Pr + xa0;
      float* rb = ring + (GG::ringN + slot) * GG::Pr + xa0;
      if (ya < 0 || ya >= H) {
        sts4(ra, 0.f, 0.f, 0.f, 0.f);
        sts4(ra + 4, 0.f, 0.f, 0.f, 0.f);
        sts4(rb, 0.f, 0.f, 0.f, 0.f);
        sts4(rb + 4, 0.f, 0.f, 0.f, 0.f);
        continue;
      }
      float hs[4][KR];
#pragma unroll
      for (int f = 0; f < 4; ++f) {
        const float* v = vs + (f * R + j) * GG::P1 + xa0;
        float w[4 * GG::nv1];
#pragma unroll
        for (int m = 0; m < GG::nv1; ++m) {
          const float4 t4 = lds4(v + 4 * m);
          w[4 * m] = t4.x;
          w[4 * m + 1] = t4.y;
          w[4 * m + 2] = t4.z;
          w[4 * m + 3] = t4.w;
        }
        float acc = 0.f;
#pragma unroll
        for (int d = 0; d < 2 * r; ++d) acc += w[GG::off + d];
#pragma unroll
        for (int k = 0; k < KR; ++k) {
          acc += w[GG::off + k + 2 * r];
          hs[f][k] = acc;
          acc -= w[GG::off + k];
        }
      }
      const float iny = fast_rcp((float)wlen(ya, H, r));
      const int gxa0 = x0 - r + xa0;  // global column of the run's first coefficient
      const bool interior = gxa0 >= r && gxa0 + KR - 1 + r <= W - 1 && xa0 + KR <= GG::W2;
      float A[KR], B[KR];
      if (interior) {  // warp-uniform except at strip edges
        const float inv = iny * inv_full;
#pragma unroll
        for (int k = 0; k < KR; ++k) {
          const float mg = hs[0][k] * inv, ms = hs[2][k] * inv;
          const float var = hs[1][k] * inv - mg * mg;
          const float cov = hs[3][k] * inv - mg * ms;
          if (eps == 0.f && !(var > 0.f)) degen = true;
          A[k] = cov * fast_rcp(var + eps);
          B[k] = (ms + sS) - A[k] * (mg + sG);
        }
      } else {
#pragma unroll
        for (int k = 0; k < KR; ++k) {
          const int gxa = gxa0 + k;
          const bool ok = xa0 + k < GG::W2 && gxa >= 0 && gxa < W;
          const float inv = iny * fast_rcp((float)wlen(gxa, W, r));
          const float mg = hs[0][k] * inv, ms = hs[2][k] * inv;
          const float var = hs[1][k] * inv - mg * mg;
          const float cov = hs[3][k] * inv - mg * ms;
          if (ok && eps == 0.f && !(var > 0.f)) degen = true;
          const float Ak = cov * fast_rcp(var + eps);
          A[k] = ok ? Ak : 0.f;
          B[k] = ok ? (ms + sS) - Ak * (mg + sG) : 0.f;
        }
      }
      sts4(ra, A[0], A[1], A[2], A[3]);
      sts4(ra + 4, A[4], A[5], A[6], A[7]);
      sts4(rb, B[0], B[1], B[2], B[3]);
      sts4(rb + 4, B[4], B[5], B[6], B[7]);
    }
    __syncthreads();  // ring rows of this batch complete

    // ---- V2 (part 2): add the entering coefficient rows ----------------
    if (v2) {
      float nc[4] = {0.f, 0.f, 0.f, 0.f};
      const float* rf = ring + fld * GG::ringN * GG::Pr + 4 * u4;
      float* vf = vs2 + fld * R * GG::P2 + 4 * u4;
#pragma unroll
      for (int j = 0; j < R; ++j) {
        if (v2ring && base + j < nrows) {
          int sn = ring_new + j;
          if (sn >= GG::ringN) sn -= GG::ringN;
          const float4 x = lds4(rf + sn * GG::Pr);
          nc[0] += x.x; nc[1] += x.y; nc[2] += x.z; nc[3] += x.w;
          if (j >= 2 * r + 1) {  // leaving row added earlier in this batch (r small)
            int so = ring_new + j - 2 * r - 1;
            if (so >= GG::ringN) so -= GG::ringN;
            const float4 o = lds4(rf + so * GG::Pr);
            nc[0] -= o.x; nc[1] -= o.y; nc[2] -= o.z; nc[3] -= o.w;
          }
        }
        const float4 pv = lds4(vf + j * GG::P2);
        c_sum[0] = pv.x + nc[0]; c_sum[1] = pv.y + nc[1];
        c_sum[2] = pv.z + nc[2]; c_sum[3] = pv.w + nc[3];
        sts4(vf + j * GG::P2, c_sum[0], c_sum[1], c_sum[2], c_sum[3]);
      }
    }
    ring_new += R;
    while (ring_new >= GG::ringN) ring_new -= GG::ringN;
    ring_old += R;
    while (ring_old >= GG::ringN) ring_old -= GG::ringN;
    __syncthreads();  // vs2 complete

    // ---- H2 -----------------------------------------------------------
    constexpr int nq2 = TX / KR;
    for (int ch = warp; ch * 4 < nq2; ch += nt / 32) {
      const int j = jl, q = ch * 4 + ql;
      const int yo = y0 + base + j - 2 * r;
      if (yo < y0 || yo >= yend) continue;
      const int xo0 = q * KR;
      const int gxo = x0 + xo0;
      if (gxo >= W) continue;
      const float* grow = G + (int64_t)yo * W + gxo;
      const bool two = gxo + 4 < W;
      const float4 g0 = __ldg(reinterpret_cast<const float4*>(grow));
      const float4 g1 = two ? __ldg(reinterpret_cast<const float4*>(grow + 4))
                            : make_float4(0.f, 0.f, 0.f, 0.f);
      const float gv[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
      float hs[2][KR];
#pragma unroll
      for (int f = 0; f < 2; ++f) {
        const float* v = vs2 + (f * R + j) * GG::P2 + xo0;
        float w[4 * GG::nv2];
#pragma unroll
        for (int m = 0; m < GG::nv2; ++m) {
          const float4 t4 = lds4(v + 4 * m);
          w[4 * m] = t4.x;
          w[4 * m + 1] = t4.y;
          w[4 * m + 2] = t4.z;
          w[4 * m + 3] = t4.w;
        }
        float acc = 0.f;
#pragma unroll
        for (int d = 0; d < 2 * r; ++d) acc += w[d];
#pragma unroll
        for (int k = 0; k < KR; ++k) {
          acc += w[k + 2 * r];
          hs[f][k] = acc;
          acc -= w[k];
        }
      }
      const float iny = fast_rcp((float)wlen(yo, H, r));
      const bool interior = gxo >= r && gxo + KR - 1 + r <= W - 1;
      float ov[KR];
#pragma unroll
      for (int k = 0; k < KR; ++k) {
        const float inv = interior ? iny * inv_full
                                   : iny * fast_rcp((float)wlen(gxo + k, W, r));
        ov[k] = (hs[0][k] * inv) * gv[k] + hs[1][k] * inv;
        if ((k < 4 || two) && !isfinite(ov[k])) bad = true;
      }
      float* orow = O + (int64_t)yo * W + gxo;
      *reinterpret_cast<float4*>(orow) = make_float4(ov[0], ov[1], ov[2], ov[3]);
      if (two) *reinterpret_cast<float4*>(orow + 4) = make_float4(ov[4], ov[5], ov[6], ov[7]);
    }
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
    default: return {nullptr, 0, 0};
  }
}

}  // namespace hrf

bool fused_highres_fwd_ok(int64_t B, int64_t Cg, int64_t C, int64_t H, int64_t W, int r) {
  if (r < 1 || r > hrf::kMaxRadius) return false;
  if (W % 4 != 0 || W < 4 || H < 1) return false;
  if (H > (1 << 30) || W > (1 << 30) || H * W > ((int64_t)1 << 40)) return false;
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
