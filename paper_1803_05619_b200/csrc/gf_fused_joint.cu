// Fused fast (joint-upsampling) guided filter, fp32 NCHW, factor-4 resize,
// on sm_100a.  gf/guided.py:152-195 (forward) and :267-283 + :236-264
// (backward).
//
// Forward, ONE kernel per call (k_joint_fwd): each CTA owns a 16 x 32
// low-res block = a 64 x 128 high-res tile of one plane.
//   1. its high-res guide tile is requested first (8 x 128-bit loads per
//      thread, held in registers) so HBM latency overlaps step 2;
//   2. the low-res x, y block plus halo (r for the box, 1 for the bilinear
//      support) is staged in shared memory, shifted by a per-CTA constant;
//      vertical then horizontal sliding window sums (fp32, <= 18 rows/cols
//      per run, so no error growth) give mean_x, mean_y, var, cov and
//      A = cov/(var+eps), b = mean_y - A mean_x for the (16+2) x (32+2) cells
//      the tile's bilinear taps touch -- never written to HBM;
//   3. out = Up(b) + Up(A) * hr_x (half-pixel centres, edge clamp; exact
//      factor-4 weights) is written with 128-bit stores.
// HBM traffic = compulsory (read hr_x, lr_x, lr_y; write out) + the lr halo
// re-reads, which hit L2.
//
// Backward, TWO kernels:
//   k_joint_bwd_hr  -- per tile: recompute A (step 2 above), write
//       d_hr_x = d_out * Up(A), and gather the exact bilinear adjoints
//       db = Up^T(d_out), dAraw = Up^T(d_out * hr_x) for the block's low-res
//       cells (hr rows/cols [4i-2, 4i+5]; deterministic, no atomics) into a
//       2-field low-res workspace;
//   k_joint_bwd_lr  -- per 32 x 32 low-res block with a 2r halo: moments,
//       the slope/intercept -> moment gradients (gf/guided.py:236-253), the
//       box-filter adjoints and d_lr_x, d_lr_y (gf/guided.py:255-263).
#include <cuda_runtime.h>

#include <algorithm>

#include "gf_common.cuh"
#include "gf_internal.h"
#include "gf_tma.cuh"
#include "gf_joint_taps.cuh"

namespace gfb {
namespace jf {

// shared pitches: rows of the horizontal pass are 16 lanes apart and start 16
// banks apart (pitch = 16 mod 32), so two rows per warp never share a bank
__host__ __device__ constexpr int pitch16(int n) { return n + ((48 - n % 32) % 32); }
constexpr int CAP = pitch16(CA);  // As / Bs row pitch
constexpr int kMaxRadius = 12;  // tail-kernel smem <= 227 KB

__device__ __forceinline__ int wlen(int i, int n, int r) {
  int a = i - r < 0 ? 0 : i - r;
  int b = i + r > n - 1 ? n - 1 : i + r;
  return b - a + 1;
}

struct SmemCoef {
  // sized for kMaxRadius; carved from dynamic shared memory
  float* xs;    // [RI][CI]
  float* ys;    // [RI][CI]
  float* vsum;  // [4][RA][VP]
  float* As;    // [RA][CAP]
  float* Bs;    // [RA][CAP]
};

__host__ __device__ inline size_t coef_smem_floats(int r) {
  const int RI = RA + 2 * r, CI = CA + 2 * r, VP = pitch16(CI);
  return (size_t)2 * RI * CI + (size_t)4 * RA * VP + (size_t)2 * RA * CAP;
}

__device__ inline SmemCoef carve(float* base, int r) {
  const int RI = RA + 2 * r, CI = CA + 2 * r, VP = pitch16(CI);
  SmemCoef s;
  s.xs = base;
  s.ys = s.xs + RI * CI;
  s.vsum = s.ys + RI * CI;
  s.As = s.vsum + 4 * RA * VP;
  s.Bs = s.As + RA * CAP;
  return s;
}

// A (and b) for low-res cells [i0-1, i0+TLY] x [k0-1, k0+TLX] of one plane.
// VCH: row chunks of the vertical pass (0: as many as the CTA's threads
// allow); HCH: column chunks per row of the horizontal pass.  Each chunk pays
// a 2r warm-up, so large radii favour fewer, longer chunks.
// MODE (where the block's low-res x, y come from):
//   kStageLdg  -- global planes X, Y: loaded, shifted and stored to sm.xs/ys;
//   kStageSmem -- raw values already in shared memory at X, Y (staged by TMA:
//                 rows i0-1-r.., columns k0-1-r-cofs.., pitch sp, zeros
//                 outside the image), copied shifted into sm.xs/ys;
//   kStageTma  -- the same raw TMA boxes read IN PLACE by the vertical pass
//                 (shift and the outside-the-image mask applied on the fly;
//                 no staging pass, no copy): sm.xs/ys are unused.
constexpr int kStageLdg = 0, kStageSmem = 1, kStageTma = 2;
// (mse_hr_body only) kStageTape: the slopes A of the block's 18 x 34 cells
// are read from the forward's tape instead of recomputed
constexpr int kStageTape = 3;
// kStageTapeTile: the tape's slopes, and the high-res gather window of hr_x
// and d_out (68 x 136 incl. the halo) staged by TMA into shared memory at CTA
// start (the whole tile's reads in flight at once, no registers held)
constexpr int kStageTapeTile = 4;
// staged window: 136 columns x 68 rows (= GR) used; 72 rows loaded and held, so
// every TMA box is 8 rows (18 copies per tile instead of 34 with 4-row boxes;
// rows 68..71 arrive and are ignored)
constexpr int kTileBox = 8;                       // rows per TMA box of the window
constexpr int HTW = THX + 8, HTH = THY + kTileBox;
constexpr int HTF = HTW * HTH;                    // floats per field (128-byte multiple)
constexpr int kTileGroups = 9;                    // mbarriers: 8 groups of 8 rows + rows 64..67

template <int RAD, bool NEED_B, int VCH = 0, int HCH = 16, int MODE = kStageLdg>
__device__ void lr_coeffs(const float* __restrict__ X, const float* __restrict__ Y, int h, int w,
                          int i0, int k0, float eps, const SmemCoef& sm, bool& degen,
                          int sp = 0, int cofs = 0) {
  constexpr int r = RAD;
  constexpr bool FROM_SMEM = MODE != kStageLdg;
  const int RI = RA + 2 * r, CI = CA + 2 * r;
  const int tid = threadIdx.x;
  // per-CTA shift (var/cov are shift invariant); any in-image sample works
  const int sy_ = min(max(i0, 0), h - 1), sx_ = min(max(k0, 0), w - 1);
  float sx, sy;
  if constexpr (FROM_SMEM) {
    const int o = (sy_ - (i0 - 1 - r)) * sp + (sx_ - (k0 - 1 - r)) + cofs;
    sx = X[o];
    sy = Y[o];
  } else {
    sx = __ldg(X + (int64_t)sy_ * w + sx_);
    sy = __ldg(Y + (int64_t)sy_ * w + sx_);
  }
  // 1) stage inputs (zero outside the image: clamped windows); every load of
  //    the block is issued before the first store, so the CTA waits for one
  //    memory latency, not one per element
  if constexpr (MODE != kStageTma) {
    constexpr int RIc = RA + 2 * r, CIc = CA + 2 * r;
    constexpr int NE = (RIc * CIc + NT - 1) / NT;
    float xv[NE], yv[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const int idx = tid + e * NT;
      const int row = idx / CIc, col = idx - row * CIc;
      const int gy = i0 - 1 - r + row, gx = k0 - 1 - r + col;
      const bool ok = idx < RIc * CIc && gy >= 0 && gy < h && gx >= 0 && gx < w;
      if constexpr (FROM_SMEM) {
        xv[e] = ok ? X[row * sp + col + cofs] - sx : 0.f;
        yv[e] = ok ? Y[row * sp + col + cofs] - sy : 0.f;
      } else {
        xv[e] = ok ? __ldg(X + (int64_t)gy * w + gx) - sx : 0.f;
        yv[e] = ok ? __ldg(Y + (int64_t)gy * w + gx) - sy : 0.f;
      }
    }
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const int idx = tid + e * NT;
      if (idx < RIc * CIc) {
        sm.xs[idx] = xv[e];
        sm.ys[idx] = yv[e];
      }
    }
    __syncthreads();
  }
  // 2) vertical sliding sums: item = (column, chunk of rows)
  {
    // item = (column, chunk of rows) with warps never straddling two chunks:
    // the columns of a chunk are padded to a multiple of 32
    constexpr int CW = (CA + 2 * r + 31) / 32 * 32;
    constexpr int VP = pitch16(CA + 2 * r);
    constexpr int nch =
        VCH > 0 ? VCH : (NT / CW > 0 ? (NT / CW < RA ? NT / CW : RA) : 1);
    constexpr int rc = (RA + nch - 1) / nch;
    for (int it = tid; it < CW * nch; it += NT) {
      const int col = it % CW, ch = it / CW;
      const int a0 = ch * rc, a1 = min(RA, a0 + rc);
      if (a0 >= a1 || col >= CI) continue;
      // element (row, col) of the block, shifted, 0 outside the image
      const bool colok = MODE != kStageTma || (unsigned)(k0 - 1 - r + col) < (unsigned)w;
      auto ld = [&](int row, float& xv, float& yv) {
        if constexpr (MODE == kStageTma) {
          const bool ok = colok && (unsigned)(i0 - 1 - r + row) < (unsigned)h;
          const float a = X[row * sp + col + cofs] - sx, b = Y[row * sp + col + cofs] - sy;
          xv = ok ? a : 0.f;
          yv = ok ? b : 0.f;
        } else {
          xv = sm.xs[row * CI + col];
          yv = sm.ys[row * CI + col];
        }
      };
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
      for (int d = 0; d < 2 * r; ++d) {
        float xv, yv;
        ld(a0 + d, xv, yv);
        s0 += xv;
        s1 += yv;
        s2 += xv * xv;
        s3 += xv * yv;
      }
      for (int a = a0; a < a1; ++a) {
        float xv, yv;
        ld(a + 2 * r, xv, yv);
        s0 += xv;
        s1 += yv;
        s2 += xv * xv;
        s3 += xv * yv;
        sm.vsum[(0 * RA + a) * VP + col] = s0;
        sm.vsum[(1 * RA + a) * VP + col] = s1;
        sm.vsum[(2 * RA + a) * VP + col] = s2;
        sm.vsum[(3 * RA + a) * VP + col] = s3;
        float xo, yo;
        ld(a, xo, yo);
        s0 -= xo;
        s1 -= yo;
        s2 -= xo * xo;
        s3 -= xo * yo;
      }
    }
  }
  __syncthreads();
  // 3) horizontal sliding sums + coefficients: item = (row, chunk of cols)
  {
    // 16 items per row (2 rows per warp, 16 banks apart), runs of 3 columns
    constexpr int nch = HCH;
    constexpr int cc = HCH == 16 ? (CA + 11) / 12 : (CA + HCH - 1) / HCH;
    constexpr int VP = pitch16(CA + 2 * r);
    for (int it = tid; it < RA * nch; it += NT) {
      const int a = it / nch, ch = it - a * nch;
      const int c0 = ch * cc, c1 = min(CA, c0 + cc);
      if (c0 >= c1) continue;
      const float* v0 = sm.vsum + (0 * RA + a) * VP;
      const float* v1 = sm.vsum + (1 * RA + a) * VP;
      const float* v2 = sm.vsum + (2 * RA + a) * VP;
      const float* v3 = sm.vsum + (3 * RA + a) * VP;
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
      for (int d = 0; d < 2 * r; ++d) {
        s0 += v0[c0 + d];
        s1 += v1[c0 + d];
        s2 += v2[c0 + d];
        s3 += v3[c0 + d];
      }
      const int gy = i0 - 1 + a;
      const bool row_ok = gy >= 0 && gy < h;
      const float ny = row_ok ? (float)wlen(gy, h, r) : 1.f;
      for (int c = c0; c < c1; ++c) {
        s0 += v0[c + 2 * r];
        s1 += v1[c + 2 * r];
        s2 += v2[c + 2 * r];
        s3 += v3[c + 2 * r];
        const int gx = k0 - 1 + c;
        float A = 0.f, B = 0.f;
        if (row_ok && gx >= 0 && gx < w) {
          const float inv = fast_rcp(ny * (float)wlen(gx, w, r));
          const float mx = s0 * inv, my = s1 * inv;
          const float var = s2 * inv - mx * mx;
          const float cov = s3 * inv - mx * my;
          if (eps == 0.f && !(var > 0.f)) degen = true;
          A = cov * fast_rcp(var + eps);
          if (NEED_B) B = (my + sy) - A * (mx + sx);
        }
        sm.As[a * CAP + c] = A;
        if (NEED_B) sm.Bs[a * CAP + c] = B;
        s0 -= v0[c];
        s1 -= v1[c];
        s2 -= v2[c];
        s3 -= v3[c];
      }
    }
  }
  __syncthreads();
}


struct FwdArgs {
  const float* lr_x;
  const float* lr_y;
  const float* hr_x;
  float* out;
  int h, w, H, W, r;
  float eps;
  uint32_t* status;
  float* A_tape = nullptr;  // optional: the low-res slope A of every cell (the tape)
};

template <int RAD, int VCH = 0, int HCH = 16>
__global__ void __launch_bounds__(NT, (RAD >= 2 && RAD <= 4) ? 4 : 3) k_joint_fwd(FwdArgs a) {
  extern __shared__ float4 smem4[];
  constexpr int r = RAD;
  const SmemCoef sm = carve(reinterpret_cast<float*>(smem4), r);
  const int64_t p = blockIdx.z;
  const int i0 = blockIdx.y * TLY, k0 = blockIdx.x * TLX;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float* __restrict__ G = a.hr_x + p * (int64_t)a.H * a.W;
  float* __restrict__ O = a.out + p * (int64_t)a.H * a.W;
  const int X0 = 4 * (k0 + lane);
  const int Yb = 4 * i0 + 8 * warp;  // this warp's 8 hr rows
  const bool col_ok = X0 < a.W;

  // 1) issue the hr loads first
  float4 g[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int Y = Yb + t;
    g[t] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (col_ok && Y < a.H) g[t] = __ldg(reinterpret_cast<const float4*>(G + (int64_t)Y * a.W + X0));
  }
  // 2) coefficients of the block
  bool degen = false;
  lr_coeffs<RAD, true, VCH, HCH>(a.lr_x + p * (int64_t)a.h * a.w, a.lr_y + p * (int64_t)a.h * a.w,
                                 a.h, a.w, i0, k0, a.eps, sm, degen);
  // the tile's own 16 x 32 slopes to the tape (the backward's hr pass reads
  // them instead of recomputing the window moments; gf/guided.py:181-194
  // keeps the slope in the tape the same way)
  if (a.A_tape) {
    for (int it = threadIdx.x; it < TLY * TLX; it += NT) {
      const int il = it / TLX, kl = it - il * TLX;
      const int i = i0 + il, kk = k0 + kl;
      if (i < a.h && kk < a.w)
        a.A_tape[p * (int64_t)a.h * a.w + (int64_t)i * a.w + kk] = sm.As[(il + 1) * CAP + kl + 1];
    }
  }
  // 3) apply
  // static column taps (measured: faster for r <= 4, 3 % slower at r = 8)
  const ColTaps ct = col_taps(X0, a.w, k0);
  const bool cin = RAD <= 4 && k0 + lane >= 1 && k0 + lane <= a.w - 2;
  // local coefficient rows 2*warp .. 2*warp+3 cover every tap of rows Yb..Yb+7
  float HA[4][4], HB[4][4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int rl = 2 * warp + q;
    if (rl < RA) {
      if (cin) {
        hrow_interior(sm.As + rl * CAP, lane, HA[q]);
        hrow_interior(sm.Bs + rl * CAP, lane, HB[q]);
      } else {
        hrow(sm.As + rl * CAP, ct, HA[q]);
        hrow(sm.Bs + rl * CAP, ct, HB[q]);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) HA[q][j] = HB[q][j] = 0.f;
    }
  }
  bool bad = false;
  const int slo_base = i0 - 1 + 2 * warp;  // global lr row of HA[0]
  if (Yb >= 2 && Yb + 7 <= 4 * a.h - 3 && Yb + 7 < a.H) {
    // interior rows (warp-uniform): unclamped taps, static phase weights
    // f = (2*phase + 5)/8 mod 1 of the half-pixel map (exact in fp32)
    if (col_ok) {
      float chk = 0.f;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int q0 = t / 4 + ((t & 3) >= 2 ? 1 : 0);
        constexpr float fph[4] = {0.625f, 0.875f, 0.125f, 0.375f};
        const float f = fph[t & 3];
        const float gv[4] = {g[t].x, g[t].y, g[t].z, g[t].w};
        float o[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float Ah = HA[q0][j] + f * (HA[q0 + 1][j] - HA[q0][j]);
          const float Bh = HB[q0][j] + f * (HB[q0 + 1][j] - HB[q0][j]);
          o[j] = Bh + Ah * gv[j];
          chk = fmaf(o[j], 0.f, chk);  // NaN iff an output is not finite
        }
        *reinterpret_cast<float4*>(O + (int64_t)(Yb + t) * a.W + X0) =
            make_float4(o[0], o[1], o[2], o[3]);
      }
      bad = chk != 0.f;
    }
  } else {
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int Y = Yb + t;
    if (!col_ok || Y >= a.H) continue;
    const Tap ty = tap4(Y, a.h);
    // static rows for interior taps: phase 0,1 -> (cell-1, cell); 2,3 -> (cell, cell+1)
    constexpr int dummy = 0;
    (void)dummy;
    const int q0 = t / 4 + ((t & 3) >= 2 ? 1 : 0);
    const int slo = slo_base + q0;
    float o[4];
    const float gv[4] = {g[t].x, g[t].y, g[t].z, g[t].w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      // exact clamped taps: lo is slo (interior / bottom clamp) or slo+1 (top clamp, f == 0)
      const float alo = ty.lo == slo ? HA[q0][j] : HA[q0 + 1][j];
      const float ahi = ty.hi == slo + 1 ? HA[q0 + 1][j] : alo;
      const float blo = ty.lo == slo ? HB[q0][j] : HB[q0 + 1][j];
      const float bhi = ty.hi == slo + 1 ? HB[q0 + 1][j] : blo;
      const float Ah = alo + ty.f * (ahi - alo);
      const float Bh = blo + ty.f * (bhi - blo);
      o[j] = Bh + Ah * gv[j];
      if (!isfinite(o[j])) bad = true;
    }
    *reinterpret_cast<float4*>(O + (int64_t)Y * a.W + X0) = make_float4(o[0], o[1], o[2], o[3]);
  }
  }
  if (degen) flag(a.status, GF_STATUS_DEGENERATE);
  if (bad) flag(a.status, GF_STATUS_NONFINITE_OUTPUT);
}

// ---------------------------------------------------------------------------
// forward, persistent TMA pipeline (k_joint_fwd_tma)
// ---------------------------------------------------------------------------
// The same per-tile arithmetic as k_joint_fwd (bit-identical results), but a
// CTA walks tiles t = blockIdx.x, +gridDim.x, ... and TMA stages each tile's
// inputs -- the 64 x 128 high-res guide tile and the low-res x, y halo blocks
// (zero-filled outside the image by the hardware) -- NS tiles ahead into a
// ring of shared-memory stages, so the SM's HBM reads for the next tiles are
// in flight while it computes and stores the current one.  One elected
// thread issues the copies; an mbarrier per stage carries the byte count.
// A TMA box must start on a 16-byte column in global memory (an unaligned
// start raises an illegal-instruction fault on sm_100a), so the low-res box
// starts PADL >= 1 + r columns left of the block, PADL a multiple of 4.
template <int RAD>
struct TmaGeo {
  static constexpr int RI = RA + 2 * RAD;
  static constexpr int PADL = (1 + RAD + 3) / 4 * 4;
  static constexpr int COFS = PADL - 1 - RAD;                // staged column of block col 0
  static constexpr int LP = (PADL + TLX + 1 + RAD + 3) / 4 * 4;  // box width: 16-byte rows
  static constexpr int HR = THY * THX;                    // floats
  static constexpr int LR = (RI * LP + 31) / 32 * 32;     // 128-byte aligned boxes
  static constexpr int STAGE = HR + 2 * LR;
  static constexpr uint32_t BYTES = (uint32_t)(HR + 2 * RI * LP) * 4u;
  static constexpr uint32_t LBYTES = (uint32_t)(2 * RI * LP) * 4u;  // low-res boxes only
};

__device__ __forceinline__ float* align128(float4* p) {
  return reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(p) + 127) &
                                  ~static_cast<uintptr_t>(127));
}

// layout of the TMA-staged tile kernels: [x box][y box][vsum][As][Bs]
// (128-byte aligned boxes; sm.xs / sm.ys unused)
template <int RAD>
__host__ __device__ constexpr int tma_coef_floats() {
  return 2 * TmaGeo<RAD>::LR + 4 * RA * pitch16(CA + 2 * RAD) + 2 * RA * CAP;
}

template <int RAD>
__device__ __forceinline__ SmemCoef carve_tma(float* base) {
  SmemCoef s;
  s.xs = s.ys = nullptr;
  s.vsum = base + 2 * TmaGeo<RAD>::LR;
  s.As = s.vsum + 4 * RA * pitch16(CA + 2 * RAD);
  s.Bs = s.As + RA * CAP;
  return s;
}

template <int RAD, int NS>
inline size_t fwd_tma_smem_bytes() {
  return 128 + (size_t)NS * TmaGeo<RAD>::STAGE * 4 + coef_smem_floats(RAD) * 4;
}

// out = Up(b) + Up(A) * g for the 8 hr rows (Yb .. Yb+7) x 4 columns (X0 ..)
// of this thread, coefficients in sm.As / sm.Bs (k_joint_fwd's step 3)
template <int RAD, int CAP = jf::CAP>  // CAP: row pitch of sm.As / sm.Bs
__device__ __forceinline__ bool apply_rows(const SmemCoef& sm, const float4 (&g)[8], float* O,
                                           int h, int w, int H, int W, int i0, int k0,
                                           int lane, int warp) {
  const int X0 = 4 * (k0 + lane);
  const int Yb = 4 * i0 + 8 * warp;
  const bool col_ok = X0 < W;
  const bool cin = RAD <= 4 && k0 + lane >= 1 && k0 + lane <= w - 2;
  ColTaps ct;
  if (!cin) ct = col_taps(X0, w, k0);
  float HA[4][4], HB[4][4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int rl = 2 * warp + q;
    if (rl < RA) {
      if (cin) {
        hrow_interior(sm.As + rl * CAP, lane, HA[q]);
        hrow_interior(sm.Bs + rl * CAP, lane, HB[q]);
      } else {
        hrow(sm.As + rl * CAP, ct, HA[q]);
        hrow(sm.Bs + rl * CAP, ct, HB[q]);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) HA[q][j] = HB[q][j] = 0.f;
    }
  }
  bool bad = false;
  const int slo_base = i0 - 1 + 2 * warp;
  if (Yb >= 2 && Yb + 7 <= 4 * h - 3 && Yb + 7 < H) {
    if (col_ok) {
      float chk = 0.f;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int q0 = t / 4 + ((t & 3) >= 2 ? 1 : 0);
        constexpr float fph[4] = {0.625f, 0.875f, 0.125f, 0.375f};
        const float f = fph[t & 3];
        const float gv[4] = {g[t].x, g[t].y, g[t].z, g[t].w};
        float o[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float Ah = HA[q0][j] + f * (HA[q0 + 1][j] - HA[q0][j]);
          const float Bh = HB[q0][j] + f * (HB[q0 + 1][j] - HB[q0][j]);
          o[j] = Bh + Ah * gv[j];
          chk = fmaf(o[j], 0.f, chk);
        }
        *reinterpret_cast<float4*>(O + (int64_t)(Yb + t) * W + X0) =
            make_float4(o[0], o[1], o[2], o[3]);
      }
      bad = chk != 0.f;
    }
  } else {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int Y = Yb + t;
      if (!col_ok || Y >= H) continue;
      const Tap ty = tap4(Y, h);
      const int q0 = t / 4 + ((t & 3) >= 2 ? 1 : 0);
      const int slo = slo_base + q0;
      float o[4];
      const float gv[4] = {g[t].x, g[t].y, g[t].z, g[t].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float alo = ty.lo == slo ? HA[q0][j] : HA[q0 + 1][j];
        const float ahi = ty.hi == slo + 1 ? HA[q0 + 1][j] : alo;
        const float blo = ty.lo == slo ? HB[q0][j] : HB[q0 + 1][j];
        const float bhi = ty.hi == slo + 1 ? HB[q0 + 1][j] : blo;
        const float Ah = alo + ty.f * (ahi - alo);
        const float Bh = blo + ty.f * (bhi - blo);
        o[j] = Bh + Ah * gv[j];
        if (!isfinite(o[j])) bad = true;
      }
      *reinterpret_cast<float4*>(O + (int64_t)Y * W + X0) = make_float4(o[0], o[1], o[2], o[3]);
    }
  }
  return bad;
}

// the tile kernel k_joint_fwd with its low-res halo blocks staged by TMA
template <int RAD, int VCH = 0, int HCH = 16>
__global__ void __launch_bounds__(NT, (RAD >= 2 && RAD <= 4) ? 4 : 3)
    k_joint_fwd_t(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmY,
                  FwdArgs a) {
  using TG = TmaGeo<RAD>;
  extern __shared__ float4 smem4[];
  __shared__ __align__(8) uint64_t tbar;
  float* base = align128(smem4);
  const SmemCoef sm = carve_tma<RAD>(base);
  const int64_t p = blockIdx.z;
  const int i0 = blockIdx.y * TLY, k0 = blockIdx.x * TLX;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float* __restrict__ G = a.hr_x + p * (int64_t)a.H * a.W;
  float* __restrict__ O = a.out + p * (int64_t)a.H * a.W;
  const int X0 = 4 * (k0 + lane);
  const int Yb = 4 * i0 + 8 * warp;
  const bool col_ok = X0 < a.W;
  if (threadIdx.x == 0) tma::mbar_init(&tbar, 1);
  // 1) the hr loads first, then the low-res blocks by TMA
  float4 g[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int Y = Yb + t;
    g[t] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (col_ok && Y < a.H) g[t] = __ldg(reinterpret_cast<const float4*>(G + (int64_t)Y * a.W + X0));
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    tma::mbar_arrive_expect_tx(&tbar, TG::LBYTES);
    tma::load_3d(base, &tmX, k0 - TG::PADL, i0 - 1 - RAD, (int)p, &tbar);
    tma::load_3d(base + TG::LR, &tmY, k0 - TG::PADL, i0 - 1 - RAD, (int)p, &tbar);
  }
  tma::mbar_wait(&tbar, 0);
  // 2) coefficients, reading the TMA boxes in place
  bool degen = false;
  lr_coeffs<RAD, true, VCH, HCH, kStageTma>(base, base + TG::LR, a.h, a.w, i0, k0, a.eps, sm,
                                            degen, TG::LP, TG::COFS);
  // 3) apply
  const bool bad = apply_rows<RAD>(sm, g, O, a.h, a.w, a.H, a.W, i0, k0, lane, warp);
  if (degen) flag(a.status, GF_STATUS_DEGENERATE);
  if (bad) flag(a.status, GF_STATUS_NONFINITE_OUTPUT);
}

template <int RAD, int NS, int MINB, int VCH = 0, int HCH = 16>
__global__ void __launch_bounds__(NT, MINB)
    k_joint_fwd_tma(const __grid_constant__ CUtensorMap tmG, const __grid_constant__ CUtensorMap tmX,
                    const __grid_constant__ CUtensorMap tmY, FwdArgs a, int tiles_x, int tiles_y,
                    int ntiles) {
  using TG = TmaGeo<RAD>;
  extern __shared__ float4 smem4[];
  __shared__ __align__(8) uint64_t bar[NS];
  float* base = reinterpret_cast<float*>(
      (reinterpret_cast<uintptr_t>(smem4) + 127) & ~static_cast<uintptr_t>(127));
  const SmemCoef sm = carve(base + NS * TG::STAGE, RAD);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) tma::mbar_init(&bar[s], 1);
  }
  __syncthreads();
  auto coords = [&](int t, int& p, int& i0, int& k0) {
    const int tx = t % tiles_x, rest = t / tiles_x;
    k0 = tx * TLX;
    i0 = (rest % tiles_y) * TLY;
    p = rest / tiles_y;
  };
  auto issue = [&](int t, int s) {
    int p, i0, k0;
    coords(t, p, i0, k0);
    float* st = base + s * TG::STAGE;
    tma::mbar_arrive_expect_tx(&bar[s], TG::BYTES);
    tma::load_3d(st, &tmG, 4 * k0, 4 * i0, p, &bar[s]);
    tma::load_3d(st + TG::HR, &tmX, k0 - TG::PADL, i0 - 1 - RAD, p, &bar[s]);
    tma::load_3d(st + TG::HR + TG::LR, &tmY, k0 - TG::PADL, i0 - 1 - RAD, p, &bar[s]);
  };
  if (tid == 0)
    for (int j = 0; j < NS - 1; ++j) {
      const int t = blockIdx.x + j * gridDim.x;
      if (t < ntiles) issue(t, j);
    }
  bool degen = false, bad = false;
  int k = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
    const int s = k % NS;
    if (tid == 0) {  // refill the stage iteration k-1 released
      const int tn = t + (NS - 1) * gridDim.x;
      if (tn < ntiles) issue(tn, (k + NS - 1) % NS);
    }
    int p, i0, k0;
    coords(t, p, i0, k0);
    tma::mbar_wait(&bar[s], (uint32_t)((k / NS) & 1));
    const float* st = base + s * TG::STAGE;
    lr_coeffs<RAD, true, VCH, HCH, kStageSmem>(st + TG::HR, st + TG::HR + TG::LR, a.h, a.w, i0, k0,
                                         a.eps, sm, degen, TG::LP, TG::COFS);
    float4 g[8];
#pragma unroll
    for (int r8 = 0; r8 < 8; ++r8)
      g[r8] = *reinterpret_cast<const float4*>(st + (8 * warp + r8) * THX + 4 * lane);
    float* O = a.out + (int64_t)p * a.H * a.W;
    bad |= apply_rows<RAD>(sm, g, O, a.h, a.w, a.H, a.W, i0, k0, lane, warp);
    // every thread's generic reads of stage s and of the coefficient scratch
    // are done before thread 0 lets TMA overwrite the stage
    tma::fence_proxy_async();
    __syncthreads();
  }
  if (degen) flag(a.status, GF_STATUS_DEGENERATE);
  if (bad) flag(a.status, GF_STATUS_NONFINITE_OUTPUT);
}

// ---------------------------------------------------------------------------
// backward, kernel 1: hr pass
// ---------------------------------------------------------------------------
struct BwdHrArgs {
  const float* lr_x;
  const float* lr_y;
  const float* hr_x;
  const float* d_out;
  float* d_hr;
  float* db;     // (P, h, w) workspace
  float* dA;     // (P, h, w) workspace
  int h, w, H, W, r;
  float eps;
  uint32_t* status;
};

constexpr int GR = THY + 4;  // gather rows: hr [4 i0 - 2, 4 i0 + 66)

__host__ __device__ inline size_t bwd_hr_smem_floats(int r) {
  return coef_smem_floats(r) + (size_t)2 * GR * TLX;
}

template <int RAD>
__global__ void __launch_bounds__(NT, 4) k_joint_bwd_hr(BwdHrArgs a) {
  extern __shared__ float4 smem4[];
  constexpr int r = RAD;
  float* base = reinterpret_cast<float*>(smem4);
  const SmemCoef sm = carve(base, r);
  float* R1 = base + coef_smem_floats(r);  // [GR][TLX]
  float* R2 = R1 + GR * TLX;
  const int64_t p = blockIdx.z;
  const int i0 = blockIdx.y * TLY, k0 = blockIdx.x * TLX;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t hplane = (int64_t)a.H * a.W;
  const float* __restrict__ G = a.hr_x + p * hplane;
  const float* __restrict__ D = a.d_out + p * hplane;
  float* __restrict__ DH = a.d_hr + p * hplane;
  const int X0 = 4 * (k0 + lane);
  const int Yb = 4 * i0 + 8 * warp;
  const bool col_ok = X0 < a.W;

  // the d_out tile is read after the coefficient phase (registers stay free
  // for it); its DRAM reads start now, into L2
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int Y = Yb + t;
    if (col_ok && Y < a.H)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(D + (int64_t)Y * a.W + X0));
  }
  // the gather below reads hr_x (and the 2-pixel halo of both fields) only
  // after the coefficient phase: start those DRAM reads now, into L2
  {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int Y = Yb + t;
      if (col_ok && Y < a.H)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(G + (int64_t)Y * a.W + X0));
    }
    // halo rows 4 i0 - 2, -1 (warp 0) and 4 i0 + 64, 65 (warp 7)
    if (warp == 0 || warp == NT / 32 - 1) {
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int Y = warp == 0 ? 4 * i0 - 2 + t : 4 * i0 + THY + t;
        if (col_ok && Y >= 0 && Y < a.H) {
          asm volatile("prefetch.global.L2 [%0];" ::"l"(G + (int64_t)Y * a.W + X0));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(D + (int64_t)Y * a.W + X0));
        }
      }
    }
    // halo columns: the 16-byte chunks left of lane 0 and right of lane 31
    const int Xh = lane == 0 ? X0 - 4 : (lane == 31 ? X0 + 4 : -1);
    if (Xh >= 0 && Xh < a.W) {
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int Y = Yb + t;
        if (Y < a.H) {
          asm volatile("prefetch.global.L2 [%0];" ::"l"(G + (int64_t)Y * a.W + Xh));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(D + (int64_t)Y * a.W + Xh));
        }
      }
    }
  }
  bool degen = false;
  lr_coeffs<RAD, false>(a.lr_x + p * (int64_t)a.h * a.w, a.lr_y + p * (int64_t)a.h * a.w, a.h, a.w,
                   i0, k0, a.eps, sm, degen);
  float4 dv[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int Y = Yb + t;
    dv[t] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (col_ok && Y < a.H) dv[t] = __ldg(reinterpret_cast<const float4*>(D + (int64_t)Y * a.W + X0));
  }
  // d_hr = d_out * Up(A)
  {
    const ColTaps ct = col_taps(X0, a.w, k0);
    const bool cin = k0 + lane >= 1 && k0 + lane <= a.w - 2;  // static column taps
    float HA[4][4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int rl = 2 * warp + q;
      if (rl < RA) {
        if (cin)
          hrow_interior(sm.As + rl * CAP, lane, HA[q]);
        else
          hrow(sm.As + rl * CAP, ct, HA[q]);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) HA[q][j] = 0.f;
      }
    }
    const int slo_base = i0 - 1 + 2 * warp;
    if (Yb >= 2 && Yb + 7 <= 4 * a.h - 3 && Yb + 7 < a.H) {  // interior rows: static taps
      if (col_ok) {
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const int q0 = t / 4 + ((t & 3) >= 2 ? 1 : 0);
          constexpr float fph[4] = {0.625f, 0.875f, 0.125f, 0.375f};
          const float f = fph[t & 3];
          const float dd[4] = {dv[t].x, dv[t].y, dv[t].z, dv[t].w};
          float o[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) o[j] = dd[j] * (HA[q0][j] + f * (HA[q0 + 1][j] - HA[q0][j]));
          *reinterpret_cast<float4*>(DH + (int64_t)(Yb + t) * a.W + X0) =
              make_float4(o[0], o[1], o[2], o[3]);
        }
      }
    } else {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int Y = Yb + t;
      if (!col_ok || Y >= a.H) continue;
      const Tap ty = tap4(Y, a.h);
      const int q0 = t / 4 + ((t & 3) >= 2 ? 1 : 0);
      const int slo = slo_base + q0;
      const float dd[4] = {dv[t].x, dv[t].y, dv[t].z, dv[t].w};
      float o[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float alo = ty.lo == slo ? HA[q0][j] : HA[q0 + 1][j];
        const float ahi = ty.hi == slo + 1 ? HA[q0 + 1][j] : alo;
        o[j] = dd[j] * (alo + ty.f * (ahi - alo));
      }
      *reinterpret_cast<float4*>(DH + (int64_t)Y * a.W + X0) = make_float4(o[0], o[1], o[2], o[3]);
    }
    }
  }
  // row partials of the adjoint: R[y][k] = sum_X wx(X, k) * (d, d*G) over
  // X in [4k-2, 4k+5] (every hr column whose taps touch lr column k): the
  // lane's own 16-byte chunk plus 2 columns of each neighbour lane by shuffle;
  // lanes 0 and 31 load the chunk outside the tile alongside their own
  {
    const int k = k0 + lane;
    float wx[8];
    if (k >= 1 && k <= a.w - 2) {  // interior: the static transposed taps
#pragma unroll
      for (int j = 0; j < 8; ++j) wx[j] = (j < 4 ? 2 * j + 1 : 15 - 2 * j) * 0.125f;
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int X = 4 * k - 2 + j;
        wx[j] = 0.f;
        if (X >= 0 && X < a.W) {
          const Tap tx = tap4(X, a.w);
          if (tx.lo == k) wx[j] += 1.f - tx.f;
          if (tx.hi == k) wx[j] += tx.f;
        }
      }
    }
    const int Xe = lane == 0 ? 4 * k - 4 : 4 * k + 4;  // edge lanes' outside chunk
    const bool edge = (lane == 0 || lane == 31) && Xe >= 0 && Xe < a.W;
#pragma unroll 2
    for (int yl = warp; yl < GR; yl += NT / 32) {
      const int Y = 4 * i0 - 2 + yl;
      const bool row = Y >= 0 && Y < a.H;
      const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
      float4 d1 = z, g1 = z, de = z, ge = z;
      if (row && k < a.w) {
        d1 = __ldg(reinterpret_cast<const float4*>(D + (int64_t)Y * a.W + 4 * k));
        g1 = __ldg(reinterpret_cast<const float4*>(G + (int64_t)Y * a.W + 4 * k));
      }
      if (row && edge) {
        de = __ldg(reinterpret_cast<const float4*>(D + (int64_t)Y * a.W + Xe));
        ge = __ldg(reinterpret_cast<const float4*>(G + (int64_t)Y * a.W + Xe));
      }
      const float4 q1 = make_float4(d1.x * g1.x, d1.y * g1.y, d1.z * g1.z, d1.w * g1.w);
      float dl0 = __shfl_up_sync(0xffffffffu, d1.z, 1), dl1 = __shfl_up_sync(0xffffffffu, d1.w, 1);
      float ql0 = __shfl_up_sync(0xffffffffu, q1.z, 1), ql1 = __shfl_up_sync(0xffffffffu, q1.w, 1);
      float dr0 = __shfl_down_sync(0xffffffffu, d1.x, 1), dr1 = __shfl_down_sync(0xffffffffu, d1.y, 1);
      float qr0 = __shfl_down_sync(0xffffffffu, q1.x, 1), qr1 = __shfl_down_sync(0xffffffffu, q1.y, 1);
      if (lane == 0) {
        dl0 = de.z;
        dl1 = de.w;
        ql0 = de.z * ge.z;
        ql1 = de.w * ge.w;
      }
      if (lane == 31) {
        dr0 = de.x;
        dr1 = de.y;
        qr0 = de.x * ge.x;
        qr1 = de.y * ge.y;
      }
      const float dd[8] = {dl0, dl1, d1.x, d1.y, d1.z, d1.w, dr0, dr1};
      const float qq[8] = {ql0, ql1, q1.x, q1.y, q1.z, q1.w, qr0, qr1};
      float s1 = 0.f, s2 = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        s1 += wx[j] * dd[j];
        s2 += wx[j] * qq[j];
      }
      if (!(row && k < a.w)) s1 = s2 = 0.f;
      R1[yl * TLX + lane] = s1;
      R2[yl * TLX + lane] = s2;
    }
  }
  __syncthreads();
  // column pass: db[i][k] = sum_Y wy(Y, i) R1[Y][k]
  for (int it = threadIdx.x; it < TLY * TLX; it += NT) {
    const int il = it / TLX, kl = it - il * TLX;
    const int i = i0 + il, k = k0 + kl;
    if (i >= a.h || k >= a.w) continue;
    float s1 = 0.f, s2 = 0.f;
    if (i >= 1 && i <= a.h - 2 && 4 * i + 5 < a.H) {
      // interior lr row: static weights of hr rows 4i-2 .. 4i+5 (the taps of
      // hrow_interior transposed: 1/8, 3/8, 5/8, 7/8, 7/8, 5/8, 3/8, 1/8)
      constexpr float wy[8] = {0.125f, 0.375f, 0.625f, 0.875f, 0.875f, 0.625f, 0.375f, 0.125f};
      const int yl0 = 4 * (i - i0);  // gather row of hr row 4i-2
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        s1 += wy[t] * R1[(yl0 + t) * TLX + kl];
        s2 += wy[t] * R2[(yl0 + t) * TLX + kl];
      }
    } else {
#pragma unroll
      for (int dy = -2; dy <= 5; ++dy) {
        const int Y = 4 * i + dy;
        if (Y < 0 || Y >= a.H) continue;
        const Tap ty = tap4(Y, a.h);
        float wgt = 0.f;
        if (ty.lo == i) wgt += 1.f - ty.f;
        if (ty.hi == i) wgt += ty.f;
        const int yl = Y - (4 * i0 - 2);
        s1 += wgt * R1[yl * TLX + kl];
        s2 += wgt * R2[yl * TLX + kl];
      }
    }
    const int64_t o = p * (int64_t)a.h * a.w + (int64_t)i * a.w + k;
    a.db[o] = s1;
    a.dA[o] = s2;
  }
  if (degen) flag(a.status, GF_STATUS_DEGENERATE);
}

// ---------------------------------------------------------------------------
// training step, fused: forward + MSE + backward hr pass
// ---------------------------------------------------------------------------
// A training step needs the loss and the gradients only (gf/training.py:230-235,
// eval_and_grads), and d_out = 2 (out - target) / (C H W B) is local
// (gf/training.py:93-101, batch mean of the per-image losses).  So per tile:
// recompute A and b (step 2 of the forward), then for every row of the
// 68-row gather window (tile + 2-pixel halo) form out = Up(b) + Up(A) hr_x,
// e = out - target, d_out, and do what k_joint_bwd_hr does with it -- the
// tile's d_hr_x = d_out Up(A) and the two bilinear adjoints -- with the
// per-CTA sum of e^2 (float64) as the loss partial.  Neither out nor d_out
// touches HBM: hr_x and target are each read once.
//
// Rows: warp w takes gather rows 8w .. 8w+7, whose taps use coefficient rows
// 2w .. 2w+2 (pre-interpolated horizontally once), and warps 0..3 one of the
// rows 64..67 (coefficient rows 16, 17).  The 2 halo columns on each side of
// the tile (taps of lr columns k0 and k0+31) are added to the row partials by
// a scalar pass per warp.
struct MseHrArgs {
  const float* lr_x;
  const float* lr_y;
  const float* hr_x;
  const float* target;  // MSE: the target; else d_out
  float* d_hr;
  float* db;
  float* dA;
  double* loss_part;  // MSE: one per CTA (plane, tile row, tile column)
  int h, w, H, W, r;
  float eps, scale2;
  uint32_t* status;
  const float* A_tape = nullptr;  // kStageTape: the forward's low-res slopes
  const float* B_tape = nullptr;  // ... and intercepts (MSE: k_joint_coeffs)
};

// MSE = false: the same single gather pass for a given d_out (k_joint_bwd_hr's
// job): `target` is d_out, A only, no loss.
// MODE kStageTma (k_joint_mse_hr_t): the low-res x, y halo blocks arrive by
// TMA (one elected thread, one mbarrier) and the coefficient pass reads them
// in place -- no per-thread staging loads, index math or copies.
// TY: low-res rows per tile (the namespace's TLY = 16, or 8: a 32-row high-res
// tile of 4 warps, each with 8 rows and one of the 4 extra rows; kStageTapeTile
// without the MSE only).  The per-pixel products, the row partials and the
// column sums do not depend on the tile height: results are bitwise the same.
template <int RAD, bool MSE, int MODE, int TY = jf::TLY>
__device__ __forceinline__ void mse_hr_body(const MseHrArgs& a, const CUtensorMap* tmX,
                                            const CUtensorMap* tmY) {
  // this tile's geometry (shadows the namespace's 16-row constants)
  constexpr int TLY = TY, THY = 4 * TY, NT = 32 * (TY / 2);
  constexpr int RA = TY + 2, GR = THY + 4, HTH = THY + kTileBox, HTF = HTW * HTH;
  constexpr int kTileGroups = TY / 2 + 1;  // 8-row groups + the 4 extra rows
  static_assert(TY == jf::TLY || (MODE == kStageTapeTile && !MSE), "8-row tiles: tape + TMA only");
  extern __shared__ float4 smem4[];
  __shared__ double red[NT / 32];
  __shared__ __align__(8) uint64_t tbar;
  __shared__ __align__(8) uint64_t gbar[kTileGroups];  // kStageTapeTile: per row group
  constexpr int r = RAD;
  float* base;
  SmemCoef sm;
  float* R1;  // [GR][TLX]
  if constexpr (MODE == kStageTma) {
    base = align128(smem4);
    sm = carve_tma<RAD>(base);
    R1 = base + tma_coef_floats<RAD>();
  } else if constexpr (MODE == kStageTape) {
    base = reinterpret_cast<float*>(smem4);
    sm.xs = sm.ys = sm.vsum = nullptr;
    sm.As = base;
    sm.Bs = base + RA * CAP;
    R1 = base + 2 * RA * CAP;
  } else if constexpr (MODE == kStageTapeTile) {
    base = align128(smem4);
    sm.xs = sm.ys = sm.vsum = nullptr;
    sm.As = base + 2 * HTF;
    sm.Bs = sm.As + RA * CAP;
    R1 = sm.Bs + RA * CAP;
  } else {
    base = reinterpret_cast<float*>(smem4);
    sm = carve(base, r);
    R1 = base + coef_smem_floats(r);
  }
  float* R2 = R1 + GR * TLX;
  const int64_t p = blockIdx.z;
  const int i0 = blockIdx.y * TLY, k0 = blockIdx.x * TLX;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t hplane = (int64_t)a.H * a.W;
  const float* __restrict__ G = a.hr_x + p * hplane;
  const float* __restrict__ T = a.target + p * hplane;
  float* __restrict__ DH = a.d_hr + p * hplane;
  const int k = k0 + lane;
  const int X0 = 4 * k;
  const bool col_ok = k < a.w;  // W == 4 w
  const int Yg = 4 * i0 - 2;    // hr row of gather row 0
  const bool extra = warp < 4;  // takes gather row THY + warp as well

  // the tile's gather rows of hr_x and target (with the 4-column halo chunk
  // on each side the scalar pass reads) start their DRAM reads into L2
  // before the coefficient phase: ONE bulk L2 prefetch per (row, field), by
  // 2 x 68 threads (one instruction each)
  const float* tG = base;        // kStageTapeTile: staged gather window
  const float* tT = base + HTF;
  if (MODE != kStageTapeTile && threadIdx.x < 2 * GR) {
    const int yl = threadIdx.x >> 1, Y = Yg + yl;
    const int xa = max(4 * k0 - 4, 0), xb = min(4 * k0 + THX + 4, a.W);
    if (Y >= 0 && Y < a.H && xb > xa) {
      const float* src = ((threadIdx.x & 1) ? T : G) + (int64_t)Y * a.W + xa;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src),
                   "r"((unsigned)(xb - xa) * 4u)
                   : "memory");
    }
  }
  bool degen = false;
  if constexpr (MODE == kStageTma) {
    using TG = TmaGeo<RAD>;
    if (threadIdx.x == 0) tma::mbar_init(&tbar, 1);
    __syncthreads();
    if (threadIdx.x == 0) {
      tma::mbar_arrive_expect_tx(&tbar, TG::LBYTES);
      tma::load_3d(base, tmX, k0 - TG::PADL, i0 - 1 - r, (int)p, &tbar);
      tma::load_3d(base + TG::LR, tmY, k0 - TG::PADL, i0 - 1 - r, (int)p, &tbar);
    }
    tma::mbar_wait(&tbar, 0);
    lr_coeffs<RAD, MSE, 0, 16, kStageTma>(base, base + TG::LR, a.h, a.w, i0, k0, a.eps, sm,
                                          degen, TG::LP, TG::COFS);
  } else if constexpr (MODE == kStageTape || MODE == kStageTapeTile) {
    static_assert(!MSE || MODE == kStageTapeTile, "the forward's tape has A only");
    // the tile's coefficient cells are requested FIRST (they gate every warp's
    // start; behind the window's 74 KB they would return last), held in
    // registers until the window's copies have been issued
    constexpr int NEA = (RA * CA + NT - 1) / NT;
    float av[NEA], bv[NEA];
    {
      const float* At = a.A_tape + p * (int64_t)a.h * a.w;
#pragma unroll
      for (int e = 0; e < NEA; ++e) {
        const int it = threadIdx.x + e * NT;
        const int ar = it / CA, c = it - ar * CA;
        const int gy = i0 - 1 + ar, gx = k0 - 1 + c;
        const bool inimg = it < RA * CA && gy >= 0 && gy < a.h && gx >= 0 && gx < a.w;
        const int64_t o = (int64_t)gy * a.w + gx;
        av[e] = inimg ? __ldg(At + o) : 0.f;
        bv[e] = 0.f;
        if constexpr (MSE) bv[e] = inimg ? __ldg(a.B_tape + p * (int64_t)a.h * a.w + o) : 0.f;
      }
    }
    if constexpr (MODE == kStageTapeTile) {
      // the window arrives as kTileBox-row boxes in row order, one mbarrier
      // per 8-row group (= per warp) and one for rows 64..67: a warp starts
      // on its rows as soon as THEY have landed, while the rest of the
      // window is still in flight
      if (threadIdx.x == 0) {
#pragma unroll
        for (int c = 0; c < kTileGroups; ++c) tma::mbar_init(&gbar[c], 1);
        tma::fence_proxy_async();
      }
      __syncthreads();
      if (threadIdx.x == 0) {
#pragma unroll
        for (int c = 0; c < kTileGroups; ++c) {
          const int rows = c < kTileGroups - 1 ? 8 : HTH - THY;
          tma::mbar_arrive_expect_tx(&gbar[c], 2u * rows * HTW * 4u);
#pragma unroll
          for (int b = 0; b < rows; b += kTileBox) {
            const int yl = 8 * c + b;
            tma::load_3d(base + yl * HTW, tmX, 4 * k0 - 4, Yg + yl, (int)p, &gbar[c]);
            tma::load_3d(base + HTF + yl * HTW, tmY, 4 * k0 - 4, Yg + yl, (int)p, &gbar[c]);
          }
        }
      }
    }
#pragma unroll
    for (int e = 0; e < NEA; ++e) {
      const int it = threadIdx.x + e * NT;
      if (it < RA * CA) {
        const int ar = it / CA, c = it - ar * CA;
        sm.As[ar * CAP + c] = av[e];
        if constexpr (MSE) sm.Bs[ar * CAP + c] = bv[e];
      }
    }
    __syncthreads();
    if constexpr (MODE == kStageTapeTile) tma::mbar_wait(&gbar[warp], 0);
  } else {
    lr_coeffs<RAD, MSE>(a.lr_x + p * (int64_t)a.h * a.w, a.lr_y + p * (int64_t)a.h * a.w, a.h,
                        a.w, i0, k0, a.eps, sm, degen);
  }

  const bool cin = k >= 1 && k <= a.w - 2;  // static column taps
  ColTaps ct;
  if (!cin) ct = col_taps(X0, a.w, k0);
  auto hrow2 = [&](int rl, float (&ha)[4], float (&hb)[4]) {
    if (cin) {
      hrow_interior(sm.As + rl * CAP, lane, ha);
      if (MSE) hrow_interior(sm.Bs + rl * CAP, lane, hb);
    } else {
      hrow(sm.As + rl * CAP, ct, ha);
      if (MSE) hrow(sm.Bs + rl * CAP, ct, hb);
    }
    if (!MSE) {
#pragma unroll
      for (int j = 0; j < 4; ++j) hb[j] = 0.f;
    }
  };
  // adjoint weights of hr columns 4k-2 .. 4k+5 into lr column k
  float wx[8];
  if (cin) {
#pragma unroll
    for (int j = 0; j < 8; ++j) wx[j] = (j < 4 ? 2 * j + 1 : 15 - 2 * j) * 0.125f;
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int X = 4 * k - 2 + j;
      wx[j] = 0.f;
      if (X >= 0 && X < a.W) {
        const Tap tx = tap4(X, a.w);
        if (tx.lo == k) wx[j] += 1.f - tx.f;
        if (tx.hi == k) wx[j] += tx.f;
      }
    }
  }

  // kStageTapeTile without the MSE: the 2 halo columns on each side of the
  // tile are in the staged window, so lanes 0 and 31 add their row partials
  // in the row pass itself (every lane runs the same 2-element load and two
  // FMAs, with zero weights except on the edge lanes) instead of a scalar pass
  // per warp; the shuffled-in neighbours of the edge lanes get zero weights
  // instead of being zeroed.  Same products, same summation order: bitwise the
  // scalar pass's result.
  constexpr bool INLINE_HALO = MODE == kStageTapeTile && !MSE;
  float wxe[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) wxe[j] = wx[j];
  float hw0 = 0.f, hw1 = 0.f;
  int hoff = 4 + 4 * lane;
  if (INLINE_HALO) {
    if (lane == 0) {
      hw0 = wx[0];
      hw1 = wx[1];
      wxe[0] = wxe[1] = 0.f;
      hoff = 2;
    }
    if (lane == 31) {
      hw0 = wx[6];
      hw1 = wx[7];
      wxe[6] = wxe[7] = 0.f;
      hoff = 4 + THX;
    }
  }

  float lsum = 0.f, chk = 0.f;
  const float scale2 = a.scale2;
  // gather row yl, its coefficient rows interpolated horizontally (lo, hi)
  // and the vertical weight f
  auto do_row = [&](int yl, const float (&alo)[4], const float (&ahi)[4], const float (&blo)[4],
                    const float (&bhi)[4], float f) {
    const int Y = Yg + yl;
    const bool in = col_ok && Y >= 0 && Y < a.H;
    const int64_t off = (int64_t)Y * a.W + X0;  // one address for the 3 accesses
    float4 g4 = make_float4(0.f, 0.f, 0.f, 0.f), t4 = g4;
    if constexpr (MODE == kStageTapeTile) {  // zeros outside the image (TMA)
      g4 = *reinterpret_cast<const float4*>(tG + yl * HTW + 4 + 4 * lane);
      t4 = *reinterpret_cast<const float4*>(tT + yl * HTW + 4 + 4 * lane);
    } else if (in) {
      g4 = __ldg(reinterpret_cast<const float4*>(G + off));
      t4 = __ldg(reinterpret_cast<const float4*>(T + off));
    }
    const float gv[4] = {g4.x, g4.y, g4.z, g4.w}, tv[4] = {t4.x, t4.y, t4.z, t4.w};
    const bool own = in && yl >= 2 && yl < 2 + THY;
    float d[4], q[4], dh[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float Ah = alo[j] + f * (ahi[j] - alo[j]);
      if (MSE) {
        const float Bh = blo[j] + f * (bhi[j] - blo[j]);
        const float o = Bh + Ah * gv[j];
        const float e = o - tv[j];
        d[j] = in ? scale2 * e : 0.f;
        if (own) {
          lsum = fmaf(e, e, lsum);
          chk = fmaf(o, 0.f, chk);  // NaN iff an output is not finite
        }
      } else {
        d[j] = tv[j];  // d_out (0 outside)
      }
      q[j] = d[j] * gv[j];
      dh[j] = d[j] * Ah;
    }
    if (own) *reinterpret_cast<float4*>(DH + off) = make_float4(dh[0], dh[1], dh[2], dh[3]);
    float dl0 = __shfl_up_sync(0xffffffffu, d[2], 1), dl1 = __shfl_up_sync(0xffffffffu, d[3], 1);
    float ql0 = __shfl_up_sync(0xffffffffu, q[2], 1), ql1 = __shfl_up_sync(0xffffffffu, q[3], 1);
    float dr0 = __shfl_down_sync(0xffffffffu, d[0], 1), dr1 = __shfl_down_sync(0xffffffffu, d[1], 1);
    float qr0 = __shfl_down_sync(0xffffffffu, q[0], 1), qr1 = __shfl_down_sync(0xffffffffu, q[1], 1);
    if (!INLINE_HALO) {
      if (lane == 0) dl0 = dl1 = ql0 = ql1 = 0.f;  // halo columns: the scalar pass
      if (lane == 31) dr0 = dr1 = qr0 = qr1 = 0.f;
    }
    const float dd[8] = {dl0, dl1, d[0], d[1], d[2], d[3], dr0, dr1};
    const float qq[8] = {ql0, ql1, q[0], q[1], q[2], q[3], qr0, qr1};
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      s1 = fmaf(wxe[j], dd[j], s1);
      s2 = fmaf(wxe[j], qq[j], s2);
    }
    if constexpr (INLINE_HALO) {
      const float2 ht = *reinterpret_cast<const float2*>(tT + yl * HTW + hoff);
      const float2 hg = *reinterpret_cast<const float2*>(tG + yl * HTW + hoff);
      s1 += fmaf(hw1, ht.y, hw0 * ht.x);
      s2 += fmaf(hw1, ht.y * hg.y, hw0 * (ht.x * hg.x));
    }
    if (!in) s1 = s2 = 0.f;
    R1[yl * TLX + lane] = s1;
    R2[yl * TLX + lane] = s2;
  };

  {
    float HA[3][4], HB[3][4];  // coefficient rows 2w, 2w+1, 2w+2
#pragma unroll
    for (int q = 0; q < 3; ++q) hrow2(2 * warp + q, HA[q], HB[q]);
    const int Yb = Yg + 8 * warp;
    if (Yb >= 2 && Yb + 7 <= 4 * a.h - 3 && Yb + 7 < a.H) {
      // interior rows (warp-uniform): rows 0..3 between coefficient rows
      // 2w, 2w+1 and rows 4..7 between 2w+1, 2w+2, f = 1/8, 3/8, 5/8, 7/8
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int q0 = t >> 2;
        do_row(8 * warp + t, HA[q0], HA[q0 + 1], HB[q0], HB[q0 + 1], (2 * (t & 3) + 1) * 0.125f);
      }
    } else {
#pragma unroll 1
      for (int t = 0; t < 8; ++t) {
        const int Y = Yb + t;
        float alo[4], ahi[4], blo[4], bhi[4], f = 0.f;
        int ql = 0, qh = 0;
        if (Y >= 0 && Y < a.H) {
          const Tap ty = tap4(Y, a.h);
          ql = ty.lo - (i0 - 1) - 2 * warp;  // in 0..2 (clamped taps stay inside)
          qh = ty.hi - (i0 - 1) - 2 * warp;
          f = ty.f;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          alo[j] = ql == 0 ? HA[0][j] : (ql == 1 ? HA[1][j] : HA[2][j]);
          ahi[j] = qh == 0 ? HA[0][j] : (qh == 1 ? HA[1][j] : HA[2][j]);
          blo[j] = ql == 0 ? HB[0][j] : (ql == 1 ? HB[1][j] : HB[2][j]);
          bhi[j] = qh == 0 ? HB[0][j] : (qh == 1 ? HB[1][j] : HB[2][j]);
        }
        do_row(8 * warp + t, alo, ahi, blo, bhi, f);
      }
    }
  }
  if (extra) {  // gather row THY + warp: coefficient rows TLY, TLY + 1
    if constexpr (MODE == kStageTapeTile) tma::mbar_wait(&gbar[kTileGroups - 1], 0);
    float HA[2][4], HB[2][4];
    hrow2(TLY, HA[0], HB[0]);
    hrow2(TLY + 1, HA[1], HB[1]);
    const int Y = Yg + THY + warp;
    float f = (2 * warp + 1) * 0.125f;
    int ql = 0, qh = 1;
    if (Y >= 0 && Y < a.H) {
      const Tap ty = tap4(Y, a.h);
      ql = ty.lo - (i0 - 1) - TLY;
      qh = ty.hi - (i0 - 1) - TLY;
      f = ty.f;
    }
    float alo[4], ahi[4], blo[4], bhi[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      alo[j] = ql == 0 ? HA[0][j] : HA[1][j];
      ahi[j] = qh == 0 ? HA[0][j] : HA[1][j];
      blo[j] = ql == 0 ? HB[0][j] : HB[1][j];
      bhi[j] = qh == 0 ? HB[0][j] : HB[1][j];
    }
    do_row(THY + warp, alo, ahi, blo, bhi, f);
  }
  __syncwarp();
  // halo columns: hr columns 4k0-2, 4k0-1 (into lr column k0's partial) and
  // 4k0+128, 4k0+129 (into k0+31's), one (row, side) item per lane
  if constexpr (!INLINE_HALO) {
    const int nrow = extra ? 9 : 8;
    if (lane < 2 * nrow) {
      const int ri = lane >> 1, side = lane & 1;
      const int yl = ri < 8 ? 8 * warp + ri : THY + warp;
      const int Y = Yg + yl;
      const int kk = side ? k0 + TLX - 1 : k0;
      const int Xa = side ? 4 * k0 + THX : 4 * k0 - 2;
      if (Y >= 0 && Y < a.H && kk < a.w) {
        const Tap ty = tap4(Y, a.h);
        const float* A0 = sm.As + (ty.lo - (i0 - 1)) * CAP;
        const float* A1 = sm.As + (ty.hi - (i0 - 1)) * CAP;
        const float* B0 = sm.Bs + (ty.lo - (i0 - 1)) * CAP;
        const float* B1 = sm.Bs + (ty.hi - (i0 - 1)) * CAP;
        float s1 = 0.f, s2 = 0.f;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int X = Xa + c;
          if (X < 0 || X >= a.W) continue;
          const Tap tx = tap4(X, a.w);
          const int cl = tx.lo - (k0 - 1), ch = tx.hi - (k0 - 1);
          // horizontal then vertical, as the row path
          float g, t;
          if constexpr (MODE == kStageTapeTile) {
            g = tG[yl * HTW + X - (4 * k0 - 4)];
            t = tT[yl * HTW + X - (4 * k0 - 4)];
          } else {
            g = __ldg(G + (int64_t)Y * a.W + X);
            t = __ldg(T + (int64_t)Y * a.W + X);
          }
          float dv = t;  // d_out
          if (MSE) {
            const float al = A0[cl] + tx.f * (A0[ch] - A0[cl]);
            const float ah = A1[cl] + tx.f * (A1[ch] - A1[cl]);
            const float bl = B0[cl] + tx.f * (B0[ch] - B0[cl]);
            const float bh = B1[cl] + tx.f * (B1[ch] - B1[cl]);
            const float Au = al + ty.f * (ah - al), Bu = bl + ty.f * (bh - bl);
            dv = scale2 * ((Bu + Au * g) - t);
          }
          float wgt = 0.f;
          if (tx.lo == kk) wgt += 1.f - tx.f;
          if (tx.hi == kk) wgt += tx.f;
          s1 += wgt * dv;
          s2 += wgt * (dv * g);
        }
        const int o = yl * TLX + (side ? TLX - 1 : 0);
        R1[o] += s1;
        R2[o] += s2;
      }
    }
  }
  // loss partial: warp sums (float64), combined in warp order below
  if (MSE) {
    double v = (double)lsum;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp] = v;
  }
  __syncthreads();
  // column pass: db[i][k] = sum_Y wy(Y, i) R1[Y][k] (as k_joint_bwd_hr)
  for (int it = threadIdx.x; it < TLY * TLX; it += NT) {
    const int il = it / TLX, kl = it - il * TLX;
    const int i = i0 + il, kc = k0 + kl;
    if (i >= a.h || kc >= a.w) continue;
    float s1 = 0.f, s2 = 0.f;
    if (i >= 1 && i <= a.h - 2 && 4 * i + 5 < a.H) {
      constexpr float wy[8] = {0.125f, 0.375f, 0.625f, 0.875f, 0.875f, 0.625f, 0.375f, 0.125f};
      const int yl0 = 4 * (i - i0);
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        s1 += wy[t] * R1[(yl0 + t) * TLX + kl];
        s2 += wy[t] * R2[(yl0 + t) * TLX + kl];
      }
    } else {
#pragma unroll
      for (int dy = -2; dy <= 5; ++dy) {
        const int Y = 4 * i + dy;
        if (Y < 0 || Y >= a.H) continue;
        const Tap ty = tap4(Y, a.h);
        float wgt = 0.f;
        if (ty.lo == i) wgt += 1.f - ty.f;
        if (ty.hi == i) wgt += ty.f;
        const int yl = Y - Yg;
        s1 += wgt * R1[yl * TLX + kl];
        s2 += wgt * R2[yl * TLX + kl];
      }
    }
    const int64_t o = p * (int64_t)a.h * a.w + (int64_t)i * a.w + kc;
    a.db[o] = s1;
    a.dA[o] = s2;
  }
  if (MSE && threadIdx.x == 0) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) s += red[w];
    a.loss_part[(p * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = s;
  }
  if (degen) flag(a.status, GF_STATUS_DEGENERATE);
  if (chk != 0.f) flag(a.status, GF_STATUS_NONFINITE_OUTPUT);
}

template <int RAD, int MINB, bool MSE>
__global__ void __launch_bounds__(NT, MINB) k_joint_mse_hr(MseHrArgs a) {
  mse_hr_body<RAD, MSE, kStageLdg>(a, nullptr, nullptr);
}

// the backward hr pass on the forward's tape of slopes (no window moments)
template <int RAD, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_joint_mse_hr_a(MseHrArgs a) {
  mse_hr_body<RAD, false, kStageTape>(a, nullptr, nullptr);
}

// ... with the gather window of hr_x and d_out staged by TMA (tmG, tmD:
// (136, 68) boxes of the high-res planes).  MSE: the fused training step on
// the coefficients of k_joint_coeffs (A and b), tmD over the target.
// TY = 8: 32-row tiles of 128 threads (52 KB of shared memory: 4 independent
// CTAs per SM instead of 2)
template <int RAD, int MINB, bool MSE = false, int TY = TLY>
__global__ void __launch_bounds__(32 * (TY / 2), MINB)
    k_joint_mse_hr_at(const __grid_constant__ CUtensorMap tmG,
                      const __grid_constant__ CUtensorMap tmD, MseHrArgs a) {
  mse_hr_body<RAD, MSE, kStageTapeTile, TY>(a, &tmG, &tmD);
}

// A and b of every low-res cell (the fused training step's coefficient tape):
// the forward's coefficient phase on 16 x 32 blocks, own cells written
template <int RAD, int VCH = 0, int HCH = 16>
__global__ void __launch_bounds__(NT, 4) k_joint_coeffs(FwdArgs a, float* A_out, float* B_out) {
  extern __shared__ float4 smem4[];
  const SmemCoef sm = carve(reinterpret_cast<float*>(smem4), RAD);
  const int64_t p = blockIdx.z;
  const int i0 = blockIdx.y * TLY, k0 = blockIdx.x * TLX;
  bool degen = false;
  lr_coeffs<RAD, true, VCH, HCH>(a.lr_x + p * (int64_t)a.h * a.w, a.lr_y + p * (int64_t)a.h * a.w,
                                 a.h, a.w, i0, k0, a.eps, sm, degen);
  for (int it = threadIdx.x; it < TLY * TLX; it += NT) {
    const int il = it / TLX, kl = it - il * TLX;
    const int i = i0 + il, kk = k0 + kl;
    if (i < a.h && kk < a.w) {
      const int64_t o = p * (int64_t)a.h * a.w + (int64_t)i * a.w + kk;
      A_out[o] = sm.As[(il + 1) * CAP + kl + 1];
      B_out[o] = sm.Bs[(il + 1) * CAP + kl + 1];
    }
  }
  if (degen) flag(a.status, GF_STATUS_DEGENERATE);
}

template <int RAD, int MINB, bool MSE>
__global__ void __launch_bounds__(NT, MINB)
    k_joint_mse_hr_t(const __grid_constant__ CUtensorMap tmX,
                     const __grid_constant__ CUtensorMap tmY, MseHrArgs a) {
  mse_hr_body<RAD, MSE, kStageTma>(a, &tmX, &tmY);
}

// ---------------------------------------------------------------------------
// backward, kernel 2: low-res tail
// ---------------------------------------------------------------------------
constexpr int TL = 32;  // low-res block of the tail kernel

struct BwdLrArgs {
  const float* lr_x;
  const float* lr_y;
  const float* db;
  const float* dA;
  float* d_lr_x;
  float* d_lr_y;
  int h, w, r;
  float eps;
};

__host__ __device__ inline size_t bwd_lr_smem_floats(int r) {
  const int NI = TL + 4 * r;   // inputs x, y
  const int NM = TL + 2 * r;   // moment region
  // xs, ys [NI][NI]; vsum [4][NM][NI]; kf [4][NM][NM]; (vs2 [4][TL][NM] reuses vsum)
  return (size_t)2 * NI * NI + (size_t)4 * NM * NI + (size_t)4 * NM * NM;
}

template <int RAD>
__global__ void __launch_bounds__(NT) k_joint_bwd_lr(BwdLrArgs a) {
  extern __shared__ float4 smem4[];
  constexpr int r = RAD;
  const int NI = TL + 4 * r, NM = TL + 2 * r;
  float* xs = reinterpret_cast<float*>(smem4);
  float* ys = xs + NI * NI;
  float* vsum = ys + NI * NI;      // [4][NM][NI], later [4][TL][NM]
  float* kf = vsum + 4 * NM * NI;  // [4][NM][NM]
  const int64_t p = blockIdx.z;
  const int i0 = blockIdx.y * TL, k0 = blockIdx.x * TL;
  const int h = a.h, w = a.w;
  const int tid = threadIdx.x;
  const float* __restrict__ X = a.lr_x + p * (int64_t)h * w;
  const float* __restrict__ Yp = a.lr_y + p * (int64_t)h * w;
  const float* __restrict__ DB = a.db + p * (int64_t)h * w;
  const float* __restrict__ DA = a.dA + p * (int64_t)h * w;
  const int sy_ = min(i0, h - 1), sx_ = min(k0, w - 1);
  const float sx = __ldg(X + (int64_t)sy_ * w + sx_);
  const float sy = __ldg(Yp + (int64_t)sy_ * w + sx_);
  // inputs over [i0-2r, i0+TL+2r)^2, shifted, zero outside the image
  {  // all loads in flight before the first store (one latency per block)
    constexpr int NIc = TL + 4 * r;
    constexpr int NE = (NIc * NIc + NT - 1) / NT;
    float xv[NE], yv[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const int idx = tid + e * NT;
      const int row = idx / NIc, col = idx - row * NIc;
      const int gy = i0 - 2 * r + row, gx = k0 - 2 * r + col;
      const bool ok = idx < NIc * NIc && gy >= 0 && gy < h && gx >= 0 && gx < w;
      xv[e] = ok ? __ldg(X + (int64_t)gy * w + gx) - sx : 0.f;
      yv[e] = ok ? __ldg(Yp + (int64_t)gy * w + gx) - sy : 0.f;
    }
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const int idx = tid + e * NT;
      if (idx < NIc * NIc) {
        xs[idx] = xv[e];
        ys[idx] = yv[e];
      }
    }
  }
  __syncthreads();
  // vertical sums for moment rows m in [0, NM) (global i0 - r + m): input rows [m, m+2r]
  {
    const int nch = max(1, min(NM, NT / NI));
    const int rc = (NM + nch - 1) / nch;
    for (int it = tid; it < NI * nch; it += NT) {
      const int col = it % NI, ch = it / NI;
      const int m0 = ch * rc, m1 = min(NM, m0 + rc);
      if (m0 >= m1) continue;
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
      for (int d = 0; d < 2 * r; ++d) {
        const float xv = xs[(m0 + d) * NI + col], yv = ys[(m0 + d) * NI + col];
        s0 += xv; s1 += yv; s2 += xv * xv; s3 += xv * yv;
      }
      for (int m = m0; m < m1; ++m) {
        const float xv = xs[(m + 2 * r) * NI + col], yv = ys[(m + 2 * r) * NI + col];
        s0 += xv; s1 += yv; s2 += xv * xv; s3 += xv * yv;
        vsum[(0 * NM + m) * NI + col] = s0;
        vsum[(1 * NM + m) * NI + col] = s1;
        vsum[(2 * NM + m) * NI + col] = s2;
        vsum[(3 * NM + m) * NI + col] = s3;
        const float xo = xs[m * NI + col], yo = ys[m * NI + col];
        s0 -= xo; s1 -= yo; s2 -= xo * xo; s3 -= xo * yo;
      }
    }
  }
  __syncthreads();
  // horizontal sums + moment gradients / N at moment cells (m, n)
  {
    const int nch = max(1, min(NM, NT / NM));
    const int cc = (NM + nch - 1) / nch;
    for (int it = tid; it < NM * nch; it += NT) {
      const int m = it / nch, ch = it - m * nch;
      const int n0 = ch * cc, n1 = min(NM, n0 + cc);
      if (n0 >= n1) continue;
      const int gy = i0 - r + m;
      const bool row_ok = gy >= 0 && gy < h;
      const float* v0 = vsum + (0 * NM + m) * NI;
      const float* v1 = vsum + (1 * NM + m) * NI;
      const float* v2 = vsum + (2 * NM + m) * NI;
      const float* v3 = vsum + (3 * NM + m) * NI;
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
      for (int d = 0; d < 2 * r; ++d) {
        s0 += v0[n0 + d]; s1 += v1[n0 + d]; s2 += v2[n0 + d]; s3 += v3[n0 + d];
      }
      const float ny = row_ok ? (float)wlen(gy, h, r) : 1.f;
      for (int n = n0; n < n1; ++n) {
        s0 += v0[n + 2 * r]; s1 += v1[n + 2 * r]; s2 += v2[n + 2 * r]; s3 += v3[n + 2 * r];
        const int gx = k0 - r + n;
        float k_cov = 0.f, k_var = 0.f, k_mx = 0.f, k_my = 0.f;
        if (row_ok && gx >= 0 && gx < w) {
          const float inv = fast_rcp(ny * (float)wlen(gx, w, r));
          const float mx = s0 * inv, my = s1 * inv;  // shifted means
          const float var = s2 * inv - mx * mx;
          const float cov = s3 * inv - mx * my;
          const float rden = fast_rcp(var + a.eps);
          const float A = cov * rden;
          const float ux = mx + sx, uy = my + sy;  // true means
          const int64_t o = (int64_t)gy * w + gx;
          const float dbv = __ldg(DB + o);
          const float dAv = __ldg(DA + o) + (-dbv * ux);   // gf/guided.py:278-280
          const float d_cov = dAv * rden;                   // :242
          const float d_var = -dAv * cov * (rden * rden);   // :243
          const float d_my = dbv + (-d_cov * ux);           // :245-247
          const float d_mx = (-dbv * A) + (-d_cov * uy) + (-2.f * d_var * ux);  // :248-252
          k_cov = d_cov * inv;
          k_var = d_var * inv;
          k_mx = d_mx * inv;
          k_my = d_my * inv;
        }
        kf[(0 * NM + m) * NM + n] = k_cov;
        kf[(1 * NM + m) * NM + n] = k_var;
        kf[(2 * NM + m) * NM + n] = k_mx;
        kf[(3 * NM + m) * NM + n] = k_my;
        s0 -= v0[n]; s1 -= v1[n]; s2 -= v2[n]; s3 -= v3[n];
      }
    }
  }
  __syncthreads();
  // box adjoint (M^T g = box_sum(g/N)): vertical sums of kf for own rows -> vsum as [4][TL][NM]
  {
    const int nch = max(1, min(TL, NT / (4 * NM)));
    const int rc = (TL + nch - 1) / nch;
    for (int it = tid; it < 4 * NM * nch; it += NT) {
      const int ch = it / (4 * NM), rem = it - ch * 4 * NM;
      const int f = rem / NM, n = rem - f * NM;
      const int m0 = ch * rc, m1 = min(TL, m0 + rc);
      if (m0 >= m1) continue;
      const float* src = kf + f * NM * NM + n;
      float s = 0.f;
      for (int d = 0; d < 2 * r; ++d) s += src[(m0 + d) * NM];
      for (int m = m0; m < m1; ++m) {
        s += src[(m + 2 * r) * NM];
        vsum[(f * TL + m) * NM + n] = s;
        s -= src[m * NM];
      }
    }
  }
  __syncthreads();
  // horizontal sums + outputs
  {
    constexpr int nch = NT / TL;  // 8
    constexpr int cc = TL / nch;  // 4
    for (int it = tid; it < TL * nch; it += NT) {
      const int m = it / nch, ch = it - m * nch;
      const int gy = i0 + m;
      if (gy >= h) continue;
      const int n0 = ch * cc;
      const float* v0 = vsum + (0 * TL + m) * NM;
      const float* v1 = vsum + (1 * TL + m) * NM;
      const float* v2 = vsum + (2 * TL + m) * NM;
      const float* v3 = vsum + (3 * TL + m) * NM;
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
      for (int d = 0; d < 2 * r; ++d) {
        s0 += v0[n0 + d]; s1 += v1[n0 + d]; s2 += v2[n0 + d]; s3 += v3[n0 + d];
      }
#pragma unroll
      for (int n = n0; n < n0 + cc; ++n) {
        s0 += v0[n + 2 * r]; s1 += v1[n + 2 * r]; s2 += v2[n + 2 * r]; s3 += v3[n + 2 * r];
        const int gx = k0 + n;
        if (gx < w) {
          const float xv = xs[(m + 2 * r) * NI + n + 2 * r] + sx;
          const float yv = ys[(m + 2 * r) * NI + n + 2 * r] + sy;
          const int64_t o = p * (int64_t)h * w + (int64_t)gy * w + gx;
          a.d_lr_y[o] = s0 * xv + s3;                      // gf/guided.py:256-258
          a.d_lr_x[o] = s0 * yv + 2.f * s1 * xv + s2;       // :259-263
        }
        s0 -= v0[n]; s1 -= v1[n]; s2 -= v2[n]; s3 -= v3[n];
      }
    }
  }
}

}  // namespace jf

thread_local int g_joint_lr_variant = 0;
thread_local int g_joint_mse_variant = 0;
thread_local int g_joint_bwd_hr_tile = 16;  // low-res rows per tile of the tape hr pass (16 or 8)
thread_local int g_joint_fwd_variant = 0;
thread_local int g_joint_bwd_hr_variant = 0;

bool fused_joint_ok(int64_t B, int64_t C, int64_t h, int64_t w, int64_t H, int64_t W, int r) {
  if (H != 4 * h || W != 4 * w) return false;
  if (r < 0 || r > jf::kMaxRadius) return false;
  if (h < 2 || w < 2) return false;
  if (H > (1 << 30) || W > (1 << 30)) return false;
  if ((h + jf::TLY - 1) / jf::TLY > 65535 || B * C > 65535) return false;
  return true;
}

static void set_smem(const void* fn, size_t bytes) {
  if (bytes > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

// kernels are instantiated per radius (0..kMaxRadius) so window loops unroll
struct JointFns {
  const void* fwd;
  const void* bwd_hr;
  const void* bwd_lr;
  const void* mse_hr;
  const void* hr_pass;
  // TMA-staged low-res blocks (w % 4 == 0): forward, fused step, hr pass
  const void* fwd_t;
  const void* mse_hr_t;
  const void* hr_pass_t;
  size_t tma_floats;  // tma_coef_floats + alignment slack
  const void* hr_pass_a;   // hr pass on the forward's tape of slopes
  const void* hr_pass_at;  // ... with the gather window staged by TMA
  const void* hr_pass_at8;  // ... on 32-row tiles (4 CTAs per SM)
  const void* coeffs;      // A, b of every low-res cell (fused step)
  const void* mse_hr_at;   // fused step on them, gather window by TMA
};

template <int RAD>
static JointFns joint_fns() {
  // r >= 2: fewer, longer coefficient-pass chunks (each pays a 2r warm-up):
  // 8 column chunks per row, and 2 row chunks for r >= 5 (config 3: r = 2
  // 1352 -> 1296 us, r = 4 1419 -> 1348 us, r = 8 1571 -> 1500 us)
  const void *fwd, *fwd_t, *coeffs;
  if constexpr (RAD >= 5)
    coeffs = (const void*)jf::k_joint_coeffs<RAD, 2, 8>;
  else if constexpr (RAD >= 2)
    coeffs = (const void*)jf::k_joint_coeffs<RAD, 0, 8>;
  else
    coeffs = (const void*)jf::k_joint_coeffs<RAD>;
  if constexpr (RAD >= 5) {
    fwd = (const void*)jf::k_joint_fwd<RAD, 2, 8>;
    fwd_t = (const void*)jf::k_joint_fwd_t<RAD, 2, 8>;
  } else if constexpr (RAD >= 2) {
    fwd = (const void*)jf::k_joint_fwd<RAD, 0, 8>;
    fwd_t = (const void*)jf::k_joint_fwd_t<RAD, 0, 8>;
  } else {
    fwd = (const void*)jf::k_joint_fwd<RAD>;
    fwd_t = (const void*)jf::k_joint_fwd_t<RAD>;
  }
  return {fwd, (const void*)jf::k_joint_bwd_hr<RAD>, (const void*)jf::k_joint_bwd_lr<RAD>,
          (const void*)jf::k_joint_mse_hr<RAD, 3, true>,
          (const void*)jf::k_joint_mse_hr<RAD, 4, false>, fwd_t,
          (const void*)jf::k_joint_mse_hr_t<RAD, 3, true>,
          (const void*)jf::k_joint_mse_hr_t<RAD, 4, false>,
          (size_t)jf::tma_coef_floats<RAD>() + 32, (const void*)jf::k_joint_mse_hr_a<RAD, 4>,
          (const void*)jf::k_joint_mse_hr_at<RAD, 2>,
          (const void*)jf::k_joint_mse_hr_at<RAD, 4, false, 8>, coeffs,
          (const void*)jf::k_joint_mse_hr_at<RAD, 2, true>};
}

static JointFns pick_joint(int r) {
  switch (r) {
    case 0: return joint_fns<0>();
    case 1: return joint_fns<1>();
    case 2: return joint_fns<2>();
    case 3: return joint_fns<3>();
    case 4: return joint_fns<4>();
    case 5: return joint_fns<5>();
    case 6: return joint_fns<6>();
    case 7: return joint_fns<7>();
    case 8: return joint_fns<8>();
    case 9: return joint_fns<9>();
    case 10: return joint_fns<10>();
    case 11: return joint_fns<11>();
    default: return joint_fns<12>();
  }
}

static void launch(const void* fn, dim3 grid, size_t smem, cudaStream_t s, void* arg) {
  void* args[] = {arg};
  cudaLaunchKernel(fn, grid, dim3(jf::NT), args, smem, s);
}

// persistent TMA forward: kernel and dynamic shared memory per radius
struct FwdTma {
  const void* fn;
  size_t smem;
};

template <int RAD>
static FwdTma fwd_tma_info() {
  constexpr int NS = 2;
  if constexpr (RAD >= 5)
    return {(const void*)jf::k_joint_fwd_tma<RAD, NS, 1, 2, 8>, jf::fwd_tma_smem_bytes<RAD, NS>()};
  else if constexpr (RAD >= 2)
    return {(const void*)jf::k_joint_fwd_tma<RAD, NS, 2, 0, 8>, jf::fwd_tma_smem_bytes<RAD, NS>()};
  else
    return {(const void*)jf::k_joint_fwd_tma<RAD, NS, 2>, jf::fwd_tma_smem_bytes<RAD, NS>()};
}

static FwdTma pick_fwd_tma(int r) {
  switch (r) {
    case 0: return fwd_tma_info<0>();
    case 1: return fwd_tma_info<1>();
    case 2: return fwd_tma_info<2>();
    case 3: return fwd_tma_info<3>();
    case 4: return fwd_tma_info<4>();
    case 5: return fwd_tma_info<5>();
    case 6: return fwd_tma_info<6>();
    case 7: return fwd_tma_info<7>();
    case 8: return fwd_tma_info<8>();
    case 9: return fwd_tma_info<9>();
    case 10: return fwd_tma_info<10>();
    case 11: return fwd_tma_info<11>();
    default: return fwd_tma_info<12>();
  }
}

// true when launched (the low-res rows must be 16-byte multiples for TMA).
// Variant hook 10 only: measured slower than the tile kernel at every config
// (config 3 r = 1: 1515 vs 1276 us; r = 8: 2397 vs 1534 us; config 4a's
// forward 3579 vs 2984 us; config 0 18.0 vs 21.7 us), because two resident
// CTAs per SM keep less of the image in flight than four tile CTAs that
// issue their 32 KB of high-res loads up front.
static bool fused_joint_fwd_tma(const float* lr_x, const float* lr_y, const float* hr_x,
                                float* out, int64_t P, int64_t h, int64_t w, int64_t H, int64_t W,
                                int r, float eps, uint32_t* status, cudaStream_t s) {
  if (w % 4 != 0 || g_joint_fwd_variant != 10) return false;
  const FwdTma F = pick_fwd_tma(r);
  const int RI = jf::RA + 2 * r, PADL = (1 + r + 3) / 4 * 4;
  const int LP = (PADL + jf::TLX + 1 + r + 3) / 4 * 4;  // as jf::TmaGeo
  CUtensorMap tmG, tmX, tmY;
  if (!tma::make_plane_map(&tmG, hr_x, W, H, P, jf::THX, jf::THY) ||
      !tma::make_plane_map(&tmX, lr_x, w, h, P, LP, RI) ||
      !tma::make_plane_map(&tmY, lr_y, w, h, P, LP, RI))
    return false;
  const LaunchCfg lc = launch_cfg(F.fn, jf::NT, F.smem);
  int tiles_x = (int)((w + jf::TLX - 1) / jf::TLX), tiles_y = (int)((h + jf::TLY - 1) / jf::TLY);
  const int64_t nt = (int64_t)tiles_x * tiles_y * P;
  if (nt > 0x7fffffff) return false;
  int ntiles = (int)nt;
  const int64_t grid = std::min<int64_t>(nt, (int64_t)lc.sms * lc.per_sm);
  jf::FwdArgs a{lr_x, lr_y, hr_x, out, (int)h, (int)w, (int)H, (int)W, r, eps, status};
  void* args[] = {&tmG, &tmX, &tmY, &a, &tiles_x, &tiles_y, &ntiles};
  cudaLaunchKernel(F.fn, dim3((unsigned)grid), dim3(jf::NT), args, F.smem, s);
  return true;
}

// tensor maps of the low-res x, y planes with the (LP, RI) halo box of the
// TMA-staged tile kernels; false when TMA does not apply (w % 4 != 0).
// The TMA-staged kernels (variant hook 11 of the forward, hr pass and fused
// step) are bitwise equal to the __ldg-staged defaults but measured ~5 %
// slower (config 4a: fwd 3.07 vs 2.92 ms, bwd 6.25 vs 5.99 ms; config 2's
// fused step 0.475 vs 0.455 ms): the in-place box reads re-apply the shift
// and the image mask to every element the vertical pass touches (about
// three times per element) where the staging pass applies them once.
static bool lr_maps(CUtensorMap* tmX, CUtensorMap* tmY, const float* lr_x, const float* lr_y,
                    int64_t P, int64_t h, int64_t w, int r) {
  if (w % 4 != 0) return false;
  const int RI = jf::RA + 2 * r, PADL = (1 + r + 3) / 4 * 4;
  const int LP = (PADL + jf::TLX + 1 + r + 3) / 4 * 4;  // as jf::TmaGeo
  return tma::make_plane_map(tmX, lr_x, w, h, P, LP, RI) &&
         tma::make_plane_map(tmY, lr_y, w, h, P, LP, RI);
}

// A, b of every low-res cell: the register-segment walk (r <= 8, w % 4 == 0),
// else the tile kernel's coefficient phase on 16 x 32 blocks
void fused_joint_coeffs(const float* lr_x, const float* lr_y, float* A, float* B, int64_t P,
                        int64_t h, int64_t w, int r, float eps, uint32_t* status, cudaStream_t s) {
  const int v = g_joint_fwd_variant;
  if (v != 21 && seg_joint_coeffs_ok(h, w, r)) {
    g_joint_coeffs_sw = v == 22 ? 8 : (v == 24 ? 4 : 0);  // 24: the register walk at 4 per lane
    seg_joint_coeffs(lr_x, lr_y, A, B, P, h, w, r, eps, status, s);
    return;
  }
  const JointFns fns = pick_joint(r);
  dim3 grid((unsigned)((w + jf::TLX - 1) / jf::TLX), (unsigned)((h + jf::TLY - 1) / jf::TLY),
            (unsigned)P);
  jf::FwdArgs fa{lr_x, lr_y, nullptr, nullptr, (int)h, (int)w, (int)(4 * h), (int)(4 * w), r, eps,
                 status};
  const size_t smc = jf::coef_smem_floats(r) * sizeof(float);
  set_smem(fns.coeffs, smc);
  void* cargs[] = {&fa, &A, &B};
  cudaLaunchKernel(fns.coeffs, grid, dim3(jf::NT), cargs, smc, s);
}

// Two-kernel forward: coefficients of every cell (A into the tape when one is
// kept, else into the workspace), then the high-res apply pass on them.
static void fused_joint_fwd_split(const float* lr_x, const float* lr_y, const float* hr_x,
                                  float* out, int64_t P, int64_t h, int64_t w, int64_t H,
                                  int64_t W, int r, float eps, uint32_t* status, cudaStream_t s,
                                  float* A_tape, float* coef_ws) {
  float* Bc = coef_ws;
  float* Ac = A_tape ? A_tape : coef_ws + P * h * w;
  fused_joint_coeffs(lr_x, lr_y, Ac, Bc, P, h, w, r, eps, status, s);
  const int v = g_joint_fwd_variant;
  g_joint_apply_variant = v == 23 || v == 25 || v == 26 ? v - 20 : 0;
  joint_apply(Ac, Bc, hr_x, out, P, h, w, H, W, status, s);
}

void fused_joint_fwd(const float* lr_x, const float* lr_y, const float* hr_x, float* out, int64_t B,
                     int64_t C, int64_t h, int64_t w, int64_t H, int64_t W, int r, float eps,
                     uint32_t* status, cudaStream_t s, float* A_tape, float* coef_ws) {
  if (!A_tape && fused_joint_fwd_tma(lr_x, lr_y, hr_x, out, B * C, h, w, H, W, r, eps, status, s))
    return;
  const JointFns fns = pick_joint(r);
  // Large calls (>= 48 M high-res elements; measured break-even ~ one 3 x 3072^2
  // image) take the two-kernel forward when the caller gave a workspace for
  // the coefficients.  Variant hook: 19 forces the one-kernel tile forward,
  // 20..29 force the split (21 tile-kernel coefficients, 22 8 columns per lane,
  // 23/25/26 CTAs per SM of the apply pass).
  const int fv = g_joint_fwd_variant;
  const bool big = B * C * H * W >= kJointSplitElems;
  if (coef_ws && ((fv == 0 && big) || (fv >= 20 && fv < 30))) {
    fused_joint_fwd_split(lr_x, lr_y, hr_x, out, B * C, h, w, H, W, r, eps, status, s, A_tape,
                          coef_ws);
    return;
  }
  CUtensorMap tmX, tmY;
  if (!A_tape && g_joint_fwd_variant == 11 && lr_maps(&tmX, &tmY, lr_x, lr_y, B * C, h, w, r)) {
    jf::FwdArgs a{lr_x, lr_y, hr_x, out, (int)h, (int)w, (int)H, (int)W, r, eps, status};
    const size_t smem = fns.tma_floats * sizeof(float);
    set_smem(fns.fwd_t, smem);
    dim3 grid((unsigned)((w + jf::TLX - 1) / jf::TLX), (unsigned)((h + jf::TLY - 1) / jf::TLY),
              (unsigned)(B * C));
    void* args[] = {&tmX, &tmY, &a};
    cudaLaunchKernel(fns.fwd_t, grid, dim3(jf::NT), args, smem, s);
    return;
  }
  jf::FwdArgs a{lr_x, lr_y, hr_x, out, (int)h, (int)w, (int)H, (int)W, r, eps, status, A_tape};
  const int tx = (int)((w + jf::TLX - 1) / jf::TLX), ty = (int)((h + jf::TLY - 1) / jf::TLY);
  const size_t smem = jf::coef_smem_floats(r) * sizeof(float);
  const void* fn = fns.fwd;
  // variant hook: coefficient-pass chunking (vertical row chunks x horizontal
  // column chunks per row; 0 = as many row chunks as the threads allow)
  switch (g_joint_fwd_variant * 100 + r) {
    case 108: fn = (const void*)jf::k_joint_fwd<8, 0, 16>; break;
    case 208: fn = (const void*)jf::k_joint_fwd<8, 1, 4>; break;
    case 308: fn = (const void*)jf::k_joint_fwd<8, 2, 4>; break;
    case 408: fn = (const void*)jf::k_joint_fwd<8, 4, 8>; break;
    case 104: fn = (const void*)jf::k_joint_fwd<4, 0, 16>; break;
    case 204: fn = (const void*)jf::k_joint_fwd<4, 2, 8>; break;
    case 304: fn = (const void*)jf::k_joint_fwd<4, 0, 4>; break;
    case 102: fn = (const void*)jf::k_joint_fwd<2, 0, 16>; break;
    case 202: fn = (const void*)jf::k_joint_fwd<2, 2, 8>; break;
    case 302: fn = (const void*)jf::k_joint_fwd<2, 0, 4>; break;
    case 101: fn = (const void*)jf::k_joint_fwd<1, 0, 8>; break;
    case 201: fn = (const void*)jf::k_joint_fwd<1, 2, 8>; break;
    case 301: fn = (const void*)jf::k_joint_fwd<1, 0, 4>; break;
    default: break;
  }
  set_smem(fn, smem);
  dim3 grid((unsigned)tx, (unsigned)ty, (unsigned)(B * C));
  launch(fn, grid, smem, s, &a);
}

size_t fused_joint_bwd_ws_bytes(int64_t B, int64_t C, int64_t h, int64_t w) {
  return (size_t)2 * B * C * h * w * sizeof(float);
}

// the low-res tail of both backward entries
static void joint_lr_tail(const JointFns& fns, const float* lr_x, const float* lr_y,
                          const float* db, const float* dA, float* d_lr_x, float* d_lr_y,
                          int64_t B, int64_t C, int64_t h, int64_t w, int r, float eps,
                          int64_t row0, cudaStream_t s) {
  if (g_joint_lr_variant != 1 && seg_joint_bwd_lr_ok(h, w, r)) {
    seg_joint_bwd_lr(lr_x, lr_y, db, dA, d_lr_x, d_lr_y, B * C, h, w, r, eps, row0, s);
  } else {
    const size_t smem = jf::bwd_lr_smem_floats(r) * sizeof(float);
    set_smem(fns.bwd_lr, smem);
    dim3 grid((unsigned)((w + jf::TL - 1) / jf::TL), (unsigned)((h + jf::TL - 1) / jf::TL),
              (unsigned)(B * C));
    jf::BwdLrArgs a{lr_x, lr_y, db, dA, d_lr_x, d_lr_y, (int)h, (int)w, r, eps};
    launch(fns.bwd_lr, grid, smem, s, &a);
  }
}

void fused_joint_bwd(const float* lr_x, const float* lr_y, const float* hr_x, const float* d_out,
                     float* d_lr_x, float* d_lr_y, float* d_hr_x, int64_t B, int64_t C, int64_t h,
                     int64_t w, int64_t H, int64_t W, int r, float eps, void* ws, int64_t row0,
                     uint32_t* status, cudaStream_t s, const float* A_tape) {
  float* db = (float*)ws;
  float* dA = db + B * C * h * w;
  const JointFns fns = pick_joint(r);
  {
    const size_t smem = jf::bwd_hr_smem_floats(r) * sizeof(float);
    set_smem(fns.bwd_hr, smem);
    dim3 grid((unsigned)((w + jf::TLX - 1) / jf::TLX), (unsigned)((h + jf::TLY - 1) / jf::TLY),
              (unsigned)(B * C));
    if (g_joint_bwd_hr_variant == 1) {  // the two-read tile kernel
      jf::BwdHrArgs a{lr_x, lr_y, hr_x, d_out, d_hr_x, db, dA, (int)h, (int)w, (int)H, (int)W, r,
                      eps, status};
      launch(fns.bwd_hr, grid, smem, s, &a);
    } else {  // single gather pass (d_hr and both adjoints from one read of hr_x,
              // d_out): 736 vs 770 us at 8 x 3 x 3072^2, r = 2 (whole backward)
      const void* fn = fns.hr_pass;
      if (r == 2 && g_joint_bwd_hr_variant == 3) fn = (const void*)jf::k_joint_mse_hr<2, 3, false>;
      if (r == 1 && g_joint_bwd_hr_variant == 3) fn = (const void*)jf::k_joint_mse_hr<1, 3, false>;
      jf::MseHrArgs a{lr_x, lr_y, hr_x, d_out, d_hr_x, db, dA, nullptr, (int)h, (int)w, (int)H,
                      (int)W, r, eps, 0.f, status};
      CUtensorMap tmX, tmY;
      CUtensorMap tmG, tmD;
      if (A_tape && g_joint_bwd_hr_variant == 0 &&
          tma::make_plane_map(&tmG, hr_x, W, H, B * C, jf::HTW, jf::kTileBox) &&
          tma::make_plane_map(&tmD, d_out, W, H, B * C, jf::HTW, jf::kTileBox)) {
        // the forward's slopes, and the gather window by TMA
        a.A_tape = A_tape;
        void* args[] = {&tmG, &tmD, &a};
        if (g_joint_bwd_hr_tile == 8 && (h + 7) / 8 <= 65535) {  // 32-row tiles, 128 threads
          constexpr int TY = 8, GR8 = 4 * TY + 4;
          const size_t sma = 128 + (2 * jf::HTW * (4 * TY + jf::kTileBox) + 2 * (TY + 2) * jf::CAP +
                                    2 * GR8 * jf::TLX) * sizeof(float);
          set_smem(fns.hr_pass_at8, sma);
          dim3 grid8(grid.x, (unsigned)((h + TY - 1) / TY), grid.z);
          cudaLaunchKernel(fns.hr_pass_at8, grid8, dim3(32 * (TY / 2)), args, sma, s);
        } else {
          const size_t sma =
              128 + (2 * jf::HTF + 2 * jf::RA * jf::CAP + 2 * jf::GR * jf::TLX) * sizeof(float);
          set_smem(fns.hr_pass_at, sma);
          cudaLaunchKernel(fns.hr_pass_at, grid, dim3(jf::NT), args, sma, s);
        }
      } else if (A_tape && g_joint_bwd_hr_variant == 12) {  // slopes, global loads
        a.A_tape = A_tape;
        const size_t sma = (2 * jf::RA * jf::CAP + 2 * jf::GR * jf::TLX) * sizeof(float);
        set_smem(fns.hr_pass_a, sma);
        launch(fns.hr_pass_a, grid, sma, s, &a);
      } else if (g_joint_bwd_hr_variant == 11 && lr_maps(&tmX, &tmY, lr_x, lr_y, B * C, h, w, r)) {
        const size_t smt = (fns.tma_floats + 2 * jf::GR * jf::TLX) * sizeof(float);
        set_smem(fns.hr_pass_t, smt);
        void* args[] = {&tmX, &tmY, &a};
        cudaLaunchKernel(fns.hr_pass_t, grid, dim3(jf::NT), args, smt, s);
      } else {
        set_smem(fn, smem);
        launch(fn, grid, smem, s, &a);
      }
    }
  }
  joint_lr_tail(fns, lr_x, lr_y, db, dA, d_lr_x, d_lr_y, B, C, h, w, r, eps, row0, s);
}

// per-CTA loss partials of the fused step: (B C) x tile rows x tile columns
static int64_t mse_tiles(int64_t C, int64_t h, int64_t w) {
  return C * ((h + jf::TLY - 1) / jf::TLY) * ((w + jf::TLX - 1) / jf::TLX);
}

// workspace of the fused step: db, dA (lr), loss partials, then A, b (lr)
size_t fused_joint_mse_ws_bytes(int64_t B, int64_t C, int64_t h, int64_t w) {
  const size_t f = ((size_t)2 * B * C * h * w * sizeof(float) + 255) / 256 * 256;
  const size_t pt = ((size_t)B * mse_tiles(C, h, w) * sizeof(double) + 255) / 256 * 256;
  return f + pt + (size_t)2 * B * C * h * w * sizeof(float);
}

void fused_joint_mse_bwd(const float* lr_x, const float* lr_y, const float* hr_x,
                         const float* target, double* loss, float* d_lr_x, float* d_lr_y,
                         float* d_hr_x, int64_t B, int64_t C, int64_t h, int64_t w, int64_t H,
                         int64_t W, int r, float eps, void* ws, uint32_t* status,
                         cudaStream_t s) {
  float* db = (float*)ws;
  float* dA = db + B * C * h * w;
  double* part =
      (double*)((char*)ws + ((size_t)2 * B * C * h * w * sizeof(float) + 255) / 256 * 256);
  const JointFns fns = pick_joint(r);
  {
    const size_t smem = jf::bwd_hr_smem_floats(r) * sizeof(float);
    // variant hook: CTAs per SM the registers are budgeted for (3 default:
    // 421 us at config 2 vs 507 us for 2 (no spills) and 441 us for 4)
    const void* fn = fns.mse_hr;
    if (r == 1 && g_joint_mse_variant == 2) fn = (const void*)jf::k_joint_mse_hr<1, 2, true>;
    if (r == 1 && g_joint_mse_variant == 4) fn = (const void*)jf::k_joint_mse_hr<1, 4, true>;
    dim3 grid((unsigned)((w + jf::TLX - 1) / jf::TLX), (unsigned)((h + jf::TLY - 1) / jf::TLY),
              (unsigned)(B * C));
    const double per_image = (double)C * (double)H * (double)W;
    jf::MseHrArgs a{lr_x, lr_y, hr_x, target, d_hr_x, db, dA, part, (int)h, (int)w, (int)H,
                    (int)W, r, eps, (float)(2.0 / per_image / (double)B), status};
    CUtensorMap tmX, tmY, tmG, tmT;
    // coefficient tape + TMA gather window: the default for large calls (config
    // 2's filter step 388 vs 436 us for the moments-recomputing kernel, since
    // the coefficients come from the register-segment walk); variant hook 15
    // forces it, 16 forces the moments-recomputing kernel
    const bool big = B * C * H * W >= kJointSplitElems;
    if (((g_joint_mse_variant == 0 && big) || g_joint_mse_variant == 15) &&
        tma::make_plane_map(&tmG, hr_x, W, H, B * C, jf::HTW, jf::kTileBox) &&
        tma::make_plane_map(&tmT, target, W, H, B * C, jf::HTW, jf::kTileBox)) {
      // coefficient tape (A, b of every cell), then the hr pass on it with the
      // gather window of hr_x and the target staged by TMA
      float* Acoef = (float*)((char*)part + ((size_t)B * mse_tiles(C, h, w) * sizeof(double) + 255) /
                                                 256 * 256);
      float* Bcoef = Acoef + B * C * h * w;
      fused_joint_coeffs(lr_x, lr_y, Acoef, Bcoef, B * C, h, w, r, eps, status, s);
      a.A_tape = Acoef;
      a.B_tape = Bcoef;
      const size_t sma =
          128 + (2 * jf::HTF + 2 * jf::RA * jf::CAP + 2 * jf::GR * jf::TLX) * sizeof(float);
      set_smem(fns.mse_hr_at, sma);
      void* args[] = {&tmG, &tmT, &a};
      cudaLaunchKernel(fns.mse_hr_at, grid, dim3(jf::NT), args, sma, s);
    } else if (g_joint_mse_variant == 11 && lr_maps(&tmX, &tmY, lr_x, lr_y, B * C, h, w, r)) {
      const size_t smt = (fns.tma_floats + 2 * jf::GR * jf::TLX) * sizeof(float);
      set_smem(fns.mse_hr_t, smt);
      void* args[] = {&tmX, &tmY, &a};
      cudaLaunchKernel(fns.mse_hr_t, grid, dim3(jf::NT), args, smt, s);
    } else {
      set_smem(fn, smem);
      launch(fn, grid, smem, s, &a);
    }
    mse_final(part, loss, B, (int)mse_tiles(C, h, w), per_image, s);
  }
  joint_lr_tail(fns, lr_x, lr_y, db, dA, d_lr_x, d_lr_y, B, C, h, w, r, eps, 0, s);
}

}  // namespace gfb
