// Fast guided filter forward, second kernel of the two-kernel split
// (gf/guided.py:170-178: bilinear_resize of the low-res slope and intercept,
// then affine_combine, gf/_kernels.py:104-124), fp32 NCHW, factor 4, sm_100a.
//
// k_joint_coeffs (gf_fused_joint.cu) writes A and b of every low-res cell
// once; k_joint_apply streams the high-res image.  Per 64 x 128 tile of one
// plane (256 threads, a warp per 8 rows, a lane per 4 columns):
//   1. every thread issues its 8 x 128-bit guide loads (held in registers);
//   2. the tile's 18 x 34 coefficient cells of A and of b (1-cell bilinear
//      halo included) arrive by TWO TMA copies issued by one elected thread:
//      boxes of 18 rows x 40 columns starting at the 16-byte column k0 - 4,
//      zero-filled outside the image, where no clamped tap ever points;
//   3. out = Up(b) + Up(A) * hr_x (half-pixel centres, edge clamp, the exact
//      factor-4 weights) is written with 128-bit stores.
// No window moments and no staging passes: ~10 instructions per output pixel,
// so the pass streams at the DRAM rate whatever the radius.  TMA = false
// (w % 4 != 0: low-res rows are not 16-byte multiples) stages the cells with
// plain loads.
#include <cuda_runtime.h>

#include "gf_common.cuh"
#include "gf_internal.h"
#include "gf_joint_taps.cuh"
#include "gf_tma.cuh"

namespace gfb {
namespace jf {

constexpr int APW = 40;                         // staged coefficient row: cells k0-4 .. k0+35
constexpr int APF = (RA * APW + 31) / 32 * 32;  // floats per field, a 128-byte multiple
constexpr int ACO = 3;                          // staged column of cell k0 - 1

struct ApplyArgs {
  const float* A;
  const float* B;
  const float* hr_x;
  float* out;
  int h, w, H, W;
  uint32_t* status;
};

// MINB: CTAs per SM the registers are budgeted for
template <bool TMA, int MINB>
__global__ void __launch_bounds__(NT, MINB)
    k_joint_apply(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                  ApplyArgs a) {
  __shared__ __align__(128) float cs[2 * APF];
  __shared__ __align__(8) uint64_t tbar;
  const int64_t p = blockIdx.z;
  const int i0 = blockIdx.y * TLY, k0 = blockIdx.x * TLX;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float* __restrict__ G = a.hr_x + p * (int64_t)a.H * a.W;
  float* __restrict__ O = a.out + p * (int64_t)a.H * a.W;
  const int k = k0 + lane;
  const int X0 = 4 * k;
  const int Yb = 4 * i0 + 8 * warp;
  const bool col_ok = X0 < a.W;
  if (TMA && threadIdx.x == 0) {
    tma::mbar_init(&tbar, 1);
    tma::fence_proxy_async();
  }
  float4 g[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int Y = Yb + t;
    g[t] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (col_ok && Y < a.H) g[t] = __ldg(reinterpret_cast<const float4*>(G + (int64_t)Y * a.W + X0));
  }
  if constexpr (TMA) {
    __syncthreads();
    if (threadIdx.x == 0) {
      tma::mbar_arrive_expect_tx(&tbar, 2u * RA * APW * 4u);
      tma::load_3d(cs, &tmA, k0 - 4, i0 - 1, (int)p, &tbar);
      tma::load_3d(cs + APF, &tmB, k0 - 4, i0 - 1, (int)p, &tbar);
    }
    tma::mbar_wait(&tbar, 0);
  } else {
    const float* Ap = a.A + p * (int64_t)a.h * a.w;
    const float* Bp = a.B + p * (int64_t)a.h * a.w;
    for (int it = threadIdx.x; it < RA * CA; it += NT) {
      const int ar = it / CA, c = it - ar * CA;
      const int gy = i0 - 1 + ar, gx = k0 - 1 + c;
      const bool in = gy >= 0 && gy < a.h && gx >= 0 && gx < a.w;
      const int64_t o = (int64_t)gy * a.w + gx;
      cs[ar * APW + ACO + c] = in ? __ldg(Ap + o) : 0.f;
      cs[APF + ar * APW + ACO + c] = in ? __ldg(Bp + o) : 0.f;
    }
    __syncthreads();
  }
  const float* As = cs + ACO;  // local column 0 = cell k0 - 1
  const float* Bs = cs + APF + ACO;
  bool bad = false;
  const bool cin = k >= 1 && k <= a.w - 2;  // static column taps
  const bool rin = Yb >= 2 && Yb + 7 <= 4 * a.h - 3 && Yb + 7 < a.H;  // static row taps
  if (rin && cin) {
    // hr rows Yb .. Yb+7 tap coefficient rows 2 warp .. 2 warp + 3 (local):
    // rows 0, 1 between q = 0, 1 (f = 5/8, 7/8), rows 2..5 between q = 1, 2
    // (f = 1/8 .. 7/8), rows 6, 7 between q = 2, 3 (f = 1/8, 3/8).  Two
    // horizontally pre-interpolated rows are live at a time.
    float chk = 0.f;
    float la[4], lb[4], ha[4], hb[4];
    const float* ra = As + (2 * warp) * APW;
    const float* rb = Bs + (2 * warp) * APW;
    hrow_interior(ra, lane, la);
    hrow_interior(rb, lane, lb);
    auto rows = [&](int t0, int t1) {
#pragma unroll
      for (int t = t0; t < t1; ++t) {
        constexpr float fph[4] = {0.625f, 0.875f, 0.125f, 0.375f};
        const float f = fph[t & 3];
        const float gv[4] = {g[t].x, g[t].y, g[t].z, g[t].w};
        float o[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float Ah = la[j] + f * (ha[j] - la[j]);
          const float Bh = lb[j] + f * (hb[j] - lb[j]);
          o[j] = Bh + Ah * gv[j];
          chk = fmaf(o[j], 0.f, chk);  // NaN iff an output is not finite
        }
        *reinterpret_cast<float4*>(O + (int64_t)(Yb + t) * a.W + X0) =
            make_float4(o[0], o[1], o[2], o[3]);
      }
    };
    auto next = [&](int q) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        la[j] = ha[j];
        lb[j] = hb[j];
      }
      hrow_interior(ra + q * APW, lane, ha);
      hrow_interior(rb + q * APW, lane, hb);
    };
    hrow_interior(ra + APW, lane, ha);
    hrow_interior(rb + APW, lane, hb);
    rows(0, 2);
    next(2);
    rows(2, 6);
    next(3);
    rows(6, 8);
    bad = chk != 0.f;
  } else if (col_ok) {
    // image borders: clamped taps, horizontal then vertical as above
    const ColTaps ct = col_taps(X0, a.w, k0);
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int Y = Yb + t;
      if (Y >= a.H) continue;
      const Tap ty = tap4(Y, a.h);
      const float* r0 = As + (ty.lo - (i0 - 1)) * APW;
      const float* r1 = As + (ty.hi - (i0 - 1)) * APW;
      float al[4], ah[4], bl[4], bh[4];
      hrow(r0, ct, al);
      hrow(r1, ct, ah);
      hrow(r0 + APF, ct, bl);
      hrow(r1 + APF, ct, bh);
      const float gv[4] = {g[t].x, g[t].y, g[t].z, g[t].w};
      float o[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float Ah = al[j] + ty.f * (ah[j] - al[j]);
        const float Bh = bl[j] + ty.f * (bh[j] - bl[j]);
        o[j] = Bh + Ah * gv[j];
        if (!isfinite(o[j])) bad = true;
      }
      *reinterpret_cast<float4*>(O + (int64_t)Y * a.W + X0) = make_float4(o[0], o[1], o[2], o[3]);
    }
  }
  if (bad) flag(a.status, GF_STATUS_NONFINITE_OUTPUT);
}

}  // namespace jf

thread_local int g_joint_apply_variant = 0;  // CTAs per SM budgeted (0: default)

void joint_apply(const float* A, const float* B, const float* hr_x, float* out, int64_t P,
                 int64_t h, int64_t w, int64_t H, int64_t W, uint32_t* status, cudaStream_t s) {
  dim3 grid((unsigned)((w + jf::TLX - 1) / jf::TLX), (unsigned)((h + jf::TLY - 1) / jf::TLY),
            (unsigned)P);
  jf::ApplyArgs a{A, B, hr_x, out, (int)h, (int)w, (int)H, (int)W, status};
  CUtensorMap tmA, tmB;
  const bool tma_ok = w % 4 == 0 && tma::make_plane_map(&tmA, A, w, h, P, jf::APW, jf::RA) &&
                      tma::make_plane_map(&tmB, B, w, h, P, jf::APW, jf::RA);
  const void* fn;
  switch (g_joint_apply_variant) {
    case 3: fn = tma_ok ? (const void*)jf::k_joint_apply<true, 3> : (const void*)jf::k_joint_apply<false, 3>; break;
    case 5: fn = tma_ok ? (const void*)jf::k_joint_apply<true, 5> : (const void*)jf::k_joint_apply<false, 5>; break;
    case 6: fn = tma_ok ? (const void*)jf::k_joint_apply<true, 6> : (const void*)jf::k_joint_apply<false, 6>; break;
    default: fn = tma_ok ? (const void*)jf::k_joint_apply<true, 4> : (const void*)jf::k_joint_apply<false, 4>; break;
  }
  void* args[] = {&tmA, &tmB, &a};
  cudaLaunchKernel(fn, grid, dim3(jf::NT), args, 0, s);
}

}  // namespace gfb
