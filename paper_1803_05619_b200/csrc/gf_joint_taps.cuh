// Tile geometry and factor-4 bilinear taps shared by the joint kernels
// (gf_fused_joint.cu, gf_joint_apply.cu).
#pragma once

#include <cuda_runtime.h>

namespace gfb {
namespace jf {

constexpr int TLY = 16, TLX = 32;      // low-res block of the hr kernels
constexpr int THY = 4 * TLY, THX = 4 * TLX;
constexpr int NT = 256;
constexpr int RA = TLY + 2, CA = TLX + 2;  // coefficient cells incl. bilinear halo

// factor-4 half-pixel tap of hr coordinate d into an axis of n low-res cells:
// s = (d + 0.5)/4 - 0.5 = (2d - 3)/8 exactly, clamped (gf/filters.py:126-131)
struct Tap {
  int lo, hi;
  float f;
};
__device__ __forceinline__ Tap tap4(int d, int n) {
  float s = (float)(2 * d - 3) * 0.125f;
  const float top = (float)(n - 1);
  s = s < 0.f ? 0.f : (s > top ? top : s);
  Tap t;
  t.lo = (int)floorf(s);
  if (t.lo > n - 1) t.lo = n - 1;
  t.f = s - (float)t.lo;
  t.hi = t.lo + 1 > n - 1 ? n - 1 : t.lo + 1;
  return t;
}

// Horizontal pre-interpolation of one coefficient row for the 4 hr phases of
// lr cell column (k0 + lane): taps into local columns.
struct ColTaps {
  int lo[4], hi[4];
  float f[4];
};

__device__ __forceinline__ ColTaps col_taps(int X0, int w, int k0) {
  ColTaps t;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    Tap tp = tap4(X0 + j, w);
    t.lo[j] = tp.lo - (k0 - 1);
    t.hi[j] = tp.hi - (k0 - 1);
    t.f[j] = tp.f;
  }
  return t;
}

// Interior lr columns (1 <= k <= w-2): the factor-4 half-pixel taps are
// static -- phases 0, 1 between cells k-1 and k (f = 5/8, 7/8), phases 2, 3
// between k and k+1 (f = 1/8, 3/8); local column of cell k-1 is the lane.
// Same arithmetic as hrow with the exact taps (bit-identical).
__device__ __forceinline__ void hrow_interior(const float* __restrict__ row, int lane,
                                              float (&o)[4]) {
  const float a0 = row[lane], a1 = row[lane + 1], a2 = row[lane + 2];
  o[0] = a0 + 0.625f * (a1 - a0);
  o[1] = a0 + 0.875f * (a1 - a0);
  o[2] = a1 + 0.125f * (a2 - a1);
  o[3] = a1 + 0.375f * (a2 - a1);
}

__device__ __forceinline__ void hrow(const float* __restrict__ row, const ColTaps& ct,
                                     float (&o)[4]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float a = row[ct.lo[j]];
    o[j] = a + ct.f[j] * (row[ct.hi[j]] - a);
  }
}

}  // namespace jf
}  // namespace gfb
