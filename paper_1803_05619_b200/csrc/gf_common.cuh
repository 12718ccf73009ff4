// Shared device helpers for the guided-filter kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/gf_b200.h"

namespace gfb {

// ---------------------------------------------------------------------------
// status word (device) -- bits of GF_STATUS_*
// ---------------------------------------------------------------------------
__device__ __forceinline__ void flag(uint32_t* status, uint32_t bit) {
  if (status) atomicOr(status, bit);
}

template <typename T>
__device__ __forceinline__ bool finite(T v) {
  return isfinite(v);
}

// One MUFU.RCP (<= 1 ulp): the fp32 kernels' reciprocal of window counts and
// of var + eps, where the IEEE-rounded __frcp_rn costs a dozen instructions.
__device__ __forceinline__ float fast_rcp(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ---------------------------------------------------------------------------
// gf/filters.py:82-93 window_counts: per-axis clamped window length.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t win_len(int64_t i, int64_t n, int r) {
  int64_t a = i - r < 0 ? 0 : i - r;
  int64_t b = i + r > n - 1 ? n - 1 : i + r;
  return b - a + 1;
}

// ---------------------------------------------------------------------------
// gf/filters.py:119-131 _axis_map, in float64 with the reference's rounding
// (explicit _rn intrinsics: no FMA contraction of (d+.5)*(in/out)-.5).
// ---------------------------------------------------------------------------
struct AxisTap {
  int64_t lo, hi;
  double f;
};

__device__ __forceinline__ AxisTap axis_map(int64_t d, int64_t n_in, int64_t n_out) {
  double scale = __ddiv_rn((double)n_in, (double)n_out);
  double s = __dadd_rn(__dmul_rn(__dadd_rn((double)d, 0.5), scale), -0.5);
  double top = (double)(n_in - 1);
  s = s < 0.0 ? 0.0 : (s > top ? top : s);
  int64_t lo = (int64_t)floor(s);
  if (lo > n_in - 1) lo = n_in - 1;
  AxisTap t;
  t.lo = lo;
  t.f = __dadd_rn(s, -(double)lo);
  t.hi = lo + 1 > n_in - 1 ? n_in - 1 : lo + 1;
  return t;
}

// gf/_kernels.py:83-95 _bilinear: rows first, then columns, lerp a + f*(b - a).
template <typename A>
__device__ __forceinline__ double bilerp(const A* __restrict__ t, int64_t w, const AxisTap& ty,
                                         const AxisTap& tx) {
  double a = (double)t[ty.lo * w + tx.lo];
  a = a + ty.f * ((double)t[ty.hi * w + tx.lo] - a);
  double b = (double)t[ty.lo * w + tx.hi];
  b = b + ty.f * ((double)t[ty.hi * w + tx.hi] - b);
  return a + tx.f * (b - a);
}

// grid-stride helper
#define GF_GRID_LOOP(i, n)                                                            \
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n);           \
       i += (int64_t)gridDim.x * blockDim.x)

inline int grid_for(int64_t n, int threads = 256) {
  int64_t b = (n + threads - 1) / threads;
  if (b > 148 * 32) b = 148 * 32;
  if (b < 1) b = 1;
  return (int)b;
}

}  // namespace gfb
