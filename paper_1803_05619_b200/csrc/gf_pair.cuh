// fp32 pair arithmetic for sm_100a (FADD2 / FMUL2 / FFMA2): two lanes of
// independent values in one 64-bit register pair, one instruction each.
#pragma once

#include <cuda_runtime.h>

namespace gfb {
namespace pr {

typedef unsigned long long u64;

__device__ __forceinline__ u64 pk(float a, float b) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ u64 bc(float a) { return pk(a, a); }
__device__ __forceinline__ float lo(u64 v) {
  return __uint_as_float((unsigned)(v & 0xffffffffull));
}
__device__ __forceinline__ float hi(u64 v) { return __uint_as_float((unsigned)(v >> 32)); }
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
  u64 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
  u64 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
  u64 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
// leaky-ReLU slope pair of (h.lo, h.hi): 1 where >= 0, else `neg`
__device__ __forceinline__ u64 slope2(u64 h, float neg) {
  return pk(lo(h) >= 0.f ? 1.f : neg, hi(h) >= 0.f ? 1.f : neg);
}

}  // namespace pr
}  // namespace gfb
