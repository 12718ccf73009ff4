// Fast guided filter forward, first kernel of the two-kernel split: the
// low-res coefficients A = cov/(var+eps), b = mean_y - A mean_x of EVERY
// low-res cell (gf/guided.py:136-149 _window_moments over the clamped
// (2r+1)^2 window, :170-173), fp32 NCHW on sm_100a, r <= 8, w % 4 == 0.
//
// Register-segment walk, one warp per work unit, no CTA barriers and no shared
// memory: a warp owns a strip of 32*SW columns (SW = 4 or 8 consecutive
// columns per lane, 16-byte loads) and walks 16-row pieces top to bottom.
// Vertical window sums of (x, y, x^2, x y) live in registers (entering row
// loaded from HBM, leaving row re-loaded from L2); horizontal windows come from
// the lane's inclusive prefix plus the neighbouring lanes' prefixes by shuffle
// (r <= SW: lanes t-1 and t+1 only, 2r+1 shuffles per field); A and b are
// written with 128-bit stores.  Output columns of a strip: [PAD, PAD + ow)
// with PAD = up4(r).
// r = 2..4 (4 columns per lane), the default: the rows travel through a per-warp
// shared-memory RING of 16 rows filled by cp.async (16 bytes per lane and
// field, zero-filled outside the image) 14 - 2r steps ahead of their use; the
// entering AND the leaving row of a step are read from the ring, so the loads
// hold no registers, the leaving rows cost no L2 re-read and the DRAM latency
// of the entering rows is hidden.  Same arithmetic, same order: bitwise the
// register walk's result.
// x and y are shifted by per-piece constants (var/cov are shift invariant)
// and every running sum restarts per piece, so rounding error is bounded by
// the piece, not the image.  Pieces start at rows 16 k - 1 (the first at row
// 0): a row band whose crop starts on a 16-row multiple at least r + 1 rows
// above its first owned row (sharding.row_bands) then has, from the row just
// above its owned rows on -- the first coefficient row its bilinear taps
// touch, which starts a piece with its whole warm-up inside the crop -- the
// full image's pieces, shifts and summation order, so the coefficients its
// owned outputs read are bitwise the 1-GPU image's.
#include <cuda_runtime.h>

#include "gf_common.cuh"
#include "gf_internal.h"

namespace gfb {
namespace jcs {

constexpr int kPiece = 16;
constexpr int kMaxRadius = 8;
constexpr int WPB = 4;  // warps per CTA (independent)

__host__ __device__ constexpr int up4(int n) { return (n + 3) / 4 * 4; }

template <int SW, int RAD>
struct Geo {
  static constexpr int NC = SW / 4;
  static constexpr int WC = 32 * SW;
  static constexpr int PAD = up4(RAD);
  static constexpr int OWMAX = (WC - PAD - RAD) / 4 * 4;
};

struct Args {
  const float* X;
  const float* Y;
  float* A;
  float* B;
  int h, w;
  int strips, ow;  // strips per plane, output columns per strip (a multiple of 4)
  int npieces;     // pieces per (plane, strip) column
  int64_t U, upw;  // pieces of all columns; pieces per warp
  int64_t nwarps;
  float eps;
  uint32_t* status;
};

__device__ __forceinline__ int wlen(int i, int n, int r) {
  const int a = i - r < 0 ? 0 : i - r;
  const int b = i + r > n - 1 ? n - 1 : i + r;
  return b - a + 1;
}

// Horizontal window sums over +-R (R <= SW) of SW values per lane (columns
// SW t .. SW t + SW-1 of the warp):
//   W_j = p[min(SW-1, j+R)] - p[j-R-1]
//         + [j < R] (T_{t-1} - p_{t-1}[SW-1+j-R]) + [j+R > SW-1] p_{t+1}[j+R-SW]
// (p inclusive prefix, p[-1] = 0, T = p[SW-1]).  Lanes 0 and 31 produce
// garbage where the window leaves the warp (halo columns).
template <int SW, int R>
__device__ __forceinline__ void hwin(const float (&v)[SW], float (&w)[SW]) {
  if constexpr (R == 0) {
#pragma unroll
    for (int j = 0; j < SW; ++j) w[j] = v[j];
  } else {
    static_assert(R <= SW, "window reaches lanes t-1 and t+1 only");
    float p[SW];
    p[0] = v[0];
#pragma unroll
    for (int j = 1; j < SW; ++j) p[j] = p[j - 1] + v[j];
    float pl[SW], pn[SW];
#pragma unroll
    for (int k = 0; k < SW; ++k) pl[k] = pn[k] = 0.f;
#pragma unroll
    for (int k = (SW - 1 - R < 0 ? 0 : SW - 1 - R); k < SW; ++k)
      pl[k] = __shfl_up_sync(0xffffffffu, p[k], 1);
#pragma unroll
    for (int k = 0; k < R; ++k) pn[k] = __shfl_down_sync(0xffffffffu, p[k], 1);
#pragma unroll
    for (int j = 0; j < SW; ++j) {
      float s = p[j + R < SW - 1 ? j + R : SW - 1];
      if (j - R - 1 >= 0) s -= p[j - R - 1];
      if (j < R) s += pl[SW - 1] - (SW - 1 + j - R >= 0 ? pl[SW - 1 + j - R] : 0.f);
      if (j + R > SW - 1) s += pn[j + R - SW];
      w[j] = s;
    }
  }
}

__device__ __forceinline__ float4 ld4(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}

// ---- cp.async ring (r <= 4, 4 columns per lane) ----
constexpr int kRingRows = 16;  // 16 KB per warp: 3 CTAs of 4 warps per SM
template <int RAD>
constexpr int ring_rows() { return kRingRows; }
template <int RAD>
constexpr int ring_ahead() { return kRingRows - 2 * RAD - 2; }  // rows in flight ahead
template <int RAD>
constexpr size_t ring_bytes() { return (size_t)ring_rows<RAD>() * 2 * 32 * sizeof(float4); }  // per warp

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const int n = valid ? 16 : 0;  // 0: the 16 bytes are zero-filled
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(n)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int NC>
struct Bufs {
  float4 ex[NC], ey[NC], lx[NC], ly[NC];  // entering / leaving rows
};

struct Piece {
  const float* X;
  const float* Y;
  float* A;
  float* B;
  int h, w, y0, y1, xl, x0, x1, lane;  // output columns [x0, x1)
  float sx, sy, eps;
};

// EDGE: some lane chunks lie outside the image or some windows are clipped by
// the image's left/right border
template <int SW, int RAD, bool EDGE, bool RING = false>
__device__ __forceinline__ void run_piece(const Piece& P, bool& degen, float4* ring = nullptr) {
  using GG = Geo<SW, RAD>;
  constexpr int r = RAD, NC = GG::NC;
  static_assert(!RING || (SW == 4 && RAD >= 1), "the ring walk: 4 columns per lane");
  constexpr int NR = ring_rows<RAD>(), PF = ring_ahead<RAD>();
  const int h = P.h, w = P.w, y0 = P.y0, y1 = P.y1, xl = P.xl;
  const float* __restrict__ X = P.X;
  const float* __restrict__ Y = P.Y;
  const float sx = P.sx, sy = P.sy, eps = P.eps;
  bool ok[NC];
  int xc[NC];
  float sxc[NC], syc[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    ok[c] = !EDGE || (xl + 4 * c >= 0 && xl + 4 * c < w);
    xc[c] = ok[c] ? xl + 4 * c : 0;
    sxc[c] = ok[c] ? sx : 0.f;  // an out-of-image chunk is masked to zero, shifted by zero
    syc[c] = ok[c] ? sy : 0.f;
  }
  float inx[SW];  // 1/nx per column (0 outside the image)
#pragma unroll
  for (int j = 0; j < SW; ++j) {
    const int x = xl + j;
    const bool in = !EDGE || (x >= 0 && x < w);
    inx[j] = in ? (EDGE ? fast_rcp((float)wlen(x, w, r)) : 1.f / (2 * r + 1)) : 0.f;
  }
  bool oout[NC];  // chunk holds output columns of this strip
#pragma unroll
  for (int c = 0; c < NC; ++c) oout[c] = xl + 4 * c >= P.x0 && xl + 4 * c < P.x1;

  auto shifted = [&](const float4 (&q)[NC], const float (&s)[NC], float (&o)[SW]) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const float4 v = (!EDGE || ok[c]) ? q[c] : make_float4(0.f, 0.f, 0.f, 0.f);
      o[4 * c] = v.x - s[c];
      o[4 * c + 1] = v.y - s[c];
      o[4 * c + 2] = v.z - s[c];
      o[4 * c + 3] = v.w - s[c];
    }
  };

  // rows of step y: entering y + r, leaving y - r - 1 (clamped; masked in the step)
  auto fetch = [&](Bufs<NC>& B, int y) {
    const int e = min(y + r, h - 1), l = max(y - r - 1, 0);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      B.ex[c] = ld4(X + (e * w + xc[c]));
      B.ey[c] = ld4(Y + (e * w + xc[c]));
      B.lx[c] = ld4(X + (l * w + xc[c]));
      B.ly[c] = ld4(Y + (l * w + xc[c]));
    }
  };
  // the first step's rows (the first two at 4 columns per lane) are requested
  // before the warm-up
  constexpr int DEPTH = SW == 4 ? 2 : 1;  // steps between a load and its use
  Bufs<NC> b0, b1;
  if constexpr (!RING) {
    fetch(b0, y0);
    if constexpr (DEPTH == 2) fetch(b1, min(y0 + 1, y1 - 1));
  }
  // RING: the piece's rows form a stream, index i <-> image row ylo + i, i in
  // [0, n): row i lives in slot i % NR; every stream row is one commit group
  // (rows outside the image: an empty group), so "all but the newest PF groups
  // are complete" always means "the entering row of this step has landed"
  const int ylo = y0 - r;
  const int nstream = (y1 - y0) + 2 * r;
  int s_issue = 0, i_issue = 0;  // slot / stream index of the next row to request
  auto issue_row = [&]() {
    const int y = ylo + i_issue;
    if (i_issue < nstream && y >= 0 && y < h) {
      float4* dst = ring + s_issue * 64 + P.lane;
      const bool v = !EDGE || ok[0];
      cp_async16(dst, X + (y * w + xc[0]), v);
      cp_async16(dst + 32, Y + (y * w + xc[0]), v);
    }
    cp_async_commit();
    ++i_issue;
    if (++s_issue == NR) s_issue = 0;
  };
  if constexpr (RING) {
    cp_async_wait<0>();  // the previous piece's tail
    __syncwarp();
#pragma unroll 1
    for (int i = 0; i < 2 * r + PF; ++i) issue_row();
  }

  // vertical warm-up: rows max(y0 - r, 0) .. min(y0 + r, h) - 1, WB rows'
  // loads in flight at a time
  float VX[SW], VY[SW], VXX[SW], VXY[SW];
#pragma unroll
  for (int j = 0; j < SW; ++j) VX[j] = VY[j] = VXX[j] = VXY[j] = 0.f;
  if constexpr (RING) {
    cp_async_wait<PF>();  // stream rows 0 .. 2r-1 (the warm-up rows) have landed
#pragma unroll 1
    for (int i = 0; i < 2 * r; ++i) {
      const int y = ylo + i;
      if (y >= 0 && y < h) {  // y < y0 + r always
        float4 qx[NC], qy[NC];
        qx[0] = ring[i * 64 + P.lane];
        qy[0] = ring[i * 64 + 32 + P.lane];
        float xv[SW], yv[SW];
        shifted(qx, sxc, xv);
        shifted(qy, syc, yv);
#pragma unroll
        for (int j = 0; j < SW; ++j) {
          VX[j] += xv[j];
          VY[j] += yv[j];
          VXX[j] = fmaf(xv[j], xv[j], VXX[j]);
          VXY[j] = fmaf(xv[j], yv[j], VXY[j]);
        }
      }
    }
  } else if constexpr (r > 0) {
    constexpr int WB = (4 / NC) < 2 * r ? (4 / NC) : 2 * r;
    const int wlo = max(y0 - r, 0), whi = min(y0 + r, h);
#pragma unroll 1
    for (int yb = wlo; yb < whi; yb += WB) {
      float4 qx[WB][NC], qy[WB][NC];
#pragma unroll
      for (int k = 0; k < WB; ++k) {
        const int y = min(yb + k, whi - 1);
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          qx[k][c] = ld4(X + (y * w + xc[c]));
          qy[k][c] = ld4(Y + (y * w + xc[c]));
        }
      }
#pragma unroll
      for (int k = 0; k < WB; ++k) {
        if (yb + k < whi) {
          float xv[SW], yv[SW];
          shifted(qx[k], sxc, xv);
          shifted(qy[k], syc, yv);
#pragma unroll
          for (int j = 0; j < SW; ++j) {
            VX[j] += xv[j];
            VY[j] += yv[j];
            VXX[j] = fmaf(xv[j], xv[j], VXX[j]);
            VXY[j] = fmaf(xv[j], yv[j], VXY[j]);
          }
        }
      }
    }
  }

  // one step: output row y from buffer `cur`, which is then refilled with the
  // rows of step y + DEPTH (RING: from the ring slots of the entering row,
  // stream index (y - y0) + 2r, and the leaving row, index (y - y0) - 1)
  int s_enter = (2 * r) % NR, s_leave = 0;
  auto step = [&](int y, Bufs<NC>& cur) {
    // the leaving row is in the sums only when it entered them (>= y0 - r)
    const bool ein = y + r < h, lin = y - r - 1 >= max(y0 - r, 0);
    {
      float ex[SW], ey[SW], lx[SW], ly[SW];
      if constexpr (RING) {
        issue_row();           // stream row (y - y0) + 2r + PF
        cp_async_wait<PF>();   // ... so row (y - y0) + 2r, the entering one, is here
        const float4* se = ring + s_enter * 64 + P.lane;
        const float4* sl = ring + s_leave * 64 + P.lane;
        cur.ex[0] = se[0];
        cur.ey[0] = se[32];
        cur.lx[0] = sl[0];
        cur.ly[0] = sl[32];
        if (++s_enter == NR) s_enter = 0;
        if (y > y0 && ++s_leave == NR) s_leave = 0;
      }
      shifted(cur.ex, sxc, ex);
      shifted(cur.ey, syc, ey);
      shifted(cur.lx, sxc, lx);
      shifted(cur.ly, syc, ly);
      if constexpr (!RING) {
        if (y + DEPTH < y1) fetch(cur, y + DEPTH);
      }
#pragma unroll
      for (int j = 0; j < SW; ++j) {
        const float e0 = ein ? ex[j] : 0.f, e1 = ein ? ey[j] : 0.f;
        const float l0 = lin ? lx[j] : 0.f, l1 = lin ? ly[j] : 0.f;
        VX[j] += e0 - l0;
        VY[j] += e1 - l1;
        VXX[j] = fmaf(-l0, l0, fmaf(e0, e0, VXX[j]));
        VXY[j] = fmaf(-l0, l1, fmaf(e0, e1, VXY[j]));
      }
    }
    float hX[SW], hY[SW], hXX[SW], hXY[SW];
    hwin<SW, r>(VX, hX);
    hwin<SW, r>(VY, hY);
    hwin<SW, r>(VXX, hXX);
    hwin<SW, r>(VXY, hXY);
    const float iny = fast_rcp((float)wlen(y, h, r));
    float Av[SW], Bv[SW];
    float vr[SW];  // variances (the eps = 0 check below)
#pragma unroll
    for (int j = 0; j < SW; ++j) {
      const float inv = inx[j] * iny;  // 1/N
      const float mx = hX[j] * inv, my = hY[j] * inv;  // shifted means
      const float var = hXX[j] * inv - mx * mx;
      const float cov = hXY[j] * inv - mx * my;
      Av[j] = cov * fast_rcp(var + eps);
      Bv[j] = (my + sy) - Av[j] * (mx + sx);
      vr[j] = var;
    }
    if (eps == 0.f) {  // gf/guided.py:142-146 (warp-uniform: off the common path)
#pragma unroll
      for (int j = 0; j < SW; ++j)
        if (oout[j >> 2] && !(vr[j] > 0.f)) degen = true;
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      if (oout[c]) {
        const int o = y * w + xl + 4 * c;
        *reinterpret_cast<float4*>(P.A + o) =
            make_float4(Av[4 * c], Av[4 * c + 1], Av[4 * c + 2], Av[4 * c + 3]);
        *reinterpret_cast<float4*>(P.B + o) =
            make_float4(Bv[4 * c], Bv[4 * c + 1], Bv[4 * c + 2], Bv[4 * c + 3]);
      }
    }
  };
  if constexpr (RING) {
#pragma unroll 1
    for (int y = y0; y < y1; ++y) step(y, b0);
  } else if constexpr (DEPTH == 2) {
#pragma unroll 1
    for (int y = y0; y < y1; y += 2) {
      step(y, b0);
      if (y + 1 < y1) step(y + 1, b1);
    }
  } else {
#pragma unroll 1
    for (int y = y0; y < y1; ++y) step(y, b0);
  }
}

template <int SW, int RAD>
__global__ void __launch_bounds__(WPB * 32, SW == 4 ? 5 : 3) k_joint_coeffs_seg(Args a) {
  using GG = Geo<SW, RAD>;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * WPB + warp;
  if (gw >= a.nwarps) return;
  const int h = a.h, w = a.w;
  const int64_t u_lo = gw * a.upw;
  const int64_t u_hi = min(u_lo + a.upw, a.U);
  const int64_t plane = (int64_t)h * w;
  bool degen = false;
  for (int64_t u = u_lo; u < u_hi; ++u) {
    const int64_t col = u / a.npieces;
    const int k = (int)(u - col * a.npieces);
    const int64_t pl = col / a.strips;
    const int strip = (int)(col - pl * a.strips);
    Piece P;
    P.y0 = max(k * kPiece - 1, 0);
    P.y1 = min(k * kPiece + kPiece - 1, h);
    P.x0 = strip * a.ow;
    P.x1 = min(P.x0 + a.ow, w);
    if (P.x0 >= w) continue;  // rounding the strip width up can leave the last strip empty
    const int xs = P.x0 - GG::PAD;
    P.X = a.X + pl * plane;
    P.Y = a.Y + pl * plane;
    P.A = a.A + pl * plane;
    P.B = a.B + pl * plane;
    P.h = h;
    P.w = w;
    P.xl = xs + SW * lane;
    P.lane = lane;
    P.sx = __ldg(P.X + (int64_t)P.y0 * w + P.x0);
    P.sy = __ldg(P.Y + (int64_t)P.y0 * w + P.x0);
    P.eps = a.eps;
    if (xs < RAD || xs + GG::WC + RAD > w)
      run_piece<SW, RAD, true>(P, degen);
    else
      run_piece<SW, RAD, false>(P, degen);
  }
  if (degen) flag(a.status, GF_STATUS_DEGENERATE);
}

// the ring walk: 4 columns per lane, WPB independent warps, ring_bytes per warp
template <int RAD>
__global__ void __launch_bounds__(WPB * 32) k_joint_coeffs_ring(Args a) {
  using GG = Geo<4, RAD>;
  extern __shared__ __align__(16) float4 ring_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float4* ring = ring_smem + warp * (ring_rows<RAD>() * 64);
  const int64_t gw = (int64_t)blockIdx.x * WPB + warp;
  if (gw >= a.nwarps) return;
  const int h = a.h, w = a.w;
  const int64_t u_lo = gw * a.upw;
  const int64_t u_hi = min(u_lo + a.upw, a.U);
  const int64_t plane = (int64_t)h * w;
  bool degen = false;
  for (int64_t u = u_lo; u < u_hi; ++u) {
    const int64_t col = u / a.npieces;
    const int k = (int)(u - col * a.npieces);
    const int64_t pl = col / a.strips;
    const int strip = (int)(col - pl * a.strips);
    Piece P;
    P.y0 = max(k * kPiece - 1, 0);
    P.y1 = min(k * kPiece + kPiece - 1, h);
    P.x0 = strip * a.ow;
    P.x1 = min(P.x0 + a.ow, w);
    if (P.x0 >= w) continue;
    const int xs = P.x0 - GG::PAD;
    P.X = a.X + pl * plane;
    P.Y = a.Y + pl * plane;
    P.A = a.A + pl * plane;
    P.B = a.B + pl * plane;
    P.h = h;
    P.w = w;
    P.xl = xs + 4 * lane;
    P.lane = lane;
    P.sx = __ldg(P.X + (int64_t)P.y0 * w + P.x0);
    P.sy = __ldg(P.Y + (int64_t)P.y0 * w + P.x0);
    P.eps = a.eps;
    if (xs < RAD || xs + GG::WC + RAD > w)
      run_piece<4, RAD, true, true>(P, degen, ring);
    else
      run_piece<4, RAD, false, true>(P, degen, ring);
  }
  cp_async_wait<0>();
  if (degen) flag(a.status, GF_STATUS_DEGENERATE);
}

struct Launch {
  const void* fn;
  int owmax;
  size_t smem = 0;  // dynamic shared memory per CTA
};

template <int SW, int RAD>
Launch launch_info() {
  return {(const void*)k_joint_coeffs_seg<SW, RAD>, Geo<SW, RAD>::OWMAX};
}

template <int RAD>
Launch ring_info() {
  return {(const void*)k_joint_coeffs_ring<RAD>, Geo<4, RAD>::OWMAX, WPB * ring_bytes<RAD>()};
}

// r = 2..4: the cp.async ring walk (4 columns per lane; narrower strips
// quantise the width better); r = 0 the register walk at 4 per lane; above, 8
// per lane.  Variant hook sw: 8 forces 8 per lane, 4 the register walk.
Launch pick(int r, int sw) {
  if (sw == 0) {
    switch (r) {
      case 1: return ring_info<1>();
      case 2: return ring_info<2>();
      case 3: return ring_info<3>();
      case 4: return ring_info<4>();
      default: break;
    }
  }
  if (sw == 8 || r > 4) {
    switch (r) {
      case 0: return launch_info<8, 0>();
      case 1: return launch_info<8, 1>();
      case 2: return launch_info<8, 2>();
      case 3: return launch_info<8, 3>();
      case 4: return launch_info<8, 4>();
      case 5: return launch_info<8, 5>();
      case 6: return launch_info<8, 6>();
      case 7: return launch_info<8, 7>();
      case 8: return launch_info<8, 8>();
      default: return {nullptr, 0};
    }
  }
  switch (r) {
    case 0: return launch_info<4, 0>();
    case 1: return launch_info<4, 1>();
    case 2: return launch_info<4, 2>();
    case 3: return launch_info<4, 3>();
    case 4: return launch_info<4, 4>();
    default: return {nullptr, 0};
  }
}

}  // namespace jcs

thread_local int g_joint_coeffs_sw = 0;  // variant hook: 8 forces 8 columns per lane

bool seg_joint_coeffs_ok(int64_t h, int64_t w, int r) {
  return r >= 0 && r <= jcs::kMaxRadius && w % 4 == 0 && w >= 4 && h >= 1 &&
         h * w < ((int64_t)1 << 31);
}

void seg_joint_coeffs(const float* lr_x, const float* lr_y, float* A, float* B, int64_t P,
                      int64_t h, int64_t w, int r, float eps, uint32_t* status, cudaStream_t s) {
  const jcs::Launch L = jcs::pick(r, g_joint_coeffs_sw);
  const LaunchCfg lc = launch_cfg(L.fn, jcs::WPB * 32, L.smem);
  const int64_t slots = (int64_t)lc.sms * lc.per_sm * jcs::WPB;
  // equal strips: as few as cover the width, each a multiple of 4 columns
  const int64_t strips = (w + L.owmax - 1) / L.owmax;
  const int64_t ow = ((w + strips - 1) / strips + 3) / 4 * 4;
  const int npieces = (int)((h + jcs::kPiece) / jcs::kPiece);  // pieces [16 k - 1, 16 k + 15)
  // pieces of all (plane, strip) columns, consecutive pieces of a column on
  // one warp (its warm-up rows are the previous piece's last rows, in L2)
  const int64_t U = P * strips * npieces;
  const int64_t upw = (U + slots - 1) / slots;
  const int64_t nw = (U + upw - 1) / upw;
  jcs::Args a{lr_x, lr_y, A, B, (int)h, (int)w, (int)strips, (int)ow, npieces, U, upw, nw, eps,
              status};
  void* args[] = {&a};
  cudaLaunchKernel(L.fn, dim3((unsigned)((nw + jcs::WPB - 1) / jcs::WPB)), dim3(jcs::WPB * 32),
                   args, L.smem, s);
}

}  // namespace gfb
