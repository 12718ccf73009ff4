// Joint guided filter backward, low-res tail (gf/guided.py:236-264 after
// :278-280), fp32 NCHW on sm_100a: register-segment walk for r <= 4.
//
// Inputs per low-res plane: lr_x, lr_y and the two adjoint fields gathered by
// k_joint_bwd_hr (db = Up^T(d_out), dA = Up^T(d_out hr_x)).  Per moment cell
//   mean_x, mean_y, var, cov over the clamped (2r+1)^2 window  (level 1)
//   dA' = dA - db mean_y ... -> d_cov, d_var, d_mx, d_my     (:242-252)
//   k = (d_cov, d_var, d_mx, d_my) / N
// and per output cell the box adjoint M^T k = box_sum(k) (level 2), then
//   d_lr_y = s_cov x + s_my,  d_lr_x = s_cov y + 2 s_var x + s_mx  (:255-263).
//
// One warp per work unit, no CTA barriers: a warp owns a strip of 128
// columns (4 per lane, 16-byte loads) and walks a piece of rows top to
// bottom.  Level-1 vertical window sums of (x, y, x^2, x y) live in
// registers (entering row loaded, leaving row re-loaded from L2); horizontal
// windows come from the lane's inclusive prefix plus the neighbouring lanes'
// prefixes by shuffle (r <= 4: lanes t-1 and t+1 only, 2r+1 shuffles per
// field); the four k fields of the last 2r+1 moment rows sit in a shared
// memory ring (level-2 vertical sums in registers, the leaving row from the
// ring).  Output columns of a strip: [PAD, PAD + OW) with PAD = up4(2r).
// x and y are shifted by per-piece constants (var/cov are shift invariant);
// the means entering the gradient formulas are the true ones.
#include <cuda_runtime.h>

#include <type_traits>

#include "gf_common.cuh"
#include "gf_internal.h"

namespace gfb {
namespace jls {

constexpr int WC = 128;  // columns per warp
constexpr int kMaxRadius = 4;
// Pieces (the rows a warp walks with one set of running sums and one shift
// constant) are cut at multiples of kPiece rows of the FULL image: a row band
// (multi-GPU config 4b) passes its first row's global index, so its pieces,
// shifts and summation order over the owned rows are the full image's and the
// band's d_lr_x, d_lr_y are bitwise equal to the 1-GPU result.
constexpr int kPiece = 64;

__host__ __device__ constexpr int up4(int n) { return (n + 3) / 4 * 4; }

template <int RAD>
struct Geo {
  static constexpr int PAD = up4(2 * RAD);
  static constexpr int OW = (WC - PAD - 2 * RAD) / 4 * 4;
  static constexpr int ringN = 2 * RAD + 1;
  static constexpr size_t smem_bytes = (size_t)ringN * 4 * 32 * sizeof(float4);  // per warp
};

constexpr int WPB = 4;  // warps per CTA (independent)

struct Args {
  const float* lr_x;
  const float* lr_y;
  const float* db;
  const float* dA;
  float* d_lr_x;
  float* d_lr_y;
  int64_t h, w;
  int strips;
  int npieces, off;     // pieces per (plane, strip) column; row0 % kPiece
  int64_t U, upw;       // pieces of all columns; pieces per warp
  int64_t nwarps;
  float eps;
};

__device__ __forceinline__ int wlen(int i, int n, int r) {
  const int a = i - r < 0 ? 0 : i - r;
  const int b = i + r > n - 1 ? n - 1 : i + r;
  return b - a + 1;
}

// Horizontal window sums over +-R (R <= 4) of 4 values per lane (columns
// 4t .. 4t+3 of the warp):
//   W_j = p[min(3, j+R)] - p[j-R-1] + [j < R] (T_{t-1} - p_{t-1}[3+j-R])
//         + [j+R > 3] p_{t+1}[j+R-4]      (p inclusive prefix, p[-1] = 0)
// Lanes 0 and 31 produce garbage where the window leaves the warp (halo).
template <int R>
__device__ __forceinline__ float4 hwin(float4 v) {
  const float p[4] = {v.x, v.x + v.y, v.x + v.y + v.z, v.x + v.y + v.z + v.w};
  if constexpr (R == 0) {
    return v;
  } else {
    float pl[4] = {0.f, 0.f, 0.f, 0.f}, pn[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int k = (3 - R < 0 ? 0 : 3 - R); k < 4; ++k) pl[k] = __shfl_up_sync(0xffffffffu, p[k], 1);
#pragma unroll
    for (int k = 0; k < R; ++k) pn[k] = __shfl_down_sync(0xffffffffu, p[k], 1);
    float w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float s = p[j + R < 3 ? j + R : 3];
      if (j - R - 1 >= 0) s -= p[j - R - 1];
      if (j < R) s += pl[3] - (3 + j - R >= 0 ? pl[3 + j - R] : 0.f);
      if (j + R > 3) s += pn[j + R - 4];
      w[j] = s;
    }
    return make_float4(w[0], w[1], w[2], w[3]);
  }
}

__device__ __forceinline__ float4 ld4(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}
__device__ __forceinline__ float4 mask4(float4 v, bool ok) {
  return ok ? v : make_float4(0.f, 0.f, 0.f, 0.f);
}
__device__ __forceinline__ float4 sub4(float4 a, float b) {
  return make_float4(a.x - b, a.y - b, a.z - b, a.w - b);
}
__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ float4 subv4(float4 a, float4 b) {
  return make_float4(a.x - b.x, a.y - b.y, a.z - b.z, a.w - b.w);
}
__device__ __forceinline__ float4 fma4(float4 a, float4 b, float4 c) {
  return make_float4(fmaf(a.x, b.x, c.x), fmaf(a.y, b.y, c.y), fmaf(a.z, b.z, c.z),
                     fmaf(a.w, b.w, c.w));
}
__device__ __forceinline__ float el(const float4& v, int j) {
  return j == 0 ? v.x : (j == 1 ? v.y : (j == 2 ? v.z : v.w));
}

struct Bufs {
  float4 ex, ey, lx, ly;  // entering / leaving rows
  float4 db, da;          // adjoint fields of the step's moment row (HBM: a step ahead)
};

struct Piece {
  const float* X;
  const float* Y;
  const float* DB;
  const float* DA;
  float* OX;
  float* OY;
  int h, w, y0, y1, xl, lane;
  float sx, sy, eps;
};

template <int RAD, bool EDGE>
__device__ __forceinline__ void run_piece(const Piece& P, float4* __restrict__ ring) {
  using GG = Geo<RAD>;
  constexpr int r = RAD, ringN = GG::ringN;
  const int h = P.h, w = P.w, y0 = P.y0, y1 = P.y1, xl = P.xl, lane = P.lane;
  const float* __restrict__ X = P.X;
  const float* __restrict__ Y = P.Y;
  const float sx = P.sx, sy = P.sy, eps = P.eps;
  const bool ok = !EDGE || (xl >= 0 && xl < w);
  const int xc = ok ? xl : 0;
  const float sxc = ok ? sx : 0.f, syc = ok ? sy : 0.f;
  float inx[4];  // 1/nx per column (0 outside the image)
  bool cin[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int x = xl + j;
    cin[j] = !EDGE || (x >= 0 && x < w);
    inx[j] = cin[j] ? (EDGE ? fast_rcp((float)wlen(x, w, r)) : 1.f / (2 * r + 1)) : 0.f;
  }
  const bool oout = 4 * lane >= GG::PAD && 4 * lane < GG::PAD + GG::OW && xl < w;

  const int ya_lo = max(y0 - r, 0);
  const int ya_end = y1 + r;  // moment rows ya in [ya_lo, ya_end)
  const int first_in = max(ya_lo - r, 0);

  float4 VX = make_float4(0.f, 0.f, 0.f, 0.f), VY = VX, VXX = VX, VXY = VX;
#pragma unroll 2
  for (int y = first_in; y < min(ya_lo + r, h); ++y) {
    const int ro = y * w + xc;
    const float4 x4 = sub4(mask4(ld4(X + ro), ok), sxc);
    const float4 y4 = sub4(mask4(ld4(Y + ro), ok), syc);
    VX = add4(VX, x4);
    VY = add4(VY, y4);
    VXX = fma4(x4, x4, VXX);
    VXY = fma4(x4, y4, VXY);
  }
  float4 K0 = make_float4(0.f, 0.f, 0.f, 0.f), K1 = K0, K2 = K0, K3 = K0;  // level-2 sums

  auto fetch = [&](auto steady, Bufs& B, int ya) {
    constexpr bool STEADY = decltype(steady)::value;
    int e = ya + r, l = ya - r - 1;
    if (!STEADY) {
      e = min(e, h - 1);
      l = max(l, 0);
    }
    B.ex = ld4(X + (e * w + xc));
    B.ey = ld4(Y + (e * w + xc));
    B.lx = ld4(X + (l * w + xc));
    B.ly = ld4(Y + (l * w + xc));
    const int ym = STEADY ? ya : min(ya, h - 1);
    B.db = ld4(P.DB + (ym * w + xc));
    B.da = ld4(P.DA + (ym * w + xc));
  };

  int slot = 0;
  auto step = [&](auto steady, int ya, Bufs& cur) {
    constexpr bool STEADY = decltype(steady)::value;
    // adjoint fields of moment row ya (fetched a step ahead with the entering
    // rows) and inputs of output row ya - r (L2)
    const float4 dbv = cur.db, dav = cur.da;
    const int yo = STEADY ? ya - r : min(max(ya - r, 0), h - 1);
    const float4 ox = ld4(X + (yo * w + xc));
    const float4 oy = ld4(Y + (yo * w + xc));
    float4 k0 = make_float4(0.f, 0.f, 0.f, 0.f), k1 = k0, k2 = k0, k3 = k0;
    if (STEADY || ya < h) {
      const bool ein = STEADY || ya + r < h, lin = STEADY || ya - r - 1 >= first_in;
      float4 ex = sub4(mask4(cur.ex, ok), sxc), ey = sub4(mask4(cur.ey, ok), syc);
      float4 lx = sub4(mask4(cur.lx, ok), sxc), ly = sub4(mask4(cur.ly, ok), syc);
      if (!STEADY) {
        if (!ein) ex = ey = make_float4(0.f, 0.f, 0.f, 0.f);
        if (!lin) lx = ly = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      VX = add4(VX, subv4(ex, lx));
      VY = add4(VY, subv4(ey, ly));
      VXX = fma4(ex, ex, VXX);
      VXX = fma4(make_float4(-lx.x, -lx.y, -lx.z, -lx.w), lx, VXX);
      VXY = fma4(ex, ey, VXY);
      VXY = fma4(make_float4(-lx.x, -lx.y, -lx.z, -lx.w), ly, VXY);
      if (STEADY || ya + 1 < ya_end) fetch(steady, cur, ya + 1);
      const float4 hX = hwin<r>(VX), hY = hwin<r>(VY), hXX = hwin<r>(VXX), hXY = hwin<r>(VXY);
      const float iny = fast_rcp((float)wlen(ya, h, r));
      float kk[4][4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float inv = inx[j] * iny;  // 1/N (0 outside the image)
        const float mx = el(hX, j) * inv, my = el(hY, j) * inv;  // shifted means
        const float var = el(hXX, j) * inv - mx * mx;
        const float cov = el(hXY, j) * inv - mx * my;
        const float rden = fast_rcp(var + eps);
        const float A = cov * rden;
        const float ux = mx + sx, uy = my + sy;  // true means
        const float dbj = el(dbv, j);
        const float dAj = el(dav, j) + (-dbj * ux);                  // gf/guided.py:278-280
        const float d_cov = dAj * rden;                              // :242
        const float d_var = -dAj * cov * (rden * rden);              // :243
        const float d_my = dbj + (-d_cov * ux);                      // :245-247
        const float d_mx = (-dbj * A) + (-d_cov * uy) + (-2.f * d_var * ux);  // :248-252
        const bool live = cin[j] && inv != 0.f;
        kk[0][j] = live ? d_cov * inv : 0.f;
        kk[1][j] = live ? d_var * inv : 0.f;
        kk[2][j] = live ? d_mx * inv : 0.f;
        kk[3][j] = live ? d_my * inv : 0.f;
      }
      k0 = make_float4(kk[0][0], kk[0][1], kk[0][2], kk[0][3]);
      k1 = make_float4(kk[1][0], kk[1][1], kk[1][2], kk[1][3]);
      k2 = make_float4(kk[2][0], kk[2][1], kk[2][2], kk[2][3]);
      k3 = make_float4(kk[3][0], kk[3][1], kk[3][2], kk[3][3]);
    } else if (ya + 1 < ya_end) {
      fetch(steady, cur, ya + 1);
    }
    // ---- level-2 vertical: ring slot of row ya holds row ya - ringN
    float4* rs = ring + slot * 128 + lane;
    if (STEADY || ya - ringN >= ya_lo) {
      K0 = subv4(K0, rs[0]);
      K1 = subv4(K1, rs[32]);
      K2 = subv4(K2, rs[64]);
      K3 = subv4(K3, rs[96]);
    }
    K0 = add4(K0, k0);
    K1 = add4(K1, k1);
    K2 = add4(K2, k2);
    K3 = add4(K3, k3);
    rs[0] = k0;
    rs[32] = k1;
    rs[64] = k2;
    rs[96] = k3;
    if (++slot == ringN) slot = 0;
    // ---- level-2 horizontal + output row y = ya - r
    const int y = ya - r;
    if (STEADY || y >= y0) {
      const float4 s0 = hwin<r>(K0), s1 = hwin<r>(K1), s2 = hwin<r>(K2), s3 = hwin<r>(K3);
      if (oout) {
        float4 gx, gy;
        gx.x = fmaf(s0.x, oy.x, fmaf(2.f * s1.x, ox.x, s2.x));
        gx.y = fmaf(s0.y, oy.y, fmaf(2.f * s1.y, ox.y, s2.y));
        gx.z = fmaf(s0.z, oy.z, fmaf(2.f * s1.z, ox.z, s2.z));
        gx.w = fmaf(s0.w, oy.w, fmaf(2.f * s1.w, ox.w, s2.w));
        gy.x = fmaf(s0.x, ox.x, s3.x);
        gy.y = fmaf(s0.y, ox.y, s3.y);
        gy.z = fmaf(s0.z, ox.z, s3.z);
        gy.w = fmaf(s0.w, ox.w, s3.w);
        *reinterpret_cast<float4*>(P.OX + (y * w + xl)) = gx;
        *reinterpret_cast<float4*>(P.OY + (y * w + xl)) = gy;
      }
    }
  };

  const std::integral_constant<bool, false> gen;
  const std::integral_constant<bool, true> sty;
  int sa = max(max(first_in + r + 1, ya_lo + ringN), y0 + r);
  const int sb = min(h - r - 1, ya_end - 1);
  Bufs b0;
  fetch(gen, b0, ya_lo);
  int ya = ya_lo;
  for (; ya < min(sa, ya_end); ++ya) step(gen, ya, b0);
  if (ya == sa)
    for (; ya < sb; ++ya) step(sty, ya, b0);
  for (; ya < ya_end; ++ya) step(gen, ya, b0);
  __syncwarp();
}

template <int RAD>
__global__ void __launch_bounds__(WPB * 32) k_joint_bwd_lr_seg(Args a) {
  using GG = Geo<RAD>;
  extern __shared__ __align__(16) float4 smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float4* ring = smem + warp * (GG::ringN * 128);
  const int64_t gw = (int64_t)blockIdx.x * WPB + warp;
  if (gw >= a.nwarps) return;
  const int h = (int)a.h, w = (int)a.w;
  const int64_t u_lo = gw * a.upw;
  const int64_t u_hi = min(u_lo + a.upw, a.U);
  const int64_t plane = (int64_t)h * w;
  for (int64_t u = u_lo; u < u_hi; ++u) {
    const int64_t col = u / a.npieces;
    const int k = (int)(u - col * a.npieces);
    Piece P;
    P.y0 = max(k * kPiece - a.off, 0);
    P.y1 = min((k + 1) * kPiece - a.off, h);
    const int64_t pl = col / a.strips;
    const int strip = (int)(col - pl * a.strips);
    const int x0 = strip * GG::OW;
    const int xs = x0 - GG::PAD;
    const int64_t off = pl * plane;
    P.X = a.lr_x + off;
    P.Y = a.lr_y + off;
    P.DB = a.db + off;
    P.DA = a.dA + off;
    P.OX = a.d_lr_x + off;
    P.OY = a.d_lr_y + off;
    P.h = h;
    P.w = w;
    P.xl = xs + 4 * lane;
    P.lane = lane;
    P.sx = __ldg(P.X + (int64_t)P.y0 * w + x0);
    P.sy = __ldg(P.Y + (int64_t)P.y0 * w + x0);
    P.eps = a.eps;
    if (xs < RAD || xs + WC + RAD > w)
      run_piece<RAD, true>(P, ring);
    else
      run_piece<RAD, false>(P, ring);
  }
}

struct Launch {
  const void* fn;
  size_t smem;
  int ow;
};

template <int RAD>
Launch launch_info() {
  return {(const void*)k_joint_bwd_lr_seg<RAD>, WPB * Geo<RAD>::smem_bytes, Geo<RAD>::OW};
}

Launch pick(int r) {
  switch (r) {
    case 0: return launch_info<0>();
    case 1: return launch_info<1>();
    case 2: return launch_info<2>();
    case 3: return launch_info<3>();
    case 4: return launch_info<4>();
    default: return {nullptr, 0, 0};
  }
}

}  // namespace jls

bool seg_joint_bwd_lr_ok(int64_t h, int64_t w, int r) {
  return r >= 0 && r <= jls::kMaxRadius && w % 4 == 0 && w >= 4 && h >= 1 &&
         h * w < ((int64_t)1 << 31);
}

void seg_joint_bwd_lr(const float* lr_x, const float* lr_y, const float* db, const float* dA,
                      float* d_lr_x, float* d_lr_y, int64_t P, int64_t h, int64_t w, int r,
                      float eps, int64_t row0, cudaStream_t s) {
  const jls::Launch L = jls::pick(r);
  const LaunchCfg lc = launch_cfg(L.fn, jls::WPB * 32, L.smem);
  const int64_t slots = (int64_t)lc.sms * lc.per_sm * jls::WPB;
  const int64_t strips = (w + L.ow - 1) / L.ow;
  const int off = (int)(row0 % jls::kPiece);
  const int npieces = (int)((off + h + jls::kPiece - 1) / jls::kPiece);
  // pieces of all (plane, strip) columns, consecutive pieces of a column on
  // one warp (its warm-up rows are the previous piece's last rows, in L2);
  // as few pieces per warp as fill one wave of warps
  const int64_t U = P * strips * npieces;
  const int64_t upw = (U + slots - 1) / slots;
  const int64_t nw = (U + upw - 1) / upw;
  jls::Args a{lr_x, lr_y, db, dA, d_lr_x, d_lr_y, h, w, (int)strips, npieces, off, U, upw, nw,
              eps};
  void* args[] = {&a};
  cudaLaunchKernel(L.fn, dim3((unsigned)((nw + jls::WPB - 1) / jls::WPB)), dim3(jls::WPB * 32),
                   args, L.smem, s);
}

}  // namespace gfb
