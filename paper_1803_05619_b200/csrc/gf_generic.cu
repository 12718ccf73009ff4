// General-shape guided-filter kernels (any ratio, any radius, fp32 or fp64).
//
// These are the GPU kernels for every case the fused fast kernels
// (gf_fused_*.cu) do not specialise: float64 (the reference's own dtype,
// reproduced to its 1e-10 bars), non-integer resize ratios, very large radii,
// tiny or unaligned images.  They mirror the reference's operator structure
// (gf/guided.py:136-297) one elementwise / separable box pass at a time, with
// every accumulation in float64, so they double as the on-device cross-check
// for the fused kernels.  Reductions are deterministic (fixed-order block
// partials, no floating-point atomics).
#include <cuda_runtime.h>

#include "gf_common.cuh"
#include "gf_internal.h"

namespace gfb {

// ===========================================================================
// primitives (gf/filters.py)
// ===========================================================================

// mean_filter (adjoint == 0) or mean_filter_adjoint (adjoint == 1) as a direct
// 2-D window sum in float64.  gf/filters.py:96-116.
template <typename T>
__global__ void k_mean2d(const T* __restrict__ in, T* __restrict__ out, int64_t P, int64_t h,
                         int64_t w, int r, int adjoint) {
  const int64_t n = P * h * w;
  GF_GRID_LOOP(i, n) {
    int64_t x = i % w;
    int64_t t = i / w;
    int64_t y = t % h;
    const T* src = in + (t / h) * h * w;
    int64_t y0 = y - r < 0 ? 0 : y - r, y1 = y + r > h - 1 ? h - 1 : y + r;
    int64_t x0 = x - r < 0 ? 0 : x - r, x1 = x + r > w - 1 ? w - 1 : x + r;
    double s = 0.0;
    if (!adjoint) {
      for (int64_t yy = y0; yy <= y1; ++yy)
        for (int64_t xx = x0; xx <= x1; ++xx) s += (double)src[yy * w + xx];
      s /= (double)((y1 - y0 + 1) * (x1 - x0 + 1));
    } else {
      for (int64_t yy = y0; yy <= y1; ++yy) {
        double ny = (double)win_len(yy, h, r);
        for (int64_t xx = x0; xx <= x1; ++xx)
          s += (double)src[yy * w + xx] / (ny * (double)win_len(xx, w, r));
      }
    }
    out[i] = (T)s;
  }
}

// ---------------------------------------------------------------------------
// Radius-independent clamped box sums (the reference's SAT is radius-free,
// gf/filters.py:32-65; SPEC.md:541 asks r = 32 to cost <= 1.5x r = 1): a
// vertical sliding pass (thread per column and segment of kSeg rows, each
// segment re-anchored by a direct sum so rounding stays bounded) and a
// horizontal pass over per-row prefix sums in shared memory (block per row;
// window = P[x1 + 1] - P[x0]).  Both cost O(1) per pixel (+ (2r+1)/kSeg).
// ---------------------------------------------------------------------------
constexpr int64_t kSeg = 256;

// vertical window sums; `weighted`: element (yy, x) scaled by 1/N(yy, x)
// (mean_filter_adjoint's g / N, gf/filters.py:106-116)
template <typename I, typename O>
__global__ void k_box_v_run(const I* __restrict__ in, O* __restrict__ out, int64_t P, int64_t h,
                            int64_t w, int r, int weighted) {
  const int64_t nseg = (h + kSeg - 1) / kSeg;
  const int64_t n = P * nseg * w;
  GF_GRID_LOOP(i, n) {
    const int64_t x = i % w;
    const int64_t t = i / w;
    const int64_t seg = t % nseg, p = t / nseg;
    const I* col = in + p * h * w + x;
    const double nx = (double)win_len(x, w, r);
    auto val = [&](int64_t yy) {
      const double v = (double)col[yy * w];
      return weighted ? v / ((double)win_len(yy, h, r) * nx) : v;
    };
    const int64_t y0 = seg * kSeg, y1 = y0 + kSeg < h ? y0 + kSeg : h;
    const int64_t a0 = y0 - r < 0 ? 0 : y0 - r, a1 = y0 + r > h - 1 ? h - 1 : y0 + r;
    double s = 0.0;
    for (int64_t yy = a0; yy <= a1; ++yy) s += val(yy);
    O* o = out + p * h * w + x;
    for (int64_t y = y0; y < y1; ++y) {
      o[y * w] = (O)s;
      if (y + r + 1 < h) s += val(y + r + 1);
      if (y - r >= 0) s -= val(y - r);
    }
  }
}

// horizontal window sums of each row via its prefix sums in shared memory
// (in may equal out: a block reads its whole row before writing it);
// `mean`: divided by N(y, x)
template <typename I, typename O>
__global__ void k_box_h_scan(const I* in, O* out, int64_t P, int64_t h, int64_t w, int r,
                             int mean) {
  extern __shared__ double pre[];  // [w + 1], then [blockDim.x] chunk totals
  double* tot = pre + w + 1;
  const int nt = blockDim.x, tid = threadIdx.x;
  const int64_t c = (w + nt - 1) / nt;  // columns per thread
  for (int64_t row = blockIdx.x; row < P * h; row += gridDim.x) {
    const I* src = in + row * w;
    const int64_t j0 = tid * c, j1 = j0 + c < w ? j0 + c : w;
    double acc = 0.0;
    for (int64_t j = j0; j < j1; ++j) {
      const double v = (double)src[j];
      pre[j + 1] = v;
      acc += v;
    }
    tot[tid] = acc;
    __syncthreads();
    if (tid < 32) {  // exclusive offsets of the chunk totals, fixed order
      const int per = (nt + 31) / 32;
      double part = 0.0;
      for (int k = 0; k < per; ++k) {
        const int q = tid * per + k;
        if (q < nt) part += tot[q];
      }
      double incl = part;
      for (int o = 1; o < 32; o <<= 1) {
        const double u = __shfl_up_sync(0xffffffffu, incl, o);
        if (tid >= o) incl += u;
      }
      double run = incl - part;
      for (int k = 0; k < per; ++k) {
        const int q = tid * per + k;
        if (q < nt) {
          const double v = tot[q];
          tot[q] = run;
          run += v;
        }
      }
    }
    __syncthreads();
    double run = tot[tid];
    if (tid == 0) pre[0] = 0.0;
    for (int64_t j = j0; j < j1; ++j) {
      run += pre[j + 1];
      pre[j + 1] = run;
    }
    __syncthreads();
    const int64_t y = row % h;
    const double ny = (double)win_len(y, h, r);
    for (int64_t x = tid; x < w; x += nt) {
      const int64_t x0 = x - r < 0 ? 0 : x - r, x1 = x + r > w - 1 ? w - 1 : x + r;
      double v = pre[x1 + 1] - pre[x0];
      if (mean) v /= (double)(x1 - x0 + 1) * ny;
      out[row * w + x] = (O)v;
    }
    __syncthreads();
  }
}

// bilinear_resize, gf/filters.py:134-156.
template <typename T>
__global__ void k_resize(const T* __restrict__ in, T* __restrict__ out, int64_t P, int64_t h,
                         int64_t w, int64_t oh, int64_t ow) {
  const int64_t n = P * oh * ow;
  GF_GRID_LOOP(i, n) {
    int64_t x = i % ow;
    int64_t t = i / ow;
    int64_t y = t % oh;
    AxisTap ty = axis_map(y, h, oh), tx = axis_map(x, w, ow);
    out[i] = (T)bilerp(in + (t / oh) * h * w, w, ty, tx);
  }
}

// Range of output coordinates d in [0, n_out) whose taps can touch source
// index i (conservative; callers test lo/hi exactly).
__device__ __forceinline__ void adj_range(int64_t i, int64_t n_in, int64_t n_out, int64_t& a,
                                          int64_t& b) {
  double k = (double)n_out / (double)n_in;
  double lo = ((double)i - 1.0 + 0.5) * k - 0.5;
  double hi = ((double)i + 1.0 + 0.5) * k - 0.5;
  a = (int64_t)floor(lo) - 2;
  b = (int64_t)ceil(hi) + 2;
  if (i == 0 || a < 0) a = 0;
  if (i == n_in - 1 || b > n_out - 1) b = n_out - 1;
}

// Weight of output coordinate d on source index i: (1-f)[lo==i] + f[hi==i].
__device__ __forceinline__ double adj_weight(int64_t d, int64_t i, int64_t n_in, int64_t n_out) {
  AxisTap t = axis_map(d, n_in, n_out);
  double wgt = 0.0;
  if (t.lo == i) wgt += 1.0 - t.f;
  if (t.hi == i) wgt += t.f;
  return wgt;
}

// bilinear_resize_adjoint as a gather, gf/filters.py:168-188.  g: (gh, gw)
// -> out: (h, w).  Optional second field g*G (for the joint backward) when
// guide != nullptr.  Accumulation in float64.
template <typename T, typename O>
__global__ void k_resize_adj(const T* __restrict__ g, const T* __restrict__ guide,
                             O* __restrict__ out, O* __restrict__ out2, int64_t P, int64_t gh,
                             int64_t gw, int64_t h, int64_t w) {
  const int64_t n = P * h * w;
  GF_GRID_LOOP(i, n) {
    int64_t k = i % w;
    int64_t t = i / w;
    int64_t iy = t % h;
    int64_t p = t / h;
    int64_t ya, yb, xa, xb;
    adj_range(iy, h, gh, ya, yb);
    adj_range(k, w, gw, xa, xb);
    const T* gp = g + p * gh * gw;
    const T* Gp = guide ? guide + p * gh * gw : nullptr;
    double s = 0.0, s2 = 0.0;
    for (int64_t Y = ya; Y <= yb; ++Y) {
      double wy = adj_weight(Y, iy, h, gh);
      if (wy == 0.0) continue;
      double row = 0.0, row2 = 0.0;
      for (int64_t X = xa; X <= xb; ++X) {
        double wx = adj_weight(X, k, w, gw);
        if (wx == 0.0) continue;
        double v = (double)gp[Y * gw + X];
        row += wx * v;
        if (Gp) row2 += wx * (v * (double)Gp[Y * gw + X]);
      }
      s += wy * row;
      s2 += wy * row2;
    }
    out[i] = (O)s;
    if (out2) out2[i] = (O)s2;
  }
}

template <typename T>
__global__ void k_check_finite(const T* __restrict__ p, int64_t n, uint32_t* status) {
  bool bad = false;
  GF_GRID_LOOP(i, n) {
    if (!finite(p[i])) bad = true;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) flag(status, GF_STATUS_NONFINITE_INPUT);
}

template <typename T>
void generic_check_finite(const T* p, int64_t n, uint32_t* status, cudaStream_t s) {
  k_check_finite<T><<<grid_for(n, 256), 256, 0, s>>>(p, n, status);
}
template void generic_check_finite<float>(const float*, int64_t, uint32_t*, cudaStream_t);
template void generic_check_finite<double>(const double*, int64_t, uint32_t*, cudaStream_t);

// ===========================================================================
// layer building blocks (all float64 intermediates)
// ===========================================================================

struct GuideMap {  // plane p = b*C + c of src -> plane of the guide
  int64_t C, Cg;
  __device__ __forceinline__ int64_t operator()(int64_t p) const {
    return Cg == C ? p : (p / C) * Cg;
  }
};

// x, y, x*x, x*y as float64 fields; finite check of both inputs.
template <typename T>
__global__ void k_products(const T* __restrict__ guide, const T* __restrict__ src,
                           double* __restrict__ f0, double* __restrict__ f1,
                           double* __restrict__ f2, double* __restrict__ f3, int64_t P,
                           int64_t hw, GuideMap gm, uint32_t* status) {
  const int64_t n = P * hw;
  GF_GRID_LOOP(i, n) {
    int64_t p = i / hw, pix = i - p * hw;
    T gx = guide[gm(p) * hw + pix];
    T sy = src[i];
    if (!finite(gx) || !finite(sy)) flag(status, GF_STATUS_NONFINITE_INPUT);
    double x = (double)gx, y = (double)sy;
    f0[i] = x;
    f1[i] = y;
    f2[i] = x * x;
    f3[i] = x * y;
  }
}

// vertical clamped window sum (float64 in/out)
__global__ void k_box_v(const double* __restrict__ in, double* __restrict__ out, int64_t P,
                        int64_t h, int64_t w, int r) {
  const int64_t n = P * h * w;
  GF_GRID_LOOP(i, n) {
    int64_t x = i % w;
    int64_t t = i / w;
    int64_t y = t % h;
    const double* col = in + (t / h) * h * w + x;
    int64_t y0 = y - r < 0 ? 0 : y - r, y1 = y + r > h - 1 ? h - 1 : y + r;
    double s = 0.0;
    for (int64_t yy = y0; yy <= y1; ++yy) s += col[yy * w];
    out[i] = s;
  }
}

// horizontal clamped window sum, optionally divided by N (mean).
__global__ void k_box_h(const double* __restrict__ in, double* __restrict__ out, int64_t P,
                        int64_t h, int64_t w, int r, int mean) {
  const int64_t n = P * h * w;
  GF_GRID_LOOP(i, n) {
    int64_t x = i % w;
    int64_t t = i / w;
    int64_t y = t % h;
    const double* row = in + t * w;
    int64_t x0 = x - r < 0 ? 0 : x - r, x1 = x + r > w - 1 ? w - 1 : x + r;
    double s = 0.0;
    for (int64_t xx = x0; xx <= x1; ++xx) s += row[xx];
    if (mean) s /= (double)((x1 - x0 + 1) * win_len(y, h, r));
    out[i] = s;
  }
}

// gf/guided.py:138-148: var, cov, degenerate check, slope and intercept.
// In: means of x, y, xx, xy.  Out: A -> a, b -> b, var -> v, cov -> c.
__global__ void k_coeffs(const double* __restrict__ mx, const double* __restrict__ my,
                         const double* __restrict__ mxx, const double* __restrict__ mxy,
                         double* __restrict__ a, double* __restrict__ b, double* __restrict__ v,
                         double* __restrict__ c, int64_t n, double eps, uint32_t* status) {
  GF_GRID_LOOP(i, n) {
    double ux = mx[i], uy = my[i];
    double var = mxx[i] - ux * ux;
    double cov = mxy[i] - ux * uy;
    if (eps == 0.0 && !(var > 0.0)) flag(status, GF_STATUS_DEGENERATE);
    double A = cov / (var + eps);
    a[i] = A;
    b[i] = uy - A * ux;
    v[i] = var;
    c[i] = cov;
  }
}

// joint apply: out = Up(b) + Up(A) * G (gf/guided.py:172-180).  With
// dout != nullptr computes d_hr = d_out * Up(A) instead (gf/guided.py:281).
template <typename T>
__global__ void k_apply_up(const double* __restrict__ A, const double* __restrict__ b,
                           const T* __restrict__ G, const T* __restrict__ dout, T* __restrict__ out,
                           int64_t P, int64_t h, int64_t w, int64_t H, int64_t W,
                           uint32_t* status) {
  const int64_t n = P * H * W;
  GF_GRID_LOOP(i, n) {
    int64_t X = i % W;
    int64_t t = i / W;
    int64_t Y = t % H;
    int64_t p = t / H;
    AxisTap ty = axis_map(Y, h, H), tx = axis_map(X, w, W);
    double Ah = bilerp(A + p * h * w, w, ty, tx);
    if (dout) {
      out[i] = (T)((double)dout[i] * Ah);
    } else {
      double bh = bilerp(b + p * h * w, w, ty, tx);
      T g = G[i];
      if (!finite(g)) flag(status, GF_STATUS_NONFINITE_INPUT);
      double o = bh + Ah * (double)g;
      T ot = (T)o;
      if (!finite(ot)) flag(status, GF_STATUS_NONFINITE_OUTPUT);
      out[i] = ot;
    }
  }
}

// highres apply: out = bh + Ah * G.
template <typename T>
__global__ void k_apply_hr(const double* __restrict__ Ah, const double* __restrict__ bh,
                           const T* __restrict__ guide, T* __restrict__ out, int64_t P,
                           int64_t hw, GuideMap gm, uint32_t* status) {
  const int64_t n = P * hw;
  GF_GRID_LOOP(i, n) {
    int64_t p = i / hw, pix = i - p * hw;
    double o = bh[i] + Ah[i] * (double)guide[gm(p) * hw + pix];
    T ot = (T)o;
    if (!finite(ot)) flag(status, GF_STATUS_NONFINITE_OUTPUT);
    out[i] = ot;
  }
}

// highres: d_out / N and d_out * G / N (inputs of the two M^T applications).
template <typename T>
__global__ void k_dout_scaled(const T* __restrict__ dout, const T* __restrict__ guide,
                              double* __restrict__ g0, double* __restrict__ g1, int64_t P,
                              int64_t H, int64_t W, int r, GuideMap gm) {
  const int64_t hw = H * W, n = P * hw;
  GF_GRID_LOOP(i, n) {
    int64_t p = i / hw, pix = i - p * hw;
    int64_t y = pix / W, x = pix - y * W;
    double inv = 1.0 / (double)(win_len(y, H, r) * win_len(x, W, r));
    double d = (double)dout[i];
    g0[i] = d * inv;
    g1[i] = (d * (double)guide[gm(p) * hw + pix]) * inv;
  }
}

// gf/guided.py:236-253: slope/intercept grads -> moment grads, each / N.
__global__ void k_mom_bwd1(const double* __restrict__ mx, const double* __restrict__ my,
                           const double* __restrict__ A, const double* __restrict__ var,
                           const double* __restrict__ cov, const double* __restrict__ db,
                           const double* __restrict__ dAraw, double* __restrict__ k0,
                           double* __restrict__ k1, double* __restrict__ k2,
                           double* __restrict__ k3, int64_t P, int64_t h, int64_t w, int r,
                           double eps) {
  const int64_t n = P * h * w;
  GF_GRID_LOOP(i, n) {
    int64_t x = i % w;
    int64_t y = (i / w) % h;
    double ux = mx[i], uy = my[i];
    double dbi = db[i];
    double dA = dAraw[i] + (-dbi * ux);
    double denom = var[i] + eps;
    double d_cov = dA / denom;
    double d_var = -dA * cov[i] / (denom * denom);
    double d_my = dbi + (-d_cov * ux);
    double d_mx = (-dbi * A[i]) + (-d_cov * uy) + (-2.0 * d_var * ux);
    double inv = 1.0 / (double)(win_len(y, h, r) * win_len(x, w, r));
    k0[i] = d_cov * inv;
    k1[i] = d_var * inv;
    k2[i] = d_mx * inv;
    k3[i] = d_my * inv;
  }
}

// gf/guided.py:255-263: d_src, d_guide from the box-summed moment grads.
// Joint: writes T outputs.  Highres: d_guide (float64, per channel) also gets
// the direct term d_out * Ah (gf/guided.py:289-295).
template <typename T>
__global__ void k_mom_bwd2(const T* __restrict__ guide, const T* __restrict__ src,
                           const double* __restrict__ bcov, const double* __restrict__ bvar,
                           const double* __restrict__ bmx, const double* __restrict__ bmy,
                           const T* __restrict__ dout, const double* __restrict__ Ah,
                           T* __restrict__ d_src, T* __restrict__ d_guide_t,
                           double* __restrict__ d_guide_d, int64_t P, int64_t hw, GuideMap gm) {
  const int64_t n = P * hw;
  GF_GRID_LOOP(i, n) {
    int64_t p = i / hw, pix = i - p * hw;
    double x = (double)guide[gm(p) * hw + pix];
    double y = (double)src[i];
    double bc = bcov[i];
    d_src[i] = (T)(bc * x + bmy[i]);
    double dg = bc * y + 2.0 * bvar[i] * x + bmx[i];
    if (d_guide_d) {
      d_guide_d[i] = (double)dout[i] * Ah[i] + dg;
    } else {
      d_guide_t[i] = (T)dg;
    }
  }
}

// per-channel float64 guide grads -> (B, Cg, H, W) in T (sum over C when Cg == 1)
template <typename T>
__global__ void k_guide_reduce(const double* __restrict__ D, T* __restrict__ dg, int64_t B,
                               int64_t C, int64_t Cg, int64_t hw) {
  const int64_t n = B * Cg * hw;
  GF_GRID_LOOP(i, n) {
    if (Cg == C) {
      dg[i] = (T)D[i];
    } else {
      int64_t b = i / hw, pix = i - b * hw;
      double s = 0.0;
      for (int64_t c = 0; c < C; ++c) s += D[(b * C + c) * hw + pix];
      dg[i] = (T)s;
    }
  }
}

// ===========================================================================
// host orchestration
// ===========================================================================

namespace {
constexpr int kThreads = 256;

template <typename K, typename... Args>
void launch(K kernel, int64_t n, cudaStream_t s, Args... args) {
  kernel<<<grid_for(n, kThreads), kThreads, 0, s>>>(args...);
}

constexpr int64_t kMaxScanW = 26000;  // row prefix sums in shared memory
// radii below this keep the direct window sums: as cheap, and exact where
// the reference is (r = 0: a window of one value, var = x^2 - x^2 = 0)
constexpr int kRunMinR = 4;

// clamped box sum of float64 fields, in -> out through tmp (mean: / N):
// radius-independent passes when a row fits shared memory, else direct sums
template <typename I, typename O>
void box2d(const I* in, O* out, double* tmp, int64_t P, int64_t h, int64_t w, int r, int mean,
           int weighted, cudaStream_t s) {
  if (w <= kMaxScanW && r >= kRunMinR) {
    const int64_t nseg = (h + kSeg - 1) / kSeg;
    launch(k_box_v_run<I, double>, P * nseg * w, s, in, tmp, P, h, w, r, weighted);
    const size_t smem = (size_t)(w + 1 + kThreads) * sizeof(double);
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(k_box_h_scan<double, O>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
    const int64_t rows = P * h;
    const int grid = (int)(rows < 148 * 16 ? rows : 148 * 16);
    k_box_h_scan<double, O><<<grid, kThreads, smem, s>>>(tmp, out, P, h, w, r, mean);
    return;
  }
  const int64_t n = P * h * w;
  launch(k_box_v, n, s, (const double*)in, tmp, P, h, w, r);  // (weighted: never, see callers)
  launch(k_box_h, n, s, (const double*)tmp, out, P, h, w, r, mean);
}

// Box-filter a float64 field in place through tmp (mean: divide by N).
void box_inplace(double* f, double* tmp, int64_t P, int64_t h, int64_t w, int r, int mean,
                 cudaStream_t s) {
  box2d<double, double>(f, f, tmp, P, h, w, r, mean, 0, s);
}

// Moments + coefficients into ws fields; returns nothing.  Field map:
//  F0 = mean x, F1 = mean y, F2 = A, F3 = b, F4 = var, F5 = cov.  Uses F6..F9.
template <typename T>
void moments(const T* guide, const T* src, double* const* F, int64_t P, int64_t h, int64_t w,
             GuideMap gm, int r, double eps, uint32_t* status, cudaStream_t s) {
  int64_t n = P * h * w;
  launch(k_products<T>, n, s, guide, src, F[6], F[7], F[8], F[9], P, h * w, gm, status);
  for (int f = 0; f < 4; ++f)
    box2d<double, double>(F[6 + f], F[6 + f], F[0 + f], P, h, w, r, 1, 0, s);
  // means now in F6..F9; coefficients
  launch(k_coeffs, n, s, (const double*)F[6], (const double*)F[7], (const double*)F[8],
         (const double*)F[9], F[2], F[3], F[4], F[5], n, eps, status);
  cudaMemcpyAsync(F[0], F[6], n * sizeof(double), cudaMemcpyDeviceToDevice, s);
  cudaMemcpyAsync(F[1], F[7], n * sizeof(double), cudaMemcpyDeviceToDevice, s);
}

void fields(void* ws, int64_t n, double** F, int count) {
  double* base = (double*)ws;
  for (int i = 0; i < count; ++i) F[i] = base + (int64_t)i * n;
}
}  // namespace

constexpr int kGenericFields = 17;

size_t generic_workspace_bytes(int64_t n_moment_plane_total, int64_t extra_doubles) {
  return (size_t)(n_moment_plane_total * kGenericFields + extra_doubles) * sizeof(double);
}

// mean_filter / mean_filter_adjoint with no workspace (the C ABI's
// primitives): the vertical sums go through `out` itself (the horizontal
// scan reads each row into shared memory before overwriting it), so the cost
// is radius-independent; float outputs hold the vertical sums in float.
// Rows wider than kMaxScanW take the direct 2-D sum.
template <typename T>
void generic_mean_filter(const T* in, T* out, int64_t P, int64_t h, int64_t w, int r,
                         int adjoint, cudaStream_t s) {
  if (w > kMaxScanW || r < kRunMinR || (const void*)in == (const void*)out) {
    launch(k_mean2d<T>, P * h * w, s, in, out, P, h, w, r, adjoint);
    return;
  }
  const int64_t nseg = (h + kSeg - 1) / kSeg;
  launch(k_box_v_run<T, T>, P * nseg * w, s, in, out, P, h, w, r, adjoint);
  const size_t smem = (size_t)(w + 1 + kThreads) * sizeof(double);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_box_h_scan<T, T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  const int64_t rows = P * h;
  const int grid = (int)(rows < 148 * 16 ? rows : 148 * 16);
  k_box_h_scan<T, T><<<grid, kThreads, smem, s>>>(out, out, P, h, w, r, adjoint ? 0 : 1);
}

template <typename T>
void generic_resize(const T* in, T* out, int64_t P, int64_t h, int64_t w, int64_t oh,
                    int64_t ow, cudaStream_t s) {
  launch(k_resize<T>, P * oh * ow, s, in, out, P, h, w, oh, ow);
}

template <typename T>
void generic_resize_adj(const T* g, T* out, int64_t P, int64_t gh, int64_t gw, int64_t h,
                        int64_t w, cudaStream_t s) {
  launch(k_resize_adj<T, T>, P * h * w, s, g, (const T*)nullptr, out, (T*)nullptr, P, gh, gw,
         h, w);
}

template <typename T>
void generic_joint_fwd(const T* lr_x, const T* lr_y, const T* hr_x, T* out, int64_t B, int64_t C,
                       int64_t h, int64_t w, int64_t H, int64_t W, int r, double eps, void* ws,
                       uint32_t* status, cudaStream_t s) {
  int64_t P = B * C, n = P * h * w;
  double* F[kGenericFields];
  fields(ws, n, F, kGenericFields);
  GuideMap gm{C, C};
  moments<T>(lr_x, lr_y, F, P, h, w, gm, r, eps, status, s);
  launch(k_apply_up<T>, P * H * W, s, (const double*)F[2], (const double*)F[3], hr_x,
         (const T*)nullptr, out, P, h, w, H, W, status);
}

template <typename T>
void generic_joint_bwd(const T* lr_x, const T* lr_y, const T* hr_x, const T* d_out, T* d_lr_x,
                       T* d_lr_y, T* d_hr_x, int64_t B, int64_t C, int64_t h, int64_t w,
                       int64_t H, int64_t W, int r, double eps, void* ws, uint32_t* status,
                       cudaStream_t s) {
  int64_t P = B * C, n = P * h * w;
  double* F[kGenericFields];
  fields(ws, n, F, kGenericFields);
  GuideMap gm{C, C};
  moments<T>(lr_x, lr_y, F, P, h, w, gm, r, eps, status, s);
  // db -> F10, dAraw -> F11 (Up^T of d_out and d_out * G), gf/guided.py:277-280
  launch(k_resize_adj<T, double>, n, s, d_out, hr_x, F[10], F[11], P, H, W, h, w);
  // d_hr = d_out * Up(A)
  launch(k_apply_up<T>, P * H * W, s, (const double*)F[2], (const double*)nullptr,
         (const T*)nullptr, d_out, d_hr_x, P, h, w, H, W, status);
  launch(k_mom_bwd1, n, s, (const double*)F[0], (const double*)F[1], (const double*)F[2],
         (const double*)F[4], (const double*)F[5], (const double*)F[10], (const double*)F[11],
         F[12], F[13], F[14], F[15], P, h, w, r, eps);
  for (int f = 12; f < 16; ++f) box_inplace(F[f], F[16], P, h, w, r, 0, s);
  launch(k_mom_bwd2<T>, n, s, lr_x, lr_y, (const double*)F[12], (const double*)F[13],
         (const double*)F[14], (const double*)F[15], (const T*)nullptr, (const double*)nullptr,
         d_lr_y, d_lr_x, (double*)nullptr, P, h * w, gm);
}

template <typename T>
void generic_highres_fwd(const T* guide, const T* src, T* out, int64_t B, int64_t Cg, int64_t C,
                         int64_t H, int64_t W, int r, double eps, void* ws, uint32_t* status,
                         cudaStream_t s) {
  int64_t P = B * C, n = P * H * W;
  double* F[kGenericFields];
  fields(ws, n, F, kGenericFields);
  GuideMap gm{C, Cg};
  moments<T>(guide, src, F, P, H, W, gm, r, eps, status, s);
  box_inplace(F[2], F[16], P, H, W, r, 1, s);  // Ah = M(A)
  box_inplace(F[3], F[16], P, H, W, r, 1, s);  // bh = M(b)
  launch(k_apply_hr<T>, n, s, (const double*)F[2], (const double*)F[3], guide, out, P, H * W,
         gm, status);
}

template <typename T>
void generic_highres_bwd(const T* guide, const T* src, const T* d_out, T* d_guide, T* d_src,
                         int64_t B, int64_t Cg, int64_t C, int64_t H, int64_t W, int r,
                         double eps, void* ws, uint32_t* status, cudaStream_t s) {
  int64_t P = B * C, n = P * H * W;
  double* F[kGenericFields];
  fields(ws, n, F, kGenericFields);
  GuideMap gm{C, Cg};
  moments<T>(guide, src, F, P, H, W, gm, r, eps, status, s);
  // Ah = M(A) -> F9 (F6..F9 are free after moments)
  cudaMemcpyAsync(F[9], F[2], n * sizeof(double), cudaMemcpyDeviceToDevice, s);
  box_inplace(F[9], F[16], P, H, W, r, 1, s);
  // db = M^T(d_out) -> F10, dAraw = M^T(d_out * G) -> F11
  launch(k_dout_scaled<T>, n, s, d_out, guide, F[10], F[11], P, H, W, r, gm);
  box_inplace(F[10], F[16], P, H, W, r, 0, s);
  box_inplace(F[11], F[16], P, H, W, r, 0, s);
  launch(k_mom_bwd1, n, s, (const double*)F[0], (const double*)F[1], (const double*)F[2],
         (const double*)F[4], (const double*)F[5], (const double*)F[10], (const double*)F[11],
         F[12], F[13], F[14], F[15], P, H, W, r, eps);
  for (int f = 12; f < 16; ++f) box_inplace(F[f], F[16], P, H, W, r, 0, s);
  // per-channel float64 d_guide -> F6, then reduce over broadcast copies
  launch(k_mom_bwd2<T>, n, s, guide, src, (const double*)F[12], (const double*)F[13],
         (const double*)F[14], (const double*)F[15], d_out, (const double*)F[9], d_src,
         (T*)nullptr, F[6], P, H * W, gm);
  launch(k_guide_reduce<T>, B * Cg * H * W, s, (const double*)F[6], d_guide, B, C, Cg, H * W);
}

// explicit instantiations
#define GF_INST(T)                                                                          \
  template void generic_mean_filter<T>(const T*, T*, int64_t, int64_t, int64_t, int, int,   \
                                       cudaStream_t);                                       \
  template void generic_resize<T>(const T*, T*, int64_t, int64_t, int64_t, int64_t,        \
                                  int64_t, cudaStream_t);                                   \
  template void generic_resize_adj<T>(const T*, T*, int64_t, int64_t, int64_t, int64_t,    \
                                      int64_t, cudaStream_t);                               \
  template void generic_joint_fwd<T>(const T*, const T*, const T*, T*, int64_t, int64_t,    \
                                     int64_t, int64_t, int64_t, int64_t, int, double,       \
                                     void*, uint32_t*, cudaStream_t);                       \
  template void generic_joint_bwd<T>(const T*, const T*, const T*, const T*, T*, T*, T*,    \
                                     int64_t, int64_t, int64_t, int64_t, int64_t, int64_t,  \
                                     int, double, void*, uint32_t*, cudaStream_t);          \
  template void generic_highres_fwd<T>(const T*, const T*, T*, int64_t, int64_t, int64_t,   \
                                       int64_t, int64_t, int, double, void*, uint32_t*,     \
                                       cudaStream_t);                                       \
  template void generic_highres_bwd<T>(const T*, const T*, const T*, T*, T*, int64_t,       \
                                       int64_t, int64_t, int64_t, int64_t, int, double,     \
                                       void*, uint32_t*, cudaStream_t);
GF_INST(float)
GF_INST(double)

}  // namespace gfb
