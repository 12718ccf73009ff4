// Standalone guidance-net layers (gf/guidance.py:52-173): ConvLayer (k x k,
// dilation, zero "same" padding, optional bias) and AdaptiveNorm
// (gain * x + norm_gain * standardize(x), per image and channel statistics,
// variance floor 1e-5), forward and backward, float and double, NCHW.
//
// These back the reference's layer objects (GuidanceNet.conv1 / .norm /
// .conv2 and the exported ConvLayer / AdaptiveNorm), not the config-2 hot
// path: GuidanceNet itself runs the fused gn_* kernels.  Every reduction is
// deterministic: one block per output scalar (or image plane), float64
// partials in a fixed per-thread order, then a fixed shared-memory tree.
#include <cuda_runtime.h>

#include "../../include/gf_b200.h"
#include "gf_common.cuh"
#include "gf_internal.h"

namespace gfb {
namespace ly {

constexpr int NT = 256;
constexpr double kVarFloor = 1e-5;  // gf/guidance.py:26 NORM_VAR_FLOOR

template <int NV>
__device__ void block_sum(double (&v)[NV], double (&out)[NV]) {
  __shared__ double sh[NV][NT];
#pragma unroll
  for (int k = 0; k < NV; ++k) sh[k][threadIdx.x] = v[k];
  __syncthreads();
  for (int s = NT / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) {
#pragma unroll
      for (int k = 0; k < NV; ++k) sh[k][threadIdx.x] += sh[k][threadIdx.x + s];
    }
    __syncthreads();
  }
#pragma unroll
  for (int k = 0; k < NV; ++k) out[k] = sh[k][0];
  __syncthreads();
}

struct ConvGeo {
  int64_t B, Cin, Cout, H, W;
  int k, d, pad;
};

// gf/guidance.py:87-104: y[co] = sum_{ky,kx} sum_ci x_pad[ci, y+ky d, x+kx d] w[co,ci,ky,kx] + b
template <typename T>
__global__ void k_conv_fwd(const T* __restrict__ x, const T* __restrict__ w,
                           const T* __restrict__ bias, T* __restrict__ y, ConvGeo g) {
  const int64_t HW = g.H * g.W, n = g.B * g.Cout * HW;
  GF_GRID_LOOP(i, n) {
    const int64_t px = i % HW, bc = i / HW;
    const int64_t co = bc % g.Cout, b = bc / g.Cout;
    const int64_t yy = px / g.W, xx = px - yy * g.W;
    double acc = 0.0;
    for (int ky = 0; ky < g.k; ++ky) {
      const int64_t sy = yy + ky * g.d - g.pad;
      if (sy < 0 || sy >= g.H) continue;
      for (int kx = 0; kx < g.k; ++kx) {
        const int64_t sx = xx + kx * g.d - g.pad;
        if (sx < 0 || sx >= g.W) continue;
        for (int64_t ci = 0; ci < g.Cin; ++ci)
          acc += (double)x[((b * g.Cin + ci) * g.H + sy) * g.W + sx] *
                 (double)w[((co * g.Cin + ci) * g.k + ky) * g.k + kx];
      }
    }
    if (bias) acc += (double)bias[co];
    y[i] = (T)acc;
  }
}

// gf/guidance.py:106-124, d_padded: dx[ci, p] = sum_{co,ky,kx} dy[co, p - (ky d - pad)] w[co,ci,ky,kx]
template <typename T>
__global__ void k_conv_dx(const T* __restrict__ dy, const T* __restrict__ w, T* __restrict__ dx,
                          ConvGeo g) {
  const int64_t HW = g.H * g.W, n = g.B * g.Cin * HW;
  GF_GRID_LOOP(i, n) {
    const int64_t px = i % HW, bc = i / HW;
    const int64_t ci = bc % g.Cin, b = bc / g.Cin;
    const int64_t yy = px / g.W, xx = px - yy * g.W;
    double acc = 0.0;
    for (int ky = 0; ky < g.k; ++ky) {
      const int64_t oy = yy - ky * g.d + g.pad;
      if (oy < 0 || oy >= g.H) continue;
      for (int kx = 0; kx < g.k; ++kx) {
        const int64_t ox = xx - kx * g.d + g.pad;
        if (ox < 0 || ox >= g.W) continue;
        for (int64_t co = 0; co < g.Cout; ++co)
          acc += (double)dy[((b * g.Cout + co) * g.H + oy) * g.W + ox] *
                 (double)w[((co * g.Cin + ci) * g.k + ky) * g.k + kx];
      }
    }
    dx[i] = (T)acc;
  }
}

// one block per weight scalar (co, ci, ky, kx), then one per bias element:
// d_w = sum_{b,y,x} dy[co] x_pad[ci, y+ky d, x+kx d];  d_b = sum dy[co]
template <typename T>
__global__ void __launch_bounds__(NT) k_conv_dw(const T* __restrict__ x, const T* __restrict__ dy,
                                                T* __restrict__ dw, T* __restrict__ db,
                                                ConvGeo g) {
  const int64_t nw = g.Cout * g.Cin * g.k * g.k;
  const int64_t j = blockIdx.x;
  const int64_t HW = g.H * g.W;
  double v[1] = {0.0};
  if (j < nw) {
    const int kx = (int)(j % g.k), ky = (int)(j / g.k % g.k);
    const int64_t ci = j / ((int64_t)g.k * g.k) % g.Cin, co = j / ((int64_t)g.k * g.k * g.Cin);
    for (int64_t b = 0; b < g.B; ++b) {
      const T* D = dy + (b * g.Cout + co) * HW;
      const T* X = x + (b * g.Cin + ci) * HW;
      for (int64_t p = threadIdx.x; p < HW; p += NT) {
        const int64_t yy = p / g.W, xx = p - yy * g.W;
        const int64_t sy = yy + ky * g.d - g.pad, sx = xx + kx * g.d - g.pad;
        if (sy < 0 || sy >= g.H || sx < 0 || sx >= g.W) continue;
        v[0] += (double)D[p] * (double)X[sy * g.W + sx];
      }
    }
  } else {
    const int64_t co = j - nw;
    for (int64_t b = 0; b < g.B; ++b) {
      const T* D = dy + (b * g.Cout + co) * HW;
      for (int64_t p = threadIdx.x; p < HW; p += NT) v[0] += (double)D[p];
    }
  }
  double s[1];
  block_sum<1>(v, s);
  if (threadIdx.x == 0) {
    if (j < nw)
      dw[j] = (T)s[0];
    else
      db[j - nw] = (T)s[0];
  }
}

// ---- AdaptiveNorm (gf/guidance.py:134-173) -------------------------------
// per (image, channel) plane: mean, inv_std = 1/sqrt(var + floor) with the
// population variance mean((x - mean)^2) (numpy x.var, two passes)
template <typename T>
__global__ void __launch_bounds__(NT) k_plane_stats(const T* __restrict__ x, double* stats,
                                                    int64_t HW) {
  const T* X = x + (int64_t)blockIdx.x * HW;
  double v[1] = {0.0}, s[1];
  for (int64_t p = threadIdx.x; p < HW; p += NT) v[0] += (double)X[p];
  block_sum<1>(v, s);
  const double mean = s[0] / (double)HW;
  v[0] = 0.0;
  for (int64_t p = threadIdx.x; p < HW; p += NT) {
    const double t = (double)X[p] - mean;
    v[0] += t * t;
  }
  block_sum<1>(v, s);
  if (threadIdx.x == 0) {
    stats[2 * blockIdx.x] = mean;
    stats[2 * blockIdx.x + 1] = 1.0 / sqrt(s[0] / (double)HW + kVarFloor);
  }
}

template <typename T>
__global__ void k_norm_apply(const T* __restrict__ x, T* __restrict__ y, const double* stats,
                             const T* gain, const T* norm_gain, int64_t HW, int64_t n) {
  const double ga = (double)gain[0], ng = (double)norm_gain[0];
  GF_GRID_LOOP(i, n) {
    const int64_t pl = i / HW;
    const double xv = (double)x[i];
    y[i] = (T)(ga * xv + ng * ((xv - stats[2 * pl]) * stats[2 * pl + 1]));
  }
}

// backward reductions per plane: sum dy x, sum dy xhat, sum g, sum g xhat
// (g = norm_gain dy), gf/guidance.py:161-173
template <typename T>
__global__ void __launch_bounds__(NT) k_norm_bwd_red(const T* __restrict__ x,
                                                     const T* __restrict__ dy,
                                                     const double* stats, const T* norm_gain,
                                                     double* red, int64_t HW) {
  const int64_t pl = blockIdx.x;
  const T* X = x + pl * HW;
  const T* D = dy + pl * HW;
  const double mean = stats[2 * pl], inv = stats[2 * pl + 1], ng = (double)norm_gain[0];
  double v[4] = {0.0, 0.0, 0.0, 0.0}, s[4];
  for (int64_t p = threadIdx.x; p < HW; p += NT) {
    const double xv = (double)X[p], d = (double)D[p];
    const double xh = (xv - mean) * inv, g = ng * d;
    v[0] += d * xv;
    v[1] += d * xh;
    v[2] += g;
    v[3] += g * xh;
  }
  block_sum<4>(v, s);
  if (threadIdx.x < 4) red[4 * pl + threadIdx.x] = s[threadIdx.x];
}

template <typename T>
__global__ void k_norm_bwd_dx(const T* __restrict__ x, const T* __restrict__ dy,
                              T* __restrict__ dx, const double* stats, const double* red,
                              const T* gain, const T* norm_gain, int64_t HW, int64_t n) {
  const double ga = (double)gain[0], ng = (double)norm_gain[0];
  GF_GRID_LOOP(i, n) {
    const int64_t pl = i / HW;
    const double mean = stats[2 * pl], inv = stats[2 * pl + 1];
    const double gm = red[4 * pl + 2] / (double)HW, gp = red[4 * pl + 3] / (double)HW;
    const double xh = ((double)x[i] - mean) * inv, d = (double)dy[i];
    dx[i] = (T)(ga * d + (ng * d - gm - xh * gp) * inv);
  }
}

// d_gain, d_norm_gain: sums over the planes in plane order
template <typename T>
__global__ void k_norm_bwd_params(const double* red, int64_t P, T* d_gain, T* d_norm_gain) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double a = 0.0, b = 0.0;
  for (int64_t pl = 0; pl < P; ++pl) {
    a += red[4 * pl];
    b += red[4 * pl + 1];
  }
  *d_gain = (T)a;
  *d_norm_gain = (T)b;
}

template <typename T>
void conv_fwd(const T* x, const T* w, const T* b, T* y, const ConvGeo& g, cudaStream_t s) {
  k_conv_fwd<T><<<grid_for(g.B * g.Cout * g.H * g.W), NT, 0, s>>>(x, w, b, y, g);
}

template <typename T>
void conv_bwd(const T* x, const T* w, const T* dy, T* dx, T* dw, T* db, const ConvGeo& g,
              cudaStream_t s) {
  k_conv_dx<T><<<grid_for(g.B * g.Cin * g.H * g.W), NT, 0, s>>>(dy, w, dx, g);
  const int64_t nw = g.Cout * g.Cin * g.k * g.k;
  k_conv_dw<T><<<(unsigned)(nw + (db ? g.Cout : 0)), NT, 0, s>>>(x, dy, dw, db, g);
}

template <typename T>
void norm_fwd(const T* x, T* y, const T* gain, const T* ng, int64_t P, int64_t HW, double* ws,
              cudaStream_t s) {
  k_plane_stats<T><<<(unsigned)P, NT, 0, s>>>(x, ws, HW);
  k_norm_apply<T><<<grid_for(P * HW), NT, 0, s>>>(x, y, ws, gain, ng, HW, P * HW);
}

template <typename T>
void norm_bwd(const T* x, const T* dy, T* dx, T* d_gain, T* d_ng, const T* gain, const T* ng,
              int64_t P, int64_t HW, double* ws, cudaStream_t s) {
  double* stats = ws;
  double* red = ws + 2 * P;
  k_plane_stats<T><<<(unsigned)P, NT, 0, s>>>(x, stats, HW);
  k_norm_bwd_red<T><<<(unsigned)P, NT, 0, s>>>(x, dy, stats, ng, red, HW);
  k_norm_bwd_dx<T><<<grid_for(P * HW), NT, 0, s>>>(x, dy, dx, stats, red, gain, ng, HW, P * HW);
  k_norm_bwd_params<T><<<1, 32, 0, s>>>(red, P, d_gain, d_ng);
}

}  // namespace ly
}  // namespace gfb

namespace {

using gfb::ly::ConvGeo;

int conv_check(int dtype, int64_t B, int64_t Cin, int64_t Cout, int64_t H, int64_t W, int k,
               int d) {
  if (dtype != GF_F32 && dtype != GF_F64) return gfb::api_fail(GF_ERR_ARG, "bad dtype");
  if (B < 1 || Cin < 1 || Cout < 1 || H < 1 || W < 1)
    return gfb::api_fail(GF_ERR_ARG, "conv2d: all dimensions must be >= 1");
  // gf/guidance.py:61-64
  if (k < 1 || k % 2 == 0) return gfb::api_fail(GF_ERR_ARG, "kernel must be odd and >= 1");
  if (d < 1) return gfb::api_fail(GF_ERR_ARG, "dilation must be >= 1");
  if (Cout * Cin * (int64_t)k * k + Cout > 0x7fffffff)
    return gfb::api_fail(GF_ERR_UNSUPPORTED, "conv2d: too many weights");
  return GF_OK;
}

int launched(const char* what) {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GF_OK : gfb::api_fail(GF_ERR_CUDA, cudaGetErrorString(e));
}

}  // namespace

extern "C" {

int gf_conv2d_fwd(int dtype, const void* x, const void* weight, const void* bias, void* y,
                  int64_t B, int64_t Cin, int64_t Cout, int64_t H, int64_t W, int kernel,
                  int dilation, void* stream) {
  if (int e = conv_check(dtype, B, Cin, Cout, H, W, kernel, dilation)) return e;
  const ConvGeo g{B, Cin, Cout, H, W, kernel, dilation, (kernel - 1) * dilation / 2};
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == GF_F32)
    gfb::ly::conv_fwd<float>((const float*)x, (const float*)weight, (const float*)bias,
                             (float*)y, g, s);
  else
    gfb::ly::conv_fwd<double>((const double*)x, (const double*)weight, (const double*)bias,
                              (double*)y, g, s);
  return launched("gf_conv2d_fwd");
}

int gf_conv2d_bwd(int dtype, const void* x, const void* weight, const void* dy, void* dx,
                  void* d_weight, void* d_bias, int64_t B, int64_t Cin, int64_t Cout, int64_t H,
                  int64_t W, int kernel, int dilation, void* stream) {
  if (int e = conv_check(dtype, B, Cin, Cout, H, W, kernel, dilation)) return e;
  const ConvGeo g{B, Cin, Cout, H, W, kernel, dilation, (kernel - 1) * dilation / 2};
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == GF_F32)
    gfb::ly::conv_bwd<float>((const float*)x, (const float*)weight, (const float*)dy, (float*)dx,
                             (float*)d_weight, (float*)d_bias, g, s);
  else
    gfb::ly::conv_bwd<double>((const double*)x, (const double*)weight, (const double*)dy,
                              (double*)dx, (double*)d_weight, (double*)d_bias, g, s);
  return launched("gf_conv2d_bwd");
}

size_t gf_adaptive_norm_workspace_bytes(int64_t B, int64_t C) {
  return (size_t)6 * B * C * sizeof(double);
}

int gf_adaptive_norm_fwd(int dtype, const void* x, void* y, const void* gain,
                         const void* norm_gain, int64_t B, int64_t C, int64_t H, int64_t W,
                         void* workspace, size_t workspace_bytes, void* stream) {
  if (dtype != GF_F32 && dtype != GF_F64) return gfb::api_fail(GF_ERR_ARG, "bad dtype");
  if (B < 1 || C < 1 || H < 1 || W < 1)
    return gfb::api_fail(GF_ERR_ARG, "adaptive_norm: all dimensions must be >= 1");
  if (workspace_bytes < gf_adaptive_norm_workspace_bytes(B, C))
    return gfb::api_fail(GF_ERR_WORKSPACE, "adaptive_norm workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == GF_F32)
    gfb::ly::norm_fwd<float>((const float*)x, (float*)y, (const float*)gain,
                             (const float*)norm_gain, B * C, H * W, (double*)workspace, s);
  else
    gfb::ly::norm_fwd<double>((const double*)x, (double*)y, (const double*)gain,
                              (const double*)norm_gain, B * C, H * W, (double*)workspace, s);
  return launched("gf_adaptive_norm_fwd");
}

int gf_adaptive_norm_bwd(int dtype, const void* x, const void* dy, void* dx, void* d_gain,
                         void* d_norm_gain, const void* gain, const void* norm_gain, int64_t B,
                         int64_t C, int64_t H, int64_t W, void* workspace,
                         size_t workspace_bytes, void* stream) {
  if (dtype != GF_F32 && dtype != GF_F64) return gfb::api_fail(GF_ERR_ARG, "bad dtype");
  if (B < 1 || C < 1 || H < 1 || W < 1)
    return gfb::api_fail(GF_ERR_ARG, "adaptive_norm: all dimensions must be >= 1");
  if (workspace_bytes < gf_adaptive_norm_workspace_bytes(B, C))
    return gfb::api_fail(GF_ERR_WORKSPACE, "adaptive_norm workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == GF_F32)
    gfb::ly::norm_bwd<float>((const float*)x, (const float*)dy, (float*)dx, (float*)d_gain,
                             (float*)d_norm_gain, (const float*)gain, (const float*)norm_gain,
                             B * C, H * W, (double*)workspace, s);
  else
    gfb::ly::norm_bwd<double>((const double*)x, (const double*)dy, (double*)dx, (double*)d_gain,
                              (double*)d_norm_gain, (const double*)gain,
                              (const double*)norm_gain, B * C, H * W, (double*)workspace, s);
  return launched("gf_adaptive_norm_bwd");
}

}  // extern "C"
