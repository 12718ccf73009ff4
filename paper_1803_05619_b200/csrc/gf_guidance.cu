// 1x1 guidance network F (gf/guidance.py:184-224) and the MSE loss
// (gf/training.py:93-101) on the GPU.
//
// F(x) = W2 lrelu(gain*h1 + ng*(h1 - mu)*inv) + b2,  h1 = W1 x,
// with per-image, per-hidden-channel population statistics of h1.  Because
// conv1 is 1x1 and bias-free, mu_j and var_j follow exactly from the image's
// input moments (sum x, sum x x^T): mu = W1 m, var_j = w_j^T Cov(x) w_j, so
// the statistics cost one pass over x instead of materialising h1.
//
// The backward needs two more per-image reductions (gf/guidance.py:161-173):
// mean(g) and mean(g * xhat) per hidden channel before dx can be formed.  All
// per-pixel quantities of hidden channel j depend only on (x, dy) and the
// parameters of channel j, so the reduction kernels parallelise over
// (pixel block, j, image) with small per-thread state.  All reductions are
// deterministic: per-block float64 partials summed in a fixed order.
#include <cuda_runtime.h>

#include "gf_common.cuh"
#include "gf_internal.h"

namespace gfb {

constexpr int kGnThreads = 256;
constexpr int kGnBlocks = 48;   // pixel blocks per (j, image)
constexpr double kLeaky = 0.2;  // gf/guidance.py:25
constexpr double kVarFloor = 1e-5;  // gf/guidance.py:26

struct GnDims {
  int64_t B, Cin, Cout, hidden, HW;
  // packed parameter offsets (gf_b200.h)
  __host__ __device__ int64_t w1(int64_t j, int64_t i) const { return j * Cin + i; }
  __host__ __device__ int64_t gain() const { return hidden * Cin; }
  __host__ __device__ int64_t ng() const { return hidden * Cin + 1; }
  __host__ __device__ int64_t w2(int64_t o, int64_t j) const {
    return hidden * Cin + 2 + o * hidden + j;
  }
  __host__ __device__ int64_t b2(int64_t o) const { return hidden * Cin + 2 + Cout * hidden + o; }
  __host__ __device__ int64_t count() const { return hidden * Cin + 2 + Cout * hidden + Cout; }
};

// block reduce of NV float64 accumulators held per thread in acc[]; writes
// the block's totals to out[0..NV).
template <int NV>
__device__ void block_reduce_store(double (&acc)[NV], double* out) {
  __shared__ double red[kGnThreads / 32][NV > 0 ? NV : 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    double a = acc[v];
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) red[warp][v] = a;
  }
  __syncthreads();
  for (int v = threadIdx.x; v < NV; v += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < kGnThreads / 32; ++w) s += red[w][v];
    out[v] = s;
  }
  __syncthreads();
}

// ---- input moments: sum x_i (Cin) and sum x_i x_k (Cin*Cin) per image ----
constexpr int kMaxCin = 4;
constexpr int kStatNV = kMaxCin + kMaxCin * kMaxCin;

template <typename T>
__global__ void k_gn_stats(const T* __restrict__ x, double* __restrict__ partials, GnDims d,
                           uint32_t* status) {
  const int64_t b = blockIdx.y;
  double acc[kStatNV];
#pragma unroll
  for (int v = 0; v < kStatNV; ++v) acc[v] = 0.0;
  const T* xb = x + b * d.Cin * d.HW;
  for (int64_t pix = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pix < d.HW;
       pix += (int64_t)gridDim.x * blockDim.x) {
    double v[kMaxCin];
#pragma unroll
    for (int i = 0; i < kMaxCin; ++i) {
      v[i] = 0.0;
      if (i < d.Cin) {
        T t = xb[i * d.HW + pix];
        if (!finite(t)) flag(status, GF_STATUS_NONFINITE_INPUT);
        v[i] = (double)t;
      }
    }
#pragma unroll
    for (int i = 0; i < kMaxCin; ++i) {
      acc[i] += v[i];
#pragma unroll
      for (int k = 0; k < kMaxCin; ++k) acc[kMaxCin + i * kMaxCin + k] += v[i] * v[k];
    }
  }
  block_reduce_store<kStatNV>(acc, partials + (b * gridDim.x + blockIdx.x) * kStatNV);
}

// per (image, hidden j): mu_j, inv_j from the summed moments.
template <typename T>
__global__ void k_gn_norm(const double* __restrict__ partials, const T* __restrict__ params,
                          double* __restrict__ norm, GnDims d, int nblk) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= d.B * d.hidden) return;
  const int64_t b = idx / d.hidden, j = idx % d.hidden;
  double S[kStatNV];
  for (int v = 0; v < kStatNV; ++v) S[v] = 0.0;
  for (int k = 0; k < nblk; ++k)
    for (int v = 0; v < kStatNV; ++v) S[v] += partials[(b * nblk + k) * kStatNV + v];
  const double N = (double)d.HW;
  double m[kMaxCin];
  for (int i = 0; i < kMaxCin; ++i) m[i] = S[i] / N;
  double mu = 0.0, var = 0.0;
  for (int i = 0; i < d.Cin; ++i) mu += (double)params[d.w1(j, i)] * m[i];
  for (int i = 0; i < d.Cin; ++i)
    for (int k = 0; k < d.Cin; ++k) {
      double cov = S[kMaxCin + i * kMaxCin + k] / N - m[i] * m[k];
      var += (double)params[d.w1(j, i)] * (double)params[d.w1(j, k)] * cov;
    }
  if (var < 0.0) var = 0.0;
  norm[idx * 2 + 0] = mu;
  norm[idx * 2 + 1] = 1.0 / sqrt(var + kVarFloor);
}

// ---- forward, one pixel per thread ----
constexpr int kMaxHidden = 64;
constexpr int kMaxCout = 4;

template <typename T>
__global__ void k_gn_fwd(const T* __restrict__ x, T* __restrict__ y, const T* __restrict__ params,
                         const double* __restrict__ norm, GnDims d) {
  const int64_t b = blockIdx.y;
  const double gain = (double)params[d.gain()], ng = (double)params[d.ng()];
  const T* xb = x + b * d.Cin * d.HW;
  T* yb = y + b * d.Cout * d.HW;
  const double* nb = norm + b * d.hidden * 2;
  for (int64_t pix = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pix < d.HW;
       pix += (int64_t)gridDim.x * blockDim.x) {
    double v[kMaxCin], out[kMaxCout];
    for (int i = 0; i < kMaxCin; ++i) v[i] = i < d.Cin ? (double)xb[i * d.HW + pix] : 0.0;
    for (int o = 0; o < kMaxCout; ++o) out[o] = 0.0;
    for (int64_t j = 0; j < d.hidden; ++j) {
      double h1 = 0.0;
      for (int i = 0; i < d.Cin; ++i) h1 += v[i] * (double)params[d.w1(j, i)];
      double xhat = (h1 - nb[2 * j]) * nb[2 * j + 1];
      double h2 = gain * h1 + ng * xhat;
      double h3 = h2 >= 0.0 ? h2 : kLeaky * h2;
      for (int o = 0; o < d.Cout; ++o) out[o] += h3 * (double)params[d.w2(o, j)];
    }
    for (int o = 0; o < d.Cout; ++o) yb[o * d.HW + pix] = (T)(out[o] + (double)params[d.b2(o)]);
  }
}

// ---- backward pass 1: per (block, j, image) sums -------------------------
// acc: [0] sum d2, [1] sum d2*xhat, [2] sum d2*h1, [3..3+Cout) sum dy_o*h3,
//      [3+Cout..3+2Cout) sum dy_o (only meaningful for j == 0)
constexpr int kP1NV = 3 + 2 * kMaxCout;

template <typename T>
__device__ __forceinline__ void gn_pixel_j(const T* __restrict__ xb, const T* __restrict__ dyb,
                                           const T* __restrict__ params, const GnDims& d,
                                           int64_t j, int64_t pix, double mu, double inv,
                                           double gain, double ng, double& h1, double& xhat,
                                           double& h3, double& d2, double* dyv) {
  h1 = 0.0;
  for (int i = 0; i < d.Cin; ++i) h1 += (double)xb[i * d.HW + pix] * (double)params[d.w1(j, i)];
  xhat = (h1 - mu) * inv;
  double h2 = gain * h1 + ng * xhat;
  bool mask = h2 >= 0.0;
  h3 = mask ? h2 : kLeaky * h2;
  double d3 = 0.0;
  for (int o = 0; o < d.Cout; ++o) {
    dyv[o] = (double)dyb[o * d.HW + pix];
    d3 += dyv[o] * (double)params[d.w2(o, j)];
  }
  d2 = mask ? d3 : kLeaky * d3;
}

template <typename T>
__global__ void k_gn_bwd1(const T* __restrict__ x, const T* __restrict__ dy,
                          const T* __restrict__ params, const double* __restrict__ norm,
                          double* __restrict__ partials, GnDims d) {
  const int64_t j = blockIdx.y, b = blockIdx.z;
  const double gain = (double)params[d.gain()], ng = (double)params[d.ng()];
  const double mu = norm[(b * d.hidden + j) * 2], inv = norm[(b * d.hidden + j) * 2 + 1];
  const T* xb = x + b * d.Cin * d.HW;
  const T* dyb = dy + b * d.Cout * d.HW;
  double acc[kP1NV];
#pragma unroll
  for (int v = 0; v < kP1NV; ++v) acc[v] = 0.0;
  for (int64_t pix = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pix < d.HW;
       pix += (int64_t)gridDim.x * blockDim.x) {
    double h1, xhat, h3, d2, dyv[kMaxCout];
    gn_pixel_j(xb, dyb, params, d, j, pix, mu, inv, gain, ng, h1, xhat, h3, d2, dyv);
    acc[0] += d2;
    acc[1] += d2 * xhat;
    acc[2] += d2 * h1;
    for (int o = 0; o < d.Cout; ++o) {
      acc[3 + o] += dyv[o] * h3;
      acc[3 + kMaxCout + o] += dyv[o];
    }
  }
  block_reduce_store<kP1NV>(acc, partials + ((b * d.hidden + j) * gridDim.x + blockIdx.x) * kP1NV);
}

// sums of pass-1 partials per (image, j) -> S1[(b*hidden + j)*kP1NV + v]
__global__ void k_gn_sum1(const double* __restrict__ partials, double* __restrict__ S1,
                          int64_t count, int nblk) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= count * kP1NV) return;
  const int64_t bj = idx / kP1NV, v = idx % kP1NV;
  double s = 0.0;
  for (int k = 0; k < nblk; ++k) s += partials[(bj * nblk + k) * kP1NV + v];
  S1[idx] = s;
}

// dh1_j for one pixel given the per-image sums (gf/guidance.py:167-172)
__device__ __forceinline__ double gn_dh1(double d2, double xhat, double inv, double gain,
                                         double ng, double g_mean, double g_proj) {
  double g = ng * d2;
  return gain * d2 + (g - g_mean - xhat * g_proj) * inv;
}

// ---- backward pass 2a: dx per pixel ----
template <typename T>
__global__ void k_gn_dx(const T* __restrict__ x, const T* __restrict__ dy, T* __restrict__ dx,
                        const T* __restrict__ params, const double* __restrict__ norm,
                        const double* __restrict__ S1, GnDims d) {
  const int64_t b = blockIdx.y;
  const double gain = (double)params[d.gain()], ng = (double)params[d.ng()];
  const double N = (double)d.HW;
  const T* xb = x + b * d.Cin * d.HW;
  const T* dyb = dy + b * d.Cout * d.HW;
  for (int64_t pix = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pix < d.HW;
       pix += (int64_t)gridDim.x * blockDim.x) {
    double acc[kMaxCin];
    for (int i = 0; i < kMaxCin; ++i) acc[i] = 0.0;
    for (int64_t j = 0; j < d.hidden; ++j) {
      const int64_t bj = b * d.hidden + j;
      double h1, xhat, h3, d2, dyv[kMaxCout];
      gn_pixel_j(xb, dyb, params, d, j, pix, norm[bj * 2], norm[bj * 2 + 1], gain, ng, h1, xhat,
                 h3, d2, dyv);
      double g_mean = ng * S1[bj * kP1NV + 0] / N;
      double g_proj = ng * S1[bj * kP1NV + 1] / N;
      double dh = gn_dh1(d2, xhat, norm[bj * 2 + 1], gain, ng, g_mean, g_proj);
      for (int i = 0; i < d.Cin; ++i) acc[i] += dh * (double)params[d.w1(j, i)];
    }
    for (int i = 0; i < d.Cin; ++i) dx[(b * d.Cin + i) * d.HW + pix] = (T)acc[i];
  }
}

// ---- backward pass 2b: dW1 partials per (block, j, image) ----
template <typename T>
__global__ void k_gn_dw1(const T* __restrict__ x, const T* __restrict__ dy,
                         const T* __restrict__ params, const double* __restrict__ norm,
                         const double* __restrict__ S1, double* __restrict__ partials, GnDims d) {
  const int64_t j = blockIdx.y, b = blockIdx.z;
  const int64_t bj = b * d.hidden + j;
  const double gain = (double)params[d.gain()], ng = (double)params[d.ng()];
  const double N = (double)d.HW;
  const double mu = norm[bj * 2], inv = norm[bj * 2 + 1];
  const double g_mean = ng * S1[bj * kP1NV + 0] / N, g_proj = ng * S1[bj * kP1NV + 1] / N;
  const T* xb = x + b * d.Cin * d.HW;
  const T* dyb = dy + b * d.Cout * d.HW;
  double acc[kMaxCin];
#pragma unroll
  for (int i = 0; i < kMaxCin; ++i) acc[i] = 0.0;
  for (int64_t pix = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pix < d.HW;
       pix += (int64_t)gridDim.x * blockDim.x) {
    double h1, xhat, h3, d2, dyv[kMaxCout];
    gn_pixel_j(xb, dyb, params, d, j, pix, mu, inv, gain, ng, h1, xhat, h3, d2, dyv);
    double dh = gn_dh1(d2, xhat, inv, gain, ng, g_mean, g_proj);
    for (int i = 0; i < d.Cin; ++i) acc[i] += dh * (double)xb[i * d.HW + pix];
  }
  block_reduce_store<kMaxCin>(acc, partials + (bj * gridDim.x + blockIdx.x) * kMaxCin);
}

// final parameter gradients (single thread block; fixed summation order)
template <typename T>
__global__ void k_gn_final(const double* __restrict__ S1, const double* __restrict__ pw1,
                           T* __restrict__ dparams, int accumulate, GnDims d, int nblk) {
  for (int64_t idx = threadIdx.x; idx < d.count(); idx += blockDim.x) {
    double s = 0.0;
    if (idx < d.hidden * d.Cin) {  // conv1.weight[j][i]
      const int64_t j = idx / d.Cin, i = idx % d.Cin;
      for (int64_t b = 0; b < d.B; ++b)
        for (int k = 0; k < nblk; ++k) s += pw1[((b * d.hidden + j) * nblk + k) * kMaxCin + i];
    } else if (idx == d.gain()) {  // sum_j sum_px d2*h1
      for (int64_t b = 0; b < d.B; ++b)
        for (int64_t j = 0; j < d.hidden; ++j) s += S1[(b * d.hidden + j) * kP1NV + 2];
    } else if (idx == d.ng()) {  // sum_j sum_px d2*xhat
      for (int64_t b = 0; b < d.B; ++b)
        for (int64_t j = 0; j < d.hidden; ++j) s += S1[(b * d.hidden + j) * kP1NV + 1];
    } else if (idx < d.b2(0)) {  // conv2.weight[o][j]
      const int64_t k = idx - (d.hidden * d.Cin + 2);
      const int64_t o = k / d.hidden, j = k % d.hidden;
      for (int64_t b = 0; b < d.B; ++b) s += S1[(b * d.hidden + j) * kP1NV + 3 + o];
    } else {  // conv2.bias[o]
      const int64_t o = idx - d.b2(0);
      for (int64_t b = 0; b < d.B; ++b) s += S1[(b * d.hidden + 0) * kP1NV + 3 + kMaxCout + o];
    }
    dparams[idx] = accumulate ? (T)((double)dparams[idx] + s) : (T)s;
  }
}

// ---- MSE (gf/training.py:93-101), batch-mean ----
template <typename T>
__global__ void k_mse(const T* __restrict__ out, const T* __restrict__ tgt, T* __restrict__ d_out,
                      double* __restrict__ partials, int64_t per_image, double scale) {
  const int64_t b = blockIdx.y;
  double acc[1] = {0.0};
  const int64_t base = b * per_image;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < per_image;
       i += (int64_t)gridDim.x * blockDim.x) {
    double diff = (double)out[base + i] - (double)tgt[base + i];
    acc[0] += diff * diff;
    d_out[base + i] = (T)(2.0 * diff * scale);
  }
  block_reduce_store<1>(acc, partials + b * gridDim.x + blockIdx.x);
}

// fp32 fast path: 128-bit accesses, fp32 per-thread sums (a few hundred
// elements each), float64 across threads and blocks
__global__ void k_mse4(const float* __restrict__ out, const float* __restrict__ tgt,
                       float* __restrict__ d_out, double* __restrict__ partials, int64_t per_image,
                       float scale2) {
  const int64_t b = blockIdx.y;
  const float4* o4 = reinterpret_cast<const float4*>(out + b * per_image);
  const float4* t4 = reinterpret_cast<const float4*>(tgt + b * per_image);
  float4* d4 = reinterpret_cast<float4*>(d_out + b * per_image);
  float s = 0.f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < per_image / 4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float4 o = __ldg(o4 + i), t = __ldg(t4 + i);
    const float e0 = o.x - t.x, e1 = o.y - t.y, e2 = o.z - t.z, e3 = o.w - t.w;
    s = fmaf(e0, e0, fmaf(e1, e1, fmaf(e2, e2, fmaf(e3, e3, s))));
    d4[i] = make_float4(scale2 * e0, scale2 * e1, scale2 * e2, scale2 * e3);
  }
  double acc[1] = {(double)s};
  block_reduce_store<1>(acc, partials + b * gridDim.x + blockIdx.x);
}

__global__ void k_mse_final(const double* __restrict__ partials, double* __restrict__ loss,
                            int64_t B, int nblk, double per_image) {
  // one warp per image sums its block partials (fixed lane order), then
  // thread 0 adds the images in order
  __shared__ double img[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double total = 0.0;
  for (int64_t b0 = 0; b0 < B; b0 += 32) {
    const int64_t b = b0 + warp;
    if (warp < 32 && b < B) {
      double s = 0.0;
      for (int k = lane; k < nblk; k += 32) s += partials[b * nblk + k];
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) img[warp] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int64_t k = 0; k < 32 && b0 + k < B; ++k) total += (img[k] / per_image) / (double)B;
    __syncthreads();
  }
  if (threadIdx.x == 0) *loss = total;
}

// ===========================================================================
// host side
// ===========================================================================

size_t gn_ws_bytes(int64_t B, int64_t hidden) {
  size_t stats = (size_t)B * kGnBlocks * kStatNV;
  size_t norm = (size_t)B * hidden * 2;
  size_t p1 = (size_t)B * hidden * kGnBlocks * kP1NV;
  size_t s1 = (size_t)B * hidden * kP1NV;
  size_t pw1 = (size_t)B * hidden * kGnBlocks * kMaxCin;
  return (stats + norm + p1 + s1 + pw1) * sizeof(double);
}

bool gn_supported(int64_t Cin, int64_t Cout, int64_t hidden) {
  return Cin >= 1 && Cin <= kMaxCin && Cout >= 1 && Cout <= kMaxCout && hidden >= 1 &&
         hidden <= kMaxHidden;
}

template <typename T>
static void gn_stats_norm(const T* x, const T* params, const GnDims& d, double* ws,
                          uint32_t* status, cudaStream_t s) {
  double* stats = ws;
  double* norm = stats + d.B * kGnBlocks * kStatNV;
  k_gn_stats<T><<<dim3(kGnBlocks, (unsigned)d.B), kGnThreads, 0, s>>>(x, stats, d, status);
  int64_t cnt = d.B * d.hidden;
  k_gn_norm<T><<<(unsigned)((cnt + 127) / 128), 128, 0, s>>>(stats, params, norm, d, kGnBlocks);
}

template <typename T>
void gn_forward_impl(const T* x, T* y, const T* params, int64_t B, int64_t Cin, int64_t Cout,
                     int64_t hidden, int64_t HW, void* ws, uint32_t* status, cudaStream_t s) {
  GnDims d{B, Cin, Cout, hidden, HW};
  double* w = (double*)ws;
  gn_stats_norm<T>(x, params, d, w, status, s);
  double* norm = w + B * kGnBlocks * kStatNV;
  int gx = (int)((HW + kGnThreads - 1) / kGnThreads);
  if (gx > 1024) gx = 1024;
  k_gn_fwd<T><<<dim3(gx, (unsigned)B), kGnThreads, 0, s>>>(x, y, params, norm, d);
}

template <typename T>
void gn_backward_impl(const T* x, const T* dy, T* dx, T* dparams, int accumulate, const T* params,
                      int64_t B, int64_t Cin, int64_t Cout, int64_t hidden, int64_t HW, void* ws,
                      uint32_t* status, cudaStream_t s) {
  GnDims d{B, Cin, Cout, hidden, HW};
  double* w = (double*)ws;
  gn_stats_norm<T>(x, params, d, w, status, s);
  double* norm = w + B * kGnBlocks * kStatNV;
  double* p1 = norm + B * hidden * 2;
  double* S1 = p1 + B * hidden * kGnBlocks * kP1NV;
  double* pw1 = S1 + B * hidden * kP1NV;
  k_gn_bwd1<T><<<dim3(kGnBlocks, (unsigned)hidden, (unsigned)B), kGnThreads, 0, s>>>(
      x, dy, params, norm, p1, d);
  int64_t cnt = B * hidden * kP1NV;
  k_gn_sum1<<<(unsigned)((cnt + 127) / 128), 128, 0, s>>>(p1, S1, B * hidden, kGnBlocks);
  int gx = (int)((HW + kGnThreads - 1) / kGnThreads);
  if (gx > 1024) gx = 1024;
  k_gn_dx<T><<<dim3(gx, (unsigned)B), kGnThreads, 0, s>>>(x, dy, dx, params, norm, S1, d);
  k_gn_dw1<T><<<dim3(kGnBlocks, (unsigned)hidden, (unsigned)B), kGnThreads, 0, s>>>(
      x, dy, params, norm, S1, pw1, d);
  k_gn_final<T><<<1, 256, 0, s>>>(S1, pw1, dparams, accumulate, d, kGnBlocks);
}

constexpr int kMseBlocks = 256;  // per image

size_t mse_ws_bytes(int64_t B) { return (size_t)B * kMseBlocks * sizeof(double); }

template <typename T>
void mse_impl(const T* out, const T* tgt, T* d_out, double* loss, int64_t B, int64_t per_image,
              void* ws, cudaStream_t s) {
  double* partials = (double*)ws;
  double scale = 1.0 / (double)per_image / (double)B;
  if (sizeof(T) == 4 && per_image % 4 == 0 && ((uintptr_t)out & 15) == 0 &&
      ((uintptr_t)tgt & 15) == 0 && ((uintptr_t)d_out & 15) == 0) {
    k_mse4<<<dim3(kMseBlocks, (unsigned)B), kGnThreads, 0, s>>>(
        (const float*)out, (const float*)tgt, (float*)d_out, partials, per_image,
        (float)(2.0 * scale));
  } else {
    k_mse<T><<<dim3(kMseBlocks, (unsigned)B), kGnThreads, 0, s>>>(out, tgt, d_out, partials,
                                                                   per_image, scale);
  }
  k_mse_final<<<1, 1024, 0, s>>>(partials, loss, B, kMseBlocks, (double)per_image);
}

void mse_final(const double* partials, double* loss, int64_t B, int nblk, double per_image,
               cudaStream_t s) {
  k_mse_final<<<1, 1024, 0, s>>>(partials, loss, B, nblk, per_image);
}

#define GN_INST(T)                                                                            \
  template void gn_forward_impl<T>(const T*, T*, const T*, int64_t, int64_t, int64_t, int64_t, \
                                   int64_t, void*, uint32_t*, cudaStream_t);                  \
  template void gn_backward_impl<T>(const T*, const T*, T*, T*, int, const T*, int64_t,       \
                                    int64_t, int64_t, int64_t, int64_t, void*, uint32_t*,     \
                                    cudaStream_t);                                            \
  template void mse_impl<T>(const T*, const T*, T*, double*, int64_t, int64_t, void*,         \
                            cudaStream_t);
GN_INST(float)
GN_INST(double)

}  // namespace gfb
