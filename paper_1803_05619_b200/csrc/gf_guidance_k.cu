// Guidance / core net with a k x k (dilated) first convolution -- the
// reference's GuidanceNet(kernel=k, dilation=d) (gf/guidance.py:184-224 with
// ConvLayer :52-124, AdaptiveNorm :134-173) as used for the low-res core net
// C_l of GuidedUpsampler (gf/training.py:186-207: k=3, hidden 24).
//
//   h1 = conv1(x)  (k x k, dilation d, zero "same" padding, no bias)
//   h2 = gain*h1 + ng*(h1 - mu)*inv     (per image, per channel; var floor 1e-5)
//   h3 = lrelu_0.2(h2);  y = W2 h3 + b2
//
// General kernels for both dtypes (fp64 reproduces the reference to its own
// bars): h1 is materialised in the workspace (B*hidden planes), channel
// statistics are two-pass (mean, then centred squares) like numpy's var, and
// every parameter gradient is a deterministic block reduction (one block per
// output scalar, fixed order, float64) -- no atomics.
#include <cuda_runtime.h>

#include "gf_common.cuh"
#include "gf_internal.h"

namespace gfb {
namespace gnk {

constexpr int NT = 256;
constexpr double kVarFloor = 1e-5;
constexpr double kLeaky = 0.2;

struct Dims {
  int64_t B, Cin, Cout, hid, H, W, HW;
  int k, d, pad;
  __host__ __device__ int64_t nw1() const { return hid * Cin * k * k; }
  __host__ __device__ int64_t gain() const { return nw1(); }
  __host__ __device__ int64_t ng() const { return nw1() + 1; }
  __host__ __device__ int64_t w2() const { return nw1() + 2; }
  __host__ __device__ int64_t b2() const { return nw1() + 2 + Cout * hid; }
  __host__ __device__ int64_t count() const { return nw1() + 2 + Cout * hid + Cout; }
};

// float64 block sum of one value per thread -> returned to every thread
__device__ double block_sum(double v) {
  __shared__ double red[NT / 32];
  __shared__ double tot;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < NT / 32; ++w) s += red[w];
    tot = s;
  }
  __syncthreads();
  const double r = tot;
  __syncthreads();
  return r;
}

// ---- forward ----------------------------------------------------------------
template <typename T>
__global__ void k_conv1(const T* __restrict__ x, const T* __restrict__ P, T* __restrict__ h1,
                        Dims D) {
  const int64_t n = D.B * D.hid * D.HW;
  for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT) {
    const int64_t px = i % D.HW, bj = i / D.HW;
    const int64_t j = bj % D.hid, b = bj / D.hid;
    const int y = (int)(px / D.W), xx = (int)(px % D.W);
    double acc = 0.0;
    for (int c = 0; c < D.Cin; ++c) {
      const T* xc = x + (b * D.Cin + c) * D.HW;
      const T* w = P + ((j * D.Cin + c) * D.k) * D.k;
      for (int ky = 0; ky < D.k; ++ky) {
        const int yy = y + ky * D.d - D.pad;
        if (yy < 0 || yy >= D.H) continue;
        for (int kx = 0; kx < D.k; ++kx) {
          const int xs = xx + kx * D.d - D.pad;
          if (xs < 0 || xs >= D.W) continue;
          acc += (double)w[ky * D.k + kx] * (double)xc[(int64_t)yy * D.W + xs];
        }
      }
    }
    h1[i] = (T)acc;
  }
}

// per (b, j): mu, inv = 1/sqrt(var + 1e-5), two-pass population variance
template <typename T>
__global__ void k_chan_stats(const T* __restrict__ h1, double* __restrict__ stats, Dims D) {
  const int64_t bj = blockIdx.x;
  const T* h = h1 + bj * D.HW;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < D.HW; i += NT) s += (double)h[i];
  const double mu = block_sum(s) / (double)D.HW;
  double q = 0.0;
  for (int64_t i = threadIdx.x; i < D.HW; i += NT) {
    const double e = (double)h[i] - mu;
    q += e * e;
  }
  const double var = block_sum(q) / (double)D.HW;
  if (threadIdx.x == 0) {
    stats[2 * bj] = mu;
    stats[2 * bj + 1] = 1.0 / sqrt(var + kVarFloor);
  }
}

template <typename T>
__device__ __forceinline__ double h2_of(double h1v, double mu, double inv, double gain, double ng) {
  return gain * h1v + ng * ((h1v - mu) * inv);
}

template <typename T>
__global__ void k_head(const T* __restrict__ h1, const double* __restrict__ stats,
                       const T* __restrict__ P, T* __restrict__ y, uint32_t* status, Dims D) {
  const double gain = (double)P[D.gain()], ng = (double)P[D.ng()];
  const int64_t n = D.B * D.HW;
  bool bad = false;
  for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT) {
    const int64_t px = i % D.HW, b = i / D.HW;
    for (int o = 0; o < D.Cout; ++o) {
      double acc = (double)P[D.b2() + o];
      for (int j = 0; j < D.hid; ++j) {
        const int64_t bj = b * D.hid + j;
        const double v = h2_of<T>((double)h1[bj * D.HW + px], stats[2 * bj], stats[2 * bj + 1],
                                  gain, ng);
        const double h3 = v >= 0.0 ? v : kLeaky * v;
        acc += (double)P[D.w2() + o * D.hid + j] * h3;
      }
      const T out = (T)acc;
      if (!finite(out)) bad = true;
      y[(b * D.Cout + o) * D.HW + px] = out;
    }
  }
  if (bad) flag(status, GF_STATUS_NONFINITE_OUTPUT);
}

// ---- backward ---------------------------------------------------------------
// d2 = lrelu'(h2) * W2^T dy, per (b, j, px)
template <typename T>
__global__ void k_d2(const T* __restrict__ h1, const double* __restrict__ stats,
                     const T* __restrict__ P, const T* __restrict__ dy, T* __restrict__ d2,
                     Dims D) {
  const double gain = (double)P[D.gain()], ng = (double)P[D.ng()];
  const int64_t n = D.B * D.hid * D.HW;
  for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT) {
    const int64_t px = i % D.HW, bj = i / D.HW;
    const int64_t j = bj % D.hid, b = bj / D.hid;
    const double v = h2_of<T>((double)h1[i], stats[2 * bj], stats[2 * bj + 1], gain, ng);
    double d3 = 0.0;
    for (int o = 0; o < D.Cout; ++o)
      d3 += (double)P[D.w2() + o * D.hid + j] * (double)dy[(b * D.Cout + o) * D.HW + px];
    d2[i] = (T)(v >= 0.0 ? d3 : kLeaky * d3);
  }
}

// per (b, j): S[0] = sum d2, S[1] = sum d2*h1, S[2] = sum d2*xhat
template <typename T>
__global__ void k_red_norm(const T* __restrict__ h1, const T* __restrict__ d2,
                           const double* __restrict__ stats, double* __restrict__ S, Dims D) {
  const int64_t bj = blockIdx.x;
  const T* h = h1 + bj * D.HW;
  const T* g = d2 + bj * D.HW;
  const double mu = stats[2 * bj], inv = stats[2 * bj + 1];
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (int64_t i = threadIdx.x; i < D.HW; i += NT) {
    const double gv = (double)g[i], hv = (double)h[i];
    s0 += gv;
    s1 += gv * hv;
    s2 += gv * ((hv - mu) * inv);
  }
  s0 = block_sum(s0);
  s1 = block_sum(s1);
  s2 = block_sum(s2);
  if (threadIdx.x == 0) {
    S[3 * bj] = s0;
    S[3 * bj + 1] = s1;
    S[3 * bj + 2] = s2;
  }
}

// per (b, o, j): sum dy_o * h3_j;  j == hid: sum dy_o (conv2 bias)
template <typename T>
__global__ void k_red_w2(const T* __restrict__ h1, const double* __restrict__ stats,
                         const T* __restrict__ P, const T* __restrict__ dy,
                         double* __restrict__ G2, Dims D) {
  const int64_t id = blockIdx.x;  // (b, o, j) with j in [0, hid]
  const int64_t j = id % (D.hid + 1), bo = id / (D.hid + 1);
  const int64_t o = bo % D.Cout, b = bo / D.Cout;
  const T* g = dy + (b * D.Cout + o) * D.HW;
  const double gain = (double)P[D.gain()], ng = (double)P[D.ng()];
  double s = 0.0;
  if (j == D.hid) {
    for (int64_t i = threadIdx.x; i < D.HW; i += NT) s += (double)g[i];
  } else {
    const int64_t bj = b * D.hid + j;
    const T* h = h1 + bj * D.HW;
    const double mu = stats[2 * bj], inv = stats[2 * bj + 1];
    for (int64_t i = threadIdx.x; i < D.HW; i += NT) {
      const double v = h2_of<T>((double)h[i], mu, inv, gain, ng);
      s += (double)g[i] * (v >= 0.0 ? v : kLeaky * v);
    }
  }
  s = block_sum(s);
  if (threadIdx.x == 0) G2[id] = s;
}

// d2 -> dh1 in place: gain*d2 + (g - mean g - xhat mean(g xhat))*inv, g = ng*d2
template <typename T>
__global__ void k_dh1(const T* __restrict__ h1, T* __restrict__ d2, const double* __restrict__ stats,
                      const double* __restrict__ S, const T* __restrict__ P, Dims D) {
  const double gain = (double)P[D.gain()], ng = (double)P[D.ng()];
  const double N = (double)D.HW;
  const int64_t n = D.B * D.hid * D.HW;
  for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT) {
    const int64_t bj = i / D.HW;
    const double mu = stats[2 * bj], inv = stats[2 * bj + 1];
    const double gm = ng * S[3 * bj] / N, gp = ng * S[3 * bj + 2] / N;
    const double dv = (double)d2[i];
    const double xhat = ((double)h1[i] - mu) * inv;
    d2[i] = (T)(gain * dv + (ng * dv - gm - xhat * gp) * inv);
  }
}

// dx = conv1^T(dh1), per (b, c, px)
template <typename T>
__global__ void k_conv1_t(const T* __restrict__ dh1, const T* __restrict__ P, T* __restrict__ dx,
                          Dims D) {
  const int64_t n = D.B * D.Cin * D.HW;
  for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT) {
    const int64_t px = i % D.HW, bc = i / D.HW;
    const int64_t c = bc % D.Cin, b = bc / D.Cin;
    const int y = (int)(px / D.W), xx = (int)(px % D.W);
    double acc = 0.0;
    for (int j = 0; j < D.hid; ++j) {
      const T* g = dh1 + (b * D.hid + j) * D.HW;
      const T* w = P + ((j * D.Cin + c) * D.k) * D.k;
      for (int ky = 0; ky < D.k; ++ky) {
        const int yy = y - ky * D.d + D.pad;
        if (yy < 0 || yy >= D.H) continue;
        for (int kx = 0; kx < D.k; ++kx) {
          const int xs = xx - kx * D.d + D.pad;
          if (xs < 0 || xs >= D.W) continue;
          acc += (double)w[ky * D.k + kx] * (double)g[(int64_t)yy * D.W + xs];
        }
      }
    }
    dx[i] = (T)acc;
  }
}

// per (b, j, c, ky, kx): sum_px dh1_j(px) * x_c(px + (ky d - pad, kx d - pad))
template <typename T>
__global__ void k_red_w1(const T* __restrict__ dh1, const T* __restrict__ x,
                         double* __restrict__ G1, Dims D) {
  const int64_t id = blockIdx.x;
  const int64_t kk = D.k * D.k;
  const int64_t t = id % kk, jc = (id / kk) % (D.hid * D.Cin), b = id / (kk * D.hid * D.Cin);
  const int ky = (int)(t / D.k), kx = (int)(t % D.k);
  const int64_t j = jc / D.Cin, c = jc % D.Cin;
  const T* g = dh1 + (b * D.hid + j) * D.HW;
  const T* xc = x + (b * D.Cin + c) * D.HW;
  const int oy = ky * D.d - D.pad, ox = kx * D.d - D.pad;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < D.HW; i += NT) {
    const int y = (int)(i / D.W) + oy, xs = (int)(i % D.W) + ox;
    if (y < 0 || y >= D.H || xs < 0 || xs >= D.W) continue;
    s += (double)g[i] * (double)xc[(int64_t)y * D.W + xs];
  }
  s = block_sum(s);
  if (threadIdx.x == 0) G1[id] = s;
}

// sum the per-image partials in image order; write or accumulate dparams
template <typename T>
__global__ void k_fin(const double* __restrict__ G1, const double* __restrict__ S,
                      const double* __restrict__ G2, T* __restrict__ dP, int accumulate, Dims D) {
  const int64_t n = D.count();
  for (int64_t v = (int64_t)blockIdx.x * NT + threadIdx.x; v < n; v += (int64_t)gridDim.x * NT) {
    double s = 0.0;
    for (int64_t b = 0; b < D.B; ++b) {
      if (v < D.nw1()) {
        s += G1[b * D.nw1() + v];
      } else if (v == D.gain() || v == D.ng()) {
        for (int j = 0; j < D.hid; ++j) s += S[3 * (b * D.hid + j) + (v == D.gain() ? 1 : 2)];
      } else if (v < D.b2()) {
        const int64_t u = v - D.w2(), o = u / D.hid, j = u % D.hid;
        s += G2[(b * D.Cout + o) * (D.hid + 1) + j];
      } else {
        const int64_t o = v - D.b2();
        s += G2[(b * D.Cout + o) * (D.hid + 1) + D.hid];
      }
    }
    dP[v] = accumulate ? (T)((double)dP[v] + s) : (T)s;
  }
}

struct WS {
  void* h1;
  void* d2;
  double* stats;
  double* S;
  double* G2;
  double* G1;
};

inline size_t up256(size_t n) { return (n + 255) / 256 * 256; }

inline WS carve(void* ws, const Dims& D, size_t es) {
  char* p = (char*)ws;
  WS w;
  const size_t plane = (size_t)D.B * D.hid * D.HW * es;
  w.h1 = p;
  p += up256(plane);
  w.d2 = p;
  p += up256(plane);
  w.stats = (double*)p;
  p += up256(sizeof(double) * 2 * D.B * D.hid);
  w.S = (double*)p;
  p += up256(sizeof(double) * 3 * D.B * D.hid);
  w.G2 = (double*)p;
  p += up256(sizeof(double) * D.B * D.Cout * (D.hid + 1));
  w.G1 = (double*)p;
  return w;
}

inline int blocks(int64_t n) {
  int64_t b = (n + NT - 1) / NT;
  return (int)(b < 1 ? 1 : (b > 148 * 16 ? 148 * 16 : b));
}

}  // namespace gnk

size_t gnk_ws_bytes_impl(int64_t B, int64_t Cin, int64_t Cout, int64_t hid, int k, int64_t HW,
                         size_t es) {
  using gnk::up256;
  const size_t plane = (size_t)B * hid * HW * es;
  return 2 * up256(plane) + up256(sizeof(double) * 2 * B * hid) +
         up256(sizeof(double) * 3 * B * hid) + up256(sizeof(double) * B * Cout * (hid + 1)) +
         up256(sizeof(double) * B * hid * Cin * k * k) + 256;
}

template <typename T>
void gnk_forward_impl(const T* x, T* y, const T* params, int64_t B, int64_t Cin, int64_t Cout,
                      int64_t hid, int k, int d, int64_t H, int64_t W, void* ws, uint32_t* status,
                      cudaStream_t s) {
  gnk::Dims D{B, Cin, Cout, hid, H, W, H * W, k, d, (k - 1) * d / 2};
  gnk::WS w = gnk::carve(ws, D, sizeof(T));
  gnk::k_conv1<T><<<gnk::blocks(B * hid * H * W), gnk::NT, 0, s>>>(x, params, (T*)w.h1, D);
  gnk::k_chan_stats<T><<<(unsigned)(B * hid), gnk::NT, 0, s>>>((const T*)w.h1, w.stats, D);
  gnk::k_head<T><<<gnk::blocks(B * H * W), gnk::NT, 0, s>>>((const T*)w.h1, w.stats, params, y,
                                                              status, D);
}

template <typename T>
void gnk_backward_impl(const T* x, const T* dy, T* dx, T* dparams, int accumulate, const T* params,
                       int64_t B, int64_t Cin, int64_t Cout, int64_t hid, int k, int d, int64_t H,
                       int64_t W, void* ws, uint32_t* status, cudaStream_t s) {
  (void)status;
  gnk::Dims D{B, Cin, Cout, hid, H, W, H * W, k, d, (k - 1) * d / 2};
  gnk::WS w = gnk::carve(ws, D, sizeof(T));
  T* h1 = (T*)w.h1;
  T* d2 = (T*)w.d2;
  const int64_t n = B * hid * H * W;
  // forward intermediates (h1, statistics) are recomputed: the tape is x only
  gnk::k_conv1<T><<<gnk::blocks(n), gnk::NT, 0, s>>>(x, params, h1, D);
  gnk::k_chan_stats<T><<<(unsigned)(B * hid), gnk::NT, 0, s>>>(h1, w.stats, D);
  gnk::k_d2<T><<<gnk::blocks(n), gnk::NT, 0, s>>>(h1, w.stats, params, dy, d2, D);
  gnk::k_red_norm<T><<<(unsigned)(B * hid), gnk::NT, 0, s>>>(h1, d2, w.stats, w.S, D);
  gnk::k_red_w2<T><<<(unsigned)(B * Cout * (hid + 1)), gnk::NT, 0, s>>>(h1, w.stats, params, dy,
                                                                       w.G2, D);
  gnk::k_dh1<T><<<gnk::blocks(n), gnk::NT, 0, s>>>(h1, d2, w.stats, w.S, params, D);
  gnk::k_conv1_t<T><<<gnk::blocks(B * Cin * H * W), gnk::NT, 0, s>>>(d2, params, dx, D);
  gnk::k_red_w1<T><<<(unsigned)(B * hid * Cin * k * k), gnk::NT, 0, s>>>(d2, x, w.G1, D);
  gnk::k_fin<T><<<gnk::blocks(D.count()), gnk::NT, 0, s>>>(w.G1, w.S, w.G2, dparams, accumulate,
                                                          D);
}

template void gnk_forward_impl<float>(const float*, float*, const float*, int64_t, int64_t, int64_t,
                                      int64_t, int, int, int64_t, int64_t, void*, uint32_t*,
                                      cudaStream_t);
template void gnk_forward_impl<double>(const double*, double*, const double*, int64_t, int64_t,
                                       int64_t, int64_t, int, int, int64_t, int64_t, void*,
                                       uint32_t*, cudaStream_t);
template void gnk_backward_impl<float>(const float*, const float*, float*, float*, int,
                                       const float*, int64_t, int64_t, int64_t, int64_t, int, int,
                                       int64_t, int64_t, void*, uint32_t*, cudaStream_t);
template void gnk_backward_impl<double>(const double*, const double*, double*, double*, int,
                                        const double*, int64_t, int64_t, int64_t, int64_t, int,
                                        int, int64_t, int64_t, void*, uint32_t*, cudaStream_t);

}  // namespace gfb
