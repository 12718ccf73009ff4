// Training-harness kernels around the guided-filter path:
//  * FixedChannelMeanGuidance (gf/guidance.py:227-255): y_o = mean_c x_c for
//    every output channel; backward dx_c = (sum_o dy_o) / Cin;
//  * adam_step (gf/training.py:66-90) over one packed parameter vector:
//    bias-corrected Adam, in place, with the reference's non-finite-gradient
//    check (TrainingError) reported through the status word.
#include <cuda_runtime.h>

#include <cmath>

#include "gf_common.cuh"
#include "gf_internal.h"

namespace gfb {
namespace trn {

constexpr int NT = 256;

template <typename T>
__global__ void k_chan_mean(const T* __restrict__ x, T* __restrict__ y, int64_t B, int64_t Cin,
                            int64_t Cout, int64_t HW) {
  GF_GRID_LOOP(i, B * HW) {
    const int64_t b = i / HW, px = i % HW;
    double s = 0.0;  // x.mean(axis=2): sum then divide
    for (int64_t c = 0; c < Cin; ++c) s += (double)x[(b * Cin + c) * HW + px];
    const T m = (T)(s / (double)Cin);
    for (int64_t o = 0; o < Cout; ++o) y[(b * Cout + o) * HW + px] = m;
  }
}

template <typename T>
__global__ void k_chan_mean_adj(const T* __restrict__ dy, T* __restrict__ dx, int64_t B,
                                int64_t Cin, int64_t Cout, int64_t HW) {
  GF_GRID_LOOP(i, B * HW) {
    const int64_t b = i / HW, px = i % HW;
    double s = 0.0;
    for (int64_t o = 0; o < Cout; ++o) s += (double)dy[(b * Cout + o) * HW + px];
    const T g = (T)(s / (double)Cin);
    for (int64_t c = 0; c < Cin; ++c) dx[(b * Cin + c) * HW + px] = g;
  }
}

// p, m, v updated in place; g read.  bc1 = 1 - beta1^t, bc2 = 1 - beta2^t.
template <typename T>
__global__ void k_adam(T* __restrict__ p, const T* __restrict__ g, T* __restrict__ m,
                       T* __restrict__ v, int64_t n, double lr, double b1, double b2, double eps,
                       double bc1, double bc2, uint32_t* status) {
  bool bad = false;
  GF_GRID_LOOP(i, n) {
    const double gi = (double)g[i];
    if (!isfinite(gi)) {
      bad = true;
      continue;
    }
    const double mi = b1 * (double)m[i] + (1.0 - b1) * gi;
    const double vi = b2 * (double)v[i] + (1.0 - b2) * gi * gi;
    const double m_hat = mi / bc1, v_hat = vi / bc2;
    p[i] = (T)((double)p[i] - lr * m_hat / (sqrt(v_hat) + eps));
    m[i] = (T)mi;
    v[i] = (T)vi;
  }
  if (bad) flag(status, GF_STATUS_NONFINITE_INPUT);
}

}  // namespace trn

template <typename T>
void chan_mean_impl(const T* x, T* y, int64_t B, int64_t Cin, int64_t Cout, int64_t HW,
                    cudaStream_t s) {
  trn::k_chan_mean<T><<<grid_for(B * HW), trn::NT, 0, s>>>(x, y, B, Cin, Cout, HW);
}
template <typename T>
void chan_mean_adj_impl(const T* dy, T* dx, int64_t B, int64_t Cin, int64_t Cout, int64_t HW,
                        cudaStream_t s) {
  trn::k_chan_mean_adj<T><<<grid_for(B * HW), trn::NT, 0, s>>>(dy, dx, B, Cin, Cout, HW);
}
template <typename T>
void adam_impl(T* p, const T* g, T* m, T* v, int64_t n, int step, double lr, double b1, double b2,
               double eps, uint32_t* status, cudaStream_t s) {
  const double t = (double)step;  // the reference's t = state.step + 1
  const double bc1 = 1.0 - pow(b1, t), bc2 = 1.0 - pow(b2, t);
  trn::k_adam<T><<<grid_for(n), trn::NT, 0, s>>>(p, g, m, v, n, lr, b1, b2, eps, bc1, bc2,
                                                  status);
}

template void chan_mean_impl<float>(const float*, float*, int64_t, int64_t, int64_t, int64_t,
                                    cudaStream_t);
template void chan_mean_impl<double>(const double*, double*, int64_t, int64_t, int64_t, int64_t,
                                     cudaStream_t);
template void chan_mean_adj_impl<float>(const float*, float*, int64_t, int64_t, int64_t, int64_t,
                                        cudaStream_t);
template void chan_mean_adj_impl<double>(const double*, double*, int64_t, int64_t, int64_t,
                                         int64_t, cudaStream_t);
template void adam_impl<float>(float*, const float*, float*, float*, int64_t, int, double, double,
                               double, double, uint32_t*, cudaStream_t);
template void adam_impl<double>(double*, const double*, double*, double*, int64_t, int, double,
                                double, double, double, uint32_t*, cudaStream_t);

}  // namespace gfb
