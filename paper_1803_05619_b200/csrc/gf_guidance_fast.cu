// Fast fp32 1x1 guidance net (gf/guidance.py:184-224) for Cin = Cout = 3 and
// a compile-time hidden width (BASELINE config 2: 3 -> 15 -> 3).
//
// Forward per image: one statistics pass (sum x, sum x x^T in float64 block
// partials), a tiny "prep" kernel that folds AdaptiveNorm into conv1,
//     h2 = gain*h1 + ng*(h1 - mu)*inv = (alpha .* W1) x + beta,
//     alpha_j = gain + ng*inv_j,  beta_j = -ng*inv_j*mu_j,
// and one streaming pass: 4 pixels per thread (128-bit loads/stores), the
// folded weights read from shared memory by broadcast.
//
// Backward per image (gf/guidance.py:161-173, 106-124): pass A streams (x, dy)
// and reduces sum d2_j, sum d2_j*h1_j, sum dy_o, sum dy_o*h3_j (fp32 per
// thread over <= 64 pixels, then float64 across threads and blocks);
// a finalize kernel turns them into mean(g), mean(g*xhat) and the dW2, db2,
// gain, norm_gain gradients; pass B streams (x, dy) again and writes
// dx = W1^T dh1 with dh1_j = alpha_j d2_j + kappa_j + lambda_j h1_j while
// reducing dW1 = sum dh1 x^T.  Every reduction is deterministic.
#include <cuda_runtime.h>

#include "gf_common.cuh"
#include "gf_internal.h"
#include "gf_pair.cuh"

namespace gfb {
namespace gnf {

constexpr int CI = 3, CO = 3;
constexpr int NT = 256;
constexpr int kBlocks = 128;  // pixel blocks per image (grid.x)
constexpr float kLeaky = 0.2f;
constexpr double kVarFloor = 1e-5;
constexpr int NST = 3;  // cp.async pipeline stages of the streaming passes

// ---- cp.async staging of the streaming passes: the two lanes of a pair
// share one 4-pixel group; the even lane copies its three x chunks, the odd
// lane its three dy chunks, and a __syncwarp after the wait_group publishes
// them to the partner (another before the refill retires the partner's reads)
__device__ __forceinline__ void cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// packed parameter layout (include/gf_b200.h)
template <int HID>
struct P {
  static constexpr int w1 = 0, gain = HID * CI, ng = HID * CI + 1, w2 = HID * CI + 2,
                       b2 = HID * CI + 2 + CO * HID, count = HID * CI + 2 + CO * HID + CO;
};

// per-image folded constants (fp32) written by prep:
//   W1f[HID*CI] (alpha .* W1), beta[HID], W1[HID*CI], alpha[HID], mu[HID], inv[HID]
template <int HID>
struct F {
  static constexpr int w1f = 0, beta = HID * CI, w1 = HID * CI + HID, alpha = 2 * HID * CI + HID,
                       mu = 2 * HID * CI + 2 * HID, inv = 2 * HID * CI + 3 * HID,
                       count = 2 * HID * CI + 4 * HID;
};

// block reduce of NV float64 accumulators per thread -> out[0..NV)
template <int NV, typename T>
__device__ void reduce_store(const T (&acc)[NV], double* out) {
  __shared__ double red[NT / 32][NV];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    double a = (double)acc[v];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) red[warp][v] = a;
  }
  __syncthreads();
  for (int v = threadIdx.x; v < NV; v += NT) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) s += red[w][v];
    out[v] = s;
  }
  __syncthreads();
}

// ---- statistics: sum x_i (3), sum x_i x_k (6) per image --------------------
__global__ void __launch_bounds__(NT) k_stats(const float* __restrict__ x, double* __restrict__ part,
                                              int64_t HW, uint32_t* status) {
  const int64_t b = blockIdx.y;
  const float4* x0 = reinterpret_cast<const float4*>(x + (b * CI + 0) * HW);
  const float4* x1 = reinterpret_cast<const float4*>(x + (b * CI + 1) * HW);
  const float4* x2 = reinterpret_cast<const float4*>(x + (b * CI + 2) * HW);
  const int64_t n4 = HW / 4;
  double acc[9];
#pragma unroll
  for (int v = 0; v < 9; ++v) acc[v] = 0.0;
  bool bad = false;
  // fp32 partials over at most 64 chunks, then folded into float64
  int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * NT;
  while (i < n4) {
    float f[9];
#pragma unroll
    for (int v = 0; v < 9; ++v) f[v] = 0.f;
    for (int k = 0; k < 64 && i < n4; ++k, i += stride) {
      const float4 a = __ldg(x0 + i), c = __ldg(x1 + i), d = __ldg(x2 + i);
      const float p0[4] = {a.x, a.y, a.z, a.w}, p1[4] = {c.x, c.y, c.z, c.w},
                  p2[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        bad |= !isfinite(p0[q]) || !isfinite(p1[q]) || !isfinite(p2[q]);
        f[0] += p0[q];
        f[1] += p1[q];
        f[2] += p2[q];
        f[3] += p0[q] * p0[q];
        f[4] += p0[q] * p1[q];
        f[5] += p0[q] * p2[q];
        f[6] += p1[q] * p1[q];
        f[7] += p1[q] * p2[q];
        f[8] += p2[q] * p2[q];
      }
    }
#pragma unroll
    for (int v = 0; v < 9; ++v) acc[v] += (double)f[v];
  }
  if (bad) flag(status, GF_STATUS_NONFINITE_INPUT);
  reduce_store<9>(acc, part + (b * gridDim.x + blockIdx.x) * 9);
}

// ---- prep: per image folded constants ------------------------------------
template <int HID>
__global__ void k_prep(const double* __restrict__ part, const float* __restrict__ params,
                       float* __restrict__ fold, int64_t HW, int nblk) {
  const int b = blockIdx.x;
  const int j = threadIdx.x;
  __shared__ double S[9];
  if (j < 9) {  // one thread per statistic, fixed block order
    double s = 0.0;
    for (int k = 0; k < nblk; ++k) s += part[((int64_t)b * nblk + k) * 9 + j];
    S[j] = s;
  }
  __syncthreads();
  if (j >= HID) return;
  const double N = (double)HW;
  const double m[3] = {S[0] / N, S[1] / N, S[2] / N};
  const int ix[3][3] = {{3, 4, 5}, {4, 6, 7}, {5, 7, 8}};
  double w[3];
  for (int i = 0; i < 3; ++i) w[i] = (double)params[P<HID>::w1 + j * CI + i];
  double mu = 0.0, var = 0.0;
  for (int i = 0; i < 3; ++i) mu += w[i] * m[i];
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 3; ++k) var += w[i] * w[k] * (S[ix[i][k]] / N - m[i] * m[k]);
  if (var < 0.0) var = 0.0;
  const double inv = 1.0 / sqrt(var + kVarFloor);
  const double gain = (double)params[P<HID>::gain], ng = (double)params[P<HID>::ng];
  const double alpha = gain + ng * inv, beta = -ng * inv * mu;
  float* f = fold + (int64_t)b * F<HID>::count;
  for (int i = 0; i < 3; ++i) {
    f[F<HID>::w1f + j * CI + i] = (float)(alpha * w[i]);
    f[F<HID>::w1 + j * CI + i] = (float)w[i];
  }
  f[F<HID>::beta + j] = (float)beta;
  f[F<HID>::alpha + j] = (float)alpha;
  f[F<HID>::mu + j] = (float)mu;
  f[F<HID>::inv + j] = (float)inv;
}

// ---- forward: y = W2 lrelu(W1f x + beta) + b2 ------------------------------
template <int HID>
__global__ void __launch_bounds__(NT) k_fwd(const float* __restrict__ x, float* __restrict__ y,
                                             const float* __restrict__ params,
                                             const float* __restrict__ fold, int64_t HW) {
  __shared__ float sw1[HID * CI], sbeta[HID], sw2[CO * HID], sb2[CO];
  const int64_t b = blockIdx.y;
  const float* f = fold + b * F<HID>::count;
  for (int i = threadIdx.x; i < HID * CI; i += NT) sw1[i] = f[F<HID>::w1f + i];
  for (int i = threadIdx.x; i < HID; i += NT) sbeta[i] = f[F<HID>::beta + i];
  for (int i = threadIdx.x; i < CO * HID; i += NT) sw2[i] = params[P<HID>::w2 + i];
  for (int i = threadIdx.x; i < CO; i += NT) sb2[i] = params[P<HID>::b2 + i];
  __syncthreads();
  const int64_t n4 = HW / 4;
  using namespace pr;
  for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < n4; i += (int64_t)gridDim.x * NT) {
    ulonglong2 X[CI];  // pixel pairs (0,1), (2,3) of each channel
#pragma unroll
    for (int c = 0; c < CI; ++c)
      X[c] = __ldg(reinterpret_cast<const ulonglong2*>(x + (b * CI + c) * HW) + i);
    u64 out[CO][2];
#pragma unroll
    for (int o = 0; o < CO; ++o) out[o][0] = out[o][1] = bc(sb2[o]);
#pragma unroll
    for (int j = 0; j < HID; ++j) {
      const u64 w0 = bc(sw1[j * CI]), w1 = bc(sw1[j * CI + 1]), w2 = bc(sw1[j * CI + 2]);
      const u64 be = bc(sbeta[j]);
      const u64 v0 = bc(sw2[0 * HID + j]), v1 = bc(sw2[1 * HID + j]), v2 = bc(sw2[2 * HID + j]);
#pragma unroll
      for (int pp = 0; pp < 2; ++pp) {
        const u64 x0 = pp ? X[0].y : X[0].x, x1 = pp ? X[1].y : X[1].x,
                  x2 = pp ? X[2].y : X[2].x;
        u64 h = fma2(w2, x2, fma2(w1, x1, fma2(w0, x0, be)));
        h = mul2(h, slope2(h, kLeaky));  // leaky ReLU 0.2 (gf/guidance.py:36-39)
        out[0][pp] = fma2(v0, h, out[0][pp]);
        out[1][pp] = fma2(v1, h, out[1][pp]);
        out[2][pp] = fma2(v2, h, out[2][pp]);
      }
    }
#pragma unroll
    for (int o = 0; o < CO; ++o)
      reinterpret_cast<ulonglong2*>(y + (b * CO + o) * HW)[i] = make_ulonglong2(out[o][0], out[o][1]);
  }
}

// ---- backward pass A: per-image sums --------------------------------------
// acc layout: [0,HID) sum d2; [HID,2HID) sum d2*h1; [2HID,2HID+CO) sum dy;
//             [2HID+CO, 2HID+CO+CO*HID) sum dy_o*h3_j
template <int HID>
struct A {
  static constexpr int d2 = 0, d2h1 = HID, dy = 2 * HID, dw2 = 2 * HID + CO,
                       nv = 2 * HID + CO + CO * HID;
};

// block reduce of NV float64 values given per thread by get(v) -> out[0..NV)
template <int NV, class Get>
__device__ void reduce_store_fn(Get get, double* out) {
  __shared__ double red[NT / 32][NV];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    double a = (double)get(v);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) red[warp][v] = a;
  }
  __syncthreads();
  for (int v = threadIdx.x; v < NV; v += NT) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) s += red[w][v];
    out[v] = s;
  }
  __syncthreads();
}

// Two threads (adjacent lanes) per 4-pixel group, each owning half of the
// hidden units: half the per-thread accumulators, so two CTAs fit an SM.
template <int HID>
__global__ void __launch_bounds__(NT, 2) k_bwd_a(const float* __restrict__ x,
                                              const float* __restrict__ dy,
                                              const float* __restrict__ params,
                                              const float* __restrict__ fold,
                                              double* __restrict__ part, int64_t HW) {
  __shared__ float sw1[HID * CI], salpha[HID], sbeta[HID], sw2[CO * HID];
  __shared__ ulonglong2 stage[NST][CI + CO][NT / 2];
  const int64_t b = blockIdx.y;
  const float* f = fold + b * F<HID>::count;
  for (int i = threadIdx.x; i < HID * CI; i += NT) sw1[i] = f[F<HID>::w1 + i];
  for (int i = threadIdx.x; i < HID; i += NT) {
    sbeta[i] = f[F<HID>::beta + i];
    salpha[i] = f[F<HID>::alpha + i];
  }
  for (int i = threadIdx.x; i < CO * HID; i += NT) sw2[i] = params[P<HID>::w2 + i];
  __syncthreads();
  constexpr int JH = (HID + 1) / 2;  // hidden units per thread
  using namespace pr;
  const int half = threadIdx.x & 1;
  const int j0 = half * JH;
  // fp32 per-thread sums on pixel pairs (a few hundred pixels each), float64
  // across threads
  u64 sd2[JH], sd2h1[JH], sdw2[CO][JH], sdy[CO];
#pragma unroll
  for (int jj = 0; jj < JH; ++jj) {
    sd2[jj] = sd2h1[jj] = 0ull;
#pragma unroll
    for (int o = 0; o < CO; ++o) sdw2[o][jj] = 0ull;
  }
#pragma unroll
  for (int o = 0; o < CO; ++o) sdy[o] = 0ull;
  const int64_t n4 = HW / 4;
  const int64_t stride = (int64_t)gridDim.x * (NT / 2);
  const int64_t first = (int64_t)blockIdx.x * (NT / 2);
  const int pr_ = threadIdx.x >> 1;
  // warp-uniform trip count: the stage hand-off below needs every lane
  const int64_t iters = n4 > first ? (n4 - first + stride - 1) / stride : 0;
  // stage iteration `it` of this pair's (x, dy) chunks (NST - 1 ahead)
  auto issue = [&](int64_t it) {
    const int64_t i = first + it * stride + pr_;
    if (it < iters && i < n4) {
      const int st = (int)(it % NST);
      const float* base = half ? dy + b * CO * HW : x + b * CI * HW;
#pragma unroll
      for (int c = 0; c < 3; ++c)
        cp16(&stage[st][3 * half + c][pr_], reinterpret_cast<const ulonglong2*>(base + c * HW) + i);
    }
    cp_commit();
  };
#pragma unroll
  for (int k = 0; k < NST - 1; ++k) issue(k);
  for (int64_t it = 0; it < iters; ++it) {
    const bool valid = first + it * stride + pr_ < n4;  // a lane pair together
    __syncwarp();  // the partner's reads of the stage refilled below are done
    issue(it + NST - 1);
    cp_wait<NST - 1>();
    __syncwarp();  // the partner's chunks of stage `it` are visible
    const int st = (int)(it % NST);
    ulonglong2 X[CI], G[CO];
#pragma unroll
    for (int c = 0; c < CI; ++c) X[c] = valid ? stage[st][c][pr_] : make_ulonglong2(0ull, 0ull);
#pragma unroll
    for (int o = 0; o < CO; ++o) {
      G[o] = valid ? stage[st][CI + o][pr_] : make_ulonglong2(0ull, 0ull);
      sdy[o] = add2(sdy[o], add2(G[o].x, G[o].y));
    }
#pragma unroll
    for (int jj = 0; jj < JH; ++jj) {
      const int j = j0 + jj;
      if (j >= HID) break;  // odd HID: the second half has one unit fewer
      const u64 a0 = bc(sw1[j * CI]), a1 = bc(sw1[j * CI + 1]), a2 = bc(sw1[j * CI + 2]);
      const u64 al = bc(salpha[j]), be = bc(sbeta[j]);
      const u64 v0 = bc(sw2[0 * HID + j]), v1 = bc(sw2[1 * HID + j]), v2 = bc(sw2[2 * HID + j]);
#pragma unroll
      for (int pp = 0; pp < 2; ++pp) {
        const u64 x0 = pp ? X[0].y : X[0].x, x1 = pp ? X[1].y : X[1].x,
                  x2 = pp ? X[2].y : X[2].x;
        const u64 g0 = pp ? G[0].y : G[0].x, g1 = pp ? G[1].y : G[1].x,
                  g2 = pp ? G[2].y : G[2].x;
        const u64 h1 = fma2(a2, x2, fma2(a1, x1, mul2(a0, x0)));
        const u64 h2 = fma2(al, h1, be);  // (alpha .* W1) x + beta
        const u64 sl = slope2(h2, kLeaky);
        const u64 h3 = mul2(h2, sl);
        const u64 d2 = mul2(fma2(v2, g2, fma2(v1, g1, mul2(v0, g0))), sl);
        sd2[jj] = add2(sd2[jj], d2);
        sd2h1[jj] = fma2(d2, h1, sd2h1[jj]);
        sdw2[0][jj] = fma2(g0, h3, sdw2[0][jj]);
        sdw2[1][jj] = fma2(g1, h3, sdw2[1][jj]);
        sdw2[2][jj] = fma2(g2, h3, sdw2[2][jj]);
      }
    }
  }
  cp_wait<0>();
  // value v of the A layout from the thread that owns it (0 elsewhere)
  auto sum2 = [](u64 p) { return lo(p) + hi(p); };
  auto get = [&](int v) -> float {
    if (v >= A<HID>::dw2) {
      const int u = v - A<HID>::dw2, o = u / HID, j = u - o * HID;
      float r = 0.f;
#pragma unroll
      for (int jj = 0; jj < JH; ++jj)
        if (j == j0 + jj) r = sum2(sdw2[o][jj]);
      return r;
    }
    if (v >= A<HID>::dy) return half == 0 ? sum2(sdy[v - A<HID>::dy]) : 0.f;
    const bool h1f = v >= A<HID>::d2h1;
    const int j = h1f ? v - A<HID>::d2h1 : v;
    float r = 0.f;
#pragma unroll
    for (int jj = 0; jj < JH; ++jj)
      if (j == j0 + jj) r = sum2(h1f ? sd2h1[jj] : sd2[jj]);
    return r;
  };
  reduce_store_fn<A<HID>::nv>(get, part + (b * gridDim.x + blockIdx.x) * A<HID>::nv);
}

// ---- finalize A: per-image constants of dh1 and the W2/b2/gain/ng grads ----
// coef (fp32, per image): kappa[HID], lambda[HID]  (alpha comes from fold)
// gsum (float64, per image): dW2 (CO*HID), db2 (CO), dgain, dng
template <int HID>
__global__ void k_fin_a(const double* __restrict__ part, const float* __restrict__ params,
                        const float* __restrict__ fold, float* __restrict__ coef,
                        double* __restrict__ gsum, int64_t HW, int nblk) {
  constexpr int NV = A<HID>::nv;
  const int b = blockIdx.x;
  __shared__ double S[NV];
  for (int v = threadIdx.x; v < NV; v += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < nblk; ++k) s += part[((int64_t)b * nblk + k) * NV + v];
    S[v] = s;
  }
  __syncthreads();
  const float* f = fold + (int64_t)b * F<HID>::count;
  const double N = (double)HW;
  const double ng = (double)params[P<HID>::ng];
  double* gs = gsum + (int64_t)b * (CO * HID + CO + 2);
  for (int v = threadIdx.x; v < CO * HID + CO; v += blockDim.x)
    gs[v] = v < CO * HID ? S[A<HID>::dw2 + v] : S[A<HID>::dy + v - CO * HID];
  if (threadIdx.x < HID) {
    const int j = threadIdx.x;
    const double mu = (double)f[F<HID>::mu + j], inv = (double)f[F<HID>::inv + j];
    const double sd2 = S[A<HID>::d2 + j], sd2h1 = S[A<HID>::d2h1 + j];
    const double sd2xhat = inv * (sd2h1 - mu * sd2);  // sum d2 * xhat
    const double gm = ng * sd2 / N;                   // mean(g), g = ng * d2
    const double gp = ng * sd2xhat / N;               // mean(g * xhat)
    // dh1 = alpha d2 + (-gm - xhat gp) inv = alpha d2 + kappa + lambda h1
    coef[(int64_t)b * 2 * HID + j] = (float)(-gm * inv + gp * inv * inv * mu);
    coef[(int64_t)b * 2 * HID + HID + j] = (float)(-gp * inv * inv);
  }
  if (threadIdx.x == 0) {
    double dg = 0.0, dn = 0.0;
    for (int j = 0; j < HID; ++j) {
      const double mu = (double)f[F<HID>::mu + j], inv = (double)f[F<HID>::inv + j];
      dg += S[A<HID>::d2h1 + j];
      dn += inv * (S[A<HID>::d2h1 + j] - mu * S[A<HID>::d2 + j]);
    }
    gs[CO * HID + CO] = dg;
    gs[CO * HID + CO + 1] = dn;
  }
}

// ---- backward pass B: dx and dW1 partials ----------------------------------
// Two threads (adjacent lanes) per 4-pixel group, each owning half of the
// hidden units; their dx contributions are summed with one shuffle.
template <int HID>
__global__ void __launch_bounds__(NT, 2) k_bwd_b(const float* __restrict__ x,
                                              const float* __restrict__ dy,
                                              float* __restrict__ dx,
                                              const float* __restrict__ params,
                                              const float* __restrict__ fold,
                                              const float* __restrict__ coef,
                                              double* __restrict__ part, int64_t HW) {
  __shared__ float sw1[HID * CI], sbeta[HID], sw2[CO * HID], salpha[HID], skap[HID], slam[HID];
  __shared__ ulonglong2 stage[NST][CI + CO][NT / 2];
  const int64_t b = blockIdx.y;
  const float* f = fold + b * F<HID>::count;
  for (int i = threadIdx.x; i < HID * CI; i += NT) sw1[i] = f[F<HID>::w1 + i];
  for (int i = threadIdx.x; i < HID; i += NT) {
    sbeta[i] = f[F<HID>::beta + i];
    salpha[i] = f[F<HID>::alpha + i];
    skap[i] = coef[b * 2 * HID + i];
    slam[i] = coef[b * 2 * HID + HID + i];
  }
  for (int i = threadIdx.x; i < CO * HID; i += NT) sw2[i] = params[P<HID>::w2 + i];
  __syncthreads();
  constexpr int JH = (HID + 1) / 2;
  using namespace pr;
  const int half = threadIdx.x & 1;
  const int j0 = half * JH;
  u64 fa[JH][CI];  // dW1 partials on pixel pairs
#pragma unroll
  for (int jj = 0; jj < JH; ++jj)
#pragma unroll
    for (int c = 0; c < CI; ++c) fa[jj][c] = 0ull;
  const int64_t n4 = HW / 4;
  const int64_t stride = (int64_t)gridDim.x * (NT / 2);
  const int64_t first = (int64_t)blockIdx.x * (NT / 2);
  // warp-uniform trip count: the dx shuffle below needs every lane
  const int64_t iters = n4 > first ? (n4 - first + stride - 1) / stride : 0;
  const int pr_ = threadIdx.x >> 1;
  // stage iteration `it` of this pair's (x, dy) chunks (NST - 1 ahead)
  auto issue = [&](int64_t it) {
    const int64_t i = first + it * stride + pr_;
    if (it < iters && i < n4) {
      const int st = (int)(it % NST);
      const float* base = half ? dy + b * CO * HW : x + b * CI * HW;
#pragma unroll
      for (int c = 0; c < 3; ++c)
        cp16(&stage[st][3 * half + c][pr_], reinterpret_cast<const ulonglong2*>(base + c * HW) + i);
    }
    cp_commit();
  };
#pragma unroll
  for (int k = 0; k < NST - 1; ++k) issue(k);
  for (int64_t it = 0; it < iters; ++it) {
    const int64_t i = first + it * stride + pr_;
    const bool valid = i < n4;  // a lane pair is valid or invalid together
    __syncwarp();  // the partner's reads of the stage refilled below are done
    issue(it + NST - 1);
    cp_wait<NST - 1>();
    __syncwarp();  // the partner's chunks of stage `it` are visible
    const int st = (int)(it % NST);
    ulonglong2 X[CI], G[CO];
    u64 dxv[CI][2];
#pragma unroll
    for (int c = 0; c < CI; ++c) {
      X[c] = valid ? stage[st][c][pr_] : make_ulonglong2(0ull, 0ull);
      dxv[c][0] = dxv[c][1] = 0ull;
    }
#pragma unroll
    for (int o = 0; o < CO; ++o)
      G[o] = valid ? stage[st][CI + o][pr_] : make_ulonglong2(0ull, 0ull);
#pragma unroll
    for (int jj = 0; jj < JH; ++jj) {
      const int j = j0 + jj;
      if (j >= HID) break;
      const u64 a0 = bc(sw1[j * CI]), a1 = bc(sw1[j * CI + 1]), a2 = bc(sw1[j * CI + 2]);
      const u64 be = bc(sbeta[j]), al = bc(salpha[j]), ka = bc(skap[j]), la = bc(slam[j]);
      const u64 v0 = bc(sw2[0 * HID + j]), v1 = bc(sw2[1 * HID + j]), v2 = bc(sw2[2 * HID + j]);
#pragma unroll
      for (int pp = 0; pp < 2; ++pp) {
        const u64 x0 = pp ? X[0].y : X[0].x, x1 = pp ? X[1].y : X[1].x,
                  x2 = pp ? X[2].y : X[2].x;
        const u64 g0 = pp ? G[0].y : G[0].x, g1 = pp ? G[1].y : G[1].x,
                  g2 = pp ? G[2].y : G[2].x;
        const u64 h1 = fma2(a2, x2, fma2(a1, x1, mul2(a0, x0)));
        const u64 h2 = fma2(al, h1, be);  // (alpha .* W1) x + beta
        const u64 d2 = mul2(fma2(v2, g2, fma2(v1, g1, mul2(v0, g0))), slope2(h2, kLeaky));
        const u64 dh = fma2(al, d2, fma2(la, h1, ka));
        dxv[0][pp] = fma2(a0, dh, dxv[0][pp]);
        dxv[1][pp] = fma2(a1, dh, dxv[1][pp]);
        dxv[2][pp] = fma2(a2, dh, dxv[2][pp]);
        fa[jj][0] = fma2(dh, x0, fa[jj][0]);
        fa[jj][1] = fma2(dh, x1, fa[jj][1]);
        fa[jj][2] = fma2(dh, x2, fa[jj][2]);
      }
    }
#pragma unroll
    for (int c = 0; c < CI; ++c)
#pragma unroll
      for (int pp = 0; pp < 2; ++pp)
        dxv[c][pp] = add2(dxv[c][pp], __shfl_xor_sync(0xffffffffu, dxv[c][pp], 1));
    if (valid && half == 0) {
#pragma unroll
      for (int c = 0; c < CI; ++c)
        reinterpret_cast<ulonglong2*>(dx + (b * CI + c) * HW)[i] =
            make_ulonglong2(dxv[c][0], dxv[c][1]);
    }
  }
  cp_wait<0>();
  auto get = [&](int v) -> float {
    const int j = v / CI, c = v - j * CI;
    float r = 0.f;
#pragma unroll
    for (int jj = 0; jj < JH; ++jj)
#pragma unroll
      for (int cc = 0; cc < CI; ++cc)
        if (j == j0 + jj && c == cc) r = pr::lo(fa[jj][cc]) + pr::hi(fa[jj][cc]);
    return r;
  };
  reduce_store_fn<HID * CI>(get, part + (b * gridDim.x + blockIdx.x) * (HID * CI));
}

// ---- per-image dW1 sums of the pass-B partials (fixed block order) --------
template <int HID>
__global__ void k_fin_b(const double* __restrict__ partb, double* __restrict__ pbi, int nblk) {
  const int64_t b = blockIdx.x;
  const int v = threadIdx.x;
  if (v >= HID * CI) return;
  double s = 0.0;
  for (int k = 0; k < nblk; ++k) s += partb[(b * nblk + k) * (HID * CI) + v];
  pbi[b * (HID * CI) + v] = s;
}

// ---- final parameter gradients (one block; fixed order over images) -------
template <int HID>
__global__ void k_fin_params(const double* __restrict__ gsum, const double* __restrict__ partb,
                             float* __restrict__ dparams, int accumulate, int64_t B, int nblk) {
  constexpr int GS = CO * HID + CO + 2;
  for (int idx = threadIdx.x; idx < P<HID>::count; idx += blockDim.x) {
    double s = 0.0;
    if (idx < HID * CI) {
      for (int64_t b = 0; b < B; ++b) s += partb[b * (HID * CI) + idx];  // per-image sums
    } else if (idx == P<HID>::gain) {
      for (int64_t b = 0; b < B; ++b) s += gsum[b * GS + CO * HID + CO];
    } else if (idx == P<HID>::ng) {
      for (int64_t b = 0; b < B; ++b) s += gsum[b * GS + CO * HID + CO + 1];
    } else if (idx < P<HID>::b2) {
      for (int64_t b = 0; b < B; ++b) s += gsum[b * GS + (idx - P<HID>::w2)];
    } else {
      for (int64_t b = 0; b < B; ++b) s += gsum[b * GS + CO * HID + (idx - P<HID>::b2)];
    }
    dparams[idx] = accumulate ? (float)((double)dparams[idx] + s) : (float)s;
  }
}

// ---- workspace -------------------------------------------------------------
template <int HID>
struct WS {
  static size_t bytes(int64_t B) {
    const size_t stats = (size_t)B * kBlocks * 9 * sizeof(double);
    const size_t fold = (size_t)B * F<HID>::count * sizeof(float);
    const size_t pa = (size_t)B * kBlocks * A<HID>::nv * sizeof(double);
    const size_t coef = (size_t)B * 2 * HID * sizeof(float);
    const size_t gsum = (size_t)B * (CO * HID + CO + 2) * sizeof(double);
    const size_t pb = (size_t)B * kBlocks * HID * CI * sizeof(double);
    return stats + fold + pa + coef + gsum + pb + 6 * 256;
  }
};

struct Carve {
  char* p;
  template <typename T>
  T* take(size_t n) {
    T* out = reinterpret_cast<T*>(p);
    p += (n * sizeof(T) + 255) / 256 * 256;
    return out;
  }
};

template <int HID>
void forward(const float* x, float* y, const float* params, int64_t B, int64_t HW, void* ws,
             uint32_t* status, cudaStream_t s) {
  Carve c{(char*)ws};
  double* stats = c.take<double>((size_t)B * kBlocks * 9);
  float* fold = c.take<float>((size_t)B * F<HID>::count);
  dim3 grid(kBlocks, (unsigned)B);
  k_stats<<<grid, NT, 0, s>>>(x, stats, HW, status);
  k_prep<HID><<<(unsigned)B, 32, 0, s>>>(stats, params, fold, HW, kBlocks);
  k_fwd<HID><<<grid, NT, 0, s>>>(x, y, params, fold, HW);
}

template <int HID>
void backward(const float* x, const float* dy, float* dx, float* dparams, int accumulate,
              const float* params, int64_t B, int64_t HW, void* ws, bool have_fold,
              uint32_t* status, cudaStream_t s) {
  Carve c{(char*)ws};
  double* stats = c.take<double>((size_t)B * kBlocks * 9);
  float* fold = c.take<float>((size_t)B * F<HID>::count);
  double* pa = c.take<double>((size_t)B * kBlocks * A<HID>::nv);
  float* coef = c.take<float>((size_t)B * 2 * HID);
  double* gsum = c.take<double>((size_t)B * (CO * HID + CO + 2));
  double* pb = c.take<double>((size_t)B * kBlocks * HID * CI);
  dim3 grid(kBlocks, (unsigned)B);
  if (!have_fold) {  // else `ws` holds forward()'s folded constants of this x and params
    k_stats<<<grid, NT, 0, s>>>(x, stats, HW, status);
    k_prep<HID><<<(unsigned)B, 32, 0, s>>>(stats, params, fold, HW, kBlocks);
  }
  k_bwd_a<HID><<<grid, NT, 0, s>>>(x, dy, params, fold, pa, HW);
  k_fin_a<HID><<<(unsigned)B, 128, 0, s>>>(pa, params, fold, coef, gsum, HW, kBlocks);
  k_bwd_b<HID><<<grid, NT, 0, s>>>(x, dy, dx, params, fold, coef, pb, HW);
  // per-image dW1 sums land in `stats` (free after prep), then the batch sum
  k_fin_b<HID><<<(unsigned)B, 64, 0, s>>>(pb, stats, kBlocks);
  k_fin_params<HID><<<1, 128, 0, s>>>(gsum, stats, dparams, accumulate, B, kBlocks);
}

}  // namespace gnf

// hidden widths with a fused fp32 path
bool gn_fast_ok(int64_t Cin, int64_t Cout, int64_t hidden, int64_t HW) {
  return Cin == 3 && Cout == 3 && HW % 4 == 0 &&
         (hidden == 4 || hidden == 8 || hidden == 15 || hidden == 16);
}

size_t gn_fast_ws_bytes(int64_t B, int64_t hidden) {
  switch (hidden) {
    case 4: return gnf::WS<4>::bytes(B);
    case 8: return gnf::WS<8>::bytes(B);
    case 15: return gnf::WS<15>::bytes(B);
    case 16: return gnf::WS<16>::bytes(B);
    default: return 0;
  }
}

void gn_fast_forward(const float* x, float* y, const float* params, int64_t B, int64_t hidden,
                     int64_t HW, void* ws, uint32_t* status, cudaStream_t s) {
  switch (hidden) {
    case 4: gnf::forward<4>(x, y, params, B, HW, ws, status, s); break;
    case 8: gnf::forward<8>(x, y, params, B, HW, ws, status, s); break;
    case 15: gnf::forward<15>(x, y, params, B, HW, ws, status, s); break;
    case 16: gnf::forward<16>(x, y, params, B, HW, ws, status, s); break;
  }
}

void gn_fast_backward(const float* x, const float* dy, float* dx, float* dparams, int accumulate,
                      const float* params, int64_t B, int64_t hidden, int64_t HW, void* ws,
                      bool have_fold, uint32_t* status, cudaStream_t s) {
  switch (hidden) {
    case 4: gnf::backward<4>(x, dy, dx, dparams, accumulate, params, B, HW, ws, have_fold, status, s); break;
    case 8: gnf::backward<8>(x, dy, dx, dparams, accumulate, params, B, HW, ws, have_fold, status, s); break;
    case 15:
      gnf::backward<15>(x, dy, dx, dparams, accumulate, params, B, HW, ws, have_fold, status, s);
      break;
    case 16:
      gnf::backward<16>(x, dy, dx, dparams, accumulate, params, B, HW, ws, have_fold, status, s);
      break;
  }
}

}  // namespace gfb
