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

#include <algorithm>

#include "gf_common.cuh"
#include "gf_internal.h"
#include "gf_pair.cuh"

namespace gfb {

thread_local int g_gn_bwd_variant = 0;

namespace gnf {

constexpr int CI = 3, CO = 3;
constexpr int NT = 256;
constexpr int kBlocks = 128;  // pixel blocks per image (grid.x)
// the one-pass backward's blocks per image: one wave of the SM's CTA slots
// spread over the batch (<= kBlocksH)
constexpr int kBlocksH = 512;
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
__global__ void __launch_bounds__(NT, 3) k_fwd(const float* __restrict__ x, float* __restrict__ y,
                                             const float* __restrict__ params,
                                             const float* __restrict__ fold, int64_t HW) {
  // per hidden unit: (W1f row, beta) and (W2 column, 0) as one 16-byte word
  // each, read by a broadcast LDS.128
  __shared__ float4 sW[HID], sV[HID];
  const int64_t b = blockIdx.y;
  const float* f = fold + b * F<HID>::count;
  for (int j = threadIdx.x; j < HID; j += NT) {
    sW[j] = make_float4(f[F<HID>::w1f + j * CI], f[F<HID>::w1f + j * CI + 1],
                        f[F<HID>::w1f + j * CI + 2], f[F<HID>::beta + j]);
    sV[j] = make_float4(params[P<HID>::w2 + j], params[P<HID>::w2 + HID + j],
                        params[P<HID>::w2 + 2 * HID + j], 0.f);
  }
  __syncthreads();
  const int64_t n4 = HW / 4;
  using namespace pr;
  const u64 B0 = bc(params[P<HID>::b2]), B1 = bc(params[P<HID>::b2 + 1]),
            B2 = bc(params[P<HID>::b2 + 2]);
  // two 4-pixel groups per iteration (i and i + stride): the seven weight
  // broadcasts of a hidden unit serve four pixel pairs.  leaky ReLU as
  // max(h, 0.2 h) (slope < 1: the same values as h * slope(h)).
  const int64_t stride = (int64_t)gridDim.x * NT;
  const u64 LK = bc(kLeaky);
  for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < n4; i += 2 * stride) {
    const bool two = i + stride < n4;
    const int64_t i1 = two ? i + stride : i;
    ulonglong2 X[2][CI];  // pixel pairs (0,1), (2,3) of each channel, both groups
#pragma unroll
    for (int c = 0; c < CI; ++c) {
      X[0][c] = __ldg(reinterpret_cast<const ulonglong2*>(x + (b * CI + c) * HW) + i);
      X[1][c] = __ldg(reinterpret_cast<const ulonglong2*>(x + (b * CI + c) * HW) + i1);
    }
    u64 out[CO][4];
#pragma unroll
    for (int pp = 0; pp < 4; ++pp) {
      out[0][pp] = B0;
      out[1][pp] = B1;
      out[2][pp] = B2;
    }
#pragma unroll
    for (int j = 0; j < HID; ++j) {
      const float4 wv = sW[j], vv = sV[j];
      const u64 w0 = bc(wv.x), w1 = bc(wv.y), w2 = bc(wv.z), be = bc(wv.w);
      const u64 v0 = bc(vv.x), v1 = bc(vv.y), v2 = bc(vv.z);
#pragma unroll
      for (int pp = 0; pp < 4; ++pp) {
        const int g = pp >> 1;
        const u64 x0 = (pp & 1) ? X[g][0].y : X[g][0].x, x1 = (pp & 1) ? X[g][1].y : X[g][1].x,
                  x2 = (pp & 1) ? X[g][2].y : X[g][2].x;
        u64 h = fma2(w2, x2, fma2(w1, x1, fma2(w0, x0, be)));
        const u64 hl = mul2(h, LK);
        h = pk(fmaxf(lo(h), lo(hl)), fmaxf(hi(h), hi(hl)));  // leaky ReLU 0.2 (gf/guidance.py:36-39)
        out[0][pp] = fma2(v0, h, out[0][pp]);
        out[1][pp] = fma2(v1, h, out[1][pp]);
        out[2][pp] = fma2(v2, h, out[2][pp]);
      }
    }
#pragma unroll
    for (int o = 0; o < CO; ++o) {
      reinterpret_cast<ulonglong2*>(y + (b * CO + o) * HW)[i] = make_ulonglong2(out[o][0], out[o][1]);
      if (two)
        reinterpret_cast<ulonglong2*>(y + (b * CO + o) * HW)[i1] =
            make_ulonglong2(out[o][2], out[o][3]);
    }
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

// ---- backward, one heavy pass (default) ------------------------------------
// The AdaptiveNorm coupling makes dh1_j = alpha_j d2_j + kappa_j + lambda_j h1_j
// (kappa, lambda per image, known only after a pass over every pixel), so
//     dx_c   = D_c(p) + K_c + sum_c' L_cc' x_c'
//              D_c = sum_j (alpha_j W1_jc) d2_j,  K_c = sum_j W1_jc kappa_j,
//              L_cc' = sum_j W1_jc lambda_j W1_jc'
//     dW1_jc = alpha_j sum_p d2_j x_c + kappa_j sum_p x_c
//              + lambda_j sum_c' W1_jc' sum_p x_c' x_c
// and sum_p d2_j h1_j = sum_c W1_jc sum_p d2_j x_c.  One heavy pass (k_bwd_h)
// streams (x, dy), writes D into dx and reduces sum d2, sum d2 x, sum dy,
// sum dy h3; the x moments come from the forward's statistics; k_fin_h forms
// kappa, lambda, K, L and every parameter gradient; k_dx adds K + L x to D.
// Four lanes share a 4-pixel group, each owning a quarter of the hidden units
// (the accumulators fit 2 CTAs per SM); D is summed over the four by shuffles.
template <int HID>
struct AH {
  static constexpr int d2 = 0, d2x = HID, dy = HID + HID * CI, dw2 = HID + HID * CI + CO,
                       nv = HID + HID * CI + CO + CO * HID;
};
// per-image fp32 constants of k_dx: K[3], L[3][3]
constexpr int KL = CI + CI * CI;
// per-image float64 gradient sums: dW2 (CO*HID), db2 (CO), dgain, dng, dW1 (HID*CI)
template <int HID>
struct GH {
  static constexpr int dw2 = 0, db2 = CO * HID, dgain = CO * HID + CO, dng = CO * HID + CO + 1,
                       dw1 = CO * HID + CO + 2, count = CO * HID + CO + 2 + HID * CI;
};

template <int HID>
__global__ void __launch_bounds__(NT, 2) k_bwd_h(const float* __restrict__ x,
                                              const float* __restrict__ dy,
                                              float* __restrict__ D,
                                              const float* __restrict__ params,
                                              const float* __restrict__ fold,
                                              double* __restrict__ part, int64_t HW) {
  constexpr int NG = NT / 4;  // 4-pixel groups per CTA iteration
  constexpr int JH = (HID + 3) / 4;  // hidden units per lane
  // unit j = q JH + jj of lane q at [jj][q]: (W1f row, beta), (W2 column, 0),
  // so the four lanes of a group read four consecutive 16-byte words
  __shared__ float4 sW[JH * 4], sV[JH * 4];
  __shared__ ulonglong2 stage[NST][CI + CO][NG];
  const int64_t b = blockIdx.y;
  const float* f = fold + b * F<HID>::count;
  for (int i = threadIdx.x; i < JH * 4; i += NT) {
    const int j = (i & 3) * JH + (i >> 2);
    sW[i] = j < HID ? make_float4(f[F<HID>::w1f + j * CI], f[F<HID>::w1f + j * CI + 1],
                                  f[F<HID>::w1f + j * CI + 2], f[F<HID>::beta + j])
                    : make_float4(0.f, 0.f, 0.f, 0.f);
    sV[i] = j < HID ? make_float4(params[P<HID>::w2 + j], params[P<HID>::w2 + HID + j],
                                  params[P<HID>::w2 + 2 * HID + j], 0.f)
                    : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __syncthreads();
  using namespace pr;
  const int q = threadIdx.x & 3;
  const int j0 = q * JH;
  const int g = threadIdx.x >> 2;
  u64 sd2[JH], sd2x[JH][CI], sdw2[CO][JH], sdy[CO];
#pragma unroll
  for (int jj = 0; jj < JH; ++jj) {
    sd2[jj] = 0ull;
#pragma unroll
    for (int c = 0; c < CI; ++c) sd2x[jj][c] = 0ull;
#pragma unroll
    for (int o = 0; o < CO; ++o) sdw2[o][jj] = 0ull;
  }
#pragma unroll
  for (int o = 0; o < CO; ++o) sdy[o] = 0ull;
  const int64_t n4 = HW / 4;
  const int64_t stride = (int64_t)gridDim.x * NG;
  const int64_t first = (int64_t)blockIdx.x * NG;
  const int64_t iters = n4 > first ? (n4 - first + stride - 1) / stride : 0;
  // lanes 0..2 of a group copy (x_q, dy_q); lane 3 copies nothing
  auto issue = [&](int64_t it) {
    const int64_t i = first + it * stride + g;
    if (it < iters && i < n4 && q < 3) {
      const int st = (int)(it % NST);
      cp16(&stage[st][q][g], reinterpret_cast<const ulonglong2*>(x + (b * CI + q) * HW) + i);
      cp16(&stage[st][CI + q][g], reinterpret_cast<const ulonglong2*>(dy + (b * CO + q) * HW) + i);
    }
    cp_commit();
  };
#pragma unroll
  for (int k = 0; k < NST - 1; ++k) issue(k);
  for (int64_t it = 0; it < iters; ++it) {
    const int64_t i = first + it * stride + g;
    const bool valid = i < n4;  // a group is valid or invalid together
    __syncwarp();  // the group's reads of the stage refilled below are done
    issue(it + NST - 1);
    cp_wait<NST - 1>();
    __syncwarp();  // the group's chunks of stage `it` are visible
    const int st = (int)(it % NST);
    ulonglong2 X[CI], G[CO];
#pragma unroll
    for (int c = 0; c < CI; ++c) X[c] = valid ? stage[st][c][g] : make_ulonglong2(0ull, 0ull);
#pragma unroll
    for (int o = 0; o < CO; ++o) {
      G[o] = valid ? stage[st][CI + o][g] : make_ulonglong2(0ull, 0ull);
      sdy[o] = add2(sdy[o], add2(G[o].x, G[o].y));
    }
    u64 dv[CI][2];
#pragma unroll
    for (int c = 0; c < CI; ++c) dv[c][0] = dv[c][1] = 0ull;
#pragma unroll
    for (int jj = 0; jj < JH; ++jj) {
      const int j = j0 + jj;
      if (j >= HID) break;
      const float4 wv = sW[jj * 4 + q], vv = sV[jj * 4 + q];
      const u64 a0 = bc(wv.x), a1 = bc(wv.y), a2 = bc(wv.z), be = bc(wv.w);
      const u64 v0 = bc(vv.x), v1 = bc(vv.y), v2 = bc(vv.z);
#pragma unroll
      for (int pp = 0; pp < 2; ++pp) {
        const u64 x0 = pp ? X[0].y : X[0].x, x1 = pp ? X[1].y : X[1].x,
                  x2 = pp ? X[2].y : X[2].x;
        const u64 g0 = pp ? G[0].y : G[0].x, g1 = pp ? G[1].y : G[1].x,
                  g2 = pp ? G[2].y : G[2].x;
        const u64 h2 = fma2(a2, x2, fma2(a1, x1, fma2(a0, x0, be)));  // (alpha .* W1) x + beta
        const u64 sl = slope2(h2, kLeaky);
        const u64 h3 = mul2(h2, sl);
        const u64 d2 = mul2(fma2(v2, g2, fma2(v1, g1, mul2(v0, g0))), sl);
        sd2[jj] = add2(sd2[jj], d2);
        sd2x[jj][0] = fma2(d2, x0, sd2x[jj][0]);
        sd2x[jj][1] = fma2(d2, x1, sd2x[jj][1]);
        sd2x[jj][2] = fma2(d2, x2, sd2x[jj][2]);
        sdw2[0][jj] = fma2(g0, h3, sdw2[0][jj]);
        sdw2[1][jj] = fma2(g1, h3, sdw2[1][jj]);
        sdw2[2][jj] = fma2(g2, h3, sdw2[2][jj]);
        dv[0][pp] = fma2(a0, d2, dv[0][pp]);
        dv[1][pp] = fma2(a1, d2, dv[1][pp]);
        dv[2][pp] = fma2(a2, d2, dv[2][pp]);
      }
    }
    // D over the group's four lanes; lane c < 3 stores channel c
#pragma unroll
    for (int c = 0; c < CI; ++c)
#pragma unroll
      for (int pp = 0; pp < 2; ++pp) {
        dv[c][pp] = add2(dv[c][pp], __shfl_xor_sync(0xffffffffu, dv[c][pp], 1));
        dv[c][pp] = add2(dv[c][pp], __shfl_xor_sync(0xffffffffu, dv[c][pp], 2));
      }
    if (valid && q < 3) {
      const u64 o0 = q == 0 ? dv[0][0] : (q == 1 ? dv[1][0] : dv[2][0]);
      const u64 o1 = q == 0 ? dv[0][1] : (q == 1 ? dv[1][1] : dv[2][1]);
      reinterpret_cast<ulonglong2*>(D + (b * CI + q) * HW)[i] = make_ulonglong2(o0, o1);
    }
  }
  cp_wait<0>();
  auto sum2 = [](u64 v) { return lo(v) + hi(v); };
  auto get = [&](int v) -> float {
    float r = 0.f;
    if (v >= AH<HID>::dw2) {
      const int u = v - AH<HID>::dw2, o = u / HID, j = u - o * HID;
#pragma unroll
      for (int jj = 0; jj < JH; ++jj)
        if (j == j0 + jj) r = sum2(sdw2[o][jj]);
      return r;
    }
    if (v >= AH<HID>::dy) return q == 0 ? sum2(sdy[v - AH<HID>::dy]) : 0.f;
    if (v >= AH<HID>::d2x) {
      const int u = v - AH<HID>::d2x, j = u / CI, c = u - j * CI;
#pragma unroll
      for (int jj = 0; jj < JH; ++jj)
#pragma unroll
        for (int cc = 0; cc < CI; ++cc)
          if (j == j0 + jj && c == cc) r = sum2(sd2x[jj][cc]);
      return r;
    }
#pragma unroll
    for (int jj = 0; jj < JH; ++jj)
      if (v == j0 + jj) r = sum2(sd2[jj]);
    return r;
  };
  reduce_store_fn<AH<HID>::nv>(get, part + (b * gridDim.x + blockIdx.x) * AH<HID>::nv);
}

// ---- the same pass with two lanes per 4-pixel group (default) --------------
// Lane q of a group owns hidden units [q UL, q UL + UL) (a padding unit has
// zero weights and contributes exact zeros), so every per-pixel cost -- the
// (x, dy) loads, the D exchange and store, the loop -- is shared by UL units
// instead of HID/4, and D needs one exchange (a reduce-scatter of its six
// pixel pairs over the two lanes) instead of two: 488 instead of 4 x 397
// SASS instructions per 4 pixels at hidden 15.  Both lanes load the group's
// 96 bytes straight from global memory one iteration ahead (one request per
// warp; the duplicate lanes coalesce).  The per-thread fp32 sums go through
// shared memory at the end: thread v < nv adds accumulator v over the 64
// owning threads in float64, in a fixed order.  The grid is one wave of the
// SMs' CTA slots spread over the batch.  Measured at config 2's high-res
// site (8 x 3 x 2048^2): whole backward 708 us vs 808 for k_bwd_h; at 232
// registers it runs 8 warps per SM (capping it at 3 CTAs per SM spills:
// 1021 us; staging (x, dy) by cp.async instead of registers: 836 us).
constexpr int NT2 = 128;
template <int HID, int MINB>
__global__ void __launch_bounds__(NT2, MINB) k_bwd_h2(const float* __restrict__ x,
                                                 const float* __restrict__ dy,
                                                 float* __restrict__ D,
                                                 const float* __restrict__ params,
                                                 const float* __restrict__ fold,
                                                 double* __restrict__ part, int64_t HW) {
  constexpr int UL = (HID + 1) / 2;  // hidden units per lane
  constexpr int NGR = NT2 / 2;       // groups per CTA
  constexpr int NA = 7 * UL + CO;    // fp32 sums per thread
  constexpr int NAP = NA + 1;        // shared pitch
  // unit j = q UL + jj at [jj][q]: (W1f row, beta), (W2 column, 0)
  __shared__ float4 sW[UL * 2], sV[UL * 2];
  __shared__ float red[NT2 * NAP];
  const int64_t b = blockIdx.y;
  const float* f = fold + b * F<HID>::count;
  for (int i = threadIdx.x; i < UL * 2; i += NT2) {
    const int j = (i & 1) * UL + (i >> 1);
    sW[i] = j < HID ? make_float4(f[F<HID>::w1f + j * CI], f[F<HID>::w1f + j * CI + 1],
                                  f[F<HID>::w1f + j * CI + 2], f[F<HID>::beta + j])
                    : make_float4(0.f, 0.f, 0.f, 0.f);
    sV[i] = j < HID ? make_float4(params[P<HID>::w2 + j], params[P<HID>::w2 + HID + j],
                                  params[P<HID>::w2 + 2 * HID + j], 0.f)
                    : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __syncthreads();
  using namespace pr;
  const int q = threadIdx.x & 1;
  const int g = threadIdx.x >> 1;
  u64 sd2[UL], sd2x[UL][CI], sdw2[CO][UL], sdy[CO];
#pragma unroll
  for (int jj = 0; jj < UL; ++jj) {
    sd2[jj] = 0ull;
#pragma unroll
    for (int c = 0; c < CI; ++c) sd2x[jj][c] = 0ull;
#pragma unroll
    for (int o = 0; o < CO; ++o) sdw2[o][jj] = 0ull;
  }
#pragma unroll
  for (int o = 0; o < CO; ++o) sdy[o] = 0ull;
  const int64_t n4 = HW / 4;
  const ulonglong2* xp[CI];
  const ulonglong2* gp[CO];
#pragma unroll
  for (int c = 0; c < CI; ++c) xp[c] = reinterpret_cast<const ulonglong2*>(x + (b * CI + c) * HW);
  u64* const dbase = reinterpret_cast<u64*>(D + b * CI * HW);
  const int64_t HW2 = HW / 2;
#pragma unroll
  for (int o = 0; o < CO; ++o) gp[o] = reinterpret_cast<const ulonglong2*>(dy + (b * CO + o) * HW);
  const int64_t stride = (int64_t)gridDim.x * NGR;
  // a warp-uniform trip count (groups past the end read zeros and store
  // nothing), so the pair exchange below runs converged
  const int64_t wfirst = (int64_t)blockIdx.x * NGR + (g & ~15);
  const int64_t iters = n4 > wfirst ? (n4 - wfirst + stride - 1) / stride : 0;
  // the group's next (x, dy), requested one iteration ahead
  ulonglong2 Xn[CI], Gn[CO];
  auto fetch = [&](int64_t i) {
    const bool ok = i < n4;
#pragma unroll
    for (int c = 0; c < CI; ++c) Xn[c] = ok ? __ldg(xp[c] + i) : make_ulonglong2(0ull, 0ull);
#pragma unroll
    for (int o = 0; o < CO; ++o) Gn[o] = ok ? __ldg(gp[o] + i) : make_ulonglong2(0ull, 0ull);
  };
  const int64_t first = (int64_t)blockIdx.x * NGR + g;
  fetch(first);
  for (int64_t it = 0; it < iters; ++it) {
    const int64_t i = first + it * stride;
    ulonglong2 X[CI], G[CO];
#pragma unroll
    for (int c = 0; c < CI; ++c) X[c] = Xn[c];
#pragma unroll
    for (int o = 0; o < CO; ++o) G[o] = Gn[o];
    fetch(i + stride);
#pragma unroll
    for (int o = 0; o < CO; ++o) sdy[o] = add2(sdy[o], add2(G[o].x, G[o].y));
    u64 dv[CI][2];
#pragma unroll
    for (int c = 0; c < CI; ++c) dv[c][0] = dv[c][1] = 0ull;
#pragma unroll
    for (int jj = 0; jj < UL; ++jj) {
      const float4 wv = sW[jj * 2 + q], vv = sV[jj * 2 + q];
      const u64 a0 = bc(wv.x), a1 = bc(wv.y), a2 = bc(wv.z), be = bc(wv.w);
      const u64 v0 = bc(vv.x), v1 = bc(vv.y), v2 = bc(vv.z);
#pragma unroll
      for (int pp = 0; pp < 2; ++pp) {
        const u64 x0 = pp ? X[0].y : X[0].x, x1 = pp ? X[1].y : X[1].x,
                  x2 = pp ? X[2].y : X[2].x;
        const u64 g0 = pp ? G[0].y : G[0].x, g1 = pp ? G[1].y : G[1].x,
                  g2 = pp ? G[2].y : G[2].x;
        const u64 h2 = fma2(a2, x2, fma2(a1, x1, fma2(a0, x0, be)));  // (alpha .* W1) x + beta
        const u64 sl = slope2(h2, kLeaky);
        const u64 h3 = mul2(h2, sl);
        const u64 d2 = mul2(fma2(v2, g2, fma2(v1, g1, mul2(v0, g0))), sl);
        sd2[jj] = add2(sd2[jj], d2);
        sd2x[jj][0] = fma2(d2, x0, sd2x[jj][0]);
        sd2x[jj][1] = fma2(d2, x1, sd2x[jj][1]);
        sd2x[jj][2] = fma2(d2, x2, sd2x[jj][2]);
        sdw2[0][jj] = fma2(g0, h3, sdw2[0][jj]);
        sdw2[1][jj] = fma2(g1, h3, sdw2[1][jj]);
        sdw2[2][jj] = fma2(g2, h3, sdw2[2][jj]);
        dv[0][pp] = fma2(a0, d2, dv[0][pp]);
        dv[1][pp] = fma2(a1, d2, dv[1][pp]);
        dv[2][pp] = fma2(a2, d2, dv[2][pp]);
      }
    }
    // D: pixel pair k = 2c + pp; lane 0 finishes k = 0..2, lane 1 k = 3..5
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      const int k0 = m, k1 = m + 3;
      const u64 mine = q ? dv[k1 >> 1][k1 & 1] : dv[k0 >> 1][k0 & 1];
      const u64 send = q ? dv[k0 >> 1][k0 & 1] : dv[k1 >> 1][k1 & 1];
      const u64 o = add2(mine, __shfl_xor_sync(0xffffffffu, send, 1));
      const int k = q ? k1 : k0;
      if (i < n4) dbase[(k >> 1) * HW2 + 2 * i + (k & 1)] = o;
    }
  }
  // per-thread sums -> shared -> float64 over the 64 threads of each lane parity
  {
    float* row = red + threadIdx.x * NAP;
    auto sum2 = [](u64 v) { return lo(v) + hi(v); };
#pragma unroll
    for (int jj = 0; jj < UL; ++jj) {
      row[jj] = sum2(sd2[jj]);
#pragma unroll
      for (int c = 0; c < CI; ++c) row[UL + jj * CI + c] = sum2(sd2x[jj][c]);
#pragma unroll
      for (int o = 0; o < CO; ++o) row[4 * UL + o * UL + jj] = sum2(sdw2[o][jj]);
    }
#pragma unroll
    for (int o = 0; o < CO; ++o) row[7 * UL + o] = q == 0 ? sum2(sdy[o]) : 0.f;
  }
  __syncthreads();
  constexpr int NV = AH<HID>::nv;
  double* out = part + (b * gridDim.x + blockIdx.x) * NV;
  for (int v = threadIdx.x; v < NV; v += NT2) {
    int slot, qq;
    if (v >= AH<HID>::dw2) {
      const int u = v - AH<HID>::dw2, o = u / HID, j = u - o * HID;
      qq = j / UL;
      slot = 4 * UL + o * UL + (j - qq * UL);
    } else if (v >= AH<HID>::dy) {
      qq = 0;
      slot = 7 * UL + (v - AH<HID>::dy);
    } else if (v >= AH<HID>::d2x) {
      const int u = v - AH<HID>::d2x, j = u / CI, c = u - j * CI;
      qq = j / UL;
      slot = UL + (j - qq * UL) * CI + c;
    } else {
      qq = v / UL;
      slot = v - qq * UL;
    }
    double s = 0.0;
    for (int t = qq; t < NT2; t += 2) s += (double)red[t * NAP + slot];
    out[v] = s;
  }
}

// ---- per image: kappa, lambda -> K, L and the parameter-gradient sums ------
template <int HID>
__global__ void k_fin_h(const double* __restrict__ part, const double* __restrict__ stats,
                        const float* __restrict__ params, const float* __restrict__ fold,
                        float* __restrict__ kl, double* __restrict__ gsum, int64_t HW, int nblk,
                        int nblk_h) {
  constexpr int NV = AH<HID>::nv;
  const int b = blockIdx.x;
  __shared__ double S[NV], X[9], kap[HID], lam[HID];
  for (int v = threadIdx.x; v < NV + 9; v += blockDim.x) {
    double s = 0.0;
    if (v < NV)
      for (int k = 0; k < nblk_h; ++k) s += part[((int64_t)b * nblk_h + k) * NV + v];
    else
      for (int k = 0; k < nblk; ++k) s += stats[((int64_t)b * nblk + k) * 9 + (v - NV)];
    if (v < NV)
      S[v] = s;
    else
      X[v - NV] = s;
  }
  __syncthreads();
  const float* f = fold + (int64_t)b * F<HID>::count;
  const double N = (double)HW;
  const double ng = (double)params[P<HID>::ng];
  auto w1 = [&](int j, int c) { return (double)params[P<HID>::w1 + j * CI + c]; };
  auto sd2h1 = [&](int j) {
    double s = 0.0;
    for (int c = 0; c < CI; ++c) s += w1(j, c) * S[AH<HID>::d2x + j * CI + c];
    return s;
  };
  if (threadIdx.x < HID) {
    const int j = threadIdx.x;
    const double mu = (double)f[F<HID>::mu + j], inv = (double)f[F<HID>::inv + j];
    const double sd2 = S[AH<HID>::d2 + j];
    const double gm = ng * sd2 / N;                        // mean(g), g = ng * d2
    const double gp = ng * inv * (sd2h1(j) - mu * sd2) / N;  // mean(g * xhat)
    kap[j] = -gm * inv + gp * inv * inv * mu;
    lam[j] = -gp * inv * inv;
  }
  __syncthreads();
  double* gs = gsum + (int64_t)b * GH<HID>::count;
  // x moments: X[0..2] = sum x_c, X[3..8] = sum x_c x_c' (00 01 02 11 12 22)
  const int ix[3][3] = {{3, 4, 5}, {4, 6, 7}, {5, 7, 8}};
  for (int v = threadIdx.x; v < GH<HID>::count; v += blockDim.x) {
    double r = 0.0;
    if (v < GH<HID>::db2) {
      r = S[AH<HID>::dw2 + v];
    } else if (v < GH<HID>::dgain) {
      r = S[AH<HID>::dy + v - GH<HID>::db2];
    } else if (v == GH<HID>::dgain) {
      for (int j = 0; j < HID; ++j) r += sd2h1(j);
    } else if (v == GH<HID>::dng) {
      for (int j = 0; j < HID; ++j) {
        const double mu = (double)f[F<HID>::mu + j], inv = (double)f[F<HID>::inv + j];
        r += inv * (sd2h1(j) - mu * S[AH<HID>::d2 + j]);
      }
    } else {
      const int u = v - GH<HID>::dw1, j = u / CI, c = u - j * CI;
      double wx = 0.0;  // sum_c' W1_jc' sum_p x_c' x_c
      for (int c2 = 0; c2 < CI; ++c2) wx += w1(j, c2) * X[ix[c2][c]];
      r = (double)f[F<HID>::alpha + j] * S[AH<HID>::d2x + j * CI + c] + kap[j] * X[c] +
          lam[j] * wx;
    }
    gs[v] = r;
  }
  if (threadIdx.x < KL) {
    const int v = threadIdx.x;
    double r = 0.0;
    if (v < CI) {
      for (int j = 0; j < HID; ++j) r += w1(j, v) * kap[j];
    } else {
      const int c = (v - CI) / CI, c2 = (v - CI) % CI;
      for (int j = 0; j < HID; ++j) r += w1(j, c) * lam[j] * w1(j, c2);
    }
    kl[(int64_t)b * KL + v] = (float)r;
  }
}

// ---- dx = D + K + L x (in place over D), 4 pixels per thread ---------------
__global__ void __launch_bounds__(NT) k_dx(const float* __restrict__ x, float* __restrict__ dx,
                                           const float* __restrict__ kl, int64_t HW) {
  const int64_t b = blockIdx.y;
  const float* c = kl + b * KL;
  using namespace pr;
  const u64 K0 = bc(c[0]), K1 = bc(c[1]), K2 = bc(c[2]);
  const u64 L00 = bc(c[3]), L01 = bc(c[4]), L02 = bc(c[5]), L10 = bc(c[6]), L11 = bc(c[7]),
            L12 = bc(c[8]), L20 = bc(c[9]), L21 = bc(c[10]), L22 = bc(c[11]);
  const int64_t n4 = HW / 4;
  const ulonglong2* x0 = reinterpret_cast<const ulonglong2*>(x + (b * CI + 0) * HW);
  const ulonglong2* x1 = reinterpret_cast<const ulonglong2*>(x + (b * CI + 1) * HW);
  const ulonglong2* x2 = reinterpret_cast<const ulonglong2*>(x + (b * CI + 2) * HW);
  ulonglong2* d0 = reinterpret_cast<ulonglong2*>(dx + (b * CI + 0) * HW);
  ulonglong2* d1 = reinterpret_cast<ulonglong2*>(dx + (b * CI + 1) * HW);
  ulonglong2* d2 = reinterpret_cast<ulonglong2*>(dx + (b * CI + 2) * HW);
  for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < n4; i += (int64_t)gridDim.x * NT) {
    const ulonglong2 a = __ldg(x0 + i), e = __ldg(x1 + i), g = __ldg(x2 + i);
    ulonglong2 p = d0[i], q = d1[i], r = d2[i];
    p.x = fma2(L02, g.x, fma2(L01, e.x, fma2(L00, a.x, add2(p.x, K0))));
    p.y = fma2(L02, g.y, fma2(L01, e.y, fma2(L00, a.y, add2(p.y, K0))));
    q.x = fma2(L12, g.x, fma2(L11, e.x, fma2(L10, a.x, add2(q.x, K1))));
    q.y = fma2(L12, g.y, fma2(L11, e.y, fma2(L10, a.y, add2(q.y, K1))));
    r.x = fma2(L22, g.x, fma2(L21, e.x, fma2(L20, a.x, add2(r.x, K2))));
    r.y = fma2(L22, g.y, fma2(L21, e.y, fma2(L20, a.y, add2(r.y, K2))));
    d0[i] = p;
    d1[i] = q;
    d2[i] = r;
  }
}

// ---- final parameter gradients of the one-pass backward --------------------
template <int HID>
__global__ void k_fin_params_h(const double* __restrict__ gsum, float* __restrict__ dparams,
                               int accumulate, int64_t B) {
  constexpr int GS = GH<HID>::count;
  for (int idx = threadIdx.x; idx < P<HID>::count; idx += blockDim.x) {
    int src;
    if (idx < HID * CI) src = GH<HID>::dw1 + idx;
    else if (idx == P<HID>::gain) src = GH<HID>::dgain;
    else if (idx == P<HID>::ng) src = GH<HID>::dng;
    else if (idx < P<HID>::b2) src = GH<HID>::dw2 + (idx - P<HID>::w2);
    else src = GH<HID>::db2 + (idx - P<HID>::b2);
    double s = 0.0;
    for (int64_t b = 0; b < B; ++b) s += gsum[b * GS + src];  // fixed image order
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
    const size_t ph = (size_t)B * kBlocksH * AH<HID>::nv * sizeof(double);
    const size_t kl = (size_t)B * KL * sizeof(float);
    const size_t gh = (size_t)B * GH<HID>::count * sizeof(double);
    return stats + fold + pa + coef + gsum + pb + ph + kl + gh + 9 * 256;
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
  double* ph = c.take<double>((size_t)B * kBlocksH * AH<HID>::nv);
  float* kl = c.take<float>((size_t)B * KL);
  double* gh = c.take<double>((size_t)B * GH<HID>::count);
  dim3 grid(kBlocks, (unsigned)B);
  if (!have_fold) {  // else `ws` holds forward()'s statistics and folded constants
    k_stats<<<grid, NT, 0, s>>>(x, stats, HW, status);
    k_prep<HID><<<(unsigned)B, 32, 0, s>>>(stats, params, fold, HW, kBlocks);
  }
  if (g_gn_bwd_variant != 1) {  // one heavy pass (default)
    // 0: two lanes per pixel group (k_bwd_h2); 2: four lanes (k_bwd_h, the
    // round-1 kernel); 3: k_bwd_h2 capped at 3 CTAs per SM (spills)
    const bool two = g_gn_bwd_variant != 2;
    const void* fn = g_gn_bwd_variant == 3   ? (const void*)k_bwd_h2<HID, 3>
                     : g_gn_bwd_variant == 2 ? (const void*)k_bwd_h<HID>
                                             : (const void*)k_bwd_h2<HID, 2>;
    const int nt = two ? NT2 : NT;
    const LaunchCfg lc = launch_cfg(fn, nt, 0);
    const int64_t slots = (int64_t)lc.sms * lc.per_sm;
    const int nbh = (int)std::min<int64_t>(kBlocksH, std::max<int64_t>(1, slots / B));
    const dim3 gh_grid((unsigned)nbh, (unsigned)B);
    if (two) {
      void* args[] = {(void*)&x, (void*)&dy, (void*)&dx, (void*)&params, (void*)&fold,
                      (void*)&ph, (void*)&HW};
      cudaLaunchKernel(fn, gh_grid, dim3(NT2), args, 0, s);
    }
    else
      k_bwd_h<HID><<<gh_grid, NT, 0, s>>>(x, dy, dx, params, fold, ph, HW);
    k_fin_h<HID><<<(unsigned)B, 128, 0, s>>>(ph, stats, params, fold, kl, gh, HW, kBlocks, nbh);
    k_dx<<<grid, NT, 0, s>>>(x, dx, kl, HW);
    k_fin_params_h<HID><<<1, 128, 0, s>>>(gh, dparams, accumulate, B);
    return;
  }
  // variant 1: two heavy passes (round-1 kernels)
  k_bwd_a<HID><<<grid, NT, 0, s>>>(x, dy, params, fold, pa, HW);
  k_fin_a<HID><<<(unsigned)B, 128, 0, s>>>(pa, params, fold, coef, gsum, HW, kBlocks);
  k_bwd_b<HID><<<grid, NT, 0, s>>>(x, dy, dx, params, fold, coef, pb, HW);
  // per-image dW1 sums in their own region (`stats` stays the forward's for
  // a later reuse), then the batch sum
  double* pbi = pa;  // free after k_fin_a
  k_fin_b<HID><<<(unsigned)B, 64, 0, s>>>(pb, pbi, kBlocks);
  k_fin_params<HID><<<1, 128, 0, s>>>(gsum, pbi, dparams, accumulate, B, kBlocks);
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
