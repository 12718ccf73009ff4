// Full-resolution guided filter backward (gf/guided.py:284-295 with
// _moment_backward :236-264) for fp32 NCHW on sm_100a.
//
// The backward is four window sums in sequence; each runs as ONE streaming
// kernel with the sum's input and output stages fused in (functors):
//
//   A  moments   sum (g, s, g^2, g s)         -> mean_g, mean_s, A, 1/(var+eps)
//   B  M(A)      sum A                        -> Ah (for d_guide's direct term)
//   C  M^T(d)    sum (d/N, d g/N)             -> db, dA_raw -> the four moment
//                                                grads, each / N (next adjoint)
//   D  M^T(k)    sum (k_cov, k_var, k_mx, k_my)-> d_src, d_guide
//
// The streaming sum (k_box_stream): a CTA owns a strip of tx output columns
// and a row chunk; per batch of 8 rows every thread updates the vertical
// running sums of one column (entering and leaving rows evaluated by the
// input functor, the leaving ones re-read from L2), then every thread slides a
// horizontal window along a run of 8 columns of one row (128-bit conflict-free
// shared-memory reads) and hands the window sums to the output functor.
// Stage A shifts g and s by a per-CTA constant (var, cov are shift invariant).
// A 1-channel guide is broadcast over the C source planes; its gradient is the
// sum of the per-plane contributions (deterministic, fixed channel order).
#include <cuda_runtime.h>

#include "gf_common.cuh"
#include "gf_internal.h"

namespace gfb {
namespace hrb {

constexpr int R = 8;     // rows per batch (= lanes per run group)
constexpr int NT = 256;  // threads; vertical phase: one column each
constexpr int K = 8;     // run length of the horizontal phase
constexpr int kMaxRadius = 64;

__host__ __device__ constexpr int pitch4(int n) { return n + ((36 - n % 32) % 32); }
constexpr int PV = pitch4(NT);  // shared row pitch (floats)

__device__ __forceinline__ int wlen(int i, int n, int r) {
  const int a = i - r < 0 ? 0 : i - r;
  const int b = i + r > n - 1 ? n - 1 : i + r;
  return b - a + 1;
}

struct Geom {
  int64_t P, H, W;  // planes (B*C), image size
  int r, tx, strips, segs, TY;
  int64_t C, Cg;
};

// In::operator()(plane, y, x, shift, v[NF]) fills the NF field values at an
// in-image pixel; Out::operator()(plane, y, x, shift, sums[NF]) consumes the
// window sums at an output pixel.  Both get the CTA's shift pair.
template <int NF, class In, class Out>
__global__ void __launch_bounds__(NT) k_box_stream(Geom g, In in, Out out) {
  extern __shared__ __align__(16) float vs[];  // [NF][R][PV]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int64_t item = blockIdx.x;
  const int strip = (int)(item % g.strips);
  item /= g.strips;
  const int seg = (int)(item % g.segs);
  const int64_t plane = item / g.segs;
  const int H = (int)g.H, W = (int)g.W, r = g.r;
  const int x0 = strip * g.tx;
  const int y0 = seg * g.TY;
  if (y0 >= H) return;
  const int yend = min(y0 + g.TY, H);
  const float2 sh = in.shift(plane, y0, min(x0, W - 1));
  // ---- column phase state: vs column tid <-> image column x0 - r + tid
  const int gx = x0 - r + tid;
  const bool col_ok = tid < g.tx + 2 * r && gx >= 0 && gx < W;
  float s[NF];
#pragma unroll
  for (int f = 0; f < NF; ++f) s[f] = 0.f;
  if (col_ok) {
    for (int y = max(y0 - r, 0); y < min(y0 + r, H); ++y) {
      float v[NF];
      in(plane, y, gx, sh, v);
#pragma unroll
      for (int f = 0; f < NF; ++f) s[f] += v[f];
    }
  }
  const int jr = lane & 7;
  const int q = warp * 4 + (lane >> 3);  // run of the horizontal phase
  for (int base = 0; y0 + base < yend; base += R) {
    // ---- vertical: rows y0+base .. +R-1 (window [y-r, y+r])
    if (tid < g.tx + 2 * r) {
      // every entering / leaving row of the batch is loaded before the first
      // is used: one memory latency per batch, not one per row
      float e[R][NF], l[R][NF];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const int y = y0 + base + j;
        const int ye = y + r, yl = y - r - 1;
#pragma unroll
        for (int f = 0; f < NF; ++f) e[j][f] = l[j][f] = 0.f;
        if (col_ok && y < yend) {
          if (ye < H) in(plane, ye, gx, sh, e[j]);
          if (yl >= 0 && yl >= y0 - r) in(plane, yl, gx, sh, l[j]);  // rows added so far
        }
      }
#pragma unroll
      for (int j = 0; j < R; ++j) {
#pragma unroll
        for (int f = 0; f < NF; ++f) {
          s[f] += e[j][f] - l[j][f];
          vs[(f * R + j) * PV + tid] = col_ok ? s[f] : 0.f;
        }
      }
    }
    __syncthreads();
    // ---- horizontal: output row y0+base+jr, columns x0 + qK .. +K-1
    {
      const int y = y0 + base + jr;
      const int xq = x0 + q * K;
      if (q * K < g.tx && y < yend && xq < W) {
        float hs[NF][K];
#pragma unroll
        for (int f = 0; f < NF; ++f) {
          const float* v = vs + (f * R + jr) * PV + q * K;  // vs column of window start
          float acc = 0.f;
          for (int c = 0; c < 2 * r; ++c) acc += v[c];
#pragma unroll
          for (int m = 0; m < K; ++m) {
            acc += v[m + 2 * r];
            hs[f][m] = acc;
            acc -= v[m];
          }
        }
#pragma unroll
        for (int m = 0; m < K; ++m) {
          const int x = xq + m;
          if (x < W && q * K + m < g.tx) {
            float o[NF];
#pragma unroll
            for (int f = 0; f < NF; ++f) o[f] = hs[f][m];
            out(plane, y, x, sh, o);
          }
        }
      }
    }
    __syncthreads();
  }
}

// ---- stage functors -----------------------------------------------------------
struct Ptrs {
  const float* guide;
  const float* src;
  const float* dout;
  float* mx;
  float* my;
  float* A;
  float* rv;
  float* Ah;
  float* k[4];   // k_cov, k_var, k_mx, k_my (each / N)
  float* dsrc;
  float* dg;     // per-plane guide gradient (Cg == 1) or d_guide (Cg == C)
  int64_t C, Cg, H, W;
  int r;
  float eps;
  uint32_t* status;
  __device__ int64_t gplane(int64_t p) const { return Cg == C ? p : (p / C) * Cg; }
  __device__ int64_t at(int64_t p, int y, int x) const { return (p * H + y) * W + x; }
  __device__ int64_t gat(int64_t p, int y, int x) const { return (gplane(p) * H + y) * W + x; }
  __device__ float invN(int y, int x) const {
    return 1.0f / (float)(wlen(y, (int)H, r) * wlen(x, (int)W, r));
  }
};

struct InMoments {
  Ptrs p;
  __device__ float2 shift(int64_t pl, int y, int x) const {
    return make_float2(__ldg(p.guide + p.gat(pl, y, x)), __ldg(p.src + p.at(pl, y, x)));
  }
  __device__ void operator()(int64_t pl, int y, int x, float2 sh, float v[4]) const {
    const float gg = __ldg(p.guide + p.gat(pl, y, x)) - sh.x;
    const float ss = __ldg(p.src + p.at(pl, y, x)) - sh.y;
    v[0] = gg;
    v[1] = ss;
    v[2] = gg * gg;
    v[3] = gg * ss;
  }
};
struct OutMoments {
  Ptrs p;
  __device__ void operator()(int64_t pl, int y, int x, float2 sh, const float s[4]) const {
    const float inv = p.invN(y, x);
    const float mg = s[0] * inv, ms = s[1] * inv;
    const float var = fmaf(s[2], inv, -mg * mg);
    const float cov = fmaf(s[3], inv, -mg * ms);
    if (p.eps == 0.f && !(var > 0.f)) flag(p.status, GF_STATUS_DEGENERATE);
    const float rv = 1.0f / (var + p.eps);
    const int64_t o = p.at(pl, y, x);
    p.mx[o] = mg + sh.x;
    p.my[o] = ms + sh.y;
    p.A[o] = cov * rv;
    p.rv[o] = rv;
  }
};

struct InPlane {  // one stored plane
  const float* f;
  Ptrs p;
  __device__ float2 shift(int64_t, int, int) const { return make_float2(0.f, 0.f); }
  __device__ void operator()(int64_t pl, int y, int x, float2, float v[1]) const {
    v[0] = __ldg(f + p.at(pl, y, x));
  }
};
struct OutMean {
  float* o;
  Ptrs p;
  __device__ void operator()(int64_t pl, int y, int x, float2, const float s[1]) const {
    o[p.at(pl, y, x)] = s[0] * p.invN(y, x);
  }
};

struct InDout {  // (d/N, d g/N)
  Ptrs p;
  __device__ float2 shift(int64_t, int, int) const { return make_float2(0.f, 0.f); }
  __device__ void operator()(int64_t pl, int y, int x, float2, float v[2]) const {
    const float inv = p.invN(y, x);
    const float d = __ldg(p.dout + p.at(pl, y, x));
    v[0] = d * inv;
    v[1] = (d * __ldg(p.guide + p.gat(pl, y, x))) * inv;
  }
};
struct OutMomGrads {  // gf/guided.py:236-253, each result / N (the next adjoint)
  Ptrs p;
  __device__ void operator()(int64_t pl, int y, int x, float2, const float s[2]) const {
    const int64_t o = p.at(pl, y, x);
    const float db = s[0];
    const float ux = p.mx[o], uy = p.my[o], A = p.A[o], rv = p.rv[o];
    const float dA = fmaf(-db, ux, s[1]);
    const float d_cov = dA * rv;
    const float d_var = -dA * A * rv;
    const float d_my = fmaf(-d_cov, ux, db);
    const float d_mx = fmaf(-2.f * d_var, ux, fmaf(-d_cov, uy, -db * A));
    const float inv = p.invN(y, x);
    p.k[0][o] = d_cov * inv;
    p.k[1][o] = d_var * inv;
    p.k[2][o] = d_mx * inv;
    p.k[3][o] = d_my * inv;
  }
};

struct InK {
  Ptrs p;
  __device__ float2 shift(int64_t, int, int) const { return make_float2(0.f, 0.f); }
  __device__ void operator()(int64_t pl, int y, int x, float2, float v[4]) const {
    const int64_t o = p.at(pl, y, x);
#pragma unroll
    for (int f = 0; f < 4; ++f) v[f] = __ldg(p.k[f] + o);
  }
};
struct OutGrads {  // gf/guided.py:255-263 + the direct term d_out * Ah (:292-295)
  Ptrs p;
  __device__ void operator()(int64_t pl, int y, int x, float2, const float s[4]) const {
    const int64_t o = p.at(pl, y, x);
    const float gx = __ldg(p.guide + p.gat(pl, y, x));
    const float sv = __ldg(p.src + o);
    p.dsrc[o] = fmaf(s[0], gx, s[3]);
    const float dg = fmaf(s[0], sv, fmaf(2.f * s[1], gx, s[2]));
    const float out = fmaf(__ldg(p.dout + o), p.Ah[o], dg);
    if (!isfinite(out)) flag(p.status, GF_STATUS_NONFINITE_OUTPUT);
    p.dg[o] = out;
  }
};

// d_guide (B, 1, H, W) = sum over the C broadcast planes (fixed order)
__global__ void k_guide_sum(const float* __restrict__ dg, float* __restrict__ out, int64_t B,
                            int64_t C, int64_t hw) {
  GF_GRID_LOOP(i, B * hw) {
    const int64_t b = i / hw, px = i - b * hw;
    float s = 0.f;
    for (int64_t c = 0; c < C; ++c) s += dg[(b * C + c) * hw + px];
    out[i] = s;
  }
}

template <int NF, class In, class Out>
void run(const Geom& g, In in, Out out, cudaStream_t s) {
  const size_t smem = (size_t)NF * R * PV * sizeof(float);
  launch_cfg((const void*)k_box_stream<NF, In, Out>, NT, smem);  // per-device smem limit
  const int64_t grid = g.P * g.strips * g.segs;
  k_box_stream<NF, In, Out><<<(unsigned)grid, NT, smem, s>>>(g, in, out);
}

}  // namespace hrb

bool fused_highres_bwd_ok(int64_t B, int64_t Cg, int64_t C, int64_t H, int64_t W, int r) {
  if (r < 1 || r > hrb::kMaxRadius) return false;
  if (H < 1 || W < 1 || H > (1 << 30) || W > (1 << 30)) return false;
  if (Cg != 1 && Cg != C) return false;
  return B >= 1 && C >= 1;
}

size_t fused_highres_bwd_ws_bytes(int64_t B, int64_t Cg, int64_t C, int64_t H, int64_t W) {
  const size_t plane = (size_t)B * C * H * W * sizeof(float);
  const size_t up = (plane + 255) / 256 * 256;
  return up * (9 + (Cg == C ? 0 : 1)) + 256;
}

void fused_highres_bwd(const float* guide, const float* src, const float* d_out, float* d_guide,
                       float* d_src, int64_t B, int64_t Cg, int64_t C, int64_t H, int64_t W, int r,
                       float eps, void* ws, uint32_t* status, cudaStream_t s) {
  const size_t plane = (size_t)B * C * H * W * sizeof(float);
  const size_t up = (plane + 255) / 256 * 256;
  char* w = (char*)ws;
  auto take = [&]() {
    float* p = (float*)w;
    w += up;
    return p;
  };
  hrb::Ptrs p;
  p.guide = guide;
  p.src = src;
  p.dout = d_out;
  p.mx = take();
  p.my = take();
  p.A = take();
  p.rv = take();
  p.Ah = take();
  for (int f = 0; f < 4; ++f) p.k[f] = take();
  p.dsrc = d_src;
  p.dg = Cg == C ? d_guide : take();
  p.C = C;
  p.Cg = Cg;
  p.H = H;
  p.W = W;
  p.r = r;
  p.eps = eps;
  p.status = status;
  // geometry: strips of equal width <= NT - 2r (multiple of K), row chunks
  // so that the grid fills the GPU about four times
  hrb::Geom g;
  g.P = B * C;
  g.H = H;
  g.W = W;
  g.r = r;
  g.C = C;
  g.Cg = Cg;
  const int txm = (hrb::NT - 2 * r) / hrb::K * hrb::K;
  const int64_t nstrip = (W + txm - 1) / txm;
  g.tx = (int)(((W + nstrip - 1) / nstrip + hrb::K - 1) / hrb::K * hrb::K);
  g.strips = (int)((W + g.tx - 1) / g.tx);
  int64_t segs = (148 * 8 + g.P * g.strips - 1) / (g.P * g.strips);
  const int64_t min_rows = 4 * r > 32 ? 4 * r : 32;  // keep the 2r warm-up rows a small share
  if (segs > H / min_rows) segs = H / min_rows > 0 ? H / min_rows : 1;
  if (segs < (H + 1023) / 1024) segs = (H + 1023) / 1024;  // bounded running-sum length
  g.TY = (int)((H + segs - 1) / segs);
  g.segs = (int)((H + g.TY - 1) / g.TY);
  hrb::run<4>(g, hrb::InMoments{p}, hrb::OutMoments{p}, s);
  hrb::run<1>(g, hrb::InPlane{p.A, p}, hrb::OutMean{p.Ah, p}, s);
  hrb::run<2>(g, hrb::InDout{p}, hrb::OutMomGrads{p}, s);
  hrb::run<4>(g, hrb::InK{p}, hrb::OutGrads{p}, s);
  if (Cg != C)
    hrb::k_guide_sum<<<grid_for(B * H * W), 256, 0, s>>>(p.dg, d_guide, B, C, H * W);
}

}  // namespace gfb
