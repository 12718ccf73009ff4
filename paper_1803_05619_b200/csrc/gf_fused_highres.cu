// Fused full-resolution guided filter forward (gf/guided.py:198-233) for fp32
// NCHW on sm_100a: ONE kernel reads guide and src once and writes out once.
//
// Work item = (plane, column strip of TX output columns, row segment of TY
// output rows).  A CTA walks its segment top to bottom in batches of R rows
// and keeps every intermediate on chip:
//
//   V1  vertical running window sums of g, g^2, s, g*s (thread per input
//       column, registers; the leaving row is re-read from L2)      -> smem vs
//   H1  horizontal window sums (sliding runs of K1 columns), window means,
//       var, cov, A = cov/(var+eps), b = mean_s - A*mean_g           -> smem ring
//   V2  vertical running sums of A and b over the ring of the last
//       2r+1+R coefficient rows (thread per coefficient column)      -> smem vs2
//   H2  horizontal sums (runs of K2=4), Ah = M(A), bh = M(b),
//       out = Ah*G + bh with 128-bit loads of G and 128-bit stores of out.
//
// Windows are clamped to the image and normalised by the true count
// N = ny*nx (gf/filters.py:82-103): out-of-image rows/columns contribute 0.
// g and s are shifted by a per-CTA constant (var/cov are shift invariant) to
// keep the fp32 sums small; running sums restart for every segment, so their
// rounding error is bounded by the segment length, not the image size.
//
// Arithmetic per output pixel is ~150 instructions: this kernel is balanced
// between the SM issue rate and HBM (28 compulsory bytes/pixel for a 1-channel
// guide); see DESIGN.md.
#include <cuda_runtime.h>

#include "gf_common.cuh"
#include "gf_internal.h"

namespace gfb {
namespace hrf {

constexpr int R = 8;     // rows per batch
constexpr int TX = 256;  // output columns per work item
constexpr int K1 = 8;    // H1 run length
constexpr int K2 = 4;    // H2 run length (one float4)
constexpr int kMaxRadius = 16;  // nt = 256 + 4r <= 320 threads, 2 CTAs/SM

struct Geo {
  int r, W1, W2, nq1, vsw, ring, ringw, nt;
  size_t smem_bytes;
};

__host__ __device__ inline Geo geometry(int r) {
  Geo g;
  g.r = r;
  g.W2 = TX + 2 * r;                  // coefficient columns
  g.nq1 = (g.W2 + K1 - 1) / K1;       // H1 runs per row
  g.vsw = g.nq1 * K1 + 2 * r;         // vs row width (>= TX + 4r, zero padded)
  g.W1 = TX + 4 * r;                  // real input columns
  g.ring = 2 * r + 1 + R;             // coefficient rows kept
  g.ringw = g.nq1 * K1;               // ring row width (>= W2)
  g.nt = ((g.vsw > g.ringw ? g.vsw : g.ringw) + 31) / 32 * 32;
  g.smem_bytes = sizeof(float) * ((size_t)R * 4 * g.vsw + (size_t)g.ring * 2 * g.ringw +
                                  (size_t)R * 2 * (TX + 2 * r));
  return g;
}

struct Args {
  const float* guide;
  const float* src;
  float* out;
  int64_t C, Cg, H, W;
  int r, TY, strips, segs;
  float eps;
  uint32_t* status;
};

__device__ __forceinline__ int wlen(int i, int n, int r) {
  int a = i - r < 0 ? 0 : i - r;
  int b = i + r > n - 1 ? n - 1 : i + r;
  return b - a + 1;
}

__global__ void __launch_bounds__(320, 2) k_highres_fused(Args a) {
  extern __shared__ float4 smem4[];
  float* smem = reinterpret_cast<float*>(smem4);
  const Geo geo = geometry(a.r);
  const int r = a.r;
  const int H = (int)a.H, W = (int)a.W;
  const int tid = threadIdx.x, nt = blockDim.x;

  float* vs = smem;                                // [R][4][vsw]
  float* ring = vs + R * 4 * geo.vsw;              // [ring][2][ringw]
  float* vs2 = ring + geo.ring * 2 * geo.ringw;    // [R][2][W2]

  // work item: plane fastest (the C planes sharing a guide run together)
  int64_t item = blockIdx.x;
  const int c = (int)(item % a.C);
  item /= a.C;
  const int strip = (int)(item % a.strips);
  item /= a.strips;
  const int seg = (int)(item % a.segs);
  const int64_t b = item / a.segs;
  const int x0 = strip * TX;
  const int y0 = seg * a.TY;
  if (y0 >= H) return;
  const int yend = min(y0 + a.TY, H);
  const int64_t plane = (int64_t)H * W;
  const float* __restrict__ G = a.guide + (a.Cg == a.C ? b * a.C + c : b * a.Cg) * plane;
  const float* __restrict__ S = a.src + (b * a.C + c) * plane;
  float* __restrict__ O = a.out + (b * a.C + c) * plane;

  const float sG = __ldg(G + (int64_t)y0 * W + x0);
  const float sS = __ldg(S + (int64_t)y0 * W + x0);

  for (int i = tid; i < geo.ring * 2 * geo.ringw; i += nt) ring[i] = 0.f;

  // ---- level-1 column state: thread = input column xi -------------------
  const int xi = tid;
  const int gx = x0 - 2 * r + xi;
  const bool col_ok = xi < geo.W1 && gx >= 0 && gx < W;
  float s_g = 0.f, s_gg = 0.f, s_s = 0.f, s_gs = 0.f;
  const int ya0 = y0 - r;                  // first coefficient row
  const int nrows = (yend - y0) + 2 * r;   // coefficient rows of this item
  const int first_add = y0 - 2 * r;        // first input row ever added
  if (col_ok) {
    for (int y = max(first_add, 0); y < min(y0, H); ++y) {
      float g = __ldg(G + (int64_t)y * W + gx) - sG;
      float s = __ldg(S + (int64_t)y * W + gx) - sS;
      s_g += g;
      s_gg += g * g;
      s_s += s;
      s_gs += g * s;
    }
  }
  // ---- level-2 column state: thread = coefficient column ----------------
  float a_sum = 0.f, b_sum = 0.f;
  bool bad = false, degen = false;

  for (int base = 0; base < nrows; base += R) {
    // ------------------------------ V1 --------------------------------
    if (xi < geo.vsw) {
      float ge[R], se[R], gl[R], sl[R];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const int ya = ya0 + base + j;
        const int e = ya + r, l = ya - r - 1;
        ge[j] = se[j] = gl[j] = sl[j] = 0.f;
        if (col_ok && base + j < nrows) {
          if (e >= 0 && e < H) {
            ge[j] = __ldg(G + (int64_t)e * W + gx) - sG;
            se[j] = __ldg(S + (int64_t)e * W + gx) - sS;
          }
          if (l >= first_add && l >= 0 && l < H) {
            gl[j] = __ldg(G + (int64_t)l * W + gx) - sG;
            sl[j] = __ldg(S + (int64_t)l * W + gx) - sS;
          }
        }
      }
#pragma unroll
      for (int j = 0; j < R; ++j) {
        s_g += ge[j] - gl[j];
        s_gg += ge[j] * ge[j] - gl[j] * gl[j];
        s_s += se[j] - sl[j];
        s_gs += ge[j] * se[j] - gl[j] * sl[j];
        float* row = vs + j * 4 * geo.vsw;
        row[xi] = col_ok ? s_g : 0.f;
        row[geo.vsw + xi] = col_ok ? s_gg : 0.f;
        row[2 * geo.vsw + xi] = col_ok ? s_s : 0.f;
        row[3 * geo.vsw + xi] = col_ok ? s_gs : 0.f;
      }
    }
    __syncthreads();

    // ------------------------------ H1 --------------------------------
    for (int it = tid; it < R * geo.nq1; it += nt) {
      const int j = it / geo.nq1, q = it - j * geo.nq1;
      if (base + j >= nrows) continue;
      const int ya = ya0 + base + j;
      const int xa0 = q * K1;
      float* rrow = ring + ((base + j) % geo.ring) * 2 * geo.ringw;
      const bool row_ok = ya >= 0 && ya < H;
      if (!row_ok) {
#pragma unroll
        for (int k = 0; k < K1; ++k) rrow[xa0 + k] = rrow[geo.ringw + xa0 + k] = 0.f;
        continue;
      }
      const float* v = vs + j * 4 * geo.vsw + xa0;
      float sg = 0.f, sgg = 0.f, ss = 0.f, sgs = 0.f;
      for (int d = 0; d < 2 * r; ++d) {
        sg += v[d];
        sgg += v[geo.vsw + d];
        ss += v[2 * geo.vsw + d];
        sgs += v[3 * geo.vsw + d];
      }
      const float ny = (float)wlen(ya, H, r);
#pragma unroll
      for (int k = 0; k < K1; ++k) {
        const int d = k + 2 * r;
        sg += v[d];
        sgg += v[geo.vsw + d];
        ss += v[2 * geo.vsw + d];
        sgs += v[3 * geo.vsw + d];
        const int gxa = x0 - r + xa0 + k;
        float A = 0.f, B = 0.f;
        if (xa0 + k < geo.W2 && gxa >= 0 && gxa < W) {
          const float inv = __frcp_rn(ny * (float)wlen(gxa, W, r));
          const float mg = sg * inv, ms = ss * inv;
          const float var = sgg * inv - mg * mg;
          const float cov = sgs * inv - mg * ms;
          if (a.eps == 0.f && !(var > 0.f)) degen = true;
          A = cov * __frcp_rn(var + a.eps);
          B = (ms + sS) - A * (mg + sG);
        }
        rrow[xa0 + k] = A;
        rrow[geo.ringw + xa0 + k] = B;
        sg -= v[k];
        sgg -= v[geo.vsw + k];
        ss -= v[2 * geo.vsw + k];
        sgs -= v[3 * geo.vsw + k];
      }
    }
    __syncthreads();

    // ------------------------------ V2 --------------------------------
    if (tid < geo.W2) {
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const int loc = base + j;
        if (loc < nrows) {
          const float* rn = ring + (loc % geo.ring) * 2 * geo.ringw;
          a_sum += rn[tid];
          b_sum += rn[geo.ringw + tid];
          const int old = loc - 2 * r - 1;
          if (old >= 0) {
            const float* ro = ring + (old % geo.ring) * 2 * geo.ringw;
            a_sum -= ro[tid];
            b_sum -= ro[geo.ringw + tid];
          }
        }
        vs2[j * 2 * geo.W2 + tid] = a_sum;
        vs2[j * 2 * geo.W2 + geo.W2 + tid] = b_sum;
      }
    }
    __syncthreads();

    // ------------------------------ H2 --------------------------------
    constexpr int nq2 = TX / K2;
    for (int it = tid; it < R * nq2; it += nt) {
      const int j = it / nq2, q = it - j * nq2;
      const int yo = y0 + base + j - 2 * r;
      if (yo < y0 || yo >= yend) continue;
      const int xo0 = q * K2;
      const int gxo = x0 + xo0;
      if (gxo >= W) continue;
      const float* va = vs2 + j * 2 * geo.W2 + xo0;
      const float* vb = va + geo.W2;
      float sa = 0.f, sb = 0.f;
      for (int d = 0; d < 2 * r; ++d) {
        sa += va[d];
        sb += vb[d];
      }
      const float ny = (float)wlen(yo, H, r);
      const float4 g4 = __ldg(reinterpret_cast<const float4*>(G + (int64_t)yo * W + gxo));
      const float gv[4] = {g4.x, g4.y, g4.z, g4.w};
      float ov[4];
#pragma unroll
      for (int k = 0; k < K2; ++k) {
        sa += va[k + 2 * r];
        sb += vb[k + 2 * r];
        const float inv = __frcp_rn(ny * (float)wlen(gxo + k, W, r));
        ov[k] = (sa * inv) * gv[k] + sb * inv;
        if (!isfinite(ov[k])) bad = true;
        sa -= va[k];
        sb -= vb[k];
      }
      *reinterpret_cast<float4*>(O + (int64_t)yo * W + gxo) = make_float4(ov[0], ov[1], ov[2], ov[3]);
    }
    // the next batch's V1 only touches vs (last read in H1, before a barrier)
    // and H1 writes ring rows no V2 of this batch reads
  }
  // Non-finite inputs are not tested per element here: they always poison
  // the output at their own pixel, so the host (gf_check_finite) classifies
  // an OUTPUT flag as an input error when the inputs are non-finite.
  if (degen) flag(a.status, GF_STATUS_DEGENERATE);
  if (bad) flag(a.status, GF_STATUS_NONFINITE_OUTPUT);
}

}  // namespace hrf

bool fused_highres_fwd_ok(int64_t B, int64_t Cg, int64_t C, int64_t H, int64_t W, int r) {
  if (r < 1 || r > hrf::kMaxRadius) return false;
  if (W % 4 != 0 || W < 4 || H < 1) return false;
  if (H > (1 << 30) || W > (1 << 30) || H * W > ((int64_t)1 << 40)) return false;
  if (Cg != 1 && Cg != C) return false;
  if (hrf::geometry(r).smem_bytes > 227 * 1024) return false;
  return B >= 1 && C >= 1;
}

void fused_highres_fwd(const float* guide, const float* src, float* out, int64_t B, int64_t Cg,
                       int64_t C, int64_t H, int64_t W, int r, float eps, uint32_t* status,
                       cudaStream_t s) {
  const hrf::Geo geo = hrf::geometry(r);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(hrf::k_highres_fused, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         227 * 1024);
    configured = true;
  }
  // resident CTAs per SM for this radius (cached: the query costs microseconds)
  static int cached_r = -1, cached_per_sm = 1, cached_sms = 148;
  if (cached_r != r) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&cached_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cached_per_sm, hrf::k_highres_fused, geo.nt,
                                                  geo.smem_bytes);
    if (cached_per_sm < 1) cached_per_sm = 1;
    cached_r = r;
  }
  const int sms = cached_sms, per_sm = cached_per_sm;
  const int64_t strips = (W + hrf::TX - 1) / hrf::TX;
  const int64_t planes = B * C;
  const int64_t slots = (int64_t)sms * per_sm;
  // segments per column: fill whole waves, keep segments <= 512 rows so the
  // running-sum rounding stays bounded
  int64_t segs = (slots + planes * strips - 1) / (planes * strips);
  if (segs < 1) segs = 1;
  int64_t min_segs = (H + 511) / 512;
  if (segs < min_segs) {
    // round up to a whole number of waves
    int64_t items = planes * strips * min_segs;
    int64_t waves = (items + slots - 1) / slots;
    segs = (waves * slots + planes * strips - 1) / (planes * strips);
  }
  if (segs > H) segs = H;
  int64_t TY = (H + segs - 1) / segs;
  if (TY < 2 * r + 1 && H > 2 * r + 1) TY = 2 * r + 1;
  segs = (H + TY - 1) / TY;
  hrf::Args a{guide, src, out, C, Cg, H, W, r, (int)TY, (int)strips, (int)segs, eps, status};
  const int64_t grid = planes * strips * segs;
  hrf::k_highres_fused<<<(unsigned)grid, geo.nt, geo.smem_bytes, s>>>(a);
}

}  // namespace gfb
