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
//   V2  vertical running sums of A and b over a ring of the last
//       max(2r+1, R) coefficient rows (thread per coefficient column; the rows leaving
//       the window are read before H1 overwrites their slots)        -> smem vs2
//   H2  horizontal sums (runs of K2=8), Ah = M(A), bh = M(b),
//       out = Ah*G + bh with 128-bit loads of G and 128-bit stores of out.
//
// H1/H2 map a warp to 8 rows x 4 runs and every shared row pitch is
// = 1 (mod 8), so the 32 lanes of a run step hit 32 distinct banks.  The
// radius is a template parameter (1..16) so every window loop is unrolled.
//
// Windows are clamped to the image and normalised by the true count
// N = ny*nx (gf/filters.py:82-103): out-of-image rows/columns contribute 0.
// g and s are shifted by a per-CTA constant (var/cov are shift invariant) to
// keep the fp32 sums small; running sums restart for every segment, so their
// rounding error is bounded by the segment length, not the image size.
#include <cuda_runtime.h>

#include "gf_common.cuh"
#include "gf_internal.h"

namespace gfb {
namespace hrf {

constexpr int R = 8;     // rows per batch
constexpr int TX = 256;  // output columns per work item
constexpr int K1 = 8;    // H1 run length
constexpr int K2 = 8;    // H2 run length (two float4)
constexpr int kMaxRadius = 16;  // nt = 256 + 4r <= 320 threads

// Row pitches are = 1 (mod 8): a warp's 32 runs (8 rows x 4 runs of 8
// columns) then touch 32 distinct banks at every step of the run.
__host__ __device__ constexpr int pitch1(int n) { return n + ((9 - n % 8) % 8); }

template <int RAD>
struct Geo {
  static constexpr int W2 = TX + 2 * RAD;          // coefficient columns
  static constexpr int nq1 = (W2 + K1 - 1) / K1;   // H1 runs per row
  static constexpr int vsw = nq1 * K1 + 2 * RAD;   // vs columns (>= TX + 4r)
  static constexpr int P1 = pitch1(vsw);
  static constexpr int W1 = TX + 4 * RAD;          // real input columns
  static constexpr int ringN = 2 * RAD + 1 > R ? 2 * RAD + 1 : R;  // coefficient rows kept
  static constexpr int ringw = nq1 * K1;           // >= W2
  static constexpr int Pr = pitch1(ringw);
  static constexpr int P2 = pitch1(W2);
  // cp.async staging of the entering input rows: 16-byte chunks covering
  // [x0 - PADL, x0 + TX + PADL) with PADL = 2r rounded up to 4
  static constexpr int PADL = (2 * RAD + 3) / 4 * 4;
  static constexpr int SW = TX + 2 * PADL;
  static constexpr int nt = ((vsw > ringw ? vsw : ringw) + 31) / 32 * 32;
  static constexpr size_t smem_floats = (size_t)4 * R * P1 + (size_t)2 * ringN * Pr +
                                        (size_t)2 * R * P2 + (size_t)2 * R * SW;
  static constexpr size_t smem_bytes = smem_floats * sizeof(float);
};

__device__ __forceinline__ void cp_async16(float* dst, const float* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const int n = valid ? 16 : 0;  // 0 -> zero fill, nothing read
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n"); }

struct Args {
  const float* guide;
  const float* src;
  float* out;
  int64_t C, Cg, H, W;
  int TY, strips, segs;
  float eps;
  uint32_t* status;
};

__device__ __forceinline__ int wlen(int i, int n, int r) {
  int a = i - r < 0 ? 0 : i - r;
  int b = i + r > n - 1 ? n - 1 : i + r;
  return b - a + 1;
}

template <int RAD>
__global__ void __launch_bounds__(320, 2) k_highres_fused(Args a) {
  using GG = Geo<RAD>;
  constexpr int r = RAD;
  extern __shared__ float4 smem4[];
  float* smem = reinterpret_cast<float*>(smem4);
  const int H = (int)a.H, W = (int)a.W;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nt = GG::nt;

  float* stg = smem;                        // [2 fields][R rows][SW] (16-B aligned for cp.async)
  float* vs = stg + 2 * R * GG::SW;         // [4 fields][R rows][P1]
  float* ring = vs + 4 * R * GG::P1;        // [2 fields][ringN slots][Pr]
  float* vs2 = ring + 2 * GG::ringN * GG::Pr;  // [2 fields][R rows][P2]

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
  const float eps = a.eps;

  for (int i = tid; i < 2 * GG::ringN * GG::Pr; i += nt) ring[i] = 0.f;

  const int ya0 = y0 - r;                 // first coefficient row
  const int nrows = (yend - y0) + 2 * r;  // coefficient rows of this item
  const int first_add = y0 - 2 * r;       // first input row ever added

  // asynchronous copy of the R entering input rows of the batch at `bb`
  // (input rows ya0 + bb + j + r) into stg; out-of-image chunks zero-fill
  auto prefetch = [&](int bb) {
    constexpr int chunks = GG::SW / 4;
    for (int idx = tid; idx < 2 * R * chunks; idx += nt) {
      const int f = idx / (R * chunks);
      const int rem = idx - f * R * chunks;
      const int j = rem / chunks, cc = rem - j * chunks;
      const int e = ya0 + bb + j + r;
      const int col = x0 - GG::PADL + 4 * cc;
      const bool ok = bb + j < nrows && e >= 0 && e < H && col >= 0 && col < W;
      const float* src = (f == 0 ? G : S) + (ok ? (int64_t)e * W + col : 0);
      cp_async16(stg + (f * R + j) * GG::SW + 4 * cc, src, ok);
    }
    cp_async_commit();
  };
  prefetch(0);

  // ---- level-1 column state: thread = input column xi -------------------
  const int xi = tid;
  const int gx = x0 - 2 * r + xi;
  const bool col_ok = xi < GG::W1 && gx >= 0 && gx < W;
  const int spos = xi + GG::PADL - 2 * r;  // column of xi in stg
  float s_g = 0.f, s_gg = 0.f, s_s = 0.f, s_gs = 0.f;
  if (col_ok) {
    for (int y = max(first_add, 0); y < min(y0, H); ++y) {
      const float g = __ldg(G + (int64_t)y * W + gx) - sG;
      const float s = __ldg(S + (int64_t)y * W + gx) - sS;
      s_g += g;
      s_gg += g * g;
      s_s += s;
      s_gs += g * s;
    }
  }
  // ---- level-2 column state: thread = coefficient column ----------------
  float a_sum = 0.f, b_sum = 0.f;
  bool bad = false, degen = false;
  int ring_new = 0;  // ring slot of coefficient row `base`
  int ring_old = ((-(2 * r + 1)) % GG::ringN + GG::ringN) % GG::ringN;  // row base-2r-1

  // run mapping shared by H1 and H2: lane -> (row j = lane % 8, run q)
  const int jl = lane & 7;
  const int ql = lane >> 3;

  for (int base = 0; base < nrows; base += R) {
    // --------------------- V1 (+ V2 old-row prefetch) ------------------
    float old_a[R], old_b[R];
    if (tid < GG::W2) {
#pragma unroll
      for (int j = 0; j < R; ++j) {
        int sl = ring_old + j;
        if (sl >= GG::ringN) sl -= GG::ringN;
        old_a[j] = ring[sl * GG::Pr + tid];
        old_b[j] = ring[(GG::ringN + sl) * GG::Pr + tid];
      }
    }
    cp_async_wait_all();
    __syncthreads();  // stg complete and visible to every thread
    if (xi < GG::vsw) {
      float ge[R], se[R], gl[R], sl[R];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const int ya = ya0 + base + j;
        const int e = ya + r, l = ya - r - 1;
        ge[j] = se[j] = gl[j] = sl[j] = 0.f;
        if (col_ok && base + j < nrows) {
          if (e >= 0 && e < H) {
            ge[j] = stg[j * GG::SW + spos] - sG;
            se[j] = stg[(R + j) * GG::SW + spos] - sS;
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
        vs[(0 * R + j) * GG::P1 + xi] = col_ok ? s_g : 0.f;
        vs[(1 * R + j) * GG::P1 + xi] = col_ok ? s_gg : 0.f;
        vs[(2 * R + j) * GG::P1 + xi] = col_ok ? s_s : 0.f;
        vs[(3 * R + j) * GG::P1 + xi] = col_ok ? s_gs : 0.f;
      }
    }
    __syncthreads();

    // the next batch's entering rows stream in while H1/V2/H2 compute
    if (base + R < nrows) prefetch(base + R);

    // ------------------------------ H1 --------------------------------
    // chunk = warp-sized group of 8 rows x 4 runs
    for (int ch = warp; ch * 4 < GG::nq1; ch += nt / 32) {
      const int j = jl, q = ch * 4 + ql;
      if (q >= GG::nq1 || base + j >= nrows) continue;
      const int ya = ya0 + base + j;
      const int xa0 = q * K1;
      int slot = ring_new + j;
      if (slot >= GG::ringN) slot -= GG::ringN;
      float* ra = ring + slot * GG::Pr + xa0;
      float* rb = ring + (GG::ringN + slot) * GG::Pr + xa0;
      if (ya < 0 || ya >= H) {
#pragma unroll
        for (int k = 0; k < K1; ++k) ra[k] = rb[k] = 0.f;
        continue;
      }
      // one field at a time keeps the live window to K1 + 2r registers
      float hs[4][K1];
#pragma unroll
      for (int f = 0; f < 4; ++f) {
        const float* v = vs + (f * R + j) * GG::P1 + xa0;
        float w[K1 + 2 * r];
#pragma unroll
        for (int d = 0; d < K1 + 2 * r; ++d) w[d] = v[d];
        float acc = 0.f;
#pragma unroll
        for (int d = 0; d < 2 * r; ++d) acc += w[d];
#pragma unroll
        for (int k = 0; k < K1; ++k) {
          acc += w[k + 2 * r];
          hs[f][k] = acc;
          acc -= w[k];
        }
      }
      const float ny = (float)wlen(ya, H, r);
#pragma unroll
      for (int k = 0; k < K1; ++k) {
        const int gxa = x0 - r + xa0 + k;
        float A = 0.f, B = 0.f;
        if (xa0 + k < GG::W2 && gxa >= 0 && gxa < W) {
          const float inv = fast_rcp(ny * (float)wlen(gxa, W, r));
          const float mg = hs[0][k] * inv, ms = hs[2][k] * inv;
          const float var = hs[1][k] * inv - mg * mg;
          const float cov = hs[3][k] * inv - mg * ms;
          if (eps == 0.f && !(var > 0.f)) degen = true;
          A = cov * fast_rcp(var + eps);
          B = (ms + sS) - A * (mg + sG);
        }
        ra[k] = A;
        rb[k] = B;
      }
    }
    __syncthreads();

    // ------------------------------ V2 --------------------------------
    if (tid < GG::W2) {
#pragma unroll
      for (int j = 0; j < R; ++j) {
        if (base + j < nrows) {
          int sn = ring_new + j;
          if (sn >= GG::ringN) sn -= GG::ringN;
          a_sum += ring[sn * GG::Pr + tid] - old_a[j];
          b_sum += ring[(GG::ringN + sn) * GG::Pr + tid] - old_b[j];
        }
        vs2[(0 * R + j) * GG::P2 + tid] = a_sum;
        vs2[(1 * R + j) * GG::P2 + tid] = b_sum;
      }
    }
    ring_new += R;
    while (ring_new >= GG::ringN) ring_new -= GG::ringN;
    ring_old += R;
    while (ring_old >= GG::ringN) ring_old -= GG::ringN;
    __syncthreads();

    // ------------------------------ H2 --------------------------------
    constexpr int nq2 = TX / K2;  // 32 runs per row
    for (int ch = warp; ch * 4 < nq2; ch += nt / 32) {
      const int j = jl, q = ch * 4 + ql;
      const int yo = y0 + base + j - 2 * r;
      if (yo < y0 || yo >= yend) continue;
      const int xo0 = q * K2;
      const int gxo = x0 + xo0;
      if (gxo >= W) continue;
      const float* grow = G + (int64_t)yo * W + gxo;
      const bool two = gxo + 4 < W;
      const float4 g0 = __ldg(reinterpret_cast<const float4*>(grow));
      const float4 g1 = two ? __ldg(reinterpret_cast<const float4*>(grow + 4))
                            : make_float4(0.f, 0.f, 0.f, 0.f);
      const float gv[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
      float ha[K2], hb[K2];
#pragma unroll
      for (int f = 0; f < 2; ++f) {
        const float* v = vs2 + (f * R + j) * GG::P2 + xo0;
        float w[K2 + 2 * r];
#pragma unroll
        for (int d = 0; d < K2 + 2 * r; ++d) w[d] = v[d];
        float acc = 0.f;
#pragma unroll
        for (int d = 0; d < 2 * r; ++d) acc += w[d];
#pragma unroll
        for (int k = 0; k < K2; ++k) {
          acc += w[k + 2 * r];
          (f == 0 ? ha : hb)[k] = acc;
          acc -= w[k];
        }
      }
      const float ny = (float)wlen(yo, H, r);
      float ov[K2];
#pragma unroll
      for (int k = 0; k < K2; ++k) {
        const float inv = fast_rcp(ny * (float)wlen(gxo + k, W, r));
        ov[k] = (ha[k] * inv) * gv[k] + hb[k] * inv;
        if (k < 4 || two) {
          if (!isfinite(ov[k])) bad = true;
        }
      }
      float* orow = O + (int64_t)yo * W + gxo;
      *reinterpret_cast<float4*>(orow) = make_float4(ov[0], ov[1], ov[2], ov[3]);
      if (two) *reinterpret_cast<float4*>(orow + 4) = make_float4(ov[4], ov[5], ov[6], ov[7]);
    }
    // next batch: V1 writes vs (last read by H1, before the V2 barrier) and
    // reads ring slots H1 wrote before that barrier; V2 writes vs2 only after
    // the next H1 barrier.
  }
  // Non-finite inputs are not tested per element here: they always poison
  // the output at their own pixel, so the host (gf_check_finite) classifies
  // an OUTPUT flag as an input error when the inputs are non-finite.
  if (degen) flag(a.status, GF_STATUS_DEGENERATE);
  if (bad) flag(a.status, GF_STATUS_NONFINITE_OUTPUT);
}

struct Launch {
  const void* fn;
  int nt;
  size_t smem;
};

template <int RAD>
Launch launch_info() {
  return {(const void*)k_highres_fused<RAD>, Geo<RAD>::nt, Geo<RAD>::smem_bytes};
}

Launch pick(int r) {
  switch (r) {
    case 1: return launch_info<1>();
    case 2: return launch_info<2>();
    case 3: return launch_info<3>();
    case 4: return launch_info<4>();
    case 5: return launch_info<5>();
    case 6: return launch_info<6>();
    case 7: return launch_info<7>();
    case 8: return launch_info<8>();
    case 9: return launch_info<9>();
    case 10: return launch_info<10>();
    case 11: return launch_info<11>();
    case 12: return launch_info<12>();
    case 13: return launch_info<13>();
    case 14: return launch_info<14>();
    case 15: return launch_info<15>();
    case 16: return launch_info<16>();
    default: return {nullptr, 0, 0};
  }
}

}  // namespace hrf

bool fused_highres_fwd_ok(int64_t B, int64_t Cg, int64_t C, int64_t H, int64_t W, int r) {
  if (r < 1 || r > hrf::kMaxRadius) return false;
  if (W % 4 != 0 || W < 4 || H < 1) return false;
  if (H > (1 << 30) || W > (1 << 30) || H * W > ((int64_t)1 << 40)) return false;
  if (Cg != 1 && Cg != C) return false;
  if (hrf::pick(r).smem > 227 * 1024) return false;
  return B >= 1 && C >= 1;
}

void fused_highres_fwd(const float* guide, const float* src, float* out, int64_t B, int64_t Cg,
                       int64_t C, int64_t H, int64_t W, int r, float eps, uint32_t* status,
                       cudaStream_t s) {
  const hrf::Launch L = hrf::pick(r);
  // per-radius launch configuration, cached (the queries cost microseconds)
  static int per_sm_cache[hrf::kMaxRadius + 1] = {0};
  static int sms = 0;
  if (per_sm_cache[r] == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(L.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, L.fn, L.nt, L.smem);
    per_sm_cache[r] = per_sm < 1 ? 1 : per_sm;
  }
  const int64_t strips = (W + hrf::TX - 1) / hrf::TX;
  const int64_t planes = B * C;
  const int64_t slots = (int64_t)sms * per_sm_cache[r];
  // choose the row segmentation: minimise waves x (rows per item incl. the
  // 4r warm-up rows), with segments of at most 1024 rows (bounded rounding)
  int64_t best_segs = 1;
  double best_cost = 1e300;
  const int64_t max_segs = H / (2 * r + 1) > 0 ? H / (2 * r + 1) : 1;
  for (int64_t sg = (H + 1023) / 1024; sg <= max_segs && sg <= 4096; ++sg) {
    const int64_t ty = (H + sg - 1) / sg;
    const int64_t items = planes * strips * ((H + ty - 1) / ty);
    const int64_t waves = (items + slots - 1) / slots;
    const double cost = (double)waves * (double)(ty + 4 * r);
    if (cost < best_cost * 0.999) {
      best_cost = cost;
      best_segs = sg;
    }
  }
  const int64_t TY = (H + best_segs - 1) / best_segs;
  const int64_t segs = (H + TY - 1) / TY;
  hrf::Args a{guide, src, out, C, Cg, H, W, (int)TY, (int)strips, (int)segs, eps, status};
  const int64_t grid = planes * strips * segs;
  void* args[] = {&a};
  cudaLaunchKernel(L.fn, dim3((unsigned)grid), dim3(L.nt), args, L.smem, s);
}

}  // namespace gfb
