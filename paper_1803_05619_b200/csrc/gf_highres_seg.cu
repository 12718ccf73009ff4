// Full-resolution guided filter forward (gf/guided.py:198-233), fp32 NCHW on
// sm_100a, register-segment variant for r <= 8: ONE kernel, one warp per work
// unit, no CTA barriers.
//
// A warp owns a strip of 256 image columns (8 consecutive columns per lane:
// two 16-byte chunks; 4 per lane as a variant) and streams a piece of rows
// top to bottom.  Per
// coefficient row ya:
//   level 1, vertical   window sums of (g, s, g^2, g*s) over rows ya-r..ya+r
//                       kept in REGISTERS per column; the entering row is
//                       loaded (HBM), the leaving row re-loaded (L2)
//   level 1, horizontal lane-local prefix sums over the lane's 8 columns; the
//                       window parts that lie in the neighbouring lanes come
//                       by shuffle (r <= 8: only lanes t-1 and t+1)
//                       -> A = cov/(var+eps), b' = mean_s - A mean_g
//   level 2, vertical   window sums of (A, b') over rows y-r..y+r in
//                       registers; the leaving coefficient row comes from a
//                       ring of 2r+1 rows in shared memory (the only smem)
//   level 2, horizontal as level 1 -> out = (Ah (G - sG) + b'h)/N + sS
// Output columns of a warp: [PAD, PAD + OW) of its 256 (the rest is halo).
//
// Arithmetic is on fp32 column PAIRS (FADD2/FFMA2/FMUL2): a 16-byte load
// lands as two pairs (c, c+1), which every stage keeps.  Windows are clamped
// to the image and normalised by the true count N = ny*nx
// (gf/filters.py:82-103).  g and s are shifted by a per-piece constant
// (sG, sS) so the fp32 second moments stay small (var/cov are shift
// invariant); running sums restart for every piece (<= 1024 rows).
#include <cuda_runtime.h>

#include <type_traits>

#include "gf_common.cuh"
#include "gf_internal.h"
#include "gf_pair.cuh"

namespace gfb {
namespace hrs {

using namespace pr;

constexpr int kMaxRadius = 8;

__host__ __device__ constexpr int up4(int n) { return (n + 3) / 4 * 4; }

// SW columns per lane (4 or 8), a warp covers 32*SW columns
template <int SW, int RAD>
struct Geo {
  static constexpr int NP = SW / 2;                        // column pairs per lane
  static constexpr int NC = SW / 4;                        // 16-byte chunks per lane
  static constexpr int WC = 32 * SW;                       // columns per warp
  static constexpr int PAD = up4(2 * RAD);                 // left halo, 16-byte aligned
  // output columns per warp; SW = 8, r = 8: 216 instead of 224 so the ring
  // spans 29 lanes (31.5 KB: 7 warps per SM instead of 6; W = 2048 still
  // needs 10 strips)
  static constexpr int OW = (SW == 8 && RAD == 8) ? 216 : (WC - PAD - 2 * RAD) / 4 * 4;
  static constexpr int ringN = 2 * RAD + 1;                // coefficient rows kept
  // lanes whose columns feed an output ([PAD - r, PAD + OW + r)): only these
  // keep a ring (the others' level-2 sums are never read)
  // (8 columns per lane only: at 4 per lane the ring does not bind occupancy
  // and the lane test measured slower)
  static constexpr int L0 = SW == 8 ? (PAD - RAD) / SW : 0;
  static constexpr int L1 =
      SW == 8 && (PAD + OW + RAD + SW - 1) / SW < 32 ? (PAD + OW + RAD + SW - 1) / SW : 32;
  static constexpr int RL = L1 - L0;
  static constexpr size_t smem_bytes = (size_t)ringN * RL * NP * 4 * sizeof(float);
};

struct Args {
  const float* guide;
  const float* src;
  float* out;
  int64_t C, Cg, H, W;
  int strips;
  int64_t U, chunk;  // rows of all (image, strip) columns; rows per warp
  float eps;
  uint32_t* status;
};

__device__ __forceinline__ u64 sub2(u64 a, u64 b) {
  u64 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

__device__ __forceinline__ int wlen(int i, int n, int r) {
  const int a = i - r < 0 ? 0 : i - r;
  const int b = i + r > n - 1 ? n - 1 : i + r;
  return b - a + 1;
}

// Horizontal window sums over +-r of one field held as SW/2 column pairs of
// this lane (columns SW*t .. SW*t+SW-1 of the warp).  Lanes near the warp's
// ends produce garbage in the columns whose window leaves the warp (unused).
//
// SW = 8, r <= 8: the window of column j reaches lanes t-1 .. t+1:
//   W_j = [T_{t-1} - p_{t-1}[7+j-r]] + [p[min(7,j+r)] - p[j-r-1]] + p_{t+1}[j+r-8]
// SW = 4, r = 4K: lanes t-K .. t+K, and with C = T_{t-K} + sum_{|d|<K} T_{t+d}
//   W_j = C + p_{t+K}[j] - p_{t-K}[j-1]
// (p = inclusive lane prefix, T = p[SW-1], p[-1] = 0, terms outside 0..7 absent)
template <int SW, int RAD>
__device__ __forceinline__ void hwin(const u64 (&v)[SW / 2], u64 (&w)[SW / 2]) {
  constexpr int r = RAD;
  float p[SW];  // inclusive prefix (scalar chain: pairs would need repacking moves)
  p[0] = lo(v[0]);
  p[1] = p[0] + hi(v[0]);
#pragma unroll
  for (int m = 1; m < SW / 2; ++m) {
    p[2 * m] = p[2 * m - 1] + lo(v[m]);
    p[2 * m + 1] = p[2 * m] + hi(v[m]);
  }
  if constexpr (SW == 4) {
    static_assert(r % 4 == 0, "SW = 4 needs r = 4K");
    constexpr int K = r / 4;
    float pl[3], pn[4];
#pragma unroll
    for (int k = 0; k < 3; ++k) pl[k] = __shfl_up_sync(0xffffffffu, p[k], K);
#pragma unroll
    for (int k = 0; k < 4; ++k) pn[k] = __shfl_down_sync(0xffffffffu, p[k], K);
    // C = sum of the 2K lane totals T_{t-K} .. T_{t+K-1}: doubling sums over
    // lanes t.. (S_n = T_t + .. + T_{t+n-1}), then one shift by K
    float sn = p[3];
#pragma unroll
    for (int n = 1; n < 2 * K; n *= 2) sn += __shfl_down_sync(0xffffffffu, sn, n);
    static_assert((2 * K & (2 * K - 1)) == 0, "2K lanes: a power of two");
    const float c = __shfl_up_sync(0xffffffffu, sn, K);
    w[0] = pk(c + pn[0], (c + pn[1]) - pl[0]);
    w[1] = add2(sub2(pk(pn[2], pn[3]), pk(pl[1], pl[2])), bc(c));
  } else {
    static_assert(SW == 8 && r <= 8, "SW = 8 needs r <= 8");
    // from lane t-1: p[k] for k = 7-r .. 7 (k = -1 reads as 0)
    // from lane t+1: p[k] for k = 0 .. r-1
    float pl[8], pn[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      pl[k] = 0.f;
      pn[k] = 0.f;
    }
#pragma unroll
    for (int k = (7 - r < 0 ? 0 : 7 - r); k < 8; ++k)
      pl[k] = __shfl_up_sync(0xffffffffu, p[k], 1);
#pragma unroll
    for (int k = 0; k < r; ++k) pn[k] = __shfl_down_sync(0xffffffffu, p[k], 1);
    // W_j = X_j + Y_j - Z_j
    float X[8], Y[8], Z[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      X[j] = j < r ? p[j + r < 7 ? j + r : 7] + pl[7] : p[j + r < 7 ? j + r : 7];
      Y[j] = j + r > 7 ? pn[j + r - 8] : 0.f;
      Z[j] = 0.f;
      if (j - r - 1 >= 0) Z[j] = p[j - r - 1];
      if (j < r && 7 + j - r >= 0) Z[j] = pl[7 + j - r];
    }
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int j = 2 * m;
      // X of the pair is one value when both columns take the same own/left terms
      const bool xsame = ((j < r) == (j + 1 < r)) &&
                         ((j + r < 7 ? j + r : 7) == (j + 1 + r < 7 ? j + 1 + r : 7));
      const bool yany = j + r > 7 || j + 1 + r > 7;
      u64 t;
      if (xsame && yany)
        t = add2(pk(Y[j], Y[j + 1]), bc(X[j]));
      else if (yany)
        t = add2(pk(X[j], X[j + 1]), pk(Y[j], Y[j + 1]));
      else
        t = pk(X[j], X[j + 1]);
      const bool zl = (j - r - 1 >= 0) || (j < r && 7 + j - r >= 0);
      const bool zh = (j - r >= 0) || (j + 1 < r && 8 + j - r >= 0);
      if (zl || zh) t = sub2(t, pk(Z[j], Z[j + 1]));
      w[m] = t;
    }
  }
}

__device__ __forceinline__ u64 lo2(float4 v) { return pk(v.x, v.y); }
__device__ __forceinline__ u64 hi2(float4 v) { return pk(v.z, v.w); }
__device__ __forceinline__ u64 half2(float4 v, int m) { return (m & 1) ? hi2(v) : lo2(v); }
__device__ __forceinline__ float4 ld4(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}
__device__ __forceinline__ float4 mask4(float4 v, bool ok) {
  return ok ? v : make_float4(0.f, 0.f, 0.f, 0.f);
}

// the rows one step prefetches: entering (g, s), leaving (g, s)
template <int NC>
struct Bufs {
  float4 eg[NC], es[NC], lg[NC], ls[NC];
};

struct Piece {
  const float* G;
  const float* S;
  float* O;
  int H, W, y0, y1, xl, lane;  // xl: image column of the lane's first column
  float sG, sS, eps;
};

// Stream one piece: output rows [y0, y1) of the warp's strip.
// EDGE: some lane chunks lie outside the image (loads clamped and masked) or
// some windows are clipped by the image's left/right border; otherwise every
// column's horizontal count is 2r+1.
template <int SW, int RAD, bool EDGE>
__device__ __forceinline__ void run_piece(const Piece& P, float4* __restrict__ ring, float& vmin,
                                          float& chk) {
  using GG = Geo<SW, RAD>;
  constexpr int r = RAD;
  constexpr int NP = GG::NP, NC = GG::NC;
  constexpr int ringN = GG::ringN;
  const int H = P.H, W = P.W, y0 = P.y0, y1 = P.y1, xl = P.xl, lane = P.lane;
  const float* __restrict__ G = P.G;
  const float* __restrict__ Sp = P.S;
  const float eps = P.eps;
  // chunk h (columns xl+4h .. xl+4h+3) is in the image or entirely outside
  bool ok[NC];
  int xc[NC];  // load column of chunk h (clamped into the image)
  u64 SGc[NC], SSc[NC];
  const u64 SG = bc(P.sG), SS = bc(P.sS);
#pragma unroll
  for (int h = 0; h < NC; ++h) {
    ok[h] = !EDGE || (xl + 4 * h >= 0 && xl + 4 * h < W);
    xc[h] = ok[h] ? xl + 4 * h : 0;
    // an out-of-image chunk is masked to zero and shifted by zero
    SGc[h] = ok[h] ? SG : 0ull;
    SSc[h] = ok[h] ? SS : 0ull;
  }
  u64 inx[NP], nxe[NP];  // 1/nx and nx per column pair (0 outside the image)
#pragma unroll
  for (int m = 0; m < NP; ++m) {
    float i[2], n[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int x = xl + 2 * m + t;
      const bool in = x >= 0 && x < W;
      const float nx = (float)wlen(x, W, r);
      i[t] = in ? fast_rcp(nx) : 0.f;
      n[t] = in ? nx : 0.f;
    }
    // interior strips: every column has the full count 2r+1 (constants)
    inx[m] = EDGE ? pk(i[0], i[1]) : bc(1.f / (2 * r + 1));
    nxe[m] = EDGE ? pk(n[0], n[1]) : bc((float)(2 * r + 1));
  }
  // coefficient columns that feed an output of this strip (vmin tracking)
  bool cok[SW];
#pragma unroll
  for (int j = 0; j < SW; ++j) {
    const int cw = SW * lane + j, x = xl + j;
    cok[j] = cw >= GG::PAD - r && cw < GG::PAD + GG::OW + r && x >= 0 && x < W;
  }

  const int ya_lo = max(y0 - r, 0);
  const int ya_end = y1 + r;  // steps ya in [ya_lo, ya_end)
  const int first_in = max(ya_lo - r, 0);

  // ---- level-1 vertical warm-up: rows first_in .. ya_lo + r - 1
  u64 VI[NP], VP[NP], VII[NP], VIP[NP];
#pragma unroll
  for (int m = 0; m < NP; ++m) VI[m] = VP[m] = VII[m] = VIP[m] = 0ull;
#pragma unroll 4
  for (int y = first_in; y < min(ya_lo + r, H); ++y) {
    const int ro = y * W;
    float4 g4[NC], s4[NC];
#pragma unroll
    for (int h = 0; h < NC; ++h) {
      g4[h] = mask4(ld4(G + ro + xc[h]), ok[h]);
      s4[h] = mask4(ld4(Sp + ro + xc[h]), ok[h]);
    }
#pragma unroll
    for (int m = 0; m < NP; ++m) {
      const u64 eI = sub2(half2(g4[m >> 1], m), SGc[m >> 1]);
      const u64 eP = sub2(half2(s4[m >> 1], m), SSc[m >> 1]);
      VI[m] = add2(VI[m], eI);
      VP[m] = add2(VP[m], eP);
      VII[m] = fma2(eI, eI, VII[m]);
      VIP[m] = fma2(eI, eP, VIP[m]);
    }
  }

  u64 VA[NP], VB[NP];  // level-2 vertical sums of A and b' (column pairs)
#pragma unroll
  for (int m = 0; m < NP; ++m) VA[m] = VB[m] = 0ull;

  // rows of step ya (clamped into the image unless STEADY; the step masks what
  // it must not use)
  auto fetch = [&](auto steady, Bufs<NC>& B, int ya) {
    constexpr bool STEADY = decltype(steady)::value;
    int e = ya + r, l = ya - r - 1;
    if (!STEADY) {
      e = min(e, H - 1);
      l = max(l, 0);
    }
    const float* ge = G + (e * W + xc[0]);
    const float* se = Sp + (e * W + xc[0]);
    const float* gl = G + (l * W + xc[0]);
    const float* sl = Sp + (l * W + xc[0]);
#pragma unroll
    for (int h = 0; h < NC; ++h) {
      const int d = xc[h] - xc[0];  // 4h unless a chunk is clamped
      B.eg[h] = ld4(ge + d);
      B.es[h] = ld4(se + d);
      B.lg[h] = ld4(gl + d);
      B.ls[h] = ld4(sl + d);
    }
  };

  int slot = 0;  // ring slot of row ya (== slot of row ya - ringN)
  // STEADY: rows ya-r-1 .. ya+r+1 inside [first_in, H), a leaving ring row,
  // an output row, and step ya+1 steady too (no clamps, no conditions)
  auto step = [&](auto steady, int ya, Bufs<NC>& cur, Bufs<NC>& nxt) {
    constexpr bool STEADY = decltype(steady)::value;
    if (STEADY || ya + 1 < ya_end) fetch(steady, nxt, ya + 1);
    // guide row of this step's output (an L2 hit: it entered 2r steps ago),
    // loaded now and used at the end of the step
    float4 og[NC];
    {
      const int o = STEADY ? ya - r : min(max(ya - r, 0), H - 1);
      const float* go = G + (o * W + xc[0]);
#pragma unroll
      for (int h = 0; h < NC; ++h) og[h] = ld4(go + (xc[h] - xc[0]));
    }
    if (EDGE) {
#pragma unroll
      for (int h = 0; h < NC; ++h) {
        cur.eg[h] = mask4(cur.eg[h], ok[h]);
        cur.es[h] = mask4(cur.es[h], ok[h]);
        cur.lg[h] = mask4(cur.lg[h], ok[h]);
        cur.ls[h] = mask4(cur.ls[h], ok[h]);
      }
    }
    u64 A2[NP], B2[NP];  // (A, b') of row ya, column pairs
    if (STEADY || ya < H) {
      // ---- level-1 vertical update (rows outside [first_in, H) contribute 0)
      const bool ein = STEADY || ya + r < H, lin = STEADY || ya - r - 1 >= first_in;
#pragma unroll
      for (int m = 0; m < NP; ++m) {
        const int h = m >> 1;
        u64 eI = sub2(half2(cur.eg[h], m), SGc[h]);
        u64 eP = sub2(half2(cur.es[h], m), SSc[h]);
        u64 nlI = sub2(SGc[h], half2(cur.lg[h], m));  // -(l_g)
        u64 lP = sub2(half2(cur.ls[h], m), SSc[h]);
        if (!STEADY) {
          if (!ein) eI = eP = 0ull;
          if (!lin) nlI = lP = 0ull;
        }
        const u64 dI = add2(eI, nlI);
        VI[m] = add2(VI[m], dI);
        VII[m] = fma2(dI, sub2(eI, nlI), VII[m]);  // e^2 - l^2
        VP[m] = add2(VP[m], sub2(eP, lP));
        VIP[m] = fma2(eI, eP, VIP[m]);
        VIP[m] = fma2(nlI, lP, VIP[m]);
      }
      // ---- level-1 horizontal + coefficients:
      //   N var = s_gg - mean_g s_g, N cov = s_gs - mean_g s_s,
      //   A = N cov / (N var + N eps), b' = mean_s - A mean_g
      u64 hI[NP], hP[NP], hII[NP], hIP[NP];
      hwin<SW, RAD>(VI, hI);
      hwin<SW, RAD>(VP, hP);
      hwin<SW, RAD>(VII, hII);
      hwin<SW, RAD>(VIP, hIP);
      const float ny = (float)wlen(ya, H, r);
      const float iny = fast_rcp(ny);
      const u64 piny = bc(iny), niny = bc(-iny), epsny = bc(eps * ny);
#pragma unroll
      for (int m = 0; m < NP; ++m) {
        const u64 nmI = mul2(hI[m], mul2(inx[m], niny));  // -mean_g
        const u64 mP = mul2(hP[m], mul2(inx[m], piny));
        const u64 vv = fma2(nmI, hI[m], hII[m]);
        const u64 cv = fma2(nmI, hP[m], hIP[m]);
        const u64 ve = fma2(nxe[m], epsny, vv);
        const u64 A = mul2(cv, pk(fast_rcp(lo(ve)), fast_rcp(hi(ve))));
        u64 B = fma2(A, nmI, mP);
        u64 Am = A;
        if (EDGE) {  // out-of-image columns carry no coefficients
          const int x = xl + 2 * m;
          const bool i0 = x >= 0 && x < W, i1 = x + 1 >= 0 && x + 1 < W;
          Am = pk(i0 ? lo(A) : 0.f, i1 ? hi(A) : 0.f);
          B = pk(i0 ? lo(B) : 0.f, i1 ? hi(B) : 0.f);
        }
        A2[m] = Am;
        B2[m] = B;
        if (eps == 0.f) {
          if (cok[2 * m]) vmin = fminf(vmin, lo(vv));
          if (cok[2 * m + 1]) vmin = fminf(vmin, hi(vv));
        }
      }
    } else {
#pragma unroll
      for (int m = 0; m < NP; ++m) A2[m] = B2[m] = 0ull;
    }

    // ---- level-2 vertical: ring slot of row ya holds row ya - ringN
    constexpr int RL = GG::RL;
    const bool rlane = lane >= GG::L0 && lane < GG::L1;
    float4* rs = ring + slot * (NP * RL) + (lane - GG::L0);
    if (rlane && (STEADY || ya - ringN >= ya_lo)) {
#pragma unroll
      for (int m = 0; m < NP; ++m) {
        const float4 q = rs[RL * m];  // (A pair m, b' pair m)
        VA[m] = sub2(VA[m], lo2(q));
        VB[m] = sub2(VB[m], hi2(q));
      }
    }
#pragma unroll
    for (int m = 0; m < NP; ++m) {
      VA[m] = add2(VA[m], A2[m]);
      VB[m] = add2(VB[m], B2[m]);
      if (rlane) rs[RL * m] = make_float4(lo(A2[m]), hi(A2[m]), lo(B2[m]), hi(B2[m]));
    }
    if (++slot == ringN) slot = 0;

    // ---- level-2 horizontal + output row y = ya - r
    const int y = ya - r;
    if (STEADY || y >= y0) {
      u64 hA[NP], hB[NP];
      hwin<SW, RAD>(VA, hA);
      hwin<SW, RAD>(VB, hB);
      const u64 iny = bc(fast_rcp((float)wlen(y, H, r)));
      float ov[SW];
#pragma unroll
      for (int m = 0; m < NP; ++m) {
        const u64 g = sub2(half2(og[m >> 1], m), SG);
        const u64 o = fma2(fma2(hA[m], g, hB[m]), mul2(inx[m], iny), SS);
        ov[2 * m] = lo(o);
        ov[2 * m + 1] = hi(o);
      }
      float* orow = P.O + y * W + xl;
#pragma unroll
      for (int h = 0; h < NC; ++h) {
        const int cw = SW * lane + 4 * h;  // warp column of the chunk
        const int x = xl + 4 * h;
        if (cw >= GG::PAD && cw < GG::PAD + GG::OW && x < W) {
          const float4 o4 = make_float4(ov[4 * h], ov[4 * h + 1], ov[4 * h + 2], ov[4 * h + 3]);
          chk = fmaf(o4.x, 0.f, chk) + fmaf(o4.y, 0.f, fmaf(o4.z, 0.f, o4.w * 0.f));
          *reinterpret_cast<float4*>(orow + 4 * h) = o4;
        }
      }
    }
  };

  // phases: general steps, steady steps (even counts keep b0 current at the
  // phase boundaries), general steps
  const std::integral_constant<bool, false> gen;
  const std::integral_constant<bool, true> sty;
  int sa = max(max(first_in + r + 1, ya_lo + ringN), y0 + r);
  sa = ya_lo + ((max(sa - ya_lo, 0) + 1) & ~1);
  const int sb = min(H - r - 1, ya_end - 1);
  Bufs<NC> b0, b1;
  fetch(gen, b0, ya_lo);
  int ya = ya_lo;
  for (; ya + 1 < min(sa, ya_end); ya += 2) {
    step(gen, ya, b0, b1);
    step(gen, ya + 1, b1, b0);
  }
  if (ya == sa) {
    for (; ya + 1 < sb; ya += 2) {
      step(sty, ya, b0, b1);
      step(sty, ya + 1, b1, b0);
    }
  }
  for (; ya < ya_end; ya += 2) {
    step(gen, ya, b0, b1);
    if (ya + 1 < ya_end) step(gen, ya + 1, b1, b0);
  }
  __syncwarp();
}

// CAP: minimum resident warps per SM asked of ptxas (a register cap; 1 = none)
template <int SW, int RAD, int CAP>
__global__ void __launch_bounds__(32, CAP) k_highres_seg(Args a) {
  using GG = Geo<SW, RAD>;
  extern __shared__ __align__(16) float4 ring[];  // [ringN][SW/2 pairs][RL ring lanes]
  const int lane = threadIdx.x;
  const int H = (int)a.H, W = (int)a.W;
  const int c = (int)(blockIdx.x % a.C);
  const int64_t chunk_id = blockIdx.x / a.C;
  const int64_t u_lo = chunk_id * a.chunk;
  const int64_t u_hi = min(u_lo + a.chunk, a.U);
  const int64_t plane = (int64_t)H * W;
  float vmin = 1.f, chk = 0.f;

  for (int64_t u = u_lo; u < u_hi;) {
    const int64_t col = u / H;
    Piece P;
    P.y0 = (int)(u - col * H);
    P.y1 = (int)min((int64_t)H, P.y0 + (u_hi - u));
    u += P.y1 - P.y0;
    const int64_t bimg = col / a.strips;
    const int strip = (int)(col - bimg * a.strips);
    const int x0 = strip * GG::OW;  // first output column
    const int xs = x0 - GG::PAD;    // image column of warp column 0
    const int64_t gplane = a.Cg == a.C ? bimg * a.C + c : bimg * a.Cg;
    const int64_t splane = bimg * a.C + c;
    P.G = a.guide + gplane * plane;
    P.S = a.src + splane * plane;
    P.O = a.out + splane * plane;
    P.H = H;
    P.W = W;
    P.xl = xs + SW * lane;
    P.lane = lane;
    P.sG = __ldg(P.G + (int64_t)P.y0 * W + x0);
    P.sS = __ldg(P.S + (int64_t)P.y0 * W + x0);
    P.eps = a.eps;
    if (xs < RAD || xs + GG::WC + RAD > W)
      run_piece<SW, RAD, true>(P, ring, vmin, chk);
    else
      run_piece<SW, RAD, false>(P, ring, vmin, chk);
  }
  if (a.eps == 0.f && !(vmin > 0.f)) flag(a.status, GF_STATUS_DEGENERATE);
  if (chk != 0.f) flag(a.status, GF_STATUS_NONFINITE_OUTPUT);
}

struct Launch {
  const void* fn;
  size_t smem;
  int ow;
};

template <int SW, int RAD, int CAP = 1>
Launch launch_info() {
  return {(const void*)k_highres_seg<SW, RAD, CAP>, Geo<SW, RAD>::smem_bytes, Geo<SW, RAD>::OW};
}

// 8 columns per lane; at r = 8 the 29-lane ring fits 7 warps per SM (293 us
// at config 1, vs 308 us for 4 columns per lane at 12 warps per SM).  Mode 2
// (test / measurement hook): 4 columns per lane at r = 8, registers capped at
// 164 (3 warps per scheduler)
Launch pick(int r, int mode) {
  switch (r) {
    case 1: return launch_info<8, 1>();
    case 2: return launch_info<8, 2>();
    case 3: return launch_info<8, 3>();
    case 4: return launch_info<8, 4>();  // 8 per lane measured faster at r = 4
    case 5: return launch_info<8, 5>();
    case 6: return launch_info<8, 6>();
    case 7: return launch_info<8, 7>();
    case 8:
      return mode == 2 ? launch_info<4, 8, 12>() : launch_info<8, 8>();
    default: return {nullptr, 0, 0};
  }
}

}  // namespace hrs

bool seg_highres_fwd_ok(int64_t B, int64_t Cg, int64_t C, int64_t H, int64_t W, int r) {
  if (r < 1 || r > hrs::kMaxRadius) return false;
  if (W % 4 != 0 || W < 4 || H < 1) return false;
  if (H * W >= ((int64_t)1 << 31)) return false;  // 32-bit in-plane offsets
  if (Cg != 1 && Cg != C) return false;
  return B >= 1 && C >= 1;
}

void seg_highres_fwd(const float* guide, const float* src, float* out, int64_t B, int64_t Cg,
                     int64_t C, int64_t H, int64_t W, int r, float eps, int mode,
                     uint32_t* status, cudaStream_t s) {
  const hrs::Launch L = hrs::pick(r, mode);
  const LaunchCfg lc = launch_cfg(L.fn, 32, L.smem);
  const int sms = lc.sms, per_sm_r = lc.per_sm;
  const int64_t strips = (W + L.ow - 1) / L.ow;
  const int64_t slots = (int64_t)sms * per_sm_r;
  // balanced pieces of the rows of all (image, strip) columns: one wave of
  // C x nch warps, more waves only to keep a piece <= 1024 rows
  const int64_t U = B * strips * H;
  const int64_t per_wave = slots / C > 0 ? slots / C : 1;
  const int64_t waves = (U + per_wave * 1024 - 1) / (per_wave * 1024);
  int64_t chunk = (U + per_wave * waves - 1) / (per_wave * waves);
  if (chunk < 8) chunk = U < 8 ? U : 8;
  const int64_t nch = (U + chunk - 1) / chunk;
  hrs::Args a{guide, src, out, C, Cg, H, W, (int)strips, U, chunk, eps, status};
  void* args[] = {&a};
  cudaLaunchKernel(L.fn, dim3((unsigned)(nch * C)), dim3(32), args, L.smem, s);
}

}  // namespace gfb
