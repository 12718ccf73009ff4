// Fused full-resolution guided filter forward (gf/guided.py:198-233) for fp32
// NCHW on sm_100a: ONE kernel reads guide and src once and writes out once.
//
// Work item = rows of (plane, column strip of tx <= 224 output columns); the
// rows of all strips are cut into equal chunks, one per CTA.  A CTA streams
// each piece of its chunk top to bottom in batches of R coefficient rows.
// Two kinds of work alternate, separated by the only two CTA barriers of a
// batch:
//
//   column phase X(k)   every thread owns one column
//     V1(k)    vertical running window sums of (g, s) and (g^2, g*s) for
//              batch k (entering rows from the TMA-staged rows, leaving rows
//              re-read from L2)                                   -> smem vs
//     V2(k-1)  vertical running sums of the coefficient rows (A, b') of
//              batch k-1: entering and leaving rows both come from the
//              coefficient ring of 2r+1+R rows                      -> vs2
//   run phase Y(k)      every thread: H1(k) on one (row, run of K=8 columns),
//                       then H2(k-1) on one (row, run)
//     H1(k)    horizontal window sums streamed over the run, A = cov/(var+eps),
//              b' = mean_s - A mean_g (shifted means)      -> coefficient ring
//     H2(k-1)  horizontal sums of (A, b') streamed over the run,
//              out = (Ah*(G - sG) + b'h)/N + sS, 128-bit loads of G and
//              stores of out
//
// Arithmetic is on fp32 PAIRS (sm_100 FADD2 / FFMA2 / FMUL2): every column,
// window and coefficient carries two fields side by side -- (s_g, s_s) and
// (s_gg, s_gs) at level 1, (A, b') at level 2 -- so one instruction updates
// both, and the shared-memory rows interleave the pair (128-bit loads fetch
// two columns).  The entering rows arrive by TMA (cp.async.bulk.tensor,
// zero-filled outside the image): the load of batch k+NSTAGE is issued at
// the start of Y(k), into the stage X(k) just consumed.
//
// Windows are clamped to the image and normalised by the true count
// N = ny*nx (gf/filters.py:82-103): out-of-image rows/columns contribute 0.
// g and s are shifted by a per-piece constant (sG, sS; var/cov are shift
// invariant) to keep the fp32 sums small; b' is the shifted intercept and the
// shift returns in the output.  Running sums restart for every piece, so
// their rounding error is bounded by the piece length (<= 1024 rows).
#include <cuda_runtime.h>

#include "gf_common.cuh"
#include "gf_internal.h"
#include "gf_tma.cuh"

namespace gfb {
namespace hrf {

constexpr int R = 8;     // coefficient rows per batch (= lanes per run group)
constexpr int NT = 256;  // threads: one vs column each in the column phase
constexpr int K = 8;     // run length of H1 and H2
constexpr int kMaxRadius = 16;
constexpr int NSTAGE = 1;  // TMA stages of the entering rows

__host__ __device__ constexpr int up4(int n) { return (n + 3) / 4 * 4; }
// smallest p >= n with p = 4 (mod 32)
__host__ __device__ constexpr int pitch4(int n) { return n + ((36 - n % 32) % 32); }
__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }
__host__ __device__ constexpr int cdiv(int a, int b) { return (a + b - 1) / b; }
// widest strip (multiple of K) whose vs columns and H1 reads fit NT columns
__host__ __device__ constexpr int tx_max(int r) {
  const int padl = up4(2 * r);
  int t = NT;
  while (t >= K && !(t + 2 * padl <= NT && cdiv(t + 2 * r, K) * K + padl <= NT)) t -= K;
  return t;
}

template <int RAD>
struct Geo {
  // vs column c <-> image column x0 - PADL + c (16-byte aligned TMA boxes); the
  // window of coefficient column a starts at vs column a + off
  static constexpr int PADL = up4(2 * RAD);
  static constexpr int off = PADL - 2 * RAD;  // 0 or 2
  static constexpr int TXM = tx_max(RAD);     // strip width bound (runtime tx <= TXM)
  static constexpr int W2M = TXM + 2 * RAD;   // coefficient columns bound
  static constexpr int RWM = cdiv(W2M, K) * K;
  static constexpr int PV = pitch4(2 * NT);   // vs rows: NT column pairs
  // coefficient rows kept: the 2r+1 of the level-2 window plus a batch, so V2
  // reads a batch's entering and leaving rows after H1 wrote the batch
  static constexpr int ringN = 2 * RAD + 1 + R;
  static constexpr int PR = pitch4(2 * RWM);  // ring rows: (A, b') pairs
  static constexpr int P2 = pitch4(2 * W2M);  // vs2 rows: (A, b') sums
  static constexpr size_t smem_floats = (size_t)NSTAGE * 2 * R * NT + (size_t)2 * R * PV +
                                        (size_t)ringN * PR + (size_t)R * P2 + 4;
  static constexpr size_t smem_bytes = smem_floats * sizeof(float);
  static constexpr uint32_t tx_bytes = 2u * R * NT * 4u;
  static constexpr int min_blocks = smem_bytes <= 113 * 1024 ? 2 : 1;
};

// ---- fp32 pair arithmetic (FADD2 / FMUL2 / FFMA2) -------------------------
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float lo(u64 v) {
  return __uint_as_float((unsigned)(v & 0xffffffffull));
}
__device__ __forceinline__ float hi(u64 v) { return __uint_as_float((unsigned)(v >> 32)); }
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
  u64 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 sub2(u64 a, u64 b) {
  u64 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
  u64 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
  u64 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ u64 lds2(const float* p) { return *reinterpret_cast<const u64*>(p); }
__device__ __forceinline__ ulonglong2 lds22(const float* p) {
  return *reinterpret_cast<const ulonglong2*>(p);
}
__device__ __forceinline__ void sts2(float* p, u64 v) { *reinterpret_cast<u64*>(p) = v; }

// CTA barrier 0
__device__ __forceinline__ void cta_sync() { asm volatile("bar.sync 0;\n" ::: "memory"); }

struct Args {
  const float* guide;
  const float* src;
  float* out;
  int64_t C, Cg, H, W;
  int tx, strips;
  int64_t U, chunk;  // rows of all (image, strip) columns; rows per CTA
  float eps;
  uint32_t* status;
};

__device__ __forceinline__ int wlen(int i, int n, int r) {
  int a = i - r < 0 ? 0 : i - r;
  int b = i + r > n - 1 ? n - 1 : i + r;
  return b - a + 1;
}

// sum of the N2 pairs p[0..N2) (16-byte aligned, N2 even)
template <int N2>
__device__ __forceinline__ u64 window_sum(const float* p) {
  u64 acc = 0;
#pragma unroll
  for (int c = 0; c < N2; c += 2) {
    const ulonglong2 v = lds22(p + 2 * c);
    acc = add2(acc, v.x);
    acc = add2(acc, v.y);
  }
  return acc;
}

// ---- run warm-up shared across lanes (r a multiple of 4, K = 8) ------------
// The window of a run's first output spans the run's own K columns and the
// next r/4 - 1 runs' columns.  Every lane loads its own K columns once (they
// are also the values that leave its window) and sums them; the neighbouring
// runs' sums arrive by shuffle (lane + 8t = same row, run q + t), except for
// the last runs of a warp, which load them.
template <int RAD>
struct Warm {
  static constexpr bool kShared = RAD % 4 == 0 && RAD >= 4 && K == 8;
  static constexpr int nS = kShared ? 2 * RAD / K : 0;
};

struct Own {
  ulonglong2 c[K / 2];  // this run's K columns (pairs), 2 per 128-bit chunk
  u64 sum;
};

__device__ __forceinline__ Own own_chunks(const float* v, bool need) {
  Own o;
  o.sum = 0;
#pragma unroll
  for (int m = 0; m < K / 2; ++m) {
    o.c[m] = need ? lds22(v + 4 * m) : make_ulonglong2(0ull, 0ull);
    o.sum = add2(o.sum, add2(o.c[m].x, o.c[m].y));
  }
  return o;
}

__device__ __forceinline__ u64 chunk_sum(const float* v) {
  u64 s = 0;
#pragma unroll
  for (int m = 0; m < K / 2; ++m) {
    const ulonglong2 c = lds22(v + 4 * m);
    s = add2(s, add2(c.x, c.y));
  }
  return s;
}

// sum of the first 2r columns of the run at v (all 32 lanes must call; only
// lanes with `task` need the result)
template <int RAD>
__device__ __forceinline__ u64 shared_warm(const float* v, u64 own_sum, int lane, bool task) {
  u64 acc = own_sum;
#pragma unroll
  for (int t = 1; t < Warm<RAD>::nS; ++t) {
    u64 nb = __shfl_down_sync(0xffffffffu, own_sum, 8 * t);
    if ((lane >> 3) + t > 3)  // run q + t belongs to the next warp
      nb = task ? chunk_sum(v + 2 * K * t) : 0ull;
    acc = add2(acc, nb);
  }
  return acc;
}

// H1 on one run: (g, s) and (gg, gs) window sums streamed over K coefficient
// columns -> (A, b') pairs into the ring row `ra`.
template <int RAD, bool INTERIOR>
__device__ __forceinline__ void h1_run(const float* vA, const float* vB, float* ra, float iny,
                                       int gxa0, int w2_left, int W, float eps, float& vmin,
                                       u64 warmA, u64 warmB, const Own& oA, const Own& oB) {
  constexpr int r = RAD;
  constexpr bool SH = Warm<RAD>::kShared;
  u64 accA = SH ? warmA : window_sum<2 * r>(vA), accB = SH ? warmB : window_sum<2 * r>(vB);
  const float inv_i = iny * (1.0f / (float)(2 * r + 1));
#pragma unroll
  for (int m = 0; m < K; m += 2) {
    const ulonglong2 eA = lds22(vA + 2 * (m + 2 * r));
    const ulonglong2 eB = lds22(vB + 2 * (m + 2 * r));
    const ulonglong2 lA = SH ? oA.c[m / 2] : lds22(vA + 2 * m);
    const ulonglong2 lB = SH ? oB.c[m / 2] : lds22(vB + 2 * m);
    u64 hA[2], hB[2];
    accA = add2(accA, eA.x); hA[0] = accA; accA = sub2(accA, lA.x);
    accB = add2(accB, eB.x); hB[0] = accB; accB = sub2(accB, lB.x);
    accA = add2(accA, eA.y); hA[1] = accA; accA = sub2(accA, lA.y);
    accB = add2(accB, eB.y); hB[1] = accB; accB = sub2(accB, lB.y);
    float cf[4];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      float inv = inv_i;
      bool ok = true;
      if constexpr (!INTERIOR) {
        const int gxa = gxa0 + m + t;
        ok = m + t < w2_left && gxa >= 0 && gxa < W;
        inv = iny * fast_rcp((float)wlen(gxa, W, r));
      }
      const u64 inv2 = pk(inv, inv);
      const u64 mA = mul2(hA[t], inv2);  // (mean g, mean s)
      const u64 mB = mul2(hB[t], inv2);  // (mean gg, mean gs)
      const float mg = lo(mA);
      const u64 vc = fma2(pk(-mg, -mg), mA, mB);  // (var, cov)
      const float var = lo(vc);
      if (ok) vmin = fminf(vmin, var);
      const float At = hi(vc) * fast_rcp(var + eps);
      cf[2 * t] = ok ? At : 0.f;
      cf[2 * t + 1] = ok ? fmaf(-At, mg, hi(mA)) : 0.f;
    }
    *reinterpret_cast<float4*>(ra + 2 * m) = make_float4(cf[0], cf[1], cf[2], cf[3]);
  }
}

// H2 on one run: window sums of (A, b') streamed over K output columns,
// out = (Ah*(G - sG) + b'h)/N + sS with 128-bit loads of G and stores of out
template <int RAD, bool INTERIOR>
__device__ __forceinline__ void h2_run(const float* v, const float* grow, float* orow,
                                       float iny, int gxo0, int W, float sG, float sS,
                                       float& chk, u64 warm, const Own& o) {
  constexpr int r = RAD;
  constexpr bool SH = Warm<RAD>::kShared;
  u64 acc = SH ? warm : window_sum<2 * r>(v);
  const float inv_i = iny * (1.0f / (float)(2 * r + 1));
#pragma unroll
  for (int m = 0; m < K; m += 4) {
    if (!INTERIOR && gxo0 + m >= W) break;  // W % 4 == 0: a float4 is all in or out
    const float4 g4 = __ldg(reinterpret_cast<const float4*>(grow + m));
    const ulonglong2 e0 = lds22(v + 2 * (m + 2 * r));
    const ulonglong2 e1 = lds22(v + 2 * (m + 2 + 2 * r));
    const ulonglong2 l0 = SH ? o.c[m / 2] : lds22(v + 2 * m);
    const ulonglong2 l1 = SH ? o.c[m / 2 + 1] : lds22(v + 2 * (m + 2));
    u64 h[4];
    acc = add2(acc, e0.x); h[0] = acc; acc = sub2(acc, l0.x);
    acc = add2(acc, e0.y); h[1] = acc; acc = sub2(acc, l0.y);
    acc = add2(acc, e1.x); h[2] = acc; acc = sub2(acc, l1.x);
    acc = add2(acc, e1.y); h[3] = acc; acc = sub2(acc, l1.y);
    const float gv[4] = {g4.x, g4.y, g4.z, g4.w};
    float ov[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      float inv = inv_i;
      if constexpr (!INTERIOR) inv = iny * fast_rcp((float)wlen(gxo0 + m + t, W, r));
      ov[t] = fmaf(fmaf(lo(h[t]), gv[t] - sG, hi(h[t])), inv, sS);
      chk += ov[t] - ov[t];  // NaN iff some output is not finite
    }
    *reinterpret_cast<float4*>(orow + m) = make_float4(ov[0], ov[1], ov[2], ov[3]);
  }
}

template <int RAD>
__global__ void __launch_bounds__(NT, Geo<RAD>::min_blocks)
    k_highres_fused(const __grid_constant__ CUtensorMap tmG,
                    const __grid_constant__ CUtensorMap tmS, Args a) {
  using GG = Geo<RAD>;
  constexpr int r = RAD;
  constexpr int ringN = GG::ringN;
  constexpr int PR = GG::PR;
  extern __shared__ __align__(128) float4 smem4[];
  float* stg = reinterpret_cast<float*>(smem4);  // [NSTAGE][2 fields][R][NT] (TMA)
  float* vsA = stg + NSTAGE * 2 * R * NT;        // [R][PV] (s_g, s_s) pairs
  float* vsB = vsA + R * GG::PV;                 // [R][PV] (s_gg, s_gs) pairs
  float* ring = vsB + R * GG::PV;                // [ringN][PR] (A, b') pairs
  float* vs2 = ring + ringN * PR;                // [R][P2] (A, b') vertical sums
  uint64_t* bar = reinterpret_cast<uint64_t*>(vs2 + R * GG::P2);  // [2 stages]
  const int H = (int)a.H, W = (int)a.W;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // Work: the rows of all (image, strip) columns of channel c, laid end to
  // end (u = (b*strips + strip)*H + y), cut into equal chunks; the C
  // channels of a chunk are consecutive CTAs so they share the guide in L2.
  // A chunk may cover the tail of one column and the head of the next: each
  // such piece is streamed separately (its own 4r warm-up rows).
  const int c = (int)(blockIdx.x % a.C);
  const int64_t chunk_id = blockIdx.x / a.C;
  const int64_t u_lo = chunk_id * a.chunk;
  const int64_t u_hi = min(u_lo + a.chunk, a.U);
  const int tx = a.tx;
  const int W2 = tx + 2 * r;  // coefficient columns of a strip
  const int64_t plane = (int64_t)H * W;
  const float eps = a.eps;
  float vmin = 1.f, chk = 0.f;
  uint32_t phases = 0;  // bit s: parity of stage s's next completion
  if (tid == 0) {
    tma::mbar_init(bar, 1);
    tma::mbar_init(bar + 1, 1);
  }
  __syncthreads();

  for (int64_t u = u_lo; u < u_hi;) {
    const int64_t col = u / H;
    const int y0 = (int)(u - col * H);
    const int yend = (int)min((int64_t)H, y0 + (u_hi - u));
    u += yend - y0;
    const int64_t b = col / a.strips;
    const int strip = (int)(col - b * a.strips);
    const int x0 = strip * tx;
    const int64_t gplane = a.Cg == a.C ? b * a.C + c : b * a.Cg;
    const int64_t splane = b * a.C + c;
    const float* __restrict__ G = a.guide + gplane * plane;
    const float* __restrict__ S = a.src + splane * plane;
    float* __restrict__ O = a.out + splane * plane;
    const float sG = __ldg(G + (int64_t)y0 * W + x0);
    const float sS = __ldg(S + (int64_t)y0 * W + x0);
    const u64 SH = pk(sG, sS);

    const int ya0 = y0 - r;                 // image row of coefficient row 0
    const int nrows = (yend - y0) + 2 * r;  // coefficient rows of this piece
    const int nb = (nrows + R - 1) / R;     // batches
    const int first_add = y0 - 2 * r;       // first input row ever added
    const int xs0 = x0 - GG::PADL;          // image column of vs / stg column 0

    // TMA of the R entering input rows of batch k (image rows ya0 + kR + r ...)
    // into stage k % NSTAGE, NSTAGE batches ahead of their use
    auto prefetch = [&](int k) {
      if (tid == 0) {
        const int st = k % NSTAGE;
        tma::fence_proxy_async();
        tma::mbar_arrive_expect_tx(bar + st, GG::tx_bytes);
        const int e0 = ya0 + k * R + r;
        float* dst = stg + st * 2 * R * NT;
        tma::load_3d(dst, &tmG, xs0, e0, (int)gplane, bar + st);
        tma::load_3d(dst + R * NT, &tmS, xs0, e0, (int)splane, bar + st);
      }
    };
#pragma unroll
    for (int k = 0; k < NSTAGE; ++k)
      if (k < nb) prefetch(k);

    // ---- column-phase state: V1 on vs column tid, V2 on coefficient column tid
    const int gx = xs0 + tid;
    const bool col_ok = gx >= 0 && gx < W;
    const char* gcb = reinterpret_cast<const char*>(G + gx);  // V1 column pointers
    const char* scb = reinterpret_cast<const char*>(S + gx);
    u64 SA = 0, SB = 0;  // (s_g, s_s), (s_gg, s_gs) of the current window
    if (col_ok) {
      for (int y = max(first_add, 0); y < y0; ++y) {
        const u64 e = sub2(pk(__ldg(G + (int64_t)y * W + gx), __ldg(S + (int64_t)y * W + gx)), SH);
        SA = add2(SA, e);
        SB = fma2(pk(lo(e), lo(e)), e, SB);
      }
    }
    const bool v2 = tid < W2;
    const float* rr = ring + 2 * tid;  // V2: ring column tid
    u64 cS = 0;                        // level-2 sums at the end of the last batch
    constexpr int dj = 2 * r + 1;      // row distance of a leaving coefficient row
    int s_cur = 0;                     // ring slot of coefficient row kR
    int s_prev = ringN - R;            // ... of row (k-1)R
    int s_lv = ringN - R - dj;         // ... of row (k-1)R - dj (its leaving row)
    const int jr = lane & 7;                      // run phase: row of the batch
    const int q = warp * 4 + (lane >> 3);         // run phase: run

    for (int k = 0; k <= nb; ++k) {
      const int base = k * R;
      // ================= column phase X(k) ===============================
      if (k < nb) {  // ---- V1(k)
        const int st = k % NSTAGE;
        float* oA = vsA + 2 * tid;
        float* oB = vsB + 2 * tid;
        const float* eg = stg + st * 2 * R * NT + tid;
        const float* es = eg + R * NT;
        const int l0 = ya0 + base - r - 1;  // leaving image row of row 0
        const bool rows_fast = base + R <= nrows && l0 >= max(first_add, 0) &&
                               ya0 + base + R - 1 + r < H;
        const bool fastc = rows_fast && col_ok;
        u64 lq[R];
        if (fastc) {  // the leaving rows (L2) load while the entering rows land
          // per-thread column pointers + CTA-uniform byte offsets of the rows
          const int64_t rowb = (int64_t)l0 * W * 4, strb = (int64_t)W * 4;
#pragma unroll
          for (int j = 0; j < R; ++j) {
            const int64_t o = rowb + j * strb;
            lq[j] = pk(__ldg(reinterpret_cast<const float*>(gcb + o)),
                       __ldg(reinterpret_cast<const float*>(scb + o)));
          }
        }
        tma::mbar_wait(bar + st, (phases >> st) & 1u);  // batch k's entering rows landed
        phases ^= 1u << st;
        if (fastc) {
          u64 ev[R];
#pragma unroll
          for (int j = 0; j < R; ++j) ev[j] = pk(eg[j * NT], es[j * NT]);
#pragma unroll
          for (int j = 0; j < R; ++j) {
            const u64 e = sub2(ev[j], SH);
            const u64 qv = sub2(lq[j], SH);
            SA = add2(SA, sub2(e, qv));
            SB = fma2(pk(lo(e), lo(e)), e, SB);
            SB = fma2(pk(-lo(qv), -lo(qv)), qv, SB);
            sts2(oA + j * GG::PV, SA);
            sts2(oB + j * GG::PV, SB);
          }
        } else if (!col_ok) {  // column outside the image: its sums stay 0
#pragma unroll
          for (int j = 0; j < R; ++j) {
            sts2(oA + j * GG::PV, 0);
            sts2(oB + j * GG::PV, 0);
          }
        } else {  // top / bottom batches: per-row predicates
#pragma unroll
          for (int j = 0; j < R; ++j) {
            const int i = base + j;
            const int e_row = ya0 + i + r, l = e_row - 2 * r - 1;
            const bool in_i = i < nrows;
            // a skipped row enters / leaves as the shift itself: contributes 0
            u64 ev = SH, lv = SH;
            if (in_i && e_row >= 0 && e_row < H) ev = pk(eg[j * NT], es[j * NT]);
            if (in_i && l >= first_add && l >= 0 && l < H)
              lv = pk(__ldg(G + (int64_t)l * W + gx), __ldg(S + (int64_t)l * W + gx));
            const u64 e = sub2(ev, SH), qv = sub2(lv, SH);
            SA = add2(SA, sub2(e, qv));
            SB = fma2(pk(lo(e), lo(e)), e, SB);
            SB = fma2(pk(-lo(qv), -lo(qv)), qv, SB);
            sts2(oA + j * GG::PV, SA);
            sts2(oB + j * GG::PV, SB);
          }
        }
      }
      if (v2 && k >= 1) {
        // ---- V2(k-1): vertical sums of batch k-1's coefficient rows -> vs2.
        // Ring rows of slots s..s+R-1 (mod ringN): rows j < w at p + j*PR, the
        // wrapped rows at p + (j - ringN)*PR.
        const int bb = base - R;             // first coefficient row of batch k-1
        const int nvalid = nrows - bb;
        const int jmin = dj - bb;            // rows j >= jmin have a leaving row
        const float* fa = rr + s_prev * PR;
        const float* fw = fa - ringN * PR;
        const int wF = ringN - s_prev;
        const float* la = rr + s_lv * PR;
        const float* lw = la - ringN * PR;
        const int wL = ringN - s_lv;
        u64 x[R], y[R];
        if (wF >= R && wL >= R && nvalid >= R && jmin <= 0) {
#pragma unroll
          for (int j = 0; j < R; ++j) {
            x[j] = lds2(fa + j * PR);
            y[j] = lds2(la + j * PR);
          }
        } else {
#pragma unroll
          for (int j = 0; j < R; ++j) {
            x[j] = 0;
            y[j] = 0;
            if (j < nvalid) {
              x[j] = lds2((j < wF ? fa : fw) + j * PR);
              if (j >= jmin) y[j] = lds2((j < wL ? la : lw) + j * PR);
            }
          }
        }
        u64 c = cS;
#pragma unroll
        for (int j = 0; j < R; ++j) {
          c = add2(c, sub2(x[j], y[j]));
          sts2(vs2 + j * GG::P2 + 2 * tid, c);
        }
        cS = c;
      }
      cta_sync();  // vs, vs2 complete; stg and the leaving ring rows consumed

      // ================= run phase Y(k) ==================================
      if (k + NSTAGE < nb) prefetch(k + NSTAGE);  // into the stage X(k) just consumed
      {  // ---- H1(k): coefficient row base+jr, columns [qK, qK+K)
        const int i = base + jr;
        const bool task = k < nb && q * K < W2 && i < nrows;
        const float* vA = vsA + jr * GG::PV + 2 * (q * K + GG::off);
        const float* vB = vA + R * GG::PV;
        Own oA, oB;
        u64 wA = 0, wB = 0;
        if constexpr (Warm<RAD>::kShared) {  // whole warp: shuffles
          // runs q - nS + 1 .. q of this row may use this run's columns
          const bool need = k < nb && q * K < W2 + (Warm<RAD>::nS - 1) * K;
          oA = own_chunks(vA, need);
          oB = own_chunks(vB, need);
          wA = shared_warm<RAD>(vA, oA.sum, lane, task);
          wB = shared_warm<RAD>(vB, oB.sum, lane, task);
        }
        if (task) {
          const int ya = ya0 + i;
          int s = s_cur + jr;
          if (s >= ringN) s -= ringN;
          float* ra = ring + s * PR + 2 * q * K;
          if (ya < 0 || ya >= H) {
#pragma unroll
            for (int m = 0; m < K; m += 2)
              *reinterpret_cast<float4*>(ra + 2 * m) = make_float4(0.f, 0.f, 0.f, 0.f);
          } else {
            const float iny = fast_rcp((float)wlen(ya, H, r));
            const int gxa0 = x0 - r + q * K;  // image column of the run's first coefficient
            if (gxa0 >= r && gxa0 + K - 1 + r <= W - 1 && q * K + K <= W2)
              h1_run<RAD, true>(vA, vB, ra, iny, gxa0, W2 - q * K, W, eps, vmin, wA, wB, oA, oB);
            else
              h1_run<RAD, false>(vA, vB, ra, iny, gxa0, W2 - q * K, W, eps, vmin, wA, wB, oA,
                                 oB);
          }
        }
      }
      {  // ---- H2(k-1): output row of coefficient row base-R+jr, columns [qK, qK+K)
        const int yo = y0 - 2 * r + base - R + jr;
        const int gxo0 = x0 + q * K;
        const bool task = k >= 1 && q * K < tx && yo >= y0 && yo < yend && gxo0 < W;
        const float* v = vs2 + jr * GG::P2 + 2 * q * K;
        Own o;
        u64 w = 0;
        if constexpr (Warm<RAD>::kShared) {
          const bool need = k >= 1 && q * K < tx + (Warm<RAD>::nS - 1) * K;
          o = own_chunks(v, need);
          w = shared_warm<RAD>(v, o.sum, lane, task);
        }
        if (task) {
          const float iny = fast_rcp((float)wlen(yo, H, r));
          const float* grow = G + (int64_t)yo * W + gxo0;
          float* orow = O + (int64_t)yo * W + gxo0;
          if (gxo0 >= r && gxo0 + K - 1 + r <= W - 1)
            h2_run<RAD, true>(v, grow, orow, iny, gxo0, W, sG, sS, chk, w, o);
          else
            h2_run<RAD, false>(v, grow, orow, iny, gxo0, W, sG, sS, chk, w, o);
        }
      }
      s_prev = s_cur;
      s_cur += R;
      if (s_cur >= ringN) s_cur -= ringN;
      s_lv += R;
      if (s_lv >= ringN) s_lv -= ringN;
      cta_sync();  // ring rows of batch k and the outputs of batch k-1 done
    }
  }
  // Non-finite inputs are not tested per element here: they always poison
  // the output at their own pixel, so the host (gf_check_finite) classifies
  // an OUTPUT flag as an input error when the inputs are non-finite.
  if (eps == 0.f && !(vmin > 0.f)) flag(a.status, GF_STATUS_DEGENERATE);
  if (chk != 0.f) flag(a.status, GF_STATUS_NONFINITE_OUTPUT);
}

struct Launch {
  const void* fn;
  int nt;
  size_t smem;
  int txm;  // widest strip
};

template <int RAD>
Launch launch_info() {
  return {(const void*)k_highres_fused<RAD>, NT, Geo<RAD>::smem_bytes, Geo<RAD>::TXM};
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
    default: return {nullptr, 0, 0, 0};
  }
}

}  // namespace hrf

bool fused_highres_fwd_ok(int64_t B, int64_t Cg, int64_t C, int64_t H, int64_t W, int r) {
  if (r < 1 || r > hrf::kMaxRadius) return false;
  if (W % 4 != 0 || W < 4 || H < 1) return false;
  if (H > (1 << 30) || W > (1 << 30) || H * W > ((int64_t)1 << 40)) return false;
  if (B * C > (1 << 30)) return false;  // TMA plane coordinate is a 32-bit int
  if (Cg != 1 && Cg != C) return false;
  if (hrf::pick(r).smem > 227 * 1024) return false;
  return B >= 1 && C >= 1;
}

void fused_highres_fwd(const float* guide, const float* src, float* out, int64_t B, int64_t Cg,
                       int64_t C, int64_t H, int64_t W, int r, float eps, uint32_t* status,
                       cudaStream_t s) {
  const hrf::Launch L = hrf::pick(r);
  const LaunchCfg lc = launch_cfg(L.fn, L.nt, L.smem);
  const int sms = lc.sms;
  // strips of equal width (multiple of K, at most the kernel's bound)
  const int64_t nstrip = (W + L.txm - 1) / L.txm;
  const int tx = (int)(((W + nstrip - 1) / nstrip + hrf::K - 1) / hrf::K * hrf::K);
  const int64_t strips = (W + tx - 1) / tx;
  const int64_t slots = (int64_t)sms * lc.per_sm;
  // balanced chunks of the rows of all (image, strip) columns: one wave of
  // C x nch CTAs, more waves only to keep a chunk <= 1024 rows (bounded
  // running-sum rounding); at least 8 rows per chunk
  const int64_t U = B * strips * H;
  const int64_t per_wave = slots / C > 0 ? slots / C : 1;
  const int64_t waves = (U + per_wave * 1024 - 1) / (per_wave * 1024);
  int64_t chunk = (U + per_wave * waves - 1) / (per_wave * waves);
  if (chunk < 8) chunk = U < 8 ? U : 8;
  const int64_t nch = (U + chunk - 1) / chunk;
  hrf::Args a{guide, src, out, C, Cg, H, W, tx, (int)strips, U, chunk, eps, status};
  const int64_t grid = nch * C;
  CUtensorMap tmG, tmS;
  if (!tma::make_plane_map(&tmG, guide, W, H, B * Cg, hrf::NT, hrf::R) ||
      !tma::make_plane_map(&tmS, src, W, H, B * C, hrf::NT, hrf::R)) {
    // surfaces as a launch error through the C ABI's cudaGetLastError check
    cudaLaunchKernel(L.fn, dim3(0), dim3(0), nullptr, 0, s);
    return;
  }
  void* args[] = {&tmG, &tmS, &a};
  cudaLaunchKernel(L.fn, dim3((unsigned)grid), dim3(L.nt), args, L.smem, s);
}

}  // namespace gfb
