// C ABI entry points (include/gf_b200.h): argument checks that mirror the
// reference's ValueError sites, then dispatch to the fused sm_100a kernels
// when the call is one they cover (fp32, NCHW, supported radius/ratio), or to
// the general kernels otherwise.  Both are CUDA; there is no CPU path.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdarg>
#include <cstring>

#include "../../include/gf_b200.h"
#include "gf_internal.h"

namespace {

thread_local char g_err[512] = "";
thread_local int g_force_generic = 0;
// full-res fp32 forward kernel: 0 = automatic, 1 = batch/TMA kernel, 2 = segment
// kernel, 3 = segment kernel with 8 columns per lane only
thread_local int g_highres_variant = 0;
// set by gn_backward_reuse for the duration of its gn_backward call
thread_local bool g_gn_reuse = false;

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(GF_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return GF_OK;
}

bool dtype_ok(int dt) { return dt == GF_F32 || dt == GF_F64; }

// GuidedFilterParams.__post_init__, gf/guided.py:50-53
int check_params(int r, double eps) {
  if (r < 0) return fail(GF_ERR_ARG, "radius must be a non-negative integer, got %d", r);
  if (!std::isfinite(eps) || eps < 0.0)
    return fail(GF_ERR_ARG, "eps must be finite and >= 0, got %g", eps);
  return GF_OK;
}

int check_dims(const char* name, int64_t a, int64_t b, int64_t c, int64_t d) {
  if (a < 1 || b < 1 || c < 1 || d < 1)
    return fail(GF_ERR_ARG, "%s: all dimensions must be >= 1, got (%lld, %lld, %lld, %lld)",
                name, (long long)a, (long long)b, (long long)c, (long long)d);
  return GF_OK;
}

cudaStream_t S(void* s) { return (cudaStream_t)s; }

bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

bool use_fused_joint(int dtype, int64_t B, int64_t C, int64_t h, int64_t w, int64_t H, int64_t W,
                     int r) {
  return !g_force_generic && dtype == GF_F32 && gfb::fused_joint_ok(B, C, h, w, H, W, r);
}

bool use_seg_highres(int dtype, int64_t B, int64_t Cg, int64_t C, int64_t H, int64_t W, int r) {
  if (g_force_generic || dtype != GF_F32 || g_highres_variant == 1) return false;
  return gfb::seg_highres_fwd_ok(B, Cg, C, H, W, r);
}

bool use_fused_highres(int dtype, int64_t B, int64_t Cg, int64_t C, int64_t H, int64_t W, int r) {
  if (use_seg_highres(dtype, B, Cg, C, H, W, r)) return true;
  return !g_force_generic && dtype == GF_F32 && g_highres_variant < 2 &&
         gfb::fused_highres_fwd_ok(B, Cg, C, H, W, r);
}

}  // namespace

extern "C" {

int gf_version(void) { return 100; }

const char* gf_last_error(void) { return g_err; }

// Test hook (like the reference's flipped_term, gf/guided.py:124-133): route
// every call of THIS thread through the general kernels.  Returns the old value.
int gf_force_generic(int on) {
  int old = g_force_generic;
  g_force_generic = on ? 1 : 0;
  return old;
}

// Introspection hooks (not in the public header): 1 when the call would take
// the fused sm_100a kernels, 0 when it takes the general kernels.
// Test hook: pick the fp32 full-res forward kernel of THIS thread (0 automatic,
// 1 batch/TMA kernel, 2 segment kernel, 3 segment kernel with 8 columns per
// lane (the automatic choice), 4 segment kernel with 4 columns per lane).
// Returns the old value.
int gf_highres_variant(int v) {
  int old = g_highres_variant;
  g_highres_variant = v;
  return old;
}

// Test hook: pick the fp32 joint-backward low-res tail of THIS thread (0
// automatic, 1 tile kernel, 2 register-segment kernel where it applies).
int gf_joint_bwd_lr_variant(int v) {
  int old = gfb::g_joint_lr_variant;
  gfb::g_joint_lr_variant = v;
  return old;
}

// Test hook: CTAs per SM the fused training-step hr kernel is compiled for
// (0 automatic = 3, or 2 or 4 at r = 1) on THIS thread.  Returns the old value.
int gf_joint_mse_variant(int v) {
  int old = gfb::g_joint_mse_variant;
  gfb::g_joint_mse_variant = v;
  return old;
}

// Test hook: coefficient-pass chunking of the r = 8 joint forward (0 default,
// 1..4 alternatives) on THIS thread.  Returns the old value.
int gf_joint_fwd_variant(int v) {
  int old = gfb::g_joint_fwd_variant;
  gfb::g_joint_fwd_variant = v;
  return old;
}

// Test hook: fused fp32 guidance-net backward of THIS thread (0 one heavy
// pass + dx fix-up, 1 the two-heavy-pass kernels).  Returns the old value.
int gf_gn_bwd_variant(int v) {
  int old = gfb::g_gn_bwd_variant;
  gfb::g_gn_bwd_variant = v;
  return old;
}

// Test hook: hr pass of the fp32 joint backward on THIS thread (0 single
// gather pass, 1 the two-read tile kernel, 3 single pass at 3 CTAs/SM for
// r <= 2).  Returns the old value.
// Test hook: low-res rows per tile of the tape hr pass of THIS thread (16 or 8)
int gf_joint_bwd_hr_tile(int v) {
  int old = gfb::g_joint_bwd_hr_tile;
  gfb::g_joint_bwd_hr_tile = v == 8 ? 8 : 16;
  return old;
}

int gf_joint_bwd_hr_variant(int v) {
  int old = gfb::g_joint_bwd_hr_variant;
  gfb::g_joint_bwd_hr_variant = v;
  return old;
}

int gf_joint_is_fused(int dtype, int64_t B, int64_t C, int64_t h, int64_t w, int64_t H,
                      int64_t W, int r) {
  return use_fused_joint(dtype, B, C, h, w, H, W, r) ? 1 : 0;
}

int gf_highres_fwd_is_fused(int dtype, int64_t B, int64_t Cg, int64_t C, int64_t H, int64_t W,
                            int r) {
  return use_fused_highres(dtype, B, Cg, C, H, W, r) ? 1 : 0;
}

int gf_sm_count(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  return n;
}

int gf_check_finite(int dtype, const void* data, int64_t n, uint32_t* status, void* stream) {
  if (!dtype_ok(dtype)) return fail(GF_ERR_ARG, "bad dtype %d", dtype);
  if (n < 0) return fail(GF_ERR_ARG, "negative length");
  if (n == 0) return GF_OK;
  if (dtype == GF_F32)
    gfb::generic_check_finite<float>((const float*)data, n, status, S(stream));
  else
    gfb::generic_check_finite<double>((const double*)data, n, status, S(stream));
  return check_launch("gf_check_finite");
}

// ---------------------------------------------------------------------------
// primitives
// ---------------------------------------------------------------------------
int gf_mean_filter(int dtype, const void* in, void* out, int64_t planes, int64_t h, int64_t w,
                   int radius, void* stream) {
  if (!dtype_ok(dtype)) return fail(GF_ERR_ARG, "bad dtype %d", dtype);
  if (radius < 0) return fail(GF_ERR_ARG, "radius must be a non-negative integer, got %d", radius);
  if (int e = check_dims("mean_filter", planes, h, w, 1)) return e;
  if (dtype == GF_F32)
    gfb::generic_mean_filter<float>((const float*)in, (float*)out, planes, h, w, radius, 0,
                                    S(stream));
  else
    gfb::generic_mean_filter<double>((const double*)in, (double*)out, planes, h, w, radius, 0,
                                     S(stream));
  return check_launch("gf_mean_filter");
}

int gf_mean_filter_adjoint(int dtype, const void* g, void* out, int64_t planes, int64_t h,
                           int64_t w, int radius, void* stream) {
  if (!dtype_ok(dtype)) return fail(GF_ERR_ARG, "bad dtype %d", dtype);
  if (radius < 0) return fail(GF_ERR_ARG, "radius must be a non-negative integer, got %d", radius);
  if (int e = check_dims("mean_filter_adjoint", planes, h, w, 1)) return e;
  if (dtype == GF_F32)
    gfb::generic_mean_filter<float>((const float*)g, (float*)out, planes, h, w, radius, 1,
                                    S(stream));
  else
    gfb::generic_mean_filter<double>((const double*)g, (double*)out, planes, h, w, radius, 1,
                                     S(stream));
  return check_launch("gf_mean_filter_adjoint");
}

int gf_bilinear_resize(int dtype, const void* in, void* out, int64_t planes, int64_t h, int64_t w,
                       int64_t out_h, int64_t out_w, void* stream) {
  if (!dtype_ok(dtype)) return fail(GF_ERR_ARG, "bad dtype %d", dtype);
  if (out_h < 1 || out_w < 1)
    return fail(GF_ERR_ARG, "output dims must be >= 1, got (%lld, %lld)", (long long)out_h,
                (long long)out_w);
  if (int e = check_dims("bilinear_resize", planes, h, w, 1)) return e;
  if (dtype == GF_F32)
    gfb::generic_resize<float>((const float*)in, (float*)out, planes, h, w, out_h, out_w,
                               S(stream));
  else
    gfb::generic_resize<double>((const double*)in, (double*)out, planes, h, w, out_h, out_w,
                                S(stream));
  return check_launch("gf_bilinear_resize");
}

int gf_bilinear_resize_adjoint(int dtype, const void* g, void* out, int64_t planes, int64_t g_h,
                               int64_t g_w, int64_t in_h, int64_t in_w, void* stream) {
  if (!dtype_ok(dtype)) return fail(GF_ERR_ARG, "bad dtype %d", dtype);
  if (in_h < 1 || in_w < 1)
    return fail(GF_ERR_ARG, "input dims must be >= 1, got (%lld, %lld)", (long long)in_h,
                (long long)in_w);
  if (int e = check_dims("bilinear_resize_adjoint", planes, g_h, g_w, 1)) return e;
  if (dtype == GF_F32)
    gfb::generic_resize_adj<float>((const float*)g, (float*)out, planes, g_h, g_w, in_h, in_w,
                                   S(stream));
  else
    gfb::generic_resize_adj<double>((const double*)g, (double*)out, planes, g_h, g_w, in_h, in_w,
                                    S(stream));
  return check_launch("gf_bilinear_resize_adjoint");
}

// ---------------------------------------------------------------------------
// joint (fast) layer
// ---------------------------------------------------------------------------
static int check_joint(int dtype, int64_t B, int64_t C, int64_t h, int64_t w, int64_t H,
                       int64_t W, int r, double eps) {
  if (!dtype_ok(dtype)) return fail(GF_ERR_ARG, "bad dtype %d", dtype);
  if (int e = check_params(r, eps)) return e;
  if (int e = check_dims("guide_lo", B, C, h, w)) return e;
  if (int e = check_dims("guide_hi", B, C, H, W)) return e;
  // gf/guided.py:165-168
  if (H < h || W < w)
    return fail(GF_ERR_ARG, "guide_hi dims (%lld, %lld) smaller than guide_lo (%lld, %lld)",
                (long long)H, (long long)W, (long long)h, (long long)w);
  return GF_OK;
}

// workspace of the general (any alignment / dtype / ratio) joint kernels
static size_t joint_generic_bytes(int64_t B, int64_t C, int64_t h, int64_t w) {
  return gfb::generic_workspace_bytes(B * C * h * w, 0);
}

// The fused kernels need 16-byte aligned buffers; the size returned here is
// for such buffers (what torch's allocator and the Python mirror hand out).
// Unaligned buffers take the general kernels, whose larger need is checked
// against the caller's workspace_bytes at the call (GF_ERR_WORKSPACE with the
// required size in gf_last_error, never an overrun).
size_t gf_joint_workspace_bytes(int dtype, int64_t B, int64_t C, int64_t h, int64_t w, int64_t H,
                                int64_t W, int radius) {
  if (use_fused_joint(dtype, B, C, h, w, H, W, radius))
    return gfb::fused_joint_bwd_ws_bytes(B, C, h, w);
  return joint_generic_bytes(B, C, h, w);
}

int gf_joint_fwd(int dtype, const void* lr_x, const void* lr_y, const void* hr_x, void* out,
                 int64_t B, int64_t C, int64_t h, int64_t w, int64_t H, int64_t W, int radius,
                 double eps, void* workspace, size_t workspace_bytes, uint32_t* status,
                 void* stream) {
  if (int e = check_joint(dtype, B, C, h, w, H, W, radius, eps)) return e;
  if (use_fused_joint(dtype, B, C, h, w, H, W, radius) && aligned16(lr_x) && aligned16(lr_y) &&
      aligned16(hr_x) && aligned16(out)) {
    // the two-kernel forward keeps A, b of every cell in the workspace when the
    // caller passed one of gf_joint_workspace_bytes
    float* coef_ws = workspace && aligned16(workspace) &&
                             workspace_bytes >= gfb::fused_joint_bwd_ws_bytes(B, C, h, w)
                         ? (float*)workspace
                         : nullptr;
    gfb::fused_joint_fwd((const float*)lr_x, (const float*)lr_y, (const float*)hr_x, (float*)out,
                         B, C, h, w, H, W, radius, (float)eps, status, S(stream), nullptr, coef_ws);
    return check_launch("gf_joint_fwd[fused]");
  }
  // general kernels (unaligned buffers, fp64, other shapes)
  size_t need = joint_generic_bytes(B, C, h, w);
  if (workspace_bytes < need)
    return fail(GF_ERR_WORKSPACE, "joint workspace %zu < %zu bytes (general kernels)",
                workspace_bytes, need);
  if (dtype == GF_F32)
    gfb::generic_joint_fwd<float>((const float*)lr_x, (const float*)lr_y, (const float*)hr_x,
                                  (float*)out, B, C, h, w, H, W, radius, eps, workspace, status,
                                  S(stream));
  else
    gfb::generic_joint_fwd<double>((const double*)lr_x, (const double*)lr_y, (const double*)hr_x,
                                   (double*)out, B, C, h, w, H, W, radius, eps, workspace, status,
                                   S(stream));
  return check_launch("gf_joint_fwd");
}

int64_t gf_joint_split_threshold(void) { return gfb::kJointSplitElems; }

int gf_joint_fwd_mode(int mode) {
  const int v = gfb::g_joint_fwd_variant;
  const int old = v == 19 ? 1 : (v == 20 ? 2 : 0);
  gfb::g_joint_fwd_variant = mode == 1 ? 19 : (mode == 2 ? 20 : 0);
  return old;
}

int gf_joint_coeffs(int dtype, const void* lr_x, const void* lr_y, void* slope_lo,
                    void* intercept_lo, int64_t B, int64_t C, int64_t h, int64_t w, int radius,
                    double eps, uint32_t* status, void* stream) {
  if (int e = check_joint(dtype, B, C, h, w, 4 * h, 4 * w, radius, eps)) return e;
  if (!(use_fused_joint(dtype, B, C, h, w, 4 * h, 4 * w, radius) && aligned16(lr_x) &&
        aligned16(lr_y) && aligned16(slope_lo) && aligned16(intercept_lo)))
    return fail(GF_ERR_UNSUPPORTED, "gf_joint_coeffs: not a fused-path call (use gf_joint_fwd)");
  gfb::fused_joint_coeffs((const float*)lr_x, (const float*)lr_y, (float*)slope_lo,
                          (float*)intercept_lo, B * C, h, w, radius, (float)eps, status, S(stream));
  return check_launch("gf_joint_coeffs");
}

int gf_joint_apply(int dtype, const void* slope_lo, const void* intercept_lo, const void* hr_x,
                   void* out, int64_t B, int64_t C, int64_t h, int64_t w, int64_t H, int64_t W,
                   uint32_t* status, void* stream) {
  if (int e = check_joint(dtype, B, C, h, w, H, W, 0, 1.0)) return e;
  if (!(use_fused_joint(dtype, B, C, h, w, H, W, 0) && aligned16(slope_lo) &&
        aligned16(intercept_lo) && aligned16(hr_x) && aligned16(out)))
    return fail(GF_ERR_UNSUPPORTED, "gf_joint_apply: not a fused-path call (use gf_joint_fwd)");
  gfb::joint_apply((const float*)slope_lo, (const float*)intercept_lo, (const float*)hr_x,
                   (float*)out, B * C, h, w, H, W, status, S(stream));
  return check_launch("gf_joint_apply");
}

int gf_joint_fwd_tape(int dtype, const void* lr_x, const void* lr_y, const void* hr_x, void* out,
                      void* slope_lo, int64_t B, int64_t C, int64_t h, int64_t w, int64_t H,
                      int64_t W, int radius, double eps, void* workspace, size_t workspace_bytes,
                      uint32_t* status, void* stream) {
  if (int e = check_joint(dtype, B, C, h, w, H, W, radius, eps)) return e;
  if (!(use_fused_joint(dtype, B, C, h, w, H, W, radius) && aligned16(lr_x) && aligned16(lr_y) &&
        aligned16(hr_x) && aligned16(out) && slope_lo))
    return fail(GF_ERR_UNSUPPORTED, "gf_joint_fwd_tape: not a fused-path call (use gf_joint_fwd)");
  // intercepts of the two-kernel forward (the slopes go to the tape)
  float* coef_ws = workspace && aligned16(workspace) &&
                           workspace_bytes >= (size_t)B * C * h * w * sizeof(float)
                       ? (float*)workspace
                       : nullptr;
  gfb::fused_joint_fwd((const float*)lr_x, (const float*)lr_y, (const float*)hr_x, (float*)out, B,
                       C, h, w, H, W, radius, (float)eps, status, S(stream), (float*)slope_lo,
                       coef_ws);
  return check_launch("gf_joint_fwd_tape");
}

int gf_joint_bwd_tape(int dtype, const void* lr_x, const void* lr_y, const void* hr_x,
                      const void* slope_lo, const void* d_out, void* d_lr_x, void* d_lr_y,
                      void* d_hr_x, int64_t B, int64_t C, int64_t h, int64_t w, int64_t H,
                      int64_t W, int radius, double eps, int64_t row0, void* workspace,
                      size_t workspace_bytes, uint32_t* status, void* stream) {
  if (int e = check_joint(dtype, B, C, h, w, H, W, radius, eps)) return e;
  if (row0 < 0) return fail(GF_ERR_ARG, "row0 must be >= 0, got %lld", (long long)row0);
  if (!(use_fused_joint(dtype, B, C, h, w, H, W, radius) && aligned16(lr_x) && aligned16(lr_y) &&
        aligned16(hr_x) && aligned16(d_out) && aligned16(d_lr_x) && aligned16(d_lr_y) &&
        aligned16(d_hr_x) && slope_lo))
    return fail(GF_ERR_UNSUPPORTED, "gf_joint_bwd_tape: not a fused-path call (use gf_joint_bwd)");
  const size_t need = gfb::fused_joint_bwd_ws_bytes(B, C, h, w);
  if (workspace_bytes < need)
    return fail(GF_ERR_WORKSPACE, "joint workspace %zu < %zu bytes", workspace_bytes, need);
  gfb::fused_joint_bwd((const float*)lr_x, (const float*)lr_y, (const float*)hr_x,
                       (const float*)d_out, (float*)d_lr_x, (float*)d_lr_y, (float*)d_hr_x, B, C,
                       h, w, H, W, radius, (float)eps, workspace, row0, status, S(stream),
                       (const float*)slope_lo);
  return check_launch("gf_joint_bwd_tape");
}

int gf_joint_bwd(int dtype, const void* lr_x, const void* lr_y, const void* hr_x,
                 const void* d_out, void* d_lr_x, void* d_lr_y, void* d_hr_x, int64_t B,
                 int64_t C, int64_t h, int64_t w, int64_t H, int64_t W, int radius, double eps,
                 void* workspace, size_t workspace_bytes, uint32_t* status, void* stream) {
  return gf_joint_bwd_band(dtype, lr_x, lr_y, hr_x, d_out, d_lr_x, d_lr_y, d_hr_x, B, C, h, w, H,
                           W, radius, eps, 0, workspace, workspace_bytes, status, stream);
}

int gf_joint_bwd_band(int dtype, const void* lr_x, const void* lr_y, const void* hr_x,
                      const void* d_out, void* d_lr_x, void* d_lr_y, void* d_hr_x, int64_t B,
                      int64_t C, int64_t h, int64_t w, int64_t H, int64_t W, int radius,
                      double eps, int64_t row0, void* workspace, size_t workspace_bytes,
                      uint32_t* status, void* stream) {
  if (int e = check_joint(dtype, B, C, h, w, H, W, radius, eps)) return e;
  if (row0 < 0) return fail(GF_ERR_ARG, "row0 must be >= 0, got %lld", (long long)row0);
  const bool fused = use_fused_joint(dtype, B, C, h, w, H, W, radius) && aligned16(lr_x) &&
                     aligned16(lr_y) && aligned16(hr_x) && aligned16(d_out) &&
                     aligned16(d_lr_x) && aligned16(d_lr_y) && aligned16(d_hr_x);
  size_t need = fused ? gfb::fused_joint_bwd_ws_bytes(B, C, h, w) : joint_generic_bytes(B, C, h, w);
  if (workspace_bytes < need)
    return fail(GF_ERR_WORKSPACE, "joint workspace %zu < %zu bytes%s", workspace_bytes, need,
                fused ? "" : " (general kernels)");
  if (fused) {
    gfb::fused_joint_bwd((const float*)lr_x, (const float*)lr_y, (const float*)hr_x,
                         (const float*)d_out, (float*)d_lr_x, (float*)d_lr_y, (float*)d_hr_x, B,
                         C, h, w, H, W, radius, (float)eps, workspace, row0, status, S(stream));
    return check_launch("gf_joint_bwd[fused]");
  }
  if (dtype == GF_F32)
    gfb::generic_joint_bwd<float>((const float*)lr_x, (const float*)lr_y, (const float*)hr_x,
                                  (const float*)d_out, (float*)d_lr_x, (float*)d_lr_y,
                                  (float*)d_hr_x, B, C, h, w, H, W, radius, eps, workspace,
                                  status, S(stream));
  else
    gfb::generic_joint_bwd<double>((const double*)lr_x, (const double*)lr_y,
                                   (const double*)hr_x, (const double*)d_out, (double*)d_lr_x,
                                   (double*)d_lr_y, (double*)d_hr_x, B, C, h, w, H, W, radius,
                                   eps, workspace, status, S(stream));
  return check_launch("gf_joint_bwd");
}

// ---------------------------------------------------------------------------
// full-resolution layer
// ---------------------------------------------------------------------------
static int check_highres(int dtype, int64_t B, int64_t Cg, int64_t C, int64_t H, int64_t W, int r,
                         double eps) {
  if (!dtype_ok(dtype)) return fail(GF_ERR_ARG, "bad dtype %d", dtype);
  if (int e = check_params(r, eps)) return e;
  if (int e = check_dims("src", B, C, H, W)) return e;
  if (int e = check_dims("guide", B, Cg, H, W)) return e;
  // gf/guided.py:204-205 requires equal shapes; a 1-channel guide is the
  // broadcast extension of BASELINE config 1.
  if (Cg != C && Cg != 1)
    return fail(GF_ERR_ARG, "guide/src channel mismatch: %lld vs %lld", (long long)Cg,
                (long long)C);
  return GF_OK;
}

size_t gf_highres_workspace_bytes(int dtype, int64_t B, int64_t Cg, int64_t C, int64_t H,
                                  int64_t W, int radius) {
  size_t gen = gfb::generic_workspace_bytes(B * C * H * W, 0);
  if (dtype == GF_F32 && gfb::fused_highres_bwd_ok(B, Cg, C, H, W, radius)) {
    size_t fast = gfb::fused_highres_bwd_ws_bytes(B, Cg, C, H, W);
    return fast > gen ? fast : gen;
  }
  return gen;
}

int gf_highres_fwd(int dtype, const void* guide, const void* src, void* out, int64_t B, int64_t Cg,
                   int64_t C, int64_t H, int64_t W, int radius, double eps, void* workspace,
                   size_t workspace_bytes, uint32_t* status, void* stream) {
  if (int e = check_highres(dtype, B, Cg, C, H, W, radius, eps)) return e;
  if (use_fused_highres(dtype, B, Cg, C, H, W, radius) && aligned16(guide) && aligned16(src) &&
      aligned16(out)) {
    if (use_seg_highres(dtype, B, Cg, C, H, W, radius)) {
      gfb::seg_highres_fwd((const float*)guide, (const float*)src, (float*)out, B, Cg, C, H, W,
                           radius, (float)eps,
                           g_highres_variant == 3 ? 1 : g_highres_variant == 4 ? 2 : 0, status,
                           S(stream));
      return check_launch("gf_highres_fwd[seg]");
    }
    gfb::fused_highres_fwd((const float*)guide, (const float*)src, (float*)out, B, Cg, C, H, W,
                           radius, (float)eps, status, S(stream));
    return check_launch("gf_highres_fwd[fused]");
  }
  // general kernels (unaligned buffers, fp64, other shapes)
  size_t need = gf_highres_workspace_bytes(dtype, B, Cg, C, H, W, radius);
  if (workspace_bytes < need)
    return fail(GF_ERR_WORKSPACE, "highres workspace %zu < %zu bytes (general kernels)",
                workspace_bytes, need);
  if (dtype == GF_F32)
    gfb::generic_highres_fwd<float>((const float*)guide, (const float*)src, (float*)out, B, Cg, C,
                                     H, W, radius, eps, workspace, status, S(stream));
  else
    gfb::generic_highres_fwd<double>((const double*)guide, (const double*)src, (double*)out, B,
                                      Cg, C, H, W, radius, eps, workspace, status, S(stream));
  return check_launch("gf_highres_fwd");
}

int gf_highres_bwd(int dtype, const void* guide, const void* src, const void* d_out,
                   void* d_guide, void* d_src, int64_t B, int64_t Cg, int64_t C, int64_t H,
                   int64_t W, int radius, double eps, void* workspace, size_t workspace_bytes,
                   uint32_t* status, void* stream) {
  if (int e = check_highres(dtype, B, Cg, C, H, W, radius, eps)) return e;
  size_t need = gf_highres_workspace_bytes(dtype, B, Cg, C, H, W, radius);
  if (workspace_bytes < need)
    return fail(GF_ERR_WORKSPACE, "highres workspace %zu < %zu bytes", workspace_bytes, need);
  if (!g_force_generic && dtype == GF_F32 && gfb::fused_highres_bwd_ok(B, Cg, C, H, W, radius)) {
    gfb::fused_highres_bwd((const float*)guide, (const float*)src, (const float*)d_out,
                           (float*)d_guide, (float*)d_src, B, Cg, C, H, W, radius, (float)eps,
                           workspace, status, S(stream));
    return check_launch("gf_highres_bwd[fused]");
  }
  if (dtype == GF_F32)
    gfb::generic_highres_bwd<float>((const float*)guide, (const float*)src, (const float*)d_out,
                                     (float*)d_guide, (float*)d_src, B, Cg, C, H, W, radius, eps,
                                     workspace, status, S(stream));
  else
    gfb::generic_highres_bwd<double>((const double*)guide, (const double*)src,
                                      (const double*)d_out, (double*)d_guide, (double*)d_src, B,
                                      Cg, C, H, W, radius, eps, workspace, status, S(stream));
  return check_launch("gf_highres_bwd");
}

// ---------------------------------------------------------------------------
// guidance net + loss
// ---------------------------------------------------------------------------
int64_t gn_param_count(int64_t Cin, int64_t Cout, int64_t hidden) {
  return hidden * Cin + 2 + Cout * hidden + Cout;
}

size_t gn_workspace_bytes(int dtype, int64_t B, int64_t Cin, int64_t Cout, int64_t hidden,
                          int64_t H, int64_t W) {
  size_t gen = gfb::gn_ws_bytes(B, hidden);
  if (dtype == GF_F32 && gfb::gn_fast_ok(Cin, Cout, hidden, H * W)) {
    size_t fast = gfb::gn_fast_ws_bytes(B, hidden);
    return fast > gen ? fast : gen;
  }
  return gen;
}

static int check_gn(int dtype, int64_t B, int64_t Cin, int64_t Cout, int64_t hidden, int64_t H,
                    int64_t W, size_t ws_bytes) {
  if (!dtype_ok(dtype)) return fail(GF_ERR_ARG, "bad dtype %d", dtype);
  if (int e = check_dims("x", B, Cin, H, W)) return e;
  if (!gfb::gn_supported(Cin, Cout, hidden))
    return fail(GF_ERR_UNSUPPORTED, "guidance net limits: Cin<=4, Cout<=4, hidden<=64 (got %lld, %lld, %lld)",
                (long long)Cin, (long long)Cout, (long long)hidden);
  size_t need = gn_workspace_bytes(dtype, B, Cin, Cout, hidden, H, W);
  if (ws_bytes < need) return fail(GF_ERR_WORKSPACE, "gn workspace %zu < %zu bytes", ws_bytes, need);
  return GF_OK;
}

int gn_forward(int dtype, const void* x, void* y, const void* params, int64_t B, int64_t Cin,
               int64_t Cout, int64_t hidden, int64_t H, int64_t W, void* workspace,
               size_t workspace_bytes, uint32_t* status, void* stream) {
  if (int e = check_gn(dtype, B, Cin, Cout, hidden, H, W, workspace_bytes)) return e;
  if (!g_force_generic && dtype == GF_F32 && gfb::gn_fast_ok(Cin, Cout, hidden, H * W) &&
      aligned16(x) && aligned16(y)) {
    gfb::gn_fast_forward((const float*)x, (float*)y, (const float*)params, B, hidden, H * W,
                         workspace, status, S(stream));
    return check_launch("gn_forward[fused]");
  }
  if (dtype == GF_F32)
    gfb::gn_forward_impl<float>((const float*)x, (float*)y, (const float*)params, B, Cin, Cout,
                                hidden, H * W, workspace, status, S(stream));
  else
    gfb::gn_forward_impl<double>((const double*)x, (double*)y, (const double*)params, B, Cin,
                                 Cout, hidden, H * W, workspace, status, S(stream));
  return check_launch("gn_forward");
}

int gn_backward(int dtype, const void* x, const void* dy, void* dx, void* dparams, int accumulate,
                const void* params, int64_t B, int64_t Cin, int64_t Cout, int64_t hidden,
                int64_t H, int64_t W, void* workspace, size_t workspace_bytes, uint32_t* status,
                void* stream) {
  if (int e = check_gn(dtype, B, Cin, Cout, hidden, H, W, workspace_bytes)) return e;
  if (!g_force_generic && dtype == GF_F32 && gfb::gn_fast_ok(Cin, Cout, hidden, H * W) &&
      aligned16(x) && aligned16(dy) && aligned16(dx)) {
    gfb::gn_fast_backward((const float*)x, (const float*)dy, (float*)dx, (float*)dparams,
                          accumulate, (const float*)params, B, hidden, H * W, workspace,
                          g_gn_reuse, status, S(stream));
    return check_launch("gn_backward[fused]");
  }
  if (dtype == GF_F32)
    gfb::gn_backward_impl<float>((const float*)x, (const float*)dy, (float*)dx, (float*)dparams,
                                 accumulate, (const float*)params, B, Cin, Cout, hidden, H * W,
                                 workspace, status, S(stream));
  else
    gfb::gn_backward_impl<double>((const double*)x, (const double*)dy, (double*)dx,
                                  (double*)dparams, accumulate, (const double*)params, B, Cin,
                                  Cout, hidden, H * W, workspace, status, S(stream));
  return check_launch("gn_backward");
}

int gn_is_fused(int dtype, int64_t Cin, int64_t Cout, int64_t hidden, int64_t H, int64_t W) {
  return !g_force_generic && dtype == GF_F32 && gfb::gn_fast_ok(Cin, Cout, hidden, H * W) ? 1
                                                                                        : 0;
}

int gn_backward_reuse(int dtype, const void* x, const void* dy, void* dx, void* dparams,
                      int accumulate, const void* params, int64_t B, int64_t Cin, int64_t Cout,
                      int64_t hidden, int64_t H, int64_t W, void* workspace,
                      size_t workspace_bytes, uint32_t* status, void* stream) {
  g_gn_reuse = true;
  const int rc = gn_backward(dtype, x, dy, dx, dparams, accumulate, params, B, Cin, Cout, hidden,
                             H, W, workspace, workspace_bytes, status, stream);
  g_gn_reuse = false;
  return rc;
}

// ---------------------------------------------------------------------------
// k x k (dilated) guidance / core net
// ---------------------------------------------------------------------------
int64_t gnk_param_count(int64_t Cin, int64_t Cout, int64_t hidden, int kernel) {
  return hidden * Cin * kernel * kernel + 2 + Cout * hidden + Cout;
}

size_t gnk_workspace_bytes(int dtype, int64_t B, int64_t Cin, int64_t Cout, int64_t hidden,
                           int kernel, int64_t H, int64_t W) {
  return gfb::gnk_ws_bytes_impl(B, Cin, Cout, hidden, kernel, H * W, dtype == GF_F64 ? 8 : 4);
}

static int check_gnk(int dtype, int64_t B, int64_t Cin, int64_t Cout, int64_t hidden, int kernel,
                     int dilation, int64_t H, int64_t W, size_t ws_bytes) {
  if (!dtype_ok(dtype)) return fail(GF_ERR_ARG, "bad dtype %d", dtype);
  if (int e = check_dims("x", B, Cin, H, W)) return e;
  // ConvLayer.__init__, gf/guidance.py:62-65
  if (kernel < 1 || kernel % 2 == 0)
    return fail(GF_ERR_ARG, "kernel must be odd and >= 1, got %d", kernel);
  if (dilation < 1) return fail(GF_ERR_ARG, "dilation must be >= 1, got %d", dilation);
  if (Cout < 1 || hidden < 1)
    return fail(GF_ERR_ARG, "Cout and hidden must be >= 1 (got %lld, %lld)", (long long)Cout,
                (long long)hidden);
  size_t need = gnk_workspace_bytes(dtype, B, Cin, Cout, hidden, kernel, H, W);
  if (ws_bytes < need) return fail(GF_ERR_WORKSPACE, "gnk workspace %zu < %zu bytes", ws_bytes, need);
  return GF_OK;
}

int gnk_forward(int dtype, const void* x, void* y, const void* params, int64_t B, int64_t Cin,
                int64_t Cout, int64_t hidden, int kernel, int dilation, int64_t H, int64_t W,
                void* workspace, size_t workspace_bytes, uint32_t* status, void* stream) {
  if (int e = check_gnk(dtype, B, Cin, Cout, hidden, kernel, dilation, H, W, workspace_bytes))
    return e;
  if (dtype == GF_F32)
    gfb::gnk_forward_impl<float>((const float*)x, (float*)y, (const float*)params, B, Cin, Cout,
                                 hidden, kernel, dilation, H, W, workspace, status, S(stream));
  else
    gfb::gnk_forward_impl<double>((const double*)x, (double*)y, (const double*)params, B, Cin,
                                  Cout, hidden, kernel, dilation, H, W, workspace, status,
                                  S(stream));
  return check_launch("gnk_forward");
}

int gnk_backward(int dtype, const void* x, const void* dy, void* dx, void* dparams,
                 int accumulate, const void* params, int64_t B, int64_t Cin, int64_t Cout,
                 int64_t hidden, int kernel, int dilation, int64_t H, int64_t W, void* workspace,
                 size_t workspace_bytes, uint32_t* status, void* stream) {
  if (int e = check_gnk(dtype, B, Cin, Cout, hidden, kernel, dilation, H, W, workspace_bytes))
    return e;
  if (dtype == GF_F32)
    gfb::gnk_backward_impl<float>((const float*)x, (const float*)dy, (float*)dx, (float*)dparams,
                                  accumulate, (const float*)params, B, Cin, Cout, hidden, kernel,
                                  dilation, H, W, workspace, status, S(stream));
  else
    gfb::gnk_backward_impl<double>((const double*)x, (const double*)dy, (double*)dx,
                                   (double*)dparams, accumulate, (const double*)params, B, Cin,
                                   Cout, hidden, kernel, dilation, H, W, workspace, status,
                                   S(stream));
  return check_launch("gnk_backward");
}

// ---------------------------------------------------------------------------
// training harness: fixed channel-mean guidance, Adam
// ---------------------------------------------------------------------------
int gf_channel_mean(int dtype, const void* x, void* y, int64_t B, int64_t Cin, int64_t Cout,
                    int64_t H, int64_t W, void* stream) {
  if (!dtype_ok(dtype)) return fail(GF_ERR_ARG, "bad dtype %d", dtype);
  if (int e = check_dims("x", B, Cin, H, W)) return e;
  if (Cout < 1) return fail(GF_ERR_ARG, "Cout must be >= 1, got %lld", (long long)Cout);
  if (dtype == GF_F32)
    gfb::chan_mean_impl<float>((const float*)x, (float*)y, B, Cin, Cout, H * W, S(stream));
  else
    gfb::chan_mean_impl<double>((const double*)x, (double*)y, B, Cin, Cout, H * W, S(stream));
  return check_launch("gf_channel_mean");
}

int gf_channel_mean_adjoint(int dtype, const void* dy, void* dx, int64_t B, int64_t Cin,
                            int64_t Cout, int64_t H, int64_t W, void* stream) {
  if (!dtype_ok(dtype)) return fail(GF_ERR_ARG, "bad dtype %d", dtype);
  if (int e = check_dims("dy", B, Cout, H, W)) return e;
  if (Cin < 1) return fail(GF_ERR_ARG, "Cin must be >= 1, got %lld", (long long)Cin);
  if (dtype == GF_F32)
    gfb::chan_mean_adj_impl<float>((const float*)dy, (float*)dx, B, Cin, Cout, H * W, S(stream));
  else
    gfb::chan_mean_adj_impl<double>((const double*)dy, (double*)dx, B, Cin, Cout, H * W,
                                    S(stream));
  return check_launch("gf_channel_mean_adjoint");
}

int gf_adam_step(int dtype, void* params, const void* grads, void* m, void* v, int64_t n, int step,
                 double lr, uint32_t* status, void* stream) {
  if (!dtype_ok(dtype)) return fail(GF_ERR_ARG, "bad dtype %d", dtype);
  if (n < 0) return fail(GF_ERR_ARG, "n must be >= 0");
  if (step < 1) return fail(GF_ERR_ARG, "step must be >= 1 (1-based), got %d", step);
  // TrainConfig.__post_init__, gf/training.py:43-45
  if (!std::isfinite(lr) || lr < 0.0)
    return fail(GF_ERR_ARG, "learning_rate must be finite and >= 0, got %g", lr);
  if (n == 0) return GF_OK;
  if (dtype == GF_F32)
    gfb::adam_impl<float>((float*)params, (const float*)grads, (float*)m, (float*)v, n, step, lr,
                          0.9, 0.999, 1e-8, status, S(stream));
  else
    gfb::adam_impl<double>((double*)params, (const double*)grads, (double*)m, (double*)v, n, step,
                           lr, 0.9, 0.999, 1e-8, status, S(stream));
  return check_launch("gf_adam_step");
}

size_t gf_mse_workspace_bytes(int64_t B, int64_t C, int64_t H, int64_t W) {
  (void)C;
  (void)H;
  (void)W;
  return gfb::mse_ws_bytes(B);
}

int gf_mse_loss(int dtype, const void* out, const void* target, void* d_out, double* loss,
                int64_t B, int64_t C, int64_t H, int64_t W, void* workspace,
                size_t workspace_bytes, void* stream) {
  if (!dtype_ok(dtype)) return fail(GF_ERR_ARG, "bad dtype %d", dtype);
  if (int e = check_dims("out", B, C, H, W)) return e;
  if (workspace_bytes < gfb::mse_ws_bytes(B))
    return fail(GF_ERR_WORKSPACE, "mse workspace too small");
  if (dtype == GF_F32)
    gfb::mse_impl<float>((const float*)out, (const float*)target, (float*)d_out, loss, B,
                         C * H * W, workspace, S(stream));
  else
    gfb::mse_impl<double>((const double*)out, (const double*)target, (double*)d_out, loss, B,
                          C * H * W, workspace, S(stream));
  return check_launch("gf_mse_loss");
}

// ---- fused training step of the fast layer (forward + MSE + backward) ----
static size_t al256(size_t n) { return (n + 255) / 256 * 256; }

// general-path layout: [joint ws | mse ws | out | d_out]
static size_t joint_mse_generic_bytes(int dtype, int64_t B, int64_t C, int64_t h, int64_t w,
                                      int64_t H, int64_t W) {
  const size_t es = dtype == GF_F64 ? 8 : 4;
  return al256(joint_generic_bytes(B, C, h, w)) + al256(gfb::mse_ws_bytes(B)) +
         2 * al256((size_t)B * C * H * W * es);
}

size_t gf_joint_mse_workspace_bytes(int dtype, int64_t B, int64_t C, int64_t h, int64_t w,
                                    int64_t H, int64_t W, int radius) {
  if (use_fused_joint(dtype, B, C, h, w, H, W, radius))
    return gfb::fused_joint_mse_ws_bytes(B, C, h, w);
  return joint_mse_generic_bytes(dtype, B, C, h, w, H, W);
}

int gf_joint_mse_bwd(int dtype, const void* lr_x, const void* lr_y, const void* hr_x,
                     const void* target, double* loss, void* d_lr_x, void* d_lr_y, void* d_hr_x,
                     int64_t B, int64_t C, int64_t h, int64_t w, int64_t H, int64_t W,
                     int radius, double eps, void* workspace, size_t workspace_bytes,
                     uint32_t* status, void* stream) {
  if (int e = check_joint(dtype, B, C, h, w, H, W, radius, eps)) return e;
  const bool fused = use_fused_joint(dtype, B, C, h, w, H, W, radius) && aligned16(lr_x) &&
                     aligned16(lr_y) && aligned16(hr_x) && aligned16(target) &&
                     aligned16(d_lr_x) && aligned16(d_lr_y) && aligned16(d_hr_x);
  const size_t need = fused ? gfb::fused_joint_mse_ws_bytes(B, C, h, w)
                            : joint_mse_generic_bytes(dtype, B, C, h, w, H, W);
  if (workspace_bytes < need)
    return fail(GF_ERR_WORKSPACE, "joint mse workspace %zu < %zu bytes%s", workspace_bytes, need,
                fused ? "" : " (general kernels)");
  if (fused) {
    gfb::fused_joint_mse_bwd((const float*)lr_x, (const float*)lr_y, (const float*)hr_x,
                             (const float*)target, loss, (float*)d_lr_x, (float*)d_lr_y,
                             (float*)d_hr_x, B, C, h, w, H, W, radius, (float)eps, workspace,
                             status, S(stream));
    return check_launch("gf_joint_mse_bwd[fused]");
  }
  // any other call: forward, MSE and backward through the general kernels,
  // with out and d_out in the workspace
  const size_t es = dtype == GF_F64 ? 8 : 4;
  const size_t jws = al256(joint_generic_bytes(B, C, h, w));
  const size_t mws = al256(gfb::mse_ws_bytes(B));
  const size_t hb = al256((size_t)B * C * H * W * es);
  char* base = (char*)workspace;
  void* out = base + jws + mws;
  void* d_out = base + jws + mws + hb;
  const int old = g_force_generic;
  g_force_generic = 1;  // the fused kernels would reject the unaligned buffers anyway
  int e = gf_joint_fwd(dtype, lr_x, lr_y, hr_x, out, B, C, h, w, H, W, radius, eps, base, jws,
                       status, stream);
  if (!e) e = gf_mse_loss(dtype, out, target, d_out, loss, B, C, H, W, base + jws, mws, stream);
  if (!e)
    e = gf_joint_bwd(dtype, lr_x, lr_y, hr_x, d_out, d_lr_x, d_lr_y, d_hr_x, B, C, h, w, H, W,
                     radius, eps, base, jws, status, stream);
  g_force_generic = old;
  return e;
}

}  // extern "C"

// checks shared with the host-buffer entries (gf_host.cu)
namespace gfb {
int api_check_highres(int dtype, int64_t B, int64_t Cg, int64_t C, int64_t H, int64_t W, int r,
                      double eps) {
  return check_highres(dtype, B, Cg, C, H, W, r, eps);
}
int api_check_joint(int dtype, int64_t B, int64_t C, int64_t h, int64_t w, int64_t H, int64_t W,
                    int r, double eps) {
  return check_joint(dtype, B, C, h, w, H, W, r, eps);
}
int api_fail(int code, const char* what) { return fail(code, "%s", what); }
}  // namespace gfb

