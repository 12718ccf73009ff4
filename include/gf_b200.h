/*
 * gf_b200.h -- C ABI of the B200-native guided-filter layer (arXiv 1803.05619).
 *
 * Drop-in boundary for the reference package's layer path
 * (/root/reference/pkg/src/guidedfilter, "gf/" below).  Every entry point is
 * plain C: raw device pointers, 64-bit sizes, a dtype tag and a CUDA stream
 * handle (cudaStream_t passed as void*; NULL = legacy default stream).  No
 * torch types cross this boundary; the library never allocates or frees:
 * callers pass every output and a workspace of the size the matching
 * *_workspace_bytes() query returns.  All launches are asynchronous on the
 * given stream; the library keeps no global state besides a thread-local
 * error string, so it is reentrant.
 *
 * Layout: every image tensor is contiguous NCHW, i.e. B*C planes of H rows
 * of W elements (index ((b*C + c)*H + y)*W + x).  The reference works on one
 * HWC float64 image at a time (gf/tensor.py:1-11); its (h, w, c) image is
 * the B=1 case after a transpose, which the Python mirror does.
 *
 * dtype: GF_F32 (float) is the production path; GF_F64 (double) reproduces
 * the reference's float64 arithmetic to its own 1e-10 test bars.
 *
 * Errors: the int return is GF_OK or a GF_ERR_* code (argument/shape errors
 * mirror the reference's ValueError sites; gf_last_error() has the text).
 * Data-dependent errors are reported through a caller-owned DEVICE uint32
 * status word that kernels OR bits into (GF_STATUS_*); the caller reads it
 * back when it wants the reference's synchronous exception semantics.
 */
#ifndef GF_B200_H
#define GF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { GF_F32 = 0, GF_F64 = 1 };

enum {
  GF_OK = 0,
  GF_ERR_ARG = 1,         /* bad shape / radius / eps / dtype  -> ValueError      */
  GF_ERR_WORKSPACE = 2,   /* workspace smaller than *_workspace_bytes()           */
  GF_ERR_CUDA = 3,        /* launch failure (gf_last_error has cudaGetErrorString) */
  GF_ERR_UNSUPPORTED = 4  /* a size beyond the library's limits                   */
};

/* Device status bits.  Priority when raising: INPUT, then DEGENERATE, then
 * OUTPUT -- the order the reference checks them (gf/guided.py:156-180). */
enum {
  GF_STATUS_NONFINITE_INPUT = 1u,   /* validate(..., finite=True), gf/tensor.py:39-40 */
  GF_STATUS_NONFINITE_OUTPUT = 2u,  /* gf/guided.py:179-180 / :216-217                */
  GF_STATUS_DEGENERATE = 4u         /* DegenerateWindowError, gf/guided.py:142-146    */
};

int gf_version(void);              /* 100 * major + minor                    */
const char* gf_last_error(void);   /* thread-local text of the last failure  */
int gf_sm_count(void);             /* SMs of the current device (for sizing) */

/* Scan n elements for NaN/Inf and OR GF_STATUS_NONFINITE_INPUT into status.
 * The fused kernels do not test every input element (a non-finite input
 * always makes the output at its own pixel non-finite); a caller that sees
 * GF_STATUS_NONFINITE_OUTPUT or GF_STATUS_DEGENERATE scans the inputs with
 * this to restore the reference's check order (inputs first,
 * gf/guided.py:156-158). */
int gf_check_finite(int dtype, const void* data, int64_t n, uint32_t* status, void* stream);

/* ---- linear operators: gf/filters.py (the reference's _kernels seam) ----
 * P planes of (h, w).  No workspace. */

/* gf/filters.py:96-103 mean_filter (and _kernels.box_sum(normalize=True),
 * gf/_kernels.py:71-80): clamped window mean, true-count normalised. */
int gf_mean_filter(int dtype, const void* in, void* out, int64_t planes, int64_t h,
                   int64_t w, int radius, void* stream);

/* gf/filters.py:106-116 mean_filter_adjoint: box_sum(g / N). */
int gf_mean_filter_adjoint(int dtype, const void* g, void* out, int64_t planes, int64_t h,
                           int64_t w, int radius, void* stream);

/* gf/filters.py:134-156 bilinear_resize (gf/_kernels.py:83-101): half-pixel
 * centres, edge clamp, rows then columns.  in (h, w) -> out (out_h, out_w). */
int gf_bilinear_resize(int dtype, const void* in, void* out, int64_t planes, int64_t h,
                       int64_t w, int64_t out_h, int64_t out_w, void* stream);

/* gf/filters.py:168-188 bilinear_resize_adjoint: exact transpose, computed
 * as a deterministic gather.  g (g_h, g_w) -> out (in_h, in_w). */
int gf_bilinear_resize_adjoint(int dtype, const void* g, void* out, int64_t planes,
                               int64_t g_h, int64_t g_w, int64_t in_h, int64_t in_w,
                               void* stream);

/* ---- the fast (joint-upsampling) layer: gf/guided.py:152-195, :267-283 ----
 * lr_x = guide_lo, lr_y = src_lo: (B, C, h, w); hr_x = guide_hi: (B, C, H, W)
 * with H >= h, W >= w (any ratio).  out: (B, C, H, W).  NO smoothing of A, b
 * on this path (gf/guided.py:170-178).
 * gf_joint_fwd on the fp32 fast path (factor 4, 16-byte aligned buffers): calls
 * of gf_joint_split_threshold() or more high-res elements run as the two
 * kernels gf_joint_coeffs + gf_joint_apply with the coefficients of every
 * low-res cell in `workspace` (gf_joint_workspace_bytes; a NULL or smaller
 * workspace keeps the one-kernel tile forward, which needs none); smaller
 * calls as one kernel.  Both agree to fp32 rounding of the coefficients. */
size_t gf_joint_workspace_bytes(int dtype, int64_t B, int64_t C, int64_t h, int64_t w,
                                int64_t H, int64_t W, int radius);

int gf_joint_fwd(int dtype, const void* lr_x, const void* lr_y, const void* hr_x, void* out,
                 int64_t B, int64_t C, int64_t h, int64_t w, int64_t H, int64_t W, int radius,
                 double eps, void* workspace, size_t workspace_bytes, uint32_t* status,
                 void* stream);

/* Gradients of dot(d_out, out): d_lr_y = d_src, d_lr_x = d_guide_lo,
 * d_hr_x = d_guide_hi (gf/guided.py:267-283).  The lr moments are recomputed
 * from lr_x, lr_y (the tape keeps input references only). */
int gf_joint_bwd(int dtype, const void* lr_x, const void* lr_y, const void* hr_x,
                 const void* d_out, void* d_lr_x, void* d_lr_y, void* d_hr_x, int64_t B,
                 int64_t C, int64_t h, int64_t w, int64_t H, int64_t W, int radius, double eps,
                 void* workspace, size_t workspace_bytes, uint32_t* status, void* stream);

/* gf_joint_bwd on a ROW BAND of a larger image (multi-GPU config 4b, SURVEY
 * 8e): the inputs are the band's aligned crop and `row0` is the FULL image's
 * low-res row index of the crop's first row.  The kernels cut their row
 * pieces and shift constants at full-image rows, so with row0 a multiple of
 * 16 (paper_1803_05619_b200.sharding.row_bands aligns crops so) every owned
 * row of every output is bitwise equal to the 1-GPU call on the whole image.
 * row0 = 0 is gf_joint_bwd. */
int gf_joint_bwd_band(int dtype, const void* lr_x, const void* lr_y, const void* hr_x,
                      const void* d_out, void* d_lr_x, void* d_lr_y, void* d_hr_x, int64_t B,
                      int64_t C, int64_t h, int64_t w, int64_t H, int64_t W, int radius,
                      double eps, int64_t row0, void* workspace, size_t workspace_bytes,
                      uint32_t* status, void* stream);

/* The two kernels of the fast forward, callable on their own (fp32 calls
 * gf_joint_is_fused accepts, 16-byte aligned buffers; else
 * GF_ERR_UNSUPPORTED).  gf_joint_coeffs: the window moments and the slope
 * A = cov / (var + eps) and intercept b = mean_y - A mean_x of EVERY low-res
 * cell (gf/guided.py:136-149, :170-173) -> slope_lo, intercept_lo (B, C, h, w).
 * gf_joint_apply: out = Up(intercept_lo) + Up(slope_lo) * hr_x, the bilinear
 * resize of both and the affine combine in one pass over hr_x
 * (gf/guided.py:174-178, gf/_kernels.py:104-124).  gf_joint_fwd on large
 * images is exactly this pair with the coefficients in its workspace. */
/* B*C*H*W from which gf_joint_fwd / gf_joint_fwd_tape (given a workspace)
 * run as this pair.  gf_joint_fwd_mode sets the choice for the CALLING THREAD
 * and returns the old one: 0 by size, 1 the one-kernel tile forward, 2 the
 * two-kernel forward (a row band passes the choice of its full image, so
 * band results stay bitwise the image's). */
int64_t gf_joint_split_threshold(void);
int gf_joint_fwd_mode(int mode);
int gf_joint_coeffs(int dtype, const void* lr_x, const void* lr_y, void* slope_lo,
                    void* intercept_lo, int64_t B, int64_t C, int64_t h, int64_t w, int radius,
                    double eps, uint32_t* status, void* stream);
int gf_joint_apply(int dtype, const void* slope_lo, const void* intercept_lo, const void* hr_x,
                   void* out, int64_t B, int64_t C, int64_t h, int64_t w, int64_t H, int64_t W,
                   uint32_t* status, void* stream);

/* Tape variants of the fast path (calls gf_joint_is_fused accepts, 16-byte
 * aligned buffers; anything else returns GF_ERR_UNSUPPORTED and computes
 * nothing -- use gf_joint_fwd / gf_joint_bwd).  gf_joint_fwd_tape also writes
 * the low-res slope A = cov / (var + eps) of every cell to `slope_lo`
 * (B, C, h, w): the reference's tape keeps it (gf/guided.py:147, :181-194).
 * gf_joint_bwd_tape reads it back, so its high-res pass streams hr_x and
 * d_out without recomputing window moments (the low-res tail still does);
 * row0 as gf_joint_bwd_band.  Results equal gf_joint_bwd's to fp32
 * rounding (a tile's halo slopes come from the neighbouring tile).
 * gf_joint_fwd_tape's workspace (gf_joint_workspace_bytes; may be NULL) lets
 * large images take the two-kernel forward, the intercepts in the workspace. */
int gf_joint_fwd_tape(int dtype, const void* lr_x, const void* lr_y, const void* hr_x, void* out,
                      void* slope_lo, int64_t B, int64_t C, int64_t h, int64_t w, int64_t H,
                      int64_t W, int radius, double eps, void* workspace, size_t workspace_bytes,
                      uint32_t* status, void* stream);

int gf_joint_bwd_tape(int dtype, const void* lr_x, const void* lr_y, const void* hr_x,
                      const void* slope_lo, const void* d_out, void* d_lr_x, void* d_lr_y,
                      void* d_hr_x, int64_t B, int64_t C, int64_t h, int64_t w, int64_t H,
                      int64_t W, int radius, double eps, int64_t row0, void* workspace,
                      size_t workspace_bytes, uint32_t* status, void* stream);

/* ---- the full-resolution layer: gf/guided.py:198-233, :284-295 ----
 * guide: (B, Cg, H, W) with Cg == C or Cg == 1 (a 1-channel guide is
 * broadcast over the C source channels, BASELINE config 1); src, out:
 * (B, C, H, W).  A and b are re-smoothed by the mean filter. */
size_t gf_highres_workspace_bytes(int dtype, int64_t B, int64_t Cg, int64_t C, int64_t H,
                                  int64_t W, int radius);

int gf_highres_fwd(int dtype, const void* guide, const void* src, void* out, int64_t B,
                   int64_t Cg, int64_t C, int64_t H, int64_t W, int radius, double eps,
                   void* workspace, size_t workspace_bytes, uint32_t* status, void* stream);

/* d_guide: (B, Cg, H, W) -- for Cg == 1 the sum over the C broadcast copies. */
int gf_highres_bwd(int dtype, const void* guide, const void* src, const void* d_out,
                   void* d_guide, void* d_src, int64_t B, int64_t Cg, int64_t C, int64_t H,
                   int64_t W, int radius, double eps, void* workspace, size_t workspace_bytes,
                   uint32_t* status, void* stream);

/* ---- 1x1 guidance net F: gf/guidance.py:184-224 ----
 * conv1 (hidden x Cin, no bias) -> AdaptiveNorm (scalar gain, norm_gain;
 * per-image per-channel population statistics, var floor 1e-5) -> leaky
 * ReLU 0.2 -> conv2 (Cout x hidden) + bias.  Parameters are one packed
 * device array of dtype, in the reference's parameters() order:
 *   conv1.weight[hidden*Cin], norm.gain[1], norm.norm_gain[1],
 *   conv2.weight[Cout*hidden], conv2.bias[Cout]
 * (gn_param_count() values).  x: (B, Cin, H, W); y: (B, Cout, H, W).
 * Statistics are per image (the reference has no batch dimension). */
int64_t gn_param_count(int64_t Cin, int64_t Cout, int64_t hidden);

size_t gn_workspace_bytes(int dtype, int64_t B, int64_t Cin, int64_t Cout, int64_t hidden,
                          int64_t H, int64_t W);

int gn_forward(int dtype, const void* x, void* y, const void* params, int64_t B, int64_t Cin,
               int64_t Cout, int64_t hidden, int64_t H, int64_t W, void* workspace,
               size_t workspace_bytes, uint32_t* status, void* stream);

/* dx: (B, Cin, H, W).  dparams (packed like params) is OVERWRITTEN with the
 * gradient summed over the batch when accumulate == 0, or added to when
 * accumulate != 0 (the two call sites of GuidedUpsampler.backward,
 * gf/training.py:168-177, accumulate low-res first). */
int gn_backward(int dtype, const void* x, const void* dy, void* dx, void* dparams,
                int accumulate, const void* params, int64_t B, int64_t Cin, int64_t Cout,
                int64_t hidden, int64_t H, int64_t W, void* workspace, size_t workspace_bytes,
                uint32_t* status, void* stream);

/* 1 when gn_forward / gn_backward of this shape take the fused fp32 kernels
 * (for 16-byte aligned x, y, dy, dx), else 0. */
int gn_is_fused(int dtype, int64_t Cin, int64_t Cout, int64_t hidden, int64_t H, int64_t W);

/* gn_backward with `workspace` being the one gn_forward filled for this x and
 * these params (same stream, parameters unchanged since): on the fused path
 * the per-image input statistics and folded AdaptiveNorm constants are read
 * from it instead of recomputed (the forward already checked x is finite).
 * Elsewhere identical to gn_backward. */
int gn_backward_reuse(int dtype, const void* x, const void* dy, void* dx, void* dparams,
                      int accumulate, const void* params, int64_t B, int64_t Cin, int64_t Cout,
                      int64_t hidden, int64_t H, int64_t W, void* workspace,
                      size_t workspace_bytes, uint32_t* status, void* stream);

/* ---- host-buffer entries: the reference's call shape (host images in, host
 * image out; gf/guided.py:152 forward_joint, :198 forward_highres) ----
 * Synchronous: the calls return when `out` (HOST memory) is written.  The
 * batch streams through the device chunk by chunk -- one plane, or one image
 * when a 1-channel guide drives C planes (copy-in of chunk b+1, kernel of
 * chunk b and copy-out of chunk b-1 overlap on three streams kept per host
 * thread and device), so page-locked host buffers make the call cost
 * ~max(H2D, D2H) of the whole batch.  `workspace` is DEVICE memory of *_host_workspace_bytes(); `status`
 * is a HOST uint32 receiving the OR of the GF_STATUS_* bits of all images. */
size_t gf_highres_host_workspace_bytes(int dtype, int64_t Cg, int64_t C, int64_t H, int64_t W,
                                       int radius);

int gf_highres_fwd_host(int dtype, const void* guide, const void* src, void* out, int64_t B,
                        int64_t Cg, int64_t C, int64_t H, int64_t W, int radius, double eps,
                        void* workspace, size_t workspace_bytes, uint32_t* status);

size_t gf_joint_host_workspace_bytes(int dtype, int64_t C, int64_t h, int64_t w, int64_t H,
                                     int64_t W, int radius);

int gf_joint_fwd_host(int dtype, const void* lr_x, const void* lr_y, const void* hr_x, void* out,
                      int64_t B, int64_t C, int64_t h, int64_t w, int64_t H, int64_t W,
                      int radius, double eps, void* workspace, size_t workspace_bytes,
                      uint32_t* status);

/* Forward AND backward of the joint layer on host images, the call a
 * training framework makes with host tensors (gf/guided.py:152 forward_joint
 * then :267 backward with d_out): per plane, lr_x, lr_y, hr_x and d_out are
 * copied in, gf_joint_fwd + gf_joint_bwd run, and out, d_lr_x, d_lr_y,
 * d_hr_x are copied out, pipelined as above. */
size_t gf_joint_fwd_bwd_host_workspace_bytes(int dtype, int64_t C, int64_t h, int64_t w,
                                             int64_t H, int64_t W, int radius);

int gf_joint_fwd_bwd_host(int dtype, const void* lr_x, const void* lr_y, const void* hr_x,
                          const void* d_out, void* out, void* d_lr_x, void* d_lr_y, void* d_hr_x,
                          int64_t B, int64_t C, int64_t h, int64_t w, int64_t H, int64_t W,
                          int radius, double eps, void* workspace, size_t workspace_bytes,
                          uint32_t* status);

/* ---- guidance / core net with a k x k dilated first convolution ----
 * gf/guidance.py:184-224 with ConvLayer(kernel=k, dilation=d) (:52-124):
 * GuidedUpsampler's low-res core net C_l (gf/training.py:186-207, k = 3).
 * Same layer chain and packed parameter order as gn_*, with conv1.weight
 * (hidden, Cin, k, k) row-major: gnk_param_count() values.  kernel odd >= 1,
 * dilation >= 1, zero "same" padding (k-1)*d/2.  kernel == 1 equals gn_*. */
int64_t gnk_param_count(int64_t Cin, int64_t Cout, int64_t hidden, int kernel);

size_t gnk_workspace_bytes(int dtype, int64_t B, int64_t Cin, int64_t Cout, int64_t hidden,
                           int kernel, int64_t H, int64_t W);

int gnk_forward(int dtype, const void* x, void* y, const void* params, int64_t B, int64_t Cin,
                int64_t Cout, int64_t hidden, int kernel, int dilation, int64_t H, int64_t W,
                void* workspace, size_t workspace_bytes, uint32_t* status, void* stream);

int gnk_backward(int dtype, const void* x, const void* dy, void* dx, void* dparams,
                 int accumulate, const void* params, int64_t B, int64_t Cin, int64_t Cout,
                 int64_t hidden, int kernel, int dilation, int64_t H, int64_t W, void* workspace,
                 size_t workspace_bytes, uint32_t* status, void* stream);

/* ---- standalone guidance layers: ConvLayer (gf/guidance.py:52-124) and
 * AdaptiveNorm (gf/guidance.py:134-173) -- the reference's layer objects
 * (GuidanceNet.conv1 / .norm / .conv2), computed in float64 internally.
 * x: (B, Cin, H, W); weight (Cout, Cin, k, k); bias (Cout) or NULL; "same"
 * zero padding (k-1)*dilation/2.  Parameter gradients are SUMMED over the
 * batch (each image is one reference call) and overwritten.  gain,
 * norm_gain and their gradients are single device scalars of dtype;
 * statistics are per image and channel (population variance, floor 1e-5). */
int gf_conv2d_fwd(int dtype, const void* x, const void* weight, const void* bias, void* y,
                  int64_t B, int64_t Cin, int64_t Cout, int64_t H, int64_t W, int kernel,
                  int dilation, void* stream);

int gf_conv2d_bwd(int dtype, const void* x, const void* weight, const void* dy, void* dx,
                  void* d_weight, void* d_bias, int64_t B, int64_t Cin, int64_t Cout, int64_t H,
                  int64_t W, int kernel, int dilation, void* stream);

size_t gf_adaptive_norm_workspace_bytes(int64_t B, int64_t C);

int gf_adaptive_norm_fwd(int dtype, const void* x, void* y, const void* gain,
                         const void* norm_gain, int64_t B, int64_t C, int64_t H, int64_t W,
                         void* workspace, size_t workspace_bytes, void* stream);

int gf_adaptive_norm_bwd(int dtype, const void* x, const void* dy, void* dx, void* d_gain,
                         void* d_norm_gain, const void* gain, const void* norm_gain, int64_t B,
                         int64_t C, int64_t H, int64_t W, void* workspace,
                         size_t workspace_bytes, void* stream);

/* ---- 8-bit images for the upsample CLI (gf/fileio.py:104-141) ----
 * unpack: interleaved (H, W, C) uint8 -> (1, C, H, W) value / 255;
 * pack: (1, C, H, W) -> (H, W, C) uint8 rint(clip(v, 0, 1) * 255) (round
 * half to even).  Device pointers; asynchronous on `stream`. */
int gf_image_unpack_u8(int dtype, const uint8_t* hwc, void* nchw, int64_t H, int64_t W,
                       int64_t C, void* stream);

int gf_image_pack_u8(int dtype, const void* nchw, uint8_t* hwc, int64_t H, int64_t W, int64_t C,
                     void* stream);

/* ---- FixedChannelMeanGuidance (gf/guidance.py:227-255) ----
 * y (B, Cout, H, W): every channel = mean over the Cin channels of x;
 * adjoint dx (B, Cin, H, W) = (sum over Cout of dy) / Cin. */
int gf_channel_mean(int dtype, const void* x, void* y, int64_t B, int64_t Cin, int64_t Cout,
                    int64_t H, int64_t W, void* stream);

int gf_channel_mean_adjoint(int dtype, const void* dy, void* dx, int64_t B, int64_t Cin,
                            int64_t Cout, int64_t H, int64_t W, void* stream);

/* ---- adam_step (gf/training.py:66-90) on one packed vector of n values ----
 * In place: m = b1 m + (1-b1) g; v = b2 v + (1-b2) g^2; p -= lr mhat /
 * (sqrt(vhat) + 1e-8) with b1 = 0.9, b2 = 0.999 and the bias corrections of
 * the 1-based step t.  A non-finite gradient sets GF_STATUS_NONFINITE_INPUT
 * (the reference's TrainingError) and leaves that element unchanged. */
int gf_adam_step(int dtype, void* params, const void* grads, void* m, void* v, int64_t n,
                 int step, double lr, uint32_t* status, void* stream);

/* ---- mse_loss: gf/training.py:93-101 (batch-mean variant of config 2) ----
 * loss = mean over the batch of per-image mean((out - target)^2); d_out =
 * 2 (out - target) / (C*H*W) / B.  loss is one device double. */
int gf_mse_loss(int dtype, const void* out, const void* target, void* d_out, double* loss,
                int64_t B, int64_t C, int64_t H, int64_t W, void* workspace,
                size_t workspace_bytes, void* stream);

/* Fused training step of the fast layer: the loss and gradients that
 * gf/training.py:230-235 (eval_and_grads) takes from forward_joint ->
 * mse_loss -> backward, i.e. loss = mean over images of mean((out -
 * target)^2) (gf/training.py:93-101) and its gradients w.r.t. lr_x (the
 * guide_lo), lr_y (src_lo) and hr_x (guide_hi), in one hr pass: out and
 * d_out = 2 (out - target) / (C H W B) never reach HBM.  target: (B, C, H, W);
 * loss: one float64 on the device. */
size_t gf_joint_mse_workspace_bytes(int dtype, int64_t B, int64_t C, int64_t h, int64_t w,
                                    int64_t H, int64_t W, int radius);

int gf_joint_mse_bwd(int dtype, const void* lr_x, const void* lr_y, const void* hr_x,
                     const void* target, double* loss, void* d_lr_x, void* d_lr_y, void* d_hr_x,
                     int64_t B, int64_t C, int64_t h, int64_t w, int64_t H, int64_t W,
                     int radius, double eps, void* workspace, size_t workspace_bytes,
                     uint32_t* status, void* stream);

size_t gf_mse_workspace_bytes(int64_t B, int64_t C, int64_t H, int64_t W);

#ifdef __cplusplus
}
#endif

#endif /* GF_B200_H */
