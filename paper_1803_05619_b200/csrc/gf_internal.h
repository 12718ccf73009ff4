// Internal declarations shared by the C-ABI layer and the kernel files.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace gfb {

// ---- per-device launch configuration (gf_launch.cu): SM count and resident
// CTAs per SM of `fn` at this block size / dynamic smem on the CURRENT device;
// also raises the kernel's dynamic shared-memory limit on that device.  Cached
// per (device, fn, threads, smem), thread-safe.
struct LaunchCfg {
  int sms;
  int per_sm;
};
LaunchCfg launch_cfg(const void* fn, int threads, size_t smem);

// ---- generic (any shape / radius / dtype) ----
size_t generic_workspace_bytes(int64_t n_moment_plane_total, int64_t extra_doubles);

template <typename T>
void generic_check_finite(const T* p, int64_t n, uint32_t* status, cudaStream_t s);
template <typename T>
void generic_mean_filter(const T* in, T* out, int64_t P, int64_t h, int64_t w, int r, int adjoint,
                         cudaStream_t s);
template <typename T>
void generic_resize(const T* in, T* out, int64_t P, int64_t h, int64_t w, int64_t oh, int64_t ow,
                    cudaStream_t s);
template <typename T>
void generic_resize_adj(const T* g, T* out, int64_t P, int64_t gh, int64_t gw, int64_t h,
                        int64_t w, cudaStream_t s);
template <typename T>
void generic_joint_fwd(const T* lr_x, const T* lr_y, const T* hr_x, T* out, int64_t B, int64_t C,
                       int64_t h, int64_t w, int64_t H, int64_t W, int r, double eps, void* ws,
                       uint32_t* status, cudaStream_t s);
template <typename T>
void generic_joint_bwd(const T* lr_x, const T* lr_y, const T* hr_x, const T* d_out, T* d_lr_x,
                       T* d_lr_y, T* d_hr_x, int64_t B, int64_t C, int64_t h, int64_t w,
                       int64_t H, int64_t W, int r, double eps, void* ws, uint32_t* status,
                       cudaStream_t s);
template <typename T>
void generic_highres_fwd(const T* guide, const T* src, T* out, int64_t B, int64_t Cg, int64_t C,
                         int64_t H, int64_t W, int r, double eps, void* ws, uint32_t* status,
                         cudaStream_t s);
template <typename T>
void generic_highres_bwd(const T* guide, const T* src, const T* d_out, T* d_guide, T* d_src,
                         int64_t B, int64_t Cg, int64_t C, int64_t H, int64_t W, int r,
                         double eps, void* ws, uint32_t* status, cudaStream_t s);

// ---- guidance net / loss ----
size_t gn_ws_bytes(int64_t B, int64_t hidden);
bool gn_supported(int64_t Cin, int64_t Cout, int64_t hidden);
template <typename T>
void gn_forward_impl(const T* x, T* y, const T* params, int64_t B, int64_t Cin, int64_t Cout,
                     int64_t hidden, int64_t HW, void* ws, uint32_t* status, cudaStream_t s);
template <typename T>
void gn_backward_impl(const T* x, const T* dy, T* dx, T* dparams, int accumulate, const T* params,
                      int64_t B, int64_t Cin, int64_t Cout, int64_t hidden, int64_t HW, void* ws,
                      uint32_t* status, cudaStream_t s);
size_t mse_ws_bytes(int64_t B);
template <typename T>
void mse_impl(const T* out, const T* tgt, T* d_out, double* loss, int64_t B, int64_t per_image,
              void* ws, cudaStream_t s);
// loss = sum_b (sum of partials[b*nblk .. b*nblk+nblk) / per_image) / B, fixed order
void mse_final(const double* partials, double* loss, int64_t B, int nblk, double per_image,
               cudaStream_t s);

// ---- fused fast paths (fp32, NCHW); return false when the shape is not
// covered, in which case the caller takes the generic path ----
// full-resolution forward, register-segment variant for r <= 8 (gf_highres_seg.cu)
bool seg_highres_fwd_ok(int64_t B, int64_t Cg, int64_t C, int64_t H, int64_t W, int r);
void seg_highres_fwd(const float* guide, const float* src, float* out, int64_t B, int64_t Cg,
                     int64_t C, int64_t H, int64_t W, int r, float eps, int mode,
                     uint32_t* status, cudaStream_t s);
bool fused_highres_fwd_ok(int64_t B, int64_t Cg, int64_t C, int64_t H, int64_t W, int r);
void fused_highres_fwd(const float* guide, const float* src, float* out, int64_t B, int64_t Cg,
                       int64_t C, int64_t H, int64_t W, int r, float eps, uint32_t* status,
                       cudaStream_t s);

// joint backward low-res tail, register-segment walk for r <= 4, w % 4 == 0
// (gf_joint_bwd_lr_seg.cu); variant hook: 0 automatic, 1 tile kernel, 2 segment
bool seg_joint_bwd_lr_ok(int64_t h, int64_t w, int r);
void seg_joint_bwd_lr(const float* lr_x, const float* lr_y, const float* db, const float* dA,
                      float* d_lr_x, float* d_lr_y, int64_t P, int64_t h, int64_t w, int r,
                      float eps, int64_t row0, cudaStream_t s);
extern thread_local int g_joint_lr_variant;
extern thread_local int g_joint_fwd_variant;  // r = 8 coefficient chunking (test hook)
extern thread_local int g_joint_mse_variant;
extern thread_local int g_joint_bwd_hr_tile;
extern thread_local int g_joint_bwd_hr_variant;  // 0 single gather pass, 1 tile kernel, 3: 3 CTAs/SM
extern thread_local int g_gn_bwd_variant;  // fused guidance backward: 0 one heavy pass (2 lanes per
                                           // pixel group), 1 two passes, 2 one pass with 4 lanes,
                                           // 3 = 0 capped at 3 CTAs per SM
bool fused_joint_ok(int64_t B, int64_t C, int64_t h, int64_t w, int64_t H, int64_t W, int r);
void fused_joint_fwd(const float* lr_x, const float* lr_y, const float* hr_x, float* out,
                     int64_t B, int64_t C, int64_t h, int64_t w, int64_t H, int64_t W, int r,
                     float eps, uint32_t* status, cudaStream_t s, float* A_tape = nullptr,
                     float* coef_ws = nullptr);  // coef_ws: 2 B C h w floats (A, b of every cell)
// second kernel of the two-kernel forward (gf_joint_apply.cu): out = Up(B) + Up(A) hr_x
void joint_apply(const float* A, const float* B, const float* hr_x, float* out, int64_t P,
                 int64_t h, int64_t w, int64_t H, int64_t W, uint32_t* status, cudaStream_t s);
extern thread_local int g_joint_apply_variant;
// high-res elements (B C H W) from which gf_joint_fwd takes the two-kernel forward
constexpr int64_t kJointSplitElems = (int64_t)48 << 20;
// first kernel of the two-kernel forward, register-segment walk for r <= 8,
// w % 4 == 0 (gf_joint_coeffs_seg.cu): A, b of every low-res cell
bool seg_joint_coeffs_ok(int64_t h, int64_t w, int r);
void seg_joint_coeffs(const float* lr_x, const float* lr_y, float* A, float* B, int64_t P,
                      int64_t h, int64_t w, int r, float eps, uint32_t* status, cudaStream_t s);
extern thread_local int g_joint_coeffs_sw;
// A, b of every low-res cell: the segment walk where it applies, else the
// tile kernel (gf_fused_joint.cu)
void fused_joint_coeffs(const float* lr_x, const float* lr_y, float* A, float* B, int64_t P,
                        int64_t h, int64_t w, int r, float eps, uint32_t* status, cudaStream_t s);
size_t fused_joint_bwd_ws_bytes(int64_t B, int64_t C, int64_t h, int64_t w);
void fused_joint_bwd(const float* lr_x, const float* lr_y, const float* hr_x, const float* d_out,
                     float* d_lr_x, float* d_lr_y, float* d_hr_x, int64_t B, int64_t C,
                     int64_t h, int64_t w, int64_t H, int64_t W, int r, float eps, void* ws,
                     int64_t row0, uint32_t* status, cudaStream_t s,
                     const float* A_tape = nullptr);
// fused training step: forward + MSE + backward (no out / d_out in HBM)
size_t fused_joint_mse_ws_bytes(int64_t B, int64_t C, int64_t h, int64_t w);
void fused_joint_mse_bwd(const float* lr_x, const float* lr_y, const float* hr_x,
                         const float* target, double* loss, float* d_lr_x, float* d_lr_y,
                         float* d_hr_x, int64_t B, int64_t C, int64_t h, int64_t w, int64_t H,
                         int64_t W, int r, float eps, void* ws, uint32_t* status,
                         cudaStream_t s);

}  // namespace gfb

namespace gfb {
// fused fp32 guidance net (Cin = Cout = 3, hidden in {4, 8, 15, 16})
bool gn_fast_ok(int64_t Cin, int64_t Cout, int64_t hidden, int64_t HW);
size_t gn_fast_ws_bytes(int64_t B, int64_t hidden);
void gn_fast_forward(const float* x, float* y, const float* params, int64_t B, int64_t hidden,
                     int64_t HW, void* ws, uint32_t* status, cudaStream_t s);
void gn_fast_backward(const float* x, const float* dy, float* dx, float* dparams, int accumulate,
                      const float* params, int64_t B, int64_t hidden, int64_t HW, void* ws,
                      bool have_fold, uint32_t* status, cudaStream_t s);
// guidance / core net with a k x k dilated first conv (gf_guidance_k.cu)
size_t gnk_ws_bytes_impl(int64_t B, int64_t Cin, int64_t Cout, int64_t hid, int k, int64_t HW,
                         size_t es);
template <typename T>
void gnk_forward_impl(const T* x, T* y, const T* params, int64_t B, int64_t Cin, int64_t Cout,
                      int64_t hid, int k, int d, int64_t H, int64_t W, void* ws, uint32_t* status,
                      cudaStream_t s);
template <typename T>
void gnk_backward_impl(const T* x, const T* dy, T* dx, T* dparams, int accumulate, const T* params,
                       int64_t B, int64_t Cin, int64_t Cout, int64_t hid, int k, int d, int64_t H,
                       int64_t W, void* ws, uint32_t* status, cudaStream_t s);

// training harness (gf_train.cu)
template <typename T>
void chan_mean_impl(const T* x, T* y, int64_t B, int64_t Cin, int64_t Cout, int64_t HW,
                    cudaStream_t s);
template <typename T>
void chan_mean_adj_impl(const T* dy, T* dx, int64_t B, int64_t Cin, int64_t Cout, int64_t HW,
                        cudaStream_t s);
template <typename T>
void adam_impl(T* p, const T* g, T* m, T* v, int64_t n, int step, double lr, double b1, double b2,
               double eps, uint32_t* status, cudaStream_t s);

// full-resolution backward, fp32 streaming window sums (gf_fused_highres_bwd.cu)
bool fused_highres_bwd_ok(int64_t B, int64_t Cg, int64_t C, int64_t H, int64_t W, int r);
size_t fused_highres_bwd_ws_bytes(int64_t B, int64_t Cg, int64_t C, int64_t H, int64_t W);
void fused_highres_bwd(const float* guide, const float* src, const float* d_out, float* d_guide,
                       float* d_src, int64_t B, int64_t Cg, int64_t C, int64_t H, int64_t W, int r,
                       float eps, void* ws, uint32_t* status, cudaStream_t s);

// argument checks / error text of the C ABI (gf_capi.cu), for gf_host.cu
int api_check_highres(int dtype, int64_t B, int64_t Cg, int64_t C, int64_t H, int64_t W, int r,
                      double eps);
int api_check_joint(int dtype, int64_t B, int64_t C, int64_t h, int64_t w, int64_t H, int64_t W,
                    int r, double eps);
int api_fail(int code, const char* what);

}  // namespace gfb
