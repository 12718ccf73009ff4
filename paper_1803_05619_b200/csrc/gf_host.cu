// Host-buffer entry points (include/gf_b200.h, "host" section): the
// reference's layer calls take host images (numpy, gf/guided.py:152, :198)
// and return host images.  These entries keep that contract and hide the PCIe
// traffic behind the kernels: the batch is streamed chunk by chunk (one plane;
// one image when a 1-channel guide drives C planes) through two device slots
// with three streams,
//
//     copy-in  (chunk b+1)  ||  kernel (chunk b)  ||  copy-out (chunk b-1)
//
// so a call costs about max(total H2D, total D2H) + one chunk of kernel and
// copy, not their sum.  Host buffers should be page-locked for the copies to
// overlap (pageable memory still gives correct results).  The caller owns the
// device workspace (size from *_host_workspace_bytes); the streams and events
// are created once per host thread and device.
#include <cuda_runtime.h>

#include "../../include/gf_b200.h"
#include "gf_internal.h"

namespace {

struct Pipe {
  cudaStream_t in = nullptr, run = nullptr, out = nullptr;
  cudaEvent_t in_done[2] = {nullptr, nullptr}, run_done[2] = {nullptr, nullptr},
              out_done[2] = {nullptr, nullptr};
  bool ok = true;
  Pipe() {
    ok &= cudaStreamCreateWithFlags(&in, cudaStreamNonBlocking) == cudaSuccess;
    ok &= cudaStreamCreateWithFlags(&run, cudaStreamNonBlocking) == cudaSuccess;
    ok &= cudaStreamCreateWithFlags(&out, cudaStreamNonBlocking) == cudaSuccess;
    for (int s = 0; s < 2; ++s) {
      ok &= cudaEventCreateWithFlags(&in_done[s], cudaEventDisableTiming) == cudaSuccess;
      ok &= cudaEventCreateWithFlags(&run_done[s], cudaEventDisableTiming) == cudaSuccess;
      ok &= cudaEventCreateWithFlags(&out_done[s], cudaEventDisableTiming) == cudaSuccess;
    }
  }
};

// one set of streams / events per (host thread, device), created on first
// use and kept (a call then costs no driver object creation)
Pipe* pipe_for_current_device() {
  constexpr int kMaxDev = 64;
  thread_local Pipe* pipes[kMaxDev] = {nullptr};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return nullptr;
  if (!pipes[dev]) pipes[dev] = new Pipe();
  return pipes[dev];
}

size_t up256(size_t n) { return (n + 255) / 256 * 256; }
size_t esize(int dtype) { return dtype == GF_F64 ? 8 : 4; }

// Copies of `nin` inputs per chunk (chunk b: in_bytes[i] at host in[i] +
// b * in_bytes[i]) and one output; `launch` runs the device entry on the slot
// buffers.  Returns a GF_* code; *status gets the OR of the device bits.
template <class Launch>
int run_pipeline(int64_t B, int nin, const void* const* in, const size_t* in_bytes, void* out,
                 size_t out_bytes, char* ws, size_t slot_bytes, uint32_t* status_dev,
                 uint32_t* status_host, Launch launch) {
  Pipe* pp = pipe_for_current_device();
  if (!pp || !pp->ok) return gfb::api_fail(GF_ERR_CUDA, "stream/event creation failed");
  Pipe& p = *pp;
  if (cudaMemsetAsync(status_dev, 0, sizeof(uint32_t), p.run) != cudaSuccess)
    return gfb::api_fail(GF_ERR_CUDA, cudaGetErrorString(cudaGetLastError()));
  for (int64_t b = 0; b < B; ++b) {
    const int s = (int)(b & 1);
    char* slot = ws + s * slot_bytes;
    // slot inputs are free once the kernel of image b-2 ran
    if (b >= 2) cudaStreamWaitEvent(p.in, p.run_done[s], 0);
    size_t off = 0;
    const void* dev_in[4];
    for (int i = 0; i < nin; ++i) {
      cudaMemcpyAsync(slot + off, (const char*)in[i] + b * in_bytes[i], in_bytes[i],
                      cudaMemcpyHostToDevice, p.in);
      dev_in[i] = slot + off;
      off += up256(in_bytes[i]);
    }
    void* dev_out = slot + off;
    cudaEventRecord(p.in_done[s], p.in);
    cudaStreamWaitEvent(p.run, p.in_done[s], 0);
    if (b >= 2) cudaStreamWaitEvent(p.run, p.out_done[s], 0);  // slot output copied out
    if (int e = launch(dev_in, dev_out, p.run)) {
      cudaStreamSynchronize(p.run);
      return e;
    }
    cudaEventRecord(p.run_done[s], p.run);
    cudaStreamWaitEvent(p.out, p.run_done[s], 0);
    cudaMemcpyAsync((char*)out + b * out_bytes, dev_out, out_bytes, cudaMemcpyDeviceToHost, p.out);
    cudaEventRecord(p.out_done[s], p.out);
  }
  cudaStreamWaitEvent(p.out, p.run_done[0], 0);  // status written by every kernel
  cudaStreamWaitEvent(p.out, p.run_done[1], 0);
  uint32_t st = 0;
  cudaMemcpyAsync(&st, status_dev, sizeof(uint32_t), cudaMemcpyDeviceToHost, p.out);
  cudaError_t e1 = cudaStreamSynchronize(p.out), e2 = cudaStreamSynchronize(p.run);
  cudaError_t e3 = cudaGetLastError();
  if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess)
    return gfb::api_fail(GF_ERR_CUDA, cudaGetErrorString(e1 != cudaSuccess ? e1
                                                         : e2 != cudaSuccess ? e2 : e3));
  if (status_host) *status_host = st;
  return GF_OK;
}

}  // namespace

extern "C" {

// ---- full-resolution layer -------------------------------------------------
// chunk = one plane (guide plane c drives src plane c), or one image when a
// 1-channel guide is broadcast over the C source planes
size_t gf_highres_host_workspace_bytes(int dtype, int64_t Cg, int64_t C, int64_t H, int64_t W,
                                       int radius) {
  const size_t plane = (size_t)H * W * esize(dtype);
  const int64_t cc = Cg == C ? 1 : C;  // source planes per chunk
  const size_t slot = up256(plane) + 2 * up256(cc * plane);
  return 2 * slot + up256(gf_highres_workspace_bytes(dtype, 1, 1, cc, H, W, radius)) + 256;
}

int gf_highres_fwd_host(int dtype, const void* guide, const void* src, void* out, int64_t B,
                        int64_t Cg, int64_t C, int64_t H, int64_t W, int radius, double eps,
                        void* workspace, size_t workspace_bytes, uint32_t* status) {
  if (int e = gfb::api_check_highres(dtype, B, Cg, C, H, W, radius, eps)) return e;
  if (!guide || !src || !out) return gfb::api_fail(GF_ERR_ARG, "null host pointer");
  const size_t need = gf_highres_host_workspace_bytes(dtype, Cg, C, H, W, radius);
  if (workspace_bytes < need) return gfb::api_fail(GF_ERR_WORKSPACE, "host workspace too small");
  const size_t plane = (size_t)H * W * esize(dtype);
  const int64_t cc = Cg == C ? 1 : C;
  const int64_t chunks = Cg == C ? B * C : B;
  const size_t in_bytes[2] = {plane, cc * plane};
  const size_t slot = up256(plane) + 2 * up256(cc * plane);
  char* ws = (char*)workspace;
  char* gws = ws + 2 * slot;
  const size_t gws_bytes = gf_highres_workspace_bytes(dtype, 1, 1, cc, H, W, radius);
  uint32_t* st_dev = (uint32_t*)(gws + up256(gws_bytes));
  const void* ins[2] = {guide, src};
  return run_pipeline(chunks, 2, ins, in_bytes, out, cc * plane, ws, slot, st_dev, status,
                      [&](const void* const* d, void* o, cudaStream_t s) {
                        return gf_highres_fwd(dtype, d[0], d[1], o, 1, 1, cc, H, W, radius, eps,
                                              gws, gws_bytes, st_dev, s);
                      });
}

// ---- joint (fast) layer ----------------------------------------------------
// chunk = one plane (the layer is independent per plane)
size_t gf_joint_host_workspace_bytes(int dtype, int64_t C, int64_t h, int64_t w, int64_t H,
                                     int64_t W, int radius) {
  (void)C;
  const size_t lo = (size_t)h * w * esize(dtype), hi = (size_t)H * W * esize(dtype);
  const size_t slot = 2 * up256(lo) + 2 * up256(hi);
  return 2 * slot + up256(gf_joint_workspace_bytes(dtype, 1, 1, h, w, H, W, radius)) + 256;
}

int gf_joint_fwd_host(int dtype, const void* lr_x, const void* lr_y, const void* hr_x, void* out,
                      int64_t B, int64_t C, int64_t h, int64_t w, int64_t H, int64_t W,
                      int radius, double eps, void* workspace, size_t workspace_bytes,
                      uint32_t* status) {
  if (int e = gfb::api_check_joint(dtype, B, C, h, w, H, W, radius, eps)) return e;
  if (!lr_x || !lr_y || !hr_x || !out) return gfb::api_fail(GF_ERR_ARG, "null host pointer");
  const size_t need = gf_joint_host_workspace_bytes(dtype, C, h, w, H, W, radius);
  if (workspace_bytes < need) return gfb::api_fail(GF_ERR_WORKSPACE, "host workspace too small");
  const size_t lo = (size_t)h * w * esize(dtype), hi = (size_t)H * W * esize(dtype);
  const size_t in_bytes[3] = {lo, lo, hi};
  const size_t slot = 2 * up256(lo) + 2 * up256(hi);
  char* ws = (char*)workspace;
  char* gws = ws + 2 * slot;
  const size_t gws_bytes = gf_joint_workspace_bytes(dtype, 1, 1, h, w, H, W, radius);
  uint32_t* st_dev = (uint32_t*)(gws + up256(gws_bytes));
  const void* ins[3] = {lr_x, lr_y, hr_x};
  return run_pipeline(B * C, 3, ins, in_bytes, out, hi, ws, slot, st_dev, status,
                      [&](const void* const* d, void* o, cudaStream_t s) {
                        return gf_joint_fwd(dtype, d[0], d[1], d[2], o, 1, 1, h, w, H, W, radius,
                                            eps, gws, gws_bytes, st_dev, s);
                      });
}

}  // extern "C"
