// Host-buffer entry points (include/gf_b200.h, "host" section): the
// reference's layer calls take host images (numpy, gf/guided.py:152, :198)
// and return host images.  These entries keep that contract and hide the PCIe
// traffic behind the kernels: the batch is streamed plane by plane through two
// device slots (a 1-channel guide is copied once per image into its own pair
// of slots) with three streams,
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

extern "C" int gf_joint_is_fused(int dtype, int64_t B, int64_t C, int64_t h, int64_t w,
                                 int64_t H, int64_t W, int r);

namespace {

// chunk slots in flight: three decouple the H2D, kernel and D2H streams (with
// two, a D2H slowed by PCIe read/write contention stalls the next H2D)
constexpr int kSlots = 3;

struct Pipe {
  cudaStream_t in = nullptr, run = nullptr, out = nullptr;
  cudaEvent_t in_done[kSlots] = {}, run_done[kSlots] = {}, out_done[kSlots] = {},
              grp_in[2] = {}, grp_done[2] = {};
  bool ok = true;
  Pipe() {
    ok &= cudaStreamCreateWithFlags(&in, cudaStreamNonBlocking) == cudaSuccess;
    ok &= cudaStreamCreateWithFlags(&run, cudaStreamNonBlocking) == cudaSuccess;
    ok &= cudaStreamCreateWithFlags(&out, cudaStreamNonBlocking) == cudaSuccess;
    for (int s = 0; s < kSlots; ++s)
      for (cudaEvent_t* e : {&in_done[s], &run_done[s], &out_done[s]})
        ok &= cudaEventCreateWithFlags(e, cudaEventDisableTiming) == cudaSuccess;
    for (int s = 0; s < 2; ++s)
      for (cudaEvent_t* e : {&grp_in[s], &grp_done[s]})
        ok &= cudaEventCreateWithFlags(e, cudaEventDisableTiming) == cudaSuccess;
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

// One pipeline input: chunk b reads host block (b / grp) of `bytes`; a group
// input (grp > 1, e.g. a guide shared by the C planes of an image) is copied
// once per group into one of two group slots.
struct Input {
  const void* host;
  size_t bytes;
  int64_t grp;
};

// One pipeline output: chunk b writes host block b of `bytes`.
struct Output {
  void* host;
  size_t bytes;
};

constexpr int kMaxIn = 4, kMaxOut = 4;

// Copies of the inputs per chunk, up to four outputs per chunk; `launch` runs
// the device entry on the slot buffers.  Returns a GF_* code; *status gets the
// OR of the device bits.
template <class Launch>
int run_pipeline(int64_t nchunk, int nin, const Input* in, int nout, const Output* outs, char* ws,
                 uint32_t* status_dev, uint32_t* status_host, Launch launch) {
  Pipe* pp = pipe_for_current_device();
  if (!pp || !pp->ok) return gfb::api_fail(GF_ERR_CUDA, "stream/event creation failed");
  Pipe& p = *pp;
  if (cudaMemsetAsync(status_dev, 0, sizeof(uint32_t), p.run) != cudaSuccess)
    return gfb::api_fail(GF_ERR_CUDA, cudaGetErrorString(cudaGetLastError()));
  // workspace: per input kSlots slots (two for a group input), then kSlots
  // slots per output
  char* slot[kMaxIn][kSlots];
  char* oslot[kMaxOut][kSlots];
  char* w = ws;
  for (int i = 0; i < nin; ++i)
    for (int s = 0; s < (in[i].grp > 1 ? 2 : kSlots); ++s) {
      slot[i][s] = w;
      w += up256(in[i].bytes);
    }
  for (int o = 0; o < nout; ++o)
    for (int s = 0; s < kSlots; ++s) {
      oslot[o][s] = w;
      w += up256(outs[o].bytes);
    }
  int64_t grp = 1;  // the (single) group size of the group inputs
  for (int i = 0; i < nin; ++i)
    if (in[i].grp > 1) grp = in[i].grp;
  for (int64_t b = 0; b < nchunk; ++b) {
    const int s = (int)(b % kSlots);
    const int64_t g = b / grp;
    const int gs = (int)(g & 1);
    const void* dev_in[kMaxIn];
    void* dev_out[kMaxOut];
    for (int o = 0; o < nout; ++o) dev_out[o] = oslot[o][s];
    bool grp_copied = false;
    for (int i = 0; i < nin; ++i) {
      if (in[i].grp > 1) {
        if (b % grp == 0) {  // first chunk of the group: its slot is free once
                             // the last chunk of group g-2 ran
          if (g >= 2) cudaStreamWaitEvent(p.in, p.grp_done[gs], 0);
          cudaMemcpyAsync(slot[i][gs], (const char*)in[i].host + g * in[i].bytes, in[i].bytes,
                          cudaMemcpyHostToDevice, p.in);
          grp_copied = true;
        }
        dev_in[i] = slot[i][gs];
      }
    }
    if (grp_copied) cudaEventRecord(p.grp_in[gs], p.in);
    // chunk slot inputs are free once the kernel of chunk b-kSlots ran
    if (b >= kSlots) cudaStreamWaitEvent(p.in, p.run_done[s], 0);
    for (int i = 0; i < nin; ++i) {
      if (in[i].grp > 1) continue;
      cudaMemcpyAsync(slot[i][s], (const char*)in[i].host + b * in[i].bytes, in[i].bytes,
                      cudaMemcpyHostToDevice, p.in);
      dev_in[i] = slot[i][s];
    }
    cudaEventRecord(p.in_done[s], p.in);
    cudaStreamWaitEvent(p.run, p.in_done[s], 0);
    if (grp > 1) cudaStreamWaitEvent(p.run, p.grp_in[gs], 0);
    if (b >= kSlots) cudaStreamWaitEvent(p.run, p.out_done[s], 0);  // output slot copied out
    if (int e = launch(dev_in, dev_out, p.run)) {
      cudaStreamSynchronize(p.run);
      return e;
    }
    cudaEventRecord(p.run_done[s], p.run);
    if (grp > 1 && (b % grp == grp - 1 || b == nchunk - 1)) cudaEventRecord(p.grp_done[gs], p.run);
    cudaStreamWaitEvent(p.out, p.run_done[s], 0);
    for (int o = 0; o < nout; ++o)
      cudaMemcpyAsync((char*)outs[o].host + b * outs[o].bytes, oslot[o][s], outs[o].bytes,
                      cudaMemcpyDeviceToHost, p.out);
    cudaEventRecord(p.out_done[s], p.out);
  }
  for (int s = 0; s < kSlots; ++s)  // status written by every kernel
    if (s < nchunk) cudaStreamWaitEvent(p.out, p.run_done[s], 0);
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

size_t pipeline_ws(const Input* in, int nin, const Output* outs, int nout) {
  size_t n = 0;
  for (int o = 0; o < nout; ++o) n += kSlots * up256(outs[o].bytes);
  for (int i = 0; i < nin; ++i) n += (in[i].grp > 1 ? 2 : kSlots) * up256(in[i].bytes);
  return n;
}

}  // namespace

extern "C" {

// ---- full-resolution layer -------------------------------------------------
// chunk = one plane; a 1-channel guide is copied once per image and shared by
// the image's C planes
size_t gf_highres_host_workspace_bytes(int dtype, int64_t Cg, int64_t C, int64_t H, int64_t W,
                                       int radius) {
  (void)Cg;
  (void)C;
  const size_t plane = (size_t)H * W * esize(dtype);
  const Input ins[2] = {{nullptr, plane, 1}, {nullptr, plane, 1}};  // the larger layout
  const Output outs[1] = {{nullptr, plane}};
  return pipeline_ws(ins, 2, outs, 1) +
         up256(gf_highres_workspace_bytes(dtype, 1, 1, 1, H, W, radius)) + 256;
}

int gf_highres_fwd_host(int dtype, const void* guide, const void* src, void* out, int64_t B,
                        int64_t Cg, int64_t C, int64_t H, int64_t W, int radius, double eps,
                        void* workspace, size_t workspace_bytes, uint32_t* status) {
  if (int e = gfb::api_check_highres(dtype, B, Cg, C, H, W, radius, eps)) return e;
  if (!guide || !src || !out) return gfb::api_fail(GF_ERR_ARG, "null host pointer");
  const size_t need = gf_highres_host_workspace_bytes(dtype, Cg, C, H, W, radius);
  if (workspace_bytes < need) return gfb::api_fail(GF_ERR_WORKSPACE, "host workspace too small");
  const size_t plane = (size_t)H * W * esize(dtype);
  const Input ins[2] = {{guide, plane, Cg == C ? 1 : C}, {src, plane, 1}};
  const Output outs[1] = {{out, plane}};
  char* ws = (char*)workspace;
  char* gws = ws + pipeline_ws(ins, 2, outs, 1);
  const size_t gws_bytes = gf_highres_workspace_bytes(dtype, 1, 1, 1, H, W, radius);
  uint32_t* st_dev = (uint32_t*)(gws + up256(gws_bytes));
  return run_pipeline(B * C, 2, ins, 1, outs, ws, st_dev, status,
                      [&](const void* const* d, void* const* o, cudaStream_t s) {
                        return gf_highres_fwd(dtype, d[0], d[1], o[0], 1, 1, 1, H, W, radius, eps,
                                              gws, gws_bytes, st_dev, s);
                      });
}

// ---- joint (fast) layer ----------------------------------------------------
// chunk = one plane (the layer is independent per plane)
size_t gf_joint_host_workspace_bytes(int dtype, int64_t C, int64_t h, int64_t w, int64_t H,
                                     int64_t W, int radius) {
  (void)C;
  const size_t lo = (size_t)h * w * esize(dtype), hi = (size_t)H * W * esize(dtype);
  const Input ins[3] = {{nullptr, lo, 1}, {nullptr, lo, 1}, {nullptr, hi, 1}};
  const Output outs[1] = {{nullptr, hi}};
  return pipeline_ws(ins, 3, outs, 1) +
         up256(gf_joint_workspace_bytes(dtype, 1, 1, h, w, H, W, radius)) + 256;
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
  const Input ins[3] = {{lr_x, lo, 1}, {lr_y, lo, 1}, {hr_x, hi, 1}};
  const Output outs[1] = {{out, hi}};
  char* ws = (char*)workspace;
  char* gws = ws + pipeline_ws(ins, 3, outs, 1);
  const size_t gws_bytes = gf_joint_workspace_bytes(dtype, 1, 1, h, w, H, W, radius);
  uint32_t* st_dev = (uint32_t*)(gws + up256(gws_bytes));
  return run_pipeline(B * C, 3, ins, 1, outs, ws, st_dev, status,
                      [&](const void* const* d, void* const* o, cudaStream_t s) {
                        return gf_joint_fwd(dtype, d[0], d[1], d[2], o[0], 1, 1, h, w, H, W, radius,
                                            eps, gws, gws_bytes, st_dev, s);
                      });
}

// forward + backward of the joint layer on host images: per plane, copy in
// lr_x, lr_y, hr_x, d_out; run gf_joint_fwd and gf_joint_bwd; copy out out,
// d_lr_x, d_lr_y, d_hr_x (a training framework's layer call with host tensors)
size_t gf_joint_fwd_bwd_host_workspace_bytes(int dtype, int64_t C, int64_t h, int64_t w,
                                             int64_t H, int64_t W, int radius) {
  (void)C;
  const size_t lo = (size_t)h * w * esize(dtype), hi = (size_t)H * W * esize(dtype);
  const Input ins[4] = {{nullptr, lo, 1}, {nullptr, lo, 1}, {nullptr, hi, 1}, {nullptr, hi, 1}};
  const Output outs[4] = {{nullptr, hi}, {nullptr, lo}, {nullptr, lo}, {nullptr, hi}};
  return pipeline_ws(ins, 4, outs, 4) +
         up256(gf_joint_workspace_bytes(dtype, 1, 1, h, w, H, W, radius)) + up256(lo) + 256;
}

int gf_joint_fwd_bwd_host(int dtype, const void* lr_x, const void* lr_y, const void* hr_x,
                          const void* d_out, void* out, void* d_lr_x, void* d_lr_y, void* d_hr_x,
                          int64_t B, int64_t C, int64_t h, int64_t w, int64_t H, int64_t W,
                          int radius, double eps, void* workspace, size_t workspace_bytes,
                          uint32_t* status) {
  if (int e = gfb::api_check_joint(dtype, B, C, h, w, H, W, radius, eps)) return e;
  if (!lr_x || !lr_y || !hr_x || !d_out || !out || !d_lr_x || !d_lr_y || !d_hr_x)
    return gfb::api_fail(GF_ERR_ARG, "null host pointer");
  const size_t need = gf_joint_fwd_bwd_host_workspace_bytes(dtype, C, h, w, H, W, radius);
  if (workspace_bytes < need) return gfb::api_fail(GF_ERR_WORKSPACE, "host workspace too small");
  const size_t lo = (size_t)h * w * esize(dtype), hi = (size_t)H * W * esize(dtype);
  const Input ins[4] = {{lr_x, lo, 1}, {lr_y, lo, 1}, {hr_x, hi, 1}, {d_out, hi, 1}};
  const Output outs[4] = {{out, hi}, {d_lr_x, lo}, {d_lr_y, lo}, {d_hr_x, hi}};
  char* ws = (char*)workspace;
  char* gws = ws + pipeline_ws(ins, 4, outs, 4);
  const size_t gws_bytes = gf_joint_workspace_bytes(dtype, 1, 1, h, w, H, W, radius);
  void* slope = gws + up256(gws_bytes);  // one plane's slope tape (fast path)
  uint32_t* st_dev = (uint32_t*)((char*)slope + up256(lo));
  // the device API's path: forward keeping the slope tape, backward on it
  // (forward_joint / backward do the same), else the moments-recomputing pair
  const bool tape = gf_joint_is_fused(dtype, 1, 1, h, w, H, W, radius) != 0;
  return run_pipeline(B * C, 4, ins, 4, outs, ws, st_dev, status,
                      [&](const void* const* d, void* const* o, cudaStream_t s) {
                        if (tape) {
                          if (int e = gf_joint_fwd_tape(dtype, d[0], d[1], d[2], o[0], slope, 1,
                                                        1, h, w, H, W, radius, eps, gws,
                                                        gws_bytes, st_dev, s))
                            return e;
                          return gf_joint_bwd_tape(dtype, d[0], d[1], d[2], slope, d[3], o[1],
                                                   o[2], o[3], 1, 1, h, w, H, W, radius, eps, 0,
                                                   gws, gws_bytes, st_dev, s);
                        }
                        if (int e = gf_joint_fwd(dtype, d[0], d[1], d[2], o[0], 1, 1, h, w, H, W,
                                                 radius, eps, gws, gws_bytes, st_dev, s))
                          return e;
                        return gf_joint_bwd(dtype, d[0], d[1], d[2], d[3], o[1], o[2], o[3], 1, 1,
                                            h, w, H, W, radius, eps, gws, gws_bytes, st_dev, s);
                      });
}

}  // extern "C"
