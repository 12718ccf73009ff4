// 8-bit image <-> planar float conversion on the device, for the upsample
// CLI (gf/cli.py:72-101 with gf/fileio.py:104-141): an image file's bytes
// cross PCIe as bytes (1 B per sample instead of 4 or 8) and are unpacked /
// packed next to the filter.
//   unpack: interleaved HWC uint8 -> NCHW (B = 1) value / 255 (fileio.py:129)
//   pack:   NCHW -> HWC uint8 of rint(clip(v, 0, 1) * 255), round half to
//           even as numpy's rint (fileio.py:137-139)
#include <cuda_runtime.h>

#include "../../include/gf_b200.h"
#include "gf_common.cuh"
#include "gf_internal.h"

namespace gfb {
namespace io {

template <typename T>
__global__ void k_unpack(const uint8_t* __restrict__ hwc, T* __restrict__ out, int64_t HW,
                         int64_t C) {
  GF_GRID_LOOP(i, HW * C) {
    const int64_t c = i / HW, px = i - c * HW;
    out[i] = (T)((double)hwc[px * C + c] / 255.0);
  }
}

template <typename T>
__global__ void k_pack(const T* __restrict__ in, uint8_t* __restrict__ hwc, int64_t HW,
                       int64_t C) {
  GF_GRID_LOOP(i, HW * C) {
    const int64_t px = i / C, c = i - px * C;
    double v = (double)in[c * HW + px];
    v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
    hwc[i] = (uint8_t)rint(v * 255.0);  // NaN never reaches here (the filter raises)
  }
}

}  // namespace io
}  // namespace gfb

extern "C" {

int gf_image_unpack_u8(int dtype, const uint8_t* hwc, void* nchw, int64_t H, int64_t W,
                       int64_t C, void* stream) {
  if (dtype != GF_F32 && dtype != GF_F64) return gfb::api_fail(GF_ERR_ARG, "bad dtype");
  if (H < 1 || W < 1 || C < 1) return gfb::api_fail(GF_ERR_ARG, "image dims must be >= 1");
  const int64_t n = H * W * C;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == GF_F32)
    gfb::io::k_unpack<float><<<gfb::grid_for(n), 256, 0, s>>>(hwc, (float*)nchw, H * W, C);
  else
    gfb::io::k_unpack<double><<<gfb::grid_for(n), 256, 0, s>>>(hwc, (double*)nchw, H * W, C);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GF_OK : gfb::api_fail(GF_ERR_CUDA, cudaGetErrorString(e));
}

int gf_image_pack_u8(int dtype, const void* nchw, uint8_t* hwc, int64_t H, int64_t W, int64_t C,
                     void* stream) {
  if (dtype != GF_F32 && dtype != GF_F64) return gfb::api_fail(GF_ERR_ARG, "bad dtype");
  if (H < 1 || W < 1 || C < 1) return gfb::api_fail(GF_ERR_ARG, "image dims must be >= 1");
  const int64_t n = H * W * C;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == GF_F32)
    gfb::io::k_pack<float><<<gfb::grid_for(n), 256, 0, s>>>((const float*)nchw, hwc, H * W, C);
  else
    gfb::io::k_pack<double><<<gfb::grid_for(n), 256, 0, s>>>((const double*)nchw, hwc, H * W,
                                                             C);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GF_OK : gfb::api_fail(GF_ERR_CUDA, cudaGetErrorString(e));
}

}  // extern "C"
