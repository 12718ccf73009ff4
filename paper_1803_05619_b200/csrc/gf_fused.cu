// placeholder: fused kernels not yet implemented
#include "gf_internal.h"
namespace gfb {
bool fused_highres_fwd_ok(int64_t, int64_t, int64_t, int64_t, int64_t, int) { return false; }
void fused_highres_fwd(const float*, const float*, float*, int64_t, int64_t, int64_t, int64_t,
                       int64_t, int, float, uint32_t*, cudaStream_t) {}
bool fused_joint_ok(int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int) { return false; }
void fused_joint_fwd(const float*, const float*, const float*, float*, int64_t, int64_t, int64_t,
                     int64_t, int64_t, int64_t, int, float, uint32_t*, cudaStream_t) {}
size_t fused_joint_bwd_ws_bytes(int64_t, int64_t, int64_t, int64_t) { return 0; }
void fused_joint_bwd(const float*, const float*, const float*, const float*, float*, float*,
                     float*, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int, float,
                     void*, uint32_t*, cudaStream_t) {}
}
