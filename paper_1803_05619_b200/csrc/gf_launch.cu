// Per-device launch configuration cache.
//
// Occupancy queries and cudaFuncSetAttribute(MaxDynamicSharedMemorySize) are
// per device (per context), so the cache is keyed by the CURRENT device as
// well as the kernel, block size and dynamic shared memory.  A process that
// drives cuda:0 and then cuda:1 therefore configures each device once, and
// concurrent host threads see a consistent entry (one mutex; a lookup costs
// tens of nanoseconds next to a kernel launch).
#include <cuda_runtime.h>

#include <mutex>
#include <tuple>
#include <map>

#include "gf_internal.h"

namespace gfb {

namespace {
using Key = std::tuple<int, const void*, int, size_t>;
std::mutex g_mu;
std::map<Key, LaunchCfg>& table() {
  static std::map<Key, LaunchCfg> t;
  return t;
}
}  // namespace

LaunchCfg launch_cfg(const void* fn, int threads, size_t smem) {
  int dev = 0;
  cudaGetDevice(&dev);
  const Key key{dev, fn, threads, smem};
  std::lock_guard<std::mutex> lock(g_mu);
  auto it = table().find(key);
  if (it != table().end()) return it->second;
  LaunchCfg c{0, 1};
  cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, dev);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  // kernels sized by their shared memory (rings, staged windows) want the
  // largest carve-out: the default heuristic can leave a 48 KB kernel with
  // fewer CTAs per SM than its shared memory allows
  if (smem >= 16 * 1024)
    cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem);
  c.per_sm = per_sm < 1 ? 1 : per_sm;
  if (c.sms < 1) c.sms = 1;
  table()[key] = c;
  return c;
}

}  // namespace gfb
