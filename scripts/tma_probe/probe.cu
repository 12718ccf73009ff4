// Standalone probe: TMA 3-D box loads (as k_joint_fwd_tma issues them) into a
// 2-stage ring, one elected thread, mbarrier per stage; checks the data.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_1803_05619_b200/csrc/gf_tma.cuh"
using namespace gfb;

__global__ void k(const __grid_constant__ CUtensorMap tm, int bw, int bh, int x, int y, float* out, int mode) {
  extern __shared__ float4 sm4[];
  __shared__ __align__(8) uint64_t bar[2];
  float* base = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(sm4) + 127) & ~(uintptr_t)127);
  if (threadIdx.x == 0) { tma::mbar_init(&bar[0], 1); tma::mbar_init(&bar[1], 1); }
  __syncthreads();
  if (threadIdx.x == 0) {
    tma::mbar_arrive_expect_tx(&bar[0], bw * bh * 4);
    tma::load_3d(base, &tm, x, y, 0, &bar[0]);
  }
  tma::mbar_wait(&bar[0], 0);
  for (int i = threadIdx.x; i < bw * bh; i += blockDim.x) out[i] = base[i];
}

int main(int argc, char** argv) {
  if (argc < 7) return 2;
  int W = atoi(argv[1]), H = atoi(argv[2]), bw = atoi(argv[3]), bh = atoi(argv[4]);
  int x = atoi(argv[5]), y = atoi(argv[6]);
  std::vector<float> h(W * H);
  for (int i = 0; i < W * H; ++i) h[i] = (float)i;
  float *d, *o;
  cudaMalloc(&d, W * H * 4);
  cudaMalloc(&o, bw * bh * 4);
  cudaMemcpy(d, h.data(), W * H * 4, cudaMemcpyHostToDevice);
  CUtensorMap tm;
  bool ok = tma::make_plane_map(&tm, d, W, H, 1, bw, bh);
  size_t smem = 128 + bw * bh * 4;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<<<1, 128, smem>>>(tm, bw, bh, x, y, o, 0);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> r(bw * bh);
  cudaMemcpy(r.data(), o, bw * bh * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int yy = 0; yy < bh; ++yy)
    for (int xx = 0; xx < bw; ++xx) {
      int gx = x + xx, gy = y + yy;
      float want = (gx >= 0 && gx < W && gy >= 0 && gy < H) ? (float)(gy * W + gx) : 0.f;
      bad += r[yy * bw + xx] != want;
    }
  printf("W=%d H=%d box=%dx%d at (%d,%d): encode %d, err %s, bad %d\n", W, H, bw, bh, x, y, ok,
         cudaGetErrorString(e), bad);
  return e != cudaSuccess;
}
