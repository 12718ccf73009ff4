// Microbenchmark: DRAM efficiency of tile-shaped streaming (read a TH x TW
// fp32 tile, write it back elsewhere) vs a linear copy, on 3072-wide planes.
// Measured (B200, gpurun_out/tc): every tile shape 64x128 .. 8x1024 copies at
// 6.78-6.84 TB/s, a grid-stride linear copy at 6.12 TB/s -- the joint
// kernels' 64 x 128 hr tiles cost no DRAM efficiency.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tilecopy tilecopy.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_linear(const float4* __restrict__ a, float4* __restrict__ b, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4;
       i += (size_t)gridDim.x * blockDim.x)
    b[i] = __ldg(a + i);
}

// one CTA of 256 threads copies a TH x TW tile; each thread holds TH*TW/1024 float4
template <int TH, int TW>
__global__ void __launch_bounds__(256) k_tile(const float* __restrict__ a, float* __restrict__ b,
                                              int H, int W) {
  constexpr int V = TH * TW / 4 / 256;  // float4 per thread
  constexpr int RW = TW / 4;            // float4 per tile row
  const int tx = W / TW;
  const int tiles_per_plane = tx * (H / TH);
  const size_t plane = (size_t)blockIdx.x / tiles_per_plane;
  const int t = blockIdx.x % tiles_per_plane;
  const int y0 = (t / tx) * TH, x0 = (t % tx) * TW;
  const float* src = a + plane * H * W;
  float* dst = b + plane * H * W;
  float4 v[V];
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const int e = k * 256 + threadIdx.x;
    const int y = y0 + e / RW, x = x0 + (e % RW) * 4;
    v[k] = __ldg(reinterpret_cast<const float4*>(src + (size_t)y * W + x));
  }
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const int e = k * 256 + threadIdx.x;
    const int y = y0 + e / RW, x = x0 + (e % RW) * 4;
    *reinterpret_cast<float4*>(dst + (size_t)y * W + x) = v[k];
  }
}

int main() {
  const int H = 3072, W = 3072, P = 48;  // 48 planes of 3072^2: 1.81 GB each way
  const size_t n = (size_t)P * H * W;
  float *a, *b;
  cudaMalloc(&a, n * 4);
  cudaMalloc(&b, n * 4);
  cudaMemset(a, 0, n * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(e0);
    for (int i = 0; i < 10; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 10;
    printf("%-12s %8.1f us  %7.1f GB/s\n", name, ms * 1e3, 2.0 * n * 4 / (ms * 1e-3) / 1e9);
  };
  run("linear", [&] { k_linear<<<148 * 16, 256>>>((const float4*)a, (float4*)b, n / 4); });
  run("64x128", [&] { k_tile<64, 128><<<P * (H / 64) * (W / 128), 256>>>(a, b, H, W); });
  run("32x256", [&] { k_tile<32, 256><<<P * (H / 32) * (W / 256), 256>>>(a, b, H, W); });
  run("16x512", [&] { k_tile<16, 512><<<P * (H / 16) * (W / 512), 256>>>(a, b, H, W); });
  run("8x1024", [&] { k_tile<8, 1024><<<P * (H / 8) * (W / 1024), 256>>>(a, b, H, W); });
  run("128x64", [&] { k_tile<128, 64><<<P * (H / 128) * (W / 64), 256>>>(a, b, H, W); });
  run("64x64", [&] { k_tile<64, 64><<<P * (H / 64) * (W / 64), 256>>>(a, b, H, W); });
  run("32x128", [&] { k_tile<32, 128><<<P * (H / 32) * (W / 128), 256>>>(a, b, H, W); });
  printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
