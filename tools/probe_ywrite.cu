// Probe: DRAM efficiency of NCHW fp32 output write patterns on B200 (config-4 shape:
// N images x 256 channels x 56 x 56).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_ywrite probe_ywrite.cu
#include <cstdio>
#include <cuda_runtime.h>
constexpr int K = 256, H = 56, W = 56, TW = 14, TP = 196;
// A: linear streaming
__global__ void k_linear(float4* y, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
    __stcs(y + i, make_float4(1.f, 2.f, 3.f, 4.f));
}
// B: sout_cw pattern. item = (tg: 8 consecutive tiles, kb: 32 channels), kb fastest; warp w -> 4 channels,
// lane = (tile8, ch); 4 rows of 16 B per lane.  TPI = tiles per item (8) ; mode 1 = tile-row items (14 tiles, 2 ch/warp-pass)
template <int MODE>
__global__ void k_tiles(float* y, int N) {
  const int T = N * TP;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (MODE == 0) {
    const int nkb = K / 32, niter = (T / 8) * nkb;
    for (int it = blockIdx.x; it < niter; it += gridDim.x) {
      const int tg = it / nkb, kb = it - tg * nkb;
      const int t = tg * 8 + (lane >> 2), k = kb * 32 + 4 * w + (lane & 3);
      const int n = t / TP, tile = t - n * TP, ty = tile / TW, tx = tile - ty * TW;
      float* row = y + (((size_t)n * K + k) * H + 4 * ty) * W + 4 * tx;
#pragma unroll
      for (int i = 0; i < 4; ++i) __stcs(reinterpret_cast<float4*>(row + i * W), make_float4(1.f, 2.f, 3.f, 4.f));
    }
  } else if (MODE == 1) {
    // item = one tile row (14 tiles = 224 B per output row) x 32 channels: per channel 4 rows x 224 B = 896 B contiguous.
    // warp w -> channels 4w..4w+3; lane = (ch2 = lane / 14 (0..1, lanes 28..31 idle), tx = lane % 14), two passes over channel pairs
    const int nkb = K / 32, niter = N * TW * nkb;
    for (int it = blockIdx.x; it < niter; it += gridDim.x) {
      const int rg = it / nkb, kb = it - rg * nkb;  // rg = n * 14 + ty
      const int n = rg / TW, ty = rg - n * TW;
      if (lane < 28) {
        const int tx = lane % 14, c2 = lane / 14;
#pragma unroll
        for (int pass = 0; pass < 2; ++pass) {
          const int k = kb * 32 + 4 * w + 2 * pass + c2;
          float* row = y + (((size_t)n * K + k) * H + 4 * ty) * W + 4 * tx;
#pragma unroll
          for (int i = 0; i < 4; ++i) __stcs(reinterpret_cast<float4*>(row + i * W), make_float4(1.f, 2.f, 3.f, 4.f));
        }
      }
    }
  } else {
    // MODE 2: item = whole plane (n, k): warp writes 12544 B contiguous with coalesced float4 (ideal NCHW order)
    const int niter = N * K / 8;
    for (int it = blockIdx.x; it < niter; it += gridDim.x) {
      float4* p = reinterpret_cast<float4*>(y + ((size_t)it * 8 + w) * H * W);
      for (int i = lane; i < H * W / 4; i += 32) __stcs(p + i, make_float4(1.f, 2.f, 3.f, 4.f));
    }
  }
}
int main() {
  const int N = 1024;
  const size_t bytes = (size_t)N * K * H * W * 4;
  float* y;
  cudaMalloc(&y, bytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto time = [&](const char* name, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-28s %8.3f ms  %8.1f GB/s  (%s)\n", name, ms / 10, bytes / (ms / 10) * 1e-6, cudaGetErrorString(cudaGetLastError()));
  };
  time("linear float4 stcs", [&] { k_linear<<<148 * 8, 256>>>(reinterpret_cast<float4*>(y), bytes / 16); });
  time("cw items 8 tiles x 32ch", [&] { k_tiles<0><<<148 * 4, 256>>>(y, N); });
  time("tile-row items 14 x 32ch", [&] { k_tiles<1><<<148 * 4, 256>>>(y, N); });
  time("whole planes per warp", [&] { k_tiles<2><<<148 * 4, 256>>>(y, N); });
  time("cw items, 8 CTAs/SM", [&] { k_tiles<0><<<148 * 8, 256>>>(y, N); });
  cudaMemset(y, 0, bytes);
  time("cudaMemset", [&] { cudaMemsetAsync(y, 0, bytes); });
  return 0;
}
