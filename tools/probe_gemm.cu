// Standalone probe: tcgen05 kind::i8 GEMM vs a CPU int32 GEMM on random codes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2004_11077_b200/csrc probe_gemm.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "gemm_i8.cuh"
#include "wl_tmap.h"

struct StoreMaxEpi {
  int32_t* D;
  unsigned* gmax;
  int T, K, rows_per_group;
  unsigned m;
  __device__ void begin(int, int, bool) { m = 0; }
  __device__ void apply(int xi, int row, int col, const int32_t* v, int n) {
    int32_t* dst = D + ((size_t)xi * T + row) * K + col;
    for (int j = 0; j < n; ++j) {
      dst[j] = v[j];
      unsigned a = (unsigned)abs(v[j]);
      m = a > m ? a : m;
    }
  }
  __device__ void finish(int, int row, bool valid) {
    if (valid) atomicMax(&gmax[row / rows_per_group], m);
  }
};

template <int BN, int SW>
int run(int T, int C, int K) {
  constexpr int ST = 4;
  using L = wl::GemmSmem<BN, SW, ST>;
  std::vector<int8_t> A((size_t)36 * T * C), B((size_t)36 * K * C);
  srand(1);
  for (auto& a : A) a = (int8_t)(rand() % 255 - 127);
  for (auto& b : B) b = (int8_t)(rand() % 255 - 127);
  int8_t *dA, *dB;
  int32_t* dD;
  unsigned* dmax;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dD, (size_t)36 * T * K * 4);
  cudaMalloc(&dmax, 64 * 4);
  cudaMemset(dmax, 0, 256);
  cudaMemset(dD, 0x7f, (size_t)36 * T * K * 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  CUtensorMap ta, tb;
  if (!wl::make_tmap_i8_3d(&ta, dA, C, T, 36, SW, 128) || !wl::make_tmap_i8_3d(&tb, dB, C, K, 36, SW, BN)) {
    printf("tmap failed\n");
    return 1;
  }
  auto kern = wl::gemm_i8_kernel<BN, SW, ST, StoreMaxEpi>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kBytes);
  StoreMaxEpi e{dD, dmax, T, K, 100000000, 0};
  dim3 grid((T + 127) / 128, K / BN, 36);
  kern<<<grid, wl::kGemmThreads, L::kBytes>>>(ta, tb, T, K, C, e);
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) {
    printf("kernel error %s\n", cudaGetErrorString(err));
    return 1;
  }
  // timing
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < 20; ++i) kern<<<grid, wl::kGemmThreads, L::kBytes>>>(ta, tb, T, K, C, e);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= 20;
  std::vector<int32_t> D((size_t)36 * T * K);
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  unsigned gm;
  cudaMemcpy(&gm, dmax, 4, cudaMemcpyDeviceToHost);
  long bad = 0;
  unsigned cm = 0;
  for (int xi = 0; xi < 36; ++xi)
    for (int t = 0; t < T; ++t)
      for (int o = 0; o < K; ++o) {
        int32_t s = 0;
        const int8_t* a = &A[((size_t)xi * T + t) * C];
        const int8_t* b = &B[((size_t)xi * K + o) * C];
        for (int c = 0; c < C; ++c) s += (int32_t)a[c] * b[c];
        unsigned as = (unsigned)abs(s);
        cm = as > cm ? as : cm;
        if (D[((size_t)xi * T + t) * K + o] != s) {
          if (bad < 5) printf("mismatch xi=%d t=%d o=%d got %d want %d\n", xi, t, o, D[((size_t)xi * T + t) * K + o], s);
          ++bad;
        }
      }
  double tops = 2.0 * 36 * T * (double)K * C / (ms * 1e-3) / 1e12;
  printf("BN=%d SW=%d T=%d C=%d K=%d : mismatches=%ld max gpu=%u cpu=%u  %.3f ms  %.1f TOPS\n", BN, SW, T, C, K, bad,
         gm, cm, ms, tops);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
  cudaFree(dmax);
  return bad != 0 || gm != cm;
}

int main() {
  int fails = 0;
  fails += run<256, 128>(1000, 256, 256);
  fails += run<128, 128>(777, 128, 128);
  fails += run<64, 64>(300, 64, 64);
  fails += run<64, 32>(200, 32, 64);
  fails += run<256, 128>(8192, 512, 512);
  printf("%s\n", fails ? "PROBE FAIL" : "PROBE PASS");
  return fails;
}
