// Throughput probe: scalar FFMA (immediate coefficient) vs packed FFMA2 (f32x2) on sm_100a.
// Each thread runs 8 independent chains; reports thread-FMAs per clock per SM.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long f2(float a, float b) {
  return ((unsigned long long)__float_as_uint(b) << 32) | __float_as_uint(a);
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
template <int N>
__global__ void k_scalar(float* out, float s) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 0.001f + i;
  for (int it = 0; it < N; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], 0.999f, 0.25f);
  float r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += a[i];
  if (r == s) out[threadIdx.x] = r;
}
template <int N>
__global__ void k_pair(float* out, float s, float c1, float c2) {
  unsigned long long a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = f2(threadIdx.x * 0.001f + i, i + 0.5f);
  const unsigned long long m = f2(c1, c1), ad = f2(c2, c2);
  for (int it = 0; it < N; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = ffma2(a[i], m, ad);
  float r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += __uint_as_float((unsigned)a[i]) + __uint_as_float((unsigned)(a[i] >> 32));
  if (r == s) out[threadIdx.x] = r;
}
template <int N>
__global__ void k_mix(float* out, float s, float c1, float c2) {  // FFMA2 + independent integer ALU work
  unsigned long long a[8];
  unsigned u[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { a[i] = f2(threadIdx.x * 0.001f + i, i + 0.5f); u[i] = threadIdx.x + i; }
  const unsigned long long m = f2(c1, c1), ad = f2(c2, c2);
  for (int it = 0; it < N; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) { a[i] = ffma2(a[i], m, ad); u[i] = (u[i] ^ (u[i] >> 3)) + 7u; }
  float r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += __uint_as_float((unsigned)a[i]) + (float)u[i];
  if (r == s) out[threadIdx.x] = r;
}
int main() {
  float* o; cudaMalloc(&o, 4096);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  constexpr int N = 4096;
  const int blocks = sms * 8, thr = 256;
  for (int which = 0; which < 3; ++which) {
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      if (which == 0) k_scalar<N><<<blocks, thr>>>(o, -1.f);
      else if (which == 1) k_pair<N><<<blocks, thr>>>(o, -1.f, 0.999f, 0.25f);
      else k_mix<N><<<blocks, thr>>>(o, -1.f, 0.999f, 0.25f);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    const double fmas = (double)blocks * thr * N * 8 * (which == 0 ? 1 : 2);
    const double instr = (double)blocks * thr * N * 8 / 32 * (which == 2 ? 3 : 1);
    printf("%s: %.3f ms  %.1f thread-FMA/clk/SM  %.2f warp-instr/clk/SM (clock %d MHz)\n",
           which == 0 ? "FFMA imm" : which == 1 ? "FFMA2   " : "FFMA2+ALU", best, fmas / (best * 1e-3) / (clk * 1e3) / sms,
           instr / (best * 1e-3) / (clk * 1e3) / sms, clk / 1000);
  }
  return 0;
}
