// Probe: a 6x6 sandwich T = L X L^T per (tile, channel) unit as one int8 tcgen05 MMA against the
// Kronecker matrix (L (x) L) split into signed base-256 digits.  A = the staged input window, MN-major
// (channels contiguous) exactly as TMA writes it with SWIZZLE_128B from the NHWC codes (box {128, 6,
// 6, 1}: 36 rows of 128 channels); B = digit matrix [112][64] K-major (SWIZZLE_64B).  D[m = channel]
// [n = digit * 36 + e] int32 in TMEM; T_e = D[e] + 256 D[36 + e] + 65536 D[72 + e], exact.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O2 -I paper_2004_11077_b200/csrc
//        tools/probe_tc_transform.cu -o /tmp/probe_tc -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "wl_ptx.cuh"
#include "wl_tmap.h"

using namespace wl;

constexpr int CP = 256, NCOL = 112;
// P^-T * 315 (input/output base change)
static const int Lm[6][6] = {{315, 0, 0, 0, 0, 0},  {0, 315, 0, 0, 0, 0},     {105, 0, 315, 0, 0, 0},
                             {0, 189, 0, 315, 0, 0}, {63, 0, 270, 0, 315, 0}, {0, 135, 0, 350, 0, 315}};

__global__ void probe_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap,
                             int* __restrict__ out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                 // 2 halves x 64 rows x 128 B
  uint8_t* sB = smem + 2 * 8192;      // 112 rows x 64 B
  uint64_t* bar = reinterpret_cast<uint64_t*>(sB + NCOL * 64);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 2 * 8192 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sA)[i] = 0x7f7f7f7fu;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<256>(tslot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar[0], 2 * 36 * 128 + NCOL * 64);
    tma_load_4d(sA, &amap, &bar[0], 0, 0, 0, 0);
    tma_load_4d(sA + 8192, &amap, &bar[0], 128, 0, 0, 0);
    tma_load_3d(sB, &bmap, &bar[0], 0, 0, 0);
  }
  mbar_wait(&bar[0], 0);
  if (warp == 1 && elect_one()) {
    tc_fence_after();
    const uint32_t idesc = idesc_i8(128, NCOL) | (1u << 15);  // A MN-major
    for (int h = 0; h < 2; ++h)
      for (int k = 0; k < 2; ++k) {
        const uint32_t a_addr = smem_u32(sA + h * 8192 + k * 32 * 128);
        uint64_t ad = (uint64_t)((a_addr >> 4) & 0x3FFF);
        ad |= (uint64_t)((8192u >> 4) & 0x3FFF) << 16;  // LBO: next 128-channel atom (unused, M = 128)
        ad |= (uint64_t)((1024u >> 4) & 0x3FFF) << 32;  // SBO: next group of 8 K rows
        ad |= 1ull << 46;
        ad |= 2ull << 61;  // SWIZZLE_128B
        const uint64_t bd = smem_desc_kmajor(sB + k * 32, 64);
        umma_i8(tbase + (uint32_t)(h * 128), ad, bd, idesc, k != 0);
      }
    umma_commit(&bar[1]);
  }
  __syncwarp();
  mbar_wait(&bar[1], 0);
  tc_fence_after();
  for (int h = 0; h < 2; ++h) {
    uint32_t r[NCOL];
    const uint32_t ta = tbase + (uint32_t(32 * (warp & 3)) << 16) + (uint32_t)(h * 128);
#pragma unroll
    for (int c = 0; c < NCOL; c += 16) tmem_ld16(ta + c, *reinterpret_cast<uint32_t(*)[16]>(r + c));
    tmem_ld_wait();
    const int ch = h * 128 + 32 * (warp & 3) + lane;
    for (int e = 0; e < 36; ++e)
      out[ch * 36 + e] = (int)r[e] + 256 * (int)r[36 + e] + 65536 * (int)r[72 + e];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(tbase);
}

int main() {
  // c0: [n=1][h=6][w=6][CP] random int8
  std::vector<int8_t> c0(6 * 6 * CP);
  srand(1);
  for (auto& v : c0) v = (int8_t)((rand() % 255) - 127);
  // digit matrix B[n][k]: n = d * 36 + e, k = xi (< 36), zero elsewhere
  std::vector<int8_t> B(NCOL * 64, 0);
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j)
      for (int p = 0; p < 6; ++p)
        for (int q = 0; q < 6; ++q) {
          int K = Lm[i][p] * Lm[j][q];
          const int e = 6 * i + j, xi = 6 * p + q;
          for (int d = 0; d < 3; ++d) {
            int dg = ((K % 256) + 256 + 128) % 256 - 128;
            B[(d * 36 + e) * 64 + xi] = (int8_t)dg;
            K = (K - dg) / 256;
          }
          if (K != 0) printf("digit overflow\n");
        }
  int8_t *dc0, *dB;
  int* dout;
  cudaMalloc(&dc0, c0.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dout, CP * 36 * 4);
  cudaMemcpy(dc0, c0.data(), c0.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  CUtensorMap amap, bmap;
  {
    EncodeTiledFn enc = get_encode_fn();
    cuuint64_t dims[4] = {CP, 6, 6, 1};
    cuuint64_t strides[3] = {CP, CP * 6, CP * 36};
    cuuint32_t box[4] = {128, 6, 6, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = enc(&amap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, dc0, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("amap failed %d\n", (int)r);
  }
  if (!make_tmap_i8_3d(&bmap, dB, 64, NCOL, 1, 64, NCOL, 1)) printf("bmap failed\n");
  const int smem = 1024 + 2 * 8192 + NCOL * 64 + 64;
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe_kernel<<<1, 128, smem>>>(amap, bmap, dout);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("kernel error %s\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<int> out(CP * 36);
  cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
  long bad = 0;
  for (int c = 0; c < CP; ++c)
    for (int i = 0; i < 6; ++i)
      for (int j = 0; j < 6; ++j) {
        long long t = 0;
        for (int p = 0; p < 6; ++p)
          for (int q = 0; q < 6; ++q) t += (long long)Lm[i][p] * c0[(p * 6 + q) * CP + c] * Lm[j][q];
        if (t != out[c * 36 + 6 * i + j]) {
          if (bad < 8) printf("mismatch c=%d e=%d: gpu %d cpu %lld\n", c, 6 * i + j, out[c * 36 + 6 * i + j], t);
          ++bad;
        }
      }
  printf("probe_tc_transform: %ld mismatches of %d\n", bad, CP * 36);
  return bad != 0;
}
