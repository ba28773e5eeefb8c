// Host launcher of the split-bf16 tcgen05 GEMM (gemm_bf16.cuh).
#include <cuda.h>
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <tuple>

#include "gemm_bf16.cuh"
#include "wl_gemm_bf16.h"
#include "wl_tmap.h"

namespace wl {

namespace {

bool tmap_bf16_sw128(CUtensorMap* map, const void* base, uint64_t kd, uint64_t rows, uint64_t batches,
                     uint32_t box_rows) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[3] = {kd, rows, batches};
  cuuint64_t strides[2] = {kd * 2, kd * rows * 2};
  cuuint32_t box[3] = {64, box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t set_attr_once(const void* kern, int smem) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int>, int> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_tuple(kern, dev);
  auto it = done.find(key);
  if (it != done.end() && it->second >= smem) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess) done[key] = smem;
  return e;
}

template <int BN>
cudaError_t launch(const CUtensorMap& ta, const CUtensorMap& tb, GemmSplitArgs a, cudaStream_t st) {
  constexpr int kMaxSmem = 220 * 1024;
  const int stage = GemmBfSmem<BN>::stage_bytes(a.PA, a.PB);
  a.stages = (kMaxSmem - 1024 - 256) / stage;
  if (a.stages > 4) a.stages = 4;
  if (a.stages < 1) return cudaErrorInvalidValue;
  // A split of kb K-blocks never uses more than kb ring stages, and when two CTAs per SM still get
  // min(kb, 2) stages each, the smaller ring wins: one CTA's TMA latency and epilogue run under the other's
  // MMAs (the config-3 backward GEMMs are one to a few K-blocks deep: a 4-stage 220 KB ring left one
  // CTA per SM running load -> MMA -> epilogue back to back, 139 us for 377 MB on 64 channels x 32 x 32).
  const int kb = (a.ks < a.Kd ? a.ks : a.Kd) / 64;
  if (a.stages > kb) a.stages = kb < 1 ? 1 : kb;
  const int half = (kMaxSmem / 2 - 1024 - 256) / stage;
  if (half >= (kb < 2 ? kb : 2) && half >= 1 && a.stages > half) a.stages = half;
  const int smem = 1024 + a.stages * stage + 256;
  auto kern = gemm_bf16_split_kernel<BN>;
  cudaError_t e = set_attr_once(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  dim3 grid((a.M + 127) / 128, (a.N + BN - 1) / BN, a.batch * a.splits);
  kern<<<grid, kGemmBfThreads, smem, st>>>(ta, tb, a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t gemm_bf16_split(const void* A, int PA, const void* B, int PB, int batch, int M, int N, int Kd, int ks,
                            float* D, int ldd, float alpha, cudaStream_t st) {
  if (Kd % 64 || ks % 64 || ks <= 0 || PA < 1 || PA > 3 || PB < 1 || PB > 3) return cudaErrorInvalidValue;
  // N tile: the whole (16-rounded) N up to 256; two planes x 3 of B at BN = 256 still fit 2 stages
  int BN = N <= 16 ? 16 : N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256;
  if (PA * 16384 + PB * BN * 128 > 110 * 1024 && BN > 128) BN = 128;  // keep >= 2 ring stages
  GemmSplitArgs a;
  a.M = M, a.N = N, a.Kd = Kd, a.batch = batch, a.PA = PA, a.PB = PB, a.ks = ks, a.splits = (Kd + ks - 1) / ks;
  a.stages = 0, a.D = D, a.ldd = ldd, a.alpha = alpha;
  CUtensorMap ta, tb;
  if (!tmap_bf16_sw128(&ta, A, Kd, M, (uint64_t)PA * batch, 128) ||
      !tmap_bf16_sw128(&tb, B, Kd, N, (uint64_t)PB * batch, BN))
    return cudaErrorInvalidValue;
  switch (BN) {
    case 16: return launch<16>(ta, tb, a, st);
    case 32: return launch<32>(ta, tb, a, st);
    case 64: return launch<64>(ta, tb, a, st);
    case 128: return launch<128>(ta, tb, a, st);
    default: return launch<256>(ta, tb, a, st);
  }
}

}  // namespace wl
