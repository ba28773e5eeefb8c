// fp32-accurate batched GEMM on the sm_100a tensor cores from split bf16 operands (kind::f16):
//
//     D[s][b][m][n] = alpha * sum_{k in split s} A[b][m][k] * B[b][n][k]        (fp32 in TMEM)
//
// An fp32 operand x is carried as P bf16 planes hi + mid + lo (x == hi + mid + lo to 24 bits;
// wl_split3 below); an operand that is already exact in bf16 (quantised codes) is one plane.  Every
// product of planes (i, j) with i + j < max(PA, PB) is issued into the same TMEM accumulator (low
// order first), so
// D carries ~fp32 products (the dropped cross terms are below 2^-24 relative) with fp32 tensor-core
// accumulation over one split; splits are reduced in fp64 by the consumer.  Used by the STE backward
// (dV = dM . U, dU^T = V^T . dM) and the float Winograd path (M = V . U^T, §8f f2).
//
// Operands are K-major bf16 in HBM, [plane][batch][rows][Kd] with Kd a multiple of 64; TMA boxes
// {64, rows} with the 128-byte swizzle; one CTA computes a 128 x BN tile of one (batch, split):
// warp 0 TMA producer, warp 1 TMEM owner + single-thread MMA issuer (M=128, N=BN, K=16), warps 2-5
// epilogue (tcgen05.ld, one row per thread).
#pragma once
#include <cuda_bf16.h>

#include "wl_ptx.cuh"

namespace wl {

// kind::f16 instruction descriptor: bf16 A and B (K-major), fp32 accumulator.
__host__ __device__ constexpr uint32_t idesc_bf16(uint32_t M, uint32_t N) {
  return (1u << 4)            // c_format = F32
         | (1u << 7)          // a_format = BF16
         | (1u << 10)         // b_format = BF16
         | ((N >> 3) << 17)   // n_dim
         | ((M >> 4) << 24);  // m_dim
}

__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// x = hi + mid + lo exactly (fp32 has 24 significand bits, each bf16 plane holds 8).
__device__ __forceinline__ void wl_split3(float x, __nv_bfloat16& hi, __nv_bfloat16& mid, __nv_bfloat16& lo) {
  hi = __float2bfloat16_rn(x);
  const float r1 = x - __bfloat162float(hi);
  mid = __float2bfloat16_rn(r1);
  lo = __float2bfloat16_rn(r1 - __bfloat162float(mid));
}

struct GemmSplitArgs {
  int M, N, Kd;   // rows of A, rows of B, reduction length (multiple of 64)
  int batch;      // batches (the 36 Winograd elements)
  int PA, PB;     // bf16 planes of A and B (1..3)
  int splits;     // reduction splits; split s covers [s * ks, min(Kd, (s + 1) * ks))
  int ks;         // multiple of 64
  int stages;     // smem ring depth (host: as many as fit)
  float* D;       // [splits][batch][M][ldd]
  int ldd;
  float alpha;
};

constexpr int kGemmBfThreads = 192;

template <int BN>
struct GemmBfSmem {
  static constexpr int kA = 128 * 128;  // one plane: 128 rows x 64 bf16
  static constexpr int kB = BN * 128;
  static constexpr int stage_bytes(int pa, int pb) { return pa * kA + pb * kB; }
};

template <int BN>
__global__ void __launch_bounds__(kGemmBfThreads, 1)
    gemm_bf16_split_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                           GemmSplitArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  using L = GemmBfSmem<BN>;
  const int STAGES = p.stages;
  const int stage_bytes = L::stage_bytes(p.PA, p.PB);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * stage_bytes);
  uint64_t* empty = full + STAGES;
  uint64_t* accfull = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accfull + 1);
  constexpr uint32_t kTmemCols = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * 128, n0 = blockIdx.y * BN;
  const int b = blockIdx.z % p.batch, s = blockIdx.z / p.batch;
  const int k0 = s * p.ks, k1 = min(p.Kd, k0 + p.ks);
  const int kblocks = (k1 - k0) / 64;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(accfull, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      for (int kb = 0; kb < kblocks; ++kb) {
        const int st = kb % STAGES;
        const uint32_t ph = (kb / STAGES) & 1;
        mbar_wait(&empty[st], ph ^ 1);
        uint8_t* sa = smem + st * stage_bytes;
        uint8_t* sb = sa + p.PA * L::kA;
        mbar_arrive_expect_tx(&full[st], (uint32_t)stage_bytes);
        const int kx = k0 + kb * 64;
        for (int q = 0; q < p.PA; ++q) tma_load_3d(sa + q * L::kA, &tmA, &full[st], kx, m0, q * p.batch + b);
        for (int q = 0; q < p.PB; ++q) tma_load_3d(sb + q * L::kB, &tmB, &full[st], kx, n0, q * p.batch + b);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_bf16(128, BN);
      const int P = p.PA > p.PB ? p.PA : p.PB;
      uint32_t acc = 0;
      for (int kb = 0; kb < kblocks; ++kb) {
        const int st = kb % STAGES;
        const uint32_t ph = (kb / STAGES) & 1;
        mbar_wait(&full[st], ph);
        tc_fence_after();
        const uint8_t* sa = smem + st * stage_bytes;
        const uint8_t* sb = sa + p.PA * L::kA;
        // smallest plane products first (i + j descending): the fp32 accumulator absorbs the low-order
        // terms before the hi x hi product, which keeps their bits
        for (int d = P - 1; d >= 0; --d)
          for (int i = 0; i < p.PA; ++i) {
            const int j = d - i;
            if (j < 0 || j >= p.PB) continue;
#pragma unroll
            for (int k = 0; k < 4; ++k) {  // 4 x K=16 per 64-element (128-byte) swizzle row
              const uint64_t ad = smem_desc_kmajor(sa + i * L::kA + k * 32, 128);
              const uint64_t bd = smem_desc_kmajor(sb + j * L::kB + k * 32, 128);
              umma_bf16(tmem_base, ad, bd, idesc, acc);
              acc = 1;
            }
          }
        umma_commit(&empty[st]);
      }
      umma_commit(accfull);
    }
    __syncwarp();
  } else {
    const int q = warp & 3;  // TMEM lane quarter of this warp
    const int row = m0 + 32 * q + lane;
    float* drow = p.D + (((size_t)s * p.batch + b) * p.M + row) * p.ldd;
    if (kblocks > 0) {
      mbar_wait(accfull, 0);
      tc_fence_after();
    }
    const uint32_t taddr = tmem_base + (uint32_t(32 * q) << 16);
#pragma unroll 1
    for (int c = 0; c < BN; c += 16) {
      uint32_t r[16];
      if (kblocks > 0) {
        tmem_ld16(taddr + c, r);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) r[j] = 0u;
      }
      const int col = n0 + c;
      if (row < p.M) {
        if (col + 16 <= p.N && (p.ldd & 3) == 0) {
#pragma unroll
          for (int j = 0; j < 16; j += 4)
            *reinterpret_cast<float4*>(drow + col + j) =
                make_float4(p.alpha * __uint_as_float(r[j]), p.alpha * __uint_as_float(r[j + 1]),
                            p.alpha * __uint_as_float(r[j + 2]), p.alpha * __uint_as_float(r[j + 3]));
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (col + j < p.N) drow[col + j] = p.alpha * __uint_as_float(r[j]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem_base);
  }
}

}  // namespace wl
