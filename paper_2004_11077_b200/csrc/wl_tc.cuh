// Tensor-core stage transforms (tcgen05 kind::i8): a 6x6 sandwich T = L X L^T of every (tile,
// channel) unit as ONE int8 MMA against the Kronecker matrix (L (x) L), split into signed base-256
// digits so every operand is int8 and every accumulator an exact int32.
//
//   A = the tile's staged codes, MN-major: TMA box {128 channels, 6, 6} with SWIZZLE_128B lands as
//       36 rows (xi = 6p + q) of 128 channels = the canonical MN-major SW128 layout (8-row K groups
//       1024 B apart); rows 36..63 are never written — the B columns there are zero.
//   B = digit matrix [NCOL][64] K-major SW64: row n = d * 36 + e holds digit d of (L (x) L)[e][xi];
//       rows 112 + d * 36 + e hold digit d of (I (x) L)[e][xi] (the first-half values tmp = X L^T,
//       whose group maximum sets the fp32 error band of the next pass's fast path).
//   D = TMEM [128 channels][NCOL] int32;  T_e = D[e] + 256 D[36 + e] + 65536 D[72 + e],
//       tmp_e = D[112 + e] + 256 D[148 + e]  (both exact: |T| <= 8.1e7 for P^-T).
// Work item = (tile, 128-channel half); warp 0 = TMA producer, warp 1 = TMEM owner + MMA issuer,
// warps 2..9 = epilogue (two per TMEM lane quarter = 32 channels, 18 outputs each); accumulators
// double-buffered by item (TMEM columns 0 and 256).
// Probe: tools/probe_tc_transform.cu (exact on random codes).
#pragma once
#include "wl_kernels2.cuh"
#include "wl_ptx.cuh"

namespace wl {
namespace tc {

constexpr int NCOL = 192;           // 108 T-digit + 72 tmp-digit columns, padded to a multiple of 16
constexpr int TMP0 = 112;           // first tmp-digit column
constexpr int STAGES = 16;          // TMA windows in flight per SM (L2-latency bound otherwise)
constexpr int A_BYTES = 40 * 128;   // one item's 36 rows, 1024-aligned; the MMA's rows 36..63 read the
                                    // next slot (or the slack below) against zero B columns
constexpr int A_SLACK = 3 * 1024;
constexpr int B_BYTES = NCOL * 64;
constexpr int SMEM_USED = 1024 + STAGES * A_BYTES + A_SLACK + B_BYTES + 256 + 2 * 128 * 8;
// > half the SM's shared memory: one CTA per SM, so no CTA ever waits on another's 512 TMEM columns
constexpr int SMEM = SMEM_USED > 120 * 1024 ? SMEM_USED : 120 * 1024;
constexpr int EPI_WARPS = 8;  // two per TMEM lane quarter, each combining half of the 36 outputs
constexpr int THREADS = 64 + 32 * EPI_WARPS;

// 32 lanes x 32 bit, 2 consecutive columns per thread.
__device__ __forceinline__ void tmem_ld2(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(taddr));
}
// 18 consecutive columns
__device__ __forceinline__ void tmem_ld18(uint32_t taddr, uint32_t* r) {
  tmem_ld16(taddr, *reinterpret_cast<uint32_t(*)[16]>(r));
  tmem_ld2(taddr + 16, r + 16);
}

// signed base-256 digit d of v
__host__ __device__ constexpr int digit(int v, int d) {
  for (int i = 0; i < d; ++i) {
    const int lo = ((v % 256) + 256 + 128) % 256 - 128;
    v = (v - lo) / 256;
  }
  return ((v % 256) + 256 + 128) % 256 - 128;
}

// Build the B operand of stage matrix L (6x6 integer) in shared memory, K-major with the 64-byte
// swizzle (16-byte chunk index ^= (row >> 1) & 3 within each 512-byte atom; sB 1024-aligned).
template <class L>
__device__ __forceinline__ void build_kron_b(uint8_t* sB) {
  for (int idx = threadIdx.x; idx < NCOL * 64; idx += blockDim.x) {
    const int n = idx >> 6, k = idx & 63;
    int v = 0;
    if (k < 36) {
      const int p = k / 6, q = k % 6;
      if (n < 108) {
        const int d = n / 36, e = n % 36, i = e / 6, j = e % 6;
        v = digit(L::e(i, p) * L::e(j, q), d);
      } else if (n >= TMP0 && n < TMP0 + 72) {
        const int d = (n - TMP0) / 36, e = (n - TMP0) % 36, l = e / 6, j = e % 6;  // tmp[l][j] = sum_q X[l][q] L[j][q]
        v = (p == l) ? digit(L::e(j, q), d) : 0;
      }
    }
    const int chunk = (k >> 4) ^ ((n >> 1) & 3);
    sB[n * 64 + chunk * 16 + (k & 15)] = (uint8_t)(int8_t)v;
  }
}

__device__ __forceinline__ uint64_t desc_mn_sw128(uint32_t addr) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((8192u >> 4) & 0x3FFF) << 16;  // LBO: next 128-channel atom (unused: M = 128)
  d |= (uint64_t)((1024u >> 4) & 0x3FFF) << 32;  // SBO: next group of 8 K rows
  d |= 1ull << 46;                                // version (sm_100)
  d |= 2ull << 61;                                // SWIZZLE_128B
  return d;
}

// Legendre input_base_change maximum (replaces sin_a_kernel<1, LD> for Cp in {128, 256}): per unit
// the exact max |T| and max |tmp|, recorded exactly like the CUDA-core pass (record_unit).
__global__ void __launch_bounds__(THREADS, 1)
    sin_a_tc_kernel(const __grid_constant__ CUtensorMap amap, Geo g, Acc* __restrict__ acc, Tables tabs) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + STAGES * A_BYTES + A_SLACK;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* accfull = empty + STAGES;  // [2]
  uint64_t* accempty = accfull + 2;    // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(accempty + 2);
  int2* part = reinterpret_cast<int2*>(sB + B_BYTES + 256);  // [2][128] partial maxima
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int halves = g.Cp >> 7;
  const int nitems = g.T * halves;
  // contiguous item range per CTA: the scale group changes only a few times per CTA, so the group
  // maxima are kept in registers and published once per group (no same-address atomic storm)
  const int i0 = (int)((long long)nitems * blockIdx.x / gridDim.x);
  const int i1 = (int)((long long)nitems * (blockIdx.x + 1) / gridDim.x);

  build_kron_b<tab::Leg_IBC>(sB);
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&amap);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&accfull[a], 1);
      mbar_init(&accempty[a], EPI_WARPS);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(tslot);
  fence_proxy_async_smem();  // the generic-proxy B writes become visible to the tensor core
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;

  if (warp == 0) {
    if (elect_one()) {
      int it = 0;
      for (int item = i0; item < i1; ++item, ++it) {
        const int s = it % STAGES;
        mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
        const int t = item / halves, h = item - t * halves;
        const int n = (int)g.fTP.div((unsigned)t), tile = t - n * g.TP;
        const int ty = (int)g.ftw.div((unsigned)tile), tx = tile - ty * g.tw;
        mbar_arrive_expect_tx(&full[s], 36 * 128);
        tma_load_4d(sA + s * A_BYTES, &amap, &full[s], h * 128, 4 * tx - g.pad, 4 * ty - g.pad, n);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_i8(128, NCOL) | (1u << 15);  // A MN-major
      int it = 0;
      for (int item = i0; item < i1; ++item, ++it) {
        const int s = it % STAGES, a = it & 1;
        mbar_wait(&accempty[a], ((it >> 1) & 1) ^ 1);
        mbar_wait(&full[s], (it / STAGES) & 1);
        tc_fence_after();
        const uint32_t base = smem_u32(sA + s * A_BYTES);
#pragma unroll
        for (int k = 0; k < 2; ++k)
          umma_i8(tbase + (uint32_t)(a * 256), desc_mn_sw128(base + k * 32 * 128), smem_desc_kmajor(sB + k * 32, 64),
                  idesc, k);
        umma_commit(&empty[s]);
        umma_commit(&accfull[a]);
      }
    }
    __syncwarp();
  } else {
    const int q = warp & 3, pt = (warp - 2) >> 2, e0 = 18 * pt;  // outputs e0 .. e0 + 17
    int cur_g = -1, run_T = 0, run_t = 0;
    auto flush = [&]() {  // publish the running group maxima (as record_unit would, in fp32 bits)
      if (cur_g >= 0 && lane == 0) {
        if (run_T > 0) atomicMax(&acc[(size_t)cur_g * ST_COUNT + ST_IBC].MF, __float_as_uint((float)run_T));
        if (run_t > 0) atomicMax(&acc[(size_t)cur_g * ST_COUNT + ST_IBC].TM, __float_as_uint((float)run_t));
      }
      run_T = run_t = 0;
    };
    int it = 0;
    for (int item = i0; item < i1; ++item, ++it) {
      const int a = it & 1;
      const int t = item / halves, h = item - t * halves;
      const int c = h * 128 + 32 * q + lane;
      mbar_wait(&accfull[a], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t ta = tbase + (uint32_t(32 * q) << 16) + (uint32_t)(a * 256);
      uint32_t r[90];
      tmem_ld18(ta + e0, r);
      tmem_ld18(ta + 36 + e0, r + 18);
      tmem_ld18(ta + 72 + e0, r + 36);
      tmem_ld18(ta + TMP0 + e0, r + 54);
      tmem_ld18(ta + TMP0 + 36 + e0, r + 72);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&accempty[a]);
      int vmax = 0, vmin = 0, wmax = 0, wmin = 0;
#pragma unroll
      for (int e = 0; e < 18; e += 2) {
        const int v0 = (int)r[e] + ((int)r[18 + e] << 8) + ((int)r[36 + e] << 16);
        const int v1 = (int)r[e + 1] + ((int)r[19 + e] << 8) + ((int)r[37 + e] << 16);
        vmax = __vimax3_s32(vmax, v0, v1);
        vmin = __vimin3_s32(vmin, v0, v1);
        const int w0 = (int)r[54 + e] + ((int)r[72 + e] << 8), w1 = (int)r[55 + e] + ((int)r[73 + e] << 8);
        wmax = __vimax3_s32(wmax, w0, w1);
        wmin = __vimin3_s32(wmin, w0, w1);
      }
      int mT = max(vmax, -vmin), mt = max(wmax, -wmin);
      // the two warps of a lane quarter meet at named barrier 1 + q; the second hands over its maxima
      int2* slot = part + (it & 1) * 128 + 32 * q + lane;
      if (pt == 1) *slot = make_int2(mT, mt);
      asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
      if (pt == 0) {
        const int2 o = *slot;
        mT = max(mT, o.x);
        mt = max(mt, o.y);
        const int grp = (int)g.fipg.div(g.fTP.div((unsigned)t));
        const bool active = c < g.C;
        if (g.C & 31) {
          record_unit((float)mT, (float)mt, grp, active, acc, ST_IBC, tabs.t[ST_IBC], t, c, g.C);
        } else {
          // the warp's 32 channels are one aligned table chunk of one group: exact warp maxima
          int wT = active ? mT : 0, wt = active ? mt : 0;
#pragma unroll
          for (int o2 = 16; o2 > 0; o2 >>= 1) {
            wT = max(wT, __shfl_xor_sync(0xffffffffu, wT, o2));
            wt = max(wt, __shfl_xor_sync(0xffffffffu, wt, o2));
          }
          if (lane == 0 && c < g.C)  // chunks past C (padding channels) have no table entry
            tabs.t[ST_IBC][(size_t)t * (g.C >> 5) + (c >> 5)] = __float_as_uint((float)wT);
          if (grp != cur_g) {
            flush();
            cur_g = grp;
          }
          run_T = max(run_T, wT);
          run_t = max(run_t, wt);
        }
      }
    }
    flush();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

}  // namespace tc
}  // namespace wl
