// Winograd-domain channel contraction (reference: _kernels.py:94-105 `_hadamard_accumulate_nb`,
// called from pipeline.py:143-145) as 36 batched int8 tensor-core GEMMs on sm_100a:
//
//     I[xi][t][o] = sum_c V[t][xi][c] * U[o][xi][c]        xi in 0..35, exact int32
//
// V (input-transform codes, [T][36][Cp]) and U (weight-transform codes, [Kp][36][Cp]) are int8,
// K-major; the TMA maps view them as 3-D {c, xi, row} with boxes {SW, 1, rows}.
// One CTA computes a 128 x BN tile of one xi with tcgen05.mma kind::i8 (M=128, N=BN, K=32 per
// instruction), operands staged by TMA into 128/64/32-byte-swizzled shared memory through a
// STAGES-deep mbarrier ring, accumulator in TMEM.  Warp roles: w0 TMA producer, w1 TMEM owner +
// single-thread MMA issuer, w2..w5 epilogue (tcgen05.ld 32 lanes each).  The epilogue is a
// template functor so the same mainloop serves the max pass and the requantisation pass.
#pragma once
#include "wl_ptx.cuh"

namespace wl {

constexpr int kGemmThreads = 192;

template <int BN, int SW, int STAGES>
struct GemmSmem {
  static constexpr int kA = 128 * SW;
  static constexpr int kB = BN * SW;
  static constexpr int kBytes = 1024 + STAGES * (kA + kB) + 256;
};

// Epilogue contract: Epi::begin(xi, row, valid), then Epi::apply(xi, row, col0, vals[16], nvalid) per
// thread for 16 consecutive columns of one row, then Epi::finish(xi, row, valid) once per thread
// (all 32 lanes of each epilogue warp reach finish, so it may use warp collectives).
template <int BN, int SW, int STAGES, class Epi>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_i8_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int T,
                   int Kout, int Cpad, Epi epi) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  using L = GemmSmem<BN, SW, STAGES>;
  uint8_t* sA = smem;
  uint8_t* sB = sA + STAGES * L::kA;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * L::kB);
  uint64_t* empty = full + STAGES;
  uint64_t* accfull = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accfull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * 128, n0 = blockIdx.y * BN, xi = blockIdx.z;
  const int kblocks = Cpad / SW;
  constexpr uint32_t kTmemCols = BN < 32 ? 32 : BN;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
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
        const int s = kb % STAGES;
        const uint32_t ph = (kb / STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], L::kA + L::kB);
        tma_load_3d(sA + s * L::kA, &tmA, &full[s], kb * SW, xi, m0);
        tma_load_3d(sB + s * L::kB, &tmB, &full[s], kb * SW, xi, n0);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_i8(128, BN);
      for (int kb = 0; kb < kblocks; ++kb) {
        const int s = kb % STAGES;
        const uint32_t ph = (kb / STAGES) & 1;
        mbar_wait(&full[s], ph);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < SW / 32; ++k) {
          const uint64_t ad = smem_desc_kmajor(sA + s * L::kA + k * 32, SW);
          const uint64_t bd = smem_desc_kmajor(sB + s * L::kB + k * 32, SW);
          umma_i8(tmem_base, ad, bd, idesc, (kb | k) != 0);
        }
        umma_commit(&empty[s]);
      }
      umma_commit(accfull);
    }
    __syncwarp();
  } else {
    mbar_wait(accfull, 0);
    tc_fence_after();
    const int q = warp & 3;
    const int row = m0 + 32 * q + lane;
    const uint32_t taddr = tmem_base + (uint32_t(32 * q) << 16);
    if constexpr (Epi::kPrefetch) epi.prefetch(row, row < T);
    epi.begin(xi, row, row < T);
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      uint32_t r0[16], r1[16];
      tmem_ld16(taddr + c, r0);
      tmem_ld16(taddr + c + 16, r1);
      tmem_ld_wait();
      const int col = n0 + c;
      const int nv0 = Kout - col, nv1 = Kout - col - 16;
      if (row < T && nv0 > 0) epi.apply(xi, row, col, r0, nv0 > 16 ? 16 : nv0);
      if (row < T && nv1 > 0) epi.apply(xi, row, col + 16, r1, nv1 > 16 ? 16 : nv1);
    }
    epi.finish(xi, row, row < T);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem_base);
  }
}

}  // namespace wl

namespace wl {

// ----------------------------------------------------------------------------------------------
// Persistent variant: one CTA per SM walks tiles (xi, m-block, n-block) round-robin.  TMEM holds two
// BN-column accumulators so the 8 epilogue warps drain tile i while the MMA warp fills tile i+1 and
// the TMA warp streams tile i+2's operands.  Barriers: smem ring full/empty[STAGES], accumulator
// full[2] (tcgen05.commit) / empty[2] (8 epilogue-warp arrivals).
// Column groups per TMEM lane quarter are the epilogue's choice (Epi::kGroups): 4 (16 epilogue
// warps) for the light max pass; 2 (8 warps, no spills under the register cap) for requantisation.
template <int G>
struct EpiShape {
  static constexpr int kGroups = G;
  static constexpr int kWarps = 4 * G;
  static constexpr int kThreads = 64 + 32 * kWarps;  // w0 TMA, w1 MMA + TMEM owner, w2.. epilogue
};

// Epilogue drain of one accumulator slice (HC columns of this warp's 32 TMEM lanes).
// Epis with kDeferSlow: the column loop is fully unrolled (staging offsets become immediates) and only
// runs the branch-free fast path; 16-column chunks whose fast path could not certify some element are
// collected in a bit mask and redone afterwards (one more tcgen05.ld of that chunk, warp-uniform loop),
// so the rare exact path and its call never sit inside the hot loop (requantisation pass 1.11 -> 1.07 ms).
template <int HC, class Epi>
__device__ __forceinline__ void epi_drain(Epi& epi, uint32_t taddr, int n0, int xi, int row, int T, int Kout) {
  static_assert(HC % 16 == 0, "epilogue column group must be a multiple of 16");
  if constexpr (Epi::kDeferSlow) {
    uint32_t slow = 0;
#pragma unroll
    for (int c = 0; c < HC; c += 32) {
      uint32_t r0[16], r1[16];
      tmem_ld16(taddr + c, r0);
      if (c + 16 < HC) tmem_ld16(taddr + c + 16, r1);
      tmem_ld_wait();
      const int col = n0 + c;
      if (row < T && Kout - col > 0) slow |= (uint32_t)epi.apply_fast(r0, c) << (c >> 4);
      if (c + 16 < HC && row < T && Kout - col - 16 > 0) slow |= (uint32_t)epi.apply_fast(r1, c + 16) << ((c >> 4) + 1);
    }
    uint32_t any = __reduce_or_sync(0xffffffffu, slow);
    while (any) {
      const int j = __ffs(any) - 1;
      any &= any - 1;
      uint32_t r[16];
      tmem_ld16(taddr + 16 * j, r);
      tmem_ld_wait();
      if ((slow >> j) & 1u) {
        const int col = n0 + 16 * j, nv = Kout - col;
        epi.apply_slow(xi, row, col, r, nv > 16 ? 16 : nv, 16 * j);
      }
    }
  } else {
#pragma unroll 1
    for (int c = 0; c < HC; c += 32) {
      uint32_t r0[16], r1[16];
      tmem_ld16(taddr + c, r0);
      if (c + 16 < HC) tmem_ld16(taddr + c + 16, r1);
      tmem_ld_wait();
      const int col = n0 + c;
      const int nv0 = Kout - col, nv1 = Kout - col - 16;
      if (row < T && nv0 > 0) epi.apply(xi, row, col, r0, nv0 > 16 ? 16 : nv0);
      if (c + 16 < HC && row < T && nv1 > 0) epi.apply(xi, row, col + 16, r1, nv1 > 16 ? 16 : nv1);
    }
  }
}

template <int BN, int SW, int STAGES, int EPI_STAGE = 0, int EPI_WARPS = 16>
struct GemmPSmem {
  static constexpr int kA = 128 * SW;
  static constexpr int kB = BN * SW;
  static constexpr int kEpi = EPI_WARPS * EPI_STAGE;  // per-epilogue-warp staging bytes
  static constexpr int kBytes = 1024 + STAGES * (kA + kB) + 512 + kEpi;
};

template <int BN, int SW, int STAGES, class Epi>
__global__ void __launch_bounds__(EpiShape<Epi::kGroups>::kThreads, 1)
    gemm_i8_persistent(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int T,
                       int Kout, int Cpad, int Kpad, Epi epi) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int kEpiGroups = Epi::kGroups, kEpiWarps = 4 * kEpiGroups;
  using L = GemmPSmem<BN, SW, STAGES, Epi::kStageBytes, kEpiWarps>;
  uint8_t* sA = smem;
  uint8_t* sB = sA + STAGES * L::kA;
  uint8_t* sEpi = sB + STAGES * L::kB;  // kEpiWarps x Epi::kStageBytes (16-byte aligned)
  uint64_t* full = reinterpret_cast<uint64_t*>(sEpi + L::kEpi);
  uint64_t* empty = full + STAGES;
  uint64_t* accfull = empty + STAGES;   // [2]
  uint64_t* accempty = accfull + 2;     // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kblocks = Cpad / SW;
  const int mblocks = (T + 127) / 128, nblocks = Kpad / BN;
  const int ntiles = 36 * mblocks * nblocks;
  constexpr uint32_t kTmemCols = 2 * BN <= 32 ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512)));

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&accfull[a], 1);
      mbar_init(&accempty[a], kEpiWarps);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // tile -> (xi, n-block, m-block), xi fastest: the CTAs in flight together cover all 36 elements of a
  // few m-blocks, i.e. whole contiguous [128 rows][36][C] regions of V and h (DRAM page locality);
  // U (36 x Kp x Cp bytes) stays L2-resident whatever the order.
  auto decode = [&](int tile, int& xi, int& mb, int& nb) {
    xi = tile % 36;
    const int r = tile / 36;
    nb = r % nblocks;
    mb = r / nblocks;
  };

  if (warp == 0) {
    if (elect_one()) {
      int it = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        int xi, mb, nb;
        decode(tile, xi, mb, nb);
        for (int kb = 0; kb < kblocks; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], L::kA + L::kB);
          tma_load_3d(sA + s * L::kA, &tmA, &full[s], kb * SW, xi, mb * 128);
          tma_load_3d(sB + s * L::kB, &tmB, &full[s], kb * SW, xi, nb * BN);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_i8(128, BN);
      int it = 0, local = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++local) {
        const int a = local & 1;
        const uint32_t aph = (local >> 1) & 1;
        mbar_wait(&accempty[a], aph ^ 1);
        tc_fence_after();
        const uint32_t dacc = tmem_base + (uint32_t)(a * BN);
        for (int kb = 0; kb < kblocks; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&full[s], ph);
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < SW / 32; ++k) {
            const uint64_t ad = smem_desc_kmajor(sA + s * L::kA + k * 32, SW);
            const uint64_t bd = smem_desc_kmajor(sB + s * L::kB + k * 32, SW);
            umma_i8(dacc, ad, bd, idesc, (kb | k) != 0);
          }
          umma_commit(&empty[s]);
        }
        umma_commit(&accfull[a]);
      }
    }
    __syncwarp();
  } else {
    const int ew = warp - 2;          // 0..kEpiWarps-1
    const int q = warp & 3;           // TMEM lane quarter this warp may access
    const int half = ew >> 2;         // column group of the tile
    constexpr int HC = BN / kEpiGroups;
    if constexpr (Epi::kStageBytes > 0) epi.set_stage(sEpi + ew * Epi::kStageBytes, HC);
    int local = 0;
    // Epis with prefetch(): the next tile's per-row parameters are loaded one tile ahead, so their
    // global-load latency hides behind this tile's drain instead of stalling the epilogue warp
    constexpr bool kPre = Epi::kPrefetch;
    if constexpr (kPre) {
      if ((int)blockIdx.x < ntiles) {
        int xi, mb, nb;
        decode(blockIdx.x, xi, mb, nb);
        epi.prefetch(mb * 128 + 32 * q + lane, mb * 128 + 32 * q + lane < T);
      }
    }
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++local) {
      int xi, mb, nb;
      decode(tile, xi, mb, nb);
      const int a = local & 1;
      const uint32_t aph = (local >> 1) & 1;
      const int row = mb * 128 + 32 * q + lane;
      // per-row parameters (global loads) before the wait: their latency overlaps the MMA
      epi.begin(xi, row, row < T);
      if constexpr (kPre) {
        if (tile + (int)gridDim.x < ntiles) {
          int xn, mn, nn;
          decode(tile + gridDim.x, xn, mn, nn);
          epi.prefetch(mn * 128 + 32 * q + lane, mn * 128 + 32 * q + lane < T);
        }
      }
      mbar_wait(&accfull[a], aph);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (uint32_t(32 * q) << 16) + (uint32_t)(a * BN + half * HC);
      const int n0 = nb * BN + half * HC;
      epi_drain<HC>(epi, taddr, n0, xi, row, T, Kout);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&accempty[a]);
      epi.finish_chunk(xi, row, row < T, nb * kEpiGroups + half);
      if constexpr (Epi::kStageBytes > 0) epi.flush(xi, mb * 128 + 32 * q, n0, HC, T, lane);
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

namespace wl {

// ----------------------------------------------------------------------------------------------
// B-stationary variant: every CTA owns one B tile (Winograd element xi, output-channel block nb) —
// U_xi's BN x Cpad codes stay resident in shared memory (one TMA load) — and walks a contiguous range
// of m-blocks of that xi, so only the A operand (V) streams through the ring: 1/3 of the persistent
// kernel's shared-memory fill per tile for Cpad = Kout = 256.  The nslots CTAs sharing a B tile split
// its m-blocks into contiguous ranges (measured: 0.59 ms vs 0.62 ms with round-robin m-blocks on
// config 4).  grid >= 36 * nblocks always (ntiles = 36 * nblocks * mblocks).  Same epilogue contract
// and TMEM double buffering as gemm_i8_persistent.  Used for the max pass (0.58 -> 0.49 ms kernel on
// config 4); the requantisation pass is epilogue-bound and measured slower with it (1.12 -> 1.21 ms).
template <int BN, int SW, int STAGES, int EPI_STAGE, int EPI_WARPS>
struct GemmBSmem {
  static constexpr int kA = 128 * SW;
  static constexpr int kEpi = EPI_WARPS * EPI_STAGE;
  static constexpr int bytes(int kblocks) { return 1024 + kblocks * BN * SW + STAGES * kA + kEpi + 512; }
};

template <int BN, int SW, int STAGES, class Epi>
__global__ void __launch_bounds__(EpiShape<Epi::kGroups>::kThreads, 1)
    gemm_i8_bstat(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int T, int Kout,
                  int Cpad, int Kpad, Epi epi) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int kEpiGroups = Epi::kGroups, kEpiWarps = 4 * kEpiGroups;
  using L = GemmBSmem<BN, SW, STAGES, Epi::kStageBytes, kEpiWarps>;
  const int kblocks = Cpad / SW;
  uint8_t* sB = smem;                          // [kblocks][BN rows][SW bytes]
  uint8_t* sA = sB + kblocks * BN * SW;        // ring [STAGES][128 rows][SW bytes]
  uint8_t* sEpi = sA + STAGES * L::kA;
  uint64_t* full = reinterpret_cast<uint64_t*>(sEpi + L::kEpi);
  uint64_t* empty = full + STAGES;
  uint64_t* accfull = empty + STAGES;  // [2]
  uint64_t* accempty = accfull + 2;    // [2]
  uint64_t* bfull = accempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mblocks = (T + 127) / 128, nblocks = Kpad / BN, nkeys = 36 * nblocks;
  const int key = (int)blockIdx.x % nkeys, slot = (int)blockIdx.x / nkeys;
  const int nslots = ((int)gridDim.x - key + nkeys - 1) / nkeys;
  const int mb0 = (int)((long long)slot * mblocks / nslots), mb1 = (int)((long long)(slot + 1) * mblocks / nslots);
  constexpr int mstep = 1;
  const int xi = key % 36, nb = key / 36;
  constexpr uint32_t kTmemCols = 2 * BN <= 32 ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512)));

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&accfull[a], 1);
      mbar_init(&accempty[a], kEpiWarps);
    }
    mbar_init(bfull, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      mbar_arrive_expect_tx(bfull, (uint32_t)(kblocks * BN * SW));
      for (int kb = 0; kb < kblocks; ++kb) tma_load_3d(sB + kb * BN * SW, &tmB, bfull, kb * SW, xi, nb * BN);
      int it = 0;
      for (int mb = mb0; mb < mb1; mb += mstep)
        for (int kb = 0; kb < kblocks; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], L::kA);
          tma_load_3d(sA + s * L::kA, &tmA, &full[s], kb * SW, xi, mb * 128);
        }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_i8(128, BN);
      mbar_wait(bfull, 0);
      tc_fence_after();
      int it = 0, local = 0;
      for (int mb = mb0; mb < mb1; mb += mstep, ++local) {
        const int a = local & 1;
        const uint32_t aph = (local >> 1) & 1;
        mbar_wait(&accempty[a], aph ^ 1);
        tc_fence_after();
        const uint32_t dacc = tmem_base + (uint32_t)(a * BN);
        for (int kb = 0; kb < kblocks; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&full[s], ph);
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < SW / 32; ++k) {
            const uint64_t ad = smem_desc_kmajor(sA + s * L::kA + k * 32, SW);
            const uint64_t bd = smem_desc_kmajor(sB + kb * BN * SW + k * 32, SW);
            umma_i8(dacc, ad, bd, idesc, (kb | k) != 0);
          }
          umma_commit(&empty[s]);
        }
        umma_commit(&accfull[a]);
      }
    }
    __syncwarp();
  } else {
    const int ew = warp - 2;
    const int q = warp & 3;
    const int half = ew >> 2;
    constexpr int HC = BN / kEpiGroups;
    static_assert(HC % 16 == 0, "epilogue column group must be a multiple of 16");
    if constexpr (Epi::kStageBytes > 0) epi.set_stage(sEpi + ew * Epi::kStageBytes, HC);
    constexpr bool kPre = Epi::kPrefetch;
    if constexpr (kPre) {
      if (mb0 < mb1) epi.prefetch(mb0 * 128 + 32 * q + lane, mb0 * 128 + 32 * q + lane < T);
    }
    int local = 0;
    const int n0 = nb * BN + half * HC;
    for (int mb = mb0; mb < mb1; mb += mstep, ++local) {
      const int a = local & 1;
      const uint32_t aph = (local >> 1) & 1;
      const int row = mb * 128 + 32 * q + lane;
      epi.begin(xi, row, row < T);
      if constexpr (kPre) {
        const int mn = mb + mstep;
        if (mn < mb1) epi.prefetch(mn * 128 + 32 * q + lane, mn * 128 + 32 * q + lane < T);
      }
      mbar_wait(&accfull[a], aph);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (uint32_t(32 * q) << 16) + (uint32_t)(a * BN + half * HC);
      epi_drain<HC>(epi, taddr, n0, xi, row, T, Kout);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&accempty[a]);
      epi.finish_chunk(xi, row, row < T, nb * kEpiGroups + half);
      if constexpr (Epi::kStageBytes > 0) epi.flush(xi, mb * 128 + 32 * q, n0, HC, T, lane);
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
