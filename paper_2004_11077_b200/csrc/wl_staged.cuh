// Persistent, double-buffered staging of the transform kernels' inputs into shared memory.
//
// The 36 codes of every (tile, channel) unit of a tile live in one contiguous block:
//   * [T][36][LD] layouts (c1, h, c4): tile t's block is 36*LD elements at t*36*LD -> one 1-D bulk
//     copy (cp.async.bulk) per TPB consecutive tiles;
//   * NHWC input codes c0: tile t's 6x6 window for all channels is a 4-D TMA box {LD, 6, 6, 1} at
//     (0, 4*tx - pad, 4*ty - pad, n); TMA zero-fills the padding and the pad-to-tile spill.
// Both land as [36][LD] (element e = 6*i + j, channel fastest).  A block of TPB*LD threads (one unit
// each, channel fastest) walks tile groups grid-stride; thread 0 prefetches group k+1 into the other
// buffer while group k is computed, completion tracked by one mbarrier per buffer.
#pragma once
#include "wl_f2.cuh"
#include "wl_kernels2.cuh"
#include "wl_ptx.cuh"

namespace wl {

template <int LD, int EB>
struct Staged {
  static_assert(LD <= 256, "staged path handles up to 256 padded channels");
  static constexpr int TPB = 256 / LD;  // tiles per iteration
  static constexpr int THREADS = TPB * LD;
  static constexpr int TILE_BYTES = 36 * LD * EB;
  static constexpr int STAGE_BYTES = TPB * TILE_BYTES;
  static constexpr int SMEM = 2 * STAGE_BYTES + 16;
  // with int8 code output staged in shared memory and bulk-stored per tile group
  static constexpr int OUT_TILE = 36 * LD;
  static constexpr int OUT_BYTES = TPB * OUT_TILE;
  static constexpr int SMEM_OUT = 2 * STAGE_BYTES + 2 * OUT_BYTES + 16;
};

// `nch` = number of real channels of the unit axis (g.C for input-side kernels, g.K for output-side).
// With `out` != nullptr the body also receives the thread's [36][LD] int8 output block in shared
// memory (element e of channel c at so[e * LD + c]); each tile group's blocks are written to
// out + t0 * 36 * LD by one cp.async.bulk store (padded channels are zero-filled), replacing 36
// byte stores per unit with 32-bit shared stores.
template <int LD, int EB, bool kC0, class Body>
__device__ __forceinline__ void staged_loop(const Geo& g, int nch, const void* planes, const CUtensorMap* c0map,
                                            Body&& body, int8_t* out = nullptr) {
  using S = Staged<LD, EB>;
  extern __shared__ __align__(128) uint8_t wl_stage_smem[];
  uint8_t* sm = wl_stage_smem;
  const bool kout = out != nullptr;
  uint8_t* osm = sm + 2 * S::STAGE_BYTES;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 2 * S::STAGE_BYTES + (kout ? 2 * S::OUT_BYTES : 0));
  const int niter = (g.T + S::TPB - 1) / S::TPB;
  const int tl = threadIdx.x / LD, c = threadIdx.x % LD;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
    if (kC0) tma_prefetch_desc(c0map);
  }
  __syncthreads();
  auto issue = [&](int it, int s) {
    const int t0 = it * S::TPB;
    const int nt = min(S::TPB, g.T - t0);
    uint8_t* dst = sm + s * S::STAGE_BYTES;
    mbar_arrive_expect_tx(&bar[s], (uint32_t)(nt * S::TILE_BYTES));
    if constexpr (!kC0) {
      bulk_g2s(dst, reinterpret_cast<const uint8_t*>(planes) + (size_t)t0 * S::TILE_BYTES, (uint32_t)(nt * S::TILE_BYTES),
               &bar[s]);
    } else {
      for (int k = 0; k < nt; ++k) {
        const int t = t0 + k, n = (int)g.fTP.div((unsigned)t), tile = t - n * g.TP;
        const int ty = (int)g.ftw.div((unsigned)tile), tx = tile - ty * g.tw;
        tma_load_4d(dst + k * S::TILE_BYTES, c0map, &bar[s], 0, 4 * tx - g.pad, 4 * ty - g.pad, n);
      }
    }
  };
  if (threadIdx.x == 0 && (int)blockIdx.x < niter) issue(blockIdx.x, 0);
  int k = 0;
  for (int it = blockIdx.x; it < niter; it += gridDim.x, ++k) {
    const int s = k & 1;
    if (threadIdx.x == 0 && it + (int)gridDim.x < niter) issue(it + gridDim.x, s ^ 1);
    mbar_wait(&bar[s], (uint32_t)((k >> 1) & 1));
    const int t = it * S::TPB + tl;
    int8_t* so = reinterpret_cast<int8_t*>(osm + s * S::OUT_BYTES + tl * S::OUT_TILE);
    body(t, c, t < g.T && c < nch, sm + s * S::STAGE_BYTES + tl * S::TILE_BYTES, so);
    if (kout) {
      if (c >= nch)
#pragma unroll
        for (int e = 0; e < 36; ++e) so[e * LD + c] = 0;
      fence_proxy_async_smem();
      if (threadIdx.x == 0) bulk_wait_read<0>();  // the store issued last iteration has read buffer s^1
    }
    __syncthreads();
    if (kout && threadIdx.x == 0) {
      const int t0 = it * S::TPB, nt = min(S::TPB, g.T - t0);
      bulk_s2g(out + (size_t)t0 * S::OUT_TILE, osm + s * S::OUT_BYTES, (uint32_t)(nt * S::OUT_TILE));
      bulk_commit();
    }
  }
  if (kout && threadIdx.x == 0) bulk_wait_all<0>();
}

// X[i][j] of unit channel c from a staged [36][LD] block.
template <int LD, typename HT, typename XT>
__device__ __forceinline__ void stage_x(const uint8_t* st, int c, XT (&X)[6][6]) {
  const HT* p = reinterpret_cast<const HT*>(st) + c;
#pragma unroll
  for (int e = 0; e < 36; ++e) X[e / 6][e % 6] = to_x<XT>((int)p[e * LD]);
}

// ---------------------------------------------------------------------------------- input side

template <int MODE, int LD>
__global__ void __launch_bounds__(Staged<LD, 1>::THREADS, WL_MINB)
    sin_a_kernel(const __grid_constant__ CUtensorMap c0map, Geo g, Acc* __restrict__ acc, Tables tabs) {
  staged_loop<LD, 1, true>(g, g.C, nullptr, &c0map, [&](int t, int c, bool active, const uint8_t* st, int8_t* so) {
    float X[6][6];
    stage_x<LD, int8_t>(st, c, X);
    const int grp = (int)g.fipg.div(g.fTP.div((unsigned)t));
    constexpr int stg = MODE == 0 ? ST_IT : ST_IBC;
    float m = 0.f, tm = 0.f;
    auto mx = [&](int, const float (&col)[6]) {
#pragma unroll
      for (int i = 0; i < 6; ++i) m = fmaxf(m, fabsf(col[i]));
    };
    if constexpr (MODE == 0)
      sandwich_cols<tab::Can_IT>(X, mx, &tm);
    else
      sandwich_cols<tab::Leg_IBC>(X, mx, &tm);
    record_unit(m, tm, grp, active, acc, stg, tabs.t[stg], active ? t : 0, c, g.C, g.lazy);
  });
}

template <int LD>
__global__ void __launch_bounds__(Staged<LD, 1>::THREADS, WL_MINB)
    sin_b_kernel(const __grid_constant__ CUtensorMap c0map, const int8_t* __restrict__ c0, int8_t* __restrict__ c1,
                 Geo g, Bits b, Acc* __restrict__ acc, const PlanF64* __restrict__ pf, Tables tabs, FixList fl) {
  staged_loop<LD, 1, true>(g, g.C, nullptr, &c0map, [&](int t, int c, bool active, const uint8_t* st, int8_t* so) {
    const int tt = active ? t : 0;
    const int n = (int)g.fTP.div((unsigned)tt), tile = (int)g.fTP.mod((unsigned)tt), grp = (int)g.fipg.div((unsigned)n);
    const Acc* ga = acc + (size_t)grp * ST_COUNT;
    const float r = ga[ST_IBC].r, thr = ga[ST_IBC].thr, ef = ga[ST_IBC].ef;
    int8_t* dst = so + c;  // staged output block, bulk-stored to c1
    float K1[6][6];
    bool deferred = false;
    {
      float X[6][6];
      stage_x<LD, int8_t>(st, c, X);
      float dmax = 0.f;
      sandwich_cols<tab::Leg_IBC>(X, [&](int j, const float (&col)[6], float cm) {
        float dcol = 0.f;
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          const int code = rq_col(col[i], r, K1[i][j], dcol);
          dst[(6 * i + j) * LD] = (int8_t)code;
        }
        dmax = fmaxf(dmax, fmaf(ef * cm, max_row_abs_sum<tab::Leg_IBC>(), dcol));
      });
      const bool want = dmax > thr && active;
      deferred = defer_fix(fl, FIX_IBC, (unsigned)tt * (unsigned)g.C + (unsigned)c, want);
      if (want && !deferred) {
        const C0Win win(c0, g, n, tile, c, LD);
        fix_unit<tab::Leg_IBC>(SrcC0{win}, r, thr, ef, ga + ST_IBC, b.q[ST_IBC], ga + ST_INPUT, b.q[ST_INPUT], true,
                               pf->ibc, [dst](int i, int j, int code) { dst[(6 * i + j) * LD] = (int8_t)code; });
#pragma unroll
        for (int e = 0; e < 36; ++e) K1[e / 6][e % 6] = (float)dst[e * LD];
      }
    }
    float m = 0.f, tm = 0.f;
    sandwich_cols<tab::Leg_IT>(K1, [&](int, const float (&col)[6]) {
#pragma unroll
      for (int i = 0; i < 6; ++i) m = fmaxf(m, fabsf(col[i]));
    }, &tm);
    if (deferred) m = tm = 0.f;  // recorded by fixup_ibc_kernel from the exact codes
    record_unit(m, tm, grp, active, acc, ST_IT, tabs.t[ST_IT], tt, c, g.C, g.lazy);
  }, c1);
}

// V codes: canonical from the c0 window (B^T), Legendre from staged c1 (B_P^T).
template <int MODE, int LD>
__global__ void __launch_bounds__(Staged<LD, 1>::THREADS, WL_MINB)
    sin_c_kernel(const __grid_constant__ CUtensorMap c0map, const int8_t* __restrict__ c0,
                 const int8_t* __restrict__ c1, int8_t* __restrict__ V, const __grid_constant__ Geo g, const __grid_constant__ Bits b, Acc* __restrict__ acc,
                 const PlanF64* __restrict__ pf, FixList fl) {
  staged_loop<LD, 1, MODE == 0>(g, g.C, c1, &c0map, [&](int t, int c, bool active, const uint8_t* st, int8_t* so) {
    if (!active) return;
    const int n = (int)g.fTP.div((unsigned)t), tile = (int)g.fTP.mod((unsigned)t), grp = (int)g.fipg.div((unsigned)n);
    const Acc* ga = acc + (size_t)grp * ST_COUNT;
    const float r = ga[ST_IT].r, thr = ga[ST_IT].thr, ef = ga[ST_IT].ef;
    int8_t* dst = so + c;  // staged output block, bulk-stored to V
    float X[6][6];
    stage_x<LD, int8_t>(st, c, X);
    float dmax = 0.f, kd;
    using LIT = std::conditional_t<MODE == 0, tab::Can_IT, tab::Leg_IT>;
    sandwich_cols<LIT>(X, [&](int j, const float (&col)[6], float cm) {
      float dcol = 0.f;
#pragma unroll
      for (int i = 0; i < 6; ++i) dst[(6 * i + j) * LD] = (int8_t)rq_col(col[i], r, kd, dcol);
      dmax = fmaxf(dmax, fmaf(ef * cm, max_row_abs_sum<LIT>(), dcol));
    });
    const bool want = dmax > thr;
    if (want && !defer_fix(fl, FIX_IT, (unsigned)t * (unsigned)g.C + (unsigned)c, want))
      fix_it_unit<MODE>(c0, c1, dst, LD, g, b, acc, pf, t, c, LD);
  }, V);
}

// ---------------------------------------------------------------------------------- output side

template <int MODE, typename HT, int LD>
__global__ void __launch_bounds__(Staged<LD, sizeof(HT)>::THREADS, WL_MINB)
    sout_a_kernel(const HT* __restrict__ h, Geo g, Acc* __restrict__ acc, Tables tabs) {
  staged_loop<LD, sizeof(HT), false>(g, g.K, h, nullptr, [&](int t, int k, bool active, const uint8_t* st, int8_t* so) {
    const int tt = active ? t : 0;
    const int n = (int)g.fTP.div((unsigned)tt), tile = (int)g.fTP.mod((unsigned)tt), grp = (int)g.fipg.div((unsigned)n);
    const int ty = (int)g.ftw.div((unsigned)tile), tx = (int)g.ftw.mod((unsigned)tile);
    float X[6][6];
    stage_x<LD, HT>(st, k, X);
    float m = 0.f, tm = 0.f;
    constexpr int stg = MODE == 0 ? ST_OUT : ST_OBC;
    if constexpr (MODE == 0) {
      sandwich_cols<tab::Can_OT>(X, [&](int j, const float (&col)[4]) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (4 * ty + i < g.Ho && 4 * tx + j < g.Wo) m = fmaxf(m, fabsf(col[i]));
      }, &tm);
    } else {
      sandwich_cols<tab::Leg_OBC>(X, [&](int, const float (&col)[6]) {
#pragma unroll
        for (int i = 0; i < 6; ++i) m = fmaxf(m, fabsf(col[i]));
      }, &tm);
    }
    record_unit(m, tm, grp, active, acc, stg, tabs.t[stg], tt, k, g.K, g.lazy);
  });
}

template <typename HT, int LD>
__global__ void __launch_bounds__(Staged<LD, sizeof(HT)>::THREADS, WL_MINB)
    sout_b_kernel(const HT* __restrict__ h, int8_t* __restrict__ c4, Geo g, Bits b, Acc* __restrict__ acc,
                  const PlanF64* __restrict__ pf, Tables tabs, FixList fl) {
  staged_loop<LD, sizeof(HT), false>(g, g.K, h, nullptr, [&](int t, int k, bool active, const uint8_t* st, int8_t* so) {
    const int tt = active ? t : 0;
    const int n = (int)g.fTP.div((unsigned)tt), tile = (int)g.fTP.mod((unsigned)tt), grp = (int)g.fipg.div((unsigned)n);
    const Acc* ga = acc + (size_t)grp * ST_COUNT;
    const float r = ga[ST_OBC].r, thr = ga[ST_OBC].thr, ef = ga[ST_OBC].ef;
    constexpr uint32_t plane = LD;
    const uint32_t off = (uint32_t)tt * 36u * LD + k;
    int8_t* dst = so + k;  // staged output block, bulk-stored to c4
    float K4[6][6];
    bool deferred = false;
    {
      float X[6][6];
      stage_x<LD, HT>(st, k, X);
      float dmax = 0.f;
      sandwich_cols<tab::Leg_OBC>(X, [&](int j, const float (&col)[6], float cm) {
        float dcol = 0.f;
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          const int code = rq_col(col[i], r, K4[i][j], dcol);
          dst[(6 * i + j) * LD] = (int8_t)code;
        }
        dmax = fmaxf(dmax, fmaf(ef * cm, max_row_abs_sum<tab::Leg_OBC>(), dcol));
      });
      const bool want = dmax > thr && active;
      deferred = defer_fix(fl, FIX_OBC, (unsigned)tt * (unsigned)g.K + (unsigned)k, want);
      if (want && !deferred) {
        fix_unit<tab::Leg_OBC>(SrcPlanes<HT>{h, plane, off}, r, thr, ef, ga + ST_OBC, b.q[ST_OBC], ga + ST_HAD,
                               b.q[ST_HAD], false, pf->obc,
                               [dst](int i, int j, int code) { dst[(6 * i + j) * LD] = (int8_t)code; });
#pragma unroll
        for (int e = 0; e < 36; ++e) K4[e / 6][e % 6] = (float)dst[e * LD];
      }
    }
    const int ty = (int)g.ftw.div((unsigned)tile), tx = (int)g.ftw.mod((unsigned)tile);
    float m = 0.f, tm = 0.f;
    sandwich_cols<tab::Leg_OT>(K4, [&](int j, const float (&col)[4]) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (4 * ty + i < g.Ho && 4 * tx + j < g.Wo) m = fmaxf(m, fabsf(col[i]));
    }, &tm);
    if (deferred) m = tm = 0.f;  // recorded by fixup_obc_kernel from the exact codes
    record_unit(m, tm, grp, active, acc, ST_OUT, tabs.t[ST_OUT], tt, k, g.K, g.lazy);
  }, c4);
}

// Output code pass (y), staged both ways.  A work item is TPB=8 consecutive tiles x KB=32 output
// channels: one 3-D TMA box {32 channels, 36 elements, 8 tiles} of the [T][36][Kp] codes (c4, or h
// for canonical) lands as [tile][36][32]; warp w computes tile w, lane = channel (conflict-free byte
// reads).  The 4x4 dequantised outputs go to a padded shared block [channel][tile][4][4(+pad)] and
// leave as float4 rows, tile fastest, so a warp stores 4 rows x 8 tiles = 4 contiguous 128-byte
// runs of y instead of 32 scattered 16-byte pieces (the plain out_c_kernel's lg_throttle).
struct StagedOut {
  static constexpr int TPB = 8, KB = 32, THREADS = 256;
  static constexpr int OT = 20;             // floats per tile (16 + 4 pad)
  static constexpr int OK = TPB * OT + 4;   // floats per channel (bank offset 4 words per channel)
  static constexpr int OUT_BYTES = KB * OK * 4;
  template <typename ST>
  static constexpr int in_bytes() { return TPB * 36 * KB * (int)sizeof(ST); }
  template <typename ST>
  static constexpr int smem() { return 2 * in_bytes<ST>() + OUT_BYTES + 16; }
};

template <int MODE, typename HT, bool TAB>
__global__ void __launch_bounds__(StagedOut::THREADS, 3)
    sout_c_kernel(const __grid_constant__ CUtensorMap srcmap, const HT* __restrict__ h,
                  const int8_t* __restrict__ c4, float* __restrict__ y, const float* __restrict__ bias,
                  const __grid_constant__ Geo g, const __grid_constant__ Bits b, const Acc* __restrict__ acc,
                  const PlanF64* __restrict__ pf, const float* __restrict__ otab, const float4* __restrict__ odq,
                  FixList fl) {
  using S = StagedOut;
  using ST = std::conditional_t<MODE == 0, HT, int8_t>;  // staged code type
  constexpr int IN_TILE = 36 * S::KB * (int)sizeof(ST);
  constexpr int IN_BYTES = S::in_bytes<ST>();
  extern __shared__ __align__(128) uint8_t wl_stage_smem[];
  uint8_t* sm = wl_stage_smem;
  float* so = reinterpret_cast<float*>(sm + 2 * IN_BYTES);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 2 * IN_BYTES + S::OUT_BYTES);
  __shared__ long long ybase[S::TPB];  // y offset of (n, k0, 4*ty, 4*tx) per tile of the item, -1 if t >= T
  __shared__ int yrows[S::TPB];        // rows of the tile inside Ho
  const int nkb = (g.K + S::KB - 1) / S::KB;
  const int niter = ((g.T + S::TPB - 1) / S::TPB) * nkb;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qo = b.q[ST_OUT];
  const long long plane = (long long)g.Ho * g.Wo;
  using LOT = std::conditional_t<MODE == 0, tab::Can_OT, tab::Leg_OT>;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
    tma_prefetch_desc(&srcmap);
  }
  __syncthreads();
  auto issue = [&](int it, int s) {
    const int tg = it / nkb, kb = it - tg * nkb;
    mbar_arrive_expect_tx(&bar[s], (uint32_t)IN_BYTES);
    tma_load_3d(sm + s * IN_BYTES, &srcmap, &bar[s], kb * S::KB, 0, tg * S::TPB);
  };
  if (threadIdx.x == 0 && (int)blockIdx.x < niter) issue(blockIdx.x, 0);
  int kk = 0;
  for (int it = blockIdx.x; it < niter; it += gridDim.x, ++kk) {
    const int s = kk & 1;
    if (threadIdx.x == 0 && it + (int)gridDim.x < niter) issue(it + gridDim.x, s ^ 1);
    const int tg = it / nkb, kb = it - tg * nkb;
    const int t0 = tg * S::TPB, k0 = kb * S::KB;
    if (threadIdx.x < S::TPB) {
      const int t = t0 + threadIdx.x;
      long long base = -1;
      int rows = 0;
      if (t < g.T) {
        const int n = (int)g.fTP.div((unsigned)t), tile = t - n * g.TP;
        const int ty = (int)g.ftw.div((unsigned)tile), tx = tile - ty * g.tw;
        base = ((long long)n * g.K + k0) * plane + (long long)(4 * ty) * g.Wo + 4 * tx;
        rows = min(4, g.Ho - 4 * ty);
      }
      ybase[threadIdx.x] = base;
      yrows[threadIdx.x] = rows;
    }
    mbar_wait(&bar[s], (uint32_t)((kk >> 1) & 1));
    {
      const int t = t0 + w, k = k0 + lane;
      const bool active = t < g.T && k < g.K;
      const int tt = active ? t : 0;
      const int grp = (int)g.fipg.div(g.fTP.div((unsigned)tt));
      const Acc* ga = acc + (size_t)grp * ST_COUNT;
      // inactive lanes (padded channels hold arbitrary codes) requantise with r = 0 -> code 0
      const float r = active ? ga[ST_OUT].r : 0.f, thr = ga[ST_OUT].thr, ef = ga[ST_OUT].ef;
      const float* tabg = TAB ? otab + (size_t)grp * (2 * qo + 1) + qo : nullptr;
      const double scale = ga[ST_OUT].scale;
      const double maxabs = __longlong_as_double((long long)ga[ST_OUT].F);
      auto deqf = [=](int code) -> float {
        if constexpr (TAB)
          return __ldg(tabg + code);
        else
          return code == qo ? (float)maxabs : (code == -qo ? (float)-maxabs : (float)((double)code * scale));
      };
      const float bk = (bias && active) ? __ldg(&bias[k]) : 0.f;
      float X[6][6];
      {
        const ST* p = reinterpret_cast<const ST*>(sm + s * IN_BYTES + w * IN_TILE) + lane;
#pragma unroll
        for (int e = 0; e < 36; ++e) X[e / 6][e % 6] = to_x<float>((int)p[e * S::KB]);
      }
      float* o = so + lane * S::OK + w * S::OT;
      float dmax = 0.f, kd;
      // group with a certified arithmetic dequantisation (out_table_kernel): two fp32 ops per output
      // instead of a table gather
      float s_hi = 0.f, s_lo = 0.f;
      bool arith = false;
      if constexpr (TAB) {
        const float4 dq = __ldg(&odq[grp]);
        s_hi = dq.x, s_lo = dq.y, arith = dq.z != 0.f;
      }
      if (arith) {
        sandwich_cols<LOT>(X, [&](int j, const float (&col)[4], float cm) {
          float dcol = 0.f;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            rq_col(col[i], r, kd, dcol);
            o[4 * i + j] = __fadd_rn(__fmaf_rn(kd, s_hi, __fmul_rn(kd, s_lo)), bk);
          }
          dmax = fmaxf(dmax, fmaf(ef * cm, max_row_abs_sum<LOT>(), dcol));
        });
      } else {
        sandwich_cols<LOT>(X, [&](int j, const float (&col)[4], float cm) {
          float dcol = 0.f;
#pragma unroll
          for (int i = 0; i < 4; ++i) o[4 * i + j] = deqf(rq_col(col[i], r, kd, dcol)) + bk;
          dmax = fmaxf(dmax, fmaf(ef * cm, max_row_abs_sum<LOT>(), dcol));
        });
      }
      const bool want = dmax > thr && active;
      if (__any_sync(0xffffffffu, want) && want && !defer_fix(fl, FIX_OUT, (unsigned)t * (unsigned)g.K + (unsigned)k, want))
        fix_out_unit_to<MODE, HT, float>(h, c4, bias, g, b, acc, pf, t, k, (uint32_t)g.Kp,
                                         [o](int i, int j, float v) { o[4 * i + j] = v; });
    }
    __syncthreads();
    // store phase: piece q = (channel kq, row i, tile tq), tile fastest
#pragma unroll
    for (int rep = 0; rep < (S::KB * 4 * S::TPB) / S::THREADS; ++rep) {
      const int q = rep * S::THREADS + threadIdx.x;
      const int tq = q & (S::TPB - 1), i = (q / S::TPB) & 3, kq = q / (4 * S::TPB);
      const long long base = ybase[tq];
      if (base < 0 || k0 + kq >= g.K || i >= yrows[tq]) continue;
      const float4 v = *reinterpret_cast<const float4*>(so + kq * S::OK + tq * S::OT + 4 * i);
      float* row = y + base + kq * plane + (long long)i * g.Wo;
      if ((g.Wo & 3) == 0 && (reinterpret_cast<uintptr_t>(y) & 15) == 0) {
        __stcs(reinterpret_cast<float4*>(row), v);
      } else {
        const int cols = g.Wo - (int)((base % g.Wo));
        const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (j < cols) row[j] = vv[j];
      }
    }
    __syncthreads();
  }
}


// ------------------------------------------------------------------ Legendre output stage via T4
// With fp32 outputs the Legendre output side stores the output stage's fp32 fast-path values
// T4 = A_P^T c4 A_P (16 floats per unit, [T][16][Kp]) plus the unit's error factor
// e4 = rowsum(A_P) * max_j |first-half column j| ([T][Kp]) instead of the 36 c4 codes: the final
// pass then reads 68 bytes per unit and only requantises (no second A_P sandwich).  c4 stays
// implicit: any unit whose decision needs exact values recomputes c4 exactly from h.

// Exact output codes of one unit (all 16 elements) from h: c4 exactly, then A_P^T c4 A_P in int64,
// ties replayed in fp64 from c4.  put(i, j, code).
template <typename HT, class Put>
__device__ __noinline__ void exact_out_from_h(const HT* __restrict__ h, const Geo& g, const Bits& b, const Acc* acc,
                                              const PlanF64* __restrict__ pf, int t, int k, Put put) {
  const int n = (int)g.fTP.div((unsigned)t), grp = (int)g.fipg.div((unsigned)n);
  const Acc* ga = acc + (size_t)grp * ST_COUNT;
  int c4[6][6];
  exact_c4_from_h<HT>(h, (uint32_t)g.Kp, (uint32_t)t * 36u * g.Kp + (uint32_t)k, ga, b, pf, c4);
  long long Y[4][4];
  sandwich<tab::Leg_OT>(c4, Y);
  const StageQ q = load_int_stage(ga[ST_OUT], b.q[ST_OUT]);
  int codes[16];
  unsigned ties = 0;
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    bool tie = false;
    codes[e] = rq(Y[e / 4][e % 4], q, tie);
    if (tie) ties |= 1u << e;
  }
  if (ties) {  // exact ties replayed in fp64 from c4, each lane walking its own tie set
    int xc[36];
#pragma unroll
    for (int u = 0; u < 36; ++u) xc[u] = c4[u / 6][u % 6];
    const StageQ qin = load_int_stage(ga[ST_OBC], b.q[ST_OBC]);
    while (ties) {
      const int e = __ffs((int)ties) - 1;
      ties &= ties - 1;
      const int code = code_of(replay_sandwich(pf->ot, 4, 6, xc, qin.qmax, qin.maxabs, qin.scale, e / 4, e % 4), q);
#pragma unroll
      for (int u = 0; u < 16; ++u)
        if (u == e) codes[u] = code;
    }
  }
#pragma unroll
  for (int e = 0; e < 16; ++e) put(e / 4, e % 4, codes[e]);
}

// Exact output values (dequantised + bias) of one unit into o[4 * i + j] (shared staging); tabg is the
// group's dequant table (or null: fp64 formula).  No closures: every argument by value.
template <typename HT>
__device__ __noinline__ void exact_out_to(const HT* __restrict__ h, const Geo& g, const Bits& b, const Acc* acc,
                                          const PlanF64* __restrict__ pf, int t, int k, float* o,
                                          const float* __restrict__ tabg, float bk) {
  const int n = (int)g.fTP.div((unsigned)t), grp = (int)g.fipg.div((unsigned)n);
  const Acc* ga = acc + (size_t)grp * ST_COUNT;
  const int qo = b.q[ST_OUT];
  const double scale = ga[ST_OUT].scale;
  const double maxabs = __longlong_as_double((long long)ga[ST_OUT].F);
  int codes[16];
  exact_out_from_h<HT>(h, g, b, acc, pf, t, k, [&codes](int i, int j, int code) { codes[4 * i + j] = code; });
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const int code = codes[e];
    const float v = tabg ? tabg[code]
                         : (code == qo ? (float)maxabs : (code == -qo ? (float)-maxabs : (float)((double)code * scale)));
    o[e] = v + bk;
  }
}

// T4 (fp32 fast path) + error factor of one unit from its float c4 codes; returns the cropped max and
// the first-half max through m / tm.
__device__ __forceinline__ void t4_of_unit(const float (&K4)[6][6], int ty, int tx, const Geo& g, float* ot, int ostride,
                                           float& efac, float& m, float& tm) {
  float cmax = 0.f;
  m = 0.f;
  tm = 0.f;
  sandwich_cols<tab::Leg_OT>(K4, [&](int j, const float (&col)[4], float cm) {
    cmax = fmaxf(cmax, cm);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      ot[(4 * i + j) * ostride] = col[i];
      if (4 * ty + i < g.Ho && 4 * tx + j < g.Wo) m = fmaxf(m, fabsf(col[i]));
    }
  }, &tm);
  efac = cmax;  // max |first-half value| of the unit: sout_cw forms the per-row band rowsum_i * efac
}

// Rare inline fallback of sout_bt (fix list full): exact c4 from h, then T4 / e4 of the unit written
// to ot / oe; returns (cropped max, first-half max).  Out of line so the fast path keeps its registers.
template <typename HT>
__device__ __noinline__ float2 exact_t4_unit(const HT* __restrict__ h, const Geo& g, const Bits& b, const Acc* ga,
                                             const PlanF64* __restrict__ pf, int t, int k, int ty, int tx, float* ot,
                                             int ostride, float* oe) {
  int c4[6][6];
  exact_c4_from_h<HT>(h, (uint32_t)g.Kp, (uint32_t)t * 36u * g.Kp + (uint32_t)k, ga, b, pf, c4);
  float K4[6][6];
#pragma unroll
  for (int e = 0; e < 36; ++e) K4[e / 6][e % 6] = (float)c4[e / 6][e % 6];
  float m, tm, efac;
  t4_of_unit(K4, ty, tx, g, ot, ostride, efac, m, tm);
  *oe = efac;
  return make_float2(m, tm);
}

// Deferred output_base_change units: exact c4 from h, the unit's T4E entries (16 T4 values + error
// factor, layout [Kp/4][T][17][4]) rewritten, output max recorded.
template <typename HT>
__global__ void __launch_bounds__(128) fixup_obct_kernel(FixList fl, const HT* __restrict__ h, float* __restrict__ t4e,
                                                         const __grid_constant__ Geo g, const __grid_constant__ Bits b,
                                                         Acc* __restrict__ acc, const PlanF64* __restrict__ pf,
                                                         Tables tabs) {
  const unsigned cnt = fix_count(fl, FIX_OBC);
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
    const unsigned u = fl.items[i];
    const int t = (int)g.fK.div(u), k = (int)g.fK.mod(u);
    const int n = (int)g.fTP.div((unsigned)t), tile = (int)g.fTP.mod((unsigned)t), grp = (int)g.fipg.div((unsigned)n);
    const Acc* ga = acc + (size_t)grp * ST_COUNT;
    int c4[6][6];
    exact_c4_from_h<HT>(h, (uint32_t)g.Kp, (uint32_t)t * 36u * g.Kp + (uint32_t)k, ga, b, pf, c4);
    float K4[6][6];
#pragma unroll
    for (int e = 0; e < 36; ++e) K4[e / 6][e % 6] = (float)c4[e / 6][e % 6];
    const int ty = (int)g.ftw.div((unsigned)tile), tx = (int)g.ftw.mod((unsigned)tile);
    float m, tm, efac;
    float* ot = t4e + ((size_t)(k >> 2) * g.T + t) * 68 + (k & 3);
    t4_of_unit(K4, ty, tx, g, ot, 4, efac, m, tm);
    ot[64] = efac;
    record_unit_single(m, tm, grp, acc, ST_OUT, tabs.t[ST_OUT], t, k, g.K);
  }
}

// Exact final outputs of one unit written straight to y (dequantised, + bias, cropped): the deferred
// fix of fixup_outt_kernel and the inline fallback of sout_cw_kernel when the fix list is full.
template <typename HT>
__device__ __noinline__ void exact_out_unit_to_y(const HT* __restrict__ h, float* __restrict__ y,
                                                 const float* __restrict__ bias, const Geo& g, const Bits& b,
                                                 const Acc* __restrict__ acc, const PlanF64* __restrict__ pf, int t,
                                                 int k) {
  const int n = (int)g.fTP.div((unsigned)t), tile = (int)g.fTP.mod((unsigned)t), grp = (int)g.fipg.div((unsigned)n);
  const int ty = (int)g.ftw.div((unsigned)tile), tx = (int)g.ftw.mod((unsigned)tile);
  const Acc* ga = acc + (size_t)grp * ST_COUNT;
  const int qo = b.q[ST_OUT];
  const double scale = ga[ST_OUT].scale;
  const double maxabs = __longlong_as_double((long long)ga[ST_OUT].F);
  const float bk = bias ? bias[k] : 0.f;
  exact_out_from_h<HT>(h, g, b, acc, pf, t, k, [&](int ii, int jj, int code) {
    const int rr = 4 * ty + ii, cc = 4 * tx + jj;
    if (rr < g.Ho && cc < g.Wo) {
      const float v = code == qo ? (float)maxabs : (code == -qo ? (float)-maxabs : (float)((double)code * scale));
      y[(((size_t)n * g.K + k) * g.Ho + rr) * g.Wo + cc] = v + bk;
    }
  });
}

// Final output pass from T4E (Legendre, fp32 output).  T4E = [Kp/4 channel groups][T tiles][17][4
// channels] floats: rows 0..15 the output stage's fp32 values T4 of the unit, row 16 the unit's max
// |first-half value| (the per-row error band is rowsum_i times it).
// Work item = R consecutive tiles x CG channel groups, staged as [CG][R][68] floats; the 8 warps are
// (pass, channel group) pairs, lane = (tile slot, channel) = (lane >> 2, lane & 3), a pass covers TPP <= 8
// tiles.  In that mapping
//   * the staged reads are conflict-free: a unit starts 68 floats (4 banks) after its neighbour tile,
//   * a warp's store of output row i is, per channel, its tiles' 16-byte pieces side by side, straight
//     from registers: no shared output staging and no CTA barrier; warps run independently on an
//     NS-deep full/empty mbarrier ring filled by one thread,
//   * R is a whole number of tile rows (CwShape), so an item writes, per channel, 4 complete output rows
//     = one contiguous 16*tw*4-byte range of y.  DRAM efficiency of the y writes depends on exactly that:
//     tools/probe_ywrite.cu measures 3.7 TB/s for 8-tile (128-byte) runs and 5.5 TB/s for whole tile rows.
struct CwShape {
  int R, TPP, CG;  // tiles per item, tiles per pass, channel groups per item; (R / TPP rounded up) * CG = 8 warps
  int vec4;        // y rows may be stored as float4 (Wo % 4 == 0 and y 16-byte aligned)
};
inline CwShape cw_shape(int tw) {
  // Items are deep in tiles and narrow in channels: per channel an item then writes one contiguous range of
  // 4 * (R / tw) output rows.  Config 4 (tw = 14): 1 / 2 / 4 tile rows per item = 1.38 / 1.33 / 1.31 ms.
#ifndef WL_CW_SMALL_PASSES
#define WL_CW_SMALL_PASSES 4
#endif
  if (tw <= 8) return {WL_CW_SMALL_PASSES * (8 / tw) * tw, (8 / tw) * tw, 8 / WL_CW_SMALL_PASSES, 0};
  if (tw <= 16) return {4 * tw, (tw + 1) / 2, 1, 0};
  if (tw <= 32) return {2 * tw, (tw + 3) / 4, 1, 0};
  return {32, 8, 2, 0};
}
struct StagedCw {
  static constexpr int THREADS = 256;
  static constexpr int STAGE_BYTES = 64 * 68 * 4;  // R * CG <= 64 units-of-4-channels per item
  static constexpr int smem(int ns) { return ns * STAGE_BYTES + 2 * ns * 8 + 16; }
};

template <typename HT, bool TAB, int NS>
__global__ void __launch_bounds__(StagedCw::THREADS, 4)
    sout_cw_kernel(const float* __restrict__ t4e, const HT* __restrict__ h, float* __restrict__ y,
                   const float* __restrict__ bias, const __grid_constant__ Geo g, const __grid_constant__ Bits b,
                   const Acc* __restrict__ acc, const PlanF64* __restrict__ pf, const float* __restrict__ otab,
                   const float4* __restrict__ odq, FixList fl, const CwShape sh) {
  using S = StagedCw;
  extern __shared__ __align__(128) uint8_t wl_stage_smem[];
  uint8_t* sm = wl_stage_smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + NS * S::STAGE_BYTES);
  uint64_t* empty = full + NS;
  const int ncb = ((g.K + 3) / 4 + sh.CG - 1) / sh.CG;
  const int niter = ((g.T + sh.R - 1) / sh.R) * ncb;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = lane >> 2, ch = lane & 3;
  const int pass = w / sh.CG, cgi = w - pass * sh.CG;
  const int tin = pass * sh.TPP + slot;                 // tile of the item this lane owns
  const bool lane_on = slot < sh.TPP && tin < sh.R;
  const int qo = b.q[ST_OUT];
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NS; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], S::THREADS / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int it, int s) {
    const int tg = it / ncb, cb = it - tg * ncb;
    // per channel group the item's tiles are one contiguous range of T4E: CG linear bulk copies
    const int t0 = tg * sh.R, nt = min(sh.R, g.T - t0);
    const int ncg = min(sh.CG, g.Kp / 4 - cb * sh.CG);
    mbar_arrive_expect_tx(&full[s], (uint32_t)(ncg * nt * 272));
    for (int q = 0; q < ncg; ++q)
      bulk_g2s(sm + s * S::STAGE_BYTES + q * sh.R * 272, t4e + ((size_t)(cb * sh.CG + q) * g.T + t0) * 68,
               (uint32_t)(nt * 272), &full[s]);
  };
  if (threadIdx.x == 0)
#pragma unroll
    for (int q = 0; q < NS - 1; ++q)
      if ((int)blockIdx.x + q * (int)gridDim.x < niter) issue(blockIdx.x + q * gridDim.x, q);
  int kk = 0;
  for (int it = blockIdx.x; it < niter; it += gridDim.x, ++kk) {
    const int s = kk % NS;
    if (threadIdx.x == 0 && it + (NS - 1) * (int)gridDim.x < niter) {
      // refill the slot of local iteration kk - 1 once all 8 warps released it
      const int j = kk + NS - 1, f = j / NS;
      if (f >= 1) mbar_wait(&empty[j % NS], (uint32_t)((f - 1) & 1));
      issue(it + (NS - 1) * gridDim.x, j % NS);
    }
    const int tg = it / ncb, cb = it - tg * ncb;
    const int t = tg * sh.R + tin, k = (cb * sh.CG + cgi) * 4 + ch;
    const bool active = lane_on && t < g.T && k < g.K;
    const int tt = active ? t : 0;
    // per-unit parameters first: their latency overlaps the wait for the box
    const int n = (int)g.fTP.div((unsigned)tt), tile = tt - n * g.TP;
    const int grp = (int)g.fipg.div((unsigned)n);
    const Acc* ga = acc + (size_t)grp * ST_COUNT;
    const float r = active ? ga[ST_OUT].r : 0.f, thr = ga[ST_OUT].thr, ef = ga[ST_OUT].ef;
    float4 dq = make_float4(0.f, 0.f, 0.f, 0.f);
    if constexpr (TAB) dq = __ldg(&odq[grp]);
    const float bk = (bias && active) ? __ldg(&bias[k]) : 0.f;
    const int ty = (int)g.ftw.div((unsigned)tile), tx = tile - ty * g.tw;
    mbar_wait(&full[s], (uint32_t)((kk / NS) & 1));
    const float* p =
        reinterpret_cast<const float*>(sm + s * S::STAGE_BYTES) + (cgi * sh.R + (lane_on ? tin : 0)) * 68 + ch;
    f2 v[8];
    float dm[4] = {0.f, 0.f, 0.f, 0.f};  // per output row: max distance of T * r to its rounded code
    if (TAB && dq.z != 0.f) {
      // certified arithmetic dequantisation (out_table_kernel): value = fma(k, s_hi, k * s_lo) + bias.
      // fma(T, -r, k) is the exact negation of rq_col's fma(T, r, -k), so dmax is the same number.
      const f2 r2 = bc2(r), nr2 = bc2(-r), shi = bc2(dq.x), slo = bc2(dq.y), bk2 = bc2(bk), mg = bc2(kMagic);
#pragma unroll
      for (int e = 0; e < 16; e += 2) {
        const f2 T = active ? mk2(p[e * 4], p[(e + 1) * 4]) : bc2(0.f);  // idle lanes: slot not filled
        const f2 k2 = sub2(fma2(T, r2, mg), mg);
        const f2 d = fma2(T, nr2, k2);
        dm[e >> 2] = fmaxf(dm[e >> 2], fmaxf(fabsf(lo2(d)), fabsf(hi2(d))));
        v[e >> 1] = add2(fma2(k2, shi, mul2(k2, slo)), bk2);
      }
    } else {
      const float* tabg = TAB ? otab + (size_t)grp * (2 * qo + 1) + qo : nullptr;
      const double scale = ga[ST_OUT].scale;
      const double maxabs = __longlong_as_double((long long)ga[ST_OUT].F);
      float kd;
#pragma unroll
      for (int e = 0; e < 16; e += 2) {
        float o2[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int code = rq_col(active ? p[(e + u) * 4] : 0.f, r, kd, dm[e >> 2]);
          if constexpr (TAB)
            o2[u] = __ldg(tabg + code) + bk;
          else
            o2[u] = (code == qo ? (float)maxabs : (code == -qo ? (float)-maxabs : (float)((double)code * scale))) + bk;
        }
        v[e >> 1] = mk2(o2[0], o2[1]);
      }
    }
    const float efac = active ? p[64] : 0.f;
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // every lane's reads of the slot are done
    // certified band of element (i, j): ef * rowsum(A_P^T row i) * max |first-half value| (>= column j's)
    const float eb = ef * efac;
    bool want = false;
#pragma unroll
    for (int i = 0; i < 4; ++i) want |= fmaf(eb, row_abs_sum<tab::Leg_OT>(i), dm[i]) > thr;
    want = want && active;
    bool skip = !active;
    if (__any_sync(0xffffffffu, want) && want &&
        !defer_fix(fl, FIX_OUT, (unsigned)t * (unsigned)g.K + (unsigned)k, want)) {
      exact_out_unit_to_y<HT>(h, y, bias, g, b, acc, pf, t, k);
      skip = true;
    }
    if (!skip) {
      float* row = y + (((size_t)n * g.K + k) * g.Ho + 4 * ty) * g.Wo + 4 * tx;
      const int rows = min(4, g.Ho - 4 * ty);
      if (sh.vec4) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (i < rows)
            __stcs(reinterpret_cast<float4*>(row + (size_t)i * g.Wo),
                   make_float4(lo2(v[2 * i]), hi2(v[2 * i]), lo2(v[2 * i + 1]), hi2(v[2 * i + 1])));
      } else {
        const int cols = min(4, g.Wo - 4 * tx);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (i < rows) {
            const float vv[4] = {lo2(v[2 * i]), hi2(v[2 * i]), lo2(v[2 * i + 1]), hi2(v[2 * i + 1])};
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (j < cols) row[(size_t)i * g.Wo + j] = vv[j];
          }
      }
    }
  }
}

// Deferred final-output units of the T4 path: exact from h, written to y.
template <typename HT>
__global__ void __launch_bounds__(128) fixup_outt_kernel(FixList fl, const HT* __restrict__ h, float* __restrict__ y,
                                                         const float* __restrict__ bias, const __grid_constant__ Geo g,
                                                         const __grid_constant__ Bits b, const Acc* __restrict__ acc,
                                                         const PlanF64* __restrict__ pf) {
  const unsigned cnt = fix_count(fl, FIX_OUT);
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
    const unsigned u = fl.items[i];
    exact_out_unit_to_y<HT>(h, y, bias, g, b, acc, pf, (int)g.fK.div(u), (int)g.fK.mod(u));
  }
}

}  // namespace wl
