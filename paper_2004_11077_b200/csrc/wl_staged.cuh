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
    record_unit(m, tm, grp, active, acc, stg, tabs.t[stg], active ? t : 0, c, g.C);
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
    record_unit(m, tm, grp, active, acc, ST_IT, tabs.t[ST_IT], tt, c, g.C);
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
    record_unit(m, tm, grp, active, acc, stg, tabs.t[stg], tt, k, g.K);
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
    record_unit(m, tm, grp, active, acc, ST_OUT, tabs.t[ST_OUT], tt, k, g.K);
  }, c4);
}

}  // namespace wl
