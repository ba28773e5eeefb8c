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
};

// `nch` = number of real channels of the unit axis (g.C for input-side kernels, g.K for output-side).
template <int LD, int EB, bool kC0, class Body>
__device__ __forceinline__ void staged_loop(const Geo& g, int nch, const void* planes, const CUtensorMap* c0map,
                                            Body&& body) {
  using S = Staged<LD, EB>;
  extern __shared__ __align__(128) uint8_t wl_stage_smem[];
  uint8_t* sm = wl_stage_smem;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 2 * S::STAGE_BYTES);
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
        const int t = t0 + k, n = t / g.TP, tile = t % g.TP;
        const int ty = tile / g.tw, tx = tile % g.tw;
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
    body(t, c, t < g.T && c < nch, sm + s * S::STAGE_BYTES + tl * S::TILE_BYTES);
    __syncthreads();
  }
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
  staged_loop<LD, 1, true>(g, g.C, nullptr, &c0map, [&](int t, int c, bool active, const uint8_t* st) {
    float X[6][6];
    stage_x<LD, int8_t>(st, c, X);
    const int grp = (t / g.TP) / g.ipg;
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
  staged_loop<LD, 1, true>(g, g.C, nullptr, &c0map, [&](int t, int c, bool active, const uint8_t* st) {
    const int tt = active ? t : 0;
    const int n = tt / g.TP, tile = tt % g.TP, grp = n / g.ipg;
    const Acc* ga = acc + (size_t)grp * ST_COUNT;
    const float r = ga[ST_IBC].r, thr = ga[ST_IBC].thr, ef = ga[ST_IBC].ef;
    constexpr uint32_t plane = LD;
    int8_t* dst = c1 + ((size_t)tt * 36 * LD + c);
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
          if (active) dst[(6 * i + j) * plane] = (int8_t)code;
        }
        dmax = fmaxf(dmax, fmaf(ef * cm, max_row_abs_sum<tab::Leg_IBC>(), dcol));
      });
      const bool want = dmax > thr && active;
      deferred = defer_fix(fl, FIX_IBC, (unsigned)tt * (unsigned)g.C + (unsigned)c, want);
      if (want && !deferred) {
        const C0Win win(c0, g, n, tile, c, LD);
        fix_unit<tab::Leg_IBC>(SrcC0{win}, r, thr, ef, ga + ST_IBC, b.q[ST_IBC], ga + ST_INPUT, b.q[ST_INPUT], true,
                               pf->ibc, [dst](int i, int j, int code) { dst[(6 * i + j) * plane] = (int8_t)code; });
#pragma unroll
        for (int e = 0; e < 36; ++e) K1[e / 6][e % 6] = (float)dst[e * plane];
      }
    }
    float m = 0.f, tm = 0.f;
    sandwich_cols<tab::Leg_IT>(K1, [&](int, const float (&col)[6]) {
#pragma unroll
      for (int i = 0; i < 6; ++i) m = fmaxf(m, fabsf(col[i]));
    }, &tm);
    if (deferred) m = tm = 0.f;  // recorded by fixup_ibc_kernel from the exact codes
    record_unit(m, tm, grp, active, acc, ST_IT, tabs.t[ST_IT], tt, c, g.C);
  });
}

// V codes: canonical from the c0 window (B^T), Legendre from staged c1 (B_P^T).
template <int MODE, int LD>
__global__ void __launch_bounds__(Staged<LD, 1>::THREADS, WL_MINB)
    sin_c_kernel(const __grid_constant__ CUtensorMap c0map, const int8_t* __restrict__ c0,
                 const int8_t* __restrict__ c1, int8_t* __restrict__ V, Geo g, Bits b, Acc* __restrict__ acc,
                 const PlanF64* __restrict__ pf, FixList fl) {
  staged_loop<LD, 1, MODE == 0>(g, g.C, c1, &c0map, [&](int t, int c, bool active, const uint8_t* st) {
    if (!active) return;
    const int n = t / g.TP, tile = t % g.TP, grp = n / g.ipg;
    const Acc* ga = acc + (size_t)grp * ST_COUNT;
    const float r = ga[ST_IT].r, thr = ga[ST_IT].thr, ef = ga[ST_IT].ef;
    constexpr uint32_t plane = LD;
    const uint32_t off = (uint32_t)t * 36u * LD + c;
    int8_t* dst = V + off;
    float X[6][6];
    stage_x<LD, int8_t>(st, c, X);
    float dmax = 0.f, kd;
    using LIT = std::conditional_t<MODE == 0, tab::Can_IT, tab::Leg_IT>;
    sandwich_cols<LIT>(X, [&](int j, const float (&col)[6], float cm) {
      float dcol = 0.f;
#pragma unroll
      for (int i = 0; i < 6; ++i) dst[(6 * i + j) * plane] = (int8_t)rq_col(col[i], r, kd, dcol);
      dmax = fmaxf(dmax, fmaf(ef * cm, max_row_abs_sum<LIT>(), dcol));
    });
    const bool want = dmax > thr;
    if (want && !defer_fix(fl, FIX_IT, (unsigned)t * (unsigned)g.C + (unsigned)c, want))
      fix_it_unit<MODE>(c0, c1, V, g, b, acc, pf, t, c, LD);
  });
}

// ---------------------------------------------------------------------------------- output side

template <int MODE, typename HT, int LD>
__global__ void __launch_bounds__(Staged<LD, sizeof(HT)>::THREADS, WL_MINB)
    sout_a_kernel(const HT* __restrict__ h, Geo g, Acc* __restrict__ acc, Tables tabs) {
  staged_loop<LD, sizeof(HT), false>(g, g.K, h, nullptr, [&](int t, int k, bool active, const uint8_t* st) {
    const int tt = active ? t : 0;
    const int n = tt / g.TP, tile = tt % g.TP, grp = n / g.ipg;
    const int ty = tile / g.tw, tx = tile % g.tw;
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
  staged_loop<LD, sizeof(HT), false>(g, g.K, h, nullptr, [&](int t, int k, bool active, const uint8_t* st) {
    const int tt = active ? t : 0;
    const int n = tt / g.TP, tile = tt % g.TP, grp = n / g.ipg;
    const Acc* ga = acc + (size_t)grp * ST_COUNT;
    const float r = ga[ST_OBC].r, thr = ga[ST_OBC].thr, ef = ga[ST_OBC].ef;
    constexpr uint32_t plane = LD;
    const uint32_t off = (uint32_t)tt * 36u * LD + k;
    int8_t* dst = c4 + off;
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
          if (active) dst[(6 * i + j) * plane] = (int8_t)code;
        }
        dmax = fmaxf(dmax, fmaf(ef * cm, max_row_abs_sum<tab::Leg_OBC>(), dcol));
      });
      const bool want = dmax > thr && active;
      deferred = defer_fix(fl, FIX_OBC, (unsigned)tt * (unsigned)g.K + (unsigned)k, want);
      if (want && !deferred) {
        fix_unit<tab::Leg_OBC>(SrcPlanes<HT>{h, plane, off}, r, thr, ef, ga + ST_OBC, b.q[ST_OBC], ga + ST_HAD,
                               b.q[ST_HAD], false, pf->obc,
                               [dst](int i, int j, int code) { dst[(6 * i + j) * plane] = (int8_t)code; });
#pragma unroll
        for (int e = 0; e < 36; ++e) K4[e / 6][e % 6] = (float)dst[e * plane];
      }
    }
    const int ty = tile / g.tw, tx = tile % g.tw;
    float m = 0.f, tm = 0.f;
    sandwich_cols<tab::Leg_OT>(K4, [&](int j, const float (&col)[4]) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (4 * ty + i < g.Ho && 4 * tx + j < g.Wo) m = fmaxf(m, fabsf(col[i]));
    }, &tm);
    if (deferred) m = tm = 0.f;  // recorded by fixup_obc_kernel from the exact codes
    record_unit(m, tm, grp, active, acc, ST_OUT, tabs.t[ST_OUT], tt, k, g.K);
  });
}

}  // namespace wl
