// Two-channel transform kernels: every thread carries the units of channels c and c+1 of one tile
// as packed fp32 pairs and runs the stage sandwich with sm_100a's f32x2 instructions
// (fma/add/sub.rn.f32x2 -> FFMA2/FADD2).  A packed instruction rounds each half exactly like its
// scalar counterpart, and the per-lane operation sequence below is the one of sandwich_cols /
// lapply / rq_col in wl_core.cuh / wl_kernels2.cuh, so every value — and therefore every code,
// stage maximum and error band — is bit-identical to the one-channel kernels.  What changes is the
// instruction count: the issue-bound transform passes (ncu: ~80 % issue-active, FMA and ALU pipes
// shared) execute one packed FMA per two channels (FFMA2 keeps the FMA pipe at 128 lanes/clk/SM
// while halving issue slots, measured by tools/probe_ffma2.cu), one 16-bit shared load per two
// codes and one 16-bit shared store per two output codes.
#pragma once
#include "wl_f2.cuh"
#include "wl_staged.cuh"

namespace wl {

// Row J (and partner P) of L dotted with the packed vector v: the lane-wise sequence of lrows_dot.
// The first product of a chain is an fma with a +0 addend in the scalar code; mul gives the same
// value (up to the sign of an exact zero, which no consumer distinguishes: |.|, rint and further
// sums map -0 and +0 alike).
template <class L, int J, int P>
__device__ __forceinline__ void lrows_dot2(const f2 (&v)[L::C], f2& oj, f2& op) {
  if constexpr (P > J) {
    f2 e = bc2(0.f), o = bc2(0.f);
    bool fe = true, fo = true;
#pragma unroll
    for (int l = 0; l < L::C; ++l) {
      const int a = L::e(J, l);
      if (a != 0) {
        if (a == L::e(P, l)) {
          e = fe ? mul2(v[l], bc2((float)a)) : fma2(v[l], bc2((float)a), e);
          fe = false;
        } else {
          o = fo ? mul2(v[l], bc2((float)a)) : fma2(v[l], bc2((float)a), o);
          fo = false;
        }
      }
    }
    oj = add2(e, o);
    op = sub2(e, o);
  } else {
    f2 s = bc2(0.f);
    bool fs = true;
#pragma unroll
    for (int l = 0; l < L::C; ++l)
      if (L::e(J, l) != 0) {
        s = fs ? mul2(v[l], bc2((float)L::e(J, l))) : fma2(v[l], bc2((float)L::e(J, l)), s);
        fs = false;
      }
    oj = s;
    op = bc2(0.f);
  }
}

template <class L>
__device__ __forceinline__ void lapply2(const f2 (&v)[L::C], f2 (&out)[L::R]) {
  static_for<0, L::R>([&](auto I) {
    constexpr int i = decltype(I)::value;
    constexpr int p = row_partner<L>(i);
    if constexpr (!(p >= 0 && p < i)) {
      f2 a, b;
      lrows_dot2<L, i, p>(v, a, b);
      out[i] = a;
      if constexpr (p > i) out[p] = b;
    }
  });
}

__device__ __forceinline__ void amax2(float& m0, float& m1, f2 x) {
  m0 = fmaxf(m0, fabsf(lo2(x)));
  m1 = fmaxf(m1, fabsf(hi2(x)));
}

// sandwich_cols on two channels: f(j, col) or f(j, col, cm0, cm1); tmax0/1 = max |first-half value|.
template <class L, class F>
__device__ __forceinline__ void sandwich_cols2(const f2 (&X)[L::C][L::C], F&& f, float* tmax0 = nullptr,
                                               float* tmax1 = nullptr) {
  auto emit = [&](int j, const f2 (&tc)[L::C]) {
    f2 col[L::R];
    lapply2<L>(tc, col);
    if constexpr (std::is_invocable_v<F, int, const f2 (&)[L::R], float, float>) {
      float c0 = 0.f, c1 = 0.f;
#pragma unroll
      for (int l = 0; l < L::C; ++l) amax2(c0, c1, tc[l]);
      f(j, col, c0, c1);
    } else {
      f(j, col);
    }
  };
  static_for<0, L::R>([&](auto J) {
    constexpr int j = decltype(J)::value;
    constexpr int p = row_partner<L>(j);
    if constexpr (!(p >= 0 && p < j)) {
      f2 tc[L::C], tp[L::C];
#pragma unroll
      for (int l = 0; l < L::C; ++l) {
        lrows_dot2<L, j, p>(X[l], tc[l], tp[l]);
        if (tmax0) {
          amax2(*tmax0, *tmax1, tc[l]);
          if constexpr (p > j) amax2(*tmax0, *tmax1, tp[l]);
        }
      }
      emit(j, tc);
      if constexpr (p > j) emit(p, tp);
    }
  });
}

// rq_col on two channels; returns the two codes' low bytes packed in a 16-bit word (the int8 codes
// sit in the low byte of y's bits since |code| < 2^22 and kMagic's low byte is 0).
__device__ __forceinline__ unsigned rq_col2(f2 T, f2 r, f2& k, float& d0, float& d1) {
  const f2 y = fma2(T, r, bc2(kMagic));
  k = sub2(y, bc2(kMagic));
  const f2 d = fma2(T, r, mk2(-lo2(k), -hi2(k)));
  d0 = fmaxf(d0, fabsf(lo2(d)));
  d1 = fmaxf(d1, fabsf(hi2(d)));
  return __byte_perm(__float_as_uint(lo2(y)), __float_as_uint(hi2(y)), 0x0040);
}

// Code pair -> packed floats: sign-extending PRMT (selector msb = replicate the byte's sign) + I2FP, no
// FMA-pipe instruction.  (The earlier mantissa splice + FADD2 cost one FMA-pipe op per pair: the transform
// passes are FMA-pipe bound; measured sin_b2 1.51 -> 1.48, sin_c2 1.10 -> 1.08, sout_bt2 1.385 -> 1.374 ms and,
// once their max|tmp| tracking was gone, the max-only passes 0.530 -> 0.524 / 0.475 -> 0.468 ms.)
template <typename HT>
__device__ __forceinline__ f2 codes2f2(unsigned v) {
  unsigned lo, hi;
  if constexpr (sizeof(HT) == 1) {
    asm("prmt.b32 %0, %1, 0, 0x8880;" : "=r"(lo) : "r"(v));
    asm("prmt.b32 %0, %1, 0, 0x9991;" : "=r"(hi) : "r"(v));
  } else {
    asm("prmt.b32 %0, %1, 0, 0x9910;" : "=r"(lo) : "r"(v));
    asm("prmt.b32 %0, %1, 0, 0xbb32;" : "=r"(hi) : "r"(v));
  }
  return mk2((float)(int)lo, (float)(int)hi);
}

// X pair of channels (c, c+1) from a staged [36][LD] block of HT codes.
template <int LD, typename HT>
__device__ __forceinline__ void stage_x2(const uint8_t* st, int c, f2 (&X)[6][6]) {
  if constexpr (sizeof(HT) == 1) {
    const uint16_t* p = reinterpret_cast<const uint16_t*>(st + c);
#pragma unroll
    for (int e = 0; e < 36; ++e) X[e / 6][e % 6] = codes2f2<HT>(p[e * LD / 2]);
  } else {
    const unsigned* p = reinterpret_cast<const unsigned*>(reinterpret_cast<const int16_t*>(st) + c);
#pragma unroll
    for (int e = 0; e < 36; ++e) X[e / 6][e % 6] = codes2f2<HT>(p[e * LD / 2]);
  }
}

// W = padded channels staged per block iteration (threads = W / 2).  Measured on config 4: the c0-fed
// IBC max pass and the V code pass run 2-5 % faster as 128-thread blocks (W = 256, twice the resident
// blocks), the other pair kernels are 1-3 % faster as 256-thread blocks.
#ifndef WL_W_SINA
#define WL_W_SINA 256
#endif
#ifndef WL_W_SINC
#define WL_W_SINC 256
#endif

template <int LD, int EB, int W = 512>
struct Staged2 {
  static_assert(LD <= 256, "staged path handles up to 256 padded channels");
  static constexpr int TPB = (W / LD) > 0 ? W / LD : 1;  // tiles per iteration (two channels per thread)
  static constexpr int THREADS = TPB * LD / 2;
  static constexpr int TILE_BYTES = 36 * LD * EB;
  static constexpr int STAGE_BYTES = TPB * TILE_BYTES;
  static constexpr int SMEM = 2 * STAGE_BYTES + 16;
  static constexpr int OUT_TILE = 36 * LD;
  static constexpr int OUT_BYTES = TPB * OUT_TILE;
  static constexpr int SMEM_OUT = 2 * STAGE_BYTES + 2 * OUT_BYTES + 16;
};

// staged_loop with two channels per thread: body(t, c, act0, act1, st, so) with c even; so points
// at the tile's [36][LD] int8 output block (the body stores 16-bit pairs at so + e * LD + c).
template <int LD, int EB, bool kC0, int W = 512, class Body>
__device__ __forceinline__ void staged_loop2(const Geo& g, int nch, const void* planes, const CUtensorMap* c0map,
                                             Body&& body, int8_t* out = nullptr) {
  using S = Staged2<LD, EB, W>;
  extern __shared__ __align__(128) uint8_t wl_stage_smem[];
  uint8_t* sm = wl_stage_smem;
  const bool kout = out != nullptr;
  uint8_t* osm = sm + 2 * S::STAGE_BYTES;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 2 * S::STAGE_BYTES + (kout ? 2 * S::OUT_BYTES : 0));
  const int niter = (g.T + S::TPB - 1) / S::TPB;
  const int tl = threadIdx.x / (LD / 2), c = 2 * (threadIdx.x % (LD / 2));
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
    body(t, c, t < g.T && c < nch, t < g.T && c + 1 < nch, sm + s * S::STAGE_BYTES + tl * S::TILE_BYTES, so);
    if (kout) {
      if (c + 1 >= nch)  // padded channels of the stored block are zero
#pragma unroll
        for (int e = 0; e < 36; ++e) {
          if (c >= nch) so[e * LD + c] = 0;
          so[e * LD + c + 1] = 0;
        }
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

// record_unit for a thread holding channels c, c+1 (c even): a 16-lane half-warp covers the 32
// channels of one table entry (t, c >> 5).
__device__ __forceinline__ void record_unit2(float m0, float m1, float tm0, float tm1, int grp, bool a0, bool a1,
                                             Acc* acc, int stage, unsigned* table, int t, int c, int C,
                                             bool lazy = false) {
  const unsigned full = 0xffffffffu;
  const bool active = a0 || a1;
  const float m = fmaxf(a0 ? m0 : 0.f, a1 ? m1 : 0.f);
  const float tm = fmaxf(a0 ? tm0 : 0.f, a1 ? tm1 : 0.f);
  const int g = active ? grp : -1;
  const int g0 = __shfl_sync(full, g, 0);
  const bool uniform = __all_sync(full, g == g0) && (C & 31) == 0;
  const int CB = (C + 31) >> 5;
  unsigned* entry = table + (size_t)t * CB + (c >> 5);
  if (uniform) {
    float w = m, tw = tm;
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) {
      w = fmaxf(w, __shfl_xor_sync(full, w, o));
      tw = fmaxf(tw, __shfl_xor_sync(full, tw, o));
    }
    if ((threadIdx.x & 15) == 0 && g >= 0) *entry = __float_as_uint(w);
    w = fmaxf(w, __shfl_xor_sync(full, w, 16));
    tw = fmaxf(tw, __shfl_xor_sync(full, tw, 16));
    if ((threadIdx.x & 31) == 0 && g >= 0) {
      if (w > 0.f) lazy_max(&acc[(size_t)g * ST_COUNT + stage].MF, __float_as_uint(w), lazy);
      if (tw > 0.f) lazy_max(&acc[(size_t)g * ST_COUNT + stage].TM, __float_as_uint(tw), lazy);
    }
  } else if (g >= 0) {
    atomicMax(entry, __float_as_uint(m));
    if (m > 0.f) lazy_max(&acc[(size_t)g * ST_COUNT + stage].MF, __float_as_uint(m), lazy);
    if (tm > 0.f) lazy_max(&acc[(size_t)g * ST_COUNT + stage].TM, __float_as_uint(tm), lazy);
  }
}

// ---------------------------------------------------------------------------------- max passes

template <int MODE, int LD>
__global__ void __launch_bounds__(Staged2<LD, 1, WL_W_SINA>::THREADS, WL_MINB * 512 / WL_W_SINA)
    sin_a2_kernel(const __grid_constant__ CUtensorMap c0map, Geo g, Acc* __restrict__ acc, Tables tabs) {
  staged_loop2<LD, 1, true, WL_W_SINA>(g, g.C, nullptr, &c0map,
                            [&](int t, int c, bool a0, bool a1, const uint8_t* st, int8_t*) {
    f2 X[6][6];
    stage_x2<LD, int8_t>(st, c, X);
    const int tt = (a0 || a1) ? t : 0;
    const int grp = (int)g.fipg.div(g.fTP.div((unsigned)tt));
    constexpr int stg = MODE == 0 ? ST_IT : ST_IBC;
    using LT = std::conditional_t<MODE == 0, tab::Can_IT, tab::Leg_IBC>;
    float m0 = 0.f, m1 = 0.f, tm0 = 0.f, tm1 = 0.f;
    sandwich_cols2<LT>(X, [&](int, const f2 (&col)[6]) {
#pragma unroll
      for (int i = 0; i < 6; ++i) amax2(m0, m1, col[i]);
    });
    record_unit2(m0, m1, tm0, tm1, grp, a0, a1, acc, stg, tabs.t[stg], tt, c, g.C, g.lazy);
  });
}

template <int MODE, typename HT, int LD>
__global__ void __launch_bounds__(Staged2<LD, sizeof(HT)>::THREADS, WL_MINB)
    sout_a2_kernel(const HT* __restrict__ h, Geo g, Acc* __restrict__ acc, Tables tabs) {
  staged_loop2<LD, sizeof(HT), false>(g, g.K, h, nullptr,
                                      [&](int t, int k, bool a0, bool a1, const uint8_t* st, int8_t*) {
    const int tt = (a0 || a1) ? t : 0;
    const int n = (int)g.fTP.div((unsigned)tt), tile = (int)g.fTP.mod((unsigned)tt), grp = (int)g.fipg.div((unsigned)n);
    f2 X[6][6];
    stage_x2<LD, HT>(st, k, X);
    float m0 = 0.f, m1 = 0.f, tm0 = 0.f, tm1 = 0.f;
    constexpr int stg = MODE == 0 ? ST_OUT : ST_OBC;
    if constexpr (MODE == 0) {
      const int ty = (int)g.ftw.div((unsigned)tile), tx = (int)g.ftw.mod((unsigned)tile);
      sandwich_cols2<tab::Can_OT>(X, [&](int j, const f2 (&col)[4]) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (4 * ty + i < g.Ho && 4 * tx + j < g.Wo) amax2(m0, m1, col[i]);
      });
    } else {
      sandwich_cols2<tab::Leg_OBC>(X, [&](int, const f2 (&col)[6]) {
#pragma unroll
        for (int i = 0; i < 6; ++i) amax2(m0, m1, col[i]);
      });
    }
    record_unit2(m0, m1, tm0, tm1, grp, a0, a1, acc, stg, tabs.t[stg], tt, k, g.K, g.lazy);
  });
}

// ---------------------------------------------------------------------------------- code passes

__device__ __forceinline__ void st_pair(int8_t* so, int c, unsigned w) {
  *reinterpret_cast<uint16_t*>(so + c) = (uint16_t)w;
}
template <int LD>
__device__ __forceinline__ void reload_k2(const int8_t* so, int c, f2 (&K)[6][6]) {
  const uint16_t* p = reinterpret_cast<const uint16_t*>(so + c);
#pragma unroll
  for (int e = 0; e < 36; ++e) K[e / 6][e % 6] = codes2f2<int8_t>(p[e * LD / 2]);
}

// sin_b on two channels: c1 codes (staged, bulk-stored) and the input_transform maximum.
template <int LD>
__global__ void __launch_bounds__(Staged2<LD, 1>::THREADS, 2)
    sin_b2_kernel(const __grid_constant__ CUtensorMap c0map, const int8_t* __restrict__ c0, int8_t* __restrict__ c1,
                  Geo g, Bits b, Acc* __restrict__ acc, const PlanF64* __restrict__ pf, Tables tabs, FixList fl) {
  staged_loop2<LD, 1, true>(g, g.C, nullptr, &c0map,
                            [&](int t, int c, bool a0, bool a1, const uint8_t* st, int8_t* so) {
    const int tt = (a0 || a1) ? t : 0;
    const int n = (int)g.fTP.div((unsigned)tt), tile = (int)g.fTP.mod((unsigned)tt), grp = (int)g.fipg.div((unsigned)n);
    const Acc* ga = acc + (size_t)grp * ST_COUNT;
    const float r = ga[ST_IBC].r, thr = ga[ST_IBC].thr, ef = ga[ST_IBC].ef;
    const f2 r2 = bc2(r);
    f2 K1[6][6];
    bool def0 = false, def1 = false;
    {
      f2 X[6][6];
      stage_x2<LD, int8_t>(st, c, X);
      float dm0 = 0.f, dm1 = 0.f;
      sandwich_cols2<tab::Leg_IBC>(X, [&](int j, const f2 (&col)[6], float cm0, float cm1) {
        float d0 = 0.f, d1 = 0.f;
#pragma unroll
        for (int i = 0; i < 6; ++i) st_pair(so + (6 * i + j) * LD, c, rq_col2(col[i], r2, K1[i][j], d0, d1));
        dm0 = fmaxf(dm0, fmaf(ef * cm0, max_row_abs_sum<tab::Leg_IBC>(), d0));
        dm1 = fmaxf(dm1, fmaf(ef * cm1, max_row_abs_sum<tab::Leg_IBC>(), d1));
      });
      const bool w0 = dm0 > thr && a0, w1 = dm1 > thr && a1;
      def0 = defer_fix(fl, FIX_IBC, (unsigned)tt * (unsigned)g.C + (unsigned)c, w0);
      def1 = defer_fix(fl, FIX_IBC, (unsigned)tt * (unsigned)g.C + (unsigned)(c + 1), w1);
      const bool f0 = w0 && !def0, f1 = w1 && !def1;
      if (f0 || f1) {
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          if (!(h ? f1 : f0)) continue;
          int8_t* dst = so + c + h;
          const C0Win win(c0, g, n, tile, c + h, LD);
          fix_unit<tab::Leg_IBC>(SrcC0{win}, r, thr, ef, ga + ST_IBC, b.q[ST_IBC], ga + ST_INPUT, b.q[ST_INPUT], true,
                                 pf->ibc, [dst](int i, int j, int code) { dst[(6 * i + j) * LD] = (int8_t)code; });
        }
        reload_k2<LD>(so, c, K1);
      }
    }
    float m0 = 0.f, m1 = 0.f, tm0 = 0.f, tm1 = 0.f;
    sandwich_cols2<tab::Leg_IT>(K1, [&](int, const f2 (&col)[6]) {
#pragma unroll
      for (int i = 0; i < 6; ++i) amax2(m0, m1, col[i]);
    });
    if (def0) m0 = tm0 = 0.f;  // recorded by fixup_ibc_kernel from the exact codes
    if (def1) m1 = tm1 = 0.f;
    record_unit2(m0, m1, tm0, tm1, grp, a0, a1, acc, ST_IT, tabs.t[ST_IT], tt, c, g.C, g.lazy);
  }, c1);
}

// Legendre V codes from staged c1 (B_P^T), two channels per thread.
template <int LD>
__global__ void __launch_bounds__(Staged2<LD, 1, WL_W_SINC>::THREADS, 2 * 512 / WL_W_SINC)
    sin_c2_kernel(const __grid_constant__ CUtensorMap c0map, const int8_t* __restrict__ c0,
                  const int8_t* __restrict__ c1, int8_t* __restrict__ V, const __grid_constant__ Geo g,
                  const __grid_constant__ Bits b, Acc* __restrict__ acc, const PlanF64* __restrict__ pf, FixList fl) {
  staged_loop2<LD, 1, false, WL_W_SINC>(g, g.C, c1, &c0map,
                                        [&](int t, int c, bool a0, bool a1, const uint8_t* st, int8_t* so) {
    if (!a0 && !a1) return;
    const int n = (int)g.fTP.div((unsigned)t), grp = (int)g.fipg.div((unsigned)n);
    const Acc* ga = acc + (size_t)grp * ST_COUNT;
    const float r = ga[ST_IT].r, thr = ga[ST_IT].thr, ef = ga[ST_IT].ef;
    const f2 r2 = bc2(r);
    f2 X[6][6];
    stage_x2<LD, int8_t>(st, c, X);
    float dm0 = 0.f, dm1 = 0.f;
    f2 kd;
    sandwich_cols2<tab::Leg_IT>(X, [&](int j, const f2 (&col)[6], float cm0, float cm1) {
      float d0 = 0.f, d1 = 0.f;
#pragma unroll
      for (int i = 0; i < 6; ++i) st_pair(so + (6 * i + j) * LD, c, rq_col2(col[i], r2, kd, d0, d1));
      dm0 = fmaxf(dm0, fmaf(ef * cm0, max_row_abs_sum<tab::Leg_IT>(), d0));
      dm1 = fmaxf(dm1, fmaf(ef * cm1, max_row_abs_sum<tab::Leg_IT>(), d1));
    });
    const bool w0 = dm0 > thr && a0, w1 = dm1 > thr && a1;
    const bool f0 = w0 && !defer_fix(fl, FIX_IT, (unsigned)t * (unsigned)g.C + (unsigned)c, w0);
    const bool f1 = w1 && !defer_fix(fl, FIX_IT, (unsigned)t * (unsigned)g.C + (unsigned)(c + 1), w1);
    if (f0) fix_it_unit<1>(c0, c1, so + c, LD, g, b, acc, pf, t, c, LD);
    if (f1) fix_it_unit<1>(c0, c1, so + c + 1, LD, g, b, acc, pf, t, c + 1, LD);
  }, V);
}

// t4_of_unit on two channels: T4 pairs stored as 8-byte words at ot + (4i+j)*ostride (channel pair
// adjacent), error factors and maxima per channel.
__device__ __forceinline__ void t4_of_unit2(const f2 (&K4)[6][6], int ty, int tx, const Geo& g, float* ot, int ostride,
                                            float& ef0, float& ef1, float& m0, float& m1, float& tm0, float& tm1) {
  float cx0 = 0.f, cx1 = 0.f;
  m0 = m1 = tm0 = tm1 = 0.f;
  sandwich_cols2<tab::Leg_OT>(K4, [&](int j, const f2 (&col)[4], float cm0, float cm1) {
    cx0 = fmaxf(cx0, cm0);
    cx1 = fmaxf(cx1, cm1);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      *reinterpret_cast<unsigned long long*>(ot + (4 * i + j) * ostride) = col[i].u;
      if (4 * ty + i < g.Ho && 4 * tx + j < g.Wo) amax2(m0, m1, col[i]);
    }
  });
  ef0 = cx0;  // max |first-half value| of the unit: sout_cw forms the per-row band rowsum_i * ef
  ef1 = cx1;
}

template <int LD, int EB>
struct StagedT42 {
  static_assert(LD <= 256, "staged path handles up to 256 padded channels");
  static constexpr int TPB = 512 / LD;
  static constexpr int THREADS = TPB * LD / 2;
  static constexpr int TILE_BYTES = 36 * LD * EB;
  static constexpr int STAGE_BYTES = TPB * TILE_BYTES;
  static constexpr int T4_TILE = 16 * LD * 4;
  static constexpr int E_TILE = LD * 4;
  static constexpr int OUT_BYTES = TPB * (T4_TILE + E_TILE);
  static constexpr int SMEM = 2 * STAGE_BYTES + 2 * OUT_BYTES + 16;
};

// sout_bt on two channels: output_base_change codes (registers) -> T4 / e4, output maximum.
template <typename HT, int LD>
__global__ void __launch_bounds__(StagedT42<LD, sizeof(HT)>::THREADS, 2)
    sout_bt2_kernel(const HT* __restrict__ h, const __grid_constant__ CUtensorMap t4map, Geo g, Bits b,
                    Acc* __restrict__ acc, const PlanF64* __restrict__ pf, Tables tabs, FixList fl) {
  using S = StagedT42<LD, sizeof(HT)>;
  extern __shared__ __align__(128) uint8_t wl_stage_smem[];
  uint8_t* sm = wl_stage_smem;
  uint8_t* osm = sm + 2 * S::STAGE_BYTES;
  uint64_t* bar = reinterpret_cast<uint64_t*>(osm + 2 * S::OUT_BYTES);
  const int niter = (g.T + S::TPB - 1) / S::TPB;
  const int tl = threadIdx.x / (LD / 2), k = 2 * (threadIdx.x % (LD / 2));
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
    tma_prefetch_desc(&t4map);
  }
  __syncthreads();
  auto issue = [&](int it, int s) {
    const int t0 = it * S::TPB;
    const int nt = min(S::TPB, g.T - t0);
    mbar_arrive_expect_tx(&bar[s], (uint32_t)(nt * S::TILE_BYTES));
    bulk_g2s(sm + s * S::STAGE_BYTES, reinterpret_cast<const uint8_t*>(h) + (size_t)t0 * S::TILE_BYTES,
             (uint32_t)(nt * S::TILE_BYTES), &bar[s]);
  };
  if (threadIdx.x == 0 && (int)blockIdx.x < niter) issue(blockIdx.x, 0);
  int kk = 0;
  for (int it = blockIdx.x; it < niter; it += gridDim.x, ++kk) {
    const int s = kk & 1;
    if (threadIdx.x == 0 && it + (int)gridDim.x < niter) issue(it + gridDim.x, s ^ 1);
    mbar_wait(&bar[s], (uint32_t)((kk >> 1) & 1));
    const int t = it * S::TPB + tl;
    const bool a0 = t < g.T && k < g.K, a1 = t < g.T && k + 1 < g.K;
    const int tt = (a0 || a1) ? t : 0;
    const int n = (int)g.fTP.div((unsigned)tt), tile = (int)g.fTP.mod((unsigned)tt), grp = (int)g.fipg.div((unsigned)n);
    const Acc* ga = acc + (size_t)grp * ST_COUNT;
    const float r = ga[ST_OBC].r, thr = ga[ST_OBC].thr, ef = ga[ST_OBC].ef;
    const f2 r2 = bc2(r);
    const uint8_t* st = sm + s * S::STAGE_BYTES + tl * S::TILE_BYTES;
    // staged block in the T4E layout [LD/4 channel groups][TPB tiles][17 rows][4 channels]: rows 0..15
    // = T4 elements, row 16 = error factors (wl_staged.cuh, sout_cw_kernel)
    float* ot = reinterpret_cast<float*>(osm + s * S::OUT_BYTES) + ((k >> 2) * S::TPB + tl) * 68 + (k & 3);
    float* oe = ot + 64;
    f2 K4[6][6];
    bool def0, def1, f0, f1;
    {
      f2 X[6][6];
      stage_x2<LD, HT>(st, k, X);
      float dm0 = 0.f, dm1 = 0.f;
      sandwich_cols2<tab::Leg_OBC>(X, [&](int j, const f2 (&col)[6], float cm0, float cm1) {
        float d0 = 0.f, d1 = 0.f;
#pragma unroll
        for (int i = 0; i < 6; ++i) rq_col2(col[i], r2, K4[i][j], d0, d1);
        dm0 = fmaxf(dm0, fmaf(ef * cm0, max_row_abs_sum<tab::Leg_OBC>(), d0));
        dm1 = fmaxf(dm1, fmaf(ef * cm1, max_row_abs_sum<tab::Leg_OBC>(), d1));
      });
      const bool w0 = dm0 > thr && a0, w1 = dm1 > thr && a1;
      def0 = defer_fix(fl, FIX_OBC, (unsigned)tt * (unsigned)g.K + (unsigned)k, w0);
      def1 = defer_fix(fl, FIX_OBC, (unsigned)tt * (unsigned)g.K + (unsigned)(k + 1), w1);
      f0 = w0 && !def0;
      f1 = w1 && !def1;
    }
    const int ty = (int)g.ftw.div((unsigned)tile), tx = (int)g.ftw.mod((unsigned)tile);
    float m0, m1, tm0, tm1, ef0, ef1;
    t4_of_unit2(K4, ty, tx, g, ot, 4, ef0, ef1, m0, m1, tm0, tm1);
    *reinterpret_cast<float2*>(oe) = make_float2(ef0, ef1);
    if (f0) {
      const float2 mm = exact_t4_unit<HT>(h, g, b, ga, pf, tt, k, ty, tx, ot, 4, oe);
      m0 = mm.x, tm0 = mm.y;
    }
    if (f1) {
      const float2 mm = exact_t4_unit<HT>(h, g, b, ga, pf, tt, k + 1, ty, tx, ot + 1, 4, oe + 1);
      m1 = mm.x, tm1 = mm.y;
    }
    if (def0) m0 = tm0 = 0.f;  // recorded by fixup_obct_kernel from the exact codes
    if (def1) m1 = tm1 = 0.f;
    record_unit2(m0, m1, tm0, tm1, grp, a0, a1, acc, ST_OUT, tabs.t[ST_OUT], tt, k, g.K, g.lazy);
    fence_proxy_async_smem();
    if (threadIdx.x == 0) bulk_wait_read<0>();  // the store issued last iteration has read buffer s^1
    __syncthreads();
    if (threadIdx.x == 0) {
      // one tensor store of the box {68 floats, TPB tiles, LD/4 channel groups}; tiles past T are clipped
      tma_store_3d(&t4map, osm + s * S::OUT_BYTES, 0, it * S::TPB, 0);
      bulk_commit();
    }
  }
  if (threadIdx.x == 0) bulk_wait_all<0>();
}

}  // namespace wl
