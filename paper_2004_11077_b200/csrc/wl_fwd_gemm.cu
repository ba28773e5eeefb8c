// Hadamard passes of the forward (reference: _kernels.py:94-105 `_hadamard_accumulate_nb` and the
// cast of pipeline.py:146): the persistent tcgen05 int8 GEMM of gemm_i8.cuh run twice over V and U,
// first with the exact max epilogue (group maxima + argmax candidates for the fp64 replay in
// finalize_hadamard), then with the requantisation epilogue writing the Hadamard codes h.
#include <cuda_runtime.h>

#include <algorithm>

#include "gemm_i8.cuh"
#include "wl_pair.cuh"
#include "wl_internal.h"

namespace wl {

// ------------------------------------------------------------------ GEMM epilogues

// Max pass: exact int32 accumulators; per-thread maximum over its row chunk; the group maximum M is
// reduced in place (atomicMax) and units that may hold the argmax are pushed as candidates for the
// fp64 replay in finalize_hadamard_kernel.
struct EpiHadMax {
  static constexpr int kGroups = 4;
  static constexpr int kStageBytes = 0;
  static constexpr bool kDeferSlow = false;
  Acc* acc;
  unsigned* table;
  Geo g;
  int nchunk;
  long long m;
  int vmax, vmin;
  int grp;
  static constexpr bool kPrefetch = false;
  __device__ __forceinline__ void prefetch(int, bool) {}
  __device__ __forceinline__ void begin(int, int row, bool valid) {
    vmax = 0;
    vmin = 0;
    grp = valid ? (int)g.fipg.div(g.fTP.div((unsigned)row)) : -1;
  }
  __device__ __forceinline__ void apply(int, int, int, const uint32_t* v, int n) {
    if (n == 16) {
#pragma unroll
      for (int j = 0; j < 16; j += 2) {
        vmax = __vimax3_s32(vmax, (int)v[j], (int)v[j + 1]);
        vmin = __vimin3_s32(vmin, (int)v[j], (int)v[j + 1]);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < n) {
          vmax = max(vmax, (int)v[j]);
          vmin = min(vmin, (int)v[j]);
        }
    }
  }
  __device__ __forceinline__ void finish_chunk(int xi, int row, bool valid, int chunk) {
    m = max((long long)vmax, -(long long)vmin);
    if (valid) table[((size_t)xi * g.T + row) * nchunk + chunk] = (unsigned)m;
    bool uniform;
    long long wmax;
    Acc* a = acc + ST_HAD;
    // (replay_gate only computes the warp reduction here; the replay itself runs in finalize)
    replay_gate(m, grp, a, ST_COUNT, uniform, wmax);
    publish_max(m, grp, a, ST_COUNT, uniform, wmax, g.lazy != 0);
  }
};

// Exact requantisation of 8 Hadamard accumulators of one row (rare path: the fp32 bracket split for
// some element of the chunk): int64 rounding, fp64 replay of exact ties.  Returns the packed codes
// (int8: 2 words, int16: 4 words).  A free function taking values, so the epilogue functor and its
// arrays stay in registers.
struct HadRqCtx {
  const Acc* acc;
  const Acc* wacc;
  const int8_t* U;
  const int8_t* V;
  int C, Cp, Kp, grp, wstage, qmax_u, qmax_v, qmax_h, xi, row;
  FixList fl;
};
template <typename HT>
static __device__ __noinline__ uint4 had_rq_slow8(HadRqCtx cx, uint4 va, uint4 vb, int col, int n) {
  const StageQ q = load_int_stage(cx.acc[(size_t)cx.grp * ST_COUNT + ST_HAD], cx.qmax_h);
  const uint32_t v[8] = {va.x, va.y, va.z, va.w, vb.x, vb.y, vb.z, vb.w};
  uint32_t c[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    bool tie = false;
    int code = rq((long long)(int)v[j], q, tie);
    // exact ties are replayed in fp64 by fixup_had_kernel (one thread each, off the epilogue's
    // critical path); only an overflowing list falls back to the inline replay
    const bool want = tie && j < n;
    const unsigned unit = ((unsigned)cx.row * 36u + (unsigned)cx.xi) * (unsigned)cx.Kp + (unsigned)(col + j);
    if (defer_fix(cx.fl, FIX_HAD, unit, want)) {
    } else if (want) {
      const StageQ qu = load_int_stage(cx.wacc[cx.wstage], cx.qmax_u);
      const StageQ qv = load_int_stage(cx.acc[(size_t)cx.grp * ST_COUNT + ST_IT], cx.qmax_v);
      code = code_of(replay_hadamard(cx.U + ((size_t)(col + j) * 36 + cx.xi) * cx.Cp,
                                     cx.V + ((size_t)cx.row * 36 + cx.xi) * cx.Cp, cx.C, qu, qv),
                     q);
    }
    c[j] = (uint32_t)code;
  }
  if constexpr (sizeof(HT) == 1)
    return make_uint4(__byte_perm(__byte_perm(c[0], c[1], 0x0040), __byte_perm(c[2], c[3], 0x0040), 0x5410),
                      __byte_perm(__byte_perm(c[4], c[5], 0x0040), __byte_perm(c[6], c[7], 0x0040), 0x5410), 0u, 0u);
  else
    return make_uint4(__byte_perm(c[0], c[1], 0x5410), __byte_perm(c[2], c[3], 0x5410), __byte_perm(c[4], c[5], 0x5410),
                      __byte_perm(c[6], c[7], 0x5410));
}

// Requantisation pass: h = rhe(qmax_h * I / M) with the fp32 magic-number fast path (I is exact and
// |I| < 2^24, so the only inexactness is the product by qmax/M); near half-integers the exact int64
// decision, and exact ties are replayed in fp64 from the U and V codes.
#ifndef WL_RQ_GROUPS
#define WL_RQ_GROUPS 2  // epilogue column groups of the requantisation pass (4 x groups epilogue warps)
#endif
template <typename HT>
struct EpiHadRq {
  // each epilogue warp stages its 32 rows x 128 columns of codes (swizzled 16-byte slots) and
  // writes them back as whole row segments
  static constexpr int kGroups = WL_RQ_GROUPS;
  static constexpr bool kDeferSlow = true;
  static constexpr int kStageBytes = 32 * (256 / kGroups) * (int)sizeof(HT);
  static constexpr int kRowBytes = (256 / kGroups) * (int)sizeof(HT);
  static constexpr int kSwz = kRowBytes / 16 - 1;  // XOR swizzle of the 16-byte slots within a row
  uint8_t* stage;
  int hc;  // columns per epilogue warp (half the N tile)
  __device__ __forceinline__ void set_stage(uint8_t* p, int half_cols) {
    stage = p;
    hc = half_cols;
  }
  Acc* acc;
  const Acc* wacc;
  const int8_t* U;
  const int8_t* V;
  HT* h;
  Geo g;
  FixList fl;
  int wstage, qmax_u, qmax_v, qmax_h;
  StageF s;
  float r_lo, r_hi;
  int grp;
  int pgrp;             // prefetched (next tile) group and its stage parameters
  float pr, pthr;
  static constexpr bool kPrefetch = true;
  __device__ __forceinline__ void prefetch(int row, bool valid) {
    pgrp = valid ? (int)g.fipg.div(g.fTP.div((unsigned)row)) : 0;
    const Acc& a = acc[(size_t)pgrp * ST_COUNT + ST_HAD];
    pr = a.r;
    pthr = a.thr;
  }
  __device__ __forceinline__ void begin(int, int row, bool valid) {
    grp = pgrp;
    const struct { float r, thr; } a = {pr, pthr};
    s.r = a.r;
    s.band = 0.5f - a.thr;
    s.qmax = qmax_h;
    // r = fl(qmax/M) is within 2^-24 (relative) of qmax/M, so [r_lo, r_hi] brackets it; I is exact,
    // hence rn(I*r_lo) == rn(I*r_hi) proves the half-even code of I*qmax/M (an exact tie always
    // splits the bracket since I != 0 then).
    r_lo = __fmul_rd(a.r, 1.f - 2.384185791015625e-7f);
    r_hi = __fmul_ru(a.r, 1.f + 2.384185791015625e-7f);
  }
  // Fast path of 16 consecutive columns starting at local column lc of this warp's slice: codes from the
  // r_lo evaluation are staged unconditionally; returns true if some element's [r_lo, r_hi] bracket
  // split (then apply_slow redoes the chunk).
  __device__ __forceinline__ bool apply_fast(const uint32_t* v, int lc) {
    // y[j] = 0x4B400000 + code: its low byte / half-word is the two's-complement code
    uint32_t y[16];
    uint32_t d0 = 0, d1 = 0, d2 = 0, d3 = 0;  // independent chains (ILP)
    f2 sq0 = bc2(0.f), sq1 = bc2(0.f);
    // column pairs on packed f32x2 (FFMA2: lane-wise identical to the scalar ops); the accumulators are
    // converted with I2FP (exact: |I| < 2^24) — measured faster than the magic-number add + FADD2 (1.07 -> 1.02 ms)
#pragma unroll
    for (int j = 0; j < 16; j += 2) {
      const f2 fi = mk2((float)(int)v[j], (float)(int)v[j + 1]);
      const f2 ya = fma2(fi, bc2(r_lo), bc2(kMagic)), yb = fma2(fi, bc2(r_hi), bc2(kMagic));
      y[j] = __float_as_uint(lo2(ya));
      y[j + 1] = __float_as_uint(hi2(ya));
#ifdef WL_RQ_XOR
      const uint32_t da = y[j] ^ __float_as_uint(lo2(yb)), db = y[j + 1] ^ __float_as_uint(hi2(yb));
      if ((j & 2) == 0) d0 |= da, d1 |= db; else d2 |= da, d3 |= db;
#else
      // bracket test on the FMA pipe (the epilogue is ALU-pipe bound): ya - yb is the exact code difference,
      // its squares accumulate to zero iff every code of the chunk agrees (two chains for ILP)
      const f2 df = sub2(ya, yb);
      if ((j & 2) == 0) sq0 = fma2(df, df, sq0); else sq1 = fma2(df, df, sq1);
#endif
    }
#ifndef WL_RQ_XOR
    {
      const f2 sq = add2(sq0, sq1);
      d0 = __float_as_uint(lo2(sq)) | __float_as_uint(hi2(sq));  // non-negative sums: bits zero iff value zero
    }
#endif
    const int lane = threadIdx.x & 31;
    const int slot0 = (lc * (int)sizeof(HT)) >> 4;
    const uint32_t rbase = smem_u32(stage) + lane * kRowBytes;
    if constexpr (sizeof(HT) == 1) {
      uint32_t w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        w[q] = __byte_perm(__byte_perm(y[4 * q], y[4 * q + 1], 0x0040), __byte_perm(y[4 * q + 2], y[4 * q + 3], 0x0040),
                           0x5410);
      st_shared_v4(rbase + ((slot0 ^ (lane & kSwz)) << 4), w[0], w[1], w[2], w[3]);
    } else {
      uint32_t w[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) w[q] = __byte_perm(y[2 * q], y[2 * q + 1], 0x5410);
      st_shared_v4(rbase + ((slot0 ^ (lane & kSwz)) << 4), w[0], w[1], w[2], w[3]);
      st_shared_v4(rbase + (((slot0 + 1) ^ (lane & kSwz)) << 4), w[4], w[5], w[6], w[7]);
    }
    return ((d0 | d1) | (d2 | d3)) != 0;  // rare: some element's bracket split
  }
  // Exact redo of a flagged chunk (int64 rounding, ties deferred to fixup_had_kernel): overwrites the
  // staged codes of the 16 columns at local column lc.
  __device__ __forceinline__ void apply_slow(int xi, int row, int col, const uint32_t* v, int n, int lc) {
    const int lane = threadIdx.x & 31;
    const int slot0 = (lc * (int)sizeof(HT)) >> 4;
    const uint32_t rbase = smem_u32(stage) + lane * kRowBytes;
    const HadRqCtx cx{acc, wacc, U, V, g.C, g.Cp, g.Kp, grp, wstage, qmax_u, qmax_v, qmax_h, xi, row, fl};
    const uint4 lo = had_rq_slow8<HT>(cx, make_uint4(v[0], v[1], v[2], v[3]), make_uint4(v[4], v[5], v[6], v[7]), col, n);
    const uint4 hi = had_rq_slow8<HT>(cx, make_uint4(v[8], v[9], v[10], v[11]), make_uint4(v[12], v[13], v[14], v[15]),
                                      col + 8, n - 8);
    if constexpr (sizeof(HT) == 1) {
      st_shared_v4(rbase + ((slot0 ^ (lane & kSwz)) << 4), lo.x, lo.y, hi.x, hi.y);
    } else {
      st_shared_v4(rbase + ((slot0 ^ (lane & kSwz)) << 4), lo.x, lo.y, lo.z, lo.w);
      st_shared_v4(rbase + (((slot0 + 1) ^ (lane & kSwz)) << 4), hi.x, hi.y, hi.z, hi.w);
    }
  }
  __device__ __forceinline__ void finish_chunk(int, int, bool, int) {}
  // write the warp's 32 staged rows: each instruction covers whole 128/256-byte row segments
  __device__ __forceinline__ void flush(int xi, int row0, int n0, int hc, int T, int lane) {
    __syncwarp();
    constexpr int kSlots = kRowBytes / 16;
    constexpr int kRowsPerInstr = 32 / kSlots;
    const int nbytes = min(hc, g.K - n0) * (int)sizeof(HT);  // valid bytes of each row segment
    for (int r0 = 0; r0 < 32; r0 += kRowsPerInstr) {
      const int r = r0 + lane / kSlots, sl = lane % kSlots;
      const int row = row0 + r;
      if (row < T && sl * 16 < nbytes) {
        const int4 v = ld_shared_v4(smem_u32(stage) + r * kRowBytes + ((sl ^ (r & kSwz)) << 4));
        *reinterpret_cast<int4*>(reinterpret_cast<uint8_t*>(h + ((size_t)row * 36 + xi) * g.Kp + n0) + sl * 16) = v;
      }
    }
    __syncwarp();
  }
};

// Deferred exact ties of the requantisation pass: fp64 replay in the reference's order
// (_kernels.py:99-104, c ascending), one thread per tie.
template <typename HT>
__global__ void __launch_bounds__(128) fixup_had_kernel(FixList fl, const int8_t* __restrict__ U,
                                                        const int8_t* __restrict__ V, HT* __restrict__ h, Geo g,
                                                        const Acc* __restrict__ acc, const Acc* __restrict__ wacc,
                                                        int wstage, int qmax_u, int qmax_v, int qmax_h) {
  const unsigned cnt = fix_count(fl, FIX_HAD);
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
    const unsigned u = fl.items[i];
    const unsigned rx = u / (unsigned)g.Kp, col = u - rx * (unsigned)g.Kp;
    const unsigned row = rx / 36u, xi = rx - row * 36u;
    const int grp = (int)g.fipg.div(g.fTP.div(row));
    const StageQ q = load_int_stage(acc[(size_t)grp * ST_COUNT + ST_HAD], qmax_h);
    const StageQ qu = load_int_stage(wacc[wstage], qmax_u);
    const StageQ qv = load_int_stage(acc[(size_t)grp * ST_COUNT + ST_IT], qmax_v);
    const double t = replay_hadamard(U + ((size_t)col * 36 + xi) * g.Cp, V + ((size_t)row * 36 + xi) * g.Cp, g.C, qu, qv);
    h[u] = (HT)code_of(t, q);
  }
}

template <int BN, int SW, class Epi>
static int launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, const Geo& g, const Epi& e, cudaStream_t st) {
  const int ntiles = 36 * ((g.T + 127) / 128) * (g.Kp / BN);
  const int grid = std::min(ntiles, num_sms());
  const int kblocks = g.Cp / SW;
  constexpr int kMaxSmem = 227 * 1024;
  // max pass: B-stationary schedule when U's tile (kblocks x BN x SW bytes) fits next to a 2..4-deep A
  // ring (the requantisation pass is epilogue-bound: it keeps the persistent tile order, gemm_i8.cuh)
  auto bstat = [&](auto stages) -> int {
    constexpr int S = decltype(stages)::value;
    using LB = GemmBSmem<BN, SW, S, Epi::kStageBytes, 4 * Epi::kGroups>;
    auto kern = gemm_i8_bstat<BN, SW, S, Epi>;
    const int smem = LB::bytes(kblocks);
    WL_CUDA(ensure_smem_attr(reinterpret_cast<const void*>(kern), smem));
    kern<<<grid, EpiShape<Epi::kGroups>::kThreads, smem, st>>>(ta, tb, g.T, g.K, g.Cp, g.Kp, e);
    WL_CUDA(cudaGetLastError());
    return WL_OK;
  };
  if (Epi::kStageBytes == 0 && grid >= 36 * (g.Kp / BN)) {
    if (GemmBSmem<BN, SW, 4, Epi::kStageBytes, 4 * Epi::kGroups>::bytes(kblocks) <= kMaxSmem)
      return bstat(std::integral_constant<int, 4>{});
    if (GemmBSmem<BN, SW, 2, Epi::kStageBytes, 4 * Epi::kGroups>::bytes(kblocks) <= kMaxSmem)
      return bstat(std::integral_constant<int, 2>{});
  }
  constexpr int STAGES = Epi::kStageBytes > 0 ? 3 : 4;
  using L = GemmPSmem<BN, SW, STAGES, Epi::kStageBytes, 4 * Epi::kGroups>;
  auto kern = gemm_i8_persistent<BN, SW, STAGES, Epi>;
  WL_CUDA(ensure_smem_attr(reinterpret_cast<const void*>(kern), L::kBytes));
  kern<<<grid, EpiShape<Epi::kGroups>::kThreads, L::kBytes, st>>>(ta, tb, g.T, g.K, g.Cp, g.Kp, e);
  WL_CUDA(cudaGetLastError());
  return WL_OK;
}

template <class Epi>
static int dispatch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, const Geo& g, int bn, int sw, const Epi& e,
                         cudaStream_t st) {
#define WL_G(BN_, SW_) \
  if (bn == BN_ && sw == SW_) return launch_gemm<BN_, SW_, Epi>(ta, tb, g, e, st);
  WL_G(64, 32) WL_G(64, 64) WL_G(64, 128) WL_G(128, 32) WL_G(128, 64) WL_G(128, 128) WL_G(256, 32) WL_G(256, 64)
  WL_G(256, 128)
#undef WL_G
  return fail(WL_ERR_ARG, "no GEMM tile for BN=%d SW=%d", bn, sw);
}

// N tile = whole padded Kout up to 256 (2 TMEM accumulators of BN columns); the max tables hold one
// entry per max-pass epilogue warp column group (BN / EpiHadMax::kGroups columns).
static void gemm_tiles(const Geo& g, int* bn, int* sw) {
  *bn = g.Kp >= 256 ? 256 : g.Kp;  // must match Layout::bn
  *sw = g.Cp % 128 == 0 ? 128 : (g.Cp % 64 == 0 ? 64 : 32);
}
int run_gemm_side(FwdCtx& c, const int8_t* U, const WeightHeader* wh) {
  const Geo& g = c.g;
  cudaStream_t st = c.st;
  int bn, sw;
  gemm_tiles(g, &bn, &sw);
  CUtensorMap ta, tbm;
  if (!tmap_i8_3d(&ta, c.V, g.Cp, 36, g.T, sw, 1, 128) || !tmap_i8_3d(&tbm, U, g.Cp, 36, g.Kp, sw, 1, bn))
    return fail(WL_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  const int wstage = c.leg ? ST_WBC : ST_WT;
  const int qu = c.b.q[wstage];
  int rc;
  {
    EpiHadMax e;
    e.acc = c.acc;
    e.table = c.tabs.t[ST_HAD];
    e.g = g;
    e.nchunk = g.Kp / c.L->bn;
    rc = dispatch_gemm(ta, tbm, g, bn, sw, e, st);
    if (rc) return rc;
#ifndef WL_FH_MULT
#define WL_FH_MULT 2
#endif
    // the table scan is one 16-byte load per (xi, tile) row: full occupancy (8 blocks of 256 per SM)
    const int fh_blocks = (int)std::max<long long>(1, std::min<long long>(4LL * WL_FH_MULT * num_sms(), (36LL * g.T + 255) / 256));
    finalize_hadamard_kernel<<<fh_blocks, 256, 0, st>>>(U, c.V, g, c.acc, wh->wacc, wstage, qu, c.b.q[ST_IT],
                                                           c.tabs.t[ST_HAD], c.L->bn, params_tail(c, ST_HAD));
    prof_mark("gemm_hadamard_max", st);
  }
  auto requant = [&](auto ht) -> int {
    using HT = decltype(ht);
    EpiHadRq<HT> e;
    e.acc = c.acc;
    e.wacc = wh->wacc;
    e.U = U;
    e.V = c.V;
    e.h = reinterpret_cast<HT*>(c.h);
    e.g = g;
    e.fl = c.fl;
    e.wstage = wstage;
    e.qmax_u = qu;
    e.qmax_v = c.b.q[ST_IT];
    e.qmax_h = c.b.q[ST_HAD];
    int r = dispatch_gemm(ta, tbm, g, bn, sw, e, st);
    if (r) return r;
    fixup_had_kernel<HT><<<c.fix_blocks, 128, 0, st>>>(c.fl, U, c.V, reinterpret_cast<HT*>(c.h), g, c.acc, wh->wacc,
                                                       wstage, qu, c.b.q[ST_IT], c.b.q[ST_HAD]);
    return WL_OK;
  };
  rc = c.L->hbytes == 1 ? requant(int8_t{}) : requant(int16_t{});
  if (rc) return rc;
  prof_mark("gemm_hadamard_codes", st);
  WL_CUDA(cudaGetLastError());
  return WL_OK;
}

}  // namespace wl
