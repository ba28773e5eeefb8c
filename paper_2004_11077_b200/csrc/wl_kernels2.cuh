// Transform kernels (v2): fp32 fast path with certified error bounds, exact integer fallback per
// element, deferred fp64 argmax replay through per-entry max tables.
//
// Every stage value T is an integer.  The fast path evaluates T in fp32: the
// first sandwich half is exact and the second rounds once per fma, so |T_f - T| <= E_stage
// (host-computed, wl_abi.cu: stage_rowsums / stage_depth).  Hence
//   * codes: y = fl(T_f * qmax/M + 1.5*2^23) is rhe(T_f * qmax/M); it equals the exact rhe() of
//     the integer stage value unless T_f*qmax/M lies within qmax*E/M (+ fp32 slack) of a
//     half-integer — those elements are recomputed in integers out of line (exact_elem), exact
//     ties replayed in fp64 in the reference's operation order;
//   * maxima: each pass writes the fp32 maximum of every 32-unit entry to a table plus the group's
//     running fp32 maximum; finalize_* recomputes exactly only the entries within 2E of it
//     (integer M, fp64 max_abs by replay), and the last block of that kernel (stage_params_tail) derives r, band and scale.
// Thread mapping: one (tile, channel) unit per thread, channel fastest, so every byte-plane access
// of a warp is one contiguous 32-byte segment; 32-bit element offsets (host-checked < 2^32).
#pragma once
#include "wl_kernels.cuh"

#ifndef WL_MINB
#define WL_MINB 3  // resident blocks per SM requested for the heavy transform kernels (measured best)
#endif

namespace wl {

struct Tables {  // max tables per stage id (only IBC, IT, HAD, OBC, OUT are used)
  unsigned* t[ST_COUNT];
};

struct StageE {  // max row abs-sum of each stage's integer matrix (error-bound factor)
  float e[ST_COUNT];
};

// Certified bound on |T_f - T|: every fma partial sum of the second half is bounded by
// rowsum(L) * max|tmp| and rounds by at most 2^-24 of itself; <= 6 roundings (+ margin).  max|tmp| is
// taken at its static bound qmax_in * rowsum(L) (the first half of the sandwich of codes |c| <= qmax_in):
// the finalize scans use it only to pick the table entries within 2E of the group's fp32 maximum, and a
// looser E just adds a few candidates — measuring max|tmp| per unit cost 36 FMNMX3 per thread in every max
// pass (7 % of the ALU-bound max-only passes).
__device__ __forceinline__ float stage_error(float rowsum, int qmax_in) {
  return 6.5f * 5.9604645e-8f * rowsum * (rowsum * (float)qmax_in);
}
// qmax of the codes a stage transforms
template <int MODE, int STAGE>
__device__ __forceinline__ int stage_in_qmax(const Bits& b) {
  if (STAGE == ST_IBC) return b.q[ST_INPUT];
  if (STAGE == ST_IT) return MODE == 0 ? b.q[ST_INPUT] : b.q[ST_IBC];
  if (STAGE == ST_OBC) return b.q[ST_HAD];
  return MODE == 0 ? b.q[ST_HAD] : b.q[ST_OBC];  // ST_OUT
}

// Small integer -> float without the (slow) I2F pipe: |v| < 2^22 placed in the mantissa of 1.5*2^23.
__device__ __forceinline__ float small_i2f(int v) { return __int_as_float(v + 0x4B400000) - kMagic; }
template <typename XT>
__device__ __forceinline__ XT to_x(int v) {
  if constexpr (sizeof(XT) == 4 && XT(0.5) != XT(0))
    return small_i2f(v);
  else
    return (XT)v;
}

// Window of one (tile, channel) unit in the NHWC input codes: base offset of pixel (r0, q0), the row
// and column strides, and bit masks of the rows / columns inside the image (zero padding).
struct C0Win {
  const int8_t* p;
  uint32_t base, rs, cs;
  unsigned rmask, cmask;
  __device__ __forceinline__ C0Win(const int8_t* c0, const Geo& g, int n, int tile, int c, uint32_t cstride)
      : p(c0) {
    const int ty = (int)g.ftw.div((unsigned)tile), tx = (int)g.ftw.mod((unsigned)tile);
    const int r0 = 4 * ty - g.pad, q0 = 4 * tx - g.pad;
    cs = cstride;
    rs = (uint32_t)g.W * cs;
    base = ((uint32_t)(n * g.H + r0) * (uint32_t)g.W + (uint32_t)q0) * cs + (uint32_t)c;
    rmask = cmask = 0;
#pragma unroll
    for (int j = 0; j < 6; ++j) {
      rmask |= (unsigned)((unsigned)(r0 + j) < (unsigned)g.H) << j;
      cmask |= (unsigned)((unsigned)(q0 + j) < (unsigned)g.W) << j;
    }
  }
  template <typename XT>
  __device__ __forceinline__ void load(XT (&X)[6][6]) const {
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        const bool v = ((rmask >> i) & (cmask >> j) & 1u) != 0;
        X[i][j] = to_x<XT>(v ? (int)__ldg(p + (base + (uint32_t)i * rs + (uint32_t)j * cs)) : 0);
      }
  }
};

// 6x6 window of input codes (NHWC int8, implicit zero padding).
template <typename XT>
__device__ __forceinline__ void load_c0(const int8_t* __restrict__ c0, const Geo& g, int n, int tile, int c,
                                        XT (&X)[6][6]) {
  C0Win(c0, g, n, tile, c, (uint32_t)g.Cp).load(X);
}

// 36 codes of one unit of a [T][36][LD] layout: element e at off + e * plane (plane = LD).
template <typename HT, typename XT>
__device__ __forceinline__ void load_planes(const HT* __restrict__ P, uint32_t plane, uint32_t off, XT (&X)[6][6]) {
  const HT* p = P + off;  // 64-bit base once; e * plane folds into the load's immediate offset
#pragma unroll
  for (int e = 0; e < 36; ++e) X[e / 6][e % 6] = to_x<XT>((int)__ldg(p + (size_t)e * plane));
}

// Max of one (unit row t, channel c) into table entry t*ceil(C/32) + c/32 and the group running max.
__device__ __forceinline__ void record_unit(float m, float tm, int grp, bool active, Acc* acc, int stage,
                                            unsigned* table, int t, int c, int C, bool lazy = false) {
  bool uniform;
  float wmax;
  const int CB = (C + 31) >> 5;
  record_max(active ? m : 0.f, active ? grp : -1, table + (size_t)t * CB + (c >> 5), (C & 31) == 0, acc + stage,
             uniform, wmax);
  publish_mf(active ? m : 0.f, active ? grp : -1, acc + stage, uniform, wmax, lazy);
  // group max of the first-half magnitudes (for the error bound)
  float tw = active ? tm : 0.f;
  if (uniform) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tw = fmaxf(tw, __shfl_xor_sync(0xffffffffu, tw, o));
    if ((threadIdx.x & 31) == 0 && grp >= 0 && tw > 0.f)
      lazy_max(&acc[(size_t)grp * ST_COUNT + stage].TM, __float_as_uint(tw), lazy);
  } else if (active && grp >= 0 && tw > 0.f) {
    lazy_max(&acc[(size_t)grp * ST_COUNT + stage].TM, __float_as_uint(tw), lazy);
  }
}

// ---------------------------------------------------------------------------------- exact elements

struct SrcC0 {  // input codes window
  C0Win w;
  template <typename XT>
  __device__ void load(XT (&X)[6][6]) const { w.load(X); }
};
template <typename HT>
struct SrcPlanes {  // [T][36][LD] codes
  const HT* p;
  uint32_t plane, off;
  template <typename XT>
  __device__ void load(XT (&X)[6][6]) const { load_planes(p, plane, off, X); }
};

// Stage matrix entry with run-time indices: a __constant__ copy of L (the constexpr L::e() folds only
// compile-time indices).
template <class L>
struct LTab {
  int v[6][6];
  constexpr LTab() : v{} {
    for (int i = 0; i < L::R; ++i)
      for (int j = 0; j < L::C; ++j) v[i][j] = L::e(i, j);
  }
};
template <class L>
__constant__ LTab<L> kLTab{};
template <class L>
__device__ __forceinline__ int ltab(int i, int j) {
  return kLTab<L>.v[i][j];
}

// Exact code of element (i, j) of stage L . X . L^T from the unit's input codes xc (row-major 6x6,
// loaded once by fix_unit); ties replayed in fp64.
template <class L>
__device__ __noinline__ int exact_elem(const int* xc, int i, int j, const Acc* a_stage, int qmax, const Acc* a_in,
                                       int qmax_in, bool in_float, const double* __restrict__ Lf) {
  long long T = 0;
#pragma unroll
  for (int l = 0; l < L::C; ++l) {
    int tmp = 0;  // first half |.| <= qmax_in * rowsum(L) < 2^31
#pragma unroll
    for (int l2 = 0; l2 < L::C; ++l2) tmp += xc[l * 6 + l2] * ltab<L>(j, l2);
    T += (long long)ltab<L>(i, l) * tmp;
  }
  const StageQ q = load_int_stage(*a_stage, qmax);
  bool tie = false;
  int code = rq(T, q, tie);
  if (tie) {
    const StageQ qin = in_float ? load_float_stage(*a_in, qmax_in) : load_int_stage(*a_in, qmax_in);
    code = code_of(replay_sandwich(Lf, L::R, L::C, xc, qin.qmax, qin.maxabs, qin.scale, i, j), q);
  }
  return code;
}

// Fast-path requantisation of one element (branch free): code from the magic-number rounding,
// float code k, and the running max distance to the rounded value (band check once per unit).
// `band` is the element's certified error bound in code units (ef * rowsum_i * max|tmp col j|).
__device__ __forceinline__ int rq_nb(float T, float r, float band, float& k, float& dmax) {
  const float y = fmaf(T, r, kMagic);
  k = y - kMagic;
  dmax = fmaxf(dmax, fabsf(fmaf(T, r, -k)) + band);
  return __float_as_int(y) - 0x4B400000;
}

// Rare path for a unit whose fast path came within the band of a half-integer: redo the fp32
// sandwich (deterministic, same values) to find the flagged elements (per-row band), then hand the
// exact code of every flagged element (exact_elem: integer evaluation of that one element, exact
// ties replayed in fp64) to out(i, j, code), which overwrites what the fast path stored.
template <class L, class Src, class Out>
__device__ __noinline__ void fix_unit(Src src, float r, float thr, float ef, const Acc* a_stage, int qmax,
                                      const Acc* a_in, int qmax_in, bool in_float, const double* __restrict__ Lf,
                                      Out out) {
  int Xi[6][6];  // the unit's codes, loaded once (the exact path reuses them)
  src.load(Xi);
  float X[6][6];
#pragma unroll
  for (int e = 0; e < 36; ++e) X[e / 6][e % 6] = (float)Xi[e / 6][e % 6];
  unsigned long long mask = 0;
  sandwich_cols<L>(X, [&](int j, const float (&col)[L::R], float cm) {
#pragma unroll
    for (int i = 0; i < L::R; ++i) {
      const float y = fmaf(col[i], r, kMagic), k = y - kMagic;
      if (fabsf(fmaf(col[i], r, -k)) + ef * cm * row_abs_sum<L>(i) > thr) mask |= 1ull << (i * 6 + j);
    }
  });
  if (!mask) return;
  // Each lane walks its own flagged elements (typically one or two of the 36) and evaluates only those exactly
  // (exact_elem: 42 integer MACs per element); the lanes of a warp iterate together.  The earlier form computed
  // the whole int64 sandwich and then ran one predicated block per element any lane had flagged.
  int xc[36];
#pragma unroll
  for (int u = 0; u < 36; ++u) xc[u] = Xi[u / 6][u % 6];
  while (mask) {
    const int bit = __ffsll((long long)mask) - 1;
    mask &= mask - 1;
    const int i = bit / 6, j = bit - 6 * i;
    out(i, j, exact_elem<L>(xc, i, j, a_stage, qmax, a_in, qmax_in, in_float, Lf));
  }
}

// Per-column fast-path requantisation: code from the magic-number rounding, float code k, and the
// column's max distance to the rounded value; the caller adds the column band
// ef * max|tmp col| * max_row_abs_sum once per column (coarser than per row, 2 fewer ops/element;
// fix_unit re-checks flagged units element by element with the per-row band).
__device__ __forceinline__ int rq_col(float T, float r, float& k, float& dcol) {
  const float y = fmaf(T, r, kMagic);
  k = y - kMagic;
  dcol = fmaxf(dcol, fabsf(fmaf(T, r, -k)));
  return __float_as_int(y) - 0x4B400000;
}

// ---------------------------------------------------------------------------------- deferred fixes
// A unit whose fast path came within the band of a half-integer is appended to a fix list instead
// of being fixed inline (which stalls its warp, and in the staged kernels the whole CTA at the next
// barrier).  A follow-up kernel fixes the listed units one per thread before anything reads them.
// If the list is full the producer fixes inline, so any capacity is correct.
enum FixListId { FIX_IBC = 0, FIX_IT, FIX_OBC, FIX_OUT, FIX_HAD, kFixLists };
struct FixList {
  unsigned* count;  // [kFixLists]
  unsigned* items;  // unit ids t * nch + c, shared by the lists (producer/fixup pairs run in sequence)
  unsigned cap;
};

// Warp-aggregated append; returns true if this lane's unit was deferred.
__device__ __forceinline__ bool defer_fix(const FixList& f, int list, unsigned unit, bool want) {
  const unsigned act = __activemask();
  const unsigned m = __ballot_sync(act, want);
  if (!m) return false;
  const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
  unsigned base = 0;
  if (lane == leader) base = atomicAdd(f.count + list, (unsigned)__popc(m));
  base = __shfl_sync(act, base, leader);
  if (!want) return false;
  const unsigned idx = base + (unsigned)__popc(m & ((1u << lane) - 1u));
  if (idx >= f.cap) return false;
  f.items[idx] = unit;
  return true;
}

__device__ __forceinline__ unsigned fix_count(const FixList& f, int list) {
  const unsigned n = *(volatile const unsigned*)(f.count + list);
  return n < f.cap ? n : f.cap;
}

// Max contribution of one unit from a fixup thread (no warp cooperation).
__device__ __forceinline__ void record_unit_single(float m, float tm, int grp, Acc* acc, int stage, unsigned* table,
                                                   int t, int c, int C) {
  const int CB = (C + 31) >> 5;
  atomicMax(table + (size_t)t * CB + (c >> 5), __float_as_uint(m));
  if (m > 0.f) lazy_max(&acc[(size_t)grp * ST_COUNT + stage].MF, __float_as_uint(m), true);
  if (tm > 0.f) lazy_max(&acc[(size_t)grp * ST_COUNT + stage].TM, __float_as_uint(tm), true);
}

// Exact fix of one input_transform unit (V codes); inline fallback and fixup_it_kernel.
// `dst` = the unit's element 0 (global V or a staged shared block), elements `dstride` apart.
template <int MODE>
__device__ __noinline__ void fix_it_unit(const int8_t* __restrict__ c0, const int8_t* __restrict__ c1, int8_t* dst,
                                         uint32_t dstride, const Geo& g, const Bits& b, const Acc* acc,
                                         const PlanF64* __restrict__ pf, int t, int c, uint32_t plane) {
  const int n = (int)g.fTP.div((unsigned)t), tile = (int)g.fTP.mod((unsigned)t), grp = (int)g.fipg.div((unsigned)n);
  const Acc* ga = acc + (size_t)grp * ST_COUNT;
  const float r = ga[ST_IT].r, thr = ga[ST_IT].thr, ef = ga[ST_IT].ef;
  const uint32_t off = (uint32_t)t * 36u * plane + (uint32_t)c;
  auto fix = [dst, dstride](int i, int j, int code) { dst[(6 * i + j) * dstride] = (int8_t)code; };
  if constexpr (MODE == 0) {
    const C0Win win(c0, g, n, tile, c, plane);
    fix_unit<tab::Can_IT>(SrcC0{win}, r, thr, ef, ga + ST_IT, b.q[ST_IT], ga + ST_INPUT, b.q[ST_INPUT], true, pf->it,
                          fix);
  } else {
    fix_unit<tab::Leg_IT>(SrcPlanes<int8_t>{c1, plane, off}, r, thr, ef, ga + ST_IT, b.q[ST_IT], ga + ST_IBC,
                          b.q[ST_IBC], false, pf->it, fix);
  }
}

// Exact fix of one output unit: every flagged element (i, j) is handed to put(i, j, value) as its
// dequantised value + bias (crop not applied: the caller decides where the value goes).
template <int MODE, typename HT, typename YT, class Put>
__device__ __noinline__ void fix_out_unit_to(const HT* __restrict__ h, const int8_t* __restrict__ c4,
                                             const YT* __restrict__ bias, const Geo& g, const Bits& b, const Acc* acc,
                                             const PlanF64* __restrict__ pf, int t, int k, uint32_t plane, Put put) {
  const int n = (int)g.fTP.div((unsigned)t), grp = (int)g.fipg.div((unsigned)n);
  const Acc* ga = acc + (size_t)grp * ST_COUNT;
  const float r = ga[ST_OUT].r, thr = ga[ST_OUT].thr, ef = ga[ST_OUT].ef;
  const double scale = ga[ST_OUT].scale;
  const double maxabs = __longlong_as_double((long long)ga[ST_OUT].F);
  const int qo = b.q[ST_OUT];
  const YT bk = bias ? bias[k] : (YT)0;
  const uint32_t off = (uint32_t)t * 36u * plane + (uint32_t)k;
  auto fix = [&](int i, int j, int code) {
    const YT v = code == qo ? (YT)maxabs : (code == -qo ? (YT)-maxabs : (YT)((double)code * scale));
    put(i, j, v + bk);
  };
  if constexpr (MODE == 0)
    fix_unit<tab::Can_OT>(SrcPlanes<HT>{h, plane, off}, r, thr, ef, ga + ST_OUT, qo, ga + ST_HAD, b.q[ST_HAD], false,
                          pf->ot, fix);
  else
    fix_unit<tab::Leg_OT>(SrcPlanes<int8_t>{c4, plane, off}, r, thr, ef, ga + ST_OUT, qo, ga + ST_OBC, b.q[ST_OBC],
                          false, pf->ot, fix);
}

// Exact fix of one output unit: flagged elements of y rewritten (dequantised, + bias, cropped).
template <int MODE, typename HT, typename YT>
__device__ __forceinline__ void fix_out_unit(const HT* __restrict__ h, const int8_t* __restrict__ c4,
                                             YT* __restrict__ y, const YT* __restrict__ bias, const Geo& g,
                                             const Bits& b, const Acc* acc, const PlanF64* __restrict__ pf, int t,
                                             int k, uint32_t plane) {
  const int n = (int)g.fTP.div((unsigned)t), tile = (int)g.fTP.mod((unsigned)t);
  const int ty = (int)g.ftw.div((unsigned)tile), tx = (int)g.ftw.mod((unsigned)tile);
  fix_out_unit_to<MODE, HT, YT>(h, c4, bias, g, b, acc, pf, t, k, plane, [&](int i, int j, YT v) {
    const int rr = 4 * ty + i, cc = 4 * tx + j;
    if (rr < g.Ho && cc < g.Wo) y[(((size_t)n * g.K + k) * g.Ho + rr) * g.Wo + cc] = v;
  });
}

// r, threshold and reference scale of one stage for every group, once its M and F are final.
// (M and F are read past L1: in the tail below other blocks' atomics produced them during this kernel.)
__device__ __forceinline__ void stage_params_of(Acc* acc, int gi, int stage, int qmax, float depth) {
  Acc& a = acc[(size_t)gi * ST_COUNT + stage];
  const long long M = (long long)__ldcg(&a.M);
  const double maxabs = __longlong_as_double((long long)__ldcg(&a.F));
  a.r = M ? (float)((double)qmax / (double)M) : 0.f;
  // per-element band = ef * rowsum_i * max|tmp col j| (the element's fp32 error E_ij times qmax/M);
  // slack for r = fl(qmax/M) (relative 2^-24 on a value <= qmax) and the fma rounding of d
  a.ef = M ? (float)((double)qmax * ((double)depth + 0.5) * 5.9604644775390625e-8 / (double)M) : 0.f;
  a.thr = M ? 0.5f - (float)((qmax + 1) * 1.25 * 5.9604644775390625e-8) : 1.f;
  a.scale = maxabs > 0.0 ? maxabs / (double)qmax : 1.0;
}

// Tail of the kernel that makes a stage's M and F final: the last block to finish derives the fast-path
// parameters of every group (one launch less per stage on the launch-bound small shapes).  `done` is the
// stage's slot of the zeroed counter block (kDoneSlot0 + stage).  Every thread of the block must call it.
constexpr int kDoneSlot0 = 16;
struct ParamsTail {
  int groups, qmax;
  float depth;
  unsigned* done;
};
__device__ __forceinline__ void stage_params_tail(Acc* acc, int stage, const ParamsTail& p) {
  __shared__ int wl_tail_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    wl_tail_last = atomicAdd(p.done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!wl_tail_last) return;
  __threadfence();
  for (int gi = threadIdx.x; gi < p.groups; gi += blockDim.x) stage_params_of(acc, gi, stage, p.qmax, p.depth);
}

// Dequantised fp32 output of every code of the output stage, per group (quantize.py:120-125:
// code * scale in fp64, +-qmax snapped to +-max_abs, then rounded to fp32): table[g][code + qmax].
// One block per group.  The block also certifies an arithmetic form of the same map for the hot
// output pass: with scale = s_hi + s_lo (fp32 head and tail of the fp64 scale) the value
// fma(k, s_hi, k * s_lo) is compared with the table entry of EVERY code of the group, +-qmax included;
// odq[g] = {s_hi, s_lo, ok}.  A group with ok = 1 dequantises with two fp32 instructions per output
// (bit-identical to the table by this exhaustive check); any other group keeps the table gather.
template <int kInTU = 0>  // header-defined kernel: instantiated only in the TUs that launch it
__global__ void __launch_bounds__(256) out_table_kernel(const Acc* __restrict__ acc, int groups, int qmax,
                                                        float* __restrict__ table, float4* __restrict__ odq) {
  const int gi = blockIdx.x;
  if (gi >= groups) return;
  const int width = 2 * qmax + 1;
  const Acc& a = acc[(size_t)gi * ST_COUNT + ST_OUT];
  const double maxabs = __longlong_as_double((long long)a.F), scale = a.scale;
  const float s_hi = (float)scale, s_lo = (float)(scale - (double)s_hi);
  bool ok = true;
  for (int i = threadIdx.x; i < width; i += blockDim.x) {
    const int code = i - qmax;
    const float v = code == qmax ? (float)maxabs : (code == -qmax ? (float)-maxabs : (float)((double)code * scale));
    table[(size_t)gi * width + i] = v;
    const float kf = (float)code;
    ok = ok && __float_as_uint(__fmaf_rn(kf, s_hi, __fmul_rn(kf, s_lo))) == __float_as_uint(v);
  }
  ok = __syncthreads_and(ok);
  if (threadIdx.x == 0) odq[gi] = make_float4(s_hi, s_lo, ok ? 1.f : 0.f, 0.f);
}

// ---------------------------------------------------------------------------------- input side

// First input stage maximum: canonical input_transform (B^T), Legendre input_base_change (P^-T).
template <int MODE, int LD>
__global__ void __launch_bounds__(256) in_a_kernel(const int8_t* __restrict__ c0, Geo g, Acc* __restrict__ acc,
                                                   Tables tabs) {
  const uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = idx < (uint32_t)g.T * (uint32_t)g.C;
  const uint32_t id = active ? idx : 0u;
  const int c = (int)g.fC.mod(id), t = (int)g.fC.div(id);
  const int n = (int)g.fTP.div((unsigned)t), tile = (int)g.fTP.mod((unsigned)t);
  const int grp = (int)g.fipg.div((unsigned)n);
  float X[6][6];
  C0Win(c0, g, n, tile, c, LD).load(X);
  constexpr int st = MODE == 0 ? ST_IT : ST_IBC;
  float m = 0.f, tm = 0.f;
  auto mx = [&](int, const float (&col)[6]) {
#pragma unroll
    for (int i = 0; i < 6; ++i) m = fmaxf(m, fabsf(col[i]));
  };
  if constexpr (MODE == 0)
    sandwich_cols<tab::Can_IT>(X, mx, &tm);
  else
    sandwich_cols<tab::Leg_IBC>(X, mx, &tm);
  record_unit(m, tm, grp, active, acc, st, tabs.t[st], t, c, g.C, g.lazy);
}

// Legendre: input_base_change codes c1 (stored) and input_transform maximum.
template <int LD>
__global__ void __launch_bounds__(256, WL_MINB) in_b_kernel(const int8_t* __restrict__ c0, int8_t* __restrict__ c1, Geo g,
                                                   Bits b, Acc* __restrict__ acc, const PlanF64* __restrict__ pf,
                                                   Tables tabs, FixList fl) {
  const uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = idx < (uint32_t)g.T * (uint32_t)g.C;
  const uint32_t id = active ? idx : 0u;
  const int c = (int)g.fC.mod(id), t = (int)g.fC.div(id);
  const int n = (int)g.fTP.div((unsigned)t), tile = (int)g.fTP.mod((unsigned)t);
  const int grp = (int)g.fipg.div((unsigned)n);
  const Acc* ga = acc + (size_t)grp * ST_COUNT;
  const float r = ga[ST_IBC].r, thr = ga[ST_IBC].thr, ef = ga[ST_IBC].ef;
  constexpr uint32_t plane = LD;
  int8_t* dst = c1 + ((size_t)t * 36 * LD + c);
  float K1[6][6];
  bool deferred = false;
  {
    const C0Win win(c0, g, n, tile, c, LD);
    float X[6][6];
    win.load(X);
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
    deferred = defer_fix(fl, FIX_IBC, id, want);
    if (want && !deferred) {
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
  record_unit(m, tm, grp, active, acc, ST_IT, tabs.t[ST_IT], t, c, g.C, g.lazy);
}

// V codes.  Canonical: from c0 through B^T.  Legendre: from the stored c1 through B_P^T.
template <int MODE, int LD>
__global__ void __launch_bounds__(256, WL_MINB) in_c_kernel(const int8_t* __restrict__ c0, const int8_t* __restrict__ c1,
                                                   int8_t* __restrict__ V, const __grid_constant__ Geo g, const __grid_constant__ Bits b, Acc* __restrict__ acc,
                                                   const PlanF64* __restrict__ pf, FixList fl) {
  const uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (uint32_t)g.T * (uint32_t)g.C) return;
  const int c = (int)g.fC.mod(idx), t = (int)g.fC.div(idx);
  const int n = (int)g.fTP.div((unsigned)t), tile = (int)g.fTP.mod((unsigned)t);
  const int grp = (int)g.fipg.div((unsigned)n);
  const Acc* ga = acc + (size_t)grp * ST_COUNT;
  const float r = ga[ST_IT].r, thr = ga[ST_IT].thr, ef = ga[ST_IT].ef;
  constexpr uint32_t plane = LD;
  const uint32_t off = (uint32_t)t * 36u * LD + c;
  int8_t* dst = V + off;
  float X[6][6];
  float dmax = 0.f, kd;
  constexpr bool kCan = MODE == 0;
  using LIT = std::conditional_t<kCan, tab::Can_IT, tab::Leg_IT>;
  auto store = [&](int j, const float (&col)[6], float cm) {
    float dcol = 0.f;
#pragma unroll
    for (int i = 0; i < 6; ++i) dst[(6 * i + j) * plane] = (int8_t)rq_col(col[i], r, kd, dcol);
    dmax = fmaxf(dmax, fmaf(ef * cm, max_row_abs_sum<LIT>(), dcol));
  };
  if constexpr (MODE == 0) {
    const C0Win win(c0, g, n, tile, c, LD);
    win.load(X);
  } else {
    load_planes(c1, plane, off, X);
  }
  sandwich_cols<LIT>(X, store);
  const bool want = dmax > thr;
  if (want && !defer_fix(fl, FIX_IT, idx, want)) fix_it_unit<MODE>(c0, c1, dst, LD, g, b, acc, pf, t, c, LD);
}

// Argmax replay of a warp whose 32 lanes hold units of ONE scale group (lane = channel of one tile row; every
// lane calls, inactive lanes with m = 0).  Only the lanes holding the warp's maximum replay, and only while
// that maximum can still be the group's (the stored maximum only grows, so a lane equal to the final maximum
// always passes); each lane walks its own set `em` of argmax elements, so a warp's replay calls run together
// instead of one after the other per distinct element (the fp64 replays were 3/4 of the instructions of the
// finalize-exec kernels: 32 lanes with 32 different argmax elements).  fp64 magnitudes order like the
// integers (gap >= 1/M relative, fp64 noise < 1e-13), so the atomicMax over replayed values is the
// reference's max_abs whichever other lanes also replay.
template <class R>
__device__ __forceinline__ void warp_argmax_replay(long long m, unsigned long long em, Acc* a, R&& replay) {
  long long wmax = m;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const long long other = __shfl_xor_sync(0xffffffffu, wmax, o);
    wmax = other > wmax ? other : wmax;
  }
  if (wmax <= 0 || m != wmax) return;
  if (m < (long long)(*(volatile const unsigned long long*)&a->M)) return;
  double f = 0.0;
  while (em) {
    const int e = __ffsll((long long)em) - 1;
    em &= em - 1;
    f = fmax(f, fabs(replay(e)));
  }
  atomicMax(&a->M, (unsigned long long)m);
  atomicMax(&a->F, dbits(f));
}

// Exact recomputation of one input-side unit: local exact max and fp64 max_abs of its argmax.
template <int MODE, int STAGE>
__device__ void exact_input_unit(const int8_t* __restrict__ c0, const int8_t* __restrict__ c1, const Geo& g,
                                 const Bits& b, Acc* acc, const PlanF64* pf, int t, int c, bool active) {
  // called by all 32 lanes of a warp with the same tile t (lane = channel, `active` = channel in range)
  const int n = (int)g.fTP.div((unsigned)t), tile = (int)g.fTP.mod((unsigned)t);
  const int grp = (int)g.fipg.div((unsigned)n);
  Acc* ga = acc + (size_t)grp * ST_COUNT;
  int xc[36];
  long long m = 0;
  unsigned long long em = 0;
  StageQ qin;
  const double* Lf = nullptr;
  if (active) {
    int Xi[6][6];
    long long T[6][6];
    if (MODE == 1 && STAGE == ST_IT) {
      load_planes(c1, (uint32_t)g.Cp, (uint32_t)t * 36u * g.Cp + c, Xi);
      sandwich<tab::Leg_IT>(Xi, T);
      qin = load_int_stage(ga[ST_IBC], b.q[ST_IBC]);
      Lf = pf->it;
    } else {
      load_c0(c0, g, n, tile, c, Xi);
      int Ti[6][6];
      if (MODE == 0)
        sandwich<tab::Can_IT>(Xi, Ti);
      else
        sandwich<tab::Leg_IBC>(Xi, Ti);
#pragma unroll
      for (int e = 0; e < 36; ++e) T[e / 6][e % 6] = Ti[e / 6][e % 6];
      qin = load_float_stage(ga[ST_INPUT], b.q[ST_INPUT]);
      Lf = MODE == 0 ? pf->it : pf->ibc;
    }
    m = absmax36(T);
#pragma unroll
    for (int e = 0; e < 36; ++e) {
      xc[e] = Xi[e / 6][e % 6];
      const long long v = T[e / 6][e % 6];
      if ((v < 0 ? -v : v) == m) em |= 1ull << e;
    }
  }
  warp_argmax_replay(m, em, ga + STAGE, [&](int e) {
    return replay_sandwich(Lf, 6, 6, xc, qin.qmax, qin.maxabs, qin.scale, e / 6, e % 6);
  });
}

// Finalize candidate lists: count slot kCandSlot0 + stage of the FixList counters (the fix lists use
// slots 0..4), items in the shared FixList buffer (free between a stage's fixup and the next
// producer).  Appends this warp's candidate lanes (entry ids) and returns the lanes that did not fit.
constexpr int kCandSlot0 = 4;
__device__ __forceinline__ unsigned defer_cands(const FixList& f, int slot, unsigned mask, unsigned entry) {
  if (!mask) return 0u;
  const int lane = threadIdx.x & 31, leader = __ffs(mask) - 1;
  unsigned base = 0;
  if (lane == leader) base = atomicAdd(f.count + slot, (unsigned)__popc(mask));
  base = __shfl_sync(0xffffffffu, base, leader);
  const bool mine = (mask >> lane) & 1u;
  const unsigned idx = base + (unsigned)__popc(mask & ((1u << lane) - 1u));
  const bool stored = mine && idx < f.cap;
  if (stored) f.items[idx] = entry;
  return mask & ~__ballot_sync(0xffffffffu, stored);
}

// Scan a stage's max table; warps recompute exactly the entries within 2E of the group's fp32 max.
template <int MODE, int STAGE>
__global__ void finalize_input_kernel(const int8_t* __restrict__ c0, const int8_t* __restrict__ c1, Geo g, Bits b,
                                      Acc* __restrict__ acc, const PlanF64* __restrict__ pf,
                                      const unsigned* __restrict__ table, float rowsum, FixList fl) {
  // thread per tile row t (group data loaded once), walking the row's CB entries; a warp's 32
  // consecutive rows read contiguous table segments.  Entries within 2E of the group's fp32 max are
  // recomputed exactly by the whole warp (lane per channel).
  const int NB = (g.C + 31) >> 5;
  const int lane = threadIdx.x & 31;
  const unsigned T = (unsigned)g.T;
  const unsigned nthr = gridDim.x * blockDim.x;
  for (unsigned t0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; t0 < T; t0 += nthr) {
    const unsigned t = t0 + lane;
    const bool valid = t < T;
    float lim = 3.4e38f;
    if (valid) {
      const int grp = (int)g.fipg.div(g.fTP.div(t));
      const Acc& a = acc[(size_t)grp * ST_COUNT + STAGE];
      lim = __uint_as_float(a.MF) - 2.f * stage_error(rowsum, stage_in_qmax<MODE, STAGE>(b));
    }
    for (int cb = 0; cb < NB; ++cb) {
      const float v = valid ? __uint_as_float(table[(size_t)t * NB + cb]) : 0.f;
      unsigned mask = __ballot_sync(0xffffffffu, v > 0.f && v >= lim);
      // candidate entries go to a list processed one warp each by finalize_*_exec (the scan's warps
      // stay short; a group whose maximum many entries reach no longer serialises on one warp);
      // a full list falls back to recomputing here
      mask = defer_cands(fl, kCandSlot0 + STAGE, mask, t * (unsigned)NB + (unsigned)cb);
      while (mask) {
        const int l = __ffs(mask) - 1;
        mask &= mask - 1;
        const int tl = (int)t0 + l, ch = cb * 32 + lane;
        exact_input_unit<MODE, STAGE>(c0, c1, g, b, acc, pf, tl, ch, ch < g.C);
      }
    }
  }
}

// Finalize candidates, one warp per listed (tile row, 32-channel block) entry, lane per channel.
template <int MODE, int STAGE>
__global__ void __launch_bounds__(256) finalize_input_exec(const int8_t* __restrict__ c0, const int8_t* __restrict__ c1,
                                                           Geo g, Bits b, Acc* __restrict__ acc,
                                                           const PlanF64* __restrict__ pf, FixList fl,
                                                           ParamsTail tail) {
  const unsigned NB = (unsigned)((g.C + 31) >> 5);
  const unsigned cnt = fix_count(fl, kCandSlot0 + STAGE);
  const int lane = threadIdx.x & 31;
  const unsigned nw = (gridDim.x * blockDim.x) >> 5;
  for (unsigned i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < cnt; i += nw) {
    const unsigned e = fl.items[i], t = e / NB, cb = e - t * NB;
    const int ch = (int)cb * 32 + lane;
    exact_input_unit<MODE, STAGE>(c0, c1, g, b, acc, pf, (int)t, ch, ch < g.C);
  }
  stage_params_tail(acc, STAGE, tail);
}

// ---------------------------------------------------------------------------------- output side

// Thread per (tile t, out channel k), k fastest.
// OUT_A: Legendre output_base_change max (P^-T on h) | canonical output max (A^T on h, cropped).
template <int MODE, typename HT, int LD>
__global__ void __launch_bounds__(256) out_a_kernel(const HT* __restrict__ h, Geo g, Acc* __restrict__ acc,
                                                    Tables tabs) {
  const uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = idx < (uint32_t)g.T * (uint32_t)g.K;
  const uint32_t id = active ? idx : 0u;
  const int k = (int)g.fK.mod(id), t = (int)g.fK.div(id);
  const int n = (int)g.fTP.div((unsigned)t), tile = (int)g.fTP.mod((unsigned)t);
  const int grp = (int)g.fipg.div((unsigned)n);
  const int ty = (int)g.ftw.div((unsigned)tile), tx = (int)g.ftw.mod((unsigned)tile);
  float X[6][6];
  load_planes(h, (uint32_t)LD, (uint32_t)t * 36u * LD + k, X);
  float m = 0.f, tm = 0.f;
  constexpr int st = MODE == 0 ? ST_OUT : ST_OBC;
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
  record_unit(m, tm, grp, active, acc, st, tabs.t[st], t, k, g.K, g.lazy);
}

// Legendre: output_base_change codes c4 (stored) and cropped output maximum.
template <typename HT, int LD>
__global__ void __launch_bounds__(256, WL_MINB) out_b_kernel(const HT* __restrict__ h, int8_t* __restrict__ c4, Geo g, Bits b,
                                                    Acc* __restrict__ acc, const PlanF64* __restrict__ pf,
                                                    Tables tabs, FixList fl) {
  const uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = idx < (uint32_t)g.T * (uint32_t)g.K;
  const uint32_t id = active ? idx : 0u;
  const int k = (int)g.fK.mod(id), t = (int)g.fK.div(id);
  const int n = (int)g.fTP.div((unsigned)t), tile = (int)g.fTP.mod((unsigned)t);
  const int grp = (int)g.fipg.div((unsigned)n);
  const Acc* ga = acc + (size_t)grp * ST_COUNT;
  const float r = ga[ST_OBC].r, thr = ga[ST_OBC].thr, ef = ga[ST_OBC].ef;
  constexpr uint32_t plane = LD;
  const uint32_t off = (uint32_t)t * 36u * LD + k;
  int8_t* dst = c4 + off;
  float K4[6][6];
  bool deferred = false;
  {
    float X[6][6];
    load_planes(h, plane, off, X);
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
    deferred = defer_fix(fl, FIX_OBC, id, want);
    if (want && !deferred) {
      fix_unit<tab::Leg_OBC>(SrcPlanes<HT>{h, plane, off}, r, thr, ef, ga + ST_OBC, b.q[ST_OBC], ga + ST_HAD,
                             b.q[ST_HAD], false, pf->obc,
                             [dst](int i, int j, int code) { dst[(6 * i + j) * plane] = (int8_t)code; });
#pragma unroll
      for (int e = 0; e < 36; ++e) K4[e / 6][e % 6] = (float)dst[e * plane];
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
  record_unit(m, tm, grp, active, acc, ST_OUT, tabs.t[ST_OUT], t, k, g.K, g.lazy);
}

// Final output: codes of the output stage, dequantised (snap +-qmax to +-max_abs), + bias, NCHW in
// fp32 (YT = float, dequant table optional) or in the reference's fp64 (YT = double, quantize.py:120-125).
template <int MODE, typename HT, int LD, typename YT = float>
__global__ void __launch_bounds__(256, WL_MINB) out_c_kernel(const HT* __restrict__ h, const int8_t* __restrict__ c4,
                                                    YT* __restrict__ y, const YT* __restrict__ bias, const __grid_constant__ Geo g,
                                                    const __grid_constant__ Bits b, Acc* __restrict__ acc, const PlanF64* __restrict__ pf,
                                                    const float* __restrict__ otab, FixList fl) {
  const uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (uint32_t)g.T * (uint32_t)g.K) return;
  const int k = (int)g.fK.mod(idx), t = (int)g.fK.div(idx);
  const int n = (int)g.fTP.div((unsigned)t), tile = (int)g.fTP.mod((unsigned)t);
  const int ty = (int)g.ftw.div((unsigned)tile), tx = (int)g.ftw.mod((unsigned)tile);
  const int grp = (int)g.fipg.div((unsigned)n);
  const Acc* ga = acc + (size_t)grp * ST_COUNT;
  const float r = ga[ST_OUT].r, thr = ga[ST_OUT].thr, ef = ga[ST_OUT].ef;
  const double scale = ga[ST_OUT].scale;
  const double maxabs = __longlong_as_double((long long)ga[ST_OUT].F);
  const int qo = b.q[ST_OUT];
  constexpr uint32_t plane = LD;
  const uint32_t off = (uint32_t)t * 36u * LD + k;
  YT Yo[4][4];
  float X[6][6];
  float dmax = 0.f, kd;
  const float* tabg = otab ? otab + (size_t)grp * (2 * qo + 1) + qo : nullptr;
  auto deqf = [=](int code) -> YT {
    if constexpr (sizeof(YT) == 4)
      if (tabg) return __ldg(tabg + code);
    return code == qo ? (YT)maxabs : (code == -qo ? (YT)-maxabs : (YT)((double)code * scale));
  };
  using LOT = std::conditional_t<MODE == 0, tab::Can_OT, tab::Leg_OT>;
  auto emit = [&](int j, const float (&col)[4], float cm) {
    float dcol = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) Yo[i][j] = deqf(rq_col(col[i], r, kd, dcol));
    dmax = fmaxf(dmax, fmaf(ef * cm, max_row_abs_sum<LOT>(), dcol));
  };
  if constexpr (MODE == 0)
    load_planes(h, plane, off, X);
  else
    load_planes(c4, plane, off, X);
  sandwich_cols<LOT>(X, emit);
  const YT bk = bias ? __ldg(&bias[k]) : (YT)0;
  const bool vec = sizeof(YT) == 4 && (g.Wo & 3) == 0 && (reinterpret_cast<uintptr_t>(y) & 15) == 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int rr = 4 * ty + i;
    if (rr >= g.Ho) continue;
    YT* row = y + (((size_t)n * g.K + k) * g.Ho + rr) * g.Wo + 4 * tx;
    if (vec) {
      *reinterpret_cast<float4*>(row) = make_float4((float)(Yo[i][0] + bk), (float)(Yo[i][1] + bk),
                                                    (float)(Yo[i][2] + bk), (float)(Yo[i][3] + bk));
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (4 * tx + j < g.Wo) row[j] = Yo[i][j] + bk;
    }
  }
  const bool want = dmax > thr;
  if (want && !defer_fix(fl, FIX_OUT, idx, want))
    fix_out_unit<MODE, HT, YT>(h, c4, y, bias, g, b, acc, pf, t, k, plane);
}

// Exact c4 codes of one unit from its h codes (int64 sandwich, ties replayed in fp64); these are the
// codes the fast path produces after its certified fixes.
template <typename HT>
__device__ __forceinline__ void exact_c4_from_h(const HT* __restrict__ h, uint32_t plane, uint32_t off, const Acc* ga,
                                                const Bits& b, const PlanF64* __restrict__ pf, int (&c4)[6][6]) {
  int Xi[6][6];
  load_planes(h, plane, off, Xi);
  long long T3[6][6];
  sandwich<tab::Leg_OBC>(Xi, T3);
  const StageQ q = load_int_stage(ga[ST_OBC], b.q[ST_OBC]);
  unsigned long long ties = 0;
#pragma unroll
  for (int e = 0; e < 36; ++e) {
    bool tie = false;
    c4[e / 6][e % 6] = rq(T3[e / 6][e % 6], q, tie);
    if (tie) ties |= 1ull << e;
  }
  if (ties) {
    // exact ties, replayed in fp64: each lane walks its own tie set (one out-of-line replay site instead of 36
    // unrolled ones), the code lands in its register through a predicated select
    int xc[36];
#pragma unroll
    for (int u = 0; u < 36; ++u) xc[u] = Xi[u / 6][u % 6];
    const StageQ qin = load_int_stage(ga[ST_HAD], b.q[ST_HAD]);
    while (ties) {
      const int e = __ffsll((long long)ties) - 1;
      ties &= ties - 1;
      const int code = code_of(replay_sandwich(pf->obc, 6, 6, xc, qin.qmax, qin.maxabs, qin.scale, e / 6, e % 6), q);
#pragma unroll
      for (int u = 0; u < 36; ++u)
        if (u == e) c4[u / 6][u % 6] = code;
    }
  }
}

template <int MODE, int STAGE, typename HT, bool FROM_H = false>
__device__ void exact_output_unit(const HT* __restrict__ h, const int8_t* __restrict__ c4, const Geo& g, const Bits& b,
                                  Acc* acc, const PlanF64* pf, int t, int k, bool active) {
  // called by all 32 lanes of a warp with the same tile t (lane = output channel, `active` = channel in range)
  const int n = (int)g.fTP.div((unsigned)t), tile = (int)g.fTP.mod((unsigned)t);
  const int ty = (int)g.ftw.div((unsigned)tile), tx = (int)g.ftw.mod((unsigned)tile);
  const int grp = (int)g.fipg.div((unsigned)n);
  Acc* ga = acc + (size_t)grp * ST_COUNT;
  int xc[36];
  long long m = 0;
  unsigned long long em = 0;
  StageQ qin;
  if (MODE == 1 && STAGE == ST_OBC) {
    if (active) {
      int Xi[6][6];
      load_planes(h, (uint32_t)g.Kp, (uint32_t)t * 36u * g.Kp + k, Xi);
      int T[6][6];
      sandwich<tab::Leg_OBC>(Xi, T);
      m = absmax36(T);
      qin = load_int_stage(ga[ST_HAD], b.q[ST_HAD]);
#pragma unroll
      for (int e = 0; e < 36; ++e) {
        xc[e] = Xi[e / 6][e % 6];
        const long long v = T[e / 6][e % 6];
        if ((v < 0 ? -v : v) == m) em |= 1ull << e;
      }
    }
    warp_argmax_replay(m, em, ga + ST_OBC, [&](int e) {
      return replay_sandwich(pf->obc, 6, 6, xc, qin.qmax, qin.maxabs, qin.scale, e / 6, e % 6);
    });
    return;
  }
  if (active) {
    int Xi[6][6];
    long long Y[4][4];
    if (MODE == 0) {
      load_planes(h, (uint32_t)g.Kp, (uint32_t)t * 36u * g.Kp + k, Xi);
      int Y32[4][4];
      sandwich<tab::Can_OT>(Xi, Y32);
#pragma unroll
      for (int e = 0; e < 16; ++e) Y[e / 4][e % 4] = Y32[e / 4][e % 4];
      qin = load_int_stage(ga[ST_HAD], b.q[ST_HAD]);
    } else {
      if constexpr (FROM_H)
        exact_c4_from_h<HT>(h, (uint32_t)g.Kp, (uint32_t)t * 36u * g.Kp + (uint32_t)k, ga, b, pf, Xi);
      else
        load_planes(c4, (uint32_t)g.Kp, (uint32_t)t * 36u * g.Kp + k, Xi);
      sandwich<tab::Leg_OT>(Xi, Y);
      qin = load_int_stage(ga[ST_OBC], b.q[ST_OBC]);
    }
    m = absmax_crop(Y, ty, tx, g);
#pragma unroll
    for (int e = 0; e < 36; ++e) xc[e] = Xi[e / 6][e % 6];
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int i = e / 4, j = e % 4;
      const long long v = Y[i][j];
      if (4 * ty + i < g.Ho && 4 * tx + j < g.Wo && (v < 0 ? -v : v) == m) em |= 1ull << e;
    }
  }
  warp_argmax_replay(m, em, ga + ST_OUT, [&](int e) {
    return replay_sandwich(pf->ot, 4, 6, xc, qin.qmax, qin.maxabs, qin.scale, e / 4, e % 4);
  });
}

template <int MODE, int STAGE, typename HT, bool FROM_H = false>
__global__ void finalize_output_kernel(const HT* __restrict__ h, const int8_t* __restrict__ c4, Geo g, Bits b,
                                       Acc* __restrict__ acc, const PlanF64* __restrict__ pf,
                                       const unsigned* __restrict__ table, float rowsum, FixList fl) {
  // thread per tile row t (group data loaded once), walking the row's KB entries; a warp's 32
  // consecutive rows read contiguous table segments.  Entries within 2E of the group's fp32 max are
  // recomputed exactly by the whole warp (lane per channel).
  const int NB = (g.K + 31) >> 5;
  const int lane = threadIdx.x & 31;
  const unsigned T = (unsigned)g.T;
  const unsigned nthr = gridDim.x * blockDim.x;
  for (unsigned t0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; t0 < T; t0 += nthr) {
    const unsigned t = t0 + lane;
    const bool valid = t < T;
    float lim = 3.4e38f;
    if (valid) {
      const int grp = (int)g.fipg.div(g.fTP.div(t));
      const Acc& a = acc[(size_t)grp * ST_COUNT + STAGE];
      lim = __uint_as_float(a.MF) - 2.f * stage_error(rowsum, stage_in_qmax<MODE, STAGE>(b));
    }
    for (int cb = 0; cb < NB; ++cb) {
      const float v = valid ? __uint_as_float(table[(size_t)t * NB + cb]) : 0.f;
      unsigned mask = __ballot_sync(0xffffffffu, v > 0.f && v >= lim);
      // candidate entries go to a list processed one warp each by finalize_*_exec (the scan's warps
      // stay short; a group whose maximum many entries reach no longer serialises on one warp);
      // a full list falls back to recomputing here
      mask = defer_cands(fl, kCandSlot0 + STAGE, mask, t * (unsigned)NB + (unsigned)cb);
      while (mask) {
        const int l = __ffs(mask) - 1;
        mask &= mask - 1;
        const int tl = (int)t0 + l, ch = cb * 32 + lane;
        exact_output_unit<MODE, STAGE, HT, FROM_H>(h, c4, g, b, acc, pf, tl, ch, ch < g.K);
      }
    }
  }
}

template <int MODE, int STAGE, typename HT, bool FROM_H = false>
__global__ void __launch_bounds__(256) finalize_output_exec(const HT* __restrict__ h, const int8_t* __restrict__ c4,
                                                            Geo g, Bits b, Acc* __restrict__ acc,
                                                            const PlanF64* __restrict__ pf, FixList fl,
                                                            ParamsTail tail) {
  const unsigned NB = (unsigned)((g.K + 31) >> 5);
  const unsigned cnt = fix_count(fl, kCandSlot0 + STAGE);
  const int lane = threadIdx.x & 31;
  const unsigned nw = (gridDim.x * blockDim.x) >> 5;
  for (unsigned i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < cnt; i += nw) {
    const unsigned e = fl.items[i], t = e / NB, cb = e - t * NB;
    const int ch = (int)cb * 32 + lane;
    exact_output_unit<MODE, STAGE, HT, FROM_H>(h, c4, g, b, acc, pf, (int)t, ch, ch < g.K);
  }
  stage_params_tail(acc, STAGE, tail);
}

// Hadamard: table[(xi*T + t)*nchunk + chunk] = exact max |I| over the row chunk (written by the GEMM
// max epilogue).  Entries equal to the group maximum are recomputed on CUDA cores (lane per column)
// and their maxima replayed in fp64.
template <int kInTU = 0>  // header-defined kernel: instantiated only in the TUs that launch it
__global__ void __launch_bounds__(256) finalize_hadamard_kernel(const int8_t* __restrict__ U, const int8_t* __restrict__ V, Geo g,
                                         Acc* __restrict__ acc, const Acc* __restrict__ wacc, int wstage, int qmax_u,
                                         int qmax_v, const unsigned* __restrict__ table, int bn, ParamsTail tail) {
  // Flat, fully parallel scan: thread per (xi, t) table row (nchunk <= 4 entries, one 16-byte load
  // when nchunk == 4); consecutive threads read consecutive rows.  An entry equal to its group's exact
  // max is recomputed by the whole warp (rare): lanes over the entry's output columns.
  __shared__ double prod[8][512];  // per-warp products of one replayed column (C <= 512)
  const int nchunk = g.Kp / bn;
  const int lane = threadIdx.x & 31;
  // 36 * T < 2^27 (make_layout rejects larger calls): 32-bit row arithmetic, no 64-bit divisions
  const unsigned T = (unsigned)g.T;
  const unsigned rows = 36u * T;
  const unsigned nthr = gridDim.x * blockDim.x;
  const bool tmajor = g.TP * g.ipg < 32;
  for (unsigned r0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; r0 < rows; r0 += nthr) {
    const unsigned rr = r0 + lane;
    const bool valid = rr < rows;
    // Lane -> table row.  Large groups: consecutive lanes are consecutive tiles of one xi (coalesced table
    // reads; a warp meets at most two groups).  Groups of fewer than 32 tiles (small images): the argmax of
    // every group tends to sit at the same xi, so that mapping would hand 32 groups' fp64 replays to one warp
    // one after the other (measured 0.99 ms on 256 images of 512 x 4 x 4); there lanes run over the 36 xi of
    // consecutive tiles, i.e. at most two groups per warp again.
    unsigned xi, t;
    if (tmajor) {
      t = valid ? rr / 36u : 0u;
      xi = valid ? rr - 36u * t : 0u;
    } else {
      xi = valid ? rr / T : 0u;
      t = valid ? rr - xi * T : 0u;
    }
    const unsigned r = xi * T + t;  // table row
    const int grp = (int)g.fipg.div(g.fTP.div(t));
    const unsigned long long M = valid ? acc[(size_t)grp * ST_COUNT + ST_HAD].M : 0ull;
    unsigned v[4] = {0u, 0u, 0u, 0u};
    if (valid) {
      if (nchunk == 4) {
        const uint4 q = *reinterpret_cast<const uint4*>(table + (size_t)r * 4);
        v[0] = q.x, v[1] = q.y, v[2] = q.z, v[3] = q.w;
      } else {
        for (int c = 0; c < nchunk && c < 4; ++c) v[c] = table[(size_t)r * nchunk + c];
      }
    }
    // entries never exceed the group maximum: one vote on the row maximum skips the chunk loop for almost
    // every warp (rows with more than 4 chunks always take it)
    const unsigned vmax = max(max(v[0], v[1]), max(v[2], v[3]));
    if (nchunk <= 4 && !__any_sync(0xffffffffu, valid && vmax != 0 && (unsigned long long)vmax == M)) continue;
    for (int chunk = 0; chunk < nchunk; ++chunk) {
      const unsigned v4 = chunk == 0 ? v[0] : chunk == 1 ? v[1] : chunk == 2 ? v[2] : v[3];
      const unsigned vc = chunk < 4 ? v4 : (valid ? table[(size_t)r * nchunk + chunk] : 0u);
      unsigned mask = __ballot_sync(0xffffffffu, valid && vc != 0 && (unsigned long long)vc == M);
      while (mask) {
        const int l = __ffs(mask) - 1;
        mask &= mask - 1;
        const int tl = (int)__shfl_sync(0xffffffffu, t, l);
        const int xl = (int)__shfl_sync(0xffffffffu, xi, l);
        const int gl = __shfl_sync(0xffffffffu, grp, l);
        Acc* ga = acc + (size_t)gl * ST_COUNT;
        const long long Ml = (long long)ga[ST_HAD].M;
        const int8_t* vrow = V + ((size_t)tl * 36 + xl) * g.Cp;
        double f = 0.0;
        const int kend = min(chunk * bn + bn, g.K);
        for (int kb = chunk * bn; kb < kend; kb += 32) {
          const int k = kb + lane;
          long long sdot = 0;
          if (k < kend) {
            const int8_t* urow = U + ((size_t)k * 36 + xl) * g.Cp;
            // exact integer dot over the zero-padded Cp channels: 16-byte loads, 4-way byte dot products
            // (|sum| <= 127 * 255 * 512 < 2^31; channels >= C are zero in U and V)
            const int4* u4 = reinterpret_cast<const int4*>(urow);
            const int4* v4 = reinterpret_cast<const int4*>(vrow);
            int s0 = 0, s1 = 0;
            for (int c = 0; c < g.Cp / 16; ++c) {
              const int4 a = __ldg(u4 + c), bb = __ldg(v4 + c);
              s0 = __dp4a(a.x, bb.x, s0);
              s1 = __dp4a(a.y, bb.y, s1);
              s0 = __dp4a(a.z, bb.z, s0);
              s1 = __dp4a(a.w, bb.w, s1);
            }
            sdot = (long long)s0 + s1;
          }
          // fp64 replay of an argmax column by the whole warp: the 32 lanes form the products
          // deq(u_c) * deq(v_c), one lane adds them c ascending from 0.0 (_kernels.py:99-104) — the same
          // roundings as replay_hadamard, with C dependent adds on the critical path instead of C times
          // (two byte loads, two dequantisations, a multiply and an add) on a single lane
          unsigned hit = __ballot_sync(0xffffffffu, k < kend && (sdot < 0 ? -sdot : sdot) == Ml);
          if (hit) {
            const StageQ qu = load_int_stage(wacc[wstage], qmax_u), qv = load_int_stage(ga[ST_IT], qmax_v);
            double* pw = prod[threadIdx.x >> 5];
            while (hit) {
              const int src = __ffs(hit) - 1;
              hit &= hit - 1;
              const int8_t* us = U + ((size_t)(kb + src) * 36 + xl) * g.Cp;
              for (int c = lane; c < g.C; c += 32)
                pw[c] = __dmul_rn(deq(us[c], qu.qmax, qu.maxabs, qu.scale), deq(vrow[c], qv.qmax, qv.maxabs, qv.scale));
              __syncwarp();
              if (lane == 0) {
                double a = 0.0;
                for (int c = 0; c < g.C; ++c) a = __dadd_rn(a, pw[c]);
                f = fmax(f, fabs(a));
              }
              __syncwarp();
            }
          }
        }
        if (f > 0.0) atomicMax(&ga[ST_HAD].F, dbits(f));
      }
    }
  }
  stage_params_tail(acc, ST_HAD, tail);
}

// ---------------------------------------------------------------------------------- fixup kernels
// One deferred unit per thread; the list length is read on the device (no host round trip).

// Legendre input_base_change: exact c1 codes, then the unit's input_transform maximum.
template <int kInTU = 0>  // header-defined kernel: instantiated only in the TUs that launch it
__global__ void __launch_bounds__(128) fixup_ibc_kernel(FixList fl, const int8_t* __restrict__ c0,
                                                        int8_t* __restrict__ c1, Geo g, Bits b, Acc* __restrict__ acc,
                                                        const PlanF64* __restrict__ pf, Tables tabs) {
  const unsigned cnt = fix_count(fl, FIX_IBC);
  const uint32_t plane = (uint32_t)g.Cp;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
    const unsigned u = fl.items[i];
    const int c = (int)g.fC.mod(u), t = (int)g.fC.div(u);
    const int n = (int)g.fTP.div((unsigned)t), tile = (int)g.fTP.mod((unsigned)t), grp = (int)g.fipg.div((unsigned)n);
    const Acc* ga = acc + (size_t)grp * ST_COUNT;
    const float r = ga[ST_IBC].r, thr = ga[ST_IBC].thr, ef = ga[ST_IBC].ef;
    int8_t* dst = c1 + ((size_t)t * 36 * plane + c);
    const C0Win win(c0, g, n, tile, c, plane);
    fix_unit<tab::Leg_IBC>(SrcC0{win}, r, thr, ef, ga + ST_IBC, b.q[ST_IBC], ga + ST_INPUT, b.q[ST_INPUT], true,
                           pf->ibc, [dst, plane](int ii, int jj, int code) { dst[(6 * ii + jj) * plane] = (int8_t)code; });
    float K1[6][6];
#pragma unroll
    for (int e = 0; e < 36; ++e) K1[e / 6][e % 6] = (float)dst[e * plane];
    float m = 0.f, tm = 0.f;
    sandwich_cols<tab::Leg_IT>(K1, [&](int, const float (&col)[6]) {
#pragma unroll
      for (int q = 0; q < 6; ++q) m = fmaxf(m, fabsf(col[q]));
    }, &tm);
    record_unit_single(m, tm, grp, acc, ST_IT, tabs.t[ST_IT], t, c, g.C);
  }
}

template <int MODE>
__global__ void __launch_bounds__(128) fixup_it_kernel(FixList fl, const int8_t* __restrict__ c0,
                                                       const int8_t* __restrict__ c1, int8_t* __restrict__ V, const __grid_constant__ Geo g,
                                                       const __grid_constant__ Bits b, const Acc* __restrict__ acc,
                                                       const PlanF64* __restrict__ pf) {
  const unsigned cnt = fix_count(fl, FIX_IT);
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
    const unsigned u = fl.items[i];
    const int t = (int)g.fC.div(u), c = (int)g.fC.mod(u);
    fix_it_unit<MODE>(c0, c1, V + ((size_t)t * 36 * g.Cp + c), (uint32_t)g.Cp, g, b, acc, pf, t, c, (uint32_t)g.Cp);
  }
}

// Legendre output_base_change: exact c4 codes, then the unit's (cropped) output maximum.
template <typename HT>
__global__ void __launch_bounds__(128) fixup_obc_kernel(FixList fl, const HT* __restrict__ h, int8_t* __restrict__ c4,
                                                        Geo g, Bits b, Acc* __restrict__ acc,
                                                        const PlanF64* __restrict__ pf, Tables tabs) {
  const unsigned cnt = fix_count(fl, FIX_OBC);
  const uint32_t plane = (uint32_t)g.Kp;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
    const unsigned u = fl.items[i];
    const int k = (int)g.fK.mod(u), t = (int)g.fK.div(u);
    const int n = (int)g.fTP.div((unsigned)t), tile = (int)g.fTP.mod((unsigned)t), grp = (int)g.fipg.div((unsigned)n);
    const int ty = (int)g.ftw.div((unsigned)tile), tx = (int)g.ftw.mod((unsigned)tile);
    const Acc* ga = acc + (size_t)grp * ST_COUNT;
    const float r = ga[ST_OBC].r, thr = ga[ST_OBC].thr, ef = ga[ST_OBC].ef;
    const uint32_t off = (uint32_t)t * 36u * plane + (uint32_t)k;
    int8_t* dst = c4 + off;
    fix_unit<tab::Leg_OBC>(SrcPlanes<HT>{h, plane, off}, r, thr, ef, ga + ST_OBC, b.q[ST_OBC], ga + ST_HAD,
                           b.q[ST_HAD], false, pf->obc,
                           [dst, plane](int ii, int jj, int code) { dst[(6 * ii + jj) * plane] = (int8_t)code; });
    float K4[6][6];
#pragma unroll
    for (int e = 0; e < 36; ++e) K4[e / 6][e % 6] = (float)dst[e * plane];
    float m = 0.f, tm = 0.f;
    sandwich_cols<tab::Leg_OT>(K4, [&](int j, const float (&col)[4]) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (4 * ty + q < g.Ho && 4 * tx + j < g.Wo) m = fmaxf(m, fabsf(col[q]));
    }, &tm);
    record_unit_single(m, tm, grp, acc, ST_OUT, tabs.t[ST_OUT], t, k, g.K);
  }
}

template <int MODE, typename HT, typename YT>
__global__ void __launch_bounds__(128) fixup_out_kernel(FixList fl, const HT* __restrict__ h,
                                                        const int8_t* __restrict__ c4, YT* __restrict__ y,
                                                        const YT* __restrict__ bias, const __grid_constant__ Geo g, const __grid_constant__ Bits b,
                                                        const Acc* __restrict__ acc, const PlanF64* __restrict__ pf) {
  const unsigned cnt = fix_count(fl, FIX_OUT);
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
    const unsigned u = fl.items[i];
    fix_out_unit<MODE, HT, YT>(h, c4, y, bias, g, b, acc, pf, (int)g.fK.div(u), (int)g.fK.mod(u),
                               (uint32_t)g.Kp);
  }
}

}  // namespace wl
