// v2 transform kernels: fp32 fast path with certified error bounds, exact integer fallback,
// deferred fp64 argmax replay through per-entry max tables.
//
// Every stage value T is an integer.  The fast path evaluates T in fp32: the
// first sandwich half is exact and the second rounds once per fma, so |T_f - T| <= E_stage
// (host-computed, see wl_forward.cu).  Hence
//   * codes: x = T_f * qmax/M rounded half-even by a magic-number add is the exact rhe() result
//     unless x is within qmax*E/M (+ fp32 slack) of a half-integer; such tile-channels are redone
//     with integer arithmetic and exact tie replay (requant36);
//   * maxima: only units whose fp32 maximum is within 2E of the running group maximum can hold the
//     exact argmax; they are pushed to a candidate list that finalize_* recomputes exactly
//     (integer M, fp64 max_abs by replay in the reference's operation order).
// Thread mapping: one (tile, channel) unit per thread, channel fastest, so every byte-plane access
// of a warp is one contiguous 32-byte segment.
#pragma once
#include "wl_kernels.cuh"

namespace wl {

struct Tables {  // max tables per stage id (only IBC, IT, HAD, OBC, OUT are used)
  unsigned* t[ST_COUNT];
};

struct StageE {  // certified fp32 error bound per stage (integer units)
  float e[ST_COUNT];
};

__device__ __forceinline__ void load_c0_f(const int8_t* __restrict__ c0, const Geo& g, int n, int tile, int c,
                                          float (&X)[6][6]) {
  const int ty = tile / g.tw, tx = tile % g.tw;
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    const int r = 4 * ty + i - g.pad;
#pragma unroll
    for (int j = 0; j < 6; ++j) {
      const int col = 4 * tx + j - g.pad;
      X[i][j] = (r >= 0 && r < g.H && col >= 0 && col < g.W)
                    ? (float)__ldg(&c0[(((size_t)n * g.H + r) * g.W + col) * g.Cp + c])
                    : 0.f;
    }
  }
}

// 36 codes of one unit from a [36][rows][ld] plane layout.
template <typename HT, typename XT>
__device__ __forceinline__ void load_planes(const HT* __restrict__ P, size_t plane, size_t off, XT (&X)[6][6]) {
#pragma unroll
  for (int e = 0; e < 36; ++e) X[e / 6][e % 6] = (XT)__ldg(&P[(size_t)e * plane + off]);
}

template <int R>
__device__ __forceinline__ float absmax_f(const float (&T)[R][R]) {
  float m = 0.f;
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < R; ++j) m = fmaxf(m, fabsf(T[i][j]));
  return m;
}

// Max of one (unit row t, channel c) into table entry t*ceil(C/32) + c/32 and the group running max.
__device__ __forceinline__ void record_unit(float m, int grp, bool active, Acc* acc, int stage, unsigned* table,
                                            int t, int c, int C) {
  bool uniform;
  float wmax;
  const int CB = (C + 31) >> 5;
  record_max(active ? m : 0.f, active ? grp : -1, table + (size_t)t * CB + (c >> 5), (C & 31) == 0, acc + stage,
             uniform, wmax);
  publish_mf(active ? m : 0.f, active ? grp : -1, acc + stage, uniform, wmax);
}

// ---------------------------------------------------------------------------------- exact fallbacks
// Out of line so the fast path keeps a small register footprint; results go through local memory.

// Legendre input_base_change codes of one unit from c0 (exact, ties replayed).
__device__ __noinline__ void exact_c1_unit(const int8_t* __restrict__ c0, const Geo g, int n, int tile, int c,
                                           const Acc* ga, const Bits b, const PlanF64* pf, int* out) {
  int Xi[6][6], T1[6][6], C1[6][6];
  load_input_tile(c0, g, n, tile, c, Xi);
  sandwich<tab::Leg_IBC>(Xi, T1);
  requant36(T1, load_int_stage(ga[ST_IBC], b.q[ST_IBC]), Xi, load_float_stage(ga[ST_INPUT], b.q[ST_INPUT]), pf->ibc,
            C1);
  for (int e = 0; e < 36; ++e) out[e] = C1[e / 6][e % 6];
}

// V codes of one unit (canonical from c0, Legendre from c1), exact with tie replay.
template <int MODE>
__device__ __noinline__ void exact_v_unit(const int8_t* __restrict__ c0, const int8_t* __restrict__ c1, const Geo g,
                                          int t, int c, const Acc* ga, const Bits b, const PlanF64* pf, int* out) {
  const int n = t / g.TP, tile = t % g.TP;
  int Xi[6][6], Cv[6][6];
  if constexpr (MODE == 0) {
    int Ti[6][6];
    load_input_tile(c0, g, n, tile, c, Xi);
    sandwich<tab::Can_IT>(Xi, Ti);
    requant36(Ti, load_int_stage(ga[ST_IT], b.q[ST_IT]), Xi, load_float_stage(ga[ST_INPUT], b.q[ST_INPUT]), pf->it,
              Cv);
  } else {
    long long Ti[6][6];
#pragma unroll
    for (int e = 0; e < 36; ++e) Xi[e / 6][e % 6] = c1[((size_t)e * g.T + t) * g.Cp + c];
    sandwich<tab::Leg_IT>(Xi, Ti);
    requant36(Ti, load_int_stage(ga[ST_IT], b.q[ST_IT]), Xi, load_int_stage(ga[ST_IBC], b.q[ST_IBC]), pf->it, Cv);
  }
  for (int e = 0; e < 36; ++e) out[e] = Cv[e / 6][e % 6];
}

// Legendre output_base_change codes of one (t, k) unit from h.
template <typename HT>
__device__ __noinline__ void exact_c4_unit(const HT* __restrict__ h, const Geo g, int t, int k, const Acc* ga,
                                           const Bits b, const PlanF64* pf, int* out) {
  int Hi[6][6], Ti[6][6], C4[6][6];
#pragma unroll
  for (int e = 0; e < 36; ++e) Hi[e / 6][e % 6] = h[((size_t)e * g.T + t) * g.Kp + k];
  sandwich<tab::Leg_OBC>(Hi, Ti);
  requant36(Ti, load_int_stage(ga[ST_OBC], b.q[ST_OBC]), Hi, load_int_stage(ga[ST_HAD], b.q[ST_HAD]), pf->obc, C4);
  for (int e = 0; e < 36; ++e) out[e] = C4[e / 6][e % 6];
}

// Output-stage codes of one (t, k) unit (canonical from h, Legendre from c4).
template <int MODE, typename HT>
__device__ __noinline__ void exact_out_unit(const HT* __restrict__ h, const int8_t* __restrict__ c4, const Geo g,
                                            int t, int k, const Acc* ga, const Bits b, const PlanF64* pf, int* out) {
  int Xi[6][6];
  long long Yi[4][4];
  StageQ qf;
  if constexpr (MODE == 0) {
#pragma unroll
    for (int e = 0; e < 36; ++e) Xi[e / 6][e % 6] = h[((size_t)e * g.T + t) * g.Kp + k];
    int Y32[4][4];
    sandwich<tab::Can_OT>(Xi, Y32);
#pragma unroll
    for (int e = 0; e < 16; ++e) Yi[e / 4][e % 4] = Y32[e / 4][e % 4];
    qf = load_int_stage(ga[ST_HAD], b.q[ST_HAD]);
  } else {
#pragma unroll
    for (int e = 0; e < 36; ++e) Xi[e / 6][e % 6] = c4[((size_t)e * g.T + t) * g.Kp + k];
    sandwich<tab::Leg_OT>(Xi, Yi);
    qf = load_int_stage(ga[ST_OBC], b.q[ST_OBC]);
  }
  const StageQ qo = load_int_stage(ga[ST_OUT], b.q[ST_OUT]);
  int xc[36];
  for (int e = 0; e < 36; ++e) xc[e] = Xi[e / 6][e % 6];
  for (int e = 0; e < 16; ++e) {
    bool tie = false;
    int code = rq(Yi[e / 4][e % 4], qo, tie);
    if (tie) code = code_of(replay_sandwich(pf->ot, 4, 6, xc, qf.qmax, qf.maxabs, qf.scale, e / 4, e % 4), qo);
    out[e] = code;
  }
}

// ---------------------------------------------------------------------------------- input side

// First input stage maximum: canonical input_transform (B^T), Legendre input_base_change (P^-T).
template <int MODE>
__global__ void __launch_bounds__(256) in_a_kernel(const int8_t* __restrict__ c0, Geo g, Acc* __restrict__ acc,
                                                   Tables tabs) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const bool active = idx < (long long)g.T * g.C;
  const long long id = active ? idx : 0;
  const int c = (int)(id % g.C), t = (int)(id / g.C);
  const int n = t / g.TP, tile = t % g.TP;
  const int grp = n / g.ipg;
  float X[6][6], T[6][6];
  load_c0_f(c0, g, n, tile, c, X);
  constexpr int st = MODE == 0 ? ST_IT : ST_IBC;
  if constexpr (MODE == 0)
    sandwich_f<tab::Can_IT>(X, T);
  else
    sandwich_f<tab::Leg_IBC>(X, T);
  record_unit(absmax_f(T), grp, active, acc, st, tabs.t[st], t, c, g.C);
}

// Legendre: input_base_change codes c1 (stored) and input_transform maximum.
__global__ void __launch_bounds__(256) in_b_kernel(const int8_t* __restrict__ c0, int8_t* __restrict__ c1, Geo g,
                                                   Bits b, Acc* __restrict__ acc, const PlanF64* __restrict__ pf,
                                                   Tables tabs, StageE E) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const bool active = idx < (long long)g.T * g.C;
  const long long id = active ? idx : 0;
  const int c = (int)(id % g.C), t = (int)(id / g.C);
  const int n = t / g.TP, tile = t % g.TP;
  const int grp = n / g.ipg;
  const Acc* ga = acc + (size_t)grp * ST_COUNT;
  float X[6][6], T[6][6];
  load_c0_f(c0, g, n, tile, c, X);
  sandwich_f<tab::Leg_IBC>(X, T);
  const StageF s1 = load_stage_f(ga[ST_IBC], b.q[ST_IBC], E.e[ST_IBC]);
  int C1[6][6];
  float dmax = 0.f;
#pragma unroll
  for (int e = 0; e < 36; ++e) C1[e / 6][e % 6] = rq_fast(T[e / 6][e % 6], s1, dmax);
  if (dmax > 0.5f - s1.band) {  // exact path for this unit
    int tmp[36];
    exact_c1_unit(c0, g, n, tile, c, ga, b, pf, tmp);
#pragma unroll
    for (int e = 0; e < 36; ++e) C1[e / 6][e % 6] = tmp[e];
  }
  if (active)
#pragma unroll
    for (int e = 0; e < 36; ++e) c1[((size_t)e * g.T + t) * g.Cp + c] = (int8_t)C1[e / 6][e % 6];
  float Xf[6][6], T2[6][6];
#pragma unroll
  for (int e = 0; e < 36; ++e) Xf[e / 6][e % 6] = (float)C1[e / 6][e % 6];
  sandwich_f<tab::Leg_IT>(Xf, T2);
  record_unit(absmax_f(T2), grp, active, acc, ST_IT, tabs.t[ST_IT], t, c, g.C);
}

// V codes.  Canonical: from c0 through B^T.  Legendre: from the stored c1 through B_P^T.
template <int MODE>
__global__ void __launch_bounds__(256) in_c_kernel(const int8_t* __restrict__ c0, const int8_t* __restrict__ c1,
                                                   int8_t* __restrict__ V, Geo g, Bits b, Acc* __restrict__ acc,
                                                   const PlanF64* __restrict__ pf, StageE E) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)g.T * g.C) return;
  const int c = (int)(idx % g.C), t = (int)(idx / g.C);
  const int n = t / g.TP, tile = t % g.TP;
  const int grp = n / g.ipg;
  const Acc* ga = acc + (size_t)grp * ST_COUNT;
  float X[6][6], T[6][6];
  if constexpr (MODE == 0) {
    load_c0_f(c0, g, n, tile, c, X);
    sandwich_f<tab::Can_IT>(X, T);
  } else {
    load_planes(c1, (size_t)g.T * g.Cp, (size_t)t * g.Cp + c, X);
    sandwich_f<tab::Leg_IT>(X, T);
  }
  const StageF s = load_stage_f(ga[ST_IT], b.q[ST_IT], E.e[ST_IT]);
  int Cv[6][6];
  float dmax = 0.f;
#pragma unroll
  for (int e = 0; e < 36; ++e) Cv[e / 6][e % 6] = rq_fast(T[e / 6][e % 6], s, dmax);
  if (dmax > 0.5f - s.band) {
    int tmp[36];
    exact_v_unit<MODE>(c0, c1, g, t, c, ga, b, pf, tmp);
#pragma unroll
    for (int e = 0; e < 36; ++e) Cv[e / 6][e % 6] = tmp[e];
  }
#pragma unroll
  for (int e = 0; e < 36; ++e) V[((size_t)e * g.T + t) * g.Cp + c] = (int8_t)Cv[e / 6][e % 6];
}

// Exact recomputation of one input-side unit: local exact max and fp64 max_abs of its argmax.
template <int MODE, int STAGE>
__device__ void exact_input_unit(const int8_t* __restrict__ c0, const int8_t* __restrict__ c1, const Geo& g,
                                 const Bits& b, Acc* acc, const PlanF64* pf, int t, int c) {
  const int n = t / g.TP, tile = t % g.TP;
  const int grp = n / g.ipg;
  Acc* ga = acc + (size_t)grp * ST_COUNT;
  int Xi[6][6];
  long long T[6][6];
  StageQ qin;
  const double* Lf;
  if (MODE == 1 && STAGE == ST_IT) {
    load_planes(c1, (size_t)g.T * g.Cp, (size_t)t * g.Cp + c, Xi);
    sandwich<tab::Leg_IT>(Xi, T);
    qin = load_int_stage(ga[ST_IBC], b.q[ST_IBC]);
    Lf = pf->it;
  } else {
    load_input_tile(c0, g, n, tile, c, Xi);
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
  const long long m = absmax36(T);
  if (m == 0) return;
  int xc[36];
  for (int e = 0; e < 36; ++e) xc[e] = Xi[e / 6][e % 6];
  double f = 0.0;
  for (int e = 0; e < 36; ++e) {
    const long long v = T[e / 6][e % 6];
    if ((v < 0 ? -v : v) == m) f = fmax(f, fabs(replay_sandwich(Lf, 6, 6, xc, qin.qmax, qin.maxabs, qin.scale, e / 6, e % 6)));
  }
  atomicMax(&ga[STAGE].M, (unsigned long long)m);
  atomicMax(&ga[STAGE].F, dbits(f));
}

// Scan a stage's max table; warps recompute exactly the entries within 2E of the group's fp32 max.
template <int MODE, int STAGE>
__global__ void finalize_input_kernel(const int8_t* __restrict__ c0, const int8_t* __restrict__ c1, Geo g, Bits b,
                                      Acc* __restrict__ acc, const PlanF64* __restrict__ pf,
                                      const unsigned* __restrict__ table, float E) {
  const int CB = (g.C + 31) >> 5;
  const long long nent = (long long)g.T * CB;
  const int lane = threadIdx.x & 31;
  const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long base = wid * 32; base < nent; base += nw * 32) {
    const long long e = base + lane;
    bool pass = false;
    if (e < nent) {
      const float v = __uint_as_float(table[e]);
      const int t = (int)(e / CB);
      const int grp = (t / g.TP) / g.ipg;
      const float mf = __uint_as_float(acc[(size_t)grp * ST_COUNT + STAGE].MF);
      pass = v > 0.f && v >= mf - 2.f * E;
    }
    unsigned mask = __ballot_sync(0xffffffffu, pass);
    while (mask) {
      const int l = __ffs(mask) - 1;
      mask &= mask - 1;
      const long long ee = base + l;
      const int t = (int)(ee / CB), c = (int)(ee % CB) * 32 + lane;
      if (c < g.C) exact_input_unit<MODE, STAGE>(c0, c1, g, b, acc, pf, t, c);
    }
  }
}

// ---------------------------------------------------------------------------------- output side

// Thread per (tile t, out channel k), k fastest.
// OUT_A: Legendre output_base_change max (P^-T on h) | canonical output max (A^T on h, cropped).
template <int MODE, typename HT>
__global__ void __launch_bounds__(256) out_a_kernel(const HT* __restrict__ h, Geo g, Acc* __restrict__ acc,
                                                    Tables tabs) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const bool active = idx < (long long)g.T * g.K;
  const long long id = active ? idx : 0;
  const int k = (int)(id % g.K), t = (int)(id / g.K);
  const int n = t / g.TP, tile = t % g.TP;
  const int grp = n / g.ipg;
  float X[6][6];
  load_planes(h, (size_t)g.T * g.Kp, (size_t)t * g.Kp + k, X);
  float m;
  constexpr int st = MODE == 0 ? ST_OUT : ST_OBC;
  if constexpr (MODE == 0) {
    float Y[4][4];
    sandwich_f<tab::Can_OT>(X, Y);
    const int ty = tile / g.tw, tx = tile % g.tw;
    m = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (4 * ty + i < g.Ho && 4 * tx + j < g.Wo) m = fmaxf(m, fabsf(Y[i][j]));
  } else {
    float T[6][6];
    sandwich_f<tab::Leg_OBC>(X, T);
    m = absmax_f(T);
  }
  record_unit(m, grp, active, acc, st, tabs.t[st], t, k, g.K);
}

// Legendre: output_base_change codes c4 (stored) and cropped output maximum.
template <typename HT>
__global__ void __launch_bounds__(256) out_b_kernel(const HT* __restrict__ h, int8_t* __restrict__ c4, Geo g, Bits b,
                                                    Acc* __restrict__ acc, const PlanF64* __restrict__ pf, Tables tabs,
                                                    StageE E) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const bool active = idx < (long long)g.T * g.K;
  const long long id = active ? idx : 0;
  const int k = (int)(id % g.K), t = (int)(id / g.K);
  const int n = t / g.TP, tile = t % g.TP;
  const int grp = n / g.ipg;
  const Acc* ga = acc + (size_t)grp * ST_COUNT;
  float X[6][6], T[6][6];
  load_planes(h, (size_t)g.T * g.Kp, (size_t)t * g.Kp + k, X);
  sandwich_f<tab::Leg_OBC>(X, T);
  const StageF s4 = load_stage_f(ga[ST_OBC], b.q[ST_OBC], E.e[ST_OBC]);
  int C4[6][6];
  float dmax = 0.f;
#pragma unroll
  for (int e = 0; e < 36; ++e) C4[e / 6][e % 6] = rq_fast(T[e / 6][e % 6], s4, dmax);
  if (dmax > 0.5f - s4.band) {
    int tmp[36];
    exact_c4_unit(h, g, t, k, ga, b, pf, tmp);
#pragma unroll
    for (int e = 0; e < 36; ++e) C4[e / 6][e % 6] = tmp[e];
  }
  if (active)
#pragma unroll
    for (int e = 0; e < 36; ++e) c4[((size_t)e * g.T + t) * g.Kp + k] = (int8_t)C4[e / 6][e % 6];
  float Xf[6][6], Y[4][4];
#pragma unroll
  for (int e = 0; e < 36; ++e) Xf[e / 6][e % 6] = (float)C4[e / 6][e % 6];
  sandwich_f<tab::Leg_OT>(Xf, Y);
  const int ty = tile / g.tw, tx = tile % g.tw;
  float m = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (4 * ty + i < g.Ho && 4 * tx + j < g.Wo) m = fmaxf(m, fabsf(Y[i][j]));
  record_unit(m, grp, active, acc, ST_OUT, tabs.t[ST_OUT], t, k, g.K);
}

// Final output: codes of the output stage, dequantised (snap +-qmax to +-max_abs), + bias, fp32 NCHW.
template <int MODE, typename HT>
__global__ void __launch_bounds__(256) out_c_kernel(const HT* __restrict__ h, const int8_t* __restrict__ c4,
                                                    float* __restrict__ y, const float* __restrict__ bias, Geo g,
                                                    Bits b, Acc* __restrict__ acc, const PlanF64* __restrict__ pf,
                                                    StageE E) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)g.T * g.K) return;
  const int k = (int)(idx % g.K), t = (int)(idx / g.K);
  const int n = t / g.TP, tile = t % g.TP;
  const int ty = tile / g.tw, tx = tile % g.tw;
  const int grp = n / g.ipg;
  const Acc* ga = acc + (size_t)grp * ST_COUNT;
  float X[6][6], Y[4][4];
  if constexpr (MODE == 0) {
    load_planes(h, (size_t)g.T * g.Kp, (size_t)t * g.Kp + k, X);
    sandwich_f<tab::Can_OT>(X, Y);
  } else {
    load_planes(c4, (size_t)g.T * g.Kp, (size_t)t * g.Kp + k, X);
    sandwich_f<tab::Leg_OT>(X, Y);
  }
  const StageF s = load_stage_f(ga[ST_OUT], b.q[ST_OUT], E.e[ST_OUT]);
  int Co[4][4];
  float dmax = 0.f;
#pragma unroll
  for (int e = 0; e < 16; ++e) Co[e / 4][e % 4] = rq_fast(Y[e / 4][e % 4], s, dmax);
  const StageQ qo = load_int_stage(ga[ST_OUT], b.q[ST_OUT]);
  if (dmax > 0.5f - s.band) {
    int tmp[16];
    exact_out_unit<MODE, HT>(h, c4, g, t, k, ga, b, pf, tmp);
#pragma unroll
    for (int e = 0; e < 16; ++e) Co[e / 4][e % 4] = tmp[e];
  }
  const float bk = bias ? __ldg(&bias[k]) : 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = 4 * ty + i;
    if (r >= g.Ho) continue;
    float* row = y + (((size_t)n * g.K + k) * g.Ho + r) * g.Wo + 4 * tx;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (4 * tx + j >= g.Wo) continue;
      float out = (float)deq(Co[i][j], qo.qmax, qo.maxabs, qo.scale);
      if (bias) out += bk;
      row[j] = out;
    }
  }
}

template <int MODE, int STAGE, typename HT>
__device__ void exact_output_unit(const HT* __restrict__ h, const int8_t* __restrict__ c4, const Geo& g, const Bits& b,
                                  Acc* acc, const PlanF64* pf, int t, int k) {
  const int n = t / g.TP, tile = t % g.TP;
  const int ty = tile / g.tw, tx = tile % g.tw;
  const int grp = n / g.ipg;
  Acc* ga = acc + (size_t)grp * ST_COUNT;
  int Xi[6][6];
  if (MODE == 1 && STAGE == ST_OBC) {
    load_planes(h, (size_t)g.T * g.Kp, (size_t)t * g.Kp + k, Xi);
    int T[6][6];
    sandwich<tab::Leg_OBC>(Xi, T);
    const long long m = absmax36(T);
    if (m == 0) return;
    const StageQ qin = load_int_stage(ga[ST_HAD], b.q[ST_HAD]);
    int xc[36];
    for (int e = 0; e < 36; ++e) xc[e] = Xi[e / 6][e % 6];
    double f = 0.0;
    for (int e = 0; e < 36; ++e) {
      const long long v = T[e / 6][e % 6];
      if ((v < 0 ? -v : v) == m) f = fmax(f, fabs(replay_sandwich(pf->obc, 6, 6, xc, qin.qmax, qin.maxabs, qin.scale, e / 6, e % 6)));
    }
    atomicMax(&ga[ST_OBC].M, (unsigned long long)m);
    atomicMax(&ga[ST_OBC].F, dbits(f));
    return;
  }
  // output stage (cropped)
  long long Y[4][4];
  StageQ qin;
  if (MODE == 0) {
    load_planes(h, (size_t)g.T * g.Kp, (size_t)t * g.Kp + k, Xi);
    int Y32[4][4];
    sandwich<tab::Can_OT>(Xi, Y32);
    for (int e = 0; e < 16; ++e) Y[e / 4][e % 4] = Y32[e / 4][e % 4];
    qin = load_int_stage(ga[ST_HAD], b.q[ST_HAD]);
  } else {
    load_planes(c4, (size_t)g.T * g.Kp, (size_t)t * g.Kp + k, Xi);
    sandwich<tab::Leg_OT>(Xi, Y);
    qin = load_int_stage(ga[ST_OBC], b.q[ST_OBC]);
  }
  const long long m = absmax_crop(Y, ty, tx, g);
  if (m == 0) return;
  int xc[36];
  for (int e = 0; e < 36; ++e) xc[e] = Xi[e / 6][e % 6];
  double f = 0.0;
  for (int e = 0; e < 16; ++e) {
    const int i = e / 4, j = e % 4;
    if (4 * ty + i >= g.Ho || 4 * tx + j >= g.Wo) continue;
    const long long v = Y[i][j];
    if ((v < 0 ? -v : v) == m) f = fmax(f, fabs(replay_sandwich(pf->ot, 4, 6, xc, qin.qmax, qin.maxabs, qin.scale, i, j)));
  }
  atomicMax(&ga[ST_OUT].M, (unsigned long long)m);
  atomicMax(&ga[ST_OUT].F, dbits(f));
}

template <int MODE, int STAGE, typename HT>
__global__ void finalize_output_kernel(const HT* __restrict__ h, const int8_t* __restrict__ c4, Geo g, Bits b,
                                       Acc* __restrict__ acc, const PlanF64* __restrict__ pf,
                                       const unsigned* __restrict__ table, float E) {
  const int KB = (g.K + 31) >> 5;
  const long long nent = (long long)g.T * KB;
  const int lane = threadIdx.x & 31;
  const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long base = wid * 32; base < nent; base += nw * 32) {
    const long long e = base + lane;
    bool pass = false;
    if (e < nent) {
      const float v = __uint_as_float(table[e]);
      const int t = (int)(e / KB);
      const int grp = (t / g.TP) / g.ipg;
      const float mf = __uint_as_float(acc[(size_t)grp * ST_COUNT + STAGE].MF);
      pass = v > 0.f && v >= mf - 2.f * E;
    }
    unsigned mask = __ballot_sync(0xffffffffu, pass);
    while (mask) {
      const int l = __ffs(mask) - 1;
      mask &= mask - 1;
      const long long ee = base + l;
      const int t = (int)(ee / KB), k = (int)(ee % KB) * 32 + lane;
      if (k < g.K) exact_output_unit<MODE, STAGE, HT>(h, c4, g, b, acc, pf, t, k);
    }
  }
}

// Hadamard: table[(xi*T + t)*nchunk + chunk] = exact max |I| over the row chunk (written by the GEMM
// max epilogue).  Entries equal to the group maximum are recomputed on CUDA cores (lane per column)
// and their maxima replayed in fp64.
__global__ void finalize_hadamard_kernel(const int8_t* __restrict__ U, const int8_t* __restrict__ V, Geo g,
                                         Acc* __restrict__ acc, const Acc* __restrict__ wacc, int wstage, int qmax_u,
                                         int qmax_v, const unsigned* __restrict__ table, int bn) {
  const int nchunk = g.Kp / bn;
  const long long nent = (long long)36 * g.T * nchunk;
  const int lane = threadIdx.x & 31;
  const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long base = wid * 32; base < nent; base += nw * 32) {
    const long long e = base + lane;
    bool pass = false;
    if (e < nent) {
      const unsigned v = table[e];
      const int t = (int)((e / nchunk) % g.T);
      const int grp = (t / g.TP) / g.ipg;
      pass = v != 0 && (unsigned long long)v == acc[(size_t)grp * ST_COUNT + ST_HAD].M;
    }
    unsigned mask = __ballot_sync(0xffffffffu, pass);
    while (mask) {
      const int l = __ffs(mask) - 1;
      mask &= mask - 1;
      const long long ee = base + l;
      const int chunk = (int)(ee % nchunk);
      const int t = (int)((ee / nchunk) % g.T), xi = (int)(ee / nchunk / g.T);
      const int grp = (t / g.TP) / g.ipg;
      Acc* ga = acc + (size_t)grp * ST_COUNT;
      const long long M = (long long)ga[ST_HAD].M;
      const int8_t* vrow = V + ((size_t)xi * g.T + t) * g.Cp;
      double f = 0.0;
      for (int k = chunk * bn + lane; k < min(chunk * bn + bn, g.K); k += 32) {
        const int8_t* urow = U + ((size_t)xi * g.Kp + k) * g.Cp;
        long long s = 0;
        for (int c = 0; c < g.C; ++c) s += (int)urow[c] * (int)vrow[c];
        if ((s < 0 ? -s : s) == M)
          f = fmax(f, fabs(replay_hadamard(urow, vrow, g.C, load_int_stage(wacc[wstage], qmax_u),
                                           load_int_stage(ga[ST_IT], qmax_v))));
      }
      if (f > 0.0) atomicMax(&ga[ST_HAD].F, dbits(f));
    }
  }
}

}  // namespace wl
