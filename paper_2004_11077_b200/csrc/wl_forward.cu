// C-ABI entry points of libwinoleg_b200.so (include/winoleg_b200.h) and the host orchestration of
// the forward dependency chain.  See wl_kernels.cuh for the data layout and DESIGN.md for the
// pass structure and rooflines.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <vector>
#include <map>
#include <mutex>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>

#include "../../include/winoleg_b200.h"
#include "gemm_i8.cuh"
#include "wl_backward.h"
#include "wl_direct.h"
#include "wl_float.h"
#include "wl_kernels2.cuh"
#include "wl_staged.cuh"
#include "wl_pair.cuh"
#include "wl_tc.cuh"
#include "wl_tmap.h"

using namespace wl;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define WL_CUDA(expr)                                                                          \
  do {                                                                                         \
    cudaError_t e_ = (expr);                                                                   \
    if (e_ != cudaSuccess) return fail(WL_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)

size_t align256(size_t v) { return (v + 255) & ~size_t(255); }
int pow2_at_least(int v, int lo) {
  int p = lo;
  while (p < v) p <<= 1;
  return p;
}

}  // namespace

struct wl_plan {
  int mode;
  PlanF64* d_pf;
};

// ------------------------------------------------------------------ optional per-kernel event timing
// (bench.py: kernel share of the step and the dominant kernel's roofline).  Process global, meant
// for single-threaded measurement only.
namespace {
struct ProfCall {
  std::vector<cudaEvent_t> ev;
  std::vector<const char*> names;
};
struct Prof {
  bool on = false;
  std::vector<ProfCall> calls;
  ProfCall* cur = nullptr;
} g_prof;

void prof_begin() {
  if (!g_prof.on) return;
  g_prof.calls.emplace_back();
  g_prof.cur = &g_prof.calls.back();
}
// WL_DEBUG_SYNC=1: synchronise after every marked kernel group and report the first failing one.
const char* g_debug_fail = nullptr;
bool debug_sync_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("WL_DEBUG_SYNC");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}
void prof_mark(const char* name, cudaStream_t st) {
  if (debug_sync_enabled() && !g_debug_fail) {
    if (cudaStreamSynchronize(st) != cudaSuccess) g_debug_fail = name;
  }
  if (!g_prof.on || !g_prof.cur) return;
  cudaEvent_t e;
  cudaEventCreate(&e);
  cudaEventRecord(e, st);
  g_prof.cur->ev.push_back(e);
  g_prof.cur->names.push_back(name);
}
}  // namespace

// ------------------------------------------------------------------ stage-width plumbing

static int check_bits(const wl_qcfg* q) {
  if (!q) return fail(WL_ERR_ARG, "qcfg is NULL");
  const int v[7] = {q->input_bits,       q->weight_bits,   q->input_transform_bits, q->weight_transform_bits,
                    q->base_change_bits, q->hadamard_bits, q->output_transform_bits};
  for (int i = 0; i < 7; ++i)
    if (v[i] < 2) return fail(WL_ERR_BITS, "stage widths must be >= 2 (quantize.py:52-55)");
  if (q->input_bits > 8 || q->weight_bits > 8 || q->input_transform_bits > 8 || q->weight_transform_bits > 8 ||
      q->base_change_bits > 8)
    return fail(WL_ERR_BITS, "input/weight/transform/base-change widths must be <= 8 (int8 tensor-core operands)");
  if (q->hadamard_bits > 9) return fail(WL_ERR_BITS, "hadamard_bits must be <= 9");
  if (q->output_transform_bits > 16) return fail(WL_ERR_BITS, "output_transform_bits must be <= 16");
  return WL_OK;
}

static Bits make_bits(const wl_qcfg* q) {
  auto qm = [](int b) { return (1 << (b - 1)) - 1; };
  Bits b;
  b.q[ST_INPUT] = qm(q->input_bits);
  b.q[ST_WEIGHTS] = qm(q->weight_bits);
  b.q[ST_WT] = qm(q->weight_transform_bits);
  b.q[ST_WBC] = qm(q->base_change_bits);
  b.q[ST_IBC] = qm(q->base_change_bits);
  b.q[ST_IT] = qm(q->input_transform_bits);
  b.q[ST_HAD] = qm(q->hadamard_bits);
  b.q[ST_OBC] = qm(q->base_change_bits);
  b.q[ST_OUT] = qm(q->output_transform_bits);
  return b;
}

static int stage_bits(const wl_qcfg* q, int st) {
  switch (st) {
    case ST_INPUT: return q->input_bits;
    case ST_WEIGHTS: return q->weight_bits;
    case ST_WT: return q->weight_transform_bits;
    case ST_IT: return q->input_transform_bits;
    case ST_HAD: return q->hadamard_bits;
    case ST_OUT: return q->output_transform_bits;
    default: return q->base_change_bits;
  }
}

static const int kCanonOrder[6] = {ST_INPUT, ST_WEIGHTS, ST_WT, ST_IT, ST_HAD, ST_OUT};
static const int kLegOrder[9] = {ST_INPUT, ST_WEIGHTS, ST_WT, ST_WBC, ST_IBC, ST_IT, ST_HAD, ST_OBC, ST_OUT};

// ------------------------------------------------------------------ geometry / workspace

constexpr int kNumTables = 5;  // IBC, IT, HAD, OBC, OUT
static const int kTableStage[kNumTables] = {ST_IBC, ST_IT, ST_HAD, ST_OBC, ST_OUT};

struct Layout {
  Geo g;
  size_t off_acc, off_c0, off_v, off_h, off_c1, off_c4, off_t4, off_e4, off_tab[kNumTables], tab_bytes[kNumTables], off_otab, off_fix,
      total;
  unsigned fix_cap;
  int groups, hbytes, bn;
};

static FastDiv make_fastdiv(unsigned d) {
  FastDiv f;
  f.d = d;
  f.s = 0;
  while ((1ull << f.s) < d) ++f.s;
  f.m = (unsigned)((((1ull << 32) * ((1ull << f.s) - d)) / d) + 1);
  return f;
}

static int make_layout(const wl_shape* s, const wl_qcfg* q, Layout* L) {
  if (!s) return fail(WL_ERR_ARG, "shape is NULL");
  if (s->n < 1 || s->c_in < 1 || s->c_out < 1 || s->pad < 0)
    return fail(WL_ERR_ARG, "bad shape n=%d c_in=%d c_out=%d pad=%d", s->n, s->c_in, s->c_out, s->pad);
  const int Hp = s->h + 2 * s->pad, Wp = s->w + 2 * s->pad;
  if (Hp < 3 || Wp < 3) return fail(WL_ERR_ARG, "input %dx%d is smaller than the 3x3 kernel", Hp, Wp);
  if (s->images_per_group < 1 || s->n % s->images_per_group)
    return fail(WL_ERR_ARG, "images_per_group=%d must divide n=%d", s->images_per_group, s->n);
  Geo& g = L->g;
  g.N = s->n;
  g.C = s->c_in;
  g.K = s->c_out;
  g.H = s->h;
  g.W = s->w;
  g.pad = s->pad;
  g.Ho = Hp - 2;
  g.Wo = Wp - 2;
  g.th = (g.Ho + 3) / 4;
  g.tw = (g.Wo + 3) / 4;
  g.TP = g.th * g.tw;
  g.T = g.N * g.TP;
  g.Cp = pow2_at_least(g.C, 32);
  g.Kp = pow2_at_least(g.K, 64);
  g.ipg = s->images_per_group;
  g.fTP = make_fastdiv((unsigned)g.TP);
  g.ftw = make_fastdiv((unsigned)g.tw);
  g.fipg = make_fastdiv((unsigned)g.ipg);
  g.fC = make_fastdiv((unsigned)g.C);
  g.fK = make_fastdiv((unsigned)g.K);
  if ((unsigned long long)g.T * std::max(g.Cp, g.Kp) * 36 >= (1ULL << 32) ||
      (unsigned long long)g.N * g.H * g.W * g.Cp >= (1ULL << 32) || g.Cp > 512 || g.Kp > 512)
    return fail(WL_ERR_ARG, "problem too large for one call (split the batch; per-image scale groups are "
                            "independent)");
  L->groups = g.N / g.ipg;
  L->hbytes = q->hadamard_bits > 8 ? 2 : 1;
  size_t o = 0;
  L->off_acc = o;
  o = align256(o + sizeof(Acc) * ST_COUNT * L->groups);
  L->off_c0 = o;
  o = align256(o + (size_t)g.N * g.H * g.W * g.Cp);
  L->off_v = o;
  o = align256(o + (size_t)36 * g.T * g.Cp);
  L->off_h = o;
  o = align256(o + (size_t)36 * g.T * g.Kp * L->hbytes);
  L->off_c1 = o;
  o = align256(o + (size_t)36 * g.T * g.Cp);
  L->off_c4 = o;
  o = align256(o + (size_t)36 * g.T * g.Kp);
  // Legendre fp32-output path: output-stage fast-path values T4 [T][16][Kp] and error factors [T][Kp]
  L->off_t4 = o;
  o = align256(o + (size_t)16 * g.T * g.Kp * sizeof(float));
  L->off_e4 = o;
  o = align256(o + (size_t)g.T * g.Kp * sizeof(float));
  L->bn = (g.Kp >= 256 ? 256 : g.Kp) / 4;  // table chunk = one max-pass epilogue warp's columns (EpiHadMax::kGroups)
  const size_t CB = (g.C + 31) / 32, KB = (g.K + 31) / 32;
  const size_t ents[kNumTables] = {g.T * CB, g.T * CB, (size_t)36 * g.T * (g.Kp / L->bn), g.T * KB, g.T * KB};
  for (int i = 0; i < kNumTables; ++i) {
    L->off_tab[i] = o;
    L->tab_bytes[i] = ents[i] * sizeof(unsigned);
    o = align256(o + L->tab_bytes[i]);
  }
  // dequantised output table (output widths <= 12 bits; wider widths dequantise in fp64 inline)
  L->off_otab = o;
  if (q->output_transform_bits <= 12) o = align256(o + sizeof(float) * (size_t)L->groups * ((1 << q->output_transform_bits) - 1));
  // deferred-fix list: counters + unit ids (expected ~0.2% of units; overflow falls back inline)
  L->off_fix = o;
  const size_t units = (size_t)g.T * std::max(g.C, g.K);
  L->fix_cap = (unsigned)std::max<size_t>(4096, units / 16);
  o = align256(o + 64 + sizeof(unsigned) * (size_t)L->fix_cap);
  L->total = o;
  return WL_OK;
}

struct WeightHeader {
  Acc wacc[ST_COUNT];
  int K, C, Kp, Cp, mode, wstage;
  wl_qcfg q;
};

static size_t weight_cache_bytes(int K, int C, int* Kp, int* Cp) {
  *Cp = pow2_at_least(C, 32);
  *Kp = pow2_at_least(K, 64);
  return align256(sizeof(WeightHeader)) + (size_t)36 * (*Kp) * (*Cp);
}

// Persistent grid for a staged kernel: resident blocks per SM (occupancy query, cached) x SMs.
template <class K>
static int staged_grid(K kern, int threads, int smem, long long work_items) {
  // keyed by kernel: instantiations with identical parameter types share K
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> cache;
  const auto key = std::make_pair(reinterpret_cast<const void*>(kern), smem);
  int per_sm = 0;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      per_sm = it->second;
    } else {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
      if (per_sm < 1) per_sm = 1;
      cache[key] = per_sm;
    }
  }
  int dev_sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, dev);
  return (int)std::max(1LL, std::min<long long>(work_items, (long long)per_sm * dev_sms));
}

// ------------------------------------------------------------------ compile-time strides
template <int V>
using IntC = std::integral_constant<int, V>;
template <class F>
static int dispatch_ld_in(int ld, F&& f) {
  switch (ld) {
    case 32: f(IntC<32>{}); return WL_OK;
    case 64: f(IntC<64>{}); return WL_OK;
    case 128: f(IntC<128>{}); return WL_OK;
    case 256: f(IntC<256>{}); return WL_OK;
    case 512: f(IntC<512>{}); return WL_OK;
  }
  return fail(WL_ERR_ARG, "unsupported padded channel count %d", ld);
}
template <class F>
static int dispatch_ld_out(int ld, F&& f) {
  switch (ld) {
    case 64: f(IntC<64>{}); return WL_OK;
    case 128: f(IntC<128>{}); return WL_OK;
    case 256: f(IntC<256>{}); return WL_OK;
    case 512: f(IntC<512>{}); return WL_OK;
  }
  return fail(WL_ERR_ARG, "unsupported padded output-channel count %d", ld);
}

// ------------------------------------------------------------------ GEMM epilogues

// Max pass: exact int32 accumulators; per-thread maximum over its row chunk; the group maximum M is
// reduced in place (atomicMax) and units that may hold the argmax are pushed as candidates for the
// fp64 replay in finalize_hadamard_kernel.
struct EpiHadMax {
  static constexpr int kGroups = 4;
  static constexpr int kStageBytes = 0;
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
    publish_max(m, grp, a, ST_COUNT, uniform, wmax);
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
  bool small;  // |I| < 2^22: int -> float by the magic-number add instead of I2F
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
    small = (long long)g.C * qmax_u * qmax_v < (1LL << 22);
  }
  __device__ __forceinline__ void apply(int xi, int row, int col, const uint32_t* v, int n) {
    // y[j] = 0x4B400000 + code: its low byte / half-word is the two's-complement code
    uint32_t y[16];
    uint32_t d0 = 0, d1 = 0, d2 = 0, d3 = 0;  // independent chains (ILP)
    if (small) {
      // column pairs on packed f32x2 (FADD2 / FFMA2: lane-wise identical to the scalar ops)
#pragma unroll
      for (int j = 0; j < 16; j += 2) {
        const f2 fi = sub2(mk2(__int_as_float((int)v[j] + 0x4B400000), __int_as_float((int)v[j + 1] + 0x4B400000)),
                           bc2(kMagic));
        const f2 ya = fma2(fi, bc2(r_lo), bc2(kMagic)), yb = fma2(fi, bc2(r_hi), bc2(kMagic));
        y[j] = __float_as_uint(lo2(ya));
        y[j + 1] = __float_as_uint(hi2(ya));
        const uint32_t da = y[j] ^ __float_as_uint(lo2(yb)), db = y[j + 1] ^ __float_as_uint(hi2(yb));
        if ((j & 2) == 0) d0 |= da, d1 |= db; else d2 |= da, d3 |= db;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float fi = (float)(int)v[j];
        y[j] = __float_as_uint(fmaf(fi, r_lo, kMagic));
        const uint32_t d = y[j] ^ __float_as_uint(fmaf(fi, r_hi, kMagic));
        if ((j & 3) == 0) d0 |= d; else if ((j & 3) == 1) d1 |= d; else if ((j & 3) == 2) d2 |= d; else d3 |= d;
      }
    }
    const bool exact = ((d0 | d1) | (d2 | d3)) != 0;  // rare: some element's bracket split
    const int lane = threadIdx.x & 31;
    const int slot0 = ((col % hc) * (int)sizeof(HT)) >> 4;
    const uint32_t rbase = smem_u32(stage) + lane * kRowBytes;
    const HadRqCtx cx{acc, wacc, U, V, g.C, g.Cp, g.Kp, grp, wstage, qmax_u, qmax_v, qmax_h, xi, row, fl};
    if constexpr (sizeof(HT) == 1) {
      uint32_t w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        w[q] = __byte_perm(__byte_perm(y[4 * q], y[4 * q + 1], 0x0040), __byte_perm(y[4 * q + 2], y[4 * q + 3], 0x0040),
                           0x5410);
      if (exact) {
        const uint4 lo = had_rq_slow8<HT>(cx, make_uint4(v[0], v[1], v[2], v[3]), make_uint4(v[4], v[5], v[6], v[7]), col, n);
        const uint4 hi = had_rq_slow8<HT>(cx, make_uint4(v[8], v[9], v[10], v[11]), make_uint4(v[12], v[13], v[14], v[15]),
                                          col + 8, n - 8);
        w[0] = lo.x, w[1] = lo.y, w[2] = hi.x, w[3] = hi.y;
      }
      st_shared_v4(rbase + ((slot0 ^ (lane & kSwz)) << 4), w[0], w[1], w[2], w[3]);
    } else {
      uint32_t w[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) w[q] = __byte_perm(y[2 * q], y[2 * q + 1], 0x5410);
      if (exact) {
        const uint4 lo = had_rq_slow8<HT>(cx, make_uint4(v[0], v[1], v[2], v[3]), make_uint4(v[4], v[5], v[6], v[7]), col, n);
        const uint4 hi = had_rq_slow8<HT>(cx, make_uint4(v[8], v[9], v[10], v[11]), make_uint4(v[12], v[13], v[14], v[15]),
                                          col + 8, n - 8);
        w[0] = lo.x, w[1] = lo.y, w[2] = lo.z, w[3] = lo.w, w[4] = hi.x, w[5] = hi.y, w[6] = hi.z, w[7] = hi.w;
      }
      st_shared_v4(rbase + ((slot0 ^ (lane & kSwz)) << 4), w[0], w[1], w[2], w[3]);
      st_shared_v4(rbase + (((slot0 + 1) ^ (lane & kSwz)) << 4), w[4], w[5], w[6], w[7]);
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

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int BN, int SW, class Epi>
static int launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, const Geo& g, const Epi& e, cudaStream_t st) {
  constexpr int STAGES = Epi::kStageBytes > 0 ? 3 : 4;
  using L = GemmPSmem<BN, SW, STAGES, Epi::kStageBytes, 4 * Epi::kGroups>;
  auto kern = gemm_i8_persistent<BN, SW, STAGES, Epi>;
  static bool attr_set = false;  // per instantiation; idempotent
  if (!attr_set) {
    WL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kBytes));
    attr_set = true;
  }
  const int ntiles = 36 * ((g.T + 127) / 128) * (g.Kp / BN);
  const int grid = std::min(ntiles, num_sms());
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

// Max row abs-sum of each stage's integer matrix: with the group's max |first-half value| it bounds
// the fp32 error of the second half (stage_error in wl_kernels2.cuh).
// fp32 second-half rounding depth of each transform stage (the fast path's certified band)
static float stage_depth(int mode, int stage) {
  const bool leg = mode == WL_LEGENDRE;
  switch (stage) {
    case ST_IBC: return (float)chain_depth<tab::Leg_IBC>();
    case ST_IT: return leg ? (float)chain_depth<tab::Leg_IT>() : (float)chain_depth<tab::Can_IT>();
    case ST_OBC: return (float)chain_depth<tab::Leg_OBC>();
    case ST_OUT: return leg ? (float)chain_depth<tab::Leg_OT>() : (float)chain_depth<tab::Can_OT>();
    default: return 6.f;
  }
}

static StageE stage_rowsums(int mode) {
  auto rowsum = [](auto tag, int R, int C) {
    using M = decltype(tag);
    long long best = 0;
    for (int i = 0; i < R; ++i) {
      long long s = 0;
      for (int j = 0; j < C; ++j) s += std::abs(M::e(i, j));
      best = std::max(best, s);
    }
    return (float)best;
  };
  StageE E;
  for (int i = 0; i < ST_COUNT; ++i) E.e[i] = 0.f;
  if (mode == WL_CANONICAL) {
    E.e[ST_IT] = rowsum(tab::Can_IT{}, 6, 6);
    E.e[ST_OUT] = rowsum(tab::Can_OT{}, 4, 6);
  } else {
    E.e[ST_IBC] = rowsum(tab::Leg_IBC{}, 6, 6);
    E.e[ST_IT] = rowsum(tab::Leg_IT{}, 6, 6);
    E.e[ST_OBC] = rowsum(tab::Leg_OBC{}, 6, 6);
    E.e[ST_OUT] = rowsum(tab::Leg_OT{}, 4, 6);
  }
  return E;
}

// ------------------------------------------------------------------ C ABI

extern "C" {

const char* wl_last_error(void) { return g_err.c_str(); }

int wl_profile_enable(int on) {
  g_prof.on = on != 0;
  return WL_OK;
}

// Sums the per-kernel event intervals of every wl_forward since the last read (synchronising).
// names_out receives up to `max` kernel names (static strings), ms_out their summed milliseconds.
int wl_profile_read(const char** names_out, double* ms_out, int max, int* n_out, int* calls_out) {
  WL_CUDA(cudaDeviceSynchronize());
  int n = 0;
  std::vector<double> acc;
  std::vector<const char*> names;
  for (auto& c : g_prof.calls) {
    for (size_t i = 1; i < c.ev.size(); ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, c.ev[i - 1], c.ev[i]);
      if (acc.size() < i) {
        acc.push_back(0.0);
        names.push_back(c.names[i]);
      }
      acc[i - 1] += ms;
    }
    for (auto e : c.ev) cudaEventDestroy(e);
  }
  n = (int)acc.size();
  for (int i = 0; i < n && i < max; ++i) {
    if (names_out) names_out[i] = names[i];
    if (ms_out) ms_out[i] = acc[i];
  }
  if (n_out) *n_out = n;
  if (calls_out) *calls_out = (int)g_prof.calls.size();
  g_prof.calls.clear();
  g_prof.cur = nullptr;
  return WL_OK;
}

int wl_plan_create(int o, int k, int mode, const int64_t* int_mats, const double* f64_mats, wl_plan** out) {
  if (!out || !int_mats || !f64_mats) return fail(WL_ERR_ARG, "NULL argument");
  if (o != 4 || k != 3) return fail(WL_ERR_PLAN, "only F(4,3) is compiled for sm_100a (got F(%d,%d))", o, k);
  if (mode != WL_CANONICAL && mode != WL_LEGENDRE) return fail(WL_ERR_ARG, "unknown mode %d", mode);
  // verify the host construction against the compiled tables
  int bad = 0;
  const int64_t* p = int_mats;
  auto check = [&](auto tag, int R, int C) {
    using M = decltype(tag);
    for (int i = 0; i < R; ++i)
      for (int j = 0; j < C; ++j)
        if (*p++ != M::e(i, j)) ++bad;
  };
  PlanF64 pf;
  memset(&pf, 0, sizeof(pf));
  const double* f = f64_mats;
  if (mode == WL_CANONICAL) {
    check(tab::Can_WT{}, 6, 3);
    check(tab::Can_IT{}, 6, 6);
    check(tab::Can_OT{}, 4, 6);
    memcpy(pf.wt, f, 18 * 8);
    memcpy(pf.it, f + 18, 36 * 8);
    memcpy(pf.ot, f + 54, 24 * 8);
  } else {
    check(tab::Leg_WT{}, 6, 3);
    check(tab::Leg_WBC{}, 6, 6);
    check(tab::Leg_IBC{}, 6, 6);
    check(tab::Leg_IT{}, 6, 6);
    check(tab::Leg_OBC{}, 6, 6);
    check(tab::Leg_OT{}, 4, 6);
    memcpy(pf.wt, f, 18 * 8);
    memcpy(pf.wbc, f + 18, 36 * 8);
    memcpy(pf.ibc, f + 54, 36 * 8);
    memcpy(pf.it, f + 90, 36 * 8);
    memcpy(pf.obc, f + 126, 36 * 8);
    memcpy(pf.ot, f + 162, 24 * 8);
  }
  if (bad)
    return fail(WL_ERR_PLAN, "plan differs from the compiled default-point F(4,3) tables in %d entries", bad);
  wl_plan* pl = new wl_plan;
  pl->mode = mode;
  cudaError_t e = cudaMalloc(&pl->d_pf, sizeof(PlanF64));
  if (e == cudaSuccess) e = cudaMemcpy(pl->d_pf, &pf, sizeof(PlanF64), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    delete pl;
    return fail(WL_ERR_CUDA, "plan upload: %s", cudaGetErrorString(e));
  }
  *out = pl;
  return WL_OK;
}

int wl_plan_destroy(wl_plan* plan) {
  if (!plan) return WL_OK;
  cudaFree(plan->d_pf);
  delete plan;
  return WL_OK;
}

int wl_plan_mode(const wl_plan* plan) { return plan ? plan->mode : WL_ERR_ARG; }

// ------------------------------------------------------------------ float (unquantized) path
static int float_geo(const wl_shape* s, FGeo* g) {
  if (!s) return fail(WL_ERR_ARG, "shape is NULL");
  if (s->n < 1 || s->c_in < 1 || s->c_out < 1 || s->pad < 0)
    return fail(WL_ERR_ARG, "bad shape n=%d c_in=%d c_out=%d pad=%d", s->n, s->c_in, s->c_out, s->pad);
  const int Hp = s->h + 2 * s->pad, Wp = s->w + 2 * s->pad;
  if (Hp < 3 || Wp < 3) return fail(WL_ERR_ARG, "input %dx%d is smaller than the 3x3 kernel", Hp, Wp);
  g->N = s->n, g->C = s->c_in, g->K = s->c_out, g->H = s->h, g->W = s->w, g->pad = s->pad;
  g->Ho = Hp - 2, g->Wo = Wp - 2, g->th = (g->Ho + 3) / 4, g->tw = (g->Wo + 3) / 4, g->TP = g->th * g->tw;
  g->T = g->N * g->TP;
  if ((unsigned long long)36 * g->T * std::max(g->C, g->K) >= (1ULL << 31))
    return fail(WL_ERR_ARG, "problem too large for one float call (split the batch)");
  return WL_OK;
}

int wl_float_workspace_size(const wl_plan* plan, const wl_shape* s, size_t* bytes) {
  if (!plan || !bytes) return fail(WL_ERR_ARG, "NULL argument");
  FGeo g;
  if (int rc = float_geo(s, &g)) return rc;
  *bytes = wl_float_workspace_bytes(g);
  return WL_OK;
}

int wl_forward_float(const wl_plan* plan, const wl_shape* s, const float* x, const float* w, const float* bias, float* y,
                     void* workspace, size_t workspace_bytes, void* stream) {
  if (!plan || !x || !w || !y || !workspace) return fail(WL_ERR_ARG, "NULL argument");
  FGeo g;
  if (int rc = float_geo(s, &g)) return rc;
  if (workspace_bytes < wl_float_workspace_bytes(g))
    return fail(WL_ERR_WORKSPACE, "workspace needs %zu bytes", wl_float_workspace_bytes(g));
  std::string err;
  if (wl_float_run(plan->mode == WL_LEGENDRE, plan->d_pf, g, x, w, bias, y, workspace, (cudaStream_t)stream, &err))
    return fail(WL_ERR_CUDA, "float path: %s", err.c_str());
  return WL_OK;
}

static int direct_geo(const wl_shape* s, DGeo* g) {
  if (!s) return fail(WL_ERR_ARG, "shape is NULL");
  if (s->n < 1 || s->c_in < 1 || s->c_out < 1 || s->pad < 0 || s->images_per_group < 1 ||
      s->n % s->images_per_group != 0)
    return fail(WL_ERR_ARG, "bad shape n=%d c_in=%d c_out=%d pad=%d images_per_group=%d", s->n, s->c_in, s->c_out,
                s->pad, s->images_per_group);
  const int Hp = s->h + 2 * s->pad, Wp = s->w + 2 * s->pad;
  if (Hp < 3 || Wp < 3) return fail(WL_ERR_ARG, "input %dx%d is smaller than the 3x3 kernel", Hp, Wp);
  g->N = s->n, g->C = s->c_in, g->K = s->c_out, g->H = s->h, g->W = s->w, g->pad = s->pad;
  g->Ho = Hp - 2, g->Wo = Wp - 2, g->ipg = s->images_per_group;
  return WL_OK;
}

static int direct_bits(const wl_qcfg* q) {
  if (!q) return fail(WL_ERR_ARG, "qconfig is NULL");
  if (q->input_bits < 2 || q->input_bits > 53 || q->weight_bits < 2 || q->weight_bits > 53 ||
      q->output_transform_bits < 2 || q->output_transform_bits > 53)
    return fail(WL_ERR_BITS, "direct baseline widths must be in [2, 53]");
  return WL_OK;
}

int wl_direct_workspace_size(const wl_shape* s, size_t* bytes) {
  if (!bytes) return fail(WL_ERR_ARG, "NULL argument");
  DGeo g;
  if (int rc = direct_geo(s, &g)) return rc;
  *bytes = wl_direct_workspace_bytes(g);
  return WL_OK;
}

}  // extern "C"

template <typename T>
static int direct_impl(const wl_qcfg* q, const wl_shape* s, const T* x, const T* w, T* y, void* workspace,
                       size_t workspace_bytes, void* stream) {
  if (!x || !w || !y || !workspace) return fail(WL_ERR_ARG, "NULL argument");
  DGeo g;
  if (int rc = direct_geo(s, &g)) return rc;
  if (int rc = direct_bits(q)) return rc;
  if (workspace_bytes < wl_direct_workspace_bytes(g))
    return fail(WL_ERR_WORKSPACE, "workspace needs %zu bytes", wl_direct_workspace_bytes(g));
  std::string err;
  if (wl_direct_run<T>(g, q->input_bits, q->weight_bits, q->output_transform_bits, x, w, y, workspace,
                       (cudaStream_t)stream, &err))
    return fail(WL_ERR_CUDA, "direct baseline: %s", err.c_str());
  return WL_OK;
}

extern "C" {

int wl_direct_quantized(const wl_qcfg* q, const wl_shape* s, const float* x, const float* w, float* y,
                        void* workspace, size_t workspace_bytes, void* stream) {
  return direct_impl<float>(q, s, x, w, y, workspace, workspace_bytes, stream);
}

int wl_direct_f64(const wl_shape* s, const double* x, const double* w, double* y, void* workspace,
                  size_t workspace_bytes, void* stream) {
  const wl_qcfg none = {0, 0, 0, 0, 0, 0, 0};  // identity casts
  if (!x || !w || !y || !workspace) return fail(WL_ERR_ARG, "NULL argument");
  DGeo g;
  if (int rc = direct_geo(s, &g)) return rc;
  if (workspace_bytes < wl_direct_workspace_bytes(g))
    return fail(WL_ERR_WORKSPACE, "workspace needs %zu bytes", wl_direct_workspace_bytes(g));
  std::string err;
  if (wl_direct_run<double>(g, none.input_bits, none.weight_bits, none.output_transform_bits, x, w, y, workspace,
                            (cudaStream_t)stream, &err))
    return fail(WL_ERR_CUDA, "direct correlation: %s", err.c_str());
  return WL_OK;
}

int wl_direct_quantized_f64(const wl_qcfg* q, const wl_shape* s, const double* x, const double* w, double* y,
                            void* workspace, size_t workspace_bytes, void* stream) {
  return direct_impl<double>(q, s, x, w, y, workspace, workspace_bytes, stream);
}

int wl_num_stages(const wl_plan* plan) { return plan ? (plan->mode == WL_LEGENDRE ? 9 : 6) : WL_ERR_ARG; }

int wl_weight_cache_size(const wl_plan* plan, int c_out, int c_in, size_t* bytes) {
  if (!plan || !bytes || c_out < 1 || c_in < 1) return fail(WL_ERR_ARG, "bad weight-cache query");
  int Kp, Cp;
  *bytes = weight_cache_bytes(c_out, c_in, &Kp, &Cp);
  return WL_OK;
}

}  // extern "C"

template <typename XT>
static int weight_transform_impl(const wl_plan* plan, const wl_qcfg* q, const XT* w, int c_out, int c_in, void* cache,
                                 size_t cache_bytes, void* stream) {
  if (!plan || !w || !cache) return fail(WL_ERR_ARG, "NULL argument");
  int rc = check_bits(q);
  if (rc) return rc;
  int Kp, Cp;
  const size_t need = weight_cache_bytes(c_out, c_in, &Kp, &Cp);
  if (cache_bytes < need) return fail(WL_ERR_WORKSPACE, "weight cache needs %zu bytes", need);
  cudaStream_t st = (cudaStream_t)stream;
  WeightHeader hdr;
  memset(&hdr, 0, sizeof(hdr));
  hdr.K = c_out;
  hdr.C = c_in;
  hdr.Kp = Kp;
  hdr.Cp = Cp;
  hdr.mode = plan->mode;
  hdr.wstage = plan->mode == WL_LEGENDRE ? ST_WBC : ST_WT;
  hdr.q = *q;
  WeightHeader* dh = reinterpret_cast<WeightHeader*>(cache);
  int8_t* U = reinterpret_cast<int8_t*>(cache) + align256(sizeof(WeightHeader));
  WL_CUDA(cudaMemcpyAsync(dh, &hdr, sizeof(hdr), cudaMemcpyHostToDevice, st));
  WL_CUDA(cudaMemsetAsync(U, 0, (size_t)36 * Kp * Cp, st));
  const Bits b = make_bits(q);
  const long long nw = (long long)c_out * c_in * 9;
  absmax_weights_kernel<XT><<<(int)std::min<long long>((nw + 255) / 256, 1024), 256, 0, st>>>(w, nw, dh->wacc);
  // "weights" stage max_abs is exact: F = fp64(max |w|) is filled by the readers from M.
  const int threads = 256, blocks = (c_out * c_in + threads - 1) / threads;
  if (plan->mode == WL_CANONICAL) {
    weight_stage_kernel<0, 0, XT><<<blocks, threads, 0, st>>>(w, c_out, c_in, Kp, Cp, U, b, dh->wacc, plan->d_pf);
    weight_stage_kernel<0, 2, XT><<<blocks, threads, 0, st>>>(w, c_out, c_in, Kp, Cp, U, b, dh->wacc, plan->d_pf);
  } else {
    weight_stage_kernel<1, 0, XT><<<blocks, threads, 0, st>>>(w, c_out, c_in, Kp, Cp, U, b, dh->wacc, plan->d_pf);
    weight_stage_kernel<1, 1, XT><<<blocks, threads, 0, st>>>(w, c_out, c_in, Kp, Cp, U, b, dh->wacc, plan->d_pf);
    weight_stage_kernel<1, 2, XT><<<blocks, threads, 0, st>>>(w, c_out, c_in, Kp, Cp, U, b, dh->wacc, plan->d_pf);
  }
  WL_CUDA(cudaGetLastError());
  return WL_OK;
}

extern "C" {

int wl_weight_transform(const wl_plan* plan, const wl_qcfg* q, const float* w, int c_out, int c_in, void* cache,
                        size_t cache_bytes, void* stream) {
  return weight_transform_impl(plan, q, w, c_out, c_in, cache, cache_bytes, stream);
}

int wl_weight_transform_f64(const wl_plan* plan, const wl_qcfg* q, const double* w, int c_out, int c_in, void* cache,
                            size_t cache_bytes, void* stream) {
  return weight_transform_impl(plan, q, w, c_out, c_in, cache, cache_bytes, stream);
}

int wl_workspace_size(const wl_plan* plan, const wl_shape* s, const wl_qcfg* q, size_t* bytes) {
  if (!plan || !bytes) return fail(WL_ERR_ARG, "NULL argument");
  int rc = check_bits(q);
  if (rc) return rc;
  Layout L;
  rc = make_layout(s, q, &L);
  if (rc) return rc;
  *bytes = L.total;
  return WL_OK;
}

int wl_debug_layout(const wl_plan* plan, const wl_shape* s, const wl_qcfg* q, size_t* off, int* dims) {
  if (!plan || !off || !dims) return fail(WL_ERR_ARG, "NULL argument");
  int rc = check_bits(q);
  if (rc) return rc;
  Layout L;
  rc = make_layout(s, q, &L);
  if (rc) return rc;
  off[0] = L.off_c0;
  off[1] = L.off_v;
  off[2] = L.off_h;
  off[3] = L.off_acc;
  dims[0] = L.g.Cp;
  dims[1] = L.g.Kp;
  dims[2] = L.g.T;
  dims[3] = L.g.TP;
  return WL_OK;
}

int wl_forward_launches(const wl_plan* plan, const wl_shape* s, const wl_qcfg* q) {
  if (!plan) return WL_ERR_ARG;
  // fp32 forward with per-image groups and W % 4 == 0, W, H <= 64: absmax + quant fused into one kernel
  const int fused = (s && s->images_per_group == 1 && (s->w & 3) == 0 && s->w <= 64 && s->h <= 64 &&
                     getenv("WL_FUSED_QUANT")) ? 1 : 0;
  // absmax, quant, [in_a|in_b(+fixup), finalize, params] x2|1, in_c, fixup, gemm max, finalize, params,
  // gemm codes, tie fixup, [out_a|out_b(+fixup), finalize, params] x2|1, output table, out_c, fixup
  const int otab = (q && q->output_transform_bits <= 12) ? 1 : 0;
  // + one finalize_*_exec per transform finalize (4 Legendre, 2 canonical)
  return (plan->mode == WL_LEGENDRE ? 29 : 19) + otab - fused;
}

}  // extern "C"

template <typename XT, typename YT>
static int forward_impl(const wl_plan* plan, const wl_qcfg* q, const wl_shape* s, const XT* x, const void* cache,
                        const YT* bias, YT* y, void* workspace, size_t workspace_bytes, void* stream) {
  if (!plan || !x || !cache || !y || !workspace) return fail(WL_ERR_ARG, "NULL argument");
  int rc = check_bits(q);
  if (rc) return rc;
  Layout L;
  rc = make_layout(s, q, &L);
  if (rc) return rc;
  if (workspace_bytes < L.total) return fail(WL_ERR_WORKSPACE, "workspace needs %zu bytes", L.total);
  const Geo& g = L.g;
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  Acc* acc = reinterpret_cast<Acc*>(ws + L.off_acc);
  int8_t* c0 = reinterpret_cast<int8_t*>(ws + L.off_c0);
  int8_t* V = reinterpret_cast<int8_t*>(ws + L.off_v);
  void* h = ws + L.off_h;
  const WeightHeader* wh = reinterpret_cast<const WeightHeader*>(cache);
  const int8_t* U = reinterpret_cast<const int8_t*>(cache) + align256(sizeof(WeightHeader));
  const Bits b = make_bits(q);
  const bool leg = plan->mode == WL_LEGENDRE;

  prof_begin();
  WL_CUDA(cudaMemsetAsync(acc, 0, sizeof(Acc) * ST_COUNT * L.groups, st));
  prof_mark("begin", st);
  {
    const long long per_image = (long long)g.C * g.H * g.W;
    // fused cast "input" (one HBM pass over x) for per-image groups: cooperative teams of g.H blocks
    bool fused = false;
    if (sizeof(XT) == 4 && g.ipg == 1 && (g.W & 3) == 0 && g.W <= 64 && g.H <= 64 && (per_image & 3) == 0 &&
        (size_t)g.N <= L.fix_cap && getenv("WL_FUSED_QUANT")) {  // opt-in: measured 1.25 ms = the two passes
      const size_t qsm_f = (size_t)g.W * (g.Cp + 4);
      static int occ = -1;
      if (occ < 0 && cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, absquant_fused_kernel, 256, qsm_f) != cudaSuccess)
        occ = 0;
      int cur_dev = 0, coop = 0;
      cudaGetDevice(&cur_dev);
      cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, cur_dev);
      const char* te = getenv("WL_FUSED_TEAM");  // blocks per image (experiments); default H/2 rows x 2
      int team = te ? atoi(te) : ((g.H & 1) == 0 && g.H >= 16 ? g.H / 2 : g.H);
      team = std::max(1, std::min(team, g.H));
      const int nteams = std::min(g.N, occ * num_sms() / team);
      if (coop && nteams >= 1) {
        unsigned* arrive = reinterpret_cast<unsigned*>(ws + L.off_fix + 64);  // fix items: unused until the transforms
        WL_CUDA(cudaMemsetAsync(arrive, 0, sizeof(unsigned) * g.N, st));
        prof_mark("absmax_input", st);
        const float* xf = reinterpret_cast<const float*>(x);
        int teamv = team;
        void* args[] = {(void*)&xf, (void*)&c0, (void*)&g, (void*)&b, (void*)&acc, (void*)&arrive, (void*)&teamv};
        WL_CUDA(cudaLaunchCooperativeKernel((const void*)absquant_fused_kernel, dim3(nteams * team), dim3(256), args,
                                            qsm_f, st));
        prof_mark("quant_input", st);
        fused = true;
      }
    }
    if (!fused) {
    int bx = (int)std::min<long long>((per_image / 4 + 255) / 256, 64);
    absmax_input_kernel<XT><<<dim3(std::max(bx, 1), g.N), 256, 0, st>>>(x, per_image, g.ipg, acc);
    prof_mark("absmax_input", st);
    const int qrow = std::max(4, std::min(64, (160000 / (g.Cp + 16)) & ~3));
    const size_t qsm = (size_t)qrow * (g.Cp + 16);
    static bool qattr = false;
    if (!qattr) {
      WL_CUDA(cudaFuncSetAttribute(quant_input_kernel<XT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      qattr = true;
    }
    if (sizeof(XT) == 4 && (g.W & 3) == 0 && g.W <= 64 && !getenv("WL_GENERIC_QUANT"))
      quant_input_w64_kernel<<<dim3(g.H, g.N), 256, (size_t)g.W * (g.Cp + 4), st>>>(
          reinterpret_cast<const float*>(x), c0, g, b, acc);
    else
      quant_input_kernel<XT><<<dim3(g.H, g.N), 256, qsm, st>>>(x, c0, g, b, acc, qrow);
    prof_mark("quant_input", st);
    }
  }
  int8_t* c1 = reinterpret_cast<int8_t*>(ws + L.off_c1);
  int8_t* c4 = reinterpret_cast<int8_t*>(ws + L.off_c4);
  float* t4 = reinterpret_cast<float*>(ws + L.off_t4);
  float* e4 = reinterpret_cast<float*>(ws + L.off_e4);
  // Legendre, fp32 output, staged output side: store T4 instead of c4 (WL_NO_T4 = the c4 path)
  const bool t4path = leg && sizeof(YT) == 4 && g.Kp <= 256 && !getenv("WL_NO_T4");
  Tables tabs;
  for (int i = 0; i < ST_COUNT; ++i) tabs.t[i] = nullptr;
  for (int i = 0; i < kNumTables; ++i) {
    tabs.t[kTableStage[i]] = reinterpret_cast<unsigned*>(ws + L.off_tab[i]);
    if (kTableStage[i] != ST_HAD) WL_CUDA(cudaMemsetAsync(ws + L.off_tab[i], 0, L.tab_bytes[i], st));
  }
  const StageE E = stage_rowsums(plan->mode);
  FixList fl;
  fl.count = reinterpret_cast<unsigned*>(ws + L.off_fix);
  fl.items = reinterpret_cast<unsigned*>(ws + L.off_fix + 64);
  fl.cap = L.fix_cap;
  WL_CUDA(cudaMemsetAsync(fl.count, 0, 64, st));
  const int fix_blocks = 16 * 148;  // one wave covers every deferred unit of config-4-sized calls (latency-bound per unit)

  const long long tc = (long long)g.T * g.C;
  const int tb = 256;
  const unsigned tgrid = (unsigned)((tc + tb - 1) / tb);
  const int fin_blocks = 4 * 148;
  const int pgrid = (L.groups + 127) / 128;
  const bool staged_in = !getenv("WL_NO_STAGED_IN"), staged_out = !getenv("WL_NO_STAGED_OUT");  // debug switches
  // the input code pass is staged (bulk-copied c0 windows / c1 blocks); the output code pass stays on
  // the plain grid (staged it measured 2.8x slower: y stores from few resident CTAs)
  const bool staged_c = !getenv("WL_PLAIN_IN_C");
  // two channels per thread on packed f32x2 (wl_pair.cuh; bit-identical, fewer issued instructions)
  const bool pair = !getenv("WL_NO_PAIR");
  CUtensorMap c0map;
  if (g.Cp <= 256 && !make_tmap_i8_4d(&c0map, c0, g.Cp, g.W, g.H, g.N, g.Cp, 6, 6))
    return fail(WL_ERR_CUDA, "cuTensorMapEncodeTiled (input window) failed");
  rc = dispatch_ld_in(g.Cp, [&](auto ldc) {
    constexpr int LD = decltype(ldc)::value;
    if (LD <= 256 && staged_in) {
      using S = Staged<(LD <= 256 ? LD : 256), 1>;
      constexpr int LDs = LD <= 256 ? LD : 256;
      const long long iters = (g.T + S::TPB - 1) / S::TPB;
      if (!leg) {
        auto ka = sin_a_kernel<0, LDs>;
        sin_a_kernel<0, LDs><<<staged_grid(ka, S::THREADS, S::SMEM, iters), S::THREADS, S::SMEM, st>>>(c0map, g, acc, tabs);
        finalize_input_kernel<0, ST_IT><<<fin_blocks, 256, 0, st>>>(c0, c1, g, b, acc, plan->d_pf, tabs.t[ST_IT], E.e[ST_IT], fl);
        finalize_input_exec<0, ST_IT><<<fin_blocks, 256, 0, st>>>(c0, c1, g, b, acc, plan->d_pf, fl);
        stage_params_kernel<<<pgrid, 128, 0, st>>>(acc, L.groups, ST_IT, b.q[ST_IT], E.e[ST_IT], stage_depth(plan->mode, ST_IT));
        prof_mark("input_transform_max", st);
        if (staged_c) {
          auto kc = sin_c_kernel<0, LDs>;
          sin_c_kernel<0, LDs><<<staged_grid(kc, S::THREADS, S::SMEM_OUT, iters), S::THREADS, S::SMEM_OUT, st>>>(c0map, c0, c1, V, g, b, acc, plan->d_pf, fl);
        } else
        in_c_kernel<0, LD><<<tgrid, tb, 0, st>>>(c0, c1, V, g, b, acc, plan->d_pf, fl);
        fixup_it_kernel<0><<<fix_blocks, 128, 0, st>>>(fl, c0, c1, V, g, b, acc, plan->d_pf);
        prof_mark("input_transform_codes", st);
      } else {
        CUtensorMap amap;
        // WL_TC_SIN_A=1: the tcgen05 Kronecker-digit pass (exact; measured 1.45 ms vs 0.67 ms for the
        // CUDA-core pass on config 4: recombining three int32 digit accumulators per output costs as
        // many instructions as the sparse P^-T sandwich itself — see DESIGN.md §4)
        if ((g.Cp == 128 || g.Cp == 256) && getenv("WL_TC_SIN_A") &&
            make_tmap_i8_4d_sw128(&amap, c0, g.Cp, g.W, g.H, g.N, 6, 6)) {
          // tensor-core pass: one int8 MMA per (tile, 128 channels) against the Kronecker digits
          static bool attr = false;
          if (!attr) {
            cudaFuncSetAttribute(tc::sin_a_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::SMEM);
            attr = true;
          }
          tc::sin_a_tc_kernel<<<num_sms(), tc::THREADS, tc::SMEM, st>>>(amap, g, acc, tabs);
        } else if (pair) {
          using S2 = Staged2<LDs, 1>;
          auto ka = sin_a2_kernel<1, LDs>;
          const long long it2 = (g.T + S2::TPB - 1) / S2::TPB;
          sin_a2_kernel<1, LDs><<<staged_grid(ka, S2::THREADS, S2::SMEM, it2), S2::THREADS, S2::SMEM, st>>>(c0map, g, acc, tabs);
        } else {
          auto ka = sin_a_kernel<1, LDs>;
          sin_a_kernel<1, LDs><<<staged_grid(ka, S::THREADS, S::SMEM, iters), S::THREADS, S::SMEM, st>>>(c0map, g, acc, tabs);
        }
        finalize_input_kernel<1, ST_IBC><<<fin_blocks, 256, 0, st>>>(c0, c1, g, b, acc, plan->d_pf, tabs.t[ST_IBC], E.e[ST_IBC], fl);
        finalize_input_exec<1, ST_IBC><<<fin_blocks, 256, 0, st>>>(c0, c1, g, b, acc, plan->d_pf, fl);
        stage_params_kernel<<<pgrid, 128, 0, st>>>(acc, L.groups, ST_IBC, b.q[ST_IBC], E.e[ST_IBC], stage_depth(plan->mode, ST_IBC));
        prof_mark("input_base_change_max", st);
        if (pair) {
          using S2 = Staged2<LDs, 1>;
          auto kb = sin_b2_kernel<LDs>;
          const long long it2 = (g.T + S2::TPB - 1) / S2::TPB;
          sin_b2_kernel<LDs><<<staged_grid(kb, S2::THREADS, S2::SMEM_OUT, it2), S2::THREADS, S2::SMEM_OUT, st>>>(c0map, c0, c1, g, b, acc, plan->d_pf, tabs, fl);
        } else {
          auto kb = sin_b_kernel<LDs>;
          sin_b_kernel<LDs><<<staged_grid(kb, S::THREADS, S::SMEM_OUT, iters), S::THREADS, S::SMEM_OUT, st>>>(c0map, c0, c1, g, b, acc, plan->d_pf, tabs, fl);
        }
        fixup_ibc_kernel<<<fix_blocks, 128, 0, st>>>(fl, c0, c1, g, b, acc, plan->d_pf, tabs);
        finalize_input_kernel<1, ST_IT><<<fin_blocks, 256, 0, st>>>(c0, c1, g, b, acc, plan->d_pf, tabs.t[ST_IT], E.e[ST_IT], fl);
        finalize_input_exec<1, ST_IT><<<fin_blocks, 256, 0, st>>>(c0, c1, g, b, acc, plan->d_pf, fl);
        stage_params_kernel<<<pgrid, 128, 0, st>>>(acc, L.groups, ST_IT, b.q[ST_IT], E.e[ST_IT], stage_depth(plan->mode, ST_IT));
        prof_mark("input_transform_max", st);
        if (staged_c && pair) {
          using S2 = Staged2<LDs, 1>;
          auto kc = sin_c2_kernel<LDs>;
          const long long it2 = (g.T + S2::TPB - 1) / S2::TPB;
          sin_c2_kernel<LDs><<<staged_grid(kc, S2::THREADS, S2::SMEM_OUT, it2), S2::THREADS, S2::SMEM_OUT, st>>>(c0map, c0, c1, V, g, b, acc, plan->d_pf, fl);
        } else if (staged_c) {
          auto kc = sin_c_kernel<1, LDs>;
          sin_c_kernel<1, LDs><<<staged_grid(kc, S::THREADS, S::SMEM_OUT, iters), S::THREADS, S::SMEM_OUT, st>>>(c0map, c0, c1, V, g, b, acc, plan->d_pf, fl);
        } else
        in_c_kernel<1, LD><<<tgrid, tb, 0, st>>>(c0, c1, V, g, b, acc, plan->d_pf, fl);
        fixup_it_kernel<1><<<fix_blocks, 128, 0, st>>>(fl, c0, c1, V, g, b, acc, plan->d_pf);
        prof_mark("input_transform_codes", st);
      }
    } else {
      if (!leg) {
        in_a_kernel<0, LD><<<tgrid, tb, 0, st>>>(c0, g, acc, tabs);
        finalize_input_kernel<0, ST_IT><<<fin_blocks, 256, 0, st>>>(c0, c1, g, b, acc, plan->d_pf, tabs.t[ST_IT], E.e[ST_IT], fl);
        finalize_input_exec<0, ST_IT><<<fin_blocks, 256, 0, st>>>(c0, c1, g, b, acc, plan->d_pf, fl);
        stage_params_kernel<<<pgrid, 128, 0, st>>>(acc, L.groups, ST_IT, b.q[ST_IT], E.e[ST_IT], stage_depth(plan->mode, ST_IT));
        prof_mark("input_transform_max", st);
        in_c_kernel<0, LD><<<tgrid, tb, 0, st>>>(c0, c1, V, g, b, acc, plan->d_pf, fl);
        fixup_it_kernel<0><<<fix_blocks, 128, 0, st>>>(fl, c0, c1, V, g, b, acc, plan->d_pf);
        prof_mark("input_transform_codes", st);
      } else {
        in_a_kernel<1, LD><<<tgrid, tb, 0, st>>>(c0, g, acc, tabs);
        finalize_input_kernel<1, ST_IBC><<<fin_blocks, 256, 0, st>>>(c0, c1, g, b, acc, plan->d_pf, tabs.t[ST_IBC], E.e[ST_IBC], fl);
        finalize_input_exec<1, ST_IBC><<<fin_blocks, 256, 0, st>>>(c0, c1, g, b, acc, plan->d_pf, fl);
        stage_params_kernel<<<pgrid, 128, 0, st>>>(acc, L.groups, ST_IBC, b.q[ST_IBC], E.e[ST_IBC], stage_depth(plan->mode, ST_IBC));
        prof_mark("input_base_change_max", st);
        in_b_kernel<LD><<<tgrid, tb, 0, st>>>(c0, c1, g, b, acc, plan->d_pf, tabs, fl);
        fixup_ibc_kernel<<<fix_blocks, 128, 0, st>>>(fl, c0, c1, g, b, acc, plan->d_pf, tabs);
        finalize_input_kernel<1, ST_IT><<<fin_blocks, 256, 0, st>>>(c0, c1, g, b, acc, plan->d_pf, tabs.t[ST_IT], E.e[ST_IT], fl);
        finalize_input_exec<1, ST_IT><<<fin_blocks, 256, 0, st>>>(c0, c1, g, b, acc, plan->d_pf, fl);
        stage_params_kernel<<<pgrid, 128, 0, st>>>(acc, L.groups, ST_IT, b.q[ST_IT], E.e[ST_IT], stage_depth(plan->mode, ST_IT));
        prof_mark("input_transform_max", st);
        in_c_kernel<1, LD><<<tgrid, tb, 0, st>>>(c0, c1, V, g, b, acc, plan->d_pf, fl);
        fixup_it_kernel<1><<<fix_blocks, 128, 0, st>>>(fl, c0, c1, V, g, b, acc, plan->d_pf);
        prof_mark("input_transform_codes", st);
      }
    }
  });
  if (rc) return rc;
  WL_CUDA(cudaGetLastError());
  // padded channels of V must be zero for the GEMM: the stage kernels only write c < C
  if (g.Cp != g.C) WL_CUDA(cudaMemset2DAsync(V + g.C, g.Cp, 0, g.Cp - g.C, (size_t)36 * g.T, st));  // [T*36][Cp]

  int bn, sw;
  gemm_tiles(g, &bn, &sw);
  CUtensorMap ta, tbm;
  if (!make_tmap_i8_3d(&ta, V, g.Cp, 36, g.T, sw, 1, 128) || !make_tmap_i8_3d(&tbm, U, g.Cp, 36, g.Kp, sw, 1, bn))
    return fail(WL_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  const int wstage = leg ? ST_WBC : ST_WT;
  const int qu = b.q[wstage];
  {
    EpiHadMax e;
    e.acc = acc;
    e.table = tabs.t[ST_HAD];
    e.g = g;
    e.nchunk = g.Kp / L.bn;
    rc = dispatch_gemm(ta, tbm, g, bn, sw, e, st);
    if (rc) return rc;
    finalize_hadamard_kernel<<<fin_blocks, 256, 0, st>>>(U, V, g, acc, wh->wacc, wstage, qu, b.q[ST_IT],
                                                         tabs.t[ST_HAD], L.bn);
    stage_params_kernel<<<pgrid, 128, 0, st>>>(acc, L.groups, ST_HAD, b.q[ST_HAD], 0.f, 0.f);
    prof_mark("gemm_hadamard_max", st);
  }
  if (L.hbytes == 1) {
    EpiHadRq<int8_t> e;
    e.acc = acc;
    e.wacc = wh->wacc;
    e.U = U;
    e.V = V;
    e.h = reinterpret_cast<int8_t*>(h);
    e.g = g;
    e.fl = fl;
    e.wstage = wstage;
    e.qmax_u = qu;
    e.qmax_v = b.q[ST_IT];
    e.qmax_h = b.q[ST_HAD];
    rc = dispatch_gemm(ta, tbm, g, bn, sw, e, st);
    if (!rc)
      fixup_had_kernel<int8_t><<<fix_blocks, 128, 0, st>>>(fl, U, V, reinterpret_cast<int8_t*>(h), g, acc, wh->wacc, wstage,
                                                          qu, b.q[ST_IT], b.q[ST_HAD]);
  } else {
    EpiHadRq<int16_t> e;
    e.acc = acc;
    e.wacc = wh->wacc;
    e.U = U;
    e.V = V;
    e.h = reinterpret_cast<int16_t*>(h);
    e.g = g;
    e.fl = fl;
    e.wstage = wstage;
    e.qmax_u = qu;
    e.qmax_v = b.q[ST_IT];
    e.qmax_h = b.q[ST_HAD];
    rc = dispatch_gemm(ta, tbm, g, bn, sw, e, st);
    if (!rc)
      fixup_had_kernel<int16_t><<<fix_blocks, 128, 0, st>>>(fl, U, V, reinterpret_cast<int16_t*>(h), g, acc, wh->wacc, wstage,
                                                          qu, b.q[ST_IT], b.q[ST_HAD]);
  }
  if (rc) return rc;
  prof_mark("gemm_hadamard_codes", st);

  const long long oc = (long long)g.T * g.K;
  const unsigned ogrid = (unsigned)((oc + tb - 1) / tb);
  float* otab = sizeof(YT) == 4 && q->output_transform_bits <= 12 ? reinterpret_cast<float*>(ws + L.off_otab) : nullptr;
  auto make_otab = [&]() {
    if (!otab) return;
    const long long n = (long long)L.groups * (2 * b.q[ST_OUT] + 1);
    out_table_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(acc, L.groups, b.q[ST_OUT], otab);
  };
  // output code pass: the staged kernel (coalesced y rows) for fp32 outputs, else the plain grid
  const bool staged_oc = sizeof(YT) == 4 && !getenv("WL_PLAIN_OUT_C");
  auto out_codes = [&](auto mode_c, auto ht, auto plain) -> int {
    constexpr int MODE = decltype(mode_c)::value;
    using HT = decltype(ht);
    const HT* hh = reinterpret_cast<const HT*>(h);
    if constexpr (sizeof(YT) == 4) {
      if (staged_oc) {
        using STT = std::conditional_t<MODE == 0, HT, int8_t>;
        CUtensorMap om;
        const void* src = MODE == 0 ? (const void*)hh : (const void*)c4;
        if (!make_tmap_3d_plain(&om, src, (int)sizeof(STT), (uint64_t)g.Kp, 36, (uint64_t)g.T, StagedOut::KB, 36,
                                StagedOut::TPB))
          return fail(WL_ERR_CUDA, "cuTensorMapEncodeTiled (output codes) failed");
        constexpr int smem = StagedOut::smem<STT>();
        const long long iters = (long long)((g.T + StagedOut::TPB - 1) / StagedOut::TPB) * ((g.K + StagedOut::KB - 1) / StagedOut::KB);
        auto launch = [&](auto tabc) {
          constexpr bool TAB = decltype(tabc)::value;
          auto kern = sout_c_kernel<MODE, HT, TAB>;
          sout_c_kernel<MODE, HT, TAB><<<staged_grid(kern, StagedOut::THREADS, smem, iters), StagedOut::THREADS, smem,
                                         st>>>(om, hh, c4, reinterpret_cast<float*>(y),
                                               reinterpret_cast<const float*>(bias), g, b, acc, plan->d_pf, otab, fl);
        };
        if (otab)
          launch(std::true_type{});
        else
          launch(std::false_type{});
        return 0;
      }
    }
    plain();
    return 0;
  };
  int oc_rc = 0;
  auto run_out = [&](auto ldc, auto ht) {
    constexpr int LD = decltype(ldc)::value;
    using HT = decltype(ht);
    const HT* hh = reinterpret_cast<const HT*>(h);
    if (LD <= 256 && staged_out) {
      constexpr int LDs = LD <= 256 ? LD : 256;
      using SH = Staged<LDs, sizeof(HT)>;
      const long long iters = (g.T + SH::TPB - 1) / SH::TPB;
      if (!leg) {
        auto ka = sout_a_kernel<0, HT, LDs>;
        sout_a_kernel<0, HT, LDs><<<staged_grid(ka, SH::THREADS, SH::SMEM, iters), SH::THREADS, SH::SMEM, st>>>(hh, g, acc, tabs);
        finalize_output_kernel<0, ST_OUT, HT><<<fin_blocks, 256, 0, st>>>(hh, c4, g, b, acc, plan->d_pf, tabs.t[ST_OUT], E.e[ST_OUT], fl);
        finalize_output_exec<0, ST_OUT, HT><<<fin_blocks, 256, 0, st>>>(hh, c4, g, b, acc, plan->d_pf, fl);
        stage_params_kernel<<<pgrid, 128, 0, st>>>(acc, L.groups, ST_OUT, b.q[ST_OUT], E.e[ST_OUT], stage_depth(plan->mode, ST_OUT));
        prof_mark("output_max", st);
        make_otab();
        oc_rc = out_codes(IntC<0>{}, HT{}, [&] { out_c_kernel<0, HT, LD, YT><<<ogrid, tb, 0, st>>>(hh, c4, y, bias, g, b, acc, plan->d_pf, otab, fl); });
        fixup_out_kernel<0, HT, YT><<<fix_blocks, 128, 0, st>>>(fl, hh, c4, y, bias, g, b, acc, plan->d_pf);
        prof_mark("output_write", st);
      } else {
        if (pair) {
          using S2 = Staged2<LDs, sizeof(HT)>;
          auto ka = sout_a2_kernel<1, HT, LDs>;
          const long long it2 = (g.T + S2::TPB - 1) / S2::TPB;
          sout_a2_kernel<1, HT, LDs><<<staged_grid(ka, S2::THREADS, S2::SMEM, it2), S2::THREADS, S2::SMEM, st>>>(hh, g, acc, tabs);
        } else {
          auto ka = sout_a_kernel<1, HT, LDs>;
          sout_a_kernel<1, HT, LDs><<<staged_grid(ka, SH::THREADS, SH::SMEM, iters), SH::THREADS, SH::SMEM, st>>>(hh, g, acc, tabs);
        }
        finalize_output_kernel<1, ST_OBC, HT><<<fin_blocks, 256, 0, st>>>(hh, c4, g, b, acc, plan->d_pf, tabs.t[ST_OBC], E.e[ST_OBC], fl);
        finalize_output_exec<1, ST_OBC, HT><<<fin_blocks, 256, 0, st>>>(hh, c4, g, b, acc, plan->d_pf, fl);
        stage_params_kernel<<<pgrid, 128, 0, st>>>(acc, L.groups, ST_OBC, b.q[ST_OBC], E.e[ST_OBC], stage_depth(plan->mode, ST_OBC));
        prof_mark("output_base_change_max", st);
        if (t4path) {
          // T4 path: the output stage's fp32 values + error factors are stored instead of c4
          if (pair) {
            using ST42 = StagedT42<LDs, sizeof(HT)>;
            auto kbt = sout_bt2_kernel<HT, LDs>;
            const long long it2 = (g.T + ST42::TPB - 1) / ST42::TPB;
            sout_bt2_kernel<HT, LDs><<<staged_grid(kbt, ST42::THREADS, ST42::SMEM, it2), ST42::THREADS, ST42::SMEM, st>>>(
                hh, t4, e4, g, b, acc, plan->d_pf, tabs, fl);
          } else {
            using ST4 = StagedT4<LDs, sizeof(HT)>;
            auto kbt = sout_bt_kernel<HT, LDs>;
            sout_bt_kernel<HT, LDs><<<staged_grid(kbt, ST4::THREADS, ST4::SMEM, iters), ST4::THREADS, ST4::SMEM, st>>>(
                hh, t4, e4, g, b, acc, plan->d_pf, tabs, fl);
          }
          fixup_obct_kernel<HT><<<fix_blocks, 128, 0, st>>>(fl, hh, t4, e4, g, b, acc, plan->d_pf, tabs);
          finalize_output_kernel<1, ST_OUT, HT, true><<<fin_blocks, 256, 0, st>>>(hh, c4, g, b, acc, plan->d_pf, tabs.t[ST_OUT], E.e[ST_OUT], fl);
        finalize_output_exec<1, ST_OUT, HT, true><<<fin_blocks, 256, 0, st>>>(hh, c4, g, b, acc, plan->d_pf, fl);
          stage_params_kernel<<<pgrid, 128, 0, st>>>(acc, L.groups, ST_OUT, b.q[ST_OUT], E.e[ST_OUT], stage_depth(plan->mode, ST_OUT));
          prof_mark("output_max", st);
          make_otab();
          if (sizeof(YT) == 4) {
            CUtensorMap tm4, em4;
            if (!make_tmap_3d_plain(&tm4, t4, 4, (uint64_t)g.Kp, 16, (uint64_t)g.T, StagedOut::KB, 16, StagedOut::TPB) ||
                !make_tmap_3d_plain(&em4, e4, 4, (uint64_t)g.Kp, 1, (uint64_t)g.T, StagedOut::KB, 1, StagedOut::TPB)) {
              oc_rc = fail(WL_ERR_CUDA, "cuTensorMapEncodeTiled (T4) failed");
              return;
            }
            // 2-deep input ring at 4 CTAs/SM; WL_CT_NS3=1 selects a 3-deep ring at 3 CTAs/SM (measured
            // slower on config 4: 2.23 vs 1.78 ms — fewer resident warps to drain the y stores)
            const bool ns2 = getenv("WL_CT_NS3") == nullptr;
            const int smem = (ns2 ? 2 : 3) * (StagedOut::TPB * 17 * StagedOut::KB * 4) + StagedOut::OUT_BYTES + 32;
            const long long oiters = (long long)((g.T + StagedOut::TPB - 1) / StagedOut::TPB) * ((g.K + StagedOut::KB - 1) / StagedOut::KB);
            auto launch = [&](auto tabc) {
              constexpr bool TAB = decltype(tabc)::value;
              if (ns2) {
                auto kern = sout_ct_kernel<HT, TAB, 2>;
                kern<<<staged_grid(kern, StagedOut::THREADS, smem, oiters), StagedOut::THREADS, smem, st>>>(
                    tm4, em4, hh, reinterpret_cast<float*>(y), reinterpret_cast<const float*>(bias), g, b, acc, plan->d_pf,
                    otab, fl);
              } else {
                auto kern = sout_ct_kernel<HT, TAB, 3>;
                kern<<<staged_grid(kern, StagedOut::THREADS, smem, oiters), StagedOut::THREADS, smem, st>>>(
                    tm4, em4, hh, reinterpret_cast<float*>(y), reinterpret_cast<const float*>(bias), g, b, acc, plan->d_pf,
                    otab, fl);
              }
            };
            if (otab)
              launch(std::true_type{});
            else
              launch(std::false_type{});
            fixup_outt_kernel<HT><<<fix_blocks, 128, 0, st>>>(fl, hh, reinterpret_cast<float*>(y),
                                                              reinterpret_cast<const float*>(bias), g, b, acc, plan->d_pf);
          }
          prof_mark("output_write", st);
          return;
        }
        auto kb = sout_b_kernel<HT, LDs>;
        sout_b_kernel<HT, LDs><<<staged_grid(kb, SH::THREADS, SH::SMEM_OUT, iters), SH::THREADS, SH::SMEM_OUT, st>>>(hh, c4, g, b, acc, plan->d_pf, tabs, fl);
        fixup_obc_kernel<HT><<<fix_blocks, 128, 0, st>>>(fl, hh, c4, g, b, acc, plan->d_pf, tabs);
        finalize_output_kernel<1, ST_OUT, HT><<<fin_blocks, 256, 0, st>>>(hh, c4, g, b, acc, plan->d_pf, tabs.t[ST_OUT], E.e[ST_OUT], fl);
        finalize_output_exec<1, ST_OUT, HT><<<fin_blocks, 256, 0, st>>>(hh, c4, g, b, acc, plan->d_pf, fl);
        stage_params_kernel<<<pgrid, 128, 0, st>>>(acc, L.groups, ST_OUT, b.q[ST_OUT], E.e[ST_OUT], stage_depth(plan->mode, ST_OUT));
        prof_mark("output_max", st);
        make_otab();
        oc_rc = out_codes(IntC<1>{}, HT{}, [&] { out_c_kernel<1, HT, LD, YT><<<ogrid, tb, 0, st>>>(hh, c4, y, bias, g, b, acc, plan->d_pf, otab, fl); });
        fixup_out_kernel<1, HT, YT><<<fix_blocks, 128, 0, st>>>(fl, hh, c4, y, bias, g, b, acc, plan->d_pf);
        prof_mark("output_write", st);
      }
    } else {
      if (!leg) {
        out_a_kernel<0, HT, LD><<<ogrid, tb, 0, st>>>(hh, g, acc, tabs);
        finalize_output_kernel<0, ST_OUT, HT><<<fin_blocks, 256, 0, st>>>(hh, c4, g, b, acc, plan->d_pf, tabs.t[ST_OUT], E.e[ST_OUT], fl);
        finalize_output_exec<0, ST_OUT, HT><<<fin_blocks, 256, 0, st>>>(hh, c4, g, b, acc, plan->d_pf, fl);
        stage_params_kernel<<<pgrid, 128, 0, st>>>(acc, L.groups, ST_OUT, b.q[ST_OUT], E.e[ST_OUT], stage_depth(plan->mode, ST_OUT));
        prof_mark("output_max", st);
        make_otab();
        oc_rc = out_codes(IntC<0>{}, HT{}, [&] { out_c_kernel<0, HT, LD, YT><<<ogrid, tb, 0, st>>>(hh, c4, y, bias, g, b, acc, plan->d_pf, otab, fl); });
        fixup_out_kernel<0, HT, YT><<<fix_blocks, 128, 0, st>>>(fl, hh, c4, y, bias, g, b, acc, plan->d_pf);
        prof_mark("output_write", st);
      } else {
        out_a_kernel<1, HT, LD><<<ogrid, tb, 0, st>>>(hh, g, acc, tabs);
        finalize_output_kernel<1, ST_OBC, HT><<<fin_blocks, 256, 0, st>>>(hh, c4, g, b, acc, plan->d_pf, tabs.t[ST_OBC], E.e[ST_OBC], fl);
        finalize_output_exec<1, ST_OBC, HT><<<fin_blocks, 256, 0, st>>>(hh, c4, g, b, acc, plan->d_pf, fl);
        stage_params_kernel<<<pgrid, 128, 0, st>>>(acc, L.groups, ST_OBC, b.q[ST_OBC], E.e[ST_OBC], stage_depth(plan->mode, ST_OBC));
        prof_mark("output_base_change_max", st);
        out_b_kernel<HT, LD><<<ogrid, tb, 0, st>>>(hh, c4, g, b, acc, plan->d_pf, tabs, fl);
        fixup_obc_kernel<HT><<<fix_blocks, 128, 0, st>>>(fl, hh, c4, g, b, acc, plan->d_pf, tabs);
        finalize_output_kernel<1, ST_OUT, HT><<<fin_blocks, 256, 0, st>>>(hh, c4, g, b, acc, plan->d_pf, tabs.t[ST_OUT], E.e[ST_OUT], fl);
        finalize_output_exec<1, ST_OUT, HT><<<fin_blocks, 256, 0, st>>>(hh, c4, g, b, acc, plan->d_pf, fl);
        stage_params_kernel<<<pgrid, 128, 0, st>>>(acc, L.groups, ST_OUT, b.q[ST_OUT], E.e[ST_OUT], stage_depth(plan->mode, ST_OUT));
        prof_mark("output_max", st);
        make_otab();
        oc_rc = out_codes(IntC<1>{}, HT{}, [&] { out_c_kernel<1, HT, LD, YT><<<ogrid, tb, 0, st>>>(hh, c4, y, bias, g, b, acc, plan->d_pf, otab, fl); });
        fixup_out_kernel<1, HT, YT><<<fix_blocks, 128, 0, st>>>(fl, hh, c4, y, bias, g, b, acc, plan->d_pf);
        prof_mark("output_write", st);
      }
    }
  };
  rc = dispatch_ld_out(g.Kp, [&](auto ldc) {
    if (L.hbytes == 1)
      run_out(ldc, int8_t{});
    else
      run_out(ldc, int16_t{});
  });
  if (rc) return rc;
  if (oc_rc) return oc_rc;

  WL_CUDA(cudaGetLastError());
  if (g_debug_fail) return fail(WL_ERR_CUDA, "kernel group '%s' failed: %s", g_debug_fail,
                                cudaGetErrorString(cudaGetLastError()));
  if (getenv("WL_FIX_STATS")) {  // debug: deferred-fix list lengths (IBC, IT, OBC, OUT, HAD) of this call
    unsigned cnt[kFixLists];
    WL_CUDA(cudaMemcpyAsync(cnt, fl.count, sizeof(cnt), cudaMemcpyDeviceToHost, st));
    WL_CUDA(cudaStreamSynchronize(st));
    const double units_in = (double)g.T * g.C, units_out = (double)g.T * g.K;
    fprintf(stderr, "wl fix lists: ibc %u (%.3f%%) it %u (%.3f%%) obc %u (%.3f%%) out %u (%.3f%%) hadamard ties %u cap %u\n",
            cnt[0], 100.0 * cnt[0] / units_in, cnt[1], 100.0 * cnt[1] / units_in, cnt[2], 100.0 * cnt[2] / units_out,
            cnt[3], 100.0 * cnt[3] / units_out, cnt[FIX_HAD], fl.cap);
  }
  return WL_OK;
}

extern "C" {

int wl_forward(const wl_plan* plan, const wl_qcfg* q, const wl_shape* s, const float* x, const void* cache,
               const float* bias, float* y, void* workspace, size_t workspace_bytes, void* stream) {
  return forward_impl(plan, q, s, x, cache, bias, y, workspace, workspace_bytes, stream);
}

int wl_forward_f64(const wl_plan* plan, const wl_qcfg* q, const wl_shape* s, const double* x, const void* cache,
                   const double* bias, double* y, void* workspace, size_t workspace_bytes, void* stream) {
  return forward_impl(plan, q, s, x, cache, bias, y, workspace, workspace_bytes, stream);
}

static BwGeo bw_geo(const Layout& L) {
  const Geo& g = L.g;
  return BwGeo{g.N, g.C, g.K, g.H, g.W, g.pad, g.Ho, g.Wo, g.th, g.tw, g.TP, g.T, g.Cp, g.Kp, g.ipg, L.groups};
}

int wl_backward_workspace_size(const wl_plan* plan, const wl_shape* s, const wl_qcfg* q, size_t* bytes) {
  if (!plan || !bytes) return fail(WL_ERR_ARG, "NULL argument");
  int rc = check_bits(q);
  if (rc) return rc;
  Layout L;
  rc = make_layout(s, q, &L);
  if (rc) return rc;
  *bytes = wl_bw_workspace_bytes(bw_geo(L));
  return WL_OK;
}

int wl_backward(const wl_plan* plan, const wl_qcfg* q, const wl_shape* s, const float* dy, const void* cache,
                const void* fwd_workspace, float* dx, float* dw, float* db, void* workspace, size_t workspace_bytes,
                void* stream) {
  if (!plan || !dy || !cache || !fwd_workspace || !dx || !dw || !workspace) return fail(WL_ERR_ARG, "NULL argument");
  int rc = check_bits(q);
  if (rc) return rc;
  Layout L;
  rc = make_layout(s, q, &L);
  if (rc) return rc;
  const BwGeo bg = bw_geo(L);
  if (workspace_bytes < wl_bw_workspace_bytes(bg)) return fail(WL_ERR_WORKSPACE, "backward workspace too small");
  const uint8_t* fws = reinterpret_cast<const uint8_t*>(fwd_workspace);
  const WeightHeader* wh = reinterpret_cast<const WeightHeader*>(cache);
  const int8_t* U = reinterpret_cast<const int8_t*>(cache) + align256(sizeof(WeightHeader));
  const Bits b = make_bits(q);
  const int wstage = plan->mode == WL_LEGENDRE ? ST_WBC : ST_WT;
  std::string err;
  rc = wl_bw_run(bg, dy, U, wh->wacc, wstage, b.q[wstage], reinterpret_cast<const int8_t*>(fws + L.off_v),
                 reinterpret_cast<const Acc*>(fws + L.off_acc), dx, dw, db, workspace, (cudaStream_t)stream, &err);
  if (rc) return fail(rc, "backward: %s", err.c_str());
  return WL_OK;
}

int wl_read_stats(const wl_plan* plan, const wl_shape* s, const wl_qcfg* q, const void* cache, const void* workspace,
                  wl_stage_stat* out, void* stream) {
  if (!plan || !cache || !workspace || !out) return fail(WL_ERR_ARG, "NULL argument");
  int rc = check_bits(q);
  if (rc) return rc;
  Layout L;
  rc = make_layout(s, q, &L);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<Acc> acc((size_t)L.groups * ST_COUNT);
  WeightHeader wh;
  WL_CUDA(cudaMemcpyAsync(acc.data(), reinterpret_cast<const uint8_t*>(workspace) + L.off_acc,
                          acc.size() * sizeof(Acc), cudaMemcpyDeviceToHost, st));
  WL_CUDA(cudaMemcpyAsync(&wh, cache, sizeof(wh), cudaMemcpyDeviceToHost, st));
  WL_CUDA(cudaStreamSynchronize(st));
  const bool leg = plan->mode == WL_LEGENDRE;
  const int ns = leg ? 9 : 6;
  const int* order = leg ? kLegOrder : kCanonOrder;
  for (int gi = 0; gi < L.groups; ++gi)
    for (int i = 0; i < ns; ++i) {
      const int stg = order[i];
      const bool wside = stg == ST_WEIGHTS || stg == ST_WT || stg == ST_WBC;
      const Acc& a = wside ? wh.wacc[stg] : acc[(size_t)gi * ST_COUNT + stg];
      const int bits = wside ? stage_bits(&wh.q, stg) : stage_bits(q, stg);
      double mx;
      if (stg == ST_INPUT || stg == ST_WEIGHTS) {
        long long mb = (long long)a.M;  // fp64 bits of max |x| (exact for fp32 and fp64 operands)
        memcpy(&mx, &mb, 8);
      } else {
        long long fb = (long long)a.F;
        memcpy(&mx, &fb, 8);
      }
      const int qmax = (1 << (bits - 1)) - 1;
      wl_stage_stat& o = out[(size_t)gi * ns + i];
      o.bits = bits;
      o.max_abs = mx;
      o.scale = mx > 0.0 ? mx / (double)qmax : 1.0;
    }
  return WL_OK;
}

}  // extern "C"
