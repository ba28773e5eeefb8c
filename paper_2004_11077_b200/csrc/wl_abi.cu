// C-ABI entry points of libwinoleg_b200.so (include/winoleg_b200.h) and the host helpers shared by
// the forward translation units (wl_internal.h).  See DESIGN.md for the pass structure.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "wl_backward.h"
#include "wl_direct.h"
#include "wl_float.h"
#include "wl_gemm_bf16.h"
#include "wl_internal.h"

namespace wl {

namespace {
thread_local std::string g_err;
}

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}
const char* last_error() { return g_err.c_str(); }

const int kTableStage[kNumTables] = {ST_IBC, ST_IT, ST_HAD, ST_OBC, ST_OUT};
unsigned g_fix_cap_override = 0;

// ------------------------------------------------------------------ per-device launch helpers
namespace {
int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}
}  // namespace

int num_sms() {
  static std::mutex mu;
  static std::map<int, int> sms;
  const int dev = current_device();
  std::lock_guard<std::mutex> lock(mu);
  auto it = sms.find(dev);
  if (it != sms.end()) return it->second;
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  if (n <= 0) n = 148;
  sms[dev] = n;
  return n;
}

cudaError_t ensure_smem_attr(const void* kern, int smem) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int>, int> done;  // (kernel, device) -> largest size set
  const int dev = current_device();
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_tuple(kern, dev);
  auto it = done.find(key);
  if (it != done.end() && it->second >= smem) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess) done[key] = smem;
  return e;
}

int staged_grid_impl(const void* kern, int threads, int smem, long long work_items) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, int>, int> occ;  // (kernel, smem, device) -> blocks / SM
  const int dev = current_device();
  ensure_smem_attr(kern, smem);
  int per_sm = 0;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto key = std::make_tuple(kern, smem, dev);
    auto it = occ.find(key);
    if (it != occ.end()) {
      per_sm = it->second;
    } else {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
      if (per_sm < 1) per_sm = 1;
      occ[key] = per_sm;
    }
  }
  return (int)std::max(1LL, std::min<long long>(work_items, (long long)per_sm * num_sms()));
}

// ------------------------------------------------------------------ tensor-map cache
namespace {
struct TmapKey {
  int kind, elem;
  const void* base;
  uint64_t d[4];
  uint32_t b[3];
  bool operator<(const TmapKey& o) const { return memcmp(this, &o, sizeof(TmapKey)) < 0; }
};
struct TmapCache {
  std::mutex mu;
  std::map<TmapKey, CUtensorMap> m;
};
TmapCache& tcache() {
  static TmapCache c;
  return c;
}
template <class F>
bool cached(const TmapKey& k, CUtensorMap* out, F&& make) {
  TmapCache& c = tcache();
  {
    std::lock_guard<std::mutex> lock(c.mu);
    auto it = c.m.find(k);
    if (it != c.m.end()) {
      *out = it->second;
      return true;
    }
  }
  if (!make(out)) return false;
  std::lock_guard<std::mutex> lock(c.mu);
  if (c.m.size() > 256) c.m.clear();  // bounded: workspaces are few and long-lived
  c.m[k] = *out;
  return true;
}
TmapKey key_of(int kind, int elem, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t d3, uint32_t b0,
               uint32_t b1, uint32_t b2) {
  TmapKey k;
  memset(&k, 0, sizeof(k));
  k.kind = kind;
  k.elem = elem;
  k.base = base;
  k.d[0] = d0, k.d[1] = d1, k.d[2] = d2, k.d[3] = d3;
  k.b[0] = b0, k.b[1] = b1, k.b[2] = b2;
  return k;
}
}  // namespace

bool tmap_i8_3d(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t b0, uint32_t b1,
                uint32_t b2) {
  return cached(key_of(0, 1, base, d0, d1, d2, 0, b0, b1, b2), m,
                [&](CUtensorMap* o) { return make_tmap_i8_3d(o, base, d0, d1, d2, b0, b1, b2); });
}
bool tmap_i8_4d(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t d3, uint32_t b0,
                uint32_t b1, uint32_t b2) {
  return cached(key_of(1, 1, base, d0, d1, d2, d3, b0, b1, b2), m,
                [&](CUtensorMap* o) { return make_tmap_i8_4d(o, base, d0, d1, d2, d3, b0, b1, b2); });
}
bool tmap_3d_plain(CUtensorMap* m, const void* base, int elem_bytes, uint64_t d0, uint64_t d1, uint64_t d2,
                   uint32_t b0, uint32_t b1, uint32_t b2) {
  return cached(key_of(2, elem_bytes, base, d0, d1, d2, 0, b0, b1, b2), m,
                [&](CUtensorMap* o) { return make_tmap_3d_plain(o, base, elem_bytes, d0, d1, d2, b0, b1, b2); });
}

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
}  // namespace

const char* g_debug_fail = nullptr;

bool debug_sync_enabled() {
  // WL_DEBUG_SYNC=1 (read once): synchronise after every kernel group and report the first failing one
  static const bool v = [] {
    const char* e = getenv("WL_DEBUG_SYNC");
    return e && e[0] == '1';
  }();
  return v;
}

void prof_begin() {
  if (!g_prof.on) return;
  g_prof.calls.emplace_back();
  g_prof.cur = &g_prof.calls.back();
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

// ------------------------------------------------------------------ stage-width plumbing

int check_bits(const wl_qcfg* q) {
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

Bits make_bits(const wl_qcfg* q) {
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

int stage_bits(const wl_qcfg* q, int st) {
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

// ------------------------------------------------------------------ geometry / workspace

FastDiv make_fastdiv(unsigned d) {
  FastDiv f;
  f.d = d;
  f.s = 0;
  while ((1ull << f.s) < d) ++f.s;
  f.m = (unsigned)((((1ull << 32) * ((1ull << f.s) - d)) / d) + 1);
  return f;
}

int make_layout(const wl_shape* s, const wl_qcfg* q, Layout* L, bool split) {
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
  g.lazy = (g.N / g.ipg) < 16 ? 1 : 0;
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
  // saved block: [acc][cast tickets][V]
  size_t o = 0;
  L->off_acc = o;
  o = align256(o + sizeof(Acc) * ST_COUNT * L->groups);
  L->off_sync = o;  // fused input cast: block ticket + one arrival counter per group
  o = align256(o + sizeof(unsigned) * ((size_t)L->groups + 1));
  L->off_v = o;
  o = align256(o + (size_t)36 * g.T * g.Cp);
  L->saved_total = o;
  if (split) o = 0;
  L->off_c0 = o;
  o = align256(o + (size_t)g.N * g.H * g.W * g.Cp);
  L->off_h = o;
  o = align256(o + (size_t)36 * g.T * g.Kp * L->hbytes);
  L->off_c1 = o;
  o = align256(o + (size_t)36 * g.T * g.Cp);
  L->off_c4 = o;
  o = align256(o + (size_t)36 * g.T * g.Kp);
  // Legendre fp32-output path: output-stage fast-path values + error factors, T4E [Kp/4][T][17][4]
  L->off_t4 = o;  // T4E [Kp/4][T][17][4] floats
  o = align256(o + (size_t)17 * g.T * g.Kp * sizeof(float));
  L->off_e4 = o;
  L->bn = (g.Kp >= 256 ? 256 : g.Kp) / 4;  // table chunk = one max-pass epilogue warp's columns (EpiHadMax::kGroups)
  const size_t CB = (g.C + 31) / 32, KB = (g.K + 31) / 32;
  const size_t ents[kNumTables] = {g.T * CB, g.T * CB, (size_t)36 * g.T * (g.Kp / L->bn), g.T * KB, g.T * KB};
  // the four transform-stage tables and the fix-list counters are zeroed by one memset per call: they are
  // laid out back to back ([IBC][IT][OBC][OUT][counters + items]); the Hadamard table (fully written by
  // the GEMM max epilogue) follows
  auto place_table = [&](int i) {
    L->off_tab[i] = o;
    L->tab_bytes[i] = ents[i] * sizeof(unsigned);
    o = align256(o + L->tab_bytes[i]);
  };
  for (int i = 0; i < kNumTables; ++i)
    if (kTableStage[i] != ST_HAD) place_table(i);
  // deferred-fix list: counters + unit ids (expected ~0.2% of units; overflow falls back inline)
  L->off_fix = o;
  const size_t units = (size_t)g.T * std::max(g.C, g.K);
  L->fix_cap = g_fix_cap_override ? g_fix_cap_override : (unsigned)std::max<size_t>(4096, units / 16);
  o = align256(o + kFixHeaderBytes + sizeof(unsigned) * (size_t)std::max<size_t>(L->fix_cap, 4096));
  for (int i = 0; i < kNumTables; ++i)
    if (kTableStage[i] == ST_HAD) place_table(i);
  // dequantised output table (output widths <= 12 bits; wider widths dequantise in fp64 inline)
  L->off_otab = o;
  if (q->output_transform_bits <= 12) o = align256(o + sizeof(float) * (size_t)L->groups * ((1 << q->output_transform_bits) - 1));
  L->off_odq = o;
  if (q->output_transform_bits <= 12) o = align256(o + sizeof(float4) * (size_t)L->groups);
  L->total = o;
  return WL_OK;
}

size_t weight_cache_bytes(int K, int C, int* Kp, int* Cp) {
  *Cp = pow2_at_least(C, 32);
  *Kp = pow2_at_least(K, 64);
  return align256(sizeof(WeightHeader)) + (size_t)36 * (*Kp) * (*Cp);
}

// fp32 second-half rounding depth of each transform stage (the fast path's certified band)
float stage_depth(int mode, int stage) {
  const bool leg = mode == WL_LEGENDRE;
  switch (stage) {
    case ST_IBC: return (float)chain_depth<tab::Leg_IBC>();
    case ST_IT: return leg ? (float)chain_depth<tab::Leg_IT>() : (float)chain_depth<tab::Can_IT>();
    case ST_OBC: return (float)chain_depth<tab::Leg_OBC>();
    case ST_OUT: return leg ? (float)chain_depth<tab::Leg_OT>() : (float)chain_depth<tab::Can_OT>();
    default: return 6.f;
  }
}

// Max row abs-sum of each stage's integer matrix: with the group's max |first-half value| it bounds
// the fp32 error of the second half (stage_error in wl_kernels2.cuh).
StageE stage_rowsums(int mode) {
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

}  // namespace wl

using namespace wl;

static const int kCanonOrder[6] = {ST_INPUT, ST_WEIGHTS, ST_WT, ST_IT, ST_HAD, ST_OUT};
static const int kLegOrder[9] = {ST_INPUT, ST_WEIGHTS, ST_WT, ST_WBC, ST_IBC, ST_IT, ST_HAD, ST_OBC, ST_OUT};

// ------------------------------------------------------------------ C ABI

extern "C" {

const char* wl_last_error(void) { return wl::last_error(); }

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

int wl_debug_gemm_bf16(const void* A, int PA, const void* B, int PB, int batch, int M, int N, int Kd, int ks,
                       float* D, int ldd, float alpha, void* stream) {
  if (!A || !B || !D) return fail(WL_ERR_ARG, "NULL argument");
  cudaError_t e = gemm_bf16_split(A, PA, B, PB, batch, M, N, Kd, ks, D, ldd, alpha, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(WL_ERR_CUDA, "gemm_bf16_split: %s", cudaGetErrorString(e));
  return WL_OK;
}

int wl_debug_set_fix_cap(unsigned cap) {
  g_fix_cap_override = cap;
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
  cudaGetDevice(&pl->device);
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

__global__ void init_weight_header_kernel(WeightHeader* dst, const WeightHeader h) {
  const uint32_t* src = reinterpret_cast<const uint32_t*>(&h);
  uint32_t* d = reinterpret_cast<uint32_t*>(dst);
  for (int i = threadIdx.x; i < (int)(sizeof(WeightHeader) / 4); i += blockDim.x) d[i] = src[i];
}

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
  // the header travels as a kernel argument (copied at launch): a cudaMemcpyAsync from this stack frame
  // would be recorded by address when the call is captured in a CUDA graph and replayed from dead memory
  init_weight_header_kernel<<<1, 32, 0, st>>>(dh, hdr);
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

static BwGeo bw_geo(const Layout& L) {
  const Geo& g = L.g;
  return BwGeo{g.N, g.C, g.K, g.H, g.W, g.pad, g.Ho, g.Wo, g.th, g.tw, g.TP, g.T, g.Cp, g.Kp, g.ipg, L.groups};
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

int wl_train_sizes(const wl_plan* plan, const wl_shape* s, const wl_qcfg* q, size_t* saved_bytes,
                   size_t* workspace_bytes) {
  if (!plan || !saved_bytes || !workspace_bytes) return fail(WL_ERR_ARG, "NULL argument");
  int rc = check_bits(q);
  if (rc) return rc;
  Layout L;
  rc = make_layout(s, q, &L, true);
  if (rc) return rc;
  *saved_bytes = L.saved_total;
  *workspace_bytes = L.total;
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
  // input cast (one fused launch, or absmax + quant), [in_a|in_b(+fixup), finalize, exec] x2|1, in_c, fixup,
  // gemm max, finalize, gemm codes, tie fixup, [out_a|out_b(+fixup), finalize, exec] x2|1, output table,
  // out_c, fixup
  // (the count assumes the fp32 entry point with a 16-byte aligned x for the fused cast)
  const int otab = (q && q->output_transform_bits <= 12) ? 1 : 0;
  const int ipg = s ? (s->images_per_group > 0 ? s->images_per_group : s->n) : 1;
  const int cast = s && cast_fusable_shape(s->c_in, s->h, s->w, ipg) ? 1 : 2;
  return (plan->mode == WL_LEGENDRE ? 22 : 14) + cast + otab;
}

int wl_forward(const wl_plan* plan, const wl_qcfg* q, const wl_shape* s, const float* x, const void* cache,
               const float* bias, float* y, void* workspace, size_t workspace_bytes, void* stream) {
  return forward_impl<float, float>(plan, q, s, x, cache, bias, y, nullptr, 0, workspace, workspace_bytes, stream);
}

int wl_forward_f64(const wl_plan* plan, const wl_qcfg* q, const wl_shape* s, const double* x, const void* cache,
                   const double* bias, double* y, void* workspace, size_t workspace_bytes, void* stream) {
  return forward_impl<double, double>(plan, q, s, x, cache, bias, y, nullptr, 0, workspace, workspace_bytes, stream);
}

int wl_forward_train(const wl_plan* plan, const wl_qcfg* q, const wl_shape* s, const float* x, const void* cache,
                     const float* bias, float* y, void* saved, size_t saved_bytes, void* workspace,
                     size_t workspace_bytes, void* stream) {
  if (!saved) return fail(WL_ERR_ARG, "NULL saved buffer");
  return forward_impl<float, float>(plan, q, s, x, cache, bias, y, saved, saved_bytes, workspace, workspace_bytes,
                                    stream);
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

// `saved` is the forward's saved block (wl_forward_train) or its whole workspace (wl_forward): both
// start with [acc][V] at the same offsets.
int wl_backward(const wl_plan* plan, const wl_qcfg* q, const wl_shape* s, const float* dy, const void* cache,
                const void* saved, float* dx, float* dw, float* db, void* workspace, size_t workspace_bytes,
                void* stream) {
  if (!plan || !dy || !cache || !saved || !dx || !dw || !workspace) return fail(WL_ERR_ARG, "NULL argument");
  int rc = check_bits(q);
  if (rc) return rc;
  Layout L;
  rc = make_layout(s, q, &L);
  if (rc) return rc;
  const BwGeo bg = bw_geo(L);
  if (workspace_bytes < wl_bw_workspace_bytes(bg)) return fail(WL_ERR_WORKSPACE, "backward workspace too small");
  const uint8_t* fws = reinterpret_cast<const uint8_t*>(saved);
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
