// Host-side internals shared by the translation units of libwinoleg_b200.so:
//   wl_abi.cu        C ABI (plan, workspace, weight transform, stats, backward / float / direct glue)
//   wl_fwd.cu        forward orchestration (input cast, stage finalizes, dependency chain)
//   wl_fwd_gemm.cu   tcgen05 Hadamard passes (max / requantisation epilogues, tie fixups)
//   wl_fwd_in_*.cu   input-side transform passes, one TU per padded channel count (wl_fwd_in.inc)
//   wl_fwd_out_*.cu  output-side transform passes, one TU per padded output-channel count (wl_fwd_out.inc)
// Splitting the forward by channel count lets `make -j` compile the kernel instantiations in parallel.
#pragma once
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstddef>
#include <cstdint>
#include <string>

#include "../../include/winoleg_b200.h"
#include "wl_kernels2.cuh"
#include "wl_tmap.h"

namespace wl {

int fail(int code, const char* fmt, ...);
const char* last_error();

#define WL_CUDA(expr)                                                                              \
  do {                                                                                             \
    cudaError_t e_ = (expr);                                                                       \
    if (e_ != cudaSuccess) return ::wl::fail(WL_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)

inline size_t align256(size_t v) { return (v + 255) & ~size_t(255); }
inline int pow2_at_least(int v, int lo) {
  int p = lo;
  while (p < v) p <<= 1;
  return p;
}

// ------------------------------------------------------------------ workspace layout
constexpr int kNumTables = 5;  // IBC, IT, HAD, OBC, OUT
// Fused input cast (cast_input_w64_kernel): fp32 x, 16-byte aligned, W % 4 == 0, W <= 64, and scale groups small
// enough that L2 is trusted to keep a group between its max pass and its quantisation.
#ifndef WL_CAST_L2_BYTES
#define WL_CAST_L2_BYTES (48ll << 20)
#endif
inline bool cast_fusable_shape(int C, int H, int W, int ipg) {
  return (W & 3) == 0 && W <= 64 && (long long)ipg * C * H * W * 4 <= WL_CAST_L2_BYTES;
}
constexpr int kFixHeaderBytes = 128;  // zeroed per call: fix-list / candidate counters [0, 16), stage done counters [16, 32)
extern const int kTableStage[kNumTables];

// The "saved" block [acc][V] comes first so that the STE backward, which reads only the per-group
// stage slots and the V codes, can keep that prefix alone (wl_forward_train puts it in its own buffer).
struct Layout {
  Geo g;
  size_t off_acc, off_sync, off_v, saved_total;  // offsets inside the saved block
  size_t off_c0, off_h, off_c1, off_c4, off_t4, off_e4, off_tab[kNumTables], tab_bytes[kNumTables], off_otab, off_odq, off_fix,
      total;  // offsets inside the workspace (split: the workspace excludes the saved block)
  unsigned fix_cap;
  int groups, hbytes, bn;
};
int make_layout(const wl_shape* s, const wl_qcfg* q, Layout* L, bool split = false);
FastDiv make_fastdiv(unsigned d);

// Test hook: cap of the deferred-fix lists (0 = automatic). Tiny caps force the inline fallback.
extern unsigned g_fix_cap_override;

int check_bits(const wl_qcfg* q);
Bits make_bits(const wl_qcfg* q);
int stage_bits(const wl_qcfg* q, int st);

struct WeightHeader {
  Acc wacc[ST_COUNT];
  int K, C, Kp, Cp, mode, wstage;
  wl_qcfg q;
};
size_t weight_cache_bytes(int K, int C, int* Kp, int* Cp);

// ------------------------------------------------------------------ launch helpers (per device)
int num_sms();
// Occupancy-sized persistent grid for a staged kernel; sets the dynamic shared-memory attribute for
// the current device on first use (the attribute is per device context).
int staged_grid_impl(const void* kern, int threads, int smem, long long work_items);
template <class K>
int staged_grid(K kern, int threads, int smem, long long work_items) {
  return staged_grid_impl(reinterpret_cast<const void*>(kern), threads, smem, work_items);
}
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device).
cudaError_t ensure_smem_attr(const void* kern, int smem);

// optional per-kernel-group event timing (bench.py) and WL_DEBUG_SYNC fault localisation
void prof_begin();
void prof_mark(const char* name, cudaStream_t st);
bool debug_sync_enabled();
extern const char* g_debug_fail;

float stage_depth(int mode, int stage);
StageE stage_rowsums(int mode);

// Tensor maps are cached per (arguments) so repeated calls on the same buffers skip the encode.
bool tmap_i8_3d(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t b0, uint32_t b1,
                uint32_t b2);
bool tmap_i8_4d(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t d3, uint32_t b0,
                uint32_t b1, uint32_t b2);
bool tmap_3d_plain(CUtensorMap* m, const void* base, int elem_bytes, uint64_t d0, uint64_t d1, uint64_t d2,
                   uint32_t b0, uint32_t b1, uint32_t b2);

// ------------------------------------------------------------------ forward context
struct FwdCtx {
  Geo g;
  const Layout* L;
  const wl_qcfg* q;
  Bits b;
  int mode;
  bool leg;
  Acc* acc;
  unsigned* sync;  // fused input cast: [0] block ticket, [1 + group] arrivals
  int8_t *c0, *c1, *V, *c4;
  void* h;
  float *t4, *e4, *otab;
  float4* odq;  // per group {s_hi, s_lo, ok}: certified arithmetic dequantisation (out_table_kernel)
  Tables tabs;
  FixList fl;
  StageE E;
  const PlanF64* pf;
  cudaStream_t st;
  const void* bias;
  void* y;
  int ybytes;  // 4 (fp32 y) or 8 (fp64 y)
  CUtensorMap c0map;  // 6x6 input-code windows (Cp <= 256)
  int fin_blocks, fix_blocks, pgrid;
};

// finalize (+ exec) + stage_params of one transform stage (wl_fwd.cu)
void finalize_input_stage(FwdCtx& c, int stage);
void finalize_output_stage(FwdCtx& c, int stage, bool t4);
void make_output_table(FwdCtx& c);
ParamsTail params_tail(const FwdCtx& c, int stage);  // stage_params_tail arguments of one stage (wl_fwd.cu)

template <int LD>
int run_input_side(FwdCtx& c);  // wl_fwd_in.inc
template <int LD, typename HT, typename YT>
int run_output_side(FwdCtx& c);  // wl_fwd_out.inc
int run_gemm_side(FwdCtx& c, const int8_t* U, const WeightHeader* wh);  // wl_fwd_gemm.cu

template <typename XT, typename YT>
int forward_impl(const wl_plan* plan, const wl_qcfg* q, const wl_shape* s, const XT* x, const void* cache,
                 const YT* bias, YT* y, void* saved, size_t saved_bytes, void* workspace, size_t workspace_bytes,
                 void* stream);

}  // namespace wl

struct wl_plan {
  int mode;
  wl::PlanF64* d_pf;  // device copy for the device that created the plan
  int device;
};
