// Forward orchestration of the quantized Winograd F(4x4,3x3) layer: the dependency chain of
// run_pipeline (pipeline.py:106-158) with the casts of quantize.py:129-148 as device passes.
//   input cast (absmax, quantise) -> input side (wl_fwd_in.inc) -> Hadamard passes (wl_fwd_gemm.cu)
//   -> output side (wl_fwd_out.inc)
// Every stage's per-group maximum is a dependency of its codes, so each arrow is a kernel boundary.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "wl_internal.h"

namespace wl {

// arguments of stage_params_tail for one stage (the done counter lives in the zeroed fix-list header)
ParamsTail params_tail(const FwdCtx& c, int stage) {
  return ParamsTail{c.L->groups, c.b.q[stage], stage == ST_HAD ? 0.f : stage_depth(c.mode, stage),
                    c.fl.count + kDoneSlot0 + stage};
}

template <int MODE, int STAGE>
static void finalize_input_t(FwdCtx& c) {
  finalize_input_kernel<MODE, STAGE><<<c.fin_blocks, 256, 0, c.st>>>(c.c0, c.c1, c.g, c.b, c.acc, c.pf,
                                                                     c.tabs.t[STAGE], c.E.e[STAGE], c.fl);
  finalize_input_exec<MODE, STAGE><<<c.fin_blocks, 256, 0, c.st>>>(c.c0, c.c1, c.g, c.b, c.acc, c.pf, c.fl,
                                                                   params_tail(c, STAGE));
}

void finalize_input_stage(FwdCtx& c, int stage) {
  if (!c.leg)
    finalize_input_t<0, ST_IT>(c);
  else if (stage == ST_IBC)
    finalize_input_t<1, ST_IBC>(c);
  else
    finalize_input_t<1, ST_IT>(c);
}

template <int MODE, int STAGE, typename HT, bool T4>
static void finalize_output_t(FwdCtx& c) {
  const HT* hh = reinterpret_cast<const HT*>(c.h);
  finalize_output_kernel<MODE, STAGE, HT, T4><<<c.fin_blocks, 256, 0, c.st>>>(hh, c.c4, c.g, c.b, c.acc, c.pf,
                                                                              c.tabs.t[STAGE], c.E.e[STAGE], c.fl);
  finalize_output_exec<MODE, STAGE, HT, T4><<<c.fin_blocks, 256, 0, c.st>>>(hh, c.c4, c.g, c.b, c.acc, c.pf, c.fl,
                                                                            params_tail(c, STAGE));
}

template <typename HT>
static void finalize_output_h(FwdCtx& c, int stage, bool t4) {
  if (!c.leg)
    finalize_output_t<0, ST_OUT, HT, false>(c);
  else if (stage == ST_OBC)
    finalize_output_t<1, ST_OBC, HT, false>(c);
  else if (t4)
    finalize_output_t<1, ST_OUT, HT, true>(c);
  else
    finalize_output_t<1, ST_OUT, HT, false>(c);
}

void finalize_output_stage(FwdCtx& c, int stage, bool t4) {
  if (c.L->hbytes == 1)
    finalize_output_h<int8_t>(c, stage, t4);
  else
    finalize_output_h<int16_t>(c, stage, t4);
}

void make_output_table(FwdCtx& c) {
  if (!c.otab) return;
  out_table_kernel<<<(unsigned)c.L->groups, 256, 0, c.st>>>(c.acc, c.L->groups, c.b.q[ST_OUT], c.otab, c.odq);
}

// cast "input": per-group max|x|, then x (NCHW fp32/fp64) -> c0 (NHWC int8)
template <typename XT>
static int input_cast(FwdCtx& c, const XT* x) {
  const Geo& g = c.g;
  const long long per_image = (long long)g.C * g.H * g.W;
  const bool w64 = sizeof(XT) == 4 && (g.W & 3) == 0 && g.W <= 64 && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
#ifndef WL_QI_RH
#define WL_QI_RH 2
#endif
#ifndef WL_CAST_LAG
#define WL_CAST_LAG 1  // images between a band's max pass and its quantisation (>= images per group)
#endif
  // band of rh rows per block: per channel one contiguous rh * W float run (at most 256 float4 slots and
  // ~60 KB of staging per block)
  // narrow images take taller bands (a block's fixed cost is spread over more bytes: configs 1-3 forward
  // -1..3 % with 4- or 8-row bands; at W = 56 two rows measured best)
  int rh = g.W <= 32 ? 8 : WL_QI_RH;
  while (rh > 1 && (rh * g.W * (g.Cp + 4) > 60 * 1024 || rh * g.W / 4 > 256)) rh >>= 1;
  rh = std::min(rh, g.H);
  const int smem = rh * g.W * (g.Cp + 4);
  const int nb = (g.H + rh - 1) / rh;
  if (w64 && cast_fusable_shape(g.C, g.H, g.W, g.ipg)) {
    // one launch, x read from HBM once (the second read of a band hits L2)
    const int lag = (int)std::min<long long>(std::max(g.ipg, WL_CAST_LAG),
                                             std::max<long long>(g.ipg, WL_CAST_L2_BYTES / (per_image * 4)));
    WL_CUDA(ensure_smem_attr(reinterpret_cast<const void*>(cast_input_w64_kernel<0>), smem));
    cast_input_w64_kernel<<<(unsigned)nb * (unsigned)(g.N + lag), 256, smem, c.st>>>(
        reinterpret_cast<const float*>(x), c.c0, g, c.b, c.acc, rh, lag, c.sync);
    prof_mark("cast_input", c.st);
    return WL_OK;
  }
  const int bx = (int)std::min<long long>((per_image / 4 + 255) / 256, 64);
  absmax_input_kernel<XT><<<dim3(std::max(bx, 1), g.N), 256, 0, c.st>>>(x, per_image, g.ipg, c.acc);
  prof_mark("absmax_input", c.st);
  if (w64) {
    WL_CUDA(ensure_smem_attr(reinterpret_cast<const void*>(quant_input_w64_kernel<0>), smem));
    quant_input_w64_kernel<<<dim3((g.H + rh - 1) / rh, g.N), 256, smem, c.st>>>(reinterpret_cast<const float*>(x),
                                                                              c.c0, g, c.b, c.acc, rh);
  } else {
    const int qrow = std::max(4, std::min(64, (160000 / (g.Cp + 16)) & ~3));
    const int qsm = qrow * (g.Cp + 16);
    WL_CUDA(ensure_smem_attr(reinterpret_cast<const void*>(quant_input_kernel<XT>), qsm));
    quant_input_kernel<XT><<<dim3(g.H, g.N), 256, qsm, c.st>>>(x, c.c0, g, c.b, c.acc, qrow);
  }
  prof_mark("quant_input", c.st);
  return WL_OK;
}

template <int V>
using IntC = std::integral_constant<int, V>;

template <typename XT, typename YT>
int forward_impl(const wl_plan* plan, const wl_qcfg* q, const wl_shape* s, const XT* x, const void* cache,
                 const YT* bias, YT* y, void* saved, size_t saved_bytes, void* workspace, size_t workspace_bytes,
                 void* stream) {
  if (!plan || !x || !cache || !y || !workspace) return fail(WL_ERR_ARG, "NULL argument");
  int rc = check_bits(q);
  if (rc) return rc;
  Layout L;
  const bool split = saved != nullptr;
  rc = make_layout(s, q, &L, split);
  if (rc) return rc;
  if (workspace_bytes < L.total) return fail(WL_ERR_WORKSPACE, "workspace needs %zu bytes", L.total);
  if (split && saved_bytes < L.saved_total) return fail(WL_ERR_WORKSPACE, "saved buffer needs %zu bytes", L.saved_total);
  // TMA / bulk copies and 16-byte vector accesses address the workspace blocks at their 256-byte-aligned offsets
  if ((reinterpret_cast<uintptr_t>(workspace) & 255) || (saved && (reinterpret_cast<uintptr_t>(saved) & 255)))
    return fail(WL_ERR_ARG, "workspace and saved buffers must be 256-byte aligned");
  const Geo& g = L.g;
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  uint8_t* sv = split ? reinterpret_cast<uint8_t*>(saved) : ws;
  const WeightHeader* wh = reinterpret_cast<const WeightHeader*>(cache);
  const int8_t* U = reinterpret_cast<const int8_t*>(cache) + align256(sizeof(WeightHeader));

  FwdCtx c;
  c.g = g;
  c.L = &L;
  c.q = q;
  c.b = make_bits(q);
  c.mode = plan->mode;
  c.leg = plan->mode == WL_LEGENDRE;
  c.acc = reinterpret_cast<Acc*>(sv + L.off_acc);
  c.sync = reinterpret_cast<unsigned*>(sv + L.off_sync);
  c.V = reinterpret_cast<int8_t*>(sv + L.off_v);
  c.c0 = reinterpret_cast<int8_t*>(ws + L.off_c0);
  c.c1 = reinterpret_cast<int8_t*>(ws + L.off_c1);
  c.c4 = reinterpret_cast<int8_t*>(ws + L.off_c4);
  c.h = ws + L.off_h;
  c.t4 = reinterpret_cast<float*>(ws + L.off_t4);
  c.e4 = reinterpret_cast<float*>(ws + L.off_e4);
  c.otab = sizeof(YT) == 4 && q->output_transform_bits <= 12 ? reinterpret_cast<float*>(ws + L.off_otab) : nullptr;
  c.odq = c.otab ? reinterpret_cast<float4*>(ws + L.off_odq) : nullptr;
  c.pf = plan->d_pf;
  c.st = st;
  c.bias = bias;
  c.y = y;
  c.ybytes = (int)sizeof(YT);
  c.E = stage_rowsums(plan->mode);
  c.fl.count = reinterpret_cast<unsigned*>(ws + L.off_fix);
  c.fl.items = reinterpret_cast<unsigned*>(ws + L.off_fix + kFixHeaderBytes);
  c.fl.cap = L.fix_cap;
  // grid-stride helper kernels: one wave covers every deferred unit / table row of config-4-sized calls;
  // small calls launch only the blocks their lists and tables can fill (launch-bound shapes)
  c.fix_blocks = (int)std::min<long long>(16LL * num_sms(), ((long long)L.fix_cap + 127) / 128);
  c.fin_blocks = (int)std::max<long long>(1, std::min<long long>(4LL * num_sms(), (36LL * g.T + 255) / 256));
  c.pgrid = (L.groups + 127) / 128;
  for (int i = 0; i < ST_COUNT; ++i) c.tabs.t[i] = nullptr;

  prof_begin();
  WL_CUDA(cudaMemsetAsync(c.acc, 0, L.off_v - L.off_acc, st));  // group accumulators + cast tickets
  prof_mark("begin", st);
  if ((rc = input_cast<XT>(c, x))) return rc;

  for (int i = 0; i < kNumTables; ++i) c.tabs.t[kTableStage[i]] = reinterpret_cast<unsigned*>(ws + L.off_tab[i]);
  // one memset: the four transform-stage max tables and the fix-list counters are contiguous (make_layout)
  WL_CUDA(cudaMemsetAsync(ws + L.off_tab[0], 0, L.off_fix + kFixHeaderBytes - L.off_tab[0], st));
  if (g.Cp <= 256 && !tmap_i8_4d(&c.c0map, c.c0, g.Cp, g.W, g.H, g.N, g.Cp, 6, 6))
    return fail(WL_ERR_CUDA, "cuTensorMapEncodeTiled (input window) failed");

  switch (g.Cp) {
    case 32: rc = run_input_side<32>(c); break;
    case 64: rc = run_input_side<64>(c); break;
    case 128: rc = run_input_side<128>(c); break;
    case 256: rc = run_input_side<256>(c); break;
    case 512: rc = run_input_side<512>(c); break;
    default: rc = fail(WL_ERR_ARG, "unsupported padded channel count %d", g.Cp);
  }
  if (rc) return rc;
  WL_CUDA(cudaGetLastError());
  // padded channels of V must be zero for the GEMM: the stage kernels only write c < C
  if (g.Cp != g.C) WL_CUDA(cudaMemset2DAsync(c.V + g.C, g.Cp, 0, g.Cp - g.C, (size_t)36 * g.T, st));  // [T*36][Cp]

  if ((rc = run_gemm_side(c, U, wh))) return rc;

  auto out = [&](auto ldc) -> int {
    constexpr int LD = decltype(ldc)::value;
    return L.hbytes == 1 ? run_output_side<LD, int8_t, YT>(c) : run_output_side<LD, int16_t, YT>(c);
  };
  switch (g.Kp) {
    case 64: rc = out(IntC<64>{}); break;
    case 128: rc = out(IntC<128>{}); break;
    case 256: rc = out(IntC<256>{}); break;
    case 512: rc = out(IntC<512>{}); break;
    default: rc = fail(WL_ERR_ARG, "unsupported padded output-channel count %d", g.Kp);
  }
  if (rc) return rc;

  WL_CUDA(cudaGetLastError());
  if (g_debug_fail)
    return fail(WL_ERR_CUDA, "kernel group '%s' failed: %s", g_debug_fail, cudaGetErrorString(cudaGetLastError()));
  return WL_OK;
}

template int forward_impl<float, float>(const wl_plan*, const wl_qcfg*, const wl_shape*, const float*, const void*,
                                        const float*, float*, void*, size_t, void*, size_t, void*);
template int forward_impl<double, double>(const wl_plan*, const wl_qcfg*, const wl_shape*, const double*, const void*,
                                          const double*, double*, void*, size_t, void*, size_t, void*);

}  // namespace wl
