/* winoleg_b200 — C ABI of the sm_100a quantized Winograd F(4x4,3x3) layer.
 *
 * This is the drop-in boundary for the reference's hot path
 *     winoleg.quantize.conv2d_winograd_quantized(x, w, plan, mode, qconfig)   (quantize.py:129-148)
 *     -> winoleg.pipeline.run_pipeline(x, w, plan, mode, cast)                (pipeline.py:106-158)
 *     -> winoleg._kernels.sandwich / hadamard_accumulate                      (_kernels.py:69-105)
 * The reference is pure Python with no FFI; the binding a maintainer would add is the ctypes
 * stub shown in INTEGRATION.md (the product package paper_2004_11077_b200 uses exactly that).
 *
 * Conventions: plain C types only; every tensor is a DEVICE pointer owned by the caller; work is
 * stream ordered on `stream` (a cudaStream_t passed as void*); no host synchronisation except in
 * wl_read_stats.  Functions return WL_OK (0) or a negative status and never throw; the message
 * of the last failure on the calling thread is returned by wl_last_error().
 */
#ifndef WINOLEG_B200_H
#define WINOLEG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum wl_status {
  WL_OK = 0,
  WL_ERR_ARG = -1,        /* invalid argument / shape (reference DimensionError / ValueError) */
  WL_ERR_PLAN = -2,       /* plan matrices differ from the compiled F(4,3) tables            */
  WL_ERR_BITS = -3,       /* a stage width the int8 tensor-core path cannot carry            */
  WL_ERR_CUDA = -4,       /* CUDA runtime / launch failure                                    */
  WL_ERR_WORKSPACE = -5   /* workspace or weight cache too small                              */
};

enum wl_mode { WL_CANONICAL = 0, WL_LEGENDRE = 1 }; /* pipeline.py:33 BASE_MODES */

/* Stage widths, field for field the reference QuantConfig (quantize.py:40-55). */
typedef struct {
  int input_bits, weight_bits, input_transform_bits, weight_transform_bits, base_change_bits, hadamard_bits,
      output_transform_bits;
} wl_qcfg;

/* x is [n][c_in][h][w] fp32 (NCHW); zero padding `pad` on every side (pad 0 == the reference's
 * valid correlation); stage scales are shared by `images_per_group` consecutive images
 * (1 == the reference's per-call semantics applied to each image; n == one scale per batch). */
typedef struct {
  int n, c_in, c_out, h, w, pad, images_per_group;
} wl_shape;

/* One StageStat (quantize.py:93-100) without the name: stage order is the reference's
 * (pipeline.py:17-21): canonical 6 rows, Legendre 9 rows. */
typedef struct {
  int bits;
  double max_abs;
  double scale;
} wl_stage_stat;

typedef struct wl_plan wl_plan;

/* Replaces build_plan + plan_to_float (construct.py:139-208) on the device side.
 * int_mats / f64_mats: the stage matrices D*L (int64) and L (fp64) in the order
 *   canonical: G (6x3), B^T (6x6), A^T (4x6)
 *   legendre:  G_P (6x3), P^-1 (6x6), P^-T (6x6), B_P^T (6x6), P^-T (6x6), A_P^T (4x6)
 * Integer matrices must equal the compiled default-point tables (else WL_ERR_PLAN). */
int wl_plan_create(int o, int k, int mode, const int64_t* int_mats, const double* f64_mats, wl_plan** out);
int wl_plan_destroy(wl_plan* plan);
int wl_plan_mode(const wl_plan* plan);

/* Weight side (pipeline.py:120, :124-137 — casts "weights", "weight_transform" and, Legendre,
 * "weight_base_change"), computed once and cached: U codes + the weight-stage statistics. */
int wl_weight_cache_size(const wl_plan* plan, int c_out, int c_in, size_t* bytes);
int wl_weight_transform(const wl_plan* plan, const wl_qcfg* q, const float* w, int c_out, int c_in, void* cache,
                        size_t cache_bytes, void* stream);
/* Same from fp64 weights: the reference's own operand dtype (pipeline.py:112-113 copies to fp64);
 * the "weights" codes are rint(w / scale) in fp64 exactly as quantize.py:118-119. */
int wl_weight_transform_f64(const wl_plan* plan, const wl_qcfg* q, const double* w, int c_out, int c_in, void* cache,
                            size_t cache_bytes, void* stream);

/* Forward: y [n][c_out][h+2pad-2][w+2pad-2] fp32 = dequantised output codes (+ bias if non-NULL).
 * workspace (and the saved buffer of wl_forward_train) must be 256-byte aligned device memory (WL_ERR_ARG
 * otherwise); x and y may have any alignment (16-byte alignment enables the vectorised paths). */
int wl_workspace_size(const wl_plan* plan, const wl_shape* s, const wl_qcfg* q, size_t* bytes);
int wl_forward(const wl_plan* plan, const wl_qcfg* q, const wl_shape* s, const float* x, const void* cache,
               const float* bias, float* y, void* workspace, size_t workspace_bytes, void* stream);
/* fp64 in / fp64 out (quantize.py:129-148 returns fp64): x is quantised in fp64 as the reference
 * does, so y is bit-identical to the reference's output for ANY fp64 input; all stages after
 * "input" run on integer codes exactly as in wl_forward. Same workspace as wl_forward. */
int wl_forward_f64(const wl_plan* plan, const wl_qcfg* q, const wl_shape* s, const double* x, const void* cache,
                   const double* bias, double* y, void* workspace, size_t workspace_bytes, void* stream);

/* Training forward: wl_forward with the part of its state the STE backward needs — the per-group
 * stage slots and the V codes — written to a separate `saved` buffer, so the caller can keep that
 * buffer until backward and release the (much larger) workspace right away.  wl_train_sizes gives
 * both sizes; the workspace of wl_forward_train is smaller than wl_forward's by the saved block. */
int wl_train_sizes(const wl_plan* plan, const wl_shape* s, const wl_qcfg* q, size_t* saved_bytes,
                   size_t* workspace_bytes);
int wl_forward_train(const wl_plan* plan, const wl_qcfg* q, const wl_shape* s, const float* x, const void* cache,
                     const float* bias, float* y, void* saved, size_t saved_bytes, void* workspace,
                     size_t workspace_bytes, void* stream);

/* Straight-through-estimator backward (no reference counterpart): casts are identity,
 * scales detached, products use the forward's quantised U and V.  `saved` is the saved buffer of the
 * wl_forward_train call being differentiated, or the whole workspace of a wl_forward call (both
 * start with the stage slots and V codes at the same offsets).
 * dx [n][c_in][h][w], dw [c_out][c_in][3][3], db [c_out] (may be NULL), all fp32. */
int wl_backward_workspace_size(const wl_plan* plan, const wl_shape* s, const wl_qcfg* q, size_t* bytes);
int wl_backward(const wl_plan* plan, const wl_qcfg* q, const wl_shape* s, const float* dy, const void* cache,
                const void* saved, float* dx, float* dw, float* db, void* workspace, size_t workspace_bytes,
                void* stream);

/* Float (unquantized) Winograd correlation in fp32 — the reference's conv2d_winograd(x, w, plan,
 * mode) (pipeline.py:161-164: run_pipeline with the identity cast), with the same batch, padding,
 * crop and bias conventions as wl_forward.  w is [c_out][c_in][3][3] fp32 (no cache: the weight
 * transform runs every call).  Accuracy: fp32 arithmetic (tolerance stated in tests/test_gpu_float.py). */
int wl_float_workspace_size(const wl_plan* plan, const wl_shape* s, size_t* bytes);
int wl_forward_float(const wl_plan* plan, const wl_shape* s, const float* x, const float* w, const float* bias, float* y,
                     void* workspace, size_t workspace_bytes, void* stream);

/* Quantized direct-convolution baseline — the reference's conv2d_direct_quantized(x, w, qconfig)
 * (quantize.py:151-160): fake-quantise x per scale group at input_bits and w at weight_bits, fp64
 * direct correlation in the reference's order (_kernels.py:53-66), fake-quantise the result per
 * group at output_transform_bits.  Computed in fp64 exactly as the reference does, so the f64 entry
 * point is bit-identical to the reference and the fp32 one is that result rounded to fp32.  x is
 * [n][c_in][h][w] with zero padding `pad`, w [c_out][c_in][3][3], y [n][c_out][h+2pad-2][w+2pad-2];
 * only input_bits, weight_bits and output_transform_bits of q are used (each in [2, 53]). */
int wl_direct_workspace_size(const wl_shape* s, size_t* bytes);
int wl_direct_quantized(const wl_qcfg* q, const wl_shape* s, const float* x, const float* w, float* y,
                        void* workspace, size_t workspace_bytes, void* stream);
/* The unquantized fp64 direct correlation, the reference's conv2d_direct (reference.py:34-39,
 * _kernels.py:53-66), same shapes and padding; bit-identical to the reference (its operation order). */
int wl_direct_f64(const wl_shape* s, const double* x, const double* w, double* y, void* workspace,
                  size_t workspace_bytes, void* stream);
int wl_direct_quantized_f64(const wl_qcfg* q, const wl_shape* s, const double* x, const double* w, double* y,
                            void* workspace, size_t workspace_bytes, void* stream);
/* Per-group StageStat rows [n/images_per_group][nstages] after wl_forward (synchronises stream). */
int wl_num_stages(const wl_plan* plan);
int wl_read_stats(const wl_plan* plan, const wl_shape* s, const wl_qcfg* q, const void* cache,
                  const void* workspace, wl_stage_stat* out, void* stream);

/* Byte offsets inside the workspace of the materialised codes (for parity tests):
 * off[0] input codes int8 [n][h][w][Cp]; off[1] V int8 [36][T][Cp]; off[2] hadamard codes
 * [36][T][Kp] (int8, int16 when hadamard_bits > 8); off[3] group maxima; dims[0..3] = Cp, Kp, T, TP. */
int wl_debug_layout(const wl_plan* plan, const wl_shape* s, const wl_qcfg* q, size_t* off, int* dims);

/* Number of kernels wl_forward launches for this shape (reported by bench.py as gpu_launches). */
int wl_forward_launches(const wl_plan* plan, const wl_shape* s, const wl_qcfg* q);

/* Optional per-kernel CUDA-event timing of wl_forward (measurement only, not thread safe):
 * wl_profile_read synchronises the device and returns, per kernel slot, the summed milliseconds
 * over every wl_forward issued since the previous read. */
int wl_profile_enable(int on);
int wl_profile_read(const char** names_out, double* ms_out, int max, int* n_out, int* calls_out);

/* Test hook: the split-bf16 tcgen05 GEMM behind the STE backward and the float path, on device
 * buffers: D[s][b][m][n] (row stride ldd) = alpha * sum_{k in split s} A[b][m][k] B[b][n][k] with
 * A bf16 [PA][batch][M][Kd], B bf16 [PB][batch][N][Kd] (planes summed: x = hi + mid + lo), Kd and ks
 * multiples of 64, splits = ceil(Kd / ks); plane products (i, j) with i + j < max(PA, PB). */
int wl_debug_gemm_bf16(const void* A, int PA, const void* B, int PB, int batch, int M, int N, int Kd, int ks,
                       float* D, int ldd, float alpha, void* stream);

/* Test hook: capacity of the deferred exact-fix lists (0 = automatic, the default).  A tiny cap forces
 * every producer onto its inline fallback; results must not change (tests/test_gpu_parity.py). */
int wl_debug_set_fix_cap(unsigned cap);

const char* wl_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* WINOLEG_B200_H */
