// Device helpers shared by the transform, GEMM-epilogue and output kernels.
//
// Integer-exact stage rule: if a stage tensor equals f * T with T integer and
// f > 0, the reference's codes rint(t / (max|t| / qmax)) (quantize.py:118-119) equal
// rhe(qmax * T / max|T|) except where that ratio is an exact half-integer ("tie").  At ties the
// fp64 reference resolves by rounding noise, so those elements — and the elements that attain the
// stage maximum, whose fp64 value IS max_abs (quantize.py:141) — are re-evaluated ("replayed") in
// fp64 with the reference's exact operation order: sandwich tmp = X.R then L.tmp with l ascending
// (_kernels.py:69-92), Hadamard sum over c ascending from 0.0 (_kernels.py:94-105), every product
// and sum rounded separately (__dmul_rn/__dadd_rn, never fused).
#pragma once
#include <cstdint>
#include <type_traits>
#include "wl_tables.cuh"

namespace wl {

enum StageId { ST_INPUT = 0, ST_WEIGHTS, ST_WT, ST_WBC, ST_IBC, ST_IT, ST_HAD, ST_OBC, ST_OUT, ST_COUNT };

// Per (group, stage) reduction slot: M = max |T| (integer stages) or fp32 bits of max |x| (input /
// weights); F = fp64 bits of the reference's max_abs (positive doubles order like uint64).
struct PlanF64 {  // fp64 left matrices (nearest doubles of the exact rationals, construct.py:191-208)
  double wt[6 * 3], wbc[36], ibc[36], it[36], obc[36], ot[4 * 6];
};

struct Acc {
  unsigned long long M;   // exact integer max |T| (fp64 bits of max|x| for input / weights)
  unsigned long long F;   // fp64 bits of the reference max_abs
  unsigned int MF;        // fp32 bits of the running max of the fp32 fast-path values
  float thr;              // fast path: 0.5 - band (set by stage_params_kernel once M is final)
  float r;                // fast path: qmax / M
  unsigned int TM;        // fp32 bits of max |first-half value| over the group (error bound input)
  float ef;               // fast path: qmax * 6.5 * 2^-24 / M (per-element band = ef * rowsum_i * tmax_j)
  float pad_;
  double scale;           // reference scale max_abs / qmax (1.0 when max_abs == 0)
};

// Max tables: every hot pass writes the maximum of each 32-unit entry (fp32 bits for the transform
// stages, exact int for the Hadamard row chunks).  A finalize kernel scans the table, recomputes
// exactly only the entries that can hold the group's argmax, and replays that argmax in fp64.
// Deterministic, no capacity limit.
struct StageQ {
  long long M;
  double maxabs, scale;
  float rcp;
  int qmax;
};

__device__ __forceinline__ StageQ load_int_stage(const Acc& a, int qmax) {
  StageQ s;
  s.M = (long long)a.M;
  s.maxabs = __longlong_as_double((long long)a.F);
  s.qmax = qmax;
  s.scale = s.maxabs > 0.0 ? s.maxabs / (double)qmax : 1.0;  // quantize.py:107-108
  s.rcp = s.M ? (float)qmax / (float)s.M : 0.f;
  return s;
}
// Input / weight stage: M holds the fp32 bits of max|v|, exact in fp64.
__device__ __forceinline__ StageQ load_float_stage(const Acc& a, int qmax) {
  StageQ s;
  s.M = 0;
  s.maxabs = __longlong_as_double((long long)a.M);
  s.qmax = qmax;
  s.scale = s.maxabs > 0.0 ? s.maxabs / (double)qmax : 1.0;
  s.rcp = s.maxabs > 0.0 ? (float)((double)qmax / s.maxabs) : 0.f;
  return s;
}

// Dequantised value of a code as the reference holds it after fake_quant (quantize.py:120-125).
__device__ __forceinline__ double deq(int c, int qmax, double maxabs, double scale) {
  return c == qmax ? maxabs : (c == -qmax ? -maxabs : (double)c * scale);
}

// rhe(qmax * |T| / M) with exact tie detection.  Fast path in fp32: x = fl(fl(|T|) * fl(qmax / M)) is
// within 3 * 2^-24 * x <= 1.8e-7 * qmax of the quotient, so within 2e-4 + 2.4e-7 * qmax of a
// half-integer (6e-3 for 16-bit outputs: a fixed 2e-4 misjudged exact ties of wide output stages,
// found by the seeded random parity sweep) the decision is redone exactly in int64.  On an exact tie
// `tie` is set and floor is returned; the caller replays the element in fp64.
__device__ __forceinline__ int rq(long long T, const StageQ& q, bool& tie) {
  if (T == 0 || q.M == 0) return 0;
  const long long a = T < 0 ? -T : T;
  const float x = __fmul_rn((float)a, q.rcp);
  const float k = floorf(x);
  const float fr = x - k;
  int c = (int)k;
  if (fabsf(fr - 0.5f) > 2e-4f + 2.4e-7f * (float)q.qmax) {
    c += fr > 0.5f;
  } else {
    const long long n2 = 2LL * q.qmax * a;
    const long long rhs = (2LL * c + 1) * q.M;
    if (n2 > rhs)
      c += 1;
    else if (n2 == rhs)
      tie = true;
  }
  return T < 0 ? -c : c;
}

// Reference code of a replayed fp64 stage value (quantize.py:118-119).
__device__ __forceinline__ int code_of(double t, const StageQ& q) {
  double c = rint(t / q.scale);
  c = c > q.qmax ? q.qmax : c;
  c = c < -q.qmax ? -q.qmax : c;
  return (int)c;
}

// Input / weight codes from fp32 values: rint(fp64(v) / scale) exactly as the reference, with an
// fp32 fast path that is only trusted away from half-integers.
__device__ __forceinline__ int quant_float(float v, const StageQ& q) {
  if (q.maxabs == 0.0) return 0;
  const float x = __fmul_rn(fabsf(v), q.rcp);
  const float k = floorf(x);
  const float fr = x - k;
  int c;
  if (fabsf(fr - 0.5f) > 1e-4f) {
    c = (int)k + (fr > 0.5f);
    c = c > q.qmax ? q.qmax : c;
    return v < 0.f ? -c : c;
  }
  double d = rint((double)v / q.scale);
  d = d > q.qmax ? q.qmax : d;
  d = d < -q.qmax ? -q.qmax : d;
  return (int)d;
}

// fp64 operand: the reference's own arithmetic (quantize.py:118-119), c = clip(rint(v / scale)).
__device__ __forceinline__ int quant_float(double v, const StageQ& q) {
  if (q.maxabs == 0.0) return 0;
  double d = rint(__ddiv_rn(v, q.scale));
  d = d > q.qmax ? q.qmax : d;
  d = d < -q.qmax ? -q.qmax : d;
  return (int)d;
}

// ---------------------------------------------------------------- fp64 replays (rare path)

// out[i][j] of L . X . L^T, L is R x B (row-major fp64), X is B x B given as codes + dequant params.
static __device__ __noinline__ double replay_sandwich(const double* __restrict__ L, int R, int B, const int* codes, int qmax,
                                               double maxabs, double scale, int i, int j) {
  (void)R;
  double tmp[6];
  for (int l = 0; l < B; ++l) {
    double s = 0.0;
    for (int l2 = 0; l2 < B; ++l2) s = __dadd_rn(s, __dmul_rn(deq(codes[l * B + l2], qmax, maxabs, scale), L[j * B + l2]));
    tmp[l] = s;
  }
  double out = 0.0;
  for (int l = 0; l < B; ++l) out = __dadd_rn(out, __dmul_rn(L[i * B + l], tmp[l]));
  return out;
}

// Hadamard element: sum_c deq(u_c) * deq(v_c), c ascending from 0.0 (_kernels.py:99-104).
template <bool kCold = true>
__device__ __noinline__ double replay_hadamard(const int8_t* __restrict__ u, const int8_t* __restrict__ v, int C,
                                               StageQ qu, StageQ qv) {
  // kCold (one tie per thread, rows not yet cached: fixup_had_kernel): the two code rows are pulled
  // into L1 up front — one prefetch per 128-byte line — and read 16 bytes at a time, so the
  // c-ascending fp64 chain reads L1 instead of paying an HBM/L2 round trip per sector (114 -> 19 us).
  // Warm callers (finalize_hadamard: rows shared by neighbouring candidates) keep the byte loop,
  // measured faster there.
  if (!kCold) {
    double acc = 0.0;
    for (int c = 0; c < C; ++c)
      acc = __dadd_rn(acc, __dmul_rn(deq(u[c], qu.qmax, qu.maxabs, qu.scale), deq(v[c], qv.qmax, qv.maxabs, qv.scale)));
    return acc;
  }
  for (int c = 0; c < C; c += 128) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(u + c));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(v + c));
  }
  double acc = 0.0;
  int c = 0;
  if ((((uintptr_t)u | (uintptr_t)v) & 15) == 0) {
    for (; c + 16 <= C; c += 16) {
      const int4 a = __ldg(reinterpret_cast<const int4*>(u + c)), b = __ldg(reinterpret_cast<const int4*>(v + c));
      const int aw[4] = {a.x, a.y, a.z, a.w}, bw[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int cu = (int)(int8_t)(aw[j >> 2] >> (8 * (j & 3))), cv = (int)(int8_t)(bw[j >> 2] >> (8 * (j & 3)));
        acc = __dadd_rn(acc, __dmul_rn(deq(cu, qu.qmax, qu.maxabs, qu.scale), deq(cv, qv.qmax, qv.maxabs, qv.scale)));
      }
    }
  }
  for (; c < C; ++c)
    acc = __dadd_rn(acc, __dmul_rn(deq(u[c], qu.qmax, qu.maxabs, qu.scale), deq(v[c], qv.qmax, qv.maxabs, qv.scale)));
  return acc;
}

// Group-wide running maxima are written with a read-first atomic: a plain L2 load (ld.global.cg, the
// coherence point of atomics) filters out every value that cannot raise the maximum, so a slot shared
// by a whole batch (scale_groups = "batch": one group) sees a handful of atomics per pass instead of
// one per warp serialised on a single L2 address (16.2 -> ~10 ms on config 4 with batch-wide scales).
// With many groups (per-image scales) the slots are uncontended and the extra load's latency would
// only stall the warp, so `lazy` (Geo::lazy: fewer than 16 groups) selects the filter.
__device__ __forceinline__ void lazy_max(unsigned int* p, unsigned int v, bool lazy) {
  if (!lazy || v > __ldcg(p)) atomicMax(p, v);
}
__device__ __forceinline__ void lazy_max(unsigned long long* p, unsigned long long v, bool lazy) {
  if (!lazy || v > __ldcg(p)) atomicMax(p, v);
}

__device__ __forceinline__ unsigned long long dbits(double d) { return (unsigned long long)__double_as_longlong(d); }

// Decide whether this lane must replay its local-argmax elements: only lanes holding the maximum
// of their warp (when the warp shares one group), and only while that maximum can still be the
// group's global maximum.  Any element equal to the final maximum passes this test because the
// global value only grows.  fp64 magnitudes are ordered like the integers (gap >= 1/M relative,
// fp64 noise < 1e-13), so an atomicMax over replayed values yields the exact max_abs.
__device__ __forceinline__ bool replay_gate(long long m, int g, const Acc* acc, int stride, bool& uniform,
                                            long long& wmax) {
  const unsigned full = 0xffffffffu;
  const int g0 = __shfl_sync(full, g, 0);
  uniform = __all_sync(full, g == g0);
  wmax = m;
  if (uniform) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      long long other = __shfl_xor_sync(full, wmax, o);
      wmax = other > wmax ? other : wmax;
    }
  }
  if (m <= 0 || g < 0) return false;
  if (uniform && m != wmax) return false;
  const long long cur = (long long)(*(volatile const unsigned long long*)&acc[(size_t)g * stride].M);
  return m >= cur;
}

__device__ __forceinline__ void publish_max(long long m, int g, Acc* acc, int stride, bool uniform, long long wmax,
                                            bool lazy = false) {
  if (uniform) {
    if ((threadIdx.x & 31) == 0 && wmax > 0 && g >= 0) lazy_max(&acc[(size_t)g * stride].M, (unsigned long long)wmax, lazy);
  } else if (m > 0 && g >= 0) {
    lazy_max(&acc[(size_t)g * stride].M, (unsigned long long)m, lazy);
  }
}

// ---------------------------------------------------------------- fp32 fast path

// Parameters of one integer stage for the fp32 fast path: x = T_f * r, rounded half-even by the
// magic-number add; elements whose x lies within `band` of a half-integer take the exact path.
struct StageF {
  float r, band;
  int qmax;
};
constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23: fma(T, r, kMagic) rounds T*r half-even to an integer
// Record the fp32 maximum `m` of this lane's unit into the entry (t, c/32) of the stage's max table
// and into the group's running fp32 maximum.  When the warp is exactly one entry (channel-aligned),
// lane 0 stores; otherwise lanes atomically max into their entries.
__device__ __forceinline__ void record_max(float m, int g, unsigned* table_entry, bool aligned, Acc* acc_stage,
                                          bool& uniform, float& wmax) {
  const unsigned full = 0xffffffffu;
  const int g0 = __shfl_sync(full, g, 0);
  uniform = __all_sync(full, g == g0) && aligned;
  wmax = m;
  if (uniform) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) wmax = fmaxf(wmax, __shfl_xor_sync(full, wmax, o));
    if ((threadIdx.x & 31) == 0 && g >= 0) *table_entry = __float_as_uint(wmax);
  } else if (g >= 0) {
    atomicMax(table_entry, __float_as_uint(m));
  }
}

__device__ __forceinline__ void publish_mf(float m, int g, Acc* acc_stage, bool uniform, float wmax, bool lazy = false) {
  if (uniform) {
    if ((threadIdx.x & 31) == 0 && wmax > 0.f && g >= 0)
      lazy_max(&acc_stage[(size_t)g * ST_COUNT].MF, __float_as_uint(wmax), lazy);
  } else if (m > 0.f && g >= 0) {
    lazy_max(&acc_stage[(size_t)g * ST_COUNT].MF, __float_as_uint(m), lazy);
  }
}

// fp32 sandwich out = L . X . L^T with compile-time integer L (R x C).  The first half X . L^T is
// exact (|partial sums| <= qmax_in * rowsum(L) < 2^24); the second half rounds once per fma, so
// |out - exact| <= 8 * 2^-24 * rowsum(L)^2 * qmax_in (the per-stage E passed to the kernels).
template <class L>
__device__ __forceinline__ void sandwich_f(const float (&X)[L::C][L::C], float (&tmp)[L::C][L::R],
                                           float (&out)[L::R][L::R]) {
#pragma unroll
  for (int i = 0; i < L::C; ++i)
#pragma unroll
    for (int j = 0; j < L::R; ++j) {
      float s = 0.f;
#pragma unroll
      for (int l = 0; l < L::C; ++l)
        if (L::e(j, l) != 0) s = fmaf(X[i][l], (float)L::e(j, l), s);
      tmp[i][j] = s;
    }
#pragma unroll
  for (int i = 0; i < L::R; ++i)
#pragma unroll
    for (int j = 0; j < L::R; ++j) {
      float s = 0.f;
#pragma unroll
      for (int l = 0; l < L::C; ++l)
        if (L::e(i, l) != 0) s = fmaf((float)L::e(i, l), tmp[l][j], s);
      out[i][j] = s;
    }
}

template <class L>
__device__ __forceinline__ void sandwich_f(const float (&X)[L::C][L::C], float (&out)[L::R][L::R]) {
  float tmp[L::C][L::R];
  sandwich_f<L>(X, tmp, out);
}

// Even/odd row pairs of a stage matrix: rows a, b with L[b][l] = +-L[a][l] for every l (at least one
// + and one - nonzero), as in B^T / B_P^T.  Both rows come from e = sum of the "+" terms and
// o = sum of the "-" terms: out[a] = e + o, out[b] = e - o, saving ~1/3 of the multiply-adds.
template <class L>
__host__ __device__ constexpr bool rows_pair(int a, int b) {
  bool ev = false, od = false;
  for (int l = 0; l < L::C; ++l) {
    const int x = L::e(a, l), y = L::e(b, l);
    if (x == y) {
      if (x != 0) ev = true;
    } else if (x == -y) {
      od = true;
    } else {
      return false;
    }
  }
  return ev && od;
}
template <class L>
__host__ __device__ constexpr int row_partner(int a) {
  // greedy in index order, so the relation is symmetric
  int p[8] = {-1, -1, -1, -1, -1, -1, -1, -1};
  for (int i = 0; i < L::R; ++i)
    if (p[i] < 0)
      for (int k = i + 1; k < L::R; ++k)
        if (p[k] < 0 && rows_pair<L>(i, k)) {
          p[i] = k;
          p[k] = i;
          break;
        }
  return p[a];
}

// Compile-time loop: f(std::integral_constant<int, i>) for i in [B, E), so per-index properties of
// the stage matrix (row partners) are constant-evaluated by the front end.
template <int B, int E, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for<B + 1, E>(f);
  }
}

// Row J (and its partner P > J, if any) of L dotted with v.
template <class L, int J, int P>
__device__ __forceinline__ void lrows_dot(const float (&v)[L::C], float& oj, float& op) {
  if constexpr (P > J) {
    float e = 0.f, o = 0.f;
#pragma unroll
    for (int l = 0; l < L::C; ++l) {
      const int a = L::e(J, l);
      if (a != 0) {
        if (a == L::e(P, l))
          e = fmaf(v[l], (float)a, e);
        else
          o = fmaf(v[l], (float)a, o);
      }
    }
    oj = e + o;
    op = e - o;
  } else {
    float s = 0.f;
#pragma unroll
    for (int l = 0; l < L::C; ++l)
      if (L::e(J, l) != 0) s = fmaf(v[l], (float)L::e(J, l), s);
    oj = s;
    op = 0.f;
  }
}

// out = L . v (second half), row pairs shared.  Rounding depth <= 4 per element, inside the
// 6.5 * 2^-24 * rowsum * max|v| bound the fast path certifies.
template <class L>
__device__ __forceinline__ void lapply(const float (&v)[L::C], float (&out)[L::R]) {
  static_for<0, L::R>([&](auto I) {
    constexpr int i = decltype(I)::value;
    constexpr int p = row_partner<L>(i);
    if constexpr (!(p >= 0 && p < i)) {
      float a, b;
      lrows_dot<L, i, p>(v, a, b);
      out[i] = a;
      if constexpr (p > i) out[p] = b;
    }
  });
}

// Column-streaming fp32 sandwich: for each output column j, tc = X . L[j]^T (exact) and
// col = L . tc; f(j, col) consumes the column before the next is formed, so only X and one or two
// columns are live.  Paired rows of L produce columns j and partner(j) together.
template <class L, class F>
__device__ __forceinline__ void sandwich_cols(const float (&X)[L::C][L::C], F&& f, float* tmax = nullptr) {
  auto emit = [&](int j, const float (&tc)[L::C]) {
    float col[L::R];
    lapply<L>(tc, col);
    if constexpr (std::is_invocable_v<F, int, const float (&)[L::R], float>) {
      float cm = 0.f;
#pragma unroll
      for (int l = 0; l < L::C; ++l) cm = fmaxf(cm, fabsf(tc[l]));
      f(j, col, cm);
    } else {
      f(j, col);
    }
  };
  static_for<0, L::R>([&](auto J) {
    constexpr int j = decltype(J)::value;
    constexpr int p = row_partner<L>(j);
    if constexpr (!(p >= 0 && p < j)) {
      float tc[L::C], tp[L::C];
#pragma unroll
      for (int l = 0; l < L::C; ++l) {
        lrows_dot<L, j, p>(X[l], tc[l], tp[l]);
        if (tmax) *tmax = fmaxf(*tmax, p > j ? fmaxf(fabsf(tc[l]), fabsf(tp[l])) : fabsf(tc[l]));
      }
      emit(j, tc);
      if constexpr (p > j) emit(p, tp);
    }
  });
}

// Rounding depth of the fp32 second half per element (sandwich_cols / lapply): a chain of n fmas
// rounds n times; a row pair rounds max(n_even, n_odd) times and once more in e +- o.  The fast path
// certifies |error| <= depth * 2^-24 * rowsum * max|tmp| (plus a 0.5 margin in stage_params_kernel).
template <class L>
__host__ __device__ constexpr int chain_depth() {
  int d = 0;
  for (int i = 0; i < L::R; ++i) {
    const int p = row_partner<L>(i);
    int ne = 0, no = 0, nz = 0;
    for (int l = 0; l < L::C; ++l) {
      const int a = L::e(i, l);
      if (a != 0) {
        ++nz;
        if (p >= 0 && a == L::e(p, l))
          ++ne;
        else if (p >= 0)
          ++no;
      }
    }
    const int di = p >= 0 ? (ne > no ? ne : no) + 1 : nz;
    d = di > d ? di : d;
  }
  return d;
}

// Largest row abs-sum of L (the per-column band uses it for every row of the column).
template <class L>
__host__ __device__ constexpr float max_row_abs_sum() {
  int m = 0;
  for (int i = 0; i < L::R; ++i) {
    int s = 0;
    for (int l = 0; l < L::C; ++l) s += L::e(i, l) < 0 ? -L::e(i, l) : L::e(i, l);
    m = s > m ? s : m;
  }
  return (float)m;
}

template <class L>
__host__ __device__ constexpr float row_abs_sum(int i) {
  int s = 0;
  for (int l = 0; l < L::C; ++l) s += L::e(i, l) < 0 ? -L::e(i, l) : L::e(i, l);
  return (float)s;
}

// Compile-time sandwich out = L . X . L^T with L a tab:: matrix (R x C), X (C x C).
template <class L, typename TO>
__device__ __forceinline__ void sandwich(const int (&X)[L::C][L::C], TO (&out)[L::R][L::R]) {
  int tmp[L::C][L::R];
#pragma unroll
  for (int i = 0; i < L::C; ++i)
#pragma unroll
    for (int j = 0; j < L::R; ++j) {
      int s = 0;
#pragma unroll
      for (int l = 0; l < L::C; ++l) s += X[i][l] * L::e(j, l);
      tmp[i][j] = s;
    }
#pragma unroll
  for (int i = 0; i < L::R; ++i)
#pragma unroll
    for (int j = 0; j < L::R; ++j) {
      TO s = 0;
#pragma unroll
      for (int l = 0; l < L::C; ++l) s += (TO)L::e(i, l) * (TO)tmp[l][j];
      out[i][j] = s;
    }
}

}  // namespace wl
