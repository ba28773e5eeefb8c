// Forward-path kernels of the quantized Winograd F(4x4,3x3) layer (canonical or Legendre base).
//
// Reference dataflow (pipeline.py:106-158 with the cast hook of quantize.py:129-148):
//   input -> [input_base_change] -> input_transform -> hadamard -> [output_base_change] -> output
// Every stage is an integer sandwich D*L . codes . (D*L)^T of the previous stage's codes; each
// stage needs its global max before its codes exist, so every kernel below is one pass of the
// dependency chain: it recomputes what it needs from the last materialised codes, reduces the
// current stage's max (and replays the argmax in fp64), or emits codes.
//
// Data layout in HBM (workspace):
//   c0  int8 [N][H][W][Cp]     input codes, channel-last so (tile, channel) threads coalesce
//   V   int8 [T][36][Cp]       input-transform codes, GEMM A operand (K-major)
//   U   int8 [Kp][36][Cp]      weight-transform codes, GEMM B operand (K-major, cached)
//   h   int8|int16 [T][36][Kp] hadamard codes (c1 [T][36][Cp], c4 [T][36][Kp] likewise)
// Cp, Kp are powers of two (>= 32 / 64, <= 512) so the 36 element offsets of a unit are
// compile-time immediates in the templated kernels.
//   acc Acc [groups][9]        per-group stage maxima
// T = N * TP tiles, TP = ceil(Ho/4)*ceil(Wo/4); element xi = 6*i + j of a 6x6 tile.
#pragma once
#include "wl_core.cuh"
#include "wl_f2.cuh"

namespace wl {

// Division by a run-time invariant d for 0 <= n < 2^31: q = (umulhi(n, m) + n) >> s
// (Granlund-Montgomery; m, s set on the host by make_fastdiv).  Replaces the ~20-instruction
// integer division sequences in the per-unit index math.
struct FastDiv {
  unsigned d, m, s;
  __device__ __forceinline__ unsigned div(unsigned n) const { return (__umulhi(n, m) + n) >> s; }
  __device__ __forceinline__ unsigned mod(unsigned n) const { return n - div(n) * d; }
};

struct Geo {
  int N, C, K, H, W, pad, Ho, Wo, th, tw, TP, T, Cp, Kp, ipg;
  int lazy;  // few scale groups: group maxima are written with the read-first atomic (lazy_max)
  FastDiv fTP, ftw, fipg, fC, fK;
};

struct Bits {
  int q[ST_COUNT];  // qmax per stage id
};


__device__ __forceinline__ int group_of_image(int n, const Geo& g) { return (int)g.fipg.div((unsigned)n); }

// ---------------------------------------------------------------------------------- input side

// max|x| per group (cast "input", quantize.py:141).  x is NCHW fp32 or fp64; grid.y = image.
// The group max is kept as fp64 bits in Acc::M (monotone for non-negative values).
__device__ __forceinline__ unsigned long long abs_bits(float v) { return __float_as_uint(fabsf(v)); }
__device__ __forceinline__ unsigned long long abs_bits(double v) {
  return (unsigned long long)__double_as_longlong(fabs(v));
}
template <typename XT>
__device__ __forceinline__ unsigned long long max_to_f64_bits(unsigned long long m) {
  if constexpr (sizeof(XT) == 4)
    return (unsigned long long)__double_as_longlong((double)__uint_as_float((unsigned)m));
  else
    return m;
}

template <typename XT>
__global__ void absmax_input_kernel(const XT* __restrict__ x, long long per_image, int ipg, Acc* acc) {
  const int n = blockIdx.y;
  const XT* xi = x + (size_t)n * per_image;
  unsigned long long m = 0;
  const bool vec = sizeof(XT) == 4 && (per_image % 4 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
  if (vec) {
    const float4* x4 = reinterpret_cast<const float4*>(xi);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < per_image / 4;
         i += (long long)gridDim.x * blockDim.x) {
      float4 v = __ldg(&x4[i]);
      m = max(m, abs_bits(v.x));
      m = max(m, abs_bits(v.y));
      m = max(m, abs_bits(v.z));
      m = max(m, abs_bits(v.w));
    }
  } else {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < per_image;
         i += (long long)gridDim.x * blockDim.x)
      m = max(m, abs_bits(__ldg(&xi[i])));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ unsigned long long sm[32];
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0 && m) atomicMax(&acc[(size_t)(n / ipg) * ST_COUNT + ST_INPUT].M, max_to_f64_bits<XT>(m));
  }
}

// c0 = rint(x / s0) (quantize.py:118-119), NCHW fp32 -> NHWC int8.  Block = (row h, image n):
// threads sweep (channel, 4-pixel chunk) with float4 loads, round with the magic-number fma (the
// exact fp64 division of the reference only within 2^-20 of a half-integer), and deposit codes in a
// shared row buffer [w][Cp+16] that is copied out as 16-byte vectors.
__device__ __forceinline__ int quant_code(float v, float rc, float thr, double scale, int qmax) {
  const float a = fabsf(v);
  const float y = fmaf(a, rc, kMagic);
  const float k = y - kMagic;
  int c = __float_as_int(y) - 0x4B400000;
  if (fabsf(fmaf(a, rc, -k)) > thr) {  // near a half-integer: the reference's fp64 quotient decides
    double d = rint((double)a / scale);
    c = (int)(d > qmax ? qmax : d);
  }
  c = c > qmax ? qmax : c;
  return v < 0.f ? -c : c;
}
// Fast path of quant_code: the fp32 magic-number code, `bad` set when the exact path must decide.
__device__ __forceinline__ int quant_fast(float v, float rc, float thr, int qmax, bool& bad) {
  const float a = fabsf(v);
  const float y = fmaf(a, rc, kMagic);
  const float k = y - kMagic;
  bad |= fabsf(fmaf(a, rc, -k)) > thr;
  const int c = min(__float_as_int(y) - 0x4B400000, qmax);
  return v < 0.f ? -c : c;
}
__device__ __forceinline__ int quant_code(double v, float, float, double scale, int qmax) {
  double d = rint(__ddiv_rn(v, scale));  // quantize.py:118-119 in the reference's own precision
  d = d > qmax ? qmax : d;
  d = d < -qmax ? -qmax : d;
  return (int)d;
}

template <typename XT>
__global__ void __launch_bounds__(256) quant_input_kernel(const XT* __restrict__ x, int8_t* __restrict__ c0, Geo g,
                                                          Bits b, const Acc* __restrict__ acc, int kQuantRowW) {
  extern __shared__ __align__(16) int8_t srow[];
  const int h = blockIdx.x, n = blockIdx.y;
  const StageQ q = load_float_stage(acc[(size_t)group_of_image(n, g) * ST_COUNT + ST_INPUT], b.q[ST_INPUT]);
  const float rc = q.maxabs > 0.0 ? (float)((double)q.qmax / q.maxabs) : 0.f;
  // fast-path error: rc relative 2^-24 on a value <= qmax, plus the fma rounding of the distance
  const float thr = 0.5f - (float)((q.qmax + 1) * 1.25 * 5.9604644775390625e-8);
  const int ld = g.Cp + 16;
  const bool vec = sizeof(XT) == 4 && (g.W & 3) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  for (int w0 = 0; w0 < g.W; w0 += kQuantRowW) {
    const int wn = min(kQuantRowW, g.W - w0);
    if (vec) {
      const int w4n = wn >> 2;
      for (int i = threadIdx.x; i < g.Cp * w4n; i += blockDim.x) {
        const int c = i / w4n, w4 = i - c * w4n;
        int8_t* dst = srow + (4 * w4) * ld + c;
        if (c < g.C) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(
                                     reinterpret_cast<const float*>(x) + (((size_t)n * g.C + c) * g.H + h) * g.W + w0) +
                                 w4);
          dst[0] = (int8_t)quant_code(v.x, rc, thr, q.scale, q.qmax);
          dst[ld] = (int8_t)quant_code(v.y, rc, thr, q.scale, q.qmax);
          dst[2 * ld] = (int8_t)quant_code(v.z, rc, thr, q.scale, q.qmax);
          dst[3 * ld] = (int8_t)quant_code(v.w, rc, thr, q.scale, q.qmax);
        } else {
          dst[0] = dst[ld] = dst[2 * ld] = dst[3 * ld] = 0;
        }
      }
    } else {
      for (int i = threadIdx.x; i < g.Cp * wn; i += blockDim.x) {
        const int c = i / wn, w = i - c * wn;
        srow[w * ld + c] = c < g.C ? (int8_t)quant_code(__ldg(x + (((size_t)n * g.C + c) * g.H + h) * g.W + w0 + w),
                                                        rc, thr, q.scale, q.qmax)
                                   : (int8_t)0;
      }
    }
    __syncthreads();
    int4* dst = reinterpret_cast<int4*>(c0 + (((size_t)n * g.H + h) * g.W + w0) * g.Cp);
    const int vpr = g.Cp >> 4;  // 16-byte vectors per pixel row
    for (int i = threadIdx.x; i < wn * vpr; i += blockDim.x) {
      const int w = i / vpr, j = i - w * vpr;
      dst[i] = *reinterpret_cast<const int4*>(srow + w * ld + 16 * j);
    }
    __syncthreads();
  }
}

// fp32 input, W % 4 == 0, W <= 64: block = (band of rh image rows, image n).  Per channel the band is one
// contiguous run of rh * W floats of x (DRAM efficiency follows the length of such runs: row-sized
// 224-byte pieces read at 5.1 TB/s, 4-row bands faster; tools/probe_ywrite.cu measured the same effect
// on NCHW writes).  Thread = (float4 i of the band, channel group of 4): it quantises a 4x4 (channel x
// pixel) block from 4 coalesced float4 loads, transposes it in registers into one 32-bit word per pixel
// (4 channels, PRMT) and stores the words into a [rh * W][Cp + 4] shared band (2-way bank conflicts at
// worst); the band leaves as coalesced 32-bit words (one contiguous rh * W * Cp byte range of c0).
// ~12 instructions per element (the generic kernel's per-item division and byte stores cost ~30).
#ifndef WL_QI_MINB
#define WL_QI_MINB 4
#endif
__device__ __forceinline__ void quant_rows_w64(const float* __restrict__ x, int8_t* __restrict__ c0, const Geo& g,
                                               const StageQ& q, int h0, int rh, int n, int8_t* srow) {
  const float rc = q.maxabs > 0.0 ? (float)((double)q.qmax / q.maxabs) : 0.f;
  const float thr = 0.5f - (float)((q.qmax + 1) * 1.25 * 5.9604644775390625e-8);
  const int ld = g.Cp + 4;
  const int nrow = min(rh, g.H - h0);
  const int nf4 = (nrow * g.W) >> 2, ncg = g.Cp >> 2;  // float4s per channel band, channel groups
  const int i = threadIdx.x % nf4, cg0 = threadIdx.x / nf4, cgstep = blockDim.x / nf4;
  if (cg0 < cgstep) {
    const size_t cstride = (size_t)g.H * g.W;
    const float* xb = x + ((size_t)n * g.C * g.H + h0) * g.W + 4 * i;
    // the channel-group pointer advances by a constant stride (the clamped tail group recomputes its four)
    const float* pc = xb + (size_t)(4 * cg0) * cstride;
    const size_t pstep = (size_t)4 * cgstep * cstride;
    int8_t* sdst = srow + (4 * i) * ld + 4 * cg0;
#pragma unroll 2
    for (int cg = cg0; cg < ncg; cg += cgstep, sdst += 4 * cgstep, pc += pstep) {
      // all four loads first (clamped channel, discarded below) so they are in flight together
      float4 v[4];
      if (4 * cg + 3 < g.C) {
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = __ldg(reinterpret_cast<const float4*>(pc + (size_t)u * cstride));
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          v[u] = __ldg(reinterpret_cast<const float4*>(xb + (size_t)min(4 * cg + u, g.C - 1) * cstride));
      }
      // pixel pairs on packed f32x2: y = fma(v, rc, 1.5 * 2^23) holds the signed half-even code in its low
      // byte (rint is odd-symmetric, so this equals the sign * rint(|v| * rc) of quant_fast); d = fma(v,
      // -rc, k) is the distance to that integer.  |v| * rc <= qmax * (1 + 2^-24), so no clamp is needed.
      uint32_t wd[4] = {0u, 0u, 0u, 0u};
      constexpr uint32_t kSel[4] = {0x3214u, 0x3240u, 0x3410u, 0x4210u};  // byte u of word p <- low byte of code
      const f2 rc2 = bc2(rc), nrc2 = bc2(-rc), mg = bc2(kMagic);
      float dmax = 0.f;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (4 * cg + u < g.C) {
          const f2 va = mk2(v[u].x, v[u].y), vb = mk2(v[u].z, v[u].w);
          const f2 ya = fma2(va, rc2, mg), yb = fma2(vb, rc2, mg);
          const f2 da = fma2(va, nrc2, sub2(ya, mg)), db = fma2(vb, nrc2, sub2(yb, mg));
          dmax = fmaxf(dmax, fmaxf(fmaxf(fabsf(lo2(da)), fabsf(hi2(da))), fmaxf(fabsf(lo2(db)), fabsf(hi2(db)))));
          wd[0] = __byte_perm(wd[0], __float_as_uint(lo2(ya)), kSel[u]);
          wd[1] = __byte_perm(wd[1], __float_as_uint(hi2(ya)), kSel[u]);
          wd[2] = __byte_perm(wd[2], __float_as_uint(lo2(yb)), kSel[u]);
          wd[3] = __byte_perm(wd[3], __float_as_uint(hi2(yb)), kSel[u]);
        }
      }
      if (dmax > thr) {  // some element within the fp32 band of a half-integer: the exact path decides
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (4 * cg + u < g.C) {
            wd[0] = __byte_perm(wd[0], (uint32_t)quant_code(v[u].x, rc, thr, q.scale, q.qmax), kSel[u]);
            wd[1] = __byte_perm(wd[1], (uint32_t)quant_code(v[u].y, rc, thr, q.scale, q.qmax), kSel[u]);
            wd[2] = __byte_perm(wd[2], (uint32_t)quant_code(v[u].z, rc, thr, q.scale, q.qmax), kSel[u]);
            wd[3] = __byte_perm(wd[3], (uint32_t)quant_code(v[u].w, rc, thr, q.scale, q.qmax), kSel[u]);
          }
      }
#pragma unroll
      for (int p = 0; p < 4; ++p) *reinterpret_cast<uint32_t*>(sdst + p * ld) = wd[p];
    }
  }
  __syncthreads();
  uint32_t* dst = reinterpret_cast<uint32_t*>(c0 + ((size_t)n * g.H + h0) * g.W * g.Cp);
  const int wpr = g.Cp >> 2, lw = __ffs(wpr) - 1;  // 32-bit words per pixel (a power of two)
  const int total = nrow * g.W * wpr;
  if (wpr <= (int)blockDim.x && (blockDim.x & (wpr - 1)) == 0) {
    // the block width is a multiple of the words per pixel: a thread keeps its word column, pixels advance
    // by blockDim / wpr per step
    const int pstride = (int)blockDim.x >> lw;
    const int8_t* sp = srow + (threadIdx.x >> lw) * ld + 4 * (threadIdx.x & (wpr - 1));
    uint32_t* dp = dst + threadIdx.x;
    const int sstep = pstride * ld;
    int j = threadIdx.x;
#pragma unroll 4
    for (; j < total; j += blockDim.x, sp += sstep, dp += blockDim.x) *dp = *reinterpret_cast<const uint32_t*>(sp);
  } else {
    for (int j = threadIdx.x; j < total; j += blockDim.x) {
      const int pix = j >> lw, jw = j & (wpr - 1);
      dst[j] = *reinterpret_cast<const uint32_t*>(srow + pix * ld + 4 * jw);
    }
  }
}

template <int kInTU = 0>  // header-defined kernel: instantiated only in the TUs that launch it
__global__ void __launch_bounds__(256, WL_QI_MINB) quant_input_w64_kernel(const float* __restrict__ x, int8_t* __restrict__ c0,
                                                              Geo g, Bits b, const Acc* __restrict__ acc, int rh) {
  extern __shared__ __align__(16) int8_t srow[];
  const int h0 = blockIdx.x * rh, n = blockIdx.y;
  const StageQ q = load_float_stage(acc[(size_t)group_of_image(n, g) * ST_COUNT + ST_INPUT], b.q[ST_INPUT]);
  quant_rows_w64(x, c0, g, q, h0, rh, n, srow);
}

// Fused cast "input" for fp32 x with W % 4 == 0 and W <= 64: one launch that reads x from HBM once.
// Block = one band of rh rows, taken from an atomic ticket (tickets start in order, so every block with a
// smaller ticket is resident or done).  Ticket t reduces max|x| of band t % nb of image n1 = t / nb into the
// group's Acc::M and arrives on the group's counter; then it quantises the same band of image n2 = n1 - lag
// exactly as quant_input_w64_kernel does, after checking that n2's group is complete.  lag >= images per
// group, so a block only ever waits for smaller tickets, whose reductions wait for nothing: no deadlock
// whatever the number of resident blocks.  The second read of a band follows the first by lag images
// (lag * C * H * W * 4 bytes of other traffic, a few tens of MB): an L2 hit.
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
struct CastShared {
  double maxabs, scale;
  float rcp;
  unsigned ticket;
  unsigned wmax[8];
};
template <int kInTU = 0>
__global__ void __launch_bounds__(256, WL_QI_MINB) cast_input_w64_kernel(const float* __restrict__ x, int8_t* __restrict__ c0,
                                                             Geo g, Bits b, Acc* acc, int rh, int lag, unsigned* sync) {
  extern __shared__ __align__(16) int8_t srow[];
  __shared__ CastShared cs;
  if (threadIdx.x == 0) cs.ticket = atomicAdd(&sync[0], 1u);
  __syncthreads();
  const int nb = (g.H + rh - 1) / rh;
  const int n1 = (int)(cs.ticket / (unsigned)nb), h0 = (int)(cs.ticket - (unsigned)n1 * nb) * rh, n2 = n1 - lag;
  if (n1 < g.N) {
    const int nrow = min(rh, g.H - h0);
#ifndef WL_CAST_NOPF
    // the whole band is requested from DRAM at once (per-line L2 prefetches: the bulk form is a uniform-datapath
    // instruction that the compiler serialises over the lanes); the loads below
    // then find their lines in L2 or in flight instead of exposing DRAM latency 8 loads at a time
    for (int ch = threadIdx.x; ch < g.C; ch += blockDim.x) {
      const char* run = reinterpret_cast<const char*>(x + (((size_t)n1 * g.C + ch) * g.H + h0) * g.W);
      const int bytes = nrow * g.W * 4;
      for (int o = 0; o < bytes; o += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(run + o));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(run + bytes - 4));
    }
#endif
    const int nf4 = (nrow * g.W) >> 2, ncg = g.Cp >> 2;
    const int i = threadIdx.x % nf4, cg0 = threadIdx.x / nf4, cgstep = blockDim.x / nf4;
    unsigned m = 0;
    if (cg0 < cgstep) {
      // per channel one pointer; max over the sign-cleared bit patterns (monotone for non-negative floats)
      const size_t cstride = (size_t)g.H * g.W;
      const float* pch = x + ((size_t)n1 * g.C * g.H + h0) * g.W + 4 * i + (size_t)(4 * cg0) * cstride;
      const size_t pstep = (size_t)4 * cgstep * cstride;
      unsigned ma = 0, mb = 0;
#pragma unroll 2
      for (int cg = cg0; cg < ncg; cg += cgstep, pch += pstep) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          v[u] = 4 * cg + u < g.C ? __ldg(reinterpret_cast<const uint4*>(pch + (size_t)u * cstride)) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          ma = max(ma, max(v[u].x & 0x7fffffffu, v[u].y & 0x7fffffffu));
          mb = max(mb, max(v[u].z & 0x7fffffffu, v[u].w & 0x7fffffffu));
        }
      }
      m = max(ma, mb);
    }
    m = __reduce_max_sync(0xffffffffu, m);
    if ((threadIdx.x & 31) == 0) cs.wmax[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {  // arrive: nobody in this block waits for it (lag >= 1)
#pragma unroll
      for (int w = 1; w < 8; ++w) m = max(m, cs.wmax[w]);
      const int grp = group_of_image(n1, g);
      if (m) atomicMax(&acc[(size_t)grp * ST_COUNT + ST_INPUT].M, max_to_f64_bits<float>(m));
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&sync[1 + grp]) : "memory");
    }
  }
  if (n2 < 0) return;
  if (threadIdx.x == 32) {  // another warp than the arriving one: the two round trips overlap
    const int grp = group_of_image(n2, g);
    const unsigned target = (unsigned)nb * (unsigned)min(g.ipg, g.N - grp * g.ipg);
    while (ld_acquire_u32(&sync[1 + grp]) < target) __nanosleep(32);
    Acc a;
    a.M = __ldcg(&acc[(size_t)grp * ST_COUNT + ST_INPUT].M);
    const StageQ q = load_float_stage(a, b.q[ST_INPUT]);
    cs.maxabs = q.maxabs;
    cs.scale = q.scale;
    cs.rcp = q.rcp;
  }
  __syncthreads();
  StageQ q;
  q.M = 0;
  q.maxabs = cs.maxabs;
  q.scale = cs.scale;
  q.rcp = cs.rcp;
  q.qmax = b.q[ST_INPUT];
  quant_rows_w64(x, c0, g, q, h0, rh, n2, srow);
}

__device__ __forceinline__ void load_input_tile(const int8_t* __restrict__ c0, const Geo& g, int n, int tile, int c,
                                                int (&X)[6][6]) {
  const int ty = (int)g.ftw.div((unsigned)tile), tx = (int)g.ftw.mod((unsigned)tile);
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    const int r = 4 * ty + i - g.pad;
#pragma unroll
    for (int j = 0; j < 6; ++j) {
      const int col = 4 * tx + j - g.pad;
      X[i][j] = (r >= 0 && r < g.H && col >= 0 && col < g.W)
                    ? (int)__ldg(&c0[(((size_t)n * g.H + r) * g.W + col) * g.Cp + c])
                    : 0;
    }
  }
}

template <typename TT>
__device__ __forceinline__ long long absmax36(const TT (&T)[6][6]) {
  long long m = 0;
#pragma unroll
  for (int i = 0; i < 6; ++i)
#pragma unroll
    for (int j = 0; j < 6; ++j) {
      long long a = (long long)T[i][j];
      a = a < 0 ? -a : a;
      m = a > m ? a : m;
    }
  return m;
}

// Requantise a 6x6 int32 stage tensor into codes; exact ties are replayed from the stage's own
// input codes `Xin` (dequantised with `qin`) through the fp64 matrix `Lf`.
template <typename TT>
__device__ __forceinline__ void requant36(const TT (&T)[6][6], const StageQ& q, const int (&Xin)[6][6],
                                          const StageQ& qin, const double* __restrict__ Lf, int (&out)[6][6]) {
  bool any_tie = false;
  bool tie[6][6];
#pragma unroll
  for (int i = 0; i < 6; ++i)
#pragma unroll
    for (int j = 0; j < 6; ++j) {
      bool t = false;
      out[i][j] = rq((long long)T[i][j], q, t);
      tie[i][j] = t;
      any_tie |= t;
    }
  if (any_tie) {
    int xc[36];
#pragma unroll
    for (int e = 0; e < 36; ++e) xc[e] = Xin[e / 6][e % 6];
    for (int e = 0; e < 36; ++e)
      if (tie[e / 6][e % 6])
        out[e / 6][e % 6] =
            code_of(replay_sandwich(Lf, 6, 6, xc, qin.qmax, qin.maxabs, qin.scale, e / 6, e % 6), q);
  }
}

// Reduce one thread's 6x6 stage tensor into the group max; replay the local argmax in fp64.
template <typename TT>
__device__ __forceinline__ void reduce36(const TT (&T)[6][6], int grp, bool active, Acc* acc, int stage,
                                         const int (&Xin)[6][6], const StageQ& qin, const double* __restrict__ Lf,
                                         int R) {
  const long long m = active ? absmax36(T) : 0;
  bool uniform;
  long long wmax;
  Acc* a = acc + stage;
  if (replay_gate(m, active ? grp : -1, a, ST_COUNT, uniform, wmax)) {
    int xc[36];
#pragma unroll
    for (int e = 0; e < 36; ++e) xc[e] = Xin[e / 6][e % 6];
    double f = 0.0;
    for (int e = 0; e < R * R; ++e) {
      long long v = (long long)T[e / R][e % R];
      if ((v < 0 ? -v : v) == m) f = fmax(f, fabs(replay_sandwich(Lf, R, 6, xc, qin.qmax, qin.maxabs, qin.scale, e / R, e % R)));
    }
    atomicMax(&a[(size_t)grp * ST_COUNT].F, dbits(f));
  }
  publish_max(m, active ? grp : -1, a, ST_COUNT, uniform, wmax);
}

// ---------------------------------------------------------------------------------- weight side

// Thread per (out channel k, in channel c), c fastest.  PASS 0: weight_transform max; PASS 1
// (Legendre): weight_base_change max; PASS 2: emit U codes [36][Kp][Cp].
template <int MODE, int PASS, typename XT>
__global__ void __launch_bounds__(256) weight_stage_kernel(const XT* __restrict__ w, int K, int C, int Kp, int Cp,
                                                           int8_t* __restrict__ U, Bits b, Acc* __restrict__ wacc,
                                                           const PlanF64* __restrict__ pf) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = idx < K * C;
  const int id = active ? idx : 0;
  const int c = id % C, k = id / C;
  const StageQ qw = load_float_stage(wacc[ST_WEIGHTS], b.q[ST_WEIGHTS]);
  int X[3][3];
#pragma unroll
  for (int i = 0; i < 9; ++i) X[i / 3][i % 3] = quant_float(__ldg(&w[(size_t)id * 9 + i]), qw);
  int xc[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) xc[i] = X[i / 3][i % 3];
  int U1[6][6];
  const double* Lwt = pf->wt;
  if constexpr (MODE == 0)
    sandwich<tab::Can_WT>(X, U1);
  else
    sandwich<tab::Leg_WT>(X, U1);
  if constexpr (PASS == 0) {
    const long long m = active ? absmax36(U1) : 0;
    bool uniform;
    long long wmax;
    if (replay_gate(m, active ? 0 : -1, wacc + ST_WT, ST_COUNT, uniform, wmax)) {
      double f = 0.0;
      for (int e = 0; e < 36; ++e) {
        long long v = U1[e / 6][e % 6];
        if ((v < 0 ? -v : v) == m)
          f = fmax(f, fabs(replay_sandwich(Lwt, 6, 3, xc, qw.qmax, qw.maxabs, qw.scale, e / 6, e % 6)));
      }
      atomicMax(&wacc[ST_WT].F, dbits(f));
    }
    publish_max(m, active ? 0 : -1, wacc + ST_WT, ST_COUNT, uniform, wmax);
    return;
  }
  const StageQ q1 = load_int_stage(wacc[ST_WT], b.q[ST_WT]);
  int C1[6][6];
  {
    bool tie[36];
    bool any = false;
#pragma unroll
    for (int e = 0; e < 36; ++e) {
      bool t = false;
      C1[e / 6][e % 6] = rq(U1[e / 6][e % 6], q1, t);
      tie[e] = t;
      any |= t;
    }
    if (any)
      for (int e = 0; e < 36; ++e)
        if (tie[e])
          C1[e / 6][e % 6] = code_of(replay_sandwich(Lwt, 6, 3, xc, qw.qmax, qw.maxabs, qw.scale, e / 6, e % 6), q1);
  }
  if constexpr (MODE == 0) {
    if (active)
#pragma unroll
      for (int e = 0; e < 36; ++e) U[((size_t)k * 36 + e) * Cp + c] = (int8_t)C1[e / 6][e % 6];
  } else {
    int U2[6][6];
    sandwich<tab::Leg_WBC>(C1, U2);
    if constexpr (PASS == 1) {
      reduce36(U2, 0, active, wacc, ST_WBC, C1, q1, pf->wbc, 6);
    } else {
      const StageQ q2 = load_int_stage(wacc[ST_WBC], b.q[ST_WBC]);
      int C2[6][6];
      requant36(U2, q2, C1, q1, pf->wbc, C2);
      if (active)
#pragma unroll
        for (int e = 0; e < 36; ++e) U[((size_t)k * 36 + e) * Cp + c] = (int8_t)C2[e / 6][e % 6];
    }
  }
}

template <typename XT>
__global__ void absmax_weights_kernel(const XT* __restrict__ w, long long n, Acc* wacc) {
  unsigned long long m = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    m = max(m, abs_bits(__ldg(&w[i])));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(&wacc[ST_WEIGHTS].M, max_to_f64_bits<XT>(m));
}

// ---------------------------------------------------------------------------------- output side

template <typename HT>
__device__ __forceinline__ void load_h(const HT* __restrict__ h, const Geo& g, int t, int k, int (&X)[6][6]) {
#pragma unroll
  for (int e = 0; e < 36; ++e) X[e / 6][e % 6] = (int)h[((size_t)e * g.T + t) * g.Kp + k];
}

// 4x4 output tile, crop-aware reduction (pipeline.py:156-158: crop before the final cast).
template <typename TT>
__device__ __forceinline__ long long absmax_crop(const TT (&Y)[4][4], int ty, int tx, const Geo& g) {
  long long m = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (4 * ty + i < g.Ho && 4 * tx + j < g.Wo) {
        long long a = (long long)Y[i][j];
        a = a < 0 ? -a : a;
        m = a > m ? a : m;
      }
    }
  return m;
}

}  // namespace wl
