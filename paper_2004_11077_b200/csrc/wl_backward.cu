// Straight-through-estimator backward of the quantized Winograd layer.
// The reference has no backward; this defines it: every fake-quant cast is the identity in
// backward with detached scales, the products use the forward's QUANTISED operands (U, V codes
// times their stage scale), and — since every Legendre composite equals the canonical transform in
// exact arithmetic (pipeline.py:9-11: P^-1 A_P = A, P^-1 B_P = B, P^-1 G_P = G) — both bases use
//   dM  = A . dY . A^T                       (6x6 per (tile, out channel))
//   dV  = sum_k U_k (.) dM_k,  dU = sum_t V_t (.) dM_t   (two 36-way batched GEMMs on tcgen05)
//   dX  = col2im( B . dV . B^T )             (gather over the <= 2x2 tiles covering a pixel)
//   dW  = G^T . dU . G,   db = sum dY
// GEMMs (gemm_bf16.cuh): the codes are exact in bf16, dM is carried as three bf16 planes
// (hi + mid + lo == fp32), fp32 accumulation in TMEM.  dV = dM . U^T over K (one pass);
// dU^T = V^T . (s_v dM) over the tiles, split into <= 4096-tile chunks whose partial sums are
// added in fp64 by the dW kernel.  The per-image V scale s_v is folded into dM's planes, the
// weight scale s_u into the dX transform.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/winoleg_b200.h"
#include "gemm_bf16.cuh"
#include "wl_backward.h"
#include "wl_gemm_bf16.h"

namespace wl {
namespace bw {

// canonical F(4,3) matrices (the reference's A, B^T, G; construct.py:161-181)
// compile-time coefficients: the unrolled sandwiches drop the zero terms (a third of A's and half of B's
// entries; fma(x, 0, s) cannot be folded by the compiler because of NaN / Inf semantics)
__host__ __device__ constexpr float kAT(int i, int j) {
  constexpr float v[4][6] = {{1, 1, 1, 1, 1, 0}, {0, 1, -1, 2, -2, 0}, {0, 1, 1, 4, 4, 0}, {0, 1, -1, 8, -8, 1}};
  return v[i][j];
}
__host__ __device__ constexpr float kBT(int i, int j) {
  constexpr float v[6][6] = {{4, 0, -5, 0, 1, 0},  {0, -4, -4, 1, 1, 0}, {0, 4, -4, -1, 1, 0},
                             {0, -2, -1, 2, 1, 0}, {0, 2, -1, -2, 1, 0}, {0, 4, 0, -5, 0, 1}};
  return v[i][j];
}
__constant__ double kG[6][3] = {{0.25, 0, 0},
                                {-1.0 / 6, -1.0 / 6, -1.0 / 6},
                                {-1.0 / 6, 1.0 / 6, -1.0 / 6},
                                {1.0 / 24, 1.0 / 12, 1.0 / 6},
                                {1.0 / 24, -1.0 / 12, 1.0 / 6},
                                {0, 0, 1}};

struct Work {  // workspace carve-up (wl_bw_workspace_bytes)
  __nv_bfloat16 *dmA, *dmB, *ut, *vt;
  float *dv, *dup, *dxt;
  int Kpad, Tpad, S, ks;
};

// dM of tile t, output channel k: A . dY_tile . A^T, dY cropped to the valid output.
__device__ __forceinline__ void dm_tile(const float* __restrict__ dy, const BwGeo& g, int t, int k, float (&out)[36]) {
  const int n = t / g.TP, tile = t % g.TP, ty = tile / g.tw, tx = tile % g.tw;
  float Y[4][4];
  const float* src = dy + (((size_t)n * g.K + k) * g.Ho + 4 * ty) * g.Wo + 4 * tx;
  if ((g.Wo & 3) == 0 && (reinterpret_cast<uintptr_t>(dy) & 15) == 0) {
    // whole tile rows: one 16-byte load per row (the lanes of a warp read different channels or tiles, so a
    // scalar load is a 32-sector request: four of them per row kept the L1 at 75 % for 31 % of the DRAM rate)
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (4 * ty + a < g.Ho) v = __ldg(reinterpret_cast<const float4*>(src + (size_t)a * g.Wo));
      Y[a][0] = v.x, Y[a][1] = v.y, Y[a][2] = v.z, Y[a][3] = v.w;
    }
  } else {
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b)
        Y[a][b] = (4 * ty + a < g.Ho && 4 * tx + b < g.Wo) ? __ldg(src + (size_t)a * g.Wo + b) : 0.f;
  }
  float tmp[4][6];  // dY . A^T
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int j = 0; j < 6; ++j) {
      float s = 0.f;
#pragma unroll
      for (int b = 0; b < 4; ++b)
        if (kAT(b, j) != 0.f) s = fmaf(Y[a][b], kAT(b, j), s);
      tmp[a][j] = s;
    }
#pragma unroll
  for (int i = 0; i < 6; ++i)
#pragma unroll
    for (int j = 0; j < 6; ++j) {
      float s = 0.f;
#pragma unroll
      for (int a = 0; a < 4; ++a)
        if (kAT(a, i) != 0.f) s = fmaf(kAT(a, i), tmp[a][j], s);
      out[6 * i + j] = s;
    }
}

// GEMM operand of dV: dM planes [3][36][T][Kpad] (k fastest: coalesced plane stores), zero padded.
__global__ void dm_rows_kernel(const float* __restrict__ dy, __nv_bfloat16* __restrict__ dmA, BwGeo g, int Kpad) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)g.T * Kpad) return;
  const int k = (int)(idx % Kpad), t = (int)(idx / Kpad);
  float m[36];
  if (k < g.K) {
    dm_tile(dy, g, t, k, m);
  } else {
#pragma unroll
    for (int e = 0; e < 36; ++e) m[e] = 0.f;
  }
  const size_t plane = (size_t)36 * g.T * Kpad;
#pragma unroll
  for (int e = 0; e < 36; ++e) {
    __nv_bfloat16 h, md, l;
    wl_split3(m[e], h, md, l);
    const size_t o = ((size_t)e * g.T + t) * Kpad + k;
    dmA[o] = h;
    dmA[plane + o] = md;
    dmA[2 * plane + o] = l;
  }
}

// GEMM operand of dU^T: s_v(t) * dM as planes [3][36][K][Tpad] (t fastest), zero padded.
__global__ void dm_cols_kernel(const float* __restrict__ dy, __nv_bfloat16* __restrict__ dmB, BwGeo g, int Tpad,
                               const Acc* __restrict__ acc) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)Tpad * g.K) return;
  const int t = (int)(idx % Tpad), k = (int)(idx / Tpad);
  float m[36];
  if (t < g.T) {
    dm_tile(dy, g, t, k, m);
    const float sv = (float)acc[(size_t)((t / g.TP) / g.ipg) * ST_COUNT + ST_IT].scale;
#pragma unroll
    for (int e = 0; e < 36; ++e) m[e] *= sv;
  } else {
#pragma unroll
    for (int e = 0; e < 36; ++e) m[e] = 0.f;
  }
  const size_t plane = (size_t)36 * g.K * Tpad;
#pragma unroll
  for (int e = 0; e < 36; ++e) {
    __nv_bfloat16 h, md, l;
    wl_split3(m[e], h, md, l);
    const size_t o = ((size_t)e * g.K + k) * Tpad + t;
    dmB[o] = h;
    dmB[plane + o] = md;
    dmB[2 * plane + o] = l;
  }
}

// Codes [rows][36][Cp] int8 -> bf16 [36][C][rows_pad] (exact), rows >= `rows` zero: the GEMM operands U^T
// (rows = K) and V^T (rows = T).  Block = 64 rows x 64 channels of one Winograd element: one 16-byte load per
// thread along the channels into a word-pitched shared tile; then a thread takes 4 rows x 4 channels (four
// 32-bit shared reads, conflict-free), converts bytes straight out of the words and stores, per channel, its
// four rows as one 8-byte piece (8 lanes = 64 bytes of a channel's row run).  3.6 instructions per code; the
// byte-per-thread version ran at 81 % issue-active (69 us on 16384 x 64 codes).
__global__ void __launch_bounds__(256) codes_t_kernel(const int8_t* __restrict__ codes, __nv_bfloat16* __restrict__ out,
                                                      int rows, int rows_pad, int C, int Cp) {
  __shared__ uint32_t sm[64][17];
  const int r0 = blockIdx.x * 64, c0 = blockIdx.y * 64, e = blockIdx.z;
  {
    const int rr = threadIdx.x >> 2, ch = threadIdx.x & 3;  // row of the tile, 16-channel chunk
    const int r = r0 + rr, c = c0 + 16 * ch;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (r < rows && c < Cp) v = __ldg(reinterpret_cast<const uint4*>(codes + ((size_t)r * 36 + e) * Cp + c));
    sm[rr][4 * ch + 0] = v.x;
    sm[rr][4 * ch + 1] = v.y;
    sm[rr][4 * ch + 2] = v.z;
    sm[rr][4 * ch + 3] = v.w;
  }
  __syncthreads();
  // lane -> (8 row quads, 4 channel words): shared bank = (4 * r4 + cw) mod 32, all distinct
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r4 = (lane & 7) + 8 * (warp & 1), cw = (lane >> 3) + 4 * (warp >> 1);
  uint32_t w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) w[i] = sm[4 * r4 + i][cw];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int c = c0 + 4 * cw + j;
    if (c < C) {
      float f[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) f[i] = (float)(int)(int8_t)(w[i] >> (8 * j));
      const __nv_bfloat162 lo = __floats2bfloat162_rn(f[0], f[1]), hi = __floats2bfloat162_rn(f[2], f[3]);
      uint2 o;
      o.x = *reinterpret_cast<const uint32_t*>(&lo);
      o.y = *reinterpret_cast<const uint32_t*>(&hi);
      *reinterpret_cast<uint2*>(out + ((size_t)e * C + c) * rows_pad + r0 + 4 * r4) = o;
    }
  }
}

// dXt = s_u * B . dV_tile . B^T, dV [36][T][C] -> dxt [T][36][C] (c fastest: coalesced both ways).
__global__ void dxt_kernel(const float* __restrict__ dv, float* __restrict__ dxt, BwGeo g, const Acc* __restrict__ wacc,
                           int wstage, int qmax_u) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)g.T * g.C) return;
  const int c = (int)(idx % g.C), t = (int)(idx / g.C);
  const float su = (float)load_int_stage(wacc[wstage], qmax_u).scale;
  float D[6][6];
#pragma unroll
  for (int e = 0; e < 36; ++e) D[e / 6][e % 6] = __ldg(&dv[((size_t)e * g.T + t) * g.C + c]);
  float tmp[6][6];  // dV . B^T  (B^T[b][j] -> B[j][b])
#pragma unroll
  for (int a = 0; a < 6; ++a)
#pragma unroll
    for (int j = 0; j < 6; ++j) {
      float s = 0.f;
#pragma unroll
      for (int b = 0; b < 6; ++b)
        if (kBT(b, j) != 0.f) s = fmaf(D[a][b], kBT(b, j), s);
      tmp[a][j] = s;
    }
#pragma unroll
  for (int i = 0; i < 6; ++i)
#pragma unroll
    for (int j = 0; j < 6; ++j) {
      float s = 0.f;
#pragma unroll
      for (int a = 0; a < 6; ++a)
        if (kBT(a, i) != 0.f) s = fmaf(kBT(a, i), tmp[a][j], s);
      dxt[((size_t)t * 36 + 6 * i + j) * g.C + c] = su * s;
    }
}

// Gather col2im: each input pixel sums the <= 2x2 tile contributions covering it (no atomics).
// Block = (image n, 32 consecutive pixels of its H x W plane, 32 channels): the sums are formed with channels
// across lanes (coalesced dxt reads) and leave through shared memory with pixels across lanes (128-byte runs
// of dx whatever the image width).  A padded coordinate p lies in tile p / 4 at offset p % 4 and, when that
// offset is 0 or 1, also in the tile before it at offset + 4; the (at most four) loads of a pixel are issued
// before their sum, tile rows then tile columns ascending.
template <int PQ>  // a block covers 8 * PQ consecutive pixels (PQ per thread) x 32 channels
__global__ void __launch_bounds__(256) dx_gather_kernel(const float* __restrict__ dxt, float* __restrict__ dx,
                                                        BwGeo g, int pblocks) {
  __shared__ float sm[8 * PQ][33];
  const int n = blockIdx.x / pblocks, p0 = (blockIdx.x % pblocks) * (8 * PQ), c0 = blockIdx.z * 32;
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int HW = g.H * g.W;
  const int c = c0 + lane;
  const int tstride = 36 * g.C;
  const float* base = dxt + (size_t)n * g.TP * tstride + c;
  const int up = g.tw * tstride - 24 * g.C, left = tstride - 4 * g.C;  // one tile up: i + 4; left: j + 4
  float v[PQ][4];
  // (row, col) of this thread's first pixel once, then stepped by 8 pixels: no division per pixel; 32-bit
  // element offsets inside the image's dxt block (TP * 36 * C floats < 2^31, host-checked); the kernel was
  // issue-bound at 85 % issue-active
  int row = (p0 + grp) / g.W, col = (p0 + grp) - row * g.W;
#pragma unroll
  for (int q = 0; q < PQ; ++q) {
    const int p = p0 + grp + 8 * q;
    v[q][0] = v[q][1] = v[q][2] = v[q][3] = 0.f;
    if (c < g.C && p < HW) {
      const int rp = row + g.pad, cp = col + g.pad;
      const int tyA = rp >> 2, iA = rp & 3, txA = cp >> 2, jA = cp & 3;
      const bool vA = tyA < g.th, vB = iA <= 1 && tyA >= 1 && tyA - 1 < g.th;
      const bool wA = txA < g.tw, wB = jA <= 1 && txA >= 1 && txA - 1 < g.tw;
      const int oa = (tyA * g.tw + txA) * tstride + (6 * iA + jA) * g.C;  // tile (tyA, txA)
      if (vB && wB) v[q][0] = __ldg(base + (oa - up - left));
      if (vB && wA) v[q][1] = __ldg(base + (oa - up));
      if (vA && wB) v[q][2] = __ldg(base + (oa - left));
      if (vA && wA) v[q][3] = __ldg(base + oa);
    }
    col += 8;
    while (col >= g.W) col -= g.W, ++row;
  }
#pragma unroll
  for (int q = 0; q < PQ; ++q) sm[grp + 8 * q][lane] = ((v[q][0] + v[q][1]) + v[q][2]) + v[q][3];
  __syncthreads();
  for (int cl = grp; cl < 32; cl += 8) {
    const int cc = c0 + cl;
    if (cc < g.C) {
#pragma unroll
      for (int hh = 0; hh < PQ / 4; ++hh) {
        const int p = p0 + 32 * hh + lane;
        if (p < HW) dx[((size_t)n * g.C + cc) * HW + p] = sm[32 * hh + lane][cl];
      }
    }
  }
}

// dW[k][c] = G^T . dU . G with dU^T[e][c][k] summed over the S split partials in fp64.
// dW = G^T . dU . G per (k, c); the dU partial sums of the S tile splits are added in fp64.  Block = 32 output
// channels x 8 input channels: the partials are read k-fastest (coalesced: [split][36][C][K]); the 9 results of
// each (k, c) go through a shared tile [32 k][8 c * 9] and leave as 288-byte runs of dw [K][C][3][3] (one thread
// per (k, c) storing its 9 floats 36 KB apart cost 162 us on 512 x 512 channels; this version ~20 us).
__global__ void __launch_bounds__(256) dw_kernel(const float* __restrict__ dup, float* __restrict__ dw, BwGeo g, int S) {
  __shared__ float tile[32][8 * 9 + 1];
  __shared__ float stage[36][256];
  const int kx = threadIdx.x & 31, cy = threadIdx.x >> 5;
  const int k0 = blockIdx.x * 32, c0 = blockIdx.y * 8;
  const int k = k0 + kx, c = c0 + cy;
  if (k < g.K && c < g.C) {
    // The 36 partials of one split go through per-thread shared slots as asynchronous copies, so all 36 loads are
    // in flight together: written as plain loads ptxas emits load -> convert -> add a few elements at a time, i.e.
    // ~36 * S serialised L2 latencies per thread (154 us on 512 x 512 channels, 70 us on 64 x 64 with 16 blocks).
    double D[6][6];
#pragma unroll
    for (int e = 0; e < 36; ++e) D[e / 6][e % 6] = 0.0;
    const size_t estride = (size_t)g.C * g.K;
    const float* src = dup + (size_t)c * g.K + k;
    const uint32_t slot = (uint32_t)__cvta_generic_to_shared(&stage[0][threadIdx.x]);
    for (int sp = 0; sp < S; ++sp, src += 36 * estride) {
#pragma unroll
      for (int e = 0; e < 36; ++e)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(slot + e * 256 * 4), "l"(src + e * estride) : "memory");
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
      for (int e = 0; e < 36; ++e) D[e / 6][e % 6] += (double)stage[e][threadIdx.x];
    }
    double tmp[6][3];  // dU . G
#pragma unroll
    for (int a = 0; a < 6; ++a)
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        double s = 0.0;
#pragma unroll
        for (int b = 0; b < 6; ++b) s += D[a][b] * kG[b][q];
        tmp[a][q] = s;
      }
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        double s = 0.0;
#pragma unroll
        for (int a = 0; a < 6; ++a) s += kG[a][p] * tmp[a][q];
        tile[kx][cy * 9 + 3 * p + q] = (float)s;
      }
  }
  __syncthreads();
  const int ncols = min(8, g.C - c0) * 9;  // valid floats of each k row of the tile
  for (int i = threadIdx.x; i < 32 * 72; i += 256) {
    const int row = i / 72, col = i - row * 72;
    if (k0 + row < g.K && col < ncols) dw[((size_t)(k0 + row) * g.C + c0) * 9 + col] = tile[row][col];
  }
}

__global__ void db_kernel(const float* __restrict__ dy, float* __restrict__ db, BwGeo g) {
  const int k = blockIdx.x;
  double s = 0.0;
  const long long per = (long long)g.Ho * g.Wo;
  for (long long i = threadIdx.x; i < (long long)g.N * per; i += blockDim.x) {
    const long long n = i / per, p = i % per;
    s += dy[((size_t)n * g.K + k) * per + p];
  }
  __shared__ double red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) db[k] = (float)s;
  }
}

size_t a256(size_t v) { return (v + 255) & ~size_t(255); }

// dU^T reduction split over the tiles: chunks of <= 4096 tiles (fp32 accumulation length), and
// enough (batch x tile x split) CTAs for two waves.
void splits(const BwGeo& g, int Tpad, int* S, int* ks) {
  const int tiles = 36 * ((g.C + 127) / 128) * ((g.K + 255) / 256);
  int s = std::max((Tpad + 4095) / 4096, (296 + tiles - 1) / tiles);
  s = std::min(s, Tpad / 64);
  s = std::max(s, 1);
  *ks = round_up((Tpad + s - 1) / s, 64);
  *S = (Tpad + *ks - 1) / *ks;
}

size_t carve(const BwGeo& g, void* ws, Work* w) {
  const size_t T = g.T, C = g.C, K = g.K;
  const int Kpad = round_up(g.K, 64), Tpad = round_up(g.T, 64);
  int S, ks;
  splits(g, Tpad, &S, &ks);
  uint8_t* p = reinterpret_cast<uint8_t*>(ws);
  size_t o = 0;
  auto take = [&](size_t bytes) {
    uint8_t* q = p ? p + o : nullptr;
    o += a256(bytes);
    return q;
  };
  Work W;
  W.dmA = reinterpret_cast<__nv_bfloat16*>(take(3 * 36 * T * Kpad * 2));
  W.dmB = reinterpret_cast<__nv_bfloat16*>(take(3 * 36 * K * (size_t)Tpad * 2));
  W.ut = reinterpret_cast<__nv_bfloat16*>(take(36 * C * (size_t)Kpad * 2));
  W.vt = reinterpret_cast<__nv_bfloat16*>(take(36 * C * (size_t)Tpad * 2));
  W.dv = reinterpret_cast<float*>(take(36 * T * C * 4));
  W.dup = reinterpret_cast<float*>(take((size_t)S * 36 * C * K * 4));
  W.dxt = reinterpret_cast<float*>(take(36 * T * C * 4));
  W.Kpad = Kpad, W.Tpad = Tpad, W.S = S, W.ks = ks;
  if (w) *w = W;
  return o;
}

}  // namespace bw
}  // namespace wl

using namespace wl;
using namespace wl::bw;

size_t wl_bw_workspace_bytes(const BwGeo& g) { return carve(g, nullptr, nullptr); }

int wl_bw_run(const BwGeo& g, const float* dy, const int8_t* ucodes, const wl::Acc* wacc, int wstage, int qmax_u,
              const int8_t* vcodes, const wl::Acc* acc, float* dx, float* dw, float* db, void* ws, cudaStream_t st,
              std::string* err) {
  Work W;
  carve(g, ws, &W);
  const int tb = 256;
  const long long T = g.T, C = g.C, K = g.K;
  dm_rows_kernel<<<(unsigned)((T * W.Kpad + tb - 1) / tb), tb, 0, st>>>(dy, W.dmA, g, W.Kpad);
  dm_cols_kernel<<<(unsigned)(((long long)W.Tpad * K + tb - 1) / tb), tb, 0, st>>>(dy, W.dmB, g, W.Tpad, acc);
  const unsigned cblk = (unsigned)((C + 63) / 64);
  codes_t_kernel<<<dim3(W.Kpad / 64, cblk, 36), 256, 0, st>>>(ucodes, W.ut, g.K, W.Kpad, g.C, g.Cp);
  codes_t_kernel<<<dim3(W.Tpad / 64, cblk, 36), 256, 0, st>>>(vcodes, W.vt, g.T, W.Tpad, g.C, g.Cp);
  // dV[e] (T x C) = dM[e] (T x K) . U[e]^T      (s_u applied in dxt_kernel)
  cudaError_t e1 = gemm_bf16_split(W.dmA, 3, W.ut, 1, 36, g.T, g.C, W.Kpad, W.Kpad, W.dv, g.C, 1.f, st);
  // dU^T[e] (C x K) = V[e]^T (C x T) . (s_v dM)[e] (T x K), split over the tiles
  cudaError_t e2 = gemm_bf16_split(W.vt, 1, W.dmB, 3, 36, g.C, g.K, W.Tpad, W.ks, W.dup, g.K, 1.f, st);
  if (e1 != cudaSuccess || e2 != cudaSuccess) {
    *err = std::string("tcgen05 backward GEMM launch: ") + cudaGetErrorString(e1 != cudaSuccess ? e1 : e2);
    return WL_ERR_CUDA;
  }
  dxt_kernel<<<(unsigned)((T * C + tb - 1) / tb), tb, 0, st>>>(W.dv, W.dxt, g, wacc, wstage, qmax_u);
  if (g.H * g.W >= 256) {  // 64 pixels per block (8 per thread: 32 loads in flight)
    const int pblocks = (g.H * g.W + 63) / 64;
    dx_gather_kernel<8><<<dim3((unsigned)(g.N * pblocks), 1, (unsigned)((C + 31) / 32)), 256, 0, st>>>(W.dxt, dx, g, pblocks);
  } else {
    const int pblocks = (g.H * g.W + 31) / 32;
    dx_gather_kernel<4><<<dim3((unsigned)(g.N * pblocks), 1, (unsigned)((C + 31) / 32)), 256, 0, st>>>(W.dxt, dx, g, pblocks);
  }
  dw_kernel<<<dim3((unsigned)((K + 31) / 32), (unsigned)((C + 7) / 8)), 256, 0, st>>>(W.dup, dw, g, W.S);
  if (db) db_kernel<<<(unsigned)K, 256, 0, st>>>(dy, db, g);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = cudaGetErrorString(e);
    return WL_ERR_CUDA;
  }
  return WL_OK;
}
