// Float (unquantized) Winograd F(4x4,3x3) correlation in fp32: the reference's
// conv2d_winograd(x, w, plan, mode) = run_pipeline with the identity cast (pipeline.py:161-164,
// stage structure pipeline.py:125-158), SURVEY §8f row 2.  Every stage is the reference's sandwich
// L . X . L^T with the plan's nearest-double matrices (construct.py:191-208) rounded to fp32:
//   canonical: U = G w G^T,                      V = B^T d B,                   Y = A^T M A
//   legendre:  U = P^-1 (G_P w G_P^T) P^-T,       V = B_P^T (P^-T d P^-1) B_P,   Y = A_P^T (P^-T M P^-1) A_P
//   M[xi] = sum_c U[xi] (.) V[xi]  (36 batched GEMMs on tcgen05, gemm_bf16.cuh: U and V carried as
//   three bf16 planes each, the six plane products with i + j <= 2 give fp32-accurate products,
//   fp32 accumulation in TMEM).
// Same batch / padding / crop conventions as the quantized layer (wl_forward).  Kernels: one
// weight transform (thread per (out, in) channel pair), one input transform (thread per (tile,
// channel), channel fastest: V stores coalesce), one output transform (thread per (tile, out
// channel)), all in fp32 with the reference's sandwich order (tmp = X . R first, then L . tmp).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <string>

#include "gemm_bf16.cuh"
#include "wl_float.h"
#include "wl_gemm_bf16.h"

namespace wl {
namespace fl32 {

struct Mats {  // fp32 copies of the plan's left matrices (row-major, L::R x L::C)
  float wt[18], wbc[36], ibc[36], it[36], obc[36], ot[24];
};

// out (R x R) = L . X . L^T, L is R x C (row-major), X is C x C; numba order: tmp = X . L^T, then L . tmp
template <int R, int C>
__device__ __forceinline__ void sandwich_f(const float* __restrict__ L, const float (&X)[C][C], float (&out)[R][R]) {
  float tmp[C][R];
#pragma unroll
  for (int i = 0; i < C; ++i)
#pragma unroll
    for (int j = 0; j < R; ++j) {
      float s = 0.f;
#pragma unroll
      for (int l = 0; l < C; ++l) s = fmaf(X[i][l], L[j * C + l], s);
      tmp[i][j] = s;
    }
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < R; ++j) {
      float s = 0.f;
#pragma unroll
      for (int l = 0; l < C; ++l) s = fmaf(L[i * C + l], tmp[l][j], s);
      out[i][j] = s;
    }
}

__global__ void mats_kernel(const wl::PlanF64* __restrict__ pf, Mats* __restrict__ m) {
  const int i = threadIdx.x;
  if (i < 18) m->wt[i] = (float)pf->wt[i];
  if (i < 36) {
    m->wbc[i] = (float)pf->wbc[i];
    m->ibc[i] = (float)pf->ibc[i];
    m->it[i] = (float)pf->it[i];
    m->obc[i] = (float)pf->obc[i];
  }
  if (i < 24) m->ot[i] = (float)pf->ot[i];
}

// three bf16 planes of v at P[o], P[o + plane], P[o + 2 plane]
__device__ __forceinline__ void put3(__nv_bfloat16* __restrict__ P, size_t plane, size_t o, float v) {
  __nv_bfloat16 h, m, l;
  wl_split3(v, h, m, l);
  P[o] = h;
  P[plane + o] = m;
  P[2 * plane + o] = l;
}

// U planes [3][36][K][Cpad] (zero padded channels)
__global__ void weight_kernel(const float* __restrict__ w, __nv_bfloat16* __restrict__ U, const Mats* __restrict__ mp,
                              FGeo g, int legendre, int Cpad) {
  __shared__ Mats m;
  if (threadIdx.x < sizeof(Mats) / 4) reinterpret_cast<float*>(&m)[threadIdx.x] = reinterpret_cast<const float*>(mp)[threadIdx.x];
  __syncthreads();
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)g.K * Cpad) return;
  const int c = (int)(idx % Cpad), k = (int)(idx / Cpad);
  const size_t plane = (size_t)36 * g.K * Cpad;
  if (c >= g.C) {
#pragma unroll
    for (int e = 0; e < 36; ++e) put3(U, plane, ((size_t)e * g.K + k) * Cpad + c, 0.f);
    return;
  }
  float X[3][3];
#pragma unroll
  for (int e = 0; e < 9; ++e) X[e / 3][e % 3] = __ldg(&w[((size_t)k * g.C + c) * 9 + e]);
  float u[6][6];
  sandwich_f<6, 3>(m.wt, X, u);
  if (legendre) {
    float v[6][6];
    sandwich_f<6, 6>(m.wbc, u, v);
#pragma unroll
    for (int e = 0; e < 36; ++e) u[e / 6][e % 6] = v[e / 6][e % 6];
  }
#pragma unroll
  for (int e = 0; e < 36; ++e) put3(U, plane, ((size_t)e * g.K + k) * Cpad + c, u[e / 6][e % 6]);
}

// V planes [3][36][T][Cpad] from the zero-padded NCHW input
__global__ void input_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ V, const Mats* __restrict__ mp,
                             FGeo g, int legendre, int Cpad) {
  __shared__ Mats m;
  if (threadIdx.x < sizeof(Mats) / 4) reinterpret_cast<float*>(&m)[threadIdx.x] = reinterpret_cast<const float*>(mp)[threadIdx.x];
  __syncthreads();
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)g.T * Cpad) return;
  const int c = (int)(idx % Cpad), t = (int)(idx / Cpad);
  const size_t plane = (size_t)36 * g.T * Cpad;
  if (c >= g.C) {
#pragma unroll
    for (int e = 0; e < 36; ++e) put3(V, plane, ((size_t)e * g.T + t) * Cpad + c, 0.f);
    return;
  }
  const int n = t / g.TP, tile = t % g.TP, ty = tile / g.tw, tx = tile % g.tw;
  float X[6][6];
#pragma unroll
  for (int i = 0; i < 6; ++i)
#pragma unroll
    for (int j = 0; j < 6; ++j) {
      const int r = 4 * ty + i - g.pad, q = 4 * tx + j - g.pad;
      X[i][j] = (r >= 0 && r < g.H && q >= 0 && q < g.W) ? __ldg(&x[(((size_t)n * g.C + c) * g.H + r) * g.W + q]) : 0.f;
    }
  float v[6][6];
  if (legendre) {
    float a[6][6];
    sandwich_f<6, 6>(m.ibc, X, a);
    sandwich_f<6, 6>(m.it, a, v);
  } else {
    sandwich_f<6, 6>(m.it, X, v);
  }
#pragma unroll
  for (int e = 0; e < 36; ++e) put3(V, plane, ((size_t)e * g.T + t) * Cpad + c, v[e / 6][e % 6]);
}

// y (cropped NCHW) from M[xi][t][k] (row-major [T][K] per xi)
__global__ void output_kernel(const float* __restrict__ M, const float* __restrict__ bias, float* __restrict__ y,
                              const Mats* __restrict__ mp, FGeo g, int legendre) {
  __shared__ Mats m;
  if (threadIdx.x < sizeof(Mats) / 4) reinterpret_cast<float*>(&m)[threadIdx.x] = reinterpret_cast<const float*>(mp)[threadIdx.x];
  __syncthreads();
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)g.T * g.K) return;
  const int k = (int)(idx % g.K), t = (int)(idx / g.K);
  const int n = t / g.TP, tile = t % g.TP, ty = tile / g.tw, tx = tile % g.tw;
  float X[6][6];
#pragma unroll
  for (int e = 0; e < 36; ++e) X[e / 6][e % 6] = __ldg(&M[((size_t)e * g.T + t) * g.K + k]);
  float Y[4][4];
  if (legendre) {
    float a[6][6];
    sandwich_f<6, 6>(m.obc, X, a);
    sandwich_f<4, 6>(m.ot, a, Y);
  } else {
    sandwich_f<4, 6>(m.ot, X, Y);
  }
  const float bk = bias ? __ldg(&bias[k]) : 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = 4 * ty + i, q = 4 * tx + j;
      if (r < g.Ho && q < g.Wo) y[(((size_t)n * g.K + k) * g.Ho + r) * g.Wo + q] = Y[i][j] + bk;
    }
}

}  // namespace fl32

static size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

size_t wl_float_workspace_bytes(const FGeo& g) {
  const size_t Cpad = round_up(g.C, 64);
  return align256(sizeof(fl32::Mats)) + align256(3 * 36 * (size_t)g.K * Cpad * 2) +
         align256(3 * 36 * (size_t)g.T * Cpad * 2) + align256((size_t)36 * g.T * g.K * 4);
}

int wl_float_run(int legendre, const PlanF64* d_pf, const FGeo& g, const float* x, const float* w, const float* bias,
                 float* y, void* ws, cudaStream_t st, std::string* err) {
  const int Cpad = round_up(g.C, 64);
  uint8_t* p = reinterpret_cast<uint8_t*>(ws);
  fl32::Mats* mats = reinterpret_cast<fl32::Mats*>(p);
  p += align256(sizeof(fl32::Mats));
  __nv_bfloat16* U = reinterpret_cast<__nv_bfloat16*>(p);
  p += align256(3 * 36 * (size_t)g.K * Cpad * 2);
  __nv_bfloat16* V = reinterpret_cast<__nv_bfloat16*>(p);
  p += align256(3 * 36 * (size_t)g.T * Cpad * 2);
  float* M = reinterpret_cast<float*>(p);
  fl32::mats_kernel<<<1, 64, 0, st>>>(d_pf, mats);
  const int tb = 256;
  fl32::weight_kernel<<<(unsigned)(((long long)g.K * Cpad + tb - 1) / tb), tb, 0, st>>>(w, U, mats, g, legendre, Cpad);
  fl32::input_kernel<<<(unsigned)(((long long)g.T * Cpad + tb - 1) / tb), tb, 0, st>>>(x, V, mats, g, legendre, Cpad);
  // M[xi] (T x K) = V[xi] (T x C) . U[xi]^T (C x K): fp32-accurate products from 3 x 3 bf16 planes
  cudaError_t ge = gemm_bf16_split(V, 3, U, 3, 36, g.T, g.K, Cpad, Cpad, M, g.K, 1.f, st);
  if (ge != cudaSuccess) {
    *err = std::string("tcgen05 float GEMM launch: ") + cudaGetErrorString(ge);
    return -1;
  }
  fl32::output_kernel<<<(unsigned)(((long long)g.T * g.K + tb - 1) / tb), tb, 0, st>>>(M, bias, y, mats, g, legendre);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = cudaGetErrorString(e);
    return -1;
  }
  return 0;
}

}  // namespace wl
