// Float (unquantized) Winograd F(4x4,3x3) correlation in fp32: the reference's
// conv2d_winograd(x, w, plan, mode) = run_pipeline with the identity cast (pipeline.py:161-164,
// stage structure pipeline.py:125-158), SURVEY §8f row 2.  Every stage is the reference's sandwich
// L . X . L^T with the plan's nearest-double matrices (construct.py:191-208) rounded to fp32:
//   canonical: U = G w G^T,                      V = B^T d B,                   Y = A^T M A
//   legendre:  U = P^-1 (G_P w G_P^T) P^-T,       V = B_P^T (P^-T d P^-1) B_P,   Y = A_P^T (P^-T M P^-1) A_P
//   M[xi] = sum_c U[xi] (.) V[xi]  (36 batched fp32 GEMMs, cuBLAS: plain library GEMMs).
// Same batch / padding / crop conventions as the quantized layer (wl_forward).  Kernels: one
// weight transform (thread per (out, in) channel pair), one input transform (thread per (tile,
// channel), channel fastest: V stores coalesce), one output transform (thread per (tile, out
// channel)), all in fp32 with the reference's sandwich order (tmp = X . R first, then L . tmp).
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <mutex>
#include <string>

#include "wl_float.h"

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

// U[xi][k][c] (row-major [K][C] per xi)
__global__ void weight_kernel(const float* __restrict__ w, float* __restrict__ U, const Mats* __restrict__ mp, FGeo g,
                              int legendre) {
  __shared__ Mats m;
  if (threadIdx.x < sizeof(Mats) / 4) reinterpret_cast<float*>(&m)[threadIdx.x] = reinterpret_cast<const float*>(mp)[threadIdx.x];
  __syncthreads();
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)g.K * g.C) return;
  const int c = (int)(idx % g.C), k = (int)(idx / g.C);
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
  for (int e = 0; e < 36; ++e) U[((size_t)e * g.K + k) * g.C + c] = u[e / 6][e % 6];
}

// V[xi][t][c] (row-major [T][C] per xi) from the zero-padded NCHW input
__global__ void input_kernel(const float* __restrict__ x, float* __restrict__ V, const Mats* __restrict__ mp, FGeo g,
                             int legendre) {
  __shared__ Mats m;
  if (threadIdx.x < sizeof(Mats) / 4) reinterpret_cast<float*>(&m)[threadIdx.x] = reinterpret_cast<const float*>(mp)[threadIdx.x];
  __syncthreads();
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)g.T * g.C) return;
  const int c = (int)(idx % g.C), t = (int)(idx / g.C);
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
  for (int e = 0; e < 36; ++e) V[((size_t)e * g.T + t) * g.C + c] = v[e / 6][e % 6];
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
  return align256(sizeof(fl32::Mats)) + align256((size_t)36 * g.K * g.C * 4) + align256((size_t)36 * g.T * g.C * 4) +
         align256((size_t)36 * g.T * g.K * 4);
}

// one handle per device, fp32 "pedantic" math (the backward's handle keeps the default mode)
static cublasHandle_t float_cublas_for_device() {
  static cublasHandle_t handles[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return nullptr;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (!handles[dev] && cublasCreate(&handles[dev]) != CUBLAS_STATUS_SUCCESS) handles[dev] = nullptr;
  return handles[dev];
}

int wl_float_run(int legendre, const PlanF64* d_pf, const FGeo& g, const float* x, const float* w, const float* bias,
                 float* y, void* ws, cudaStream_t st, std::string* err) {
  uint8_t* p = reinterpret_cast<uint8_t*>(ws);
  fl32::Mats* mats = reinterpret_cast<fl32::Mats*>(p);
  p += align256(sizeof(fl32::Mats));
  float* U = reinterpret_cast<float*>(p);
  p += align256((size_t)36 * g.K * g.C * 4);
  float* V = reinterpret_cast<float*>(p);
  p += align256((size_t)36 * g.T * g.C * 4);
  float* M = reinterpret_cast<float*>(p);
  fl32::mats_kernel<<<1, 64, 0, st>>>(d_pf, mats);
  const int tb = 256;
  fl32::weight_kernel<<<(unsigned)(((long long)g.K * g.C + tb - 1) / tb), tb, 0, st>>>(w, U, mats, g, legendre);
  fl32::input_kernel<<<(unsigned)(((long long)g.T * g.C + tb - 1) / tb), tb, 0, st>>>(x, V, mats, g, legendre);
  cublasHandle_t h = float_cublas_for_device();
  if (!h) {
    *err = "cublasCreate failed";
    return -1;
  }
  cublasSetStream(h, st);
  cublasSetMathMode(h, CUBLAS_PEDANTIC_MATH);  // true fp32 FMA products (no tf32 / bf16x3 emulation)
  const float one = 1.f, zero = 0.f;
  // column-major view: M_xi (K x T) = U_xi^T (K x C) . V_xi (C x T)
  cublasStatus_t s = cublasSgemmStridedBatched(h, CUBLAS_OP_T, CUBLAS_OP_N, g.K, g.T, g.C, &one, U, g.C,
                                               (long long)g.K * g.C, V, g.C, (long long)g.T * g.C, &zero, M, g.K,
                                               (long long)g.T * g.K, 36);
  if (s != CUBLAS_STATUS_SUCCESS) {
    *err = "cublasSgemmStridedBatched failed";
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
