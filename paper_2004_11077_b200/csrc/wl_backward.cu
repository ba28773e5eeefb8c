// Straight-through-estimator backward of the quantized Winograd layer.
// The reference has no backward; this defines it: every fake-quant cast is the identity in
// backward with detached scales, the products use the forward's QUANTISED operands (U, V codes
// times their stage scale), and — since every Legendre composite equals the canonical transform in
// exact arithmetic (pipeline.py:9-11: P^-1 A_P = A, P^-1 B_P = B, P^-1 G_P = G) — both bases use
//   dM  = A . dY . A^T                       (6x6 per (tile, out channel))
//   dV  = sum_k U_k (.) dM_k,  dU = sum_t V_t (.) dM_t   (36 batched fp32 GEMMs, cuBLAS)
//   dX  = col2im( B . dV . B^T )             (gather over the <= 2x2 tiles covering a pixel)
//   dW  = G^T . dU . G,   db = sum dY
// Transform / gather kernels are hand written; the batched GEMMs are plain library GEMMs.
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/winoleg_b200.h"
#include "wl_backward.h"

namespace wl {
namespace bw {

// canonical F(4,3) matrices (the reference's A, B^T, G; construct.py:161-181)
__constant__ float kAT[4][6] = {{1, 1, 1, 1, 1, 0}, {0, 1, -1, 2, -2, 0}, {0, 1, 1, 4, 4, 0}, {0, 1, -1, 8, -8, 1}};
__constant__ float kBT[6][6] = {{4, 0, -5, 0, 1, 0},  {0, -4, -4, 1, 1, 0}, {0, 4, -4, -1, 1, 0},
                                {0, -2, -1, 2, 1, 0}, {0, 2, -1, -2, 1, 0}, {0, 4, 0, -5, 0, 1}};
__constant__ float kG[6][3] = {{0.25f, 0, 0},
                               {-1.f / 6, -1.f / 6, -1.f / 6},
                               {-1.f / 6, 1.f / 6, -1.f / 6},
                               {1.f / 24, 1.f / 12, 1.f / 6},
                               {1.f / 24, -1.f / 12, 1.f / 6},
                               {0, 0, 1}};

// dM[e][t][k] = (A . dY_tile . A^T)[e], dY cropped to the valid output (pad-to-tile spill is zero).
__global__ void dm_kernel(const float* __restrict__ dy, float* __restrict__ dm, BwGeo g) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)g.T * g.K) return;
  const int k = (int)(idx % g.K), t = (int)(idx / g.K);
  const int n = t / g.TP, tile = t % g.TP, ty = tile / g.tw, tx = tile % g.tw;
  float Y[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int r = 4 * ty + a, c = 4 * tx + b;
      Y[a][b] = (r < g.Ho && c < g.Wo) ? __ldg(&dy[(((size_t)n * g.K + k) * g.Ho + r) * g.Wo + c]) : 0.f;
    }
  float tmp[4][6];  // dY . A^T
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int j = 0; j < 6; ++j) {
      float s = 0.f;
#pragma unroll
      for (int b = 0; b < 4; ++b) s = fmaf(Y[a][b], kAT[b][j], s);
      tmp[a][j] = s;
    }
#pragma unroll
  for (int i = 0; i < 6; ++i)
#pragma unroll
    for (int j = 0; j < 6; ++j) {
      float s = 0.f;
#pragma unroll
      for (int a = 0; a < 4; ++a) s = fmaf(kAT[a][i], tmp[a][j], s);
      dm[((size_t)(6 * i + j) * g.T + t) * g.K + k] = s;
    }
}

// Dequantised GEMM operands: U [36][K][C] and V [36][T][C] fp32 from the int8 codes.
__global__ void deq_u_kernel(const int8_t* __restrict__ ucodes, float* __restrict__ ud, BwGeo g,
                             const Acc* __restrict__ wacc, int wstage, int qmax_u) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= 36LL * g.K * g.C) return;
  const double su = load_int_stage(wacc[wstage], qmax_u).scale;
  const int c = (int)(idx % g.C);
  const long long r = idx / g.C;
  const int k = (int)(r % g.K), e = (int)(r / g.K);
  ud[idx] = (float)((double)ucodes[((size_t)k * 36 + e) * g.Cp + c] * su);
}
__global__ void deq_v_kernel(const int8_t* __restrict__ vcodes, float* __restrict__ vd, BwGeo g,
                             const Acc* __restrict__ acc) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= 36LL * g.T * g.C) return;
  const int c = (int)(idx % g.C);
  const long long r = idx / g.C;
  const int t = (int)(r % g.T), e = (int)(r / g.T);
  const int grp = (t / g.TP) / g.ipg;
  vd[idx] = (float)((double)vcodes[((size_t)t * 36 + e) * g.Cp + c] * acc[(size_t)grp * ST_COUNT + ST_IT].scale);
}

// dXt[t][c][36] = B . dV_tile . B^T (dV gathered from [36][T][C]).
__global__ void dxt_kernel(const float* __restrict__ dv, float* __restrict__ dxt, BwGeo g) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)g.T * g.C) return;
  const int c = (int)(idx % g.C), t = (int)(idx / g.C);
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
      for (int b = 0; b < 6; ++b) s = fmaf(D[a][b], kBT[b][j], s);
      tmp[a][j] = s;
    }
  float* out = dxt + idx * 36;
#pragma unroll
  for (int i = 0; i < 6; ++i)
#pragma unroll
    for (int j = 0; j < 6; ++j) {
      float s = 0.f;
#pragma unroll
      for (int a = 0; a < 6; ++a) s = fmaf(kBT[a][i], tmp[a][j], s);
      out[6 * i + j] = s;
    }
}

// Gather col2im: each input pixel sums the <= 2x2 tile contributions covering it (no atomics).
__global__ void dx_gather_kernel(const float* __restrict__ dxt, float* __restrict__ dx, BwGeo g) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)g.N * g.C * g.H * g.W) return;
  const int col = (int)(idx % g.W);
  long long r_ = idx / g.W;
  const int row = (int)(r_ % g.H);
  r_ /= g.H;
  const int c = (int)(r_ % g.C), n = (int)(r_ / g.C);
  const int rp = row + g.pad, cp = col + g.pad;
  float s = 0.f;
  for (int ty = max(0, (rp - 2) / 4); ty <= min(g.th - 1, rp / 4); ++ty) {
    const int i = rp - 4 * ty;
    if (i < 0 || i > 5) continue;
    for (int tx = max(0, (cp - 2) / 4); tx <= min(g.tw - 1, cp / 4); ++tx) {
      const int j = cp - 4 * tx;
      if (j < 0 || j > 5) continue;
      const int t = n * g.TP + ty * g.tw + tx;
      s += __ldg(&dxt[((size_t)t * g.C + c) * 36 + 6 * i + j]);
    }
  }
  dx[idx] = s;
}

// dW[k][c] = G^T . dU . G with dU[e][c][k] from the batched GEMM.
__global__ void dw_kernel(const float* __restrict__ du, float* __restrict__ dw, BwGeo g) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= g.K * g.C) return;
  const int c = idx % g.C, k = idx / g.C;
  float D[6][6];
#pragma unroll
  for (int e = 0; e < 36; ++e) D[e / 6][e % 6] = du[((size_t)e * g.C + c) * g.K + k];
  float tmp[6][3];  // dU . G
#pragma unroll
  for (int a = 0; a < 6; ++a)
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      float s = 0.f;
#pragma unroll
      for (int b = 0; b < 6; ++b) s = fmaf(D[a][b], kG[b][q], s);
      tmp[a][q] = s;
    }
#pragma unroll
  for (int p = 0; p < 3; ++p)
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      float s = 0.f;
#pragma unroll
      for (int a = 0; a < 6; ++a) s = fmaf(kG[a][p], tmp[a][q], s);
      dw[(size_t)idx * 9 + 3 * p + q] = s;
    }
}

__global__ void db_kernel(const float* __restrict__ dy, float* __restrict__ db, BwGeo g) {
  const int k = blockIdx.x;
  float s = 0.f;
  const long long per = (long long)g.Ho * g.Wo;
  for (long long i = threadIdx.x; i < (long long)g.N * per; i += blockDim.x) {
    const long long n = i / per, p = i % per;
    s += dy[((size_t)n * g.K + k) * per + p];
  }
  __shared__ float red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) db[k] = s;
  }
}

}  // namespace bw
}  // namespace wl

using namespace wl::bw;

namespace {
std::mutex g_cublas_mu;
cublasHandle_t cublas_for_device() {
  static cublasHandle_t handles[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_cublas_mu);
  if (!handles[dev]) cublasCreate(&handles[dev]);
  return handles[dev];
}
size_t a256(size_t v) { return (v + 255) & ~size_t(255); }
}  // namespace

size_t wl_bw_workspace_bytes(const BwGeo& g) {
  const size_t T = g.T, C = g.C, K = g.K;
  return a256(36 * T * K * 4) + a256(36 * K * C * 4) + a256(36 * T * C * 4) + a256(36 * T * C * 4) +
         a256(36 * C * K * 4);
}

int wl_bw_run(const BwGeo& g, const float* dy, const int8_t* ucodes, const wl::Acc* wacc, int wstage, int qmax_u,
              const int8_t* vcodes, const wl::Acc* acc, float* dx, float* dw, float* db, void* ws, cudaStream_t st,
              std::string* err) {
  const size_t T = g.T, C = g.C, K = g.K;
  uint8_t* p = reinterpret_cast<uint8_t*>(ws);
  float* dm = reinterpret_cast<float*>(p);
  p += a256(36 * T * K * 4);
  float* ud = reinterpret_cast<float*>(p);
  p += a256(36 * K * C * 4);
  float* vd = reinterpret_cast<float*>(p);
  p += a256(36 * T * C * 4);
  float* dv = reinterpret_cast<float*>(p);
  p += a256(36 * T * C * 4);
  float* du = reinterpret_cast<float*>(p);
  const int tb = 256;
  dm_kernel<<<(unsigned)((T * K + tb - 1) / tb), tb, 0, st>>>(dy, dm, g);
  deq_u_kernel<<<(unsigned)((36 * K * C + tb - 1) / tb), tb, 0, st>>>(ucodes, ud, g, wacc, wstage, qmax_u);
  deq_v_kernel<<<(unsigned)((36 * T * C + tb - 1) / tb), tb, 0, st>>>(vcodes, vd, g, acc);
  cublasHandle_t h = cublas_for_device();
  cublasSetStream(h, st);
  const float one = 1.f, zero = 0.f;
  // dV_e [T x C] = dM_e [T x K] . U_e [K x C]   (row-major; column-major view: dV^T = U^T . dM^T)
  cublasStatus_t s1 = cublasSgemmStridedBatched(h, CUBLAS_OP_N, CUBLAS_OP_N, (int)C, (int)T, (int)K, &one, ud,
                                                (int)C, (long long)K * C, dm, (int)K, (long long)T * K, &zero, dv,
                                                (int)C, (long long)T * C, 36);
  // dU_e [C x K] = V_e^T [C x T] . dM_e [T x K]  (column-major result dU^T [K x C] = dM^T . V)
  cublasStatus_t s2 = cublasSgemmStridedBatched(h, CUBLAS_OP_N, CUBLAS_OP_T, (int)K, (int)C, (int)T, &one, dm,
                                                (int)K, (long long)T * K, vd, (int)C, (long long)T * C, &zero, du,
                                                (int)K, (long long)C * K, 36);
  if (s1 != CUBLAS_STATUS_SUCCESS || s2 != CUBLAS_STATUS_SUCCESS) {
    *err = "cublasSgemmStridedBatched failed";
    return WL_ERR_CUDA;
  }
  // dX: tile transforms into vd (no longer needed), then the gather
  float* dxt = vd;
  dxt_kernel<<<(unsigned)((T * C + tb - 1) / tb), tb, 0, st>>>(dv, dxt, g);
  dx_gather_kernel<<<(unsigned)(((size_t)g.N * C * g.H * g.W + tb - 1) / tb), tb, 0, st>>>(dxt, dx, g);
  dw_kernel<<<(unsigned)((K * C + tb - 1) / tb), tb, 0, st>>>(du, dw, g);
  if (db) db_kernel<<<(unsigned)K, 256, 0, st>>>(dy, db, g);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = cudaGetErrorString(e);
    return WL_ERR_CUDA;
  }
  return WL_OK;
}
