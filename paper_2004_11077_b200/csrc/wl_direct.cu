// Quantized direct-convolution baseline: the reference's conv2d_direct_quantized(x, w, qconfig)
// (quantize.py:151-160), SURVEY §8f row 3 — the "direct" rows of the error experiment
// (harness.py:233-236).  The reference fake-quantises x and w (quantize.py:111-126), correlates the
// dequantised fp64 operands with _conv2d_direct_nb (_kernels.py:53-66: out[oc,i,j] += w*x, c, p, q
// ascending, separate multiply and add) and fake-quantises the result at output_transform_bits.
//
// Everything here runs in the reference's own fp64 arithmetic and order, so the result is the
// reference's bit for bit (no integer restatement, no replay): the per-group maxima are exact
// (max is order independent; |fp64| bit patterns order like the values), every element's sum
// uses the same operation sequence, and the casts are the reference's divide / rint / clip / snap.
// Kernels (thread per element, grid-stride): absmax (atomicMax on the |value| bit pattern per
// scale group), fake_quant to dequantised fp64, direct correlation + output group max, output
// fake_quant (+ conversion to the caller's dtype).  This is a comparison baseline, not the hot
// path: fp64 CUDA-core arithmetic, no tensor cores.
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "wl_direct.h"

namespace wl {
namespace dq {

__device__ __forceinline__ unsigned long long abs_bits(double v) {
  return (unsigned long long)__double_as_longlong(fabs(v));
}

// per-group max |x| as fp64 bits (x: groups of `per` consecutive elements)
template <typename T>
__global__ void absmax_kernel(const T* __restrict__ x, long long total, long long per,
                              unsigned long long* __restrict__ gmax) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= total) return;
  long long g = i / per, gend = (g + 1) * per;
  unsigned long long m = 0;
  for (; i < total; i += stride) {
    if (i >= gend) {  // crossed into a later group: flush
      atomicMax(&gmax[g], m);
      m = 0;
      g = i / per;
      gend = (g + 1) * per;
    }
    m = max(m, abs_bits((double)x[i]));
  }
  atomicMax(&gmax[g], m);
}

// fake_quant (quantize.py:111-126): scale = M/qmax, codes = clip(rint(v/scale)), out = codes*scale,
// codes == +-qmax snapped to +-M; M == 0 leaves the (all-zero) tensor unchanged (and, with no
// absmax pass, makes the cast the identity: the unquantized conv2d_direct).
__device__ __forceinline__ double fake_quant1(double v, double M, double qmax) {
  if (M == 0.0 || qmax == 0.0) return v;  // qmax 0: identity cast (width 0)
  const double scale = __ddiv_rn(M, qmax);
  double c = rint(__ddiv_rn(v, scale));
  c = fmin(fmax(c, -qmax), qmax);
  if (c == qmax) return M;
  if (c == -qmax) return -M;
  return __dmul_rn(c, scale);
}

template <typename T>
__global__ void quant_kernel(const T* __restrict__ x, double* __restrict__ xq, long long total, long long per,
                             const unsigned long long* __restrict__ gmax, double qmax) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += stride)
    xq[i] = fake_quant1((double)x[i], __longlong_as_double((long long)gmax[i / per]), qmax);
}

// z[n][k][i][j] = sum_{c,p,q ascending} wq[k][c][p][q] * xp[n][c][i+p][j+q]   (xp: x zero-padded)
__global__ void direct_kernel(const double* __restrict__ xq, const double* __restrict__ wq, double* __restrict__ z,
                              DGeo g, unsigned long long* __restrict__ zmax) {
  const long long total = (long long)g.N * g.K * g.Ho * g.Wo;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total; idx += stride) {
    const int j = (int)(idx % g.Wo);
    long long r = idx / g.Wo;
    const int i = (int)(r % g.Ho);
    r /= g.Ho;
    const int k = (int)(r % g.K);
    const int n = (int)(r / g.K);
    const double* xn = xq + (size_t)n * g.C * g.H * g.W;
    const double* wk = wq + (size_t)k * g.C * 9;
    double acc = 0.0;
    for (int c = 0; c < g.C; ++c) {
      const double* xc = xn + (size_t)c * g.H * g.W;
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        const int y = i + p - g.pad;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const int x = j + q - g.pad;
          const double xv = (y >= 0 && y < g.H && x >= 0 && x < g.W) ? __ldg(&xc[(size_t)y * g.W + x]) : 0.0;
          acc = __dadd_rn(acc, __dmul_rn(__ldg(&wk[c * 9 + p * 3 + q]), xv));
        }
      }
    }
    z[idx] = acc;
    atomicMax(&zmax[n / g.ipg], abs_bits(acc));
  }
}

template <typename T>
__global__ void out_kernel(const double* __restrict__ z, T* __restrict__ y, long long total, long long per,
                           const unsigned long long* __restrict__ gmax, double qmax) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += stride)
    y[i] = (T)fake_quant1(z[i], __longlong_as_double((long long)gmax[i / per]), qmax);
}

}  // namespace dq

static size_t al256(size_t v) { return (v + 255) & ~size_t(255); }

size_t wl_direct_workspace_bytes(const DGeo& g) {
  const int groups = g.N / g.ipg;
  return al256((size_t)(2 * groups + 1) * 8) + al256((size_t)g.N * g.C * g.H * g.W * 8) +
         al256((size_t)g.K * g.C * 9 * 8) + al256((size_t)g.N * g.K * g.Ho * g.Wo * 8);
}

static unsigned grid_for(long long n, int tb) {
  long long b = (n + tb - 1) / tb;
  const long long cap = 148LL * 16;  // grid-stride beyond 16 blocks per SM
  return (unsigned)(b < 1 ? 1 : (b > cap ? cap : b));
}

template <typename T>
int wl_direct_run(const DGeo& g, int in_bits, int w_bits, int out_bits, const T* x, const T* w, T* y, void* ws,
                  cudaStream_t st, std::string* err) {
  const int groups = g.N / g.ipg;
  uint8_t* p = reinterpret_cast<uint8_t*>(ws);
  unsigned long long* gx = reinterpret_cast<unsigned long long*>(p);  // [groups] x max, [1] w max, [groups] z max
  unsigned long long* gw = gx + groups;
  unsigned long long* gz = gw + 1;
  p += al256((size_t)(2 * groups + 1) * 8);
  double* xq = reinterpret_cast<double*>(p);
  p += al256((size_t)g.N * g.C * g.H * g.W * 8);
  double* wq = reinterpret_cast<double*>(p);
  p += al256((size_t)g.K * g.C * 9 * 8);
  double* z = reinterpret_cast<double*>(p);
  const long long nx = (long long)g.N * g.C * g.H * g.W, per_x = (long long)g.ipg * g.C * g.H * g.W;
  const long long nw = (long long)g.K * g.C * 9;
  const long long ny = (long long)g.N * g.K * g.Ho * g.Wo, per_y = (long long)g.ipg * g.K * g.Ho * g.Wo;
  const int tb = 256;
  cudaMemsetAsync(gx, 0, (size_t)(2 * groups + 1) * 8, st);
  // width 0 = identity cast: the group maximum stays 0 and fake_quant1 passes the value through
  auto qmax = [](int bits) { return bits > 0 ? (double)((1LL << (bits - 1)) - 1) : 0.0; };
  if (in_bits > 0) dq::absmax_kernel<T><<<grid_for(nx, tb), tb, 0, st>>>(x, nx, per_x, gx);
  if (w_bits > 0) dq::absmax_kernel<T><<<grid_for(nw, tb), tb, 0, st>>>(w, nw, nw, gw);
  dq::quant_kernel<T><<<grid_for(nx, tb), tb, 0, st>>>(x, xq, nx, per_x, gx, qmax(in_bits));
  dq::quant_kernel<T><<<grid_for(nw, tb), tb, 0, st>>>(w, wq, nw, nw, gw, qmax(w_bits));
  dq::direct_kernel<<<grid_for(ny, tb), tb, 0, st>>>(xq, wq, z, g, gz);
  dq::out_kernel<T><<<grid_for(ny, tb), tb, 0, st>>>(z, y, ny, per_y, gz, qmax(out_bits));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = cudaGetErrorString(e);
    return -1;
  }
  return 0;
}

template int wl_direct_run<float>(const DGeo&, int, int, int, const float*, const float*, float*, void*, cudaStream_t,
                                  std::string*);
template int wl_direct_run<double>(const DGeo&, int, int, int, const double*, const double*, double*, void*,
                                   cudaStream_t, std::string*);

}  // namespace wl
