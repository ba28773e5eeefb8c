// Host interface of the quantized direct-convolution baseline (wl_direct.cu), used by the C ABI in
// wl_forward.cu.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <string>

namespace wl {

struct DGeo {
  int N, C, K, H, W, pad, Ho, Wo, ipg;
};

size_t wl_direct_workspace_bytes(const DGeo& g);
template <typename T>
int wl_direct_run(const DGeo& g, int in_bits, int w_bits, int out_bits, const T* x, const T* w, T* y, void* ws,
                  cudaStream_t st, std::string* err);

}  // namespace wl
