// Host interface of the float (unquantized) Winograd path (wl_float.cu), used by the C ABI in
// wl_forward.cu.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "wl_core.cuh"

namespace wl {

struct FGeo {
  int N, C, K, H, W, pad, Ho, Wo, th, tw, TP, T;
};

size_t wl_float_workspace_bytes(const FGeo& g);
int wl_float_run(int legendre, const PlanF64* d_pf, const FGeo& g, const float* x, const float* w, const float* bias,
                 float* y, void* ws, cudaStream_t st, std::string* err);

}  // namespace wl
