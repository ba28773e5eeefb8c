// Host interface of the STE backward (wl_backward.cu), used by the C ABI in wl_abi.cu.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "wl_core.cuh"

struct BwGeo {
  int N, C, K, H, W, pad, Ho, Wo, th, tw, TP, T, Cp, Kp, ipg, groups;
};

size_t wl_bw_workspace_bytes(const BwGeo& g);
// ucodes [Kp][36][Cp] with their stage slot wacc[wstage]; vcodes [T][36][Cp] with per-group scale
// acc[g*ST_COUNT + ST_IT].scale (set by the forward).
int wl_bw_run(const BwGeo& g, const float* dy, const int8_t* ucodes, const wl::Acc* wacc, int wstage, int qmax_u,
              const int8_t* vcodes, const wl::Acc* acc, float* dx, float* dw, float* db, void* ws, cudaStream_t st,
              std::string* err);
