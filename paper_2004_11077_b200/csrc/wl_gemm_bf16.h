// Host launcher of the split-bf16 tcgen05 GEMM (gemm_bf16.cuh), shared by the STE backward and the
// float Winograd path.
#pragma once
#include <cuda_runtime.h>

namespace wl {

// D[s][b][m][n] (row stride ldd) = alpha * sum_{k in split s} A[b][m][k] B[b][n][k].
// A: bf16 [PA][batch][M][Kd], B: bf16 [PB][batch][N][Kd] (Kd a multiple of 64, zero padded);
// splits = ceil(Kd / ks), ks a multiple of 64.  Returns a cudaError_t.
cudaError_t gemm_bf16_split(const void* A, int PA, const void* B, int PB, int batch, int M, int N, int Kd, int ks,
                            float* D, int ldd, float alpha, cudaStream_t st);

inline int round_up(int v, int m) { return (v + m - 1) / m * m; }

}  // namespace wl
