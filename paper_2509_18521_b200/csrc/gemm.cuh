// tcgen05 GEMM for the decoder projections (K4).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"

namespace ab {

enum GemmEpi : int {
  kEpiBF16 = 0,     // out bf16 = acc (+ bias)
  kEpiF32 = 1,      // out f32 = acc
  kEpiAddF32 = 2,   // out f32 += acc   (residual stream)
  kEpiSwiGLU = 3,   // weight rows interleaved in 64-row halves: out bf16[j] = silu(gate_j) * up_j
};

// D[M, N] = A[M, K] . W[N, K]^T, A = activations (rows dynamic), W = weights.
// Swap-AB on the tensor core: the 128-row UMMA M side walks W, the UMMA N
// side (BN) walks the activation rows, so small decode batches still issue
// full 128-wide MMAs.
struct GemmPlan {
  CUtensorMap tw;        // weights [N, K] bf16, box {64, 128}, 128B swizzle
  CUtensorMap ta;        // activations [M_cap, K] bf16, box {64, BN}, 128B swizzle
  int N = 0, K = 0, M_cap = 0, BN = 0, epi = 0;
  void* out = nullptr;
  int64_t ldo = 0;
  const __nv_bfloat16* bias = nullptr;
  const int* rows_dev = nullptr;  // live row count on device (nullptr: M_cap)
  const int* stop_dev = nullptr;  // engine stop flag (nullptr: never stop)
  int splits = 1;                 // split-K factor (kEpiAddF32 / kEpiF32-atomic only)
};

void gemm_plan(GemmPlan& p, const __nv_bfloat16* W, int N, int K, const __nv_bfloat16* A, int M_cap, int64_t lda,
               int BN, int epi, void* out, int64_t ldo, const __nv_bfloat16* bias, const int* rows_dev,
               const int* stop_dev);
void gemm_launch(const GemmPlan& p, cudaStream_t s);

}  // namespace ab
