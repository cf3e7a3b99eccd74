#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace vpe {
// Fused MLP block (mlp.cu): resid[M, D] += ls2 * (GELU(X W1^T + b1) W2^T + b2), X = LN2 output.
struct MlpPlan {
  CUtensorMap tx, tw1, tw2;
  const float *b1 = nullptr, *b2 = nullptr, *ls2 = nullptr;
  float* resid = nullptr;
  int M = 0, hidden = 0, grid = 0;
};
// D must be 384 (ViT-S/14) and hidden a multiple of 64; VPE_E_SHAPE otherwise (caller falls
// back to the FC1 / FC2 GEMM pair).
int plan_mlp(MlpPlan* m, const __nv_bfloat16* X, int M, int D, int hidden, const __nv_bfloat16* W1, const float* b1,
             const __nv_bfloat16* W2, const float* b2, const float* ls2, float* resid);
int launch_mlp(const MlpPlan& m, cudaStream_t s);
}  // namespace vpe
