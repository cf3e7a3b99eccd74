#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "gemm.cuh"

namespace vpe {
struct AttnPlan {
  CUtensorMap tqkv;
  __nv_bfloat16* out;
  int B, T, D, heads;
  int grid;        // persistent CTAs (<= #SMs)
  const int* sched;  // device CSR schedule: [grid + 1] offsets, then unit ids (LPT order per CTA)
  int single = 0;    // 1: a unit is one Q tile (slot B idle) -- small batches, more CTAs busy
};
// qkv: [B*T, 3D] bf16 (q | k | v column blocks, head-major inside each); out: [B*T, D] bf16
int plan_attention(AttnPlan* a, const __nv_bfloat16* qkv, __nv_bfloat16* out, int B, int T, int D, int heads);
int launch_attention(const AttnPlan& a, cudaStream_t s);
}  // namespace vpe
