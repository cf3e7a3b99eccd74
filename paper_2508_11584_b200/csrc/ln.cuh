#pragma once
// LayerNorm row math shared by the standalone kernel (misc.cu) and the GEMM that computes its A
// operand as LN(residual) in its prologue (gemm.cu, gemm_ln_kernel): one warp per row of D = NV*128
// fp32, lane l holding float4 i*32 + l. Every rounding step is spelled out so that both produce
// bit-identical bf16 (the fused path must reproduce the unfused one exactly).
#include <cuda_bf16.h>
#include <stdint.h>

#include "tc.cuh"

namespace vpe {

template <int NV>
VPE_DEV void ln_load(const float* __restrict__ x, int64_t row, int D, int lane, float4 (&v)[NV]) {
  const float4* xr = reinterpret_cast<const float4*>(x + row * D);
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = xr[i * 32 + lane];
}

// two-pass mean / variance over the warp's row (matches torch's reduction numerics closely)
template <int NV>
VPE_DEV void ln_stats(const float4 (&v)[NV], int D, float eps, float& mean, float& rstd) {
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) s = __fadd_rn(s, __fadd_rn(__fadd_rn(v[i].x, v[i].y), __fadd_rn(v[i].z, v[i].w)));
#pragma unroll
  for (int o = 16; o; o >>= 1) s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
  mean = __fdiv_rn(s, (float)D);
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const float a = __fsub_rn(v[i].x, mean), b = __fsub_rn(v[i].y, mean);
    const float c = __fsub_rn(v[i].z, mean), d = __fsub_rn(v[i].w, mean);
    q = __fadd_rn(q, __fadd_rn(__fmaf_rn(a, a, __fmul_rn(b, b)), __fmaf_rn(c, c, __fmul_rn(d, d))));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) q = __fadd_rn(q, __shfl_xor_sync(0xffffffffu, q, o));
  rstd = rsqrtf(__fadd_rn(__fdiv_rn(q, (float)D), eps));
}

// four normalised values -> w * n + b -> packed bf16 (column c = (i*32 + lane) * 4)
VPE_DEV uint2 ln_affine4(float4 v, float mean, float rstd, const float* __restrict__ w, const float* __restrict__ b,
                         int c) {
  const float4 ww = __ldg(reinterpret_cast<const float4*>(w + c));
  const float4 bb = __ldg(reinterpret_cast<const float4*>(b + c));
  uint2 u;
  u.x = pack_bf16(__fmaf_rn(__fmul_rn(__fsub_rn(v.x, mean), rstd), ww.x, bb.x),
                  __fmaf_rn(__fmul_rn(__fsub_rn(v.y, mean), rstd), ww.y, bb.y));
  u.y = pack_bf16(__fmaf_rn(__fmul_rn(__fsub_rn(v.z, mean), rstd), ww.z, bb.z),
                  __fmaf_rn(__fmul_rn(__fsub_rn(v.w, mean), rstd), ww.w, bb.w));
  return u;
}

}  // namespace vpe
