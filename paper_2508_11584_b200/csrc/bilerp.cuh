// align_corners=True bilinear sampling shared by the resize kernels (misc.cu) and the
// upsample-fused 3x3 conv (gemm.cu conv_up_kernel), so every path rounds identically and the
// fused conv sees bit-for-bit the tensor the standalone resize would have written.
// Oracle: F.interpolate(mode="bilinear", align_corners=True) (modeling_depth_anything.py:157-200,
// 288-293): src = o * (n_in - 1) / (n_out - 1).
#pragma once
#include <cuda_runtime.h>

namespace vpe {

__host__ __device__ inline float ac_scale(int n_in, int n_out) {
  return n_out > 1 ? (float)(n_in - 1) / (float)(n_out - 1) : 0.f;
}

struct AcCoord {
  int i0, i1;   // source taps (i1 == i0 on the last source row/column)
  float l, h;   // weights of i1 and i0
};

// Products and differences spelled as _rn intrinsics: no FMA contraction, so the host planner
// and every kernel agree on i0 (the planner sizes the fused conv's source boxes from it).
__device__ __forceinline__ AcCoord ac_coord(float s, int o, int n_in) {
  const float f = __fmul_rn(s, (float)o);
  AcCoord c;
  c.i0 = (int)f;
  c.i1 = c.i0 + (c.i0 < n_in - 1);
  c.l = __fsub_rn(f, (float)c.i0);
  c.h = __fsub_rn(1.f, c.l);
  return c;
}
inline int ac_i0_host(float s, int o) {
  volatile float f = s * (float)o;  // IEEE single multiply, as __fmul_rn
  return (int)f;
}

// hy*(hx*a + lx*b) + ly*(hx*c + lx*d) with the FMA contraction spelled out
__device__ __forceinline__ float bilerp(float a, float b, float c, float d, float hx, float lx, float hy, float ly) {
  const float t0 = __fmaf_rn(lx, b, __fmul_rn(hx, a));
  const float t1 = __fmaf_rn(lx, d, __fmul_rn(hx, c));
  return __fmaf_rn(ly, t1, __fmul_rn(hy, t0));
}

}  // namespace vpe
