#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace vpe {
int launch_patch_im2col(const uint8_t* px, __nv_bfloat16* A, int B, int R, int KP, float* resid,
                        const float* cls_pos0, int D, cudaStream_t s);
int launch_camera_im2col(const uint8_t* hwc, int Hc, int Wc, __nv_bfloat16* A, int B, int R, int KP, float* resid,
                         const float* cls_pos0, int D, cudaStream_t s);
int launch_layernorm(const float* x, int M, int D, const float* w, const float* b, float eps, __nv_bfloat16* out,
                     const float* w2, const float* b2, __nv_bfloat16* out2, cudaStream_t s);
int launch_bilinear_ac(const __nv_bfloat16* in, int B, int Hi, int Wi, int cp, __nv_bfloat16* out, int Ho, int Wo,
                       int C, cudaStream_t s);
int launch_im2col_s2(const __nv_bfloat16* x, int B, int H, int W, int C, __nv_bfloat16* out, cudaStream_t s);
}  // namespace vpe
