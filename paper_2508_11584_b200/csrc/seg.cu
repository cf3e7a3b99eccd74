// Linear segmentation head ("b200_linseg"): BN-folded 1x1 conv D->C read in place from the ring's
// `final` tap (as an NHWC image, cls row skipped) on tcgen05 with split-precision weights
// (hi+lo bf16 -> ~fp32 logits), then ONE fused bilinear(align_corners=False)-upsample + argmax
// pass that never materialises the [C, R, R] logit volume (the CPU oracle's 120 MB temporary).
// Oracle: oracle/seg.py.
#include <cuda_runtime.h>

#include <new>

#include "gemm.cuh"
#include "runtime.h"
#include "util.cuh"

using namespace vpe;

struct vpe_seg {
  vpe_seg_config cfg;
  vpe_seg_weights w;
  int h = 0, cpitch = 0;
  float* logits = nullptr;  // [B, h*h, cpitch]
  const void* bound = nullptr;
  GemmPlan g;
};

namespace {

// source index per torch's area_pixel_compute_source_index (align_corners=False, no cubic)
__device__ __forceinline__ void src_index(float scale, int dst, int in_size, int& i0, int& i1, float& l0,
                                          float& l1) {
  float s = scale * ((float)dst + 0.5f) - 0.5f;
  if (s < 0.f) s = 0.f;
  i0 = (int)s;
  i1 = i0 + ((i0 < in_size - 1) ? 1 : 0);
  l1 = fminf(fmaxf(s - (float)i0, 0.f), 1.f);
  l0 = 1.f - l1;
}

// Fused bilinear (align_corners=False) upsample + argmax, torch's rounding order
//   out = (x00*w0 + x01*w1)*h0 + (x10*w0 + x11*w1)*h1.
// A CTA owns half a source band: the 7 output rows that all read the same two source rows, every
// output column of them (one thread per column). Per class a thread loads the 4 corner logits
// once, forms the two x-interpolations once and reuses them for its 7 output pixels, keeping 7
// running (max, argmax) pairs in registers; the [C, R, R] logit volume never exists.
constexpr int HALF_ROWS = 7;  // R / h / 2
__global__ void __launch_bounds__(1024)
    seg_upsample_argmax_kernel(const float* __restrict__ logits, int h, int C, int cp, int R,
                               uint8_t* __restrict__ labels) {
  extern __shared__ float s_src[];  // [2 rows][h cols][C]
  const int hb = blockIdx.x, b = blockIdx.y;
  const float scale = (float)h / (float)R;
  const int oy0 = hb * HALF_ROWS;
  int y0, y1;
  float hy0_unused, hy1_unused;
  src_index(scale, oy0, h, y0, y1, hy0_unused, hy1_unused);
  const float* src = logits + (int64_t)b * h * h * cp;
  for (int i = threadIdx.x; i < 2 * h * C; i += blockDim.x) {
    const int c = i % C, pix = i / C;
    const int yy = pix / h ? y1 : y0, xx = pix % h;
    s_src[i] = src[((int64_t)yy * h + xx) * cp + c];
  }
  __syncthreads();
  const int ox = threadIdx.x;
  if (ox >= R) return;
  int x0, x1;
  float wx0, wx1;
  src_index(scale, ox, h, x0, x1, wx0, wx1);
  float hy0[HALF_ROWS], hy1[HALF_ROWS], best[HALF_ROWS];
  int arg[HALF_ROWS];
#pragma unroll
  for (int k = 0; k < HALF_ROWS; ++k) {
    int a0, a1;
    src_index(scale, oy0 + k, h, a0, a1, hy0[k], hy1[k]);
    best[k] = -INFINITY;
    arg[k] = 0;
  }
  const float* r0 = s_src;
  const float* r1 = s_src + h * C;
#pragma unroll 2
  for (int c = 0; c < C; ++c) {
    const float t0 = __fadd_rn(__fmul_rn(r0[x0 * C + c], wx0), __fmul_rn(r0[x1 * C + c], wx1));
    const float t1 = __fadd_rn(__fmul_rn(r1[x0 * C + c], wx0), __fmul_rn(r1[x1 * C + c], wx1));
#pragma unroll
    for (int k = 0; k < HALF_ROWS; ++k) {
      const float v = __fadd_rn(__fmul_rn(t0, hy0[k]), __fmul_rn(t1, hy1[k]));
      if (v > best[k]) {
        best[k] = v;
        arg[k] = c;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < HALF_ROWS; ++k) labels[((int64_t)b * R + oy0 + k) * R + ox] = (uint8_t)arg[k];
}
}  // namespace

extern "C" int vpe_seg_create(const vpe_seg_config* cfg, const vpe_seg_weights* w, vpe_seg** out) {
  if (!cfg || !w || !out) return VPE_E_VALUE;
  if (cfg->classes < 1 || cfg->classes > 256 || cfg->resolution % 14 || cfg->dim % 64) return VPE_E_CONFIG;
  vpe_seg* s = new (std::nothrow) vpe_seg();
  if (!s) return VPE_E_RESOURCE;
  s->cfg = *cfg;
  s->w = *w;
  s->h = cfg->resolution / 14;
  s->cpitch = (cfg->classes + 31) / 32 * 32;
  if (cudaMalloc(&s->logits, (size_t)cfg->batch * s->h * s->h * s->cpitch * 4) != cudaSuccess) {
    delete s;
    return VPE_E_RESOURCE;
  }
  *out = s;
  return VPE_OK;
}

extern "C" int vpe_seg_destroy(vpe_seg* s) {
  if (!s) return VPE_OK;
  cudaFree(s->logits);
  delete s;
  return VPE_OK;
}

extern "C" int vpe_seg_forward(vpe_seg* s, const void* final_tap, uint8_t* labels, float* logits_out, void* stream) {
  if (!s || !final_tap || !labels) return VPE_E_VALUE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int D = s->cfg.dim, h = s->h, B = s->cfg.batch, T = h * h + 1, C = s->cfg.classes;
  if (s->bound != final_tap) {
    EpiParams ep;
    ep.kind = EPI_F32;
    ep.N = C;
    ep.bias = s->w.b;
    ep.out = s->logits;
    ep.ldo = s->cpitch;
    const __nv_bfloat16* x = static_cast<const __nv_bfloat16*>(final_tap) + D;  // skip cls row
    VPE_TRY(plan_gemm_conv(&s->g, x, B, h, h, D, D, (int64_t)h * D, (int64_t)T * D, 1, 64,
                           static_cast<const __nv_bfloat16*>(s->w.w_split), C, 2 * D, 2 * D, ep, 32));
    s->bound = final_tap;
  }
  VPE_TRY(launch_gemm(s->g, st));
  const int R = s->cfg.resolution;
  dim3 grid(2 * h, B);
  const size_t smem = (size_t)2 * h * C * sizeof(float);
  static bool attr = false;
  if (!attr) {
    VPE_CUDA_TRY(cudaFuncSetAttribute(seg_upsample_argmax_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      227 * 1024));
    attr = true;
  }
  if (R > 1024 || R != 14 * h || smem > 227 * 1024) return VPE_E_CONFIG;
  seg_upsample_argmax_kernel<<<grid, (R + 31) / 32 * 32, smem, st>>>(s->logits, h, C, s->cpitch, R, labels);
  VPE_CUDA_TRY(cudaGetLastError());
  count_launches(2);
  if (logits_out) {
    VPE_CUDA_TRY(cudaMemcpy2DAsync(logits_out, (size_t)C * 4, s->logits, (size_t)s->cpitch * 4, (size_t)C * 4,
                                   (size_t)B * h * h, cudaMemcpyDeviceToDevice, st));
  }
  return VPE_OK;
}
