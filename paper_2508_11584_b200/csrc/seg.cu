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
constexpr int BAND_COLS = 112;  // output columns per CTA (8 source cells)
constexpr int SEG_THREADS = 256;

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

// Separable form of torch's bilinear (align_corners=False) + argmax, identical rounding order:
//   out = (x00*w0 + x01*w1)*h0 + (x10*w0 + x11*w1)*h1 = A(y0)*h0 + A(y1)*h1,
//   A(y, ox) = x(y, x0)*w0 + x(y, x1)*w1.
// A CTA owns half a source band (7 output rows, which all read the same two source rows) and 56
// output columns; A for those 2 rows x 56 columns x all classes is built once in SMEM
// ([row][class][column], conflict-free), then every pixel does 2 loads + 3 flops per class.
constexpr int SEG_COLS = 56;
__global__ void __launch_bounds__(SEG_THREADS)
    seg_upsample_argmax_kernel(const float* __restrict__ logits, int h, int C, int cp, int R,
                               uint8_t* __restrict__ labels) {
  extern __shared__ float s_mem[];
  const int wcols = 6;
  float* s_src = s_mem;                      // [2 rows][6 cols][C]
  float* s_a = s_mem + 2 * wcols * C;        // [2 rows][C][SEG_COLS]
  const int hb = blockIdx.x, chunk = blockIdx.y, b = blockIdx.z;
  const int rows_per_band = R / h;   // 14
  const int half_rows = rows_per_band / 2;
  const float scale = (float)h / (float)R;
  const int oy0 = hb * half_rows, ox0 = chunk * SEG_COLS;
  int y0, y1;
  float hy0_unused, hy1_unused;
  src_index(scale, oy0, h, y0, y1, hy0_unused, hy1_unused);
  const int sx0 = max(chunk * (SEG_COLS / rows_per_band) - 1, 0);
  const float* src = logits + (int64_t)b * h * h * cp;
  for (int i = threadIdx.x; i < 2 * wcols * C; i += blockDim.x) {
    const int c = i % C, pix = i / C;
    const int yy = pix / wcols ? y1 : y0, xx = sx0 + pix % wcols;
    s_src[i] = xx < h ? src[((int64_t)yy * h + xx) * cp + c] : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * C * SEG_COLS; i += blockDim.x) {
    const int ox = i % SEG_COLS, rc = i / SEG_COLS;
    const int c = rc % C, yy = rc / C;
    int x0, x1;
    float wx0, wx1;
    src_index(scale, min(ox0 + ox, R - 1), h, x0, x1, wx0, wx1);
    const float* row = s_src + yy * wcols * C + c;
    s_a[i] = __fadd_rn(__fmul_rn(row[(x0 - sx0) * C], wx0), __fmul_rn(row[(x1 - sx0) * C], wx1));
  }
  __syncthreads();
  for (int p = threadIdx.x; p < half_rows * SEG_COLS; p += blockDim.x) {
    const int oy = oy0 + p / SEG_COLS, ox = p % SEG_COLS;
    int yy0, yy1;
    float hy0, hy1;
    src_index(scale, oy, h, yy0, yy1, hy0, hy1);
    const float* a0 = s_a + ox;
    const float* a1 = s_a + C * SEG_COLS + ox;
    float best = -INFINITY;
    int arg = 0;
#pragma unroll 4
    for (int c = 0; c < C; ++c) {
      const float v = __fadd_rn(__fmul_rn(a0[c * SEG_COLS], hy0), __fmul_rn(a1[c * SEG_COLS], hy1));
      if (v > best) {
        best = v;
        arg = c;
      }
    }
    if (ox0 + ox < R) labels[((int64_t)b * R + oy) * R + ox0 + ox] = (uint8_t)arg;
  }
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
  dim3 grid(2 * h, (R + SEG_COLS - 1) / SEG_COLS, B);
  const size_t smem = ((size_t)2 * 6 * C + 2 * C * SEG_COLS) * sizeof(float);
  static bool attr = false;
  if (!attr) {
    VPE_CUDA_TRY(cudaFuncSetAttribute(seg_upsample_argmax_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)((2 * 6 * 256 + 2 * 256 * SEG_COLS) * sizeof(float))));
    attr = true;
  }
  seg_upsample_argmax_kernel<<<grid, SEG_THREADS, smem, st>>>(s->logits, h, C, s->cpitch, R, labels);
  VPE_CUDA_TRY(cudaGetLastError());
  count_launches(2);
  if (logits_out) {
    VPE_CUDA_TRY(cudaMemcpy2DAsync(logits_out, (size_t)C * 4, s->logits, (size_t)s->cpitch * 4, (size_t)C * 4,
                                   (size_t)B * h * h, cudaMemcpyDeviceToDevice, st));
  }
  return VPE_OK;
}
