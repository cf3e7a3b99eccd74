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

__global__ void __launch_bounds__(SEG_THREADS)
    seg_upsample_argmax_kernel(const float* __restrict__ logits, int h, int C, int cp, int R,
                               uint8_t* __restrict__ labels) {
  extern __shared__ float s_log[];  // [3 rows][10 cols][C]
  const int band = blockIdx.x, chunk = blockIdx.y, b = blockIdx.z;
  const int rows_per_band = R / h;  // 14
  const float scale = (float)h / (float)R;
  const int oy0 = band * rows_per_band, ox0 = chunk * BAND_COLS;
  // source window (rows band-1..band+1, cols 8*chunk-1 .. 8*chunk+8), clamped
  const int sy0 = max(band - 1, 0);
  const int sx0 = max(chunk * (BAND_COLS / rows_per_band) - 1, 0);
  const int wcols = 10, wrows = 3;
  const float* src = logits + (int64_t)b * h * h * cp;
  for (int i = threadIdx.x; i < wrows * wcols * C; i += blockDim.x) {
    const int c = i % C, pix = i / C;
    const int yy = sy0 + pix / wcols, xx = sx0 + pix % wcols;
    s_log[i] = (yy < h && xx < h) ? src[((int64_t)yy * h + xx) * cp + c] : 0.f;
  }
  __syncthreads();
  const int npx = rows_per_band * BAND_COLS;
  for (int p = threadIdx.x; p < npx; p += blockDim.x) {
    const int oy = oy0 + p / BAND_COLS, ox = ox0 + p % BAND_COLS;
    if (oy >= R || ox >= R) continue;
    int y0, y1, x0, x1;
    float hy0, hy1, wx0, wx1;
    src_index(scale, oy, h, y0, y1, hy0, hy1);
    src_index(scale, ox, h, x0, x1, wx0, wx1);
    const float* r00 = s_log + ((y0 - sy0) * wcols + (x0 - sx0)) * C;
    const float* r01 = s_log + ((y0 - sy0) * wcols + (x1 - sx0)) * C;
    const float* r10 = s_log + ((y1 - sy0) * wcols + (x0 - sx0)) * C;
    const float* r11 = s_log + ((y1 - sy0) * wcols + (x1 - sx0)) * C;
    float best = -INFINITY;
    int arg = 0;
    for (int c = 0; c < C; ++c) {
      // torch CPU order: (x00*w0 + x01*w1)*h0 + (x10*w0 + x11*w1)*h1
      const float t0 = __fadd_rn(__fmul_rn(r00[c], wx0), __fmul_rn(r01[c], wx1));
      const float t1 = __fadd_rn(__fmul_rn(r10[c], wx0), __fmul_rn(r11[c], wx1));
      const float v = __fadd_rn(__fmul_rn(t0, hy0), __fmul_rn(t1, hy1));
      if (v > best) {
        best = v;
        arg = c;
      }
    }
    labels[((int64_t)b * R + oy) * R + ox] = (uint8_t)arg;
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
  dim3 grid(h, (R + BAND_COLS - 1) / BAND_COLS, B);
  const size_t smem = (size_t)3 * 10 * C * sizeof(float);
  seg_upsample_argmax_kernel<<<grid, SEG_THREADS, smem, st>>>(s->logits, h, C, s->cpitch, R, labels);
  VPE_CUDA_TRY(cudaGetLastError());
  count_launches(2);
  if (logits_out) {
    VPE_CUDA_TRY(cudaMemcpy2DAsync(logits_out, (size_t)C * 4, s->logits, (size_t)s->cpitch * 4, (size_t)C * 4,
                                   (size_t)B * h * h, cudaMemcpyDeviceToDevice, st));
  }
  return VPE_OK;
}
