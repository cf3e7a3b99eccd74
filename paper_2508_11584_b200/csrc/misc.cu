// Memory-bound kernels of the backbone and DPT neck: patch im2col + normalisation, LayerNorm
// (optionally writing the tap LayerNorm straight into a ring slot), bilinear resize, stride-2
// im2col. All coalesced, 16-byte vectorised, one pass over HBM/L2.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>

#include "bilerp.cuh"
#include "ln.cuh"
#include "misc.cuh"
#include "tc.cuh"
#include "util.cuh"

namespace vpe {

// ---------------------------------------------------------------------------------------------
// u8 NCHW frames -> normalised bf16 im2col rows [B*Np, KP] (k = c*196 + ky*14 + kx, zero pad to KP)
// Oracle: torchvision-style ImageNet normalisation + modeling_dinov2.py:139-149.
// Also writes the cls rows of the fp32 residual stream: h[b*T] = cls_token + pos[0].
__global__ void patch_im2col_kernel(const uint8_t* __restrict__ px, __nv_bfloat16* __restrict__ A, int B, int R,
                                    int KP, float* __restrict__ resid, const float* __restrict__ cls_pos0, int D) {
  pdl_wait();
  pdl_trigger();
  const int h = R / 14, np = h * h;
  const int blk = blockIdx.x;
  if (blk >= B * np) {
    const int b = blk - B * np;
    float* dst = resid + (int64_t)b * (np + 1) * D;
    for (int i = threadIdx.x; i < D; i += blockDim.x) dst[i] = cls_pos0[i];
    return;
  }
  const int b = blk / np, p = blk - b * np;
  const int py = p / h, pxx = p - py * h;
  const float mean[3] = {0.485f, 0.456f, 0.406f};
  const float stdv[3] = {0.229f, 0.224f, 0.225f};
  __nv_bfloat16* row = A + (int64_t)blk * KP;
  for (int k = threadIdx.x; k < KP; k += blockDim.x) {
    float v = 0.f;
    if (k < 588) {
      const int c = k / 196, r = k - c * 196, ky = r / 14, kx = r - ky * 14;
      const uint8_t u = px[(((int64_t)b * 3 + c) * R + (py * 14 + ky)) * R + pxx * 14 + kx];
      v = ((float)u / 255.0f - mean[c]) / stdv[c];
    }
    row[k] = __float2bfloat16_rn(v);
  }
}

// Same output, a block per 8 horizontally adjacent patches: the 3 x 14 x 112-byte source window
// is staged in smem with coalesced 4-byte loads, then written as consecutive bf16 pairs of the
// 8 im2col rows (the one-block-per-patch version issued byte loads and 2-byte scattered stores:
// 48 us at B = 16, 448). Identical arithmetic. Needs h % 8 == 0 and R % 4 == 0.
constexpr int IM_PPB = 8;
// ((u / 255) - mean) / std for every byte and channel, as a module-initialised device table:
// the host compiler's constant evaluation does the same correctly rounded IEEE single divisions
// the kernel did per CTA (768 x 2 of them: a third of its issued instructions)
struct NormLut {
  float v[3][256];
};
constexpr NormLut make_norm_lut() {
  NormLut t{};
  const float mean[3] = {0.485f, 0.456f, 0.406f};
  const float stdv[3] = {0.229f, 0.224f, 0.225f};
  for (int c = 0; c < 3; ++c)
    for (int i = 0; i < 256; ++i) t.v[c][i] = ((float)i / 255.0f - mean[c]) / stdv[c];
  return t;
}
__device__ NormLut g_norm_lut = make_norm_lut();

__global__ void __launch_bounds__(256) patch_im2col8_kernel(const uint8_t* __restrict__ px,
                                                            __nv_bfloat16* __restrict__ A, int B, int R, int KP,
                                                            float* __restrict__ resid,
                                                            const float* __restrict__ cls_pos0, int D) {
  pdl_wait();
  pdl_trigger();
  __shared__ __align__(16) uint8_t win[3 * 14][IM_PPB * 14];
  __shared__ float lut[3][256];  // ((u / 255) - mean) / std for every byte: the same IEEE divisions once
  const int h = R / 14, np = h * h, gpr = h / IM_PPB;  // patch groups per patch row
  const int blk = blockIdx.x;
  if (blk >= B * np / IM_PPB) {
    const int b = blk - B * np / IM_PPB;
    float* dst = resid + (int64_t)b * (np + 1) * D;
    for (int i = threadIdx.x; i < D; i += blockDim.x) dst[i] = cls_pos0[i];
    return;
  }
  const int b = blk / (np / IM_PPB), g = blk - b * (np / IM_PPB);
  const int py = g / gpr, gx = g - py * gpr;
  constexpr int WW = IM_PPB * 14 / 4;  // 4-byte words per window row
  for (int i = threadIdx.x; i < 42 * WW; i += blockDim.x) {
    const int rr = i / WW, w = i - rr * WW;
    const int c = rr / 14, ky = rr - c * 14;
    const uint32_t* src = reinterpret_cast<const uint32_t*>(px + (((int64_t)b * 3 + c) * R + (py * 14 + ky)) * R +
                                                            gx * IM_PPB * 14);
    reinterpret_cast<uint32_t*>(win[rr])[w] = __ldg(src + w);
  }
  for (int i = threadIdx.x; i < 3 * 256; i += blockDim.x) (&lut[0][0])[i] = (&g_norm_lut.v[0][0])[i];
  __syncthreads();
  const int pairs = KP / 2;
  __nv_bfloat16* rows = A + ((int64_t)b * np + py * h + gx * IM_PPB) * KP;
  // (patch j, pair kp) of flat index i, stepped incrementally (no runtime division by pairs)
  int j = (int)threadIdx.x / pairs, kp = (int)threadIdx.x - j * pairs;
  const int jstep = (int)blockDim.x / pairs, kstep = (int)blockDim.x - jstep * pairs;
  for (int i = threadIdx.x; i < IM_PPB * pairs; i += blockDim.x) {
    const int k = 2 * kp;
    uint32_t out = 0u;
    if (k < 588) {
      const int c = k / 196, r = k - c * 196, ky = r / 14, kx = r - ky * 14;
      const uint8_t* wr = &win[c * 14 + ky][j * 14 + kx];
      out = pack_bf16(lut[c][wr[0]], lut[c][wr[1]]);
    }
    reinterpret_cast<uint32_t*>(rows + (int64_t)j * KP)[kp] = out;
    j += jstep;
    kp += kstep;
    if (kp >= pairs) {
      kp -= pairs;
      ++j;
    }
  }
}

int launch_patch_im2col(const uint8_t* px, __nv_bfloat16* A, int B, int R, int KP, float* resid,
                        const float* cls_pos0, int D, cudaStream_t s) {
  const int np = (R / 14) * (R / 14);
  PdlKind pk(16);
  static OncePerDevice co;
  if (co.first()) {
    max_smem_carveout(patch_im2col_kernel);
  }
  const char* generic = getenv("VPE_IM2COL_GENERIC");  // parity test hook
  if ((R / 14) % IM_PPB == 0 && R % 4 == 0 && KP % 2 == 0 && !(generic && generic[0] == '1')) {
    static OncePerDevice co8;
    if (co8.first()) {
      max_smem_carveout(patch_im2col8_kernel);
    }
    return launch_k(patch_im2col8_kernel, dim3(B * np / IM_PPB + B), dim3(256), 0, s, px, A, B, R, KP, resid,
                    cls_pos0, D) == cudaSuccess
               ? VPE_OK
               : VPE_E_CUDA;
  }
  return launch_k(patch_im2col_kernel, dim3(B * np + B), dim3(128), 0, s, px, A, B, R, KP, resid, cls_pos0, D) ==
                 cudaSuccess
             ? VPE_OK
             : VPE_E_CUDA;
}

// ---------------------------------------------------------------------------------------------
// Camera ingest fused into the patch embedding: u8 HWC camera frames
// [B, Hc, Wc, 3] -> centre crop to the largest square -> bilinear resize to R x R (half-pixel
// centres, align_corners=False, no antialias: torch F.interpolate) -> ImageNet normalisation ->
// bf16 im2col rows, in one pass. Oracle: oracle/camera.py camera_preprocess.
__global__ void camera_im2col_kernel(const uint8_t* __restrict__ hwc, int Hc, int Wc, __nv_bfloat16* __restrict__ A,
                                     int B, int R, int KP, float* __restrict__ resid,
                                     const float* __restrict__ cls_pos0, int D) {
  pdl_wait();
  pdl_trigger();
  const int h = R / 14, np = h * h;
  const int blk = blockIdx.x;
  if (blk >= B * np) {
    const int b = blk - B * np;
    float* dst = resid + (int64_t)b * (np + 1) * D;
    for (int i = threadIdx.x; i < D; i += blockDim.x) dst[i] = cls_pos0[i];
    return;
  }
  const int b = blk / np, p = blk - b * np;
  const int py = p / h, pxx = p - py * h;
  const int S = Hc < Wc ? Hc : Wc;
  const int oy = (Hc - S) / 2, ox = (Wc - S) / 2;
  const float scale = (float)S / (float)R;
  const float mean[3] = {0.485f, 0.456f, 0.406f};
  const float stdv[3] = {0.229f, 0.224f, 0.225f};
  const uint8_t* img = hwc + (int64_t)b * Hc * Wc * 3;
  __nv_bfloat16* row = A + (int64_t)blk * KP;
  for (int k = threadIdx.x; k < KP; k += blockDim.x) {
    float v = 0.f;
    if (k < 588) {
      const int c = k / 196, r = k - c * 196, ky = r / 14, kx = r - ky * 14;
      const int y = py * 14 + ky, x = pxx * 14 + kx;
      float sy = (y + 0.5f) * scale - 0.5f, sx = (x + 0.5f) * scale - 0.5f;
      sy = sy < 0.f ? 0.f : sy;
      sx = sx < 0.f ? 0.f : sx;
      const int y0 = (int)sy, x0 = (int)sx;
      const int y1 = y0 + (y0 < S - 1), x1 = x0 + (x0 < S - 1);
      const float ly = sy - y0, lx = sx - x0, hy = 1.f - ly, hx = 1.f - lx;
      const uint8_t* r0 = img + ((int64_t)(oy + y0) * Wc + ox) * 3 + c;
      const uint8_t* r1 = img + ((int64_t)(oy + y1) * Wc + ox) * 3 + c;
      const float u = hy * (hx * (float)__ldg(r0 + x0 * 3) + lx * (float)__ldg(r0 + x1 * 3)) +
                      ly * (hx * (float)__ldg(r1 + x0 * 3) + lx * (float)__ldg(r1 + x1 * 3));
      v = (u / 255.0f - mean[c]) / stdv[c];
    }
    row[k] = __float2bfloat16_rn(v);
  }
}

int launch_camera_im2col(const uint8_t* hwc, int Hc, int Wc, __nv_bfloat16* A, int B, int R, int KP, float* resid,
                         const float* cls_pos0, int D, cudaStream_t s) {
  if (Hc < 1 || Wc < 1 || R % 14) return VPE_E_SHAPE;
  const int np = (R / 14) * (R / 14);
  return launch_k(camera_im2col_kernel, dim3(B * np + B), dim3(128), 0, s, hwc, Hc, Wc, A, B, R, KP, resid, cls_pos0,
                  D) == cudaSuccess
             ? VPE_OK
             : VPE_E_CUDA;
}

// ---------------------------------------------------------------------------------------------
// LayerNorm over D (multiple of 128) for fp32 rows -> bf16; optional second affine (tap LN).
// Two-pass mean/variance in registers (matches torch's reduction numerics closely).
template <int NV>
__global__ void layernorm_kernel(const float* __restrict__ x, int M, int D, const float* __restrict__ w,
                                 const float* __restrict__ b, float eps, __nv_bfloat16* __restrict__ out,
                                 const float* __restrict__ w2, const float* __restrict__ b2,
                                 __nv_bfloat16* __restrict__ out2) {
  pdl_wait();
  pdl_trigger();
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= M) return;
  float4 v[NV];
  ln_load<NV>(x, row, D, lane, v);
  float mean, rstd;
  ln_stats<NV>(v, D, eps, mean, rstd);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = (i * 32 + lane) * 4;
    if (out) *reinterpret_cast<uint2*>(out + (int64_t)row * D + c) = ln_affine4(v[i], mean, rstd, w, b, c);
    if (out2) *reinterpret_cast<uint2*>(out2 + (int64_t)row * D + c) = ln_affine4(v[i], mean, rstd, w2, b2, c);
  }
}

int launch_layernorm(const float* x, int M, int D, const float* w, const float* b, float eps, __nv_bfloat16* out,
                     const float* w2, const float* b2, __nv_bfloat16* out2, cudaStream_t s) {
  if (D % 128) return VPE_E_SHAPE;
  const int rows_per_block = 8;
  dim3 grid((M + rows_per_block - 1) / rows_per_block), block(32 * rows_per_block);
  PdlKind pk(4);
  switch (D / 128) {
#define VPE_LN(NV_) \
  case NV_: {                                                                                       \
    static OncePerDevice co;                                                                          \
    if (co.first()) {                                                                                       \
      max_smem_carveout(layernorm_kernel<NV_>);                                                      \
    }                                                                                                \
  }                                                                                                  \
    if (launch_k(layernorm_kernel<NV_>, grid, block, 0, s, x, M, D, w, b, eps, out, w2, b2, out2) != cudaSuccess) \
      return VPE_E_CUDA;                                                                             \
    break;
    VPE_LN(1) VPE_LN(2) VPE_LN(3) VPE_LN(4) VPE_LN(5) VPE_LN(6) VPE_LN(8) VPE_LN(10) VPE_LN(12)
#undef VPE_LN
    default:
      return VPE_E_SHAPE;
  }
  return cudaGetLastError() == cudaSuccess ? VPE_OK : VPE_E_CUDA;
}

// ---------------------------------------------------------------------------------------------
// Bilinear resize on NHWC bf16, align_corners=True (modeling_depth_anything.py:157-200, 288-293).
// Thread = up to 32 channels (4 x 16 B) of one output pixel: the bilinear weights are computed
// once and 16 independent 16-byte loads are in flight per thread. Channel pitch cp, C real.
template <int NV>
__global__ void __launch_bounds__(256) bilinear_ac_kernel(const __nv_bfloat16* __restrict__ in, int B, int Hi,
                                                          int Wi, int cp, __nv_bfloat16* __restrict__ out, int Ho,
                                                          int Wo, int C) {
  // 32-bit index math (64-bit div/mod is a long software sequence; B*Ho*Wo*groups < 2^31 is
  // checked by the launcher)
  const int groups = C / (8 * NV);
  const int total = B * Ho * Wo * groups;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= total) return;
  const int g = groups == 1 ? 0 : t % groups;
  int pix = groups == 1 ? t : t / groups;
  const int ox = pix % Wo;
  pix /= Wo;
  const int oy = pix % Ho;
  const int b = pix / Ho;
  const AcCoord cy = ac_coord(ac_scale(Hi, Ho), oy, Hi), cx = ac_coord(ac_scale(Wi, Wo), ox, Wi);
  const int y0 = cy.i0, y1 = cy.i1, x0 = cx.i0, x1 = cx.i1;
  const float ly = cy.l, hy = cy.h, lx = cx.l, hx = cx.h;
  const __nv_bfloat16* base = in + (int64_t)b * Hi * Wi * cp + g * 8 * NV;
  const uint4* p00 = reinterpret_cast<const uint4*>(base + ((int64_t)y0 * Wi + x0) * cp);
  const uint4* p01 = reinterpret_cast<const uint4*>(base + ((int64_t)y0 * Wi + x1) * cp);
  const uint4* p10 = reinterpret_cast<const uint4*>(base + ((int64_t)y1 * Wi + x0) * cp);
  const uint4* p11 = reinterpret_cast<const uint4*>(base + ((int64_t)y1 * Wi + x1) * cp);
  uint4 a[NV], bq[NV], c[NV], d[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    a[v] = __ldg(p00 + v);
    bq[v] = __ldg(p01 + v);
    c[v] = __ldg(p10 + v);
    d[v] = __ldg(p11 + v);
  }
  uint4* dst = reinterpret_cast<uint4*>(out + (((int64_t)b * Ho + oy) * Wo + ox) * cp + g * 8 * NV);
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const __nv_bfloat162* pa = reinterpret_cast<const __nv_bfloat162*>(&a[v]);
    const __nv_bfloat162* pb = reinterpret_cast<const __nv_bfloat162*>(&bq[v]);
    const __nv_bfloat162* pc = reinterpret_cast<const __nv_bfloat162*>(&c[v]);
    const __nv_bfloat162* pd = reinterpret_cast<const __nv_bfloat162*>(&d[v]);
    uint4 o;
    uint32_t* po = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 fa = __bfloat1622float2(pa[j]), fb = __bfloat1622float2(pb[j]);
      const float2 fc = __bfloat1622float2(pc[j]), fd = __bfloat1622float2(pd[j]);
      const float r0 = bilerp(fa.x, fb.x, fc.x, fd.x, hx, lx, hy, ly);
      const float r1 = bilerp(fa.y, fb.y, fc.y, fd.y, hx, lx, hy, ly);
      po[j] = pack_bf16(r0, r1);
    }
    dst[v] = o;
  }
}

// Row-staged variant: a CTA produces one output row of one image. The two source rows it reads
// are staged in shared memory with coalesced 16-byte loads, so the per-pixel corner gathers hit
// smem instead of issuing 16 scattered L1/L2 requests per thread (the gather version ran at
// ~1.5-2 TB/s). Same fp32 arithmetic and rounding order as bilinear_ac_kernel.
__global__ void __launch_bounds__(256) bilinear_ac_rows_kernel(const __nv_bfloat16* __restrict__ in, int Hi, int Wi,
                                                               int cp, __nv_bfloat16* __restrict__ out, int Ho,
                                                               int Wo, int C) {
  extern __shared__ __align__(16) uint8_t s_rows[];  // [2][Wi][cp] bf16
  const int oy = blockIdx.x, b = blockIdx.y;
  const float sw = ac_scale(Wi, Wo);
  const AcCoord cy = ac_coord(ac_scale(Hi, Ho), oy, Hi);
  const int y0 = cy.i0, y1 = cy.i1;
  const float ly = cy.l, hy = cy.h;
  const int row_vec = Wi * cp / 8;  // uint4 per source row
  const uint4* src0 = reinterpret_cast<const uint4*>(in + ((int64_t)b * Hi + y0) * Wi * cp);
  const uint4* src1 = reinterpret_cast<const uint4*>(in + ((int64_t)b * Hi + y1) * Wi * cp);
  uint4* r0 = reinterpret_cast<uint4*>(s_rows);
  uint4* r1 = r0 + row_vec;
  for (int i = threadIdx.x; i < row_vec; i += blockDim.x) {
    r0[i] = __ldg(src0 + i);
    r1[i] = __ldg(src1 + i);
  }
  __syncthreads();
  const int groups = C / 8;
  const int lg = (groups & (groups - 1)) == 0 ? __ffs(groups) - 1 : -1;  // power of two: shift
  uint4* dst = reinterpret_cast<uint4*>(out + ((int64_t)b * Ho + oy) * Wo * cp);
  const uint64_t hy2 = f2_pack(hy, hy), ly2 = f2_pack(ly, ly);
  // bf16 pair -> f32x2 (exact), then bilerp() per lane on f32x2: the same IEEE operations and
  // order, half the FP instructions
  auto up = [](uint32_t w) { return f2_pack(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u)); };
  for (int t = threadIdx.x; t < Wo * groups; t += blockDim.x) {
    const int ox = lg >= 0 ? t >> lg : t / groups, g = t - ox * groups;
    const AcCoord cx = ac_coord(sw, ox, Wi);
    const int x0 = cx.i0, x1 = cx.i1;
    const uint64_t hx2 = f2_pack(cx.h, cx.h), lx2 = f2_pack(cx.l, cx.l);
    const uint4 a = r0[(x0 * cp) / 8 + g], bq = r0[(x1 * cp) / 8 + g];
    const uint4 c = r1[(x0 * cp) / 8 + g], d = r1[(x1 * cp) / 8 + g];
    const uint32_t aw[4] = {a.x, a.y, a.z, a.w}, bw[4] = {bq.x, bq.y, bq.z, bq.w};
    const uint32_t cw[4] = {c.x, c.y, c.z, c.w}, dw[4] = {d.x, d.y, d.z, d.w};
    uint32_t po[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint64_t t0 = ffma2(lx2, up(bw[j]), fmul2(hx2, up(aw[j])));
      const uint64_t t1 = ffma2(lx2, up(dw[j]), fmul2(hx2, up(cw[j])));
      float v0, v1;
      f2_unpack(ffma2(ly2, t1, fmul2(hy2, t0)), v0, v1);
      po[j] = pack_bf16(v0, v1);
    }
    dst[(ox * cp) / 8 + g] = make_uint4(po[0], po[1], po[2], po[3]);
  }
}

int launch_bilinear_ac(const __nv_bfloat16* in, int B, int Hi, int Wi, int cp, __nv_bfloat16* out, int Ho, int Wo,
                       int C, cudaStream_t s) {
  if (C % 8 || cp % 8) return VPE_E_SHAPE;
  const size_t row_bytes = (size_t)Wi * cp * 2;
  // (tried: bands of up to 8 output rows sharing one bulk-copied source span per CTA -- 207 vs
  // 178 us for the step's five resizes, fewer CTAs in flight)
  static const int mode = getenv("VPE_BILINEAR_GATHER") ? 2 : 0;
  const size_t rows_smem = 2 * row_bytes;
  if (rows_smem <= 96 * 1024 && mode != 2) {
    static OncePerDevice attr;
    if (attr.first()) {
      cudaFuncSetAttribute(bilinear_ac_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
      max_smem_carveout(bilinear_ac_rows_kernel);
    }
    bilinear_ac_rows_kernel<<<dim3(Ho, B), 256, rows_smem, s>>>(in, Hi, Wi, cp, out, Ho, Wo, C);
    return cudaGetLastError() == cudaSuccess ? VPE_OK : VPE_E_CUDA;
  }
  if ((int64_t)B * Ho * Wo * (C / 8) >= (int64_t)1 << 31) return VPE_E_SHAPE;
  const int nv = (C % 32 == 0) ? 4 : 1;
  const int64_t total = (int64_t)B * Ho * Wo * (C / (8 * nv));
  const unsigned blocks = (unsigned)((total + 255) / 256);
  if (nv == 4)
    bilinear_ac_kernel<4><<<blocks, 256, 0, s>>>(in, B, Hi, Wi, cp, out, Ho, Wo, C);
  else
    bilinear_ac_kernel<1><<<blocks, 256, 0, s>>>(in, B, Hi, Wi, cp, out, Ho, Wo, C);
  return cudaGetLastError() == cudaSuccess ? VPE_OK : VPE_E_CUDA;
}

// ---------------------------------------------------------------------------------------------
// im2col for a 3x3 stride-2 pad-1 conv on NHWC bf16 [B,H,W,C] -> [B*Ho*Wo, 9*C] (tap-major)
__global__ void im2col_s2_kernel(const __nv_bfloat16* __restrict__ x, int B, int H, int W, int C,
                                 __nv_bfloat16* __restrict__ out, int Ho, int Wo) {
  const int cv = C / 8;
  const int total = B * Ho * Wo * 9 * cv;  // < 2^31 (checked by the launcher): 32-bit div/mod
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= total) return;
  const int c8 = t % cv;
  int r = t / cv;
  const int tap = r % 9;
  r /= 9;
  const int ox = r % Wo;
  r /= Wo;
  const int oy = r % Ho;
  const int b = r / Ho;
  const int iy = 2 * oy - 1 + tap / 3, ix = 2 * ox - 1 + tap % 3;
  uint4 v = make_uint4(0, 0, 0, 0);
  if (iy >= 0 && iy < H && ix >= 0 && ix < W)
    v = *reinterpret_cast<const uint4*>(x + (((int64_t)b * H + iy) * W + ix) * C + c8 * 8);
  *reinterpret_cast<uint4*>(out + ((((int64_t)b * Ho + oy) * Wo + ox) * 9 + tap) * C + c8 * 8) = v;
}

int launch_im2col_s2(const __nv_bfloat16* x, int B, int H, int W, int C, __nv_bfloat16* out, cudaStream_t s) {
  if (C % 8) return VPE_E_SHAPE;
  const int Ho = (H + 1) / 2, Wo = (W + 1) / 2;
  const int64_t total = (int64_t)B * Ho * Wo * 9 * (C / 8);
  if (total >= ((int64_t)1 << 31)) return VPE_E_SHAPE;
  static OncePerDevice co;
  if (co.first()) {
    max_smem_carveout(im2col_s2_kernel);
  }
  im2col_s2_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(x, B, H, W, C, out, Ho, Wo);
  return cudaGetLastError() == cudaSuccess ? VPE_OK : VPE_E_CUDA;
}

}  // namespace vpe
