// Linear segmentation head ("b200_linseg"): BN-folded 1x1 conv D->C read in place from the ring's
// `final` tap (as an NHWC image, cls row skipped) on tcgen05 with split-precision weights
// (hi+lo bf16 -> ~fp32 logits), then ONE fused bilinear(align_corners=False)-upsample + argmax
// pass that never materialises the [C, R, R] logit volume (the CPU oracle's 120 MB temporary).
// Oracle: oracle/seg.py.
#include <cuda_runtime.h>

#include <cstdlib>
#include <new>

#include "gemm.cuh"
#include "tc.cuh"
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
  float s = __fmaf_rn(scale, (float)dst + 0.5f, -0.5f);  // explicit: this file builds with --fmad=false
  if (s < 0.f) s = 0.f;
  i0 = (int)s;
  i1 = i0 + ((i0 < in_size - 1) ? 1 : 0);
  l1 = fminf(fmaxf(s - (float)i0, 0.f), 1.f);
  l0 = 1.f - l1;
}

// Fused bilinear (align_corners=False) upsample + argmax, torch's rounding order
//   out = (x00*w0 + x01*w1)*h0 + (x10*w0 + x11*w1)*h1.
// A CTA owns half a source band: the 7 output rows that all read the same two source rows, every
// output column of them (one thread per column); the [C, R, R] logit volume never exists.
// Instruction diet (the kernel is issue-bound): classes go two at a time through packed f32x2
// mul/add (IEEE RN per lane, so bit-identical to the scalar formula), the x-interpolations are
// shared by the 7 rows, and the running argmax is kept per chunk of SEG_G classes — a 3-input max
// per class pair, one compare per chunk — with the index recovered at the end by re-evaluating
// only the winning chunk and taking its first class equal to the maximum (torch's first-occurrence
// tie rule: a later chunk only wins on a strictly greater maximum).
constexpr int HALF_ROWS = 7;  // R / h / 2
constexpr int SEG_G = 8;      // classes per argmax chunk

__device__ __forceinline__ float seg_fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
// a*b rounded once, as fma(a, b, z) with z a +0 pair the compiler cannot see: ptxas contracts
// mul.rn.f32x2 + add.rn.f32x2 into FFMA2 even under --fmad=false, which would change the rounding
// (only the sign of an exact-zero product can differ from mul.rn, and -0 == +0 in every compare)
__device__ __forceinline__ uint64_t seg_mul2(uint64_t a, uint64_t b, uint64_t z) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(z));
  return d;
}
__device__ __forceinline__ float seg_value(const float* r0, const float* r1, int x0, int x1, int cs, int c, float wx0,
                                           float wx1, float h0, float h1) {
  const float t0 = __fadd_rn(__fmul_rn(r0[x0 * cs + c], wx0), __fmul_rn(r0[x1 * cs + c], wx1));
  const float t1 = __fadd_rn(__fmul_rn(r1[x0 * cs + c], wx0), __fmul_rn(r1[x1 * cs + c], wx1));
  return __fadd_rn(__fmul_rn(t0, h0), __fmul_rn(t1, h1));
}

__global__ void __launch_bounds__(1024)
    seg_upsample_argmax_kernel(const float* __restrict__ logits, int h, int C, int cp, int R,
                               uint8_t* __restrict__ labels, float zero) {
  extern __shared__ float s_src[];  // [2 rows][h cols][cs], cs = C rounded up to even
  const int cs = (C + 1) & ~1;
  const int hb = blockIdx.x, b = blockIdx.y;
  const float scale = (float)h / (float)R;
  const int oy0 = hb * HALF_ROWS;
  int y0, y1;
  float hy0_unused, hy1_unused;
  src_index(scale, oy0, h, y0, y1, hy0_unused, hy1_unused);
  const float* src = logits + (int64_t)b * h * h * cp;
  {  // stage the two source rows: one warp per source pixel, lanes across classes (no div/mod)
    const int nw = blockDim.x >> 5, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int pix = wid; pix < 2 * h; pix += nw) {
      const int yy = pix < h ? y0 : y1, xx = pix < h ? pix : pix - h;
      const float* g = src + ((int64_t)yy * h + xx) * cp;
      float* d = s_src + pix * cs;
#pragma unroll 4
      for (int c = lane; c < cs; c += 32) d[c] = c < C ? __ldg(g + c) : 0.f;
    }
  }
  __syncthreads();
  const int ox = threadIdx.x;
  if (ox >= R) return;
  int x0, x1;
  float wx0, wx1;
  src_index(scale, ox, h, x0, x1, wx0, wx1);
  float hy0[HALF_ROWS], hy1[HALF_ROWS], best[HALF_ROWS];
  uint64_t H0[HALF_ROWS], H1[HALF_ROWS];
  int arg[HALF_ROWS];
#pragma unroll
  for (int k = 0; k < HALF_ROWS; ++k) {
    int a0, a1;
    src_index(scale, oy0 + k, h, a0, a1, hy0[k], hy1[k]);
    H0[k] = f2_pack(hy0[k], hy0[k]);
    H1[k] = f2_pack(hy1[k], hy1[k]);
    best[k] = -INFINITY;
    arg[k] = 0;  // chunk start until the final pass
  }
  const uint64_t W0 = f2_pack(wx0, wx0), W1 = f2_pack(wx1, wx1), Z = f2_pack(zero, zero);
  const float* r0 = s_src;
  const float* r1 = s_src + h * cs;
  const uint64_t* p00 = reinterpret_cast<const uint64_t*>(r0 + x0 * cs);
  const uint64_t* p01 = reinterpret_cast<const uint64_t*>(r0 + x1 * cs);
  const uint64_t* p10 = reinterpret_cast<const uint64_t*>(r1 + x0 * cs);
  const uint64_t* p11 = reinterpret_cast<const uint64_t*>(r1 + x1 * cs);
  const int cg = C / SEG_G * SEG_G;
#pragma unroll 1
  for (int c0 = 0; c0 < cg; c0 += SEG_G) {
    float m[HALF_ROWS];
#pragma unroll
    for (int k = 0; k < HALF_ROWS; ++k) m[k] = -INFINITY;
#pragma unroll
    for (int pc = 0; pc < SEG_G / 2; ++pc) {
      const int q = (c0 >> 1) + pc;  // class pair (c, c + 1)
      const uint64_t T0 = fadd2(seg_mul2(p00[q], W0, Z), seg_mul2(p01[q], W1, Z));
      const uint64_t T1 = fadd2(seg_mul2(p10[q], W0, Z), seg_mul2(p11[q], W1, Z));
#pragma unroll
      for (int k = 0; k < HALF_ROWS; ++k) {
        float va, vb;
        f2_unpack(fadd2(seg_mul2(T0, H0[k], Z), seg_mul2(T1, H1[k], Z)), va, vb);
        m[k] = seg_fmax3(m[k], va, vb);
      }
    }
#pragma unroll
    for (int k = 0; k < HALF_ROWS; ++k) {
      if (m[k] > best[k]) {
        best[k] = m[k];
        arg[k] = c0;
      }
    }
  }
#pragma unroll 1
  for (int c = cg; c < C; ++c) {  // tail classes: a chunk of one
#pragma unroll
    for (int k = 0; k < HALF_ROWS; ++k) {
      const float v = seg_value(r0, r1, x0, x1, cs, c, wx0, wx1, hy0[k], hy1[k]);
      if (v > best[k]) {
        best[k] = v;
        arg[k] = c;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < HALF_ROWS; ++k) {
    const int c0 = arg[k];
    if (c0 < cg) {  // winning chunk: first class of it equal to the max, two classes at a time
#pragma unroll 1
      for (int q = c0 >> 1; q < (c0 + SEG_G) >> 1; ++q) {
        const uint64_t T0 = fadd2(seg_mul2(p00[q], W0, Z), seg_mul2(p01[q], W1, Z));
        const uint64_t T1 = fadd2(seg_mul2(p10[q], W0, Z), seg_mul2(p11[q], W1, Z));
        float va, vb;
        f2_unpack(fadd2(seg_mul2(T0, H0[k], Z), seg_mul2(T1, H1[k], Z)), va, vb);
        if (va == best[k]) {
          arg[k] = 2 * q;
          break;
        }
        if (vb == best[k]) {
          arg[k] = 2 * q + 1;
          break;
        }
      }
    }  // else a tail class won outright and arg[k] is already its index
    labels[((int64_t)b * R + oy0 + k) * R + ox] = (uint8_t)arg[k];
  }
}
// Candidate-pruned variant (default). Within a 7 x 7 output block that samples one source cell
// (the CTA's 7 rows share the source rows; 7-column blocks never straddle a source column
// boundary: boundaries fall at 14k + 7), every class's upsampled logit is bilinear in the
// block's interpolation weights, so its range over the block is spanned by the 4 corner pixels.
// A class whose corner maximum is below tau = max over classes of the corner minimum (less a
// rounding margin) cannot be the argmax anywhere in the block; warps build each block's list of
// the remaining classes (ascending, by ballot), then every pixel evaluates only those, with the
// exact per-pixel formula and first-index tie rule above -- identical labels. Measured on the
// seeded C2 head: ~12 of 150 classes survive per block.
constexpr int SEG_BLK = 7;         // block width (columns) = HALF_ROWS
constexpr int SEG_CMAX = 256;      // classes supported

__device__ __forceinline__ float seg_t(const float* r, int x0, int x1, int cs, int c, float w0, float w1) {
  return __fadd_rn(__fmul_rn(r[x0 * cs + c], w0), __fmul_rn(r[x1 * cs + c], w1));
}

// MAXT / MINB: the C2 shape (448 threads) is instantiated for 3 CTAs per SM (<= 48 registers;
// at the generic 1024-thread bound ptxas used 61 and only 2 fit, 3.5 waves of 296 CTAs)
template <int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT, MINB)
    seg_upsample_argmax_pruned_kernel(const float* __restrict__ logits, int h, int C, int cp, int R,
                                      uint8_t* __restrict__ labels) {
  extern __shared__ float s_src[];  // [2 rows][h cols][cs], then the candidate lists
  const int cs = (C + 1) & ~1;
  const int nblk = R / SEG_BLK;
  uint8_t* s_cand = reinterpret_cast<uint8_t*>(s_src + 2 * h * cs);  // [nblk][C]
  int* s_ncand = reinterpret_cast<int*>(s_cand + ((nblk * C + 15) & ~15));
  const int hb = blockIdx.x, b = blockIdx.y;
  const float scale = (float)h / (float)R;
  const int oy0 = hb * HALF_ROWS;
  int y0, y1;
  float hy0_unused, hy1_unused;
  src_index(scale, oy0, h, y0, y1, hy0_unused, hy1_unused);
  const float* src = logits + (int64_t)b * h * h * cp;
  const int nw = blockDim.x >> 5, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // largest |logit| of the two source rows (the pruning margin's scale), per warp, while loading
  __shared__ float s_wmag[32];
  float wmag = 0.f;
  for (int pix = wid; pix < 2 * h; pix += nw) {
    const int yy = pix < h ? y0 : y1, xx = pix < h ? pix : pix - h;
    const float* g = src + ((int64_t)yy * h + xx) * cp;
    float* d = s_src + pix * cs;
#pragma unroll 4
    for (int c = lane; c < cs; c += 32) {
      const float v = c < C ? __ldg(g + c) : 0.f;
      d[c] = v;
      wmag = fmaxf(wmag, fabsf(v));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) wmag = fmaxf(wmag, __shfl_xor_sync(0xffffffffu, wmag, o));
  if (lane == 0) s_wmag[wid] = wmag;
  __syncthreads();
  const float* r0 = s_src;
  const float* r1 = s_src + h * cs;
  // ---- candidate lists, one warp per block
  {
    int a0, a1;
    float ht0, ht1, hb0, hb1;  // vertical weights of the band's first and last row
    src_index(scale, oy0, h, a0, a1, ht0, ht1);
    src_index(scale, oy0 + HALF_ROWS - 1, h, a0, a1, hb0, hb1);
    float mag = lane < nw ? s_wmag[lane] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mag = fmaxf(mag, __shfl_xor_sync(0xffffffffu, mag, o));
    for (int blk = wid; blk < nblk; blk += nw) {
      int xa0, xa1, xb0, xb1;
      float wa0, wa1, wb0, wb1;
      src_index(scale, blk * SEG_BLK, h, xa0, xa1, wa0, wa1);
      src_index(scale, blk * SEG_BLK + SEG_BLK - 1, h, xb0, xb1, wb0, wb1);
      float lb[SEG_CMAX / 32], ub[SEG_CMAX / 32];
      float tau = -INFINITY;
#pragma unroll
      for (int j = 0; j < SEG_CMAX / 32; ++j) {
        const int c = lane + 32 * j;
        lb[j] = -INFINITY;
        ub[j] = -INFINITY;
        if (c < C) {
          const float ta0 = seg_t(r0, xa0, xa1, cs, c, wa0, wa1), ta1 = seg_t(r1, xa0, xa1, cs, c, wa0, wa1);
          const float tb0 = seg_t(r0, xb0, xb1, cs, c, wb0, wb1), tb1 = seg_t(r1, xb0, xb1, cs, c, wb0, wb1);
          const float v00 = __fadd_rn(__fmul_rn(ta0, ht0), __fmul_rn(ta1, ht1));
          const float v01 = __fadd_rn(__fmul_rn(tb0, ht0), __fmul_rn(tb1, ht1));
          const float v10 = __fadd_rn(__fmul_rn(ta0, hb0), __fmul_rn(ta1, hb1));
          const float v11 = __fadd_rn(__fmul_rn(tb0, hb0), __fmul_rn(tb1, hb1));
          lb[j] = fminf(fminf(v00, v01), fminf(v10, v11));
          ub[j] = fmaxf(fmaxf(v00, v01), fmaxf(v10, v11));
          tau = fmaxf(tau, lb[j]);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tau = fmaxf(tau, __shfl_xor_sync(0xffffffffu, tau, o));
      // every computed value (pixel or corner) is within a few roundings (2^-24 each) of the
      // exact bilinear value, relative to the largest source logit: keep a 2^-16 margin (scaled
      // by the band's largest |logit|, which bounds the block's)
      const float thr = tau - mag * 0x1p-16f;
      int n = 0;
#pragma unroll
      for (int j = 0; j < SEG_CMAX / 32; ++j) {
        const int c = lane + 32 * j;
        const bool keep = c < C && ub[j] >= thr;
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (keep) s_cand[blk * C + n + __popc(bal & ((1u << lane) - 1u))] = (uint8_t)c;
        n += __popc(bal);
      }
      if (lane == 0) s_ncand[blk] = n;
    }
  }
  __syncthreads();
  // ---- per pixel: the block's candidates in ascending class order, exact formula
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
  const int blk = ox / SEG_BLK;
  const int n = s_ncand[blk];
  const uint8_t* cl = s_cand + blk * C;
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
    const int c = cl[i];
    const float t0 = seg_t(r0, x0, x1, cs, c, wx0, wx1), t1 = seg_t(r1, x0, x1, cs, c, wx0, wx1);
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

int launch_upsample_argmax(const float* logits, int B, int h, int C, int cp, int R, uint8_t* labels,
                           cudaStream_t st) {
  const size_t smem = (size_t)2 * h * ((C + 1) & ~1) * sizeof(float);
  if (B < 1 || h < 1 || C < 1 || C > 256 || cp < C || R > 1024 || R != 14 * h || smem > 227 * 1024)
    return VPE_E_CONFIG;
  static OncePerDevice attr;
  if (attr.first()) {
    VPE_CUDA_TRY(cudaFuncSetAttribute(seg_upsample_argmax_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      227 * 1024));
    max_smem_carveout(seg_upsample_argmax_kernel);
    VPE_CUDA_TRY(cudaFuncSetAttribute(seg_upsample_argmax_pruned_kernel<448, 3>,  // + its static s_wmag
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024 - 256));
    max_smem_carveout(seg_upsample_argmax_pruned_kernel<448, 3>);
    VPE_CUDA_TRY(cudaFuncSetAttribute(seg_upsample_argmax_pruned_kernel<1024, 1>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024 - 256));
    max_smem_carveout(seg_upsample_argmax_pruned_kernel<1024, 1>);
  }
  static const bool prune = !(getenv("VPE_SEG_PRUNE") && getenv("VPE_SEG_PRUNE")[0] == '0');  // A/B
  const int nblk = R / SEG_BLK;
  const size_t smem_p = smem + (((size_t)nblk * C + 15) & ~(size_t)15) + (size_t)nblk * sizeof(int);
  if (prune && R % SEG_BLK == 0 && HALF_ROWS == SEG_BLK && smem_p <= 227 * 1024 - 256) {
    const int nt = (R + 31) / 32 * 32;
    static const bool narrow = !(getenv("VPE_SEG_NARROW") && getenv("VPE_SEG_NARROW")[0] == '0');  // A/B
    if (nt <= 448 && narrow)
      seg_upsample_argmax_pruned_kernel<448, 3><<<dim3(2 * h, B), nt, smem_p, st>>>(logits, h, C, cp, R, labels);
    else
      seg_upsample_argmax_pruned_kernel<1024, 1><<<dim3(2 * h, B), nt, smem_p, st>>>(logits, h, C, cp, R, labels);
  } else {
    seg_upsample_argmax_kernel<<<dim3(2 * h, B), (R + 31) / 32 * 32, smem, st>>>(logits, h, C, cp, R, labels, 0.f);
  }
  VPE_CUDA_TRY(cudaGetLastError());
  return VPE_OK;
}
}  // namespace

extern "C" int vpe_op_upsample_argmax(const float* logits, int32_t B, int32_t h, int32_t C, int32_t cp,
                                      int32_t resolution, uint8_t* labels, void* stream) {
  if (!logits || !labels) return VPE_E_VALUE;
  VPE_TRY(launch_upsample_argmax(logits, B, h, C, cp, resolution, labels, static_cast<cudaStream_t>(stream)));
  count_launches(1);
  return VPE_OK;
}

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
    // one N tile covering all classes when there are enough pixel tiles to fill the GPU (the
    // tap is then read once, not once per 32-class tile); narrow tiles for small batches
    static const int bn_env = getenv("VPE_SEG_BN") ? atoi(getenv("VPE_SEG_BN")) : 0;  // A/B
    const int m_tiles = (B * h * h + 127) / 128;
    const int bn = bn_env ? bn_env : ((C <= 192 && m_tiles >= 64) ? (C <= 128 ? 128 : 192) : 32);
    VPE_TRY(plan_gemm_conv(&s->g, x, B, h, h, D, D, (int64_t)h * D, (int64_t)T * D, 1, 64,
                           static_cast<const __nv_bfloat16*>(s->w.w_split), C, 2 * D, 2 * D, ep, bn));
    s->bound = final_tap;
  }
  VPE_TRY(launch_gemm(s->g, st));
  VPE_TRY(launch_upsample_argmax(s->logits, B, h, C, s->cpitch, s->cfg.resolution, labels, st));
  count_launches(2);
  if (logits_out) {
    VPE_CUDA_TRY(cudaMemcpy2DAsync(logits_out, (size_t)C * 4, s->logits, (size_t)s->cpitch * 4, (size_t)C * 4,
                                   (size_t)B * h * h, cudaMemcpyDeviceToDevice, st));
  }
  return VPE_OK;
}
