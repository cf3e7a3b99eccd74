// tcgen05 GEMM engine (see gemm.cuh). sm_100a only.
//
// Persistent, warp-specialised: grid = min(tiles, #SMs); each CTA walks tiles t = blockIdx.x,
// += gridDim.x (M-major over N so co-resident CTAs share the A tile in L2).
//   warp 0      TMA producer (A: 2D rows or 4D NHWC implicit-conv boxes; B: K-major weights)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2-9   epilogue: 2 warps per TMEM lane quadrant, split over 32-column chunks
// The accumulator is double-buffered in TMEM (2 x BN columns), so tile i's epilogue overlaps
// tile i+1's mainloop. Row-major bf16/f32 outputs leave through per-warp smem staging and TMA
// bulk tensor stores (coalesced, OOB-clipped); the fp32 residual update uses TMA reduce-add
// (cp.reduce.async.bulk .add.f32), so the SM never reads the residual stream.
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "bilerp.cuh"
#include "gemm.cuh"
#include "tc.cuh"
#include "util.cuh"

namespace vpe {

// EPI_SPLIT warps per TMEM lane quadrant share a tile's 32-column chunks round-robin; more warps
// per SMSP hide the dependent-FMA / MUFU latency of the GELU epilogue (ncu: "wait" stalls).
constexpr int EPI_SPLIT = 4;
constexpr int EPI_WARPS = 4 * EPI_SPLIT;
constexpr int GEMM_THREADS = 64 + 32 * EPI_WARPS;
// per epilogue warp: 4 KB = two 2-KB halves for bf16 tiles (32x32) or one 4-KB fp32 tile
constexpr int STAGE_BUF = 32 * 32 * 4;

template <int BN, int BK>
struct GemmCfg {
  static constexpr int A_BYTES = 128 * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int PIPE_BUDGET = 150 * 1024;
  static constexpr int STAGES_RAW = PIPE_BUDGET / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : (STAGES_RAW < 2 ? 2 : STAGES_RAW);
  static constexpr int TMEM_COLS = (2 * BN) <= 32 ? 32 : ((2 * BN) <= 64 ? 64 : ((2 * BN) <= 128 ? 128 : ((2 * BN) <= 256 ? 256 : 512)));
  static constexpr int SWZ_LAYOUT = BK == 64 ? 2 : 4;  // UMMA SWIZZLE_128B / SWIZZLE_64B
  static constexpr int SBO = 8 * BK * 2;               // bytes between 8-row core groups
  static constexpr size_t SMEM = 1024 + (size_t)STAGES * STAGE_BYTES + EPI_WARPS * STAGE_BUF + 256;
};

VPE_DEV void store_bf16x32(__nv_bfloat16* dst, const float (&v)[32]) {
  uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint4 u;
    u.x = pack_bf16(v[8 * i + 0], v[8 * i + 1]);
    u.y = pack_bf16(v[8 * i + 2], v[8 * i + 3]);
    u.z = pack_bf16(v[8 * i + 4], v[8 * i + 5]);
    u.w = pack_bf16(v[8 * i + 6], v[8 * i + 7]);
    d[i] = u;
  }
}
VPE_DEV void load_bf16x32_add(const __nv_bfloat16* src, float (&v)[32]) {
  const uint4* s = reinterpret_cast<const uint4*>(src);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint4 u = s[i];
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float2 f = __bfloat1622float2(h[j]);
      v[8 * i + 2 * j] += f.x;
      v[8 * i + 2 * j + 1] += f.y;
    }
  }
}

// Activation over a whole chunk behind one (warp-uniform) branch per kind: a per-element
// apply_act() let the compiler if-convert the erf-GELU into every element's path (measured: the
// predicated-off MUFU/FFMA sequence ran for ReLU / identity epilogues too).
// (GELU here is an out-of-line call: no engine conv uses it, and inlined it costs every
// ReLU / identity epilogue registers.)
__device__ __noinline__ float gelu_erf_call(float x) { return gelu_erf(x); }
template <int NV>
VPE_DEV void apply_act_n(float* v, int act) {
  if (act == ACT_RELU) {
#pragma unroll
    for (int j = 0; j < NV; ++j) v[j] = fmaxf(v[j], 0.f);
  } else if (act == ACT_GELU) {
#pragma unroll
    for (int j = 0; j < NV; ++j) v[j] = gelu_erf_call(v[j]);
  }
}

VPE_DEV float apply_act(float x, int act) {
  if (act == ACT_GELU) return gelu_erf(x);  // scalar path; the TMA-store epilogue uses gelu_poly32
  if (act == ACT_RELU) return fmaxf(x, 0.f);
  return x;
}

// v[j] += vec[col0 + j] for the valid columns (vectorised when the chunk is full)
VPE_DEV void add_vec32(float (&v)[32], const float* __restrict__ vec, int col0, int N, bool full) {
  if (full) {
    const float4* b4 = reinterpret_cast<const float4*>(vec + col0);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float4 b = __ldg(b4 + i);
      v[4 * i] += b.x;
      v[4 * i + 1] += b.y;
      v[4 * i + 2] += b.z;
      v[4 * i + 3] += b.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (col0 + j < N) v[j] += __ldg(vec + col0 + j);
  }
}
VPE_DEV void mul_vec32(float (&v)[32], const float* __restrict__ vec, int col0, int N, bool full) {
  if (full) {
    const float4* b4 = reinterpret_cast<const float4*>(vec + col0);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float4 b = __ldg(b4 + i);
      v[4 * i] *= b.x;
      v[4 * i + 1] *= b.y;
      v[4 * i + 2] *= b.z;
      v[4 * i + 3] *= b.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] *= (col0 + j < N) ? __ldg(vec + col0 + j) : 0.f;
  }
}

// DPT head conv3 (1x1, 32 -> 1) on relu(conv2): b3 + sum_c relu(v_c) w3_c, as four interleaved
// partial sums (a 32-long dependent FMA chain was the epilogue's latency). w3 may be global or smem.
VPE_DEV float depth_dot(const float (&v)[32], const float* w3, float b3) {
  float a[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int j = 0; j < 32; ++j) a[j & 3] = __fmaf_rn(fmaxf(v[j], 0.f), w3[j], a[j & 3]);
  return b3 + ((a[0] + a[1]) + (a[2] + a[3]));
}

// Direct (non-TMA) epilogue for one thread: one output row (gpix), 32 consecutive columns.
VPE_DEV void epilogue_direct(const EpiParams& ep, int64_t gpix, int col0, float (&v)[32]) {
  const int N = ep.N;
  const bool full = (col0 + 32 <= N);
  if (ep.bias) add_vec32(v, ep.bias, col0, N, full);
  switch (ep.kind) {
    case EPI_BF16:
    case EPI_CONV: {
      __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(ep.out) + gpix * ep.ldo + col0;
      if (ep.kind == EPI_CONV) {
        if (full) {
          if (ep.add1) load_bf16x32_add(ep.add1 + gpix * ep.ldo + col0, v);
          if (ep.add2) load_bf16x32_add(ep.add2 + gpix * ep.ldo + col0, v);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            if (col0 + j < N) {
              if (ep.add1) v[j] += __bfloat162float(ep.add1[gpix * ep.ldo + col0 + j]);
              if (ep.add2) v[j] += __bfloat162float(ep.add2[gpix * ep.ldo + col0 + j]);
            }
          }
        }
      }
#pragma unroll
      apply_act_n<32>(v, ep.act);
      if (full) {
        store_bf16x32(out, v);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (col0 + j < N) out[j] = __float2bfloat16_rn(v[j]);
      }
      if (ep.out_relu) {
        __nv_bfloat16* o2 = ep.out_relu + gpix * ep.ldo + col0;
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j], 0.f);
        if (full) {
          store_bf16x32(o2, v);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (col0 + j < N) o2[j] = __float2bfloat16_rn(v[j]);
        }
      }
      break;
    }
    case EPI_RESID: {
      float* r = ep.resid + gpix * ep.ldr + col0;
      mul_vec32(v, ep.scale, col0, N, full);
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (col0 + j < N) r[j] += v[j];
      break;
    }
    case EPI_PATCH: {
      const int img = (int)gpix / ep.rows_per_img;  // 32-bit: rows < 2^31
      const int64_t p = gpix - (int64_t)img * ep.rows_per_img;
      float* r = ep.resid + (gpix + img + 1) * ep.ldr + col0;
      add_vec32(v, ep.pos + (p + 1) * (int64_t)N, col0, N, full);
      if (full) {
        float4* r4 = reinterpret_cast<float4*>(r);
#pragma unroll
        for (int i = 0; i < 8; ++i) r4[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (col0 + j < N) r[j] = v[j];
      }
      break;
    }
    case EPI_F32: {
      float* o = reinterpret_cast<float*>(ep.out) + gpix * ep.ldo + col0;
      apply_act_n<32>(v, ep.act);
      if (full) {
        float4* o4 = reinterpret_cast<float4*>(o);
#pragma unroll
        for (int i = 0; i < 8; ++i) o4[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (col0 + j < N) o[j] = v[j];
      }
      break;
    }
    case EPI_CONVT: {
      // gpix indexes the input grid (img, y, x); each group of ct_cout columns is one sub-pixel.
      const int HW = ep.ct_H * ep.ct_W;
      const int img = (int)gpix / HW;  // 32-bit: pixels < 2^31
      const int rem = (int)gpix - img * HW;
      const int y = rem / ep.ct_W, x = rem - (rem / ep.ct_W) * ep.ct_W;
      // ct_cout is a multiple of 32, so a 32-column chunk is 32 contiguous channels of one
      // output sub-pixel: one 64-byte vector store
      const int k = ep.ct_k, Wo = ep.ct_W * k, Ho = ep.ct_H * k;
      const int s = col0 / ep.ct_cout, co0 = col0 - s * ep.ct_cout;
      const int ky = s / k, kx = s - ky * k;
      const int64_t op = (img * Ho + (int64_t)(y * k + ky)) * Wo + (x * k + kx);
      __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(ep.out) + op * ep.ldo + co0;
      if (full) {
        store_bf16x32(dst, v);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (col0 + j < N) dst[j] = __float2bfloat16_rn(v[j]);
      }
      break;
    }
    case EPI_DEPTH: {
      const float pre = depth_dot(v, ep.w3, ep.b3);
      ep.depth_pre[gpix] = pre;
      ep.depth[gpix] = fmaxf(pre, 0.f) * ep.max_depth;
      break;
    }
    default:
      break;
  }
}

// EPI_CONV through a per-warp smem stage (halo conv): the warp's 32 lanes are 32 pixels of 32
// channels at pitch ldo. Written per thread, each 16-byte store of the warp lands in a different
// pixel (half sectors) -- measured ~1.5x slower for the whole conv than contiguous runs. So the
// add operands are loaded and the results stored cooperatively, in passes of 8U channels:
// piece q = 32 j + lane is 16-byte unit (q % U) of pixel q / U, i.e. each instruction moves
// 32/U pixels x 16U contiguous bytes (U = 4: the warp's whole 2 KB when ldo = 32). Stage row of
// pixel p: 16U bytes, units XOR-swizzled (conflict-free per pixel and per piece).
template <int U>
VPE_DEV uint32_t conv_stg_off(int px, int unit) {
  constexpr int SH = U == 4 ? 1 : 2;
  return (uint32_t)(px * 16 * U + ((unit ^ ((px >> SH) & (U - 1))) << 4));
}

template <int U>
VPE_DEV void epilogue_conv_staged(const EpiParams& ep, int64_t gpix, bool valid, int col0, float (&v)[32],
                                  uint8_t* stg) {
  constexpr int PASSES = 4 / U, CH = 8 * U, PPI = 32 / U;  // channel passes, channels/pass, pixels/instr
  const uint32_t lane = lane_id();
  if (ep.bias) add_vec32(v, ep.bias, col0, ep.N, true);
  int64_t pg[U];  // pixel of each piece this lane moves, and whether it exists
  bool pv[U];
#pragma unroll
  for (int j = 0; j < U; ++j) {
    const int src = PPI * j + lane / U;
    pg[j] = __shfl_sync(0xffffffffu, gpix, src);
    pv[j] = __shfl_sync(0xffffffffu, valid ? 1 : 0, src) != 0;
  }
  const __nv_bfloat16* adds[2] = {ep.add1, ep.add2};
  __nv_bfloat16* outs[2] = {reinterpret_cast<__nv_bfloat16*>(ep.out), ep.out_relu};
#pragma unroll
  for (int h = 0; h < PASSES; ++h) {
    const int c = col0 + CH * h;
    float* vh = v + CH * h;
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      if (!adds[a]) continue;  // warp-uniform
#pragma unroll
      for (int j = 0; j < U; ++j) {
        uint4 u = make_uint4(0, 0, 0, 0);
        if (pv[j]) u = __ldg(reinterpret_cast<const uint4*>(adds[a] + pg[j] * ep.ldo + c) + (lane % U));
        *reinterpret_cast<uint4*>(stg + conv_stg_off<U>(PPI * j + lane / U, lane % U)) = u;
      }
      __syncwarp();
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint4 w = *reinterpret_cast<const uint4*>(stg + conv_stg_off<U>(lane, u));
        const __nv_bfloat162* hh = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const float2 f = __bfloat1622float2(hh[t]);
          vh[8 * u + 2 * t] += f.x;
          vh[8 * u + 2 * t + 1] += f.y;
        }
      }
      __syncwarp();
    }
    apply_act_n<CH>(vh, ep.act);
#pragma unroll
    for (int o = 0; o < 2; ++o) {
      if (!outs[o]) continue;  // warp-uniform
#pragma unroll
      for (int u = 0; u < U; ++u) {
        float f[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) f[t] = o ? fmaxf(vh[8 * u + t], 0.f) : vh[8 * u + t];
        uint4 w;
        w.x = pack_bf16(f[0], f[1]);
        w.y = pack_bf16(f[2], f[3]);
        w.z = pack_bf16(f[4], f[5]);
        w.w = pack_bf16(f[6], f[7]);
        *reinterpret_cast<uint4*>(stg + conv_stg_off<U>(lane, u)) = w;
      }
      __syncwarp();
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const uint4 w = *reinterpret_cast<const uint4*>(stg + conv_stg_off<U>(PPI * j + lane / U, lane % U));
        if (pv[j]) *(reinterpret_cast<uint4*>(outs[o] + pg[j] * ep.ldo + c) + (lane % U)) = w;
      }
      __syncwarp();
    }
  }
}

// optional MMA-thread timeline of CTA 0: a diagnostics build only (nvcc -DVPE_TRACE_BUILD, then
// VPE_GEMM_TRACE=1 and vpe_debug_gemm_trace); the product build compiles the probes out
__device__ unsigned long long g_gemm_trace[4096];
static int g_gemm_trace_on = -1;
#ifdef VPE_TRACE_BUILD
#define GEMM_TRACE(idx, code)                                                        \
  do {                                                                               \
    if (p.trace && blockIdx.x == 0 && (idx) < 2040) {                                \
      g_gemm_trace[2 * (idx)] = (unsigned long long)(code);                          \
      g_gemm_trace[2 * (idx) + 1] = (unsigned long long)clock64();                   \
      ++(idx);                                                                       \
    }                                                                                \
  } while (0)
#else
#define GEMM_TRACE(idx, code) \
  do {                        \
  } while (0)
#endif

// per-role variant: slots [base, base + 600) of CTA 0's timeline (halo conv: MMA 0, TMA 680,
// epilogue warp 2 at 1360)
#ifdef VPE_TRACE_BUILD
#define ROLE_TRACE(base, idx, code)                                                  \
  do {                                                                               \
    if (p.trace && blockIdx.x == 0 && (idx) < 600) {                                 \
      g_gemm_trace[2 * ((base) + (idx))] = (unsigned long long)(code);               \
      g_gemm_trace[2 * ((base) + (idx)) + 1] = (unsigned long long)clock64();        \
      ++(idx);                                                                       \
    }                                                                                \
  } while (0)
#else
#define ROLE_TRACE(base, idx, code) \
  do {                              \
  } while (0)
#endif

// One 32-column chunk of a row-major tile through the TMA-store epilogue: bias / LayerScale /
// activation in registers, swizzled smem staging (per-warp double buffer), then a TMA bulk store
// (bf16 / f32) or bulk reduce-add (fp32 residual). Lane 0 issues; row0 = first of the warp's 32 rows.
VPE_DEV void epilogue_tma_chunk(const GemmParams& p, const CUtensorMap* tout, float (&v)[32], int col0, int row0,
                                uint8_t* stg_base, int& nstore) {
  const uint32_t lane = lane_id();
  const int N = p.ep.N;
  const bool fullc = col0 + 32 <= N;
  if (p.ep.bias) add_vec32(v, p.ep.bias, col0, N, fullc);
  if (p.ep.kind == EPI_RESID) mul_vec32(v, p.ep.scale, col0, N, fullc);
  if (p.ep.act == ACT_GELU) {
    gelu_poly32(v);
  } else if (p.ep.act != ACT_NONE) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = apply_act(v[j], p.ep.act);
  }
  const bool bf = p.ep.kind == EPI_BF16;
  uint8_t* stg = stg_base + (bf ? (nstore & 1) * (STAGE_BUF / 2) : 0);
  if (lane == 0) {  // the store that last used this buffer has finished reading it
    if (bf)
      bulk_wait_read1();
    else
      bulk_wait_read0();
  }
  __syncwarp();
  // staging rows are written in the TMA swizzle layout (bank-conflict free):
  // bf16: 64-B rows, SWIZZLE_64B (chunk ^ ((row>>1)&3)); f32: 128-B rows, SWIZZLE_128B
  if (p.ep.kind == EPI_BF16) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint4 u;
      u.x = pack_bf16(v[8 * k + 0], v[8 * k + 1]);
      u.y = pack_bf16(v[8 * k + 2], v[8 * k + 3]);
      u.z = pack_bf16(v[8 * k + 4], v[8 * k + 5]);
      u.w = pack_bf16(v[8 * k + 6], v[8 * k + 7]);
      *reinterpret_cast<uint4*>(stg + lane * 64 + ((k ^ ((lane >> 1) & 3)) << 4)) = u;
    }
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      *reinterpret_cast<float4*>(stg + lane * 128 + ((k ^ (lane & 7)) << 4)) =
          make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
  }
  fence_async_smem();
  __syncwarp();
  if (lane == 0) {
    if (p.ep.kind == EPI_RESID)
      tma_reduce_add_2d(tout, stg, col0, row0);
    else
      tma_store_2d(tout, stg, col0, row0);
    bulk_commit();
  }
  ++nstore;
}

template <int BN, int BK>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                   const __grid_constant__ CUtensorMap tout, const GemmParams p) {
  using C = GemmCfg<BN, BK>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint8_t* sStage = sB + C::STAGES * C::B_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sStage + EPI_WARPS * STAGE_BUF);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;  // [2]
  uint64_t* tempty = tfull + 2;         // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = warp_id(), lane = lane_id();
  if (warp == 0 && lane == 0) {
    tma_prefetch(&ta);
    tma_prefetch(&tb);
    if (p.tma_out) tma_prefetch(&tout);
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], EPI_WARPS);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tslot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  pdl_wait();
  if (!p.pdl_late) pdl_trigger();
  const int ntiles = p.m_tiles * p.n_tiles;

  if (warp == 0) {
    if (lane == 0) {
      const int half = p.ks / 2;
      int it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int mt = t / p.n_tiles, nt = t - mt * p.n_tiles;
        const int n0 = nt * BN;
        int m0 = 0, img = 0, y0 = 0, x0 = 0;
        if (p.mode == 0) {
          m0 = mt * 128;
        } else {
          img = mt / p.tiles_per_img;
          const int r = mt - img * p.tiles_per_img;
          y0 = (r / p.tiles_x) * p.bh;
          x0 = (r % p.tiles_x) * p.bw;
        }
        for (int kb = 0; kb < p.kblocks; ++kb, ++it) {
          const int s = it % C::STAGES;
          const uint32_t ph = (it / C::STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          mbar_expect_tx(&full[s], C::STAGE_BYTES);
          const int ka = kb % p.kblocks_a;
          if (p.mode == 0) {
            tma_load_2d(sA + s * C::A_BYTES, &ta, &full[s], ka * BK, m0);
          } else {
            const int tap = ka / p.cchunks, cc = ka - tap * p.cchunks;
            const int dy = tap / p.ks - half, dx = tap % p.ks - half;
            tma_load_4d(sA + s * C::A_BYTES, &ta, &full[s], cc * BK, x0 + dx, y0 + dy, img);
          }
          tma_load_2d(sB + s * C::B_BYTES, &tb, &full[s], kb * BK, n0);
        }
      }
      if (p.pdl_late) pdl_trigger();  // every load issued: the dependent grid may come in
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(128, BN);
      // descriptor words of stage 0; a stage / K-step is a constant added to the address field
      // (16-byte units): the single issuing thread is latency-bound, so keep its chain short
      const uint64_t a_desc0 = smem_desc(smem_u32(sA), 16, C::SBO, C::SWZ_LAYOUT);
      const uint64_t b_desc0 = smem_desc(smem_u32(sB), 16, C::SBO, C::SWZ_LAYOUT);
      const uint32_t a_hi = (uint32_t)(a_desc0 >> 32), b_hi = (uint32_t)(b_desc0 >> 32);
      int s = 0, i = 0, tn = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
        const int acc = i & 1;
        GEMM_TRACE(tn, 1);
        mbar_wait(&tempty[acc], ((i >> 1) & 1) ^ 1);
        tc_fence_after();
        GEMM_TRACE(tn, 2);
        const uint32_t d = tmem + acc * BN;
        for (int kb = 0; kb < p.kblocks; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t a_lo = (uint32_t)a_desc0 + (uint32_t)s * (C::A_BYTES >> 4);
          const uint32_t b_lo = (uint32_t)b_desc0 + (uint32_t)s * (C::B_BYTES >> 4);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = ((uint64_t)a_hi << 32) | (a_lo + 2 * k);
            const uint64_t bd = ((uint64_t)b_hi << 32) | (b_lo + 2 * k);
            umma_f16(d, ad, bd, idesc, (kb | k) != 0);
          }
          umma_commit(&empty[s]);
          if (++s == C::STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else {
    // epilogue warps: TMEM lane quadrant = warp % 4, column slice = (warp - 2) / 4
    const int e = warp - 2;
    const int q = warp & 3;
    const int chalf = e >> 2;
    const int r = q * 32 + lane;
    uint8_t* stg_base = sStage + e * STAGE_BUF;
    int nstore = 0;  // staging double buffer: store n uses half n & 1
    int i = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
      const int acc = i & 1;
      const int mt = t / p.n_tiles, nt = t - mt * p.n_tiles;
      const int n0 = nt * BN;
      int64_t gpix;
      bool valid;
      int m0 = 0;
      if (p.mode == 0) {
        m0 = mt * 128;
        gpix = m0 + r;
        valid = gpix < p.M;
      } else {
        const int img = mt / p.tiles_per_img;
        const int rr = mt - img * p.tiles_per_img;
        const int y = (rr / p.tiles_x) * p.bh + r / p.bw, x = (rr % p.tiles_x) * p.bw + r % p.bw;
        valid = (y < p.H) && (x < p.W);
        gpix = ((int64_t)img * p.H + y) * p.W + x;
      }
      mbar_wait(&tfull[acc], (i >> 1) & 1);
      tc_fence_after();
      if (chalf >= BN / 32) {  // narrow tile: this column slice has no chunk, release at once
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
      }
#pragma unroll 1
      for (int c = chalf; c < BN / 32; c += EPI_SPLIT) {
        const int c0 = c * 32;
        float v[32];
        tmem_ld32(tmem + acc * BN + ((uint32_t)(q * 32) << 16) + c0, v);
        tmem_ld_wait();
        if (c + EPI_SPLIT >= BN / 32) {  // this warp's last TMEM read of the tile: release it now
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);  // one arrival per warp (512 per-thread
                                                      // arrivals serialise on the barrier)
        }
        const int col0 = n0 + c0;
        if (col0 >= p.ep.N) continue;  // warp-uniform
        if (p.tma_out) {
          epilogue_tma_chunk(p, &tout, v, col0, m0 + q * 32, stg_base, nstore);
        } else if (valid) {
          epilogue_direct(p.ep, gpix, col0, v);
        }
      }
    }
    if (lane == 0) bulk_wait0();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// ------------------------------------------------------------------------------------------
// Residual GEMM with the next LayerNorm in its epilogue (backbone proj / FC2 at D = 384):
//   resid += LayerScale * (A W^T + bias);  xln = LN(resid) (bf16, the next GEMM's A);
//   optionally tap = LN'(resid) with a second affine (the ring's tap / final norm).
// A CTA owns whole 384-wide rows (one 128 x 384 accumulator: an N=256 and an N=128 MMA per K
// step), so the row statistics never leave the CTA. Epilogue: 8 warps, two per TMEM lane
// quadrant (192 columns each). The drained pipeline stages become the epilogue's staging: the old
// residual arrives by TMA, the new one leaves by TMA, row sums are exchanged between the two
// warps of a quadrant through smem + a named barrier. Replaces TMA reduce-add epilogue + the
// standalone LayerNorm kernel; the new residual is bit-identical (same single fp32 add), the LN
// differs from layernorm_kernel only in summation order.
// ------------------------------------------------------------------------------------------
constexpr int RL_N = 384, RL_ST = 3;
constexpr int RL_SPLIT = 4;                          // epilogue warps per TMEM lane quadrant
constexpr int RL_EW = 4 * RL_SPLIT;                  // epilogue warps
constexpr int RL_CH = RL_N / 32 / RL_SPLIT;          // 32-column chunks per epilogue warp
constexpr int RL_THREADS = 32 * (2 + RL_EW);         // warps: 0 TMA, 1 MMA, then the epilogue
struct RlCfg {
  static constexpr int A_BYTES = 128 * 64 * 2;
  static constexpr int B_BYTES = RL_N * 64 * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;  // 64 KB; the 3 stages double as epilogue staging
  static constexpr size_t SMEM = 1024 + (size_t)RL_ST * STAGE + 2 * RL_SPLIT * 128 * 4 + 256;
};

__global__ void __launch_bounds__(RL_THREADS, 1)
    gemm_resid_ln_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                         const __grid_constant__ CUtensorMap tres, const __grid_constant__ CUtensorMap txln,
                         const __grid_constant__ CUtensorMap ttap, const GemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* xs = reinterpret_cast<float*>(smem + RL_ST * RlCfg::STAGE);  // [2 uses][RL_SPLIT parts][128 rows]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + RL_ST * RlCfg::STAGE + 2 * RL_SPLIT * 128 * 4);
  uint64_t* empty = full + RL_ST;
  uint64_t* tfull = empty + RL_ST;
  uint64_t* tempty = tfull + 1;
  uint64_t* epi_done = tempty + 1;
  uint64_t* ebar = epi_done + 1;  // [RL_EW] per epilogue warp: old-residual TMA loads
  uint32_t* tslot = reinterpret_cast<uint32_t*>(ebar + RL_EW);
  const uint32_t warp = warp_id(), lane = lane_id();
  if (warp == 0 && lane == 0) {
    tma_prefetch(&ta);
    tma_prefetch(&tb);
    tma_prefetch(&tres);
    tma_prefetch(&txln);
    for (int i = 0; i < RL_ST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, RL_EW);
    mbar_init(epi_done, RL_EW);
    for (int i = 0; i < RL_EW; ++i) mbar_init(&ebar[i], 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  pdl_wait();
  if (!p.pdl_late) pdl_trigger();
  const int m_tiles = p.m_tiles, kblocks = p.kblocks;

  if (warp == 0) {
    if (lane == 0) {
      int s = 0, i = 0;
      uint32_t ph = 0;
      for (int mt = blockIdx.x; mt < m_tiles; mt += gridDim.x, ++i) {
        // the stages double as the previous tile's epilogue staging
        if (i > 0) mbar_wait(epi_done, (i - 1) & 1);
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          mbar_expect_tx(&full[s], RlCfg::STAGE);
          uint8_t* st = smem + s * RlCfg::STAGE;
          tma_load_2d(st, &ta, &full[s], kb * 64, mt * 128);
          for (int nb = 0; nb < 3; ++nb)
            tma_load_2d(st + RlCfg::A_BYTES + nb * 16384, &tb, &full[s], kb * 64, nb * 128);
          if (++s == RL_ST) {
            s = 0;
            ph ^= 1;
          }
        }
      }
      if (p.pdl_late) pdl_trigger();
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id256 = idesc_bf16(128, 256), id128 = idesc_bf16(128, 128);
      const uint64_t d0 = smem_desc(smem_u32(smem), 16, 1024, 2);
      const uint32_t lo0 = (uint32_t)d0, hi = (uint32_t)(d0 >> 32);
      int s = 0, i = 0;
      uint32_t ph = 0;
      for (int mt = blockIdx.x; mt < m_tiles; mt += gridDim.x, ++i) {
        mbar_wait(tempty, (i & 1) ^ 1);
        tc_fence_after();
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t a_lo = lo0 + (uint32_t)s * (RlCfg::STAGE >> 4);
          const uint32_t b_lo = a_lo + (RlCfg::A_BYTES >> 4);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t ad = ((uint64_t)hi << 32) | (a_lo + 2 * k);
            umma_f16(tmem, ad, ((uint64_t)hi << 32) | (b_lo + 2 * k), id256, (kb | k) != 0);
            umma_f16(tmem + 256, ad, ((uint64_t)hi << 32) | (b_lo + (32768 >> 4) + 2 * k), id128, (kb | k) != 0);
          }
          umma_commit(&empty[s]);
          if (++s == RL_ST) {
            s = 0;
            ph ^= 1;
          }
        }
        umma_commit(tfull);
      }
    }
  } else {
    const int e = warp - 2, q = warp & 3, h = e >> 2;  // h: this warp's column part of the row
    const int r = q * 32 + lane;                        // row of the tile
    uint8_t* stg = smem + e * (RL_CH * 4096);           // RL_CH chunks of 32 x 32 fp32
    const int bar_id = 1 + q;                           // the quadrant's RL_SPLIT warps
    auto pair_sync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(32 * RL_SPLIT) : "memory"); };
    int i = 0;
    for (int mt = blockIdx.x; mt < m_tiles; mt += gridDim.x, ++i) {
      const int row0 = mt * 128 + q * 32;
      mbar_wait(tfull, i & 1);  // mainloop done: every stage is free for staging
      tc_fence_after();
      if (lane == 0) {
        mbar_expect_tx(&ebar[e], RL_CH * 4096);
        for (int c = 0; c < RL_CH; ++c) tma_load_2d(stg + c * 4096, &tres, &ebar[e], (h * RL_CH + c) * 32, row0);
      }
      mbar_wait(&ebar[e], i & 1);
      float sum = 0.f;
#pragma unroll 1
      for (int c = 0; c < RL_CH; ++c) {
        const int col0 = (h * RL_CH + c) * 32;
        float v[32];
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + col0, v);
        tmem_ld_wait();
        add_vec32(v, p.ep.bias, col0, RL_N, true);
        mul_vec32(v, p.ep.scale, col0, RL_N, true);
        uint8_t* cb = stg + c * 4096 + lane * 128;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          float4* sp = reinterpret_cast<float4*>(cb + ((k ^ (lane & 7)) << 4));
          float4 o = *sp;
          o.x = __fadd_rn(o.x, v[4 * k]);
          o.y = __fadd_rn(o.y, v[4 * k + 1]);
          o.z = __fadd_rn(o.z, v[4 * k + 2]);
          o.w = __fadd_rn(o.w, v[4 * k + 3]);
          *sp = o;
          sum = __fadd_rn(sum, __fadd_rn(__fadd_rn(o.x, o.y), __fadd_rn(o.z, o.w)));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty);  // accumulator read out
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        for (int c = 0; c < RL_CH; ++c) tma_store_2d(&tres, stg + c * 4096, (h * RL_CH + c) * 32, row0);
        bulk_commit();
      }
      // row statistics: the RL_SPLIT column parts of the row meet in smem (fixed order)
      xs[h * 128 + r] = sum;
      pair_sync();
      float tot = xs[r];
#pragma unroll
      for (int j = 1; j < RL_SPLIT; ++j) tot = __fadd_rn(tot, xs[j * 128 + r]);
      const float mean = __fdiv_rn(tot, (float)RL_N);
      float sq = 0.f;
#pragma unroll 1
      for (int c = 0; c < RL_CH; ++c) {
        const uint8_t* cb = stg + c * 4096 + lane * 128;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float4 o = *reinterpret_cast<const float4*>(cb + ((k ^ (lane & 7)) << 4));
          const float a = __fsub_rn(o.x, mean), b = __fsub_rn(o.y, mean);
          const float cc = __fsub_rn(o.z, mean), d = __fsub_rn(o.w, mean);
          sq = __fadd_rn(sq, __fadd_rn(__fmaf_rn(a, a, __fmul_rn(b, b)), __fmaf_rn(cc, cc, __fmul_rn(d, d))));
        }
      }
      xs[RL_SPLIT * 128 + h * 128 + r] = sq;
      pair_sync();
      float tq = xs[RL_SPLIT * 128 + r];
#pragma unroll
      for (int j = 1; j < RL_SPLIT; ++j) tq = __fadd_rn(tq, xs[RL_SPLIT * 128 + j * 128 + r]);
      const float rstd = rsqrtf(__fadd_rn(__fdiv_rn(tq, (float)RL_N), p.ln.eps));
      if (lane == 0) bulk_wait_read0();  // the new-residual stores have read the staging
      __syncwarp();
      const bool tap = p.ln.tap != nullptr;
#pragma unroll 1
      for (int c = 0; c < RL_CH; ++c) {
        const int col0 = (h * RL_CH + c) * 32;
        uint8_t* cb = stg + c * 4096;
        float x[32];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float4 o = *reinterpret_cast<const float4*>(cb + lane * 128 + ((k ^ (lane & 7)) << 4));
          x[4 * k] = o.x;
          x[4 * k + 1] = o.y;
          x[4 * k + 2] = o.z;
          x[4 * k + 3] = o.w;
        }
        __syncwarp();  // the bf16 rows below overwrite fp32 rows other lanes read above
        for (int o = 0; o < 2; ++o) {
          const float* w = o ? p.ln.tw : p.ln.w;
          const float* b = o ? p.ln.tb : p.ln.b;
          if (!w) continue;  // uniform: no second affine
          uint8_t* ob = cb + o * 2048 + lane * 64;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float4 w0 = __ldg(reinterpret_cast<const float4*>(w + col0 + 8 * k));
            const float4 w1 = __ldg(reinterpret_cast<const float4*>(w + col0 + 8 * k + 4));
            const float4 b0 = __ldg(reinterpret_cast<const float4*>(b + col0 + 8 * k));
            const float4 b1 = __ldg(reinterpret_cast<const float4*>(b + col0 + 8 * k + 4));
            const float* xx = x + 8 * k;
            uint4 u;
            u.x = pack_bf16(__fmaf_rn(__fmul_rn(__fsub_rn(xx[0], mean), rstd), w0.x, b0.x),
                            __fmaf_rn(__fmul_rn(__fsub_rn(xx[1], mean), rstd), w0.y, b0.y));
            u.y = pack_bf16(__fmaf_rn(__fmul_rn(__fsub_rn(xx[2], mean), rstd), w0.z, b0.z),
                            __fmaf_rn(__fmul_rn(__fsub_rn(xx[3], mean), rstd), w0.w, b0.w));
            u.z = pack_bf16(__fmaf_rn(__fmul_rn(__fsub_rn(xx[4], mean), rstd), w1.x, b1.x),
                            __fmaf_rn(__fmul_rn(__fsub_rn(xx[5], mean), rstd), w1.y, b1.y));
            u.w = pack_bf16(__fmaf_rn(__fmul_rn(__fsub_rn(xx[6], mean), rstd), w1.z, b1.z),
                            __fmaf_rn(__fmul_rn(__fsub_rn(xx[7], mean), rstd), w1.w, b1.w));
            *reinterpret_cast<uint4*>(ob + ((k ^ ((lane >> 1) & 3)) << 4)) = u;
          }
        }
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        for (int c = 0; c < RL_CH; ++c) {
          if (p.ln.w) tma_store_2d(&txln, stg + c * 4096, (h * RL_CH + c) * 32, row0);
          if (tap) tma_store_2d(&ttap, stg + c * 4096 + 2048, (h * RL_CH + c) * 32, row0);
        }
        bulk_commit();
        bulk_wait_read0();  // staging free for the next tile's loads
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(epi_done);
    }
    if (lane == 0) bulk_wait0();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ------------------------------------------------------------------------------------------
// 3x3 convolution with a shared halo tile (mode 2).
//
// The 4D-box implicit GEMM above re-reads the input once per tap (9x the L2->SMEM traffic).
// Here one TMA (5D map {8ch, x, y, chunk, img}) brings the (rows+2) x P halo of a 128-pixel
// output tile for a whole channel group into SMEM in the UMMA no-swizzle K-major layout
// ("core matrix" = 8 pixels x 16 B, pixels 16 B apart, 8-channel chunks LBO apart). Every tap
// is then just a different descriptor start address: + (dy*P + dx) * 16 B. Output pixels are
// "virtual" positions v = ry*P + rx of the padded row pitch P; the 2 halo columns per row are
// computed and discarded by the epilogue.
// ------------------------------------------------------------------------------------------
// RT = output rows of 128 pixels per tile (W >= 128 only): RT accumulators of 128 x BN share one
// (RT+2)-row halo, so the A traffic per output row drops from 3 to (RT+2)/RT halo rows.
// WRES: every weight tile of the conv (parts x 9 taps x channel groups, <= 72 KB) is loaded
// into shared memory once per CTA and stays resident for all of the CTA's tiles, so only the A
// halo streams and the MMA issuer waits once per tile instead of once per tap (the DPT 3x3
// convs: 64->64 RCUs 72 KB, head convs 36 / 18 KB).
constexpr int WRES_BYTES = 72 * 1024;

template <int BN, int KC, int RT, bool WRES = false>
struct HaloCfg {
  static constexpr int GCH = 8 * KC;                 // channels per group
  // The halo is one swizzled row of 16*KC bytes per pixel: SWIZZLE_128B for 64-channel groups,
  // SWIZZLE_64B for 32 (TMA moves whole rows; the 16-byte rows of a no-swizzle K-major layout
  // capped TMA at ~11 B/clk/SM, below the MMA rate). Shifted taps are plain start offsets.
  static constexpr bool SW = true;
  static constexpr int RB = 16 * KC;                 // bytes per halo pixel
  static constexpr uint32_t A_LAYOUT = KC == 8 ? 2 : 4;  // UMMA SWIZZLE_128B / SWIZZLE_64B
  static constexpr int A_MAX = (KC * 130 * (RT + 2) * 16 + 1023) / 1024 * 1024;  // largest stage (P=130)
  static constexpr int A_STAGES = 2;
  static constexpr int B_BYTES = BN * GCH * 2;       // one tap's weight tile
  static constexpr int B_STAGES = BN >= 128 ? 4 : 8;
  static constexpr int B_REGION = WRES ? WRES_BYTES : B_STAGES * B_BYTES;
  static constexpr int TMEM_COLS = GemmCfg<BN * RT, 64>::TMEM_COLS;
  static constexpr int B_SWZ = GCH == 64 ? 2 : 4;
  static constexpr int B_SBO = 8 * GCH * 2;
  // EPI_CONV smem stage: 16 KB, as 2 KB for each of 8 warps when a tile has <= 2 chunks per lane
  // quadrant (whole-chunk passes, U = 4), else 1 KB for each of the 16 warps (half chunks, U = 2)
  static constexpr int NCHUNK = RT * (BN / 32);
  static constexpr int STG_U = NCHUNK <= 2 ? 4 : 2;
  static constexpr int STG_SPLIT = NCHUNK <= 2 ? 2 : EPI_SPLIT;
  static constexpr int STG_BYTES = STG_U * 512;
  static constexpr size_t SMEM = 1024 + (size_t)A_STAGES * A_MAX + (size_t)B_REGION + 16384 + 256;
};

template <int BN, int KC, int RT, bool WRES = false>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    conv_halo_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                     const GemmParams p) {
  using C = HaloCfg<BN, KC, RT, WRES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sB = smem;  // 1024-aligned for the swizzled weight tiles
  uint8_t* sA = sB + C::B_REGION;
  uint8_t* sStg = sA + C::A_STAGES * C::A_MAX;
  uint64_t* a_full = reinterpret_cast<uint64_t*>(sStg + 16384);
  uint64_t* a_empty = a_full + C::A_STAGES;
  uint64_t* b_full = a_empty + C::A_STAGES;
  uint64_t* b_empty = b_full + C::B_STAGES;
  uint64_t* tfull = b_empty + C::B_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = warp_id(), lane = lane_id();
  const int P = p.hp, rows_box = p.rows_box;
  const int a_bytes = KC * P * rows_box * 16;
  const int chunk_stride = P * rows_box * 16;  // LBO: distance between 8-channel chunks
  const int nb = p.parts * 9;                  // weight tiles per halo stage
  if (warp == 0 && lane == 0) {
    tma_prefetch(&ta);
    tma_prefetch(&tb);
    for (int i = 0; i < C::A_STAGES; ++i) {
      mbar_init(&a_full[i], 1);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < C::B_STAGES; ++i) {
      mbar_init(&b_full[i], 1);
      mbar_init(&b_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], EPI_WARPS);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tslot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const int ntiles = p.m_tiles * p.n_tiles;
  const int groups = p.cchunks;  // channel groups of GCH
  // dy-stacked MMAs (RT >= 2 output rows on one halo, weights resident, one part / group): the
  // three kernel rows of a tap column sit as one [dy2; dy1; dy0] x BN tile, so a single MMA on
  // halo row h (N = 64 / 128 / .. BN-blocks) adds into the accumulators of every output row it
  // touches (rows h-2..h, BN TMEM columns apart): (RT+2) x 3 x KC/2 MMAs per tile instead of
  // 9 x RT x KC/2, the A operand read once per halo row instead of once per (row, dy). Same
  // per-row accumulation order as the tap loop (dy-major, dx, k). Every MMA accumulates, so the
  // epilogue zeroes each accumulator chunk after reading it (and all of TMEM starts at zero).
  const bool dys = RT >= 2 && WRES && p.parts == 1 && groups == 1 && p.bh == RT;
  if (dys && warp >= 2) {
    const int e = warp - 2;
    for (int c = e >> 2; c < C::TMEM_COLS / 32; c += EPI_SPLIT)
      tmem_zero32(tmem + ((uint32_t)((warp & 3) * 32) << 16) + c * 32);
    tmem_st_wait();
  }
  if (dys) {
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  pdl_wait();
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      int ia = 0, ib = 0;
      if (WRES && dys) {  // tap (dy, dx) -> rows (2 - dy) * BN of the dx tile [dy2; dy1; dy0]
        mbar_expect_tx(&b_full[0], 9 * C::B_BYTES);
        for (int tap = 0; tap < 9; ++tap)
          tma_load_2d(sB + ((tap % 3) * 3 + (2 - tap / 3)) * C::B_BYTES, &tb, &b_full[0], tap * p.kcp, 0);
      } else if (WRES) {  // all weight tiles once (single N tile: the planner guarantees n_tiles == 1)
        mbar_expect_tx(&b_full[0], groups * nb * C::B_BYTES);
        for (int g = 0; g < groups; ++g)
          for (int j = 0; j < nb; ++j) {
            const int part = j / 9, tap = j - part * 9;
            tma_load_2d(sB + (g * nb + j) * C::B_BYTES, &tb, &b_full[0], (part * 9 + tap) * p.kcp + g * C::GCH, 0);
          }
      }
      int tix = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int mt = t / p.n_tiles, nt = t - mt * p.n_tiles;
        const int img = mt / p.tiles_per_img, rr = mt - img * p.tiles_per_img;
        // flat: the box starts one row above the tile's first position, at column -1
        const int y0 = p.flat ? (rr * 128) / P : (rr / p.tiles_x) * p.bh, x0 = p.flat ? 0 : (rr % p.tiles_x) * p.bw;
        for (int g = 0; g < groups; ++g, ++ia) {
          const int sa = ia % C::A_STAGES;
          mbar_wait(&a_empty[sa], ((ia / C::A_STAGES) & 1) ^ 1);
          ROLE_TRACE(680, tix, 11);
          if ((p.dbg & 2) && ia >= C::A_STAGES) {
            mbar_arrive(&a_full[sa]);
          } else {
            mbar_expect_tx(&a_full[sa], a_bytes);
            if (C::SW)
              tma_load_4d(sA + sa * C::A_MAX, &ta, &a_full[sa], g * C::GCH, x0 - 1, y0 - 1, img);
            else
              tma_load_5d(sA + sa * C::A_MAX, &ta, &a_full[sa], 0, x0 - 1, y0 - 1, g * KC, img);
          }
          if (WRES) continue;
          for (int j = 0; j < nb; ++j, ++ib) {
            const int sb = ib % C::B_STAGES;
            mbar_wait(&b_empty[sb], ((ib / C::B_STAGES) & 1) ^ 1);
            mbar_expect_tx(&b_full[sb], C::B_BYTES);
            const int part = j / 9, tap = j - part * 9;
            tma_load_2d(sB + sb * C::B_BYTES, &tb, &b_full[sb], (part * 9 + tap) * p.kcp + g * C::GCH, nt * BN);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(128, BN);
      int ia = 0, ib = 0, i = 0;
      // descriptor words (the start-address field is the low 14 bits, in 16-byte units)
      const uint64_t a_desc0 =
          C::SW ? smem_desc(smem_u32(sA), 16, 8 * C::RB, C::A_LAYOUT) : smem_desc(smem_u32(sA), chunk_stride, 128, 0);
      const uint64_t b_desc0 = smem_desc(smem_u32(sB), 16, C::B_SBO, C::B_SWZ);
      const uint32_t a_lo0 = (uint32_t)a_desc0, a_hi = (uint32_t)(a_desc0 >> 32);
      const uint32_t b_lo0 = (uint32_t)b_desc0, b_hi = (uint32_t)(b_desc0 >> 32);
      const uint32_t kstep = C::SW ? 2u : (uint32_t)(2 * chunk_stride) >> 4;  // one K16 step, 16 B units
      // SW128 starts that are not 1024-aligned (any halo pixel) need no descriptor "base offset":
      // the swizzle is a function of the absolute smem address, which TMA and UMMA share
      // (measured: base offset = (addr >> 7) & 7 breaks every shifted tap)
      const int rsub = p.bh / RT;  // output rows per 128-position sub-tile
      uint32_t toff[9 * RT];
      {
#pragma unroll
        for (int tap = 0; tap < 9; ++tap)
#pragma unroll
          for (int rt = 0; rt < RT; ++rt) {
            const uint32_t px = (uint32_t)((rt * rsub + tap / 3) * P + tap % 3);  // halo pixel of the tap
            toff[tap * RT + rt] = C::SW ? px * (C::RB / 16) : px;
          }
      }
      if (WRES) {  // every weight tile, loaded once
        mbar_wait(&b_full[0], 0);
        tc_fence_after();
      }
      int tix = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
        const int acc = i & 1;
        mbar_wait(&tempty[acc], ((i >> 1) & 1) ^ 1);
        ROLE_TRACE(0, tix, 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * BN * RT;
        // flat tiles: position 0 of the tile sits (128 rr) mod P pixels into the box's second row
        uint32_t foff = 0;
        if (p.flat) {
          const int rr = (t / p.n_tiles) % p.tiles_per_img;
          foff = (uint32_t)((rr * 128) % P) * (C::SW ? C::RB / 16 : 1);
        }
        // The 9 taps x RT rows x KC/2 K-steps are unrolled with every descriptor a precomputed
        // word + constant: the lone issuing thread is latency-bound (~4 clk per dependent
        // instruction), and at ~20 instructions per MMA it could not keep the N=32..128 MMAs
        // (45-65 clk each) fed -- the tile ran at half the tensor rate. Streamed weights (not
        // WRES) arrive one tap tile per ring slot.
        if (dys) {
          const int sa = ia % C::A_STAGES;
          mbar_wait(&a_full[sa], (ia / C::A_STAGES) & 1);
          ROLE_TRACE(0, tix, 2);
          tc_fence_after();
          const uint32_t a_lo = a_lo0 + (uint32_t)sa * (C::A_MAX >> 4);
#pragma unroll
          for (int h = 0; h < RT + 2; ++h) {
            const int r_lo = h > 2 ? h - 2 : 0, r_hi = h < RT - 1 ? h : RT - 1;
            const uint32_t id = idesc_bf16(128, (r_hi - r_lo + 1) * BN);
            const int blk0 = 2 - (h - r_lo);  // block of row r_lo's kernel row dy = h - r_lo
#pragma unroll
            for (int dx = 0; dx < 3; ++dx) {
              const uint32_t at = a_lo + (uint32_t)(h * P + dx) * (C::RB / 16);
              const uint32_t bt = b_lo0 + (uint32_t)((dx * 3 + blk0) * (C::B_BYTES >> 4));
#pragma unroll
              for (int k = 0; k < KC / 2; ++k) {
                const uint64_t ad = ((uint64_t)a_hi << 32) | (at + (uint32_t)k * kstep);
                const uint64_t bd = ((uint64_t)b_hi << 32) | (bt + (uint32_t)(k * 2));
                umma_f16(d + r_lo * BN, ad, bd, id, 1u);
              }
            }
          }
          umma_commit(&a_empty[sa]);
          ++ia;
          ROLE_TRACE(0, tix, 3);
          umma_commit(&tfull[acc]);
          continue;
        }
        for (int g = 0; g < groups; ++g, ++ia) {
          const int sa = ia % C::A_STAGES;
          mbar_wait(&a_full[sa], (ia / C::A_STAGES) & 1);
          ROLE_TRACE(0, tix, 2);
          tc_fence_after();
          const uint32_t a_lo = a_lo0 + (uint32_t)sa * (C::A_MAX >> 4);
          for (int part = 0; part < p.parts; ++part) {
            const uint32_t keep = (g | part) != 0 ? 1u : 0u;
#pragma unroll
            for (int tap = 0; tap < 9; ++tap) {
              uint32_t b_lo;
              int sb = 0;
              if (WRES) {
                b_lo = b_lo0 + (uint32_t)((g * nb + part * 9 + tap) * (C::B_BYTES >> 4));
              } else {
                sb = ib & (C::B_STAGES - 1);
                mbar_wait(&b_full[sb], (ib / C::B_STAGES) & 1);
                tc_fence_after();
                b_lo = b_lo0 + (uint32_t)sb * (C::B_BYTES >> 4);
              }
#pragma unroll
              for (int rt = 0; rt < RT; ++rt) {
                const uint32_t at = a_lo + foff + toff[tap * RT + rt];
#pragma unroll
                for (int k = 0; k < KC / 2; ++k) {
                  const uint64_t ad = ((uint64_t)a_hi << 32) | (at + (uint32_t)k * kstep);
                  const uint64_t bd = ((uint64_t)b_hi << 32) | (b_lo + (uint32_t)(k * 2));
                  umma_f16(d + rt * BN, ad, bd, idesc, (tap | k) != 0 ? 1u : keep);
                }
              }
              if (!WRES) {
                umma_commit(&b_empty[sb]);
                ++ib;
              }
            }
          }
          umma_commit(&a_empty[sa]);
        }
        ROLE_TRACE(0, tix, 3);
        umma_commit(&tfull[acc]);
      }
    }
  } else {
    int tix = 0;
    const bool tr = warp == 2 && lane == 0;
    const int e = warp - 2;
    const int q = warp & 3;
    // EPI_CONV goes through the per-warp smem stage (epilogue_conv_staged)
    const bool staged =
        p.ep.kind == EPI_CONV && (p.ep.ldo & 7) == 0 &&
        ((reinterpret_cast<uintptr_t>(p.ep.out) | reinterpret_cast<uintptr_t>(p.ep.out_relu) |
          reinterpret_cast<uintptr_t>(p.ep.add1) | reinterpret_cast<uintptr_t>(p.ep.add2)) & 15) == 0;
    const int split = staged ? C::STG_SPLIT : EPI_SPLIT;
    const int chalf = (staged && C::STG_SPLIT == 2) ? (e < 8 ? e >> 2 : 1 << 20) : e >> 2;
    uint8_t* stg = sStg + (e & (16384 / C::STG_BYTES - 1)) * C::STG_BYTES;
    const int r = q * 32 + lane;  // virtual output position within a 128-row sub-tile
    const int ry = r / P, rx = r - (r / P) * P;
    const int rows_sub = p.bh / RT;  // output rows per 128-row sub-tile (1 when RT > 1)
    int i = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
      const int acc = i & 1;
      const int mt = t / p.n_tiles, nt = t - mt * p.n_tiles;
      const int img = mt / p.tiles_per_img, rr = mt - img * p.tiles_per_img;
      const int ytile = (rr / p.tiles_x) * p.bh, x = (rr % p.tiles_x) * p.bw + rx;
      mbar_wait(&tfull[acc], (i >> 1) & 1);
      if (tr) ROLE_TRACE(1360, tix, 21);
      tc_fence_after();
      if (chalf >= RT * (BN / 32)) {  // this column slice has no chunk: release at once
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
      }
#pragma unroll 1
      for (int k = chalf; k < RT * (BN / 32); k += split) {
        const int rt = k / (BN / 32), c0 = (k - rt * (BN / 32)) * 32;
        float v[32];
        if (p.dbg & 32) {
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) v[jj] = 0.f;
        } else {
          tmem_ld32(tmem + (acc * RT + rt) * BN + ((uint32_t)(q * 32) << 16) + c0, v);
          tmem_ld_wait();
          if (dys) {
            tmem_zero32(tmem + (acc * RT + rt) * BN + ((uint32_t)(q * 32) << 16) + c0);
            tmem_st_wait();
          }
        }
        if (k + split >= RT * (BN / 32)) {  // last TMEM read of the tile by this warp
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
        int y = ytile + rt * rows_sub + ry, xo = x;
        bool valid = ry < rows_sub && rx < p.bw && y < p.H && x < p.W;
        if (p.flat) {  // position rr * 128 + r of the image's P-pitched layout
          const int gp = rr * 128 + r;
          y = gp / P;
          xo = gp - y * P;
          valid = xo < p.W && y < p.H;
        }
        const int64_t gpix = ((int64_t)img * p.H + y) * p.W + xo;
        const int col0 = nt * BN + c0;
        if (staged && col0 + 32 <= p.ep.N) {
          if (!(p.dbg & 1)) epilogue_conv_staged<C::STG_U>(p.ep, gpix, valid, col0, v, stg);
        } else if (valid && col0 < p.ep.N && !(p.dbg & 1)) epilogue_direct(p.ep, gpix, col0, v);
      }
      if (tr) ROLE_TRACE(1360, tix, 23);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// ------------------------------------------------------------------------------------------
// Upsample-fused 3x3 conv (DPT head: conv1 after the last fusion stage's x2 resize, conv2 after
// the resize to 14h x 14w). The resized map is never written to HBM: per tile, warp 0 TMA-loads
// the small source box the tile's halo samples from (no swizzle, [rows][cols][C] bf16), eight
// builder warps interpolate the (RT+2) x 130-pixel halo straight into the swizzled K-major layout
// conv_halo_kernel gets from TMA (bilerp on f32x2, same rounding as bilinear_ac_rows_kernel, so
// the tile is bit-identical to the resized tensor), and the MMA warp / eight epilogue warps run
// the halo conv's schedule unchanged (weights resident, taps as descriptor start offsets).
// Traffic per output row drops from (RT+2)/RT halo rows of the resized map to ~(RT+2)/RT x the
// resize ratio of source rows, and the resize kernel's write + re-read of the large map goes.
// 20 warps (640 threads, 96 registers): TMA, MMA, two epilogue warps per TMEM lane quadrant,
// ten builders (520 / 1040 jobs per tile in 2 / 4 rounds)
constexpr int UP_EPI_WARPS = 8;
constexpr int UP_BUILD_WARPS = 10;
constexpr int UP_THREADS = 32 * (2 + UP_EPI_WARPS + UP_BUILD_WARPS);
constexpr int UP_MAX_SRC = 4;

template <int BN, int KC, int RT>
struct UpCfg {
  static_assert(BN == 32, "conv_up_kernel: 32 output channels");
  static constexpr int GCH = 8 * KC;   // channels (one group: Cp == GCH)
  static constexpr int RB = 16 * KC;   // bytes per halo pixel
  static constexpr int P = 130;        // halo pitch: 128 output pixels + 2
  static constexpr uint32_t A_LAYOUT = KC == 8 ? 2 : 4;  // UMMA SWIZZLE_128B / SWIZZLE_64B
  static constexpr int A_BYTES = (RB * P * (RT + 2) + 1023) / 1024 * 1024;
  // dy-stacked weights: per dx one [96 = 3 x 32, GCH] K-major tile whose row block b holds the
  // kernel row dy = 2 - b, so one N = 96 MMA on halo row h adds into the accumulators of output
  // rows h-2, h-1, h, laid out 32 TMEM columns apart (see conv_up_kernel)
  static constexpr int NS3 = 3 * BN;
  static constexpr int B_BYTES = NS3 * GCH * 2;  // one dx tile
  static constexpr int W_BYTES = (3 * B_BYTES + 1023) / 1024 * 1024;
  static constexpr int B_SWZ = GCH == 64 ? 2 : 4;
  static constexpr int B_SBO = 8 * GCH * 2;
  static constexpr int AST = 2;        // halo stages
  static constexpr int NACC = RT + 4;  // 32-column accumulators per tile: rows -2 .. RT+1
  static constexpr int ACC = 2;        // tile accumulator sets in TMEM
  static constexpr int TMEM_COLS = GemmCfg<NACC * BN, 64>::TMEM_COLS;
  static constexpr int JOBS = P * KC;  // builder jobs per tile: (halo column, 16-byte channel chunk)
  static constexpr size_t FIXED = 1024 + W_BYTES + AST * (size_t)A_BYTES + UP_EPI_WARPS * 2048 + 256;
};

// 8 channels: bf16x2 words unpacked to f32x2 (exact), bilerp as in bilerp() per lane
VPE_DEV uint32_t bilerp_bf16x2(uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint64_t hx, uint64_t lx, uint64_t hy,
                               uint64_t ly) {
  auto up = [](uint32_t w) {
    return f2_pack(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
  };
  const uint64_t t0 = ffma2(lx, up(b), fmul2(hx, up(a)));
  const uint64_t t1 = ffma2(lx, up(d), fmul2(hx, up(c)));
  float r0, r1;
  f2_unpack(ffma2(ly, t1, fmul2(hy, t0)), r0, r1);
  return pack_bf16(r0, r1);
}

// diagnostics timeline (VPE_TRACE_BUILD + VPE_GEMM_TRACE=1): CTA 0, 500 events per role at
// slots base.. (MMA 0, TMA 510, first builder warp 1020, first epilogue warp 1530)
#ifdef VPE_TRACE_BUILD
#define UP_TRACE(base, idx, code)                                                    \
  do {                                                                               \
    if (p.trace && blockIdx.x == 0 && (idx) < 500) {                                 \
      g_gemm_trace[2 * ((base) + (idx))] = (unsigned long long)(code);               \
      g_gemm_trace[2 * ((base) + (idx)) + 1] = (unsigned long long)clock64();        \
      ++(idx);                                                                       \
    }                                                                                \
  } while (0)
#else
#define UP_TRACE(base, idx, code) \
  do {                            \
  } while (0)
#endif

template <int BN, int KC, int RT>
__global__ void __launch_bounds__(UP_THREADS, 1)
    conv_up_kernel(const __grid_constant__ CUtensorMap ts, const __grid_constant__ CUtensorMap tb,
                   const GemmParams p) {
  using C = UpCfg<BN, KC, RT>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int NS = p.up_stages, SB = p.up_src_bytes;
  uint8_t* sB = smem;
  uint8_t* sA = sB + C::W_BYTES;
  uint8_t* sS = sA + C::AST * C::A_BYTES;
  uint8_t* sStg = sS + NS * SB;
  uint64_t* a_full = reinterpret_cast<uint64_t*>(sStg + UP_EPI_WARPS * 2048);
  uint64_t* a_empty = a_full + C::AST;
  uint64_t* s_full = a_empty + C::AST;
  uint64_t* s_empty = s_full + UP_MAX_SRC;
  uint64_t* w_full = s_empty + UP_MAX_SRC;
  uint64_t* tfull = w_full + 1;
  uint64_t* tempty = tfull + C::ACC;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + C::ACC);

  __shared__ float s_bias[32], s_w3[32];  // epilogue constants (N <= 32), broadcast reads
  const uint32_t warp = warp_id(), lane = lane_id();
  if (warp == 2) {
    s_bias[lane] = (p.ep.bias && (int)lane < p.ep.N) ? p.ep.bias[lane] : 0.f;
    s_w3[lane] = p.ep.w3 ? p.ep.w3[lane] : 0.f;
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&ts);
    tma_prefetch(&tb);
    for (int i = 0; i < C::AST; ++i) {
      mbar_init(&a_full[i], UP_BUILD_WARPS);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < C::ACC; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], UP_EPI_WARPS);
    }
    for (int i = 0; i < NS; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], UP_BUILD_WARPS);
    }
    mbar_init(w_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tslot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  if (warp >= 2 && warp < 2 + UP_EPI_WARPS) {  // every MMA accumulates: start from zero
    float z[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) z[j] = 0.f;
    for (int c = (warp - 2) >> 2; c < C::TMEM_COLS / 32; c += UP_EPI_WARPS / 4)
      tmem_st32(tmem + ((uint32_t)((warp & 3) * 32) << 16) + c * 32, z);
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait();
  pdl_trigger();
  const int ntiles = p.m_tiles;
  const float sh = p.up_sh, sw = p.up_sw;
  // tile t -> image, first output row, first output column; source box origin
  auto tile_of = [&](int t, int& img, int& y0, int& x0) {
    img = t / p.tiles_per_img;
    const int rr = t - img * p.tiles_per_img;
    y0 = (rr / p.tiles_x) * RT;
    x0 = (rr - (rr / p.tiles_x) * p.tiles_x) * 128;
  };
  auto src_origin = [&](int y0, int x0, int& sy, int& sx) {
    sy = ac_coord(sh, y0 > 0 ? y0 - 1 : 0, p.up_hs).i0;
    sx = ac_coord(sw, x0 > 0 ? x0 - 1 : 0, p.up_ws).i0;
  };

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(w_full, 3 * C::B_BYTES);
      for (int dx = 0; dx < 3; ++dx) tma_load_2d(sB + dx * C::B_BYTES, &tb, w_full, 0, dx * C::NS3);
      int i = 0, tix = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
        const int ss = i % NS;
        mbar_wait_sleep(&s_empty[ss], ((i / NS) & 1) ^ 1);
        UP_TRACE(510, tix, 11);
        int img, y0, x0, sy, sx;
        tile_of(t, img, y0, x0);
        src_origin(y0, x0, sy, sx);
        mbar_expect_tx(&s_full[ss], p.up_box_bytes);
        tma_load_4d(sS + ss * SB, &ts, &s_full[ss], 0, sx, sy, img);
      }
    }
  } else if (warp == 1) {
    // the whole warp walks the loop (warp-voted waits keep descriptors in uniform registers);
    // one elected lane issues
    constexpr uint32_t idesc = idesc_bf16(128, C::NS3);
    const uint64_t a_desc0 = smem_desc(smem_u32(sA), 16, 8 * C::RB, C::A_LAYOUT);
    const uint64_t b_desc0 = smem_desc(smem_u32(sB), 16, C::B_SBO, C::B_SWZ);
    const uint32_t a_lo0 = (uint32_t)a_desc0, a_hi = (uint32_t)(a_desc0 >> 32);
    const uint32_t b_lo0 = (uint32_t)b_desc0, b_hi = (uint32_t)(b_desc0 >> 32);
    mbar_wait_warp(w_full, 0);
    tc_fence_after();
    int i = 0, tix = 0;
    const bool tr = lane == 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
      const int acc = i % C::ACC, sa = i % C::AST;
      mbar_wait_warp(&tempty[acc], ((i / C::ACC) & 1) ^ 1);
      if (tr) UP_TRACE(0, tix, 1);
      tc_fence_after();
      mbar_wait_warp(&a_full[sa], (i / C::AST) & 1);
      if (tr) UP_TRACE(0, tix, 2);
      tc_fence_after();
      const uint32_t d = tmem + acc * C::NACC * BN;
      const uint32_t a_lo = a_lo0 + (uint32_t)sa * (C::A_BYTES >> 4);
      // halo row h, shift dx: columns [h*32, h*32 + 96) = accumulators of output rows h-2..h
#pragma unroll
      for (int h = 0; h < ((p.dbg & 2) ? 0 : RT + 2); ++h) {
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) {
          const uint32_t at = a_lo + (uint32_t)(h * C::P + dx) * (C::RB / 16);
          const uint32_t b_lo = b_lo0 + (uint32_t)(dx * (C::B_BYTES >> 4));
#pragma unroll
          for (int k = 0; k < KC / 2; ++k) {
            const uint64_t ad = ((uint64_t)a_hi << 32) | (at + (uint32_t)k * 2u);
            const uint64_t bd = ((uint64_t)b_hi << 32) | (b_lo + (uint32_t)(k * 2));
            if (elect_one()) umma_f16(d + h * BN, ad, bd, idesc, 1u);
          }
        }
      }
      if (elect_one()) umma_commit(&a_empty[sa]);
      if (elect_one()) umma_commit(&tfull[acc]);
      __syncwarp();
      if (tr) UP_TRACE(0, tix, 3);
    }
  } else if (warp < 2 + UP_EPI_WARPS) {
    const int e = warp - 2, q = warp & 3, chalf = e >> 2;  // two warps per TMEM lane quadrant
    const bool staged =
        p.ep.kind == EPI_CONV && (p.ep.ldo & 7) == 0 &&
        ((reinterpret_cast<uintptr_t>(p.ep.out) | reinterpret_cast<uintptr_t>(p.ep.out_relu) |
          reinterpret_cast<uintptr_t>(p.ep.add1) | reinterpret_cast<uintptr_t>(p.ep.add2)) & 15) == 0;
    uint8_t* stg = sStg + e * 2048;
    const int r = q * 32 + lane;  // output pixel within the tile's 128-wide row
    int i = 0, tix = 0;
    const bool tr = e == 0 && lane == 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
      const int acc = i % C::ACC;
      int img, y0, x0;
      tile_of(t, img, y0, x0);
      mbar_wait_sleep(&tfull[acc], (i / C::ACC) & 1);
      if (tr) UP_TRACE(1530, tix, 31);
      tc_fence_after();
      const uint32_t tbase = tmem + acc * C::NACC * BN + ((uint32_t)(q * 32) << 16);
      float z[32];
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) z[jj] = 0.f;
      // rows -2, -1, RT, RT+1 collect the dy-stack's out-of-tile partial sums: clear them
      for (int k = chalf; k < 4; k += UP_EPI_WARPS / 4) tmem_st32(tbase + (k < 2 ? k : RT + k) * BN, z);
#pragma unroll 1
      for (int k = chalf; k < RT; k += UP_EPI_WARPS / 4) {
        const int rt = k, c0 = 0;
        float v[32];
        tmem_ld32(tbase + (rt + 2) * BN, v);
        tmem_ld_wait();
        tmem_st32(tbase + (rt + 2) * BN, z);
        if (k + UP_EPI_WARPS / 4 >= RT) {  // last TMEM access of the tile by this warp
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
        const int y = y0 + rt, x = x0 + r;
        const bool valid = y < p.H && x < p.W;
        const int64_t gpix = ((int64_t)img * p.H + y) * p.W + x;
        if (p.ep.kind == EPI_DEPTH) {  // N == 32: bias and w3 from smem
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) v[jj] += s_bias[jj];
          const float pre = depth_dot(v, s_w3, p.ep.b3);
          if (valid) {
            p.ep.depth_pre[gpix] = pre;
            p.ep.depth[gpix] = fmaxf(pre, 0.f) * p.ep.max_depth;
          }
        } else if (staged && c0 + 32 <= p.ep.N) {
          epilogue_conv_staged<4>(p.ep, gpix, valid, c0, v, stg);
        } else if (valid && c0 < p.ep.N) {
          epilogue_direct(p.ep, gpix, c0, v);
        }
      }
      if (tr) UP_TRACE(1530, tix, 32);
    }
  } else {
    // builders. Job = (halo column c, 16-byte channel chunk g) for all RT+2 halo rows: the
    // horizontal lerp t = lx*b + hx*a of a source row is computed once and kept while consecutive
    // halo rows sample that row (ratio < 1: a source row serves ~1/ratio halo rows), then
    // out = ly*t(i1) + hy*t(i0) -- bilerp()'s exact operation order, on f32x2. Rows are the outer
    // loop (their sampling is tile-uniform: no divergence) and each thread carries two jobs
    // through it side by side, so the two dependent LDS -> FMA -> STS chains overlap.
    constexpr int NB = UP_BUILD_WARPS * 32;
    const int bt = (int)(warp - 2 - UP_EPI_WARPS) * 32 + (int)lane;
    const int row_bytes = p.up_cols * C::GCH * 2;
    int i = 0, tix = 0;
    const bool tr = bt == 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
      const int sa = i % C::AST, ss = i % NS;
      int img, y0, x0, sy, sx;
      tile_of(t, img, y0, x0);
      src_origin(y0, x0, sy, sx);
      mbar_wait_sleep(&a_empty[sa], ((i / C::AST) & 1) ^ 1);
      if (tr) UP_TRACE(1020, tix, 21);
      mbar_wait_sleep(&s_full[ss], (i / NS) & 1);
      if (tr) UP_TRACE(1020, tix, 22);
      const uint32_t src = smem_u32(sS + ss * SB);
      const uint32_t dst = smem_u32(sA + sa * C::A_BYTES);
      // Each pass hands 2 jobs to each of the first `act` threads (the rest skip it) instead of
      // 1-2 jobs to all of them: with KC = 4 (520 jobs, 320 threads) only 8 warps do the work.
#pragma unroll 1
      for (int base = ((p.dbg & 1) ? C::JOBS : 0); base < C::JOBS; base += 2 * NB) {
        const int rem = C::JOBS - base < 2 * NB ? C::JOBS - base : 2 * NB, act = (rem + 1) >> 1;
        if (bt >= act) continue;
        const int jb = base + bt;
        uint32_t s0[2], s1[2];
        uint64_t hx[2], lx[2], hl[2][4], hh[2][4];
        int cj[2], gj[2];
        bool xv[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int j = jb + q * act < base + rem ? jb + q * act : jb;  // odd count: the last thread redoes its job
          cj[q] = j / KC;
          gj[q] = j - cj[q] * KC;
          const int X = x0 - 1 + cj[q];
          xv[q] = X >= 0 && X < p.W;  // lane-dependent: applied as a select at the store
          const AcCoord cx = ac_coord(sw, xv[q] ? X : 0, p.up_ws);
          s0[q] = src + ((cx.i0 - sx) * C::GCH + gj[q] * 8) * 2;
          s1[q] = src + ((cx.i1 - sx) * C::GCH + gj[q] * 8) * 2;
          hx[q] = f2_pack(cx.h, cx.h);
          lx[q] = f2_pack(cx.l, cx.l);
        }
        auto hlerp = [&](int q, int roff, uint64_t (&h)[4]) {
          const uint4 a = lds128(s0[q] + roff);
          const uint4 b = lds128(s1[q] + roff);
          const uint32_t aw[4] = {a.x, a.y, a.z, a.w}, bw[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t av = f2_pack(__uint_as_float(aw[k] << 16), __uint_as_float(aw[k] & 0xffff0000u));
            const uint64_t bv = f2_pack(__uint_as_float(bw[k] << 16), __uint_as_float(bw[k] & 0xffff0000u));
            h[k] = ffma2(lx[q], bv, fmul2(hx[q], av));
          }
        };
        int cur0 = -1, cur1 = -1;  // source rows (byte offsets) held in hl / hh: tile-uniform
#pragma unroll
        for (int r = 0; r < RT + 2; ++r) {
          const int Y = y0 - 1 + r;
          uint32_t o[2];
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int px = r * C::P + cj[q];
            const int swz = KC == 8 ? (px & 7) : ((px >> 1) & 3);  // TMA/UMMA 128B / 64B swizzle
            o[q] = dst + px * C::RB + ((gj[q] ^ swz) << 4);
          }
          if (Y < 0 || Y >= p.H) {
            sts128(o[0], make_uint4(0, 0, 0, 0));
            sts128(o[1], make_uint4(0, 0, 0, 0));
            continue;
          }
          const AcCoord cy = ac_coord(sh, Y, p.up_hs);
          const int n0 = (cy.i0 - sy) * row_bytes, n1 = (cy.i1 - sy) * row_bytes;
          if (n0 != cur0) {
            if (n0 == cur1) {
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                hl[0][k] = hh[0][k];
                hl[1][k] = hh[1][k];
              }
            } else {
              hlerp(0, n0, hl[0]);
              hlerp(1, n0, hl[1]);
            }
            cur0 = n0;
          }
          if (n1 != cur1) {
            if (n1 == cur0) {
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                hh[0][k] = hl[0][k];
                hh[1][k] = hl[1][k];
              }
            } else {
              hlerp(0, n1, hh[0]);
              hlerp(1, n1, hh[1]);
            }
            cur1 = n1;
          }
          const uint64_t hy = f2_pack(cy.h, cy.h), ly = f2_pack(cy.l, cy.l);
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            uint32_t w[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              float v0, v1;
              f2_unpack(ffma2(ly, hh[q][k], fmul2(hy, hl[q][k])), v0, v1);
              w[k] = xv[q] ? pack_bf16(v0, v1) : 0u;
            }
            sts128(o[q], make_uint4(w[0], w[1], w[2], w[3]));
          }
        }
      }
      fence_async_smem();  // generic-proxy halo writes -> tensor-core (async proxy) reads
      __syncwarp();
      if (tr) UP_TRACE(1020, tix, 23);
      if (lane == 0) {
        mbar_arrive(&a_full[sa]);
        mbar_arrive(&s_empty[ss]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// ------------------------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static int g_num_sms = 0;

bool tma_available() {
  if (g_encode) return true;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || fn == nullptr)
    return false;
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return true;
}

static int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

int encode_tma_t(CUtensorMap* m, CUtensorMapDataType dt, int rank, const void* ptr, const uint64_t* dims,
                 const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapSwizzle swz) {
  if (!tma_available()) return VPE_E_CUDA;
  uint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = g_encode(m, dt, rank, const_cast<void*>(ptr), dims, strides_bytes, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    fprintf(stderr, "[vpe] cuTensorMapEncodeTiled failed (%d) rank=%d dims=%llu,%llu box=%u,%u\n", (int)r, rank,
            (unsigned long long)dims[0], (unsigned long long)dims[1], box[0], box[1]);
    return VPE_E_SHAPE;
  }
  return VPE_OK;
}

int encode_tma(CUtensorMap* m, int rank, const void* ptr, const uint64_t* dims, const uint64_t* strides_bytes,
               const uint32_t* box, CUtensorMapSwizzle swz) {
  return encode_tma_t(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, ptr, dims, strides_bytes, box, swz);
}

static int smem_for(int bn, int bk) {
#define VPE_SM(BN_, BK_) \
  if (bn == BN_ && bk == BK_) return (int)GemmCfg<BN_, BK_>::SMEM;
  VPE_SM(32, 64) VPE_SM(64, 64) VPE_SM(128, 64) VPE_SM(192, 64) VPE_SM(256, 64) VPE_SM(32, 32) VPE_SM(64, 32)
#undef VPE_SM
  return -1;
}

static int make_b_map(GemmPlan* g, const __nv_bfloat16* B, int N, int Kb, int64_t ldb, int bn, int bk) {
  if ((ldb * 2) % 16 || (reinterpret_cast<uintptr_t>(B) % 16)) return VPE_E_SHAPE;
  uint64_t dims[2] = {(uint64_t)Kb, (uint64_t)N};
  uint64_t strides[1] = {(uint64_t)ldb * 2};
  uint32_t box[2] = {(uint32_t)bk, (uint32_t)bn};
  return encode_tma(&g->tb, 2, B, dims, strides, box, bk == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B);
}

// TMA-store epilogue for row-major outputs (bf16 / f32 store, f32 residual reduce-add)
static int make_out_map(GemmPlan* g, int M) {
  const EpiParams& ep = g->p.ep;
  if (ep.kind != EPI_BF16 && ep.kind != EPI_F32 && ep.kind != EPI_RESID) return VPE_OK;
  if (ep.out_relu) return VPE_OK;
  const bool bf = ep.kind == EPI_BF16;
  void* base = ep.kind == EPI_RESID ? static_cast<void*>(ep.resid) : ep.out;
  const int64_t ld = ep.kind == EPI_RESID ? ep.ldr : ep.ldo;
  const int esz = bf ? 2 : 4;
  if ((ld * esz) % 16 || reinterpret_cast<uintptr_t>(base) % 16 || ep.N % (16 / esz)) return VPE_OK;
  uint64_t dims[2] = {(uint64_t)ep.N, (uint64_t)M};
  uint64_t strides[1] = {(uint64_t)ld * esz};
  uint32_t box[2] = {32u, 32u};
  VPE_TRY(encode_tma_t(&g->tout, bf ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims,
                       strides, box, bf ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B));
  g->p.tma_out = 1;
  return VPE_OK;
}

static void finish_grid(GemmPlan* g, int N, int bn, int m_tiles) {
  g->p.n_tiles = (N + bn - 1) / bn;
  g->p.m_tiles = m_tiles;
  const int tiles = g->p.n_tiles * m_tiles;
  int ctas = tiles < num_sms() ? tiles : num_sms();
  static int mult = -1;  // experiment: VPE_GEMM_GRID=k -> k CTAs per SM worth of grid (tiles spread)
  if (mult < 0) {
    const char* e = getenv("VPE_GEMM_GRID");
    mult = e ? atoi(e) : 1;
  }
  if (mult > 1) ctas = tiles < num_sms() * mult ? tiles : num_sms() * mult;
  g->grid = dim3(ctas, 1, 1);
}

int plan_gemm_rows(GemmPlan* g, const __nv_bfloat16* A, int M, int K, int64_t lda, const __nv_bfloat16* B, int N,
                   int Kb, int64_t ldb, const EpiParams& ep, int bn) {
  const int bk = 64;
  if (K % bk || Kb % K || smem_for(bn, bk) < 0) return VPE_E_SHAPE;
  if ((lda * 2) % 16 || (reinterpret_cast<uintptr_t>(A) % 16)) return VPE_E_SHAPE;
  memset(g, 0, sizeof(*g));
  uint64_t dims[2] = {(uint64_t)K, (uint64_t)M};
  uint64_t strides[1] = {(uint64_t)lda * 2};
  uint32_t box[2] = {(uint32_t)bk, 128u};
  int rc = encode_tma(&g->ta, 2, A, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  if ((rc = make_b_map(g, B, N, Kb, ldb, bn, bk))) return rc;
  g->p.kblocks = Kb / bk;
  g->p.kblocks_a = K / bk;
  g->p.mode = 0;
  g->p.M = M;
  g->p.ks = 1;
  g->p.cchunks = 1;
  g->p.ep = ep;
  if ((rc = make_out_map(g, M))) return rc;
  finish_grid(g, N, bn, (M + 127) / 128);
  g->bn = bn;
  g->bk = bk;
  g->smem = smem_for(bn, bk);
  return VPE_OK;
}

int plan_gemm_conv(GemmPlan* g, const __nv_bfloat16* X, int nimg, int H, int W, int C, int64_t pitch_px,
                   int64_t pitch_row, int64_t pitch_img, int ks, int bk, const __nv_bfloat16* B, int N, int Kb,
                   int64_t ldb, const EpiParams& ep, int bn) {
  if ((bk != 64 && bk != 32) || smem_for(bn, bk) < 0 || (ks != 1 && ks != 3)) return VPE_E_SHAPE;
  const int cchunks = (C + bk - 1) / bk;
  const int ka = ks * ks * cchunks;
  if (Kb % (ka * bk)) return VPE_E_SHAPE;
  if ((pitch_px * 2) % 16 || (pitch_row * 2) % 16 || (pitch_img * 2) % 16 || reinterpret_cast<uintptr_t>(X) % 16)
    return VPE_E_SHAPE;
  memset(g, 0, sizeof(*g));
  // spatial tile bw x bh = 128 pixels; pick bw (power of two <= 128) minimising padded area
  int best_bw = 128, best_cost = 1 << 30;
  for (int bw = 128; bw >= 1; bw >>= 1) {
    const int bh = 128 / bw;
    const int cost = ((W + bw - 1) / bw) * bw * (((H + bh - 1) / bh) * bh);
    if (cost < best_cost) {
      best_cost = cost;
      best_bw = bw;
    }
  }
  const int bw = best_bw, bh = 128 / bw;
  uint64_t dims[4] = {(uint64_t)C, (uint64_t)W, (uint64_t)H, (uint64_t)nimg};
  uint64_t strides[3] = {(uint64_t)pitch_px * 2, (uint64_t)pitch_row * 2, (uint64_t)pitch_img * 2};
  uint32_t box[4] = {(uint32_t)bk, (uint32_t)bw, (uint32_t)bh, 1u};
  int rc = encode_tma(&g->ta, 4, X, dims, strides, box, bk == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B);
  if (rc) return rc;
  if ((rc = make_b_map(g, B, N, Kb, ldb, bn, bk))) return rc;
  g->p.kblocks = Kb / bk;
  g->p.kblocks_a = ka;
  g->p.mode = 1;
  g->p.ks = ks;
  g->p.cchunks = cchunks;
  g->p.H = H;
  g->p.W = W;
  g->p.bw = bw;
  g->p.bh = bh;
  g->p.tiles_x = (W + bw - 1) / bw;
  g->p.tiles_per_img = g->p.tiles_x * ((H + bh - 1) / bh);
  g->p.M = nimg * H * W;
  g->p.ep = ep;
  finish_grid(g, N, bn, nimg * g->p.tiles_per_img);
  g->bn = bn;
  g->bk = bk;
  g->smem = smem_for(bn, bk);
  return VPE_OK;
}

int plan_conv_halo(GemmPlan* g, const __nv_bfloat16* X, int nimg, int H, int W, int Cp, int64_t pitch_px,
                   int64_t pitch_row, int64_t pitch_img, int parts, const __nv_bfloat16* B, int N, int64_t ldb,
                   const EpiParams& ep, int bn) {
  if (Cp % 32 || (bn != 32 && bn != 64 && bn != 128)) return VPE_E_SHAPE;
  const int kc = (Cp % 64 == 0) ? 8 : 4;
  if (Cp == 32) {
    if (kc != 4) return VPE_E_SHAPE;
  } else if (Cp % 64) {
    return VPE_E_SHAPE;
  }
  int bw, P, rows, rt = 1;
  if (W >= 128) {
    bw = 128;
    P = 130;
    // stack RT output rows on one halo when the channel group is narrow (A traffic per output
    // row (RT+2)/RT); keep the 2 x RT x BN TMEM columns and the two halo stages within budget
    if (kc == 4 && bn == 32) rt = 4;
    else if (kc == 8 && bn <= 64) rt = 2;
    rows = rt;
  } else {
    bw = W;
    P = W + 2;
    rows = 128 / P;
    // streamed weights (too large to stay resident, e.g. the det head's 384 -> 384 hi+lo conv):
    // two multi-row sub-tiles share each weight tile, halving the L2 -> SMEM weight traffic that
    // bounds those convs (measured 7.3 TB/s of weight re-reads at 32 x 32)
    const bool streamed = (size_t)parts * 9 * Cp * bn * 2 > (size_t)WRES_BYTES || (N + bn - 1) / bn > 1;
    if (kc == 8 && bn == 128 && streamed && !getenv("VPE_HALO_NO_RT2")) {
      const int rb2 = rows + 129 / P + 3;
      if (rb2 * P <= 130 * 4) rt = 2;
    }
  }
  static const double min_fill = getenv("VPE_HALO_FILL") ? atof(getenv("VPE_HALO_FILL")) : 0.7;
  static const bool flat_ok = !getenv("VPE_HALO_FLAT") || atoi(getenv("VPE_HALO_FLAT")) != 0;
  const int rows_sub = W >= 128 ? 1 : rows;  // output rows per 128-position sub-tile
  // Whole rows per 128-position tile would leave it under-filled (W = 64: one 66-position row):
  // tile the image's P-pitched position space in runs of 128 instead (rows straddle tiles; the
  // two pad columns per row are the only idle MMA rows, 64 / 66 filled). The box spans the
  // rows a run touches plus the halo: 3 + ceil(128 / P).
  const bool flat = W < 128 && flat_ok && (rows < 1 || (double)(rows_sub * bw) / 128.0 < min_fill);
  if (flat) {
    rt = 1;
    rows = 1;
  } else if (rows < 1 || (double)(rows_sub * bw) / 128.0 < min_fill) {
    return VPE_E_SHAPE;
  }
  if (W < 128 && !flat) rows = rows_sub * rt;  // output rows per tile
  const int rows_box = flat ? 3 + (128 + P - 1) / P
                            : (W >= 128 ? (rt > 1 ? rt + 2 : 129 / P + 3) : (rt - 1) * rows_sub + 129 / P + 3);
  if (P > 256 || rows_box > 256) return VPE_E_SHAPE;
  if (flat && P * rows_box > 130 * 3) return VPE_E_SHAPE;  // the RT = 1 instances' A stage (A_MAX)
  if ((pitch_px * 2) % 16 || (pitch_row * 2) % 16 || (pitch_img * 2) % 16 || reinterpret_cast<uintptr_t>(X) % 16)
    return VPE_E_SHAPE;
  memset(g, 0, sizeof(*g));
  {
    // 4D view {ch, x, y, img}, box {8 kc, P, rows, 1}, SWIZZLE_128B / 64B: one row per pixel
    uint64_t dims[4] = {(uint64_t)Cp, (uint64_t)W, (uint64_t)H, (uint64_t)nimg};
    uint64_t strides[3] = {(uint64_t)pitch_px * 2, (uint64_t)pitch_row * 2, (uint64_t)pitch_img * 2};
    uint32_t box[4] = {8u * kc, (uint32_t)P, (uint32_t)rows_box, 1u};
    VPE_TRY(encode_tma(&g->ta, 4, X, dims, strides, box,
                       kc == 8 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B));
  }
  const int gch = 8 * kc;
  VPE_TRY(make_b_map(g, B, N, parts * 9 * Cp, ldb, bn, gch));
  g->p.mode = 2;
  g->p.hp = P;
  g->p.rows_box = rows_box;
  g->p.parts = parts;
  g->p.kcp = Cp;
  g->p.cchunks = Cp / gch;  // channel groups
  g->p.ks = 3;
  g->p.H = H;
  g->p.W = W;
  g->p.bw = bw;
  g->p.bh = rows;
  g->p.tiles_x = (W + bw - 1) / bw;
  g->p.tiles_per_img = g->p.tiles_x * ((H + rows - 1) / rows);
  if (flat) {
    g->p.flat = 1;
    g->p.tiles_x = 1;
    g->p.tiles_per_img = (H * P - 2 + 127) / 128;  // the last row's 2 pad positions need no tile
  }
  g->p.M = nimg * H * W;
  g->p.ep = ep;
  finish_grid(g, N, bn, nimg * g->p.tiles_per_img);
  g->bn = bn;
  g->bk = gch;
  g->halo_kc = kc;
  g->halo_rt = rt;
  // weights resident in smem when the whole conv fits (single N tile)
  g->halo_wres = (g->p.n_tiles == 1 && (size_t)parts * 9 * Cp * bn * 2 <= (size_t)WRES_BYTES &&
                  !getenv("VPE_NO_WRES"));
#define VPE_HS(BN_, KC_, RT_)                                                        \
  if (bn == BN_ && kc == KC_ && rt == RT_)                                           \
    g->smem = g->halo_wres ? HaloCfg<BN_, KC_, RT_, true>::SMEM : HaloCfg<BN_, KC_, RT_>::SMEM;
  VPE_HS(32, 4, 1) VPE_HS(64, 4, 1) VPE_HS(128, 4, 1) VPE_HS(32, 8, 1) VPE_HS(64, 8, 1) VPE_HS(128, 8, 1)
  VPE_HS(32, 4, 4) VPE_HS(32, 8, 2) VPE_HS(64, 8, 2) VPE_HS(128, 8, 2)
#undef VPE_HS
  return VPE_OK;
}

int pack_conv_up_weights(const __nv_bfloat16* B, int Cp, __nv_bfloat16* wpack, cudaStream_t stream) {
  // dy-stacked weights: wpack[dx][b * 32 + co][c] = W[co][tap (2 - b, dx)][c] (UpCfg)
  for (int dx = 0; dx < 3; ++dx)
    for (int b = 0; b < 3; ++b)
      VPE_CUDA_TRY(cudaMemcpy2DAsync(wpack + (size_t)(dx * 96 + b * 32) * Cp, (size_t)Cp * 2,
                                     B + (size_t)((2 - b) * 3 + dx) * Cp, (size_t)9 * Cp * 2, (size_t)Cp * 2, 32,
                                     cudaMemcpyDeviceToDevice, stream));
  return VPE_OK;
}

int plan_conv_up(GemmPlan* g, const __nv_bfloat16* X, int nimg, int Hs, int Ws, int Cp, int Ho, int Wo,
                 const __nv_bfloat16* B, int N, const EpiParams& ep, __nv_bfloat16* wpack, cudaStream_t stream) {
  if ((Cp != 32 && Cp != 64) || N != 32 || Wo < 128 || Ho < 2 || Hs < 1 || Ws < 1 || !wpack) return VPE_E_SHAPE;
  if (reinterpret_cast<uintptr_t>(X) % 16 || reinterpret_cast<uintptr_t>(B) % 16 ||
      reinterpret_cast<uintptr_t>(wpack) % 16)  // B null: wpack already holds the packed weights
    return VPE_E_SHAPE;
  const int kc = Cp / 8, rt = Cp == 32 ? 4 : 2, bn = 32;
  memset(g, 0, sizeof(*g));
  const float sh = ac_scale(Hs, Ho), sw = ac_scale(Ws, Wo);
  // source box: the largest span any tile's halo samples (same float math as the kernel)
  auto span = [](float s, int n_in, int n_out, int step, int len) {
    int m = 0;
    for (int o0 = 0; o0 < n_out; o0 += step) {
      const int lo = o0 > 0 ? o0 - 1 : 0, hi = o0 + len < n_out ? o0 + len : n_out - 1;
      const int i_lo = ac_i0_host(s, lo), i_hi0 = ac_i0_host(s, hi);
      const int i_hi = i_hi0 + (i_hi0 < n_in - 1);
      if (i_hi - i_lo + 1 > m) m = i_hi - i_lo + 1;
    }
    return m;
  };
  const int rows = span(sh, Hs, Ho, rt, rt), cols = span(sw, Ws, Wo, 128, 128);
  if (rows > 256 || cols > 256) return VPE_E_SHAPE;
  {
    uint64_t dims[4] = {(uint64_t)Cp, (uint64_t)Ws, (uint64_t)Hs, (uint64_t)nimg};
    uint64_t strides[3] = {(uint64_t)Cp * 2, (uint64_t)Ws * Cp * 2, (uint64_t)Hs * Ws * Cp * 2};
    uint32_t box[4] = {(uint32_t)Cp, (uint32_t)cols, (uint32_t)rows, 1u};
    VPE_TRY(encode_tma(&g->ta, 4, X, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE));
  }
  if (B) VPE_TRY(pack_conv_up_weights(B, Cp, wpack, stream));
  {
    uint64_t dims[2] = {(uint64_t)Cp, 288};
    uint64_t strides[1] = {(uint64_t)Cp * 2};
    uint32_t box[2] = {(uint32_t)Cp, 96};
    VPE_TRY(encode_tma(&g->tb, 2, wpack, dims, strides, box,
                       Cp == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B));
  }
  const int box_bytes = rows * cols * Cp * 2;
  const int src_bytes = (box_bytes + 127) / 128 * 128;
  const size_t fixed = Cp == 32 ? UpCfg<32, 4, 4>::FIXED : UpCfg<32, 8, 2>::FIXED;
  const size_t budget = 227 * 1024 - 512;  // dynamic + the kernel's static epilogue constants
  int stages = 0;
  while (stages < UP_MAX_SRC && fixed + (size_t)(stages + 1) * src_bytes <= budget) ++stages;
  if (stages < 1) return VPE_E_SHAPE;
  static const int max_st = getenv("VPE_UP_STAGES") ? atoi(getenv("VPE_UP_STAGES")) : UP_MAX_SRC;
  if (max_st >= 1 && stages > max_st) stages = max_st;
  g->p.mode = 3;
  g->p.kcp = Cp;
  g->p.cchunks = 1;
  g->p.ks = 3;
  g->p.H = Ho;
  g->p.W = Wo;
  g->p.bw = 128;
  g->p.bh = rt;
  g->p.hp = 130;
  g->p.tiles_x = (Wo + 127) / 128;
  g->p.tiles_per_img = g->p.tiles_x * ((Ho + rt - 1) / rt);
  g->p.M = nimg * Ho * Wo;
  g->p.up_hs = Hs;
  g->p.up_ws = Ws;
  g->p.up_rows = rows;
  g->p.up_cols = cols;
  g->p.up_stages = stages;
  g->p.up_src_bytes = src_bytes;
  g->p.up_box_bytes = box_bytes;
  g->p.up_sh = sh;
  g->p.up_sw = sw;
  g->p.ep = ep;
  finish_grid(g, N, bn, nimg * g->p.tiles_per_img);
  g->bn = bn;
  g->bk = Cp;
  g->up_kc = kc;
  g->halo_rt = rt;
  g->smem = fixed + (size_t)stages * src_bytes;
  return VPE_OK;
}

template <int BN, int KC, int RT>
static int launch_up_t(const GemmPlan& g, cudaStream_t s) {
  auto k = conv_up_kernel<BN, KC, RT>;
  static OncePerDevice attr_set;
  if (attr_set.first()) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024 - 512);
    max_smem_carveout(k);
  }
  PdlKind pk(8);
  static const int dbg = getenv("VPE_UP_DBG") ? atoi(getenv("VPE_UP_DBG")) : 0;  // 1 no build, 2 no MMA
  GemmParams p = g.p;
  p.dbg = dbg;
  if (g_gemm_trace_on < 0) {
    const char* e = getenv("VPE_GEMM_TRACE");
    g_gemm_trace_on = (e && e[0] == '1') ? 1 : 0;
  }
  p.trace = g_gemm_trace_on;
  return launch_k(k, g.grid, dim3(UP_THREADS), g.smem, s, g.ta, g.tb, p) == cudaSuccess ? VPE_OK : VPE_E_CUDA;
}

template <int BN, int KC, int RT, bool WRES = false>
static int launch_halo_t(const GemmPlan& g0, cudaStream_t s) {
  auto k = conv_halo_kernel<BN, KC, RT, WRES>;
  static const int dbg = getenv("VPE_HALO_DBG") ? atoi(getenv("VPE_HALO_DBG")) : 0;
  GemmPlan g = g0;
  g.p.dbg = dbg;
  if (g_gemm_trace_on < 0) {
    const char* e = getenv("VPE_GEMM_TRACE");
    g_gemm_trace_on = (e && e[0] == '1') ? 1 : 0;
  }
  g.p.trace = g_gemm_trace_on;
  static OncePerDevice attr_set;
  if (attr_set.first()) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)HaloCfg<BN, KC, RT, WRES>::SMEM);
    max_smem_carveout(k);
  }
  PdlKind pk(8);
  return launch_k(k, g.grid, dim3(GEMM_THREADS), HaloCfg<BN, KC, RT, WRES>::SMEM, s, g.ta, g.tb, g.p) == cudaSuccess
             ? VPE_OK
             : VPE_E_CUDA;
}

template <int BN, int BK>
static int launch_t(const GemmPlan& g, cudaStream_t s) {
  auto k = gemm_tc_kernel<BN, BK>;
  static OncePerDevice attr_set;
  if (attr_set.first()) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GemmCfg<BN, BK>::SMEM);
    max_smem_carveout(k);
  }
  if (g_gemm_trace_on < 0) {
    const char* e = getenv("VPE_GEMM_TRACE");
    g_gemm_trace_on = (e && e[0] == '1') ? 1 : 0;
  }
  GemmParams p = g.p;
  p.trace = g_gemm_trace_on;
  p.pdl_late = pdl_late();
  PdlKind pk(1);
  return launch_k(k, g.grid, dim3(GEMM_THREADS), GemmCfg<BN, BK>::SMEM, s, g.ta, g.tb, g.tout, p) == cudaSuccess
             ? VPE_OK
             : VPE_E_CUDA;
}

static int bf16_rows_map(CUtensorMap* m, const __nv_bfloat16* base, int M, int N) {
  if (reinterpret_cast<uintptr_t>(base) % 16) return VPE_E_SHAPE;
  uint64_t dims[2] = {(uint64_t)N, (uint64_t)M};
  uint64_t strides[1] = {(uint64_t)N * 2};
  uint32_t box[2] = {32u, 32u};
  return encode_tma_t(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_64B);
}

int plan_gemm_resid_ln(GemmPlan* g, const __nv_bfloat16* A, int M, int K, const __nv_bfloat16* W, const float* bias,
                       const float* ls, float* resid, const float* ln_w, const float* ln_b, float eps,
                       __nv_bfloat16* xln, const float* tw, const float* tb) {
  if (K % 64 || !bias || !ls || !resid || !ln_w || !ln_b) return VPE_E_SHAPE;
  if (reinterpret_cast<uintptr_t>(A) % 16 || reinterpret_cast<uintptr_t>(resid) % 16) return VPE_E_SHAPE;
  memset(g, 0, sizeof(*g));
  uint64_t dims[2] = {(uint64_t)K, (uint64_t)M};
  uint64_t strides[1] = {(uint64_t)K * 2};
  uint32_t box[2] = {64u, 128u};
  VPE_TRY(encode_tma(&g->ta, 2, A, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B));
  VPE_TRY(make_b_map(g, W, RL_N, K, K, 128, 64));
  {
    uint64_t rd[2] = {(uint64_t)RL_N, (uint64_t)M};
    uint64_t rs[1] = {(uint64_t)RL_N * 4};
    uint32_t rb[2] = {32u, 32u};
    VPE_TRY(encode_tma_t(&g->tout, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, resid, rd, rs, rb, CU_TENSOR_MAP_SWIZZLE_128B));
  }
  if (xln) VPE_TRY(bf16_rows_map(&g->tx, xln, M, RL_N));
  g->p.ep.kind = EPI_RESID;
  g->p.ep.N = RL_N;
  g->p.ep.bias = bias;
  g->p.ep.scale = ls;
  g->p.ep.resid = resid;
  g->p.ep.ldr = RL_N;
  g->p.ep.out = xln;
  g->p.M = M;
  g->p.kblocks = K / 64;
  g->p.m_tiles = (M + 127) / 128;
  g->p.ln.w = ln_w;
  g->p.ln.b = ln_b;
  g->p.ln.eps = eps;
  g->p.ln.tw = tw;
  g->p.ln.tb = tb;
  g->grid = dim3(g->p.m_tiles < num_sms() ? g->p.m_tiles : num_sms(), 1, 1);
  g->resid_ln = 1;
  g->smem = RlCfg::SMEM;
  return VPE_OK;
}

int launch_gemm_resid_ln(const GemmPlan& g0, __nv_bfloat16* xln, __nv_bfloat16* tap, cudaStream_t s) {
  if (!g0.resid_ln) return VPE_E_SHAPE;
  GemmPlan g = g0;
  if (xln && xln != g0.p.ep.out) {
    VPE_TRY(bf16_rows_map(&g.tx, xln, g.p.M, RL_N));
    g.p.ep.out = xln;
  }
  if (!g.p.ep.out) g.p.ln.w = nullptr;  // no LayerNorm output wanted (tap only)
  g.p.pdl_late = pdl_late();
  CUtensorMap ttap;
  memset(&ttap, 0, sizeof(ttap));
  g.p.ln.tap = tap;
  if (tap) {
    if (!g.p.ln.tw || !g.p.ln.tb) return VPE_E_VALUE;
    VPE_TRY(bf16_rows_map(&ttap, tap, g.p.M, RL_N));
  }
  static OncePerDevice attr_set;
  if (attr_set.first()) {
    cudaFuncSetAttribute(gemm_resid_ln_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RlCfg::SMEM);
    max_smem_carveout(gemm_resid_ln_kernel);
  }
  PdlKind pk(1);
  return launch_k(gemm_resid_ln_kernel, g.grid, dim3(RL_THREADS), RlCfg::SMEM, s, g.ta, g.tb, g.tout, g.tx, ttap,
                  g.p) == cudaSuccess
             ? VPE_OK
             : VPE_E_CUDA;
}

int launch_gemm(const GemmPlan& g, cudaStream_t s) {
  if (g.resid_ln) return launch_gemm_resid_ln(g, nullptr, nullptr, s);
  if (g.up_kc == 4 && g.halo_rt == 4 && g.bn == 32) return launch_up_t<32, 4, 4>(g, s);
  if (g.up_kc == 8 && g.halo_rt == 2 && g.bn == 32) return launch_up_t<32, 8, 2>(g, s);
  if (g.up_kc) return VPE_E_SHAPE;
  if (g.halo_kc) {
#define VPE_LH(BN_, KC_, RT_)                                                         \
  if (g.bn == BN_ && g.halo_kc == KC_ && g.halo_rt == RT_)                            \
    return g.halo_wres ? launch_halo_t<BN_, KC_, RT_, true>(g, s) : launch_halo_t<BN_, KC_, RT_>(g, s);
    VPE_LH(32, 4, 1) VPE_LH(64, 4, 1) VPE_LH(128, 4, 1) VPE_LH(32, 8, 1) VPE_LH(64, 8, 1) VPE_LH(128, 8, 1)
    VPE_LH(32, 4, 4) VPE_LH(32, 8, 2) VPE_LH(64, 8, 2) VPE_LH(128, 8, 2)
#undef VPE_LH
    return VPE_E_SHAPE;
  }
#define VPE_L(BN_, BK_) \
  if (g.bn == BN_ && g.bk == BK_) return launch_t<BN_, BK_>(g, s);
  VPE_L(32, 64) VPE_L(64, 64) VPE_L(128, 64) VPE_L(192, 64) VPE_L(256, 64) VPE_L(32, 32) VPE_L(64, 32)
#undef VPE_L
  return VPE_E_SHAPE;
}

}  // namespace vpe

extern "C" int vpe_debug_gemm_trace(unsigned long long* host, int n) {
  if (!host || n < 0 || n > 4096) return VPE_E_VALUE;
  VPE_CUDA_TRY(cudaMemcpyFromSymbol(host, vpe::g_gemm_trace, n * sizeof(unsigned long long)));
  return VPE_OK;
}
