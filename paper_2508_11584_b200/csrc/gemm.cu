// tcgen05 GEMM engine (see gemm.cuh). sm_100a only.
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstring>

#include "gemm.cuh"
#include "tc.cuh"
#include "util.cuh"

namespace vpe {

// ------------------------------------------------------------------------------------------
// device side
// ------------------------------------------------------------------------------------------
template <int BN, int BK>
struct GemmCfg {
  static constexpr int A_BYTES = 128 * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (BN >= 256) ? 4 : (BN >= 128 ? 4 : 5);
  static constexpr int TMEM_COLS = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
  static constexpr int SWZ_LAYOUT = BK == 64 ? 2 : 4;   // UMMA SWIZZLE_128B / SWIZZLE_64B
  static constexpr int SBO = 8 * BK * 2;                // bytes between 8-row core groups
  static constexpr size_t SMEM = 1024 + (size_t)STAGES * STAGE_BYTES + 256;
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

VPE_DEV float apply_act(float x, int act) {
  if (act == ACT_GELU) return gelu_erf(x);
  if (act == ACT_RELU) return fmaxf(x, 0.f);
  return x;
}

// Epilogue for one thread: one output row (gpix), 32 consecutive columns starting at col0.
VPE_DEV void epilogue32(const EpiParams& ep, int64_t gpix, int col0, float (&v)[32]) {
  const int N = ep.N;
  const bool full = (col0 + 32 <= N);
  if (ep.bias) {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (col0 + j < N) v[j] += __ldg(ep.bias + col0 + j);
  }
  switch (ep.kind) {
    case EPI_BF16:
    case EPI_CONV: {
      __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(ep.out) + gpix * ep.ldo + col0;
      if (ep.kind == EPI_CONV) {
        if (full) {
          if (ep.add1) load_bf16x32_add(ep.add1 + gpix * ep.ldo + col0, v);
          if (ep.add2) load_bf16x32_add(ep.add2 + gpix * ep.ldo + col0, v);
        } else {
          for (int j = 0; j < 32; ++j) {
            if (col0 + j >= N) break;
            if (ep.add1) v[j] += __bfloat162float(ep.add1[gpix * ep.ldo + col0 + j]);
            if (ep.add2) v[j] += __bfloat162float(ep.add2[gpix * ep.ldo + col0 + j]);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = apply_act(v[j], ep.act);
      if (full) {
        store_bf16x32(out, v);
      } else {
        for (int j = 0; j < 32 && col0 + j < N; ++j) out[j] = __float2bfloat16_rn(v[j]);
      }
      if (ep.out_relu) {
        __nv_bfloat16* o2 = ep.out_relu + gpix * ep.ldo + col0;
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j], 0.f);
        if (full) {
          store_bf16x32(o2, v);
        } else {
          for (int j = 0; j < 32 && col0 + j < N; ++j) o2[j] = __float2bfloat16_rn(v[j]);
        }
      }
      break;
    }
    case EPI_RESID: {
      float* r = ep.resid + gpix * ep.ldr + col0;
      if (full) {
        float4* r4 = reinterpret_cast<float4*>(r);
        const float4* s4 = reinterpret_cast<const float4*>(ep.scale + col0);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float4 h = r4[i], s = __ldg(s4 + i);
          h.x += s.x * v[4 * i + 0];
          h.y += s.y * v[4 * i + 1];
          h.z += s.z * v[4 * i + 2];
          h.w += s.w * v[4 * i + 3];
          r4[i] = h;
        }
      } else {
        for (int j = 0; j < 32 && col0 + j < N; ++j) r[j] += ep.scale[col0 + j] * v[j];
      }
      break;
    }
    case EPI_PATCH: {
      const int64_t img = gpix / ep.rows_per_img;
      const int64_t p = gpix - img * ep.rows_per_img;
      float* r = ep.resid + (gpix + img + 1) * ep.ldr + col0;
      const float* pos = ep.pos + (p + 1) * (int64_t)N + col0;
      for (int j = 0; j < 32 && col0 + j < N; ++j) r[j] = v[j] + __ldg(pos + j);
      break;
    }
    case EPI_F32: {
      float* o = reinterpret_cast<float*>(ep.out) + gpix * ep.ldo + col0;
      if (ep.act != ACT_NONE) {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = apply_act(v[j], ep.act);
      }
      if (full) {
        float4* o4 = reinterpret_cast<float4*>(o);
#pragma unroll
        for (int i = 0; i < 8; ++i) o4[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
      } else {
        for (int j = 0; j < 32 && col0 + j < N; ++j) o[j] = v[j];
      }
      break;
    }
    case EPI_CONVT: {
      // gpix indexes the input grid (img, y, x); each group of ct_cout columns is one sub-pixel.
      const int HW = ep.ct_H * ep.ct_W;
      const int64_t img = gpix / HW;
      const int rem = (int)(gpix - img * HW);
      const int y = rem / ep.ct_W, x = rem - (rem / ep.ct_W) * ep.ct_W;
      const int k = ep.ct_k, Wo = ep.ct_W * k, Ho = ep.ct_H * k;
      __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(ep.out);
      for (int j = 0; j < 32; ++j) {
        const int c = col0 + j;
        if (c >= N) break;
        const int s = c / ep.ct_cout, co = c - s * ep.ct_cout;
        const int ky = s / k, kx = s - ky * k;
        const int64_t op = (img * Ho + (int64_t)(y * k + ky)) * Wo + (x * k + kx);
        out[op * ep.ldo + co] = __float2bfloat16_rn(v[j]);
      }
      break;
    }
    case EPI_DEPTH: {
      float pre = ep.b3;
#pragma unroll
      for (int j = 0; j < 32; ++j) pre += fmaxf(v[j], 0.f) * __ldg(ep.w3 + j);
      ep.depth_pre[gpix] = pre;
      ep.depth[gpix] = fmaxf(pre, 0.f) * ep.max_depth;
      break;
    }
    default:
      break;
  }
}

template <int BN, int BK>
__global__ void __launch_bounds__(192, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                   const GemmParams p) {
  using C = GemmCfg<BN, BK>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + C::STAGES * C::B_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tfull + 1);

  const uint32_t warp = warp_id(), lane = lane_id();
  if (warp == 0 && lane == 0) {
    tma_prefetch(&ta);
    tma_prefetch(&tb);
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(tfull, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tslot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  const int n0 = blockIdx.x * BN;
  // tile geometry
  int m0 = 0, img = 0, y0 = 0, x0 = 0;
  if (p.mode == 0) {
    m0 = blockIdx.y * 128;
  } else {
    img = blockIdx.y / p.tiles_per_img;
    const int r = blockIdx.y - img * p.tiles_per_img;
    y0 = (r / p.tiles_x) * p.bh;
    x0 = (r % p.tiles_x) * p.bw;
  }

  if (warp == 0) {
    if (lane == 0) {
      const int half = p.ks / 2;
      for (int kb = 0; kb < p.kblocks; ++kb) {
        const int s = kb % C::STAGES;
        const uint32_t ph = (kb / C::STAGES) & 1;
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
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(128, BN);
      for (int kb = 0; kb < p.kblocks; ++kb) {
        const int s = kb % C::STAGES;
        const uint32_t ph = (kb / C::STAGES) & 1;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t a0 = smem_u32(sA + s * C::A_BYTES);
        const uint32_t b0 = smem_u32(sB + s * C::B_BYTES);
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          const uint64_t ad = smem_desc(a0 + k * 32, 16, C::SBO, C::SWZ_LAYOUT);
          const uint64_t bd = smem_desc(b0 + k * 32, 16, C::SBO, C::SWZ_LAYOUT);
          umma_f16(tmem, ad, bd, idesc, (kb | k) != 0);
        }
        umma_commit(&empty[s]);
      }
      umma_commit(tfull);
    }
  } else {
    // epilogue: warps 2..5 -> TMEM lane quadrant (warp % 4)
    mbar_wait(tfull, 0);
    tc_fence_after();
    const int q = warp & 3;
    const int r = q * 32 + lane;
    int64_t gpix;
    bool valid;
    if (p.mode == 0) {
      gpix = m0 + r;
      valid = gpix < p.M;
    } else {
      const int y = y0 + r / p.bw, x = x0 + r % p.bw;
      valid = (y < p.H) && (x < p.W);
      gpix = ((int64_t)img * p.H + y) * p.W + x;
    }
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      float v[32];
      tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + c0, v);
      tmem_ld_wait();
      if (valid && n0 + c0 < p.ep.N) epilogue32(p.ep, gpix, n0 + c0, v);
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

int encode_tma(CUtensorMap* m, int rank, const void* ptr, const uint64_t* dims, const uint64_t* strides_bytes,
                  const uint32_t* box, CUtensorMapSwizzle swz) {
  if (!tma_available()) return VPE_E_CUDA;
  uint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(ptr), dims, strides_bytes, box,
                        es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    fprintf(stderr, "[vpe] cuTensorMapEncodeTiled failed (%d) rank=%d dims=%llu,%llu box=%u,%u\n", (int)r, rank,
            (unsigned long long)dims[0], (unsigned long long)dims[1], box[0], box[1]);
    return VPE_E_SHAPE;
  }
  return VPE_OK;
}

static int smem_for(int bn, int bk) {
#define VPE_SM(BN_, BK_) \
  if (bn == BN_ && bk == BK_) return (int)GemmCfg<BN_, BK_>::SMEM;
  VPE_SM(32, 64) VPE_SM(64, 64) VPE_SM(128, 64) VPE_SM(256, 64) VPE_SM(32, 32) VPE_SM(64, 32)
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
  g->grid = dim3((N + bn - 1) / bn, (M + 127) / 128, 1);
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
  // spatial tile bw x bh = 128 pixels; pick bw (power of two <= 128) minimising padded width
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
  g->grid = dim3((N + bn - 1) / bn, nimg * g->p.tiles_per_img, 1);
  g->bn = bn;
  g->bk = bk;
  g->smem = smem_for(bn, bk);
  return VPE_OK;
}

template <int BN, int BK>
static int launch_t(const GemmPlan& g, cudaStream_t s) {
  auto k = gemm_tc_kernel<BN, BK>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GemmCfg<BN, BK>::SMEM);
    attr_set = true;
  }
  k<<<g.grid, 192, GemmCfg<BN, BK>::SMEM, s>>>(g.ta, g.tb, g.p);
  return cudaGetLastError() == cudaSuccess ? VPE_OK : VPE_E_CUDA;
}

int launch_gemm(const GemmPlan& g, cudaStream_t s) {
#define VPE_L(BN_, BK_) \
  if (g.bn == BN_ && g.bk == BK_) return launch_t<BN_, BK_>(g, s);
  VPE_L(32, 64) VPE_L(64, 64) VPE_L(128, 64) VPE_L(256, 64) VPE_L(32, 32) VPE_L(64, 32)
#undef VPE_L
  return VPE_E_SHAPE;
}

}  // namespace vpe
