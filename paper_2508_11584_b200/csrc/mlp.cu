// Fused DINOv2 MLP block on tcgen05 (modeling_dinov2.py:312-328 + the LayerScale residual of
// :378-386):  resid += ls2 * (GELU(X W1^T + b1) W2^T + b2)  with X = LN2(resid) [M, D].
//
// The hidden activation [M, 4D] never leaves the SM. A CTA owns a 128-row block of X, keeps it
// resident in shared memory, and walks the hidden dimension in 64-wide chunks:
//   H_i = X W1[64i:64i+64]^T          (TMEM, double-buffered, N = 64)
//   P_i = bf16(GELU(H_i + b1))        (epilogue warps -> smem, UMMA SW128 K-major layout)
//   O  += P_i W2[:, 64i:64i+64]^T     (TMEM, N = D as two MMAs of D/2)
// so the separate FC1 -> HBM/L2 -> FC2 round trip (2 x 50 MB at C2) and the FC1 output stores
// that stall the next tile's TMA loads (profiles/round1_ubench.md) disappear.
//   warp 0      TMA producer: X once per block; W1 boxes (64 K x 64 rows) through a 6-slot ring,
//               W2 boxes (64 K x D/2 rows) through a 2-slot ring, in MMA consumption order
//   warp 1      MMA issuer: H_0, H_1, O_0, H_2, O_1, ... (H_{i+1} overlaps the GELU of H_i)
//   warps 2-9   epilogue: 2 warps per TMEM lane quadrant (32 hidden columns each); at the end of a
//               block the O accumulator goes straight into the fp32 residual (vector reductions)
// Requires D == 384 (ViT-S: TMEM = O 384 + 2 x 64 H columns = 512) and hidden % 64 == 0.
#include <cudaTypedefs.h>

#include <cstdlib>

#include "gemm.cuh"
#include "mlp.cuh"
#include "tc.cuh"
#include "util.cuh"

namespace vpe {

namespace {
constexpr int MD = 384;                 // model width handled by this kernel
constexpr int HC = 64;                  // hidden chunk
constexpr int KB = MD / 64;             // 64-wide K blocks of X (6)
constexpr int X_BYTES = 128 * MD * 2;   // 96 KB resident A block
constexpr int W1_BOX = HC * 64 * 2;     // 8 KB
constexpr int W1_SLOTS = 6;
constexpr int W2_BOX = (MD / 2) * 64 * 2;  // 24 KB
constexpr int W2_SLOTS = 2;
constexpr int P_BYTES = 128 * HC * 2;   // 16 KB
constexpr int MLP_THREADS = 64 + 32 * 8;
constexpr int SMEM_MLP = 1024 + X_BYTES + W1_SLOTS * W1_BOX + W2_SLOTS * W2_BOX + 2 * P_BYTES + 512;
constexpr uint32_t O_COL = 0, H_COL = 384;
}  // namespace

VPE_DEV void add_bias32(float (&v)[32], const float* __restrict__ b) {
  const float4* b4 = reinterpret_cast<const float4*>(b);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float4 x = __ldg(b4 + i);
    v[4 * i] += x.x;
    v[4 * i + 1] += x.y;
    v[4 * i + 2] += x.z;
    v[4 * i + 3] += x.w;
  }
}

VPE_DEV void red_add_v4f(float* dst, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

__device__ unsigned long long g_mlp_trace[4096];
#define MLP_TRACE(code)                                                              \
  do {                                                                               \
    if (trace && blockIdx.x == 0 && tn < 2040) {                                     \
      g_mlp_trace[2 * tn] = (unsigned long long)(code);                              \
      g_mlp_trace[2 * tn + 1] = (unsigned long long)clock64();                       \
      ++tn;                                                                          \
    }                                                                                \
  } while (0)

__global__ void __launch_bounds__(MLP_THREADS, 1)
    mlp_fused_kernel(const __grid_constant__ CUtensorMap tx, const __grid_constant__ CUtensorMap tw1,
                     const __grid_constant__ CUtensorMap tw2, const float* __restrict__ b1,
                     const float* __restrict__ b2, const float* __restrict__ ls2, float* __restrict__ resid,
                     int M, int hidden, int trace) {
  extern __shared__ uint8_t smem_raw[];
  int tn = 0;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sX = smem;                          // KB boxes of [128 rows][64] SW128
  uint8_t* sW1 = sX + X_BYTES;                 // [W1_SLOTS][64 rows][64] SW128
  uint8_t* sW2 = sW1 + W1_SLOTS * W1_BOX;      // [W2_SLOTS][192 rows][64] SW128
  uint8_t* sP = sW2 + W2_SLOTS * W2_BOX;       // [2][128 rows][64] SW128
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + 2 * P_BYTES);
  uint64_t* x_full = bars;
  uint64_t* x_empty = bars + 1;
  uint64_t* w1_full = bars + 2;                 // [W1_SLOTS]
  uint64_t* w1_empty = w1_full + W1_SLOTS;      // [W1_SLOTS]
  uint64_t* w2_full = w1_empty + W1_SLOTS;      // [W2_SLOTS]
  uint64_t* w2_empty = w2_full + W2_SLOTS;      // [W2_SLOTS]
  uint64_t* h_full = w2_empty + W2_SLOTS;       // [2]
  uint64_t* h_empty = h_full + 2;               // [2]
  uint64_t* p_full = h_empty + 2;               // [2]
  uint64_t* p_empty = p_full + 2;               // [2]
  uint64_t* o_full = p_empty + 2;
  uint64_t* o_empty = o_full + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(o_empty + 1);

  const uint32_t warp = warp_id(), lane = lane_id();
  const int nblk = (M + 127) / 128;
  const int nch = hidden / HC;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tx);
    tma_prefetch(&tw1);
    tma_prefetch(&tw2);
    mbar_init(x_full, 1);
    mbar_init(x_empty, 1);
    for (int i = 0; i < W1_SLOTS; ++i) {
      mbar_init(&w1_full[i], 1);
      mbar_init(&w1_empty[i], 1);
    }
    for (int i = 0; i < W2_SLOTS; ++i) {
      mbar_init(&w2_full[i], 1);
      mbar_init(&w2_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&h_full[i], 1);
      mbar_init(&h_empty[i], 8);
      mbar_init(&p_full[i], 8);
      mbar_init(&p_empty[i], 1);
    }
    mbar_init(o_full, 1);
    mbar_init(o_empty, 8);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  pdl_wait();
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      int n1 = 0, n2 = 0, nb = 0;
      auto load_w1 = [&](int chunk) {
        for (int k = 0; k < KB; ++k, ++n1) {
          const int s = n1 % W1_SLOTS;
          mbar_wait(&w1_empty[s], ((n1 / W1_SLOTS) & 1) ^ 1);
          mbar_expect_tx(&w1_full[s], W1_BOX);
          tma_load_2d(sW1 + s * W1_BOX, &tw1, &w1_full[s], k * 64, chunk * HC);
        }
      };
      auto load_w2 = [&](int chunk) {
        for (int h = 0; h < 2; ++h, ++n2) {
          const int s = n2 % W2_SLOTS;
          mbar_wait(&w2_empty[s], ((n2 / W2_SLOTS) & 1) ^ 1);
          mbar_expect_tx(&w2_full[s], W2_BOX);
          tma_load_2d(sW2 + s * W2_BOX, &tw2, &w2_full[s], chunk * HC, h * (MD / 2));
        }
      };
      for (int blk = blockIdx.x; blk < nblk; blk += gridDim.x, ++nb) {
        mbar_wait(x_empty, (nb & 1) ^ 1);
        mbar_expect_tx(x_full, X_BYTES);
        for (int k = 0; k < KB; ++k) tma_load_2d(sX + k * (128 * 128), &tx, x_full, k * 64, blk * 128);
        for (int i = 0; i < nch; ++i) {
          load_w1(i);
          if (i > 0) load_w2(i - 1);
        }
        load_w2(nch - 1);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_h = idesc_bf16(128, HC);
      constexpr uint32_t idesc_o = idesc_bf16(128, MD / 2);
      int n1 = 0, n2 = 0, nb = 0, gh = 0, go = 0;  // gh/go: global H / O chunk counters
      for (int blk = blockIdx.x; blk < nblk; blk += gridDim.x, ++nb) {
        mbar_wait(x_full, nb & 1);
        tc_fence_after();
        auto issue_h = [&](int i) {
          const int hb = gh & 1;
          MLP_TRACE(100 + i);
          mbar_wait(&h_empty[hb], ((gh >> 1) & 1) ^ 1);  // epilogue has read H from 2 chunks ago
          tc_fence_after();
          MLP_TRACE(200 + i);
          const uint32_t d = tmem + H_COL + hb * HC;
          for (int k = 0; k < KB; ++k, ++n1) {
            const int s = n1 % W1_SLOTS;
            mbar_wait(&w1_full[s], (n1 / W1_SLOTS) & 1);
            tc_fence_after();
            if (k == 0) MLP_TRACE(300 + i);
            const uint32_t a0 = smem_u32(sX + k * (128 * 128));
            const uint32_t b0 = smem_u32(sW1 + s * W1_BOX);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              umma_f16(d, smem_desc(a0 + kk * 32, 16, 1024, 2), smem_desc(b0 + kk * 32, 16, 1024, 2), idesc_h,
                       (k | kk) != 0);
            umma_commit(&w1_empty[s]);
          }
          umma_commit(&h_full[hb]);
          if (i == nch - 1) umma_commit(x_empty);  // every H of the block issued: X may be replaced
          ++gh;
        };
        auto issue_o = [&](int j) {
          const int pb = go & 1;
          if (j == 0) {  // the previous block's O has been read out
            mbar_wait(o_empty, (nb & 1) ^ 1);
            tc_fence_after();
          }
          MLP_TRACE(400 + j);
          mbar_wait(&p_full[pb], (go >> 1) & 1);
          tc_fence_after();
          MLP_TRACE(500 + j);
          const uint32_t a0 = smem_u32(sP + pb * P_BYTES);
          for (int h = 0; h < 2; ++h, ++n2) {
            const int s = n2 % W2_SLOTS;
            mbar_wait(&w2_full[s], (n2 / W2_SLOTS) & 1);
            tc_fence_after();
            if (h == 0) MLP_TRACE(600 + j);
            const uint32_t b0 = smem_u32(sW2 + s * W2_BOX);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              umma_f16(tmem + O_COL + h * (MD / 2), smem_desc(a0 + kk * 32, 16, 1024, 2),
                       smem_desc(b0 + kk * 32, 16, 1024, 2), idesc_o, (j | kk) != 0);
            umma_commit(&w2_empty[s]);
          }
          umma_commit(&p_empty[pb]);
          ++go;
        };
        for (int i = 0; i < nch; ++i) {
          issue_h(i);
          if (i > 0) issue_o(i - 1);
        }
        issue_o(nch - 1);
        umma_commit(o_full);
      }
    }
  } else {
    // epilogue warps: quadrant q = warp % 4 (TMEM lanes), half hh = which 32 of the 64 hidden
    // columns (and which 192 of the 384 output columns)
    const int e = (int)warp - 2;
    const int q = warp & 3, hh = e >> 2;
    const int r = q * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    int gh = 0, nb = 0;
    for (int blk = blockIdx.x; blk < nblk; blk += gridDim.x, ++nb) {
      for (int i = 0; i < nch; ++i, ++gh) {
        const int hb = gh & 1;
        mbar_wait(&h_full[hb], (gh >> 1) & 1);
        tc_fence_after();
        float v[32];
        tmem_ld32(lane_base + H_COL + hb * HC + hh * 32, v);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&h_empty[hb]);
        add_bias32(v, b1 + i * HC + hh * 32);
        gelu_poly32(v);
        // P_i rows in the UMMA SW128 K-major layout: 128-B rows, 16-B chunk c at slot c ^ (row & 7)
        mbar_wait(&p_empty[hb], ((gh >> 1) & 1) ^ 1);  // O of two chunks ago has read this buffer
        uint8_t* prow = sP + hb * P_BYTES + r * 128;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int c = hh * 4 + j;
          uint4 u;
          u.x = pack_bf16(v[8 * j + 0], v[8 * j + 1]);
          u.y = pack_bf16(v[8 * j + 2], v[8 * j + 3]);
          u.z = pack_bf16(v[8 * j + 4], v[8 * j + 5]);
          u.w = pack_bf16(v[8 * j + 6], v[8 * j + 7]);
          *reinterpret_cast<uint4*>(prow + ((c ^ (r & 7)) << 4)) = u;
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[hb]);
      }
      // block done: resid[rows] += ls2 * (O + b2)
      mbar_wait(o_full, nb & 1);
      tc_fence_after();
      const int64_t row = (int64_t)blk * 128 + r;
#pragma unroll 1
      for (int c = 0; c < 6; ++c) {
        const int col0 = hh * (MD / 2) + c * 32;
        float o[32];
        tmem_ld32(lane_base + O_COL + col0, o);
        tmem_ld_wait();
        if (c == 5) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(o_empty);
        }
        if (row < M) {
          float* dst = resid + row * MD + col0;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const float4 bb = __ldg(reinterpret_cast<const float4*>(b2 + col0) + k);
            const float4 ll = __ldg(reinterpret_cast<const float4*>(ls2 + col0) + k);
            red_add_v4f(dst + 4 * k, ll.x * (o[4 * k] + bb.x), ll.y * (o[4 * k + 1] + bb.y),
                        ll.z * (o[4 * k + 2] + bb.z), ll.w * (o[4 * k + 3] + bb.w));
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

int plan_mlp(MlpPlan* m, const __nv_bfloat16* X, int M, int D, int hidden, const __nv_bfloat16* W1, const float* b1,
             const __nv_bfloat16* W2, const float* b2, const float* ls2, float* resid) {
  if (D != MD || hidden % HC || hidden < 2 * HC) return VPE_E_SHAPE;
  if (reinterpret_cast<uintptr_t>(X) % 16 || reinterpret_cast<uintptr_t>(W1) % 16 ||
      reinterpret_cast<uintptr_t>(W2) % 16 || reinterpret_cast<uintptr_t>(resid) % 16)
    return VPE_E_SHAPE;
  {
    uint64_t dims[2] = {(uint64_t)D, (uint64_t)M};
    uint64_t strides[1] = {(uint64_t)D * 2};
    uint32_t box[2] = {64u, 128u};
    VPE_TRY(encode_tma(&m->tx, 2, X, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B));
  }
  {
    uint64_t dims[2] = {(uint64_t)D, (uint64_t)hidden};
    uint64_t strides[1] = {(uint64_t)D * 2};
    uint32_t box[2] = {64u, (uint32_t)HC};
    VPE_TRY(encode_tma(&m->tw1, 2, W1, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B));
  }
  {
    uint64_t dims[2] = {(uint64_t)hidden, (uint64_t)D};
    uint64_t strides[1] = {(uint64_t)hidden * 2};
    uint32_t box[2] = {64u, (uint32_t)(D / 2)};
    VPE_TRY(encode_tma(&m->tw2, 2, W2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B));
  }
  m->b1 = b1;
  m->b2 = b2;
  m->ls2 = ls2;
  m->resid = resid;
  m->M = M;
  m->hidden = hidden;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int nblk = (M + 127) / 128;
  m->grid = nblk < sms ? nblk : sms;
  return VPE_OK;
}

int launch_mlp(const MlpPlan& m, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(mlp_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_MLP);
    attr = true;
  }
  static int trace = -1;
  if (trace < 0) {
    const char* e = getenv("VPE_MLP_TRACE");
    trace = (e && e[0] == '1') ? 1 : 0;
  }
  mlp_fused_kernel<<<m.grid, MLP_THREADS, SMEM_MLP, s>>>(m.tx, m.tw1, m.tw2, m.b1, m.b2, m.ls2, m.resid, m.M,
                                                          m.hidden, trace);
  return cudaGetLastError() == cudaSuccess ? VPE_OK : VPE_E_CUDA;
}

}  // namespace vpe

extern "C" int vpe_debug_mlp_trace(unsigned long long* host, int n) {
  if (!host || n < 0 || n > 4096) return VPE_E_VALUE;
  VPE_CUDA_TRY(cudaMemcpyFromSymbol(host, vpe::g_mlp_trace, n * sizeof(unsigned long long)));
  return VPE_OK;
}
