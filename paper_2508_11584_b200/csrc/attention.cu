// Non-causal multi-head attention (head_dim 64) on tcgen05: S = Q K^T and O += P V run on the
// tensor cores with both accumulators in TMEM; softmax runs on 4 warps, one thread per query row;
// O is rescaled in TMEM only when the running max jumps (see the softmax branch below).
// Tried and measured slower on B200 (round 1): a two-Q-tile ping-pong CTA (265 vs 112 us at B=16)
// and S-in-registers with early S release + polynomial exp2 (148 us, register-capped with spills).
//
// Oracle: transformers modeling_dinov2.py:153-178 (eager softmax(QK^T * 1/8) V).
// Q/K/V are read in place from the fused QKV GEMM output [B*T, 3D] through a 2D TMA map
// (box 64 cols x 128 rows), so no head re-layout pass is needed.
#include <cudaTypedefs.h>

#include "attention.cuh"
#include "tc.cuh"
#include "util.cuh"

namespace vpe {

namespace {
constexpr int TILE = 16 * 1024;  // one [128][64] bf16 SW128 tile
// Q + K double-buffered + V single-buffered + P: 96 KB -> two CTAs per SM, so one CTA's
// softmax overlaps the other's tensor-core work (ncu: 1 CTA/SM left the tensor pipe 88% idle)
constexpr int SMEM_ATT = 1024 + TILE /*Q*/ + 2 * TILE /*K*/ + TILE /*V*/ + 2 * TILE /*P*/ + 256;
constexpr int S_COL = 0, O_COL = 128, TMEM_COLS = 256;
}  // namespace

__global__ void __launch_bounds__(192, 2)
    attention_tc_kernel(const __grid_constant__ CUtensorMap tqkv, __nv_bfloat16* __restrict__ out, int T, int D,
                        float scale_log2) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + TILE;
  uint8_t* sV = sK + 2 * TILE;
  uint8_t* sP = sV + TILE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + 2 * TILE);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;   // [2]
  uint64_t* k_empty = bars + 3;  // [2] freed when S_j completes
  uint64_t* v_full = bars + 5;
  uint64_t* v_empty = bars + 6;  // freed when PV_j completes
  uint64_t* s_full = bars + 7;
  uint64_t* p_full = bars + 8;
  uint64_t* o_full = bars + 9;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 10);

  const int qt = blockIdx.x, head = blockIdx.y, b = blockIdx.z;
  const int q0 = qt * 128;
  const int row_base = b * T;
  const int nkv = (T + 127) / 128;
  const uint32_t warp = warp_id(), lane = lane_id();

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tqkv);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    mbar_init(v_full, 1);
    mbar_init(v_empty, 1);
    mbar_init(s_full, 1);
    mbar_init(p_full, 128);
    mbar_init(o_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tslot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(q_full, TILE);
      tma_load_2d(sQ, &tqkv, q_full, head * 64, row_base + q0);
      mbar_expect_tx(&k_full[0], TILE);
      tma_load_2d(sK, &tqkv, &k_full[0], D + head * 64, row_base);
      // order K_{j+1} before V_j: K_{j+1} only waits for S_{j-1}, V_j waits for PV_{j-1}
      for (int j = 0; j < nkv; ++j) {
        if (j + 1 < nkv) {
          const int s = (j + 1) & 1;
          mbar_wait(&k_empty[s], (((j + 1) >> 1) & 1) ^ 1);
          mbar_expect_tx(&k_full[s], TILE);
          tma_load_2d(sK + s * TILE, &tqkv, &k_full[s], D + head * 64, row_base + (j + 1) * 128);
        }
        mbar_wait(v_empty, (j & 1) ^ 1);
        mbar_expect_tx(v_full, TILE);
        tma_load_2d(sV, &tqkv, v_full, 2 * D + head * 64, row_base + j * 128);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_bf16(128, 128);
      constexpr uint32_t idesc_o = idesc_bf16(128, 64, /*b_mn_major=*/true);
      const uint32_t q_addr = smem_u32(sQ);
      mbar_wait(q_full, 0);
      mbar_wait(&k_full[0], 0);
      tc_fence_after();
      {
        const uint32_t k_addr = smem_u32(sK);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          umma_f16(tmem + S_COL, smem_desc(q_addr + k * 32, 16, 1024, 2), smem_desc(k_addr + k * 32, 16, 1024, 2),
                   idesc_s, k > 0);
        umma_commit(s_full);
        umma_commit(&k_empty[0]);
      }
      for (int j = 0; j < nkv; ++j) {
        mbar_wait(p_full, j & 1);
        tc_fence_after();
        if (j + 1 < nkv) {
          const int s1 = (j + 1) & 1;
          mbar_wait(&k_full[s1], ((j + 1) >> 1) & 1);
          tc_fence_after();
          const uint32_t k_addr = smem_u32(sK + s1 * TILE);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_f16(tmem + S_COL, smem_desc(q_addr + k * 32, 16, 1024, 2), smem_desc(k_addr + k * 32, 16, 1024, 2),
                     idesc_s, k > 0);
          umma_commit(s_full);
          umma_commit(&k_empty[s1]);
        }
        mbar_wait(v_full, j & 1);
        tc_fence_after();
        const uint32_t v_addr = smem_u32(sV);
        const uint32_t p_addr = smem_u32(sP);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t pa = p_addr + (k >> 2) * TILE + (k & 3) * 32;
          umma_f16(tmem + O_COL, smem_desc(pa, 16, 1024, 2), smem_desc(v_addr + k * 2048, 1024, 1024, 2), idesc_o,
                   (j | k) > 0);
        }
        umma_commit(o_full);
        umma_commit(v_empty);
      }
    }
  } else {
    // softmax / correction warps: one thread per query row. O accumulates in TMEM across KV
    // blocks (PV_j issued with accumulate=1); the running max used for the exponentials is only
    // raised when a block's max exceeds it by > 8 (log2 units, i.e. p <= 256), and only then is
    // O rescaled in TMEM (tcgen05.ld/st) -- with real data that is once or twice per row.
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const uint32_t lane_addr = tmem + ((uint32_t)(q * 32) << 16);
    float m_used = -INFINITY, l = 0.f;
    uint8_t* prow0 = sP + r * 128;
    for (int j = 0; j < nkv; ++j) {
      mbar_wait(s_full, j & 1);
      tc_fence_after();
      const int kvalid = T - j * 128;  // keys >= kvalid are padding
      // pass 1: block row max
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < 4; c += 2) {
        float t[32], u[32];
        tmem_ld32(lane_addr + S_COL + c * 32, t);
        tmem_ld32(lane_addr + S_COL + (c + 1) * 32, u);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          if (c * 32 + i < kvalid) mx = fmaxf(mx, t[i] * scale_log2);
          if ((c + 1) * 32 + i < kvalid) mx = fmaxf(mx, u[i] * scale_log2);
        }
      }
      // PV_{j-1} must be finished (P buffer free, O stable) before P_j / any O rescale
      if (j > 0) {
        mbar_wait(o_full, (j - 1) & 1);
        tc_fence_after();
      }
      if (mx > m_used + 8.f) {
        const float alpha = fast_exp2(m_used - mx);  // 0 on the first block
        l *= alpha;
        if (j > 0) {
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            float t[32];
            tmem_ld32(lane_addr + O_COL + c * 32, t);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) t[i] *= alpha;
            tmem_st32(lane_addr + O_COL + c * 32, t);
          }
          tmem_st_wait();
        }
        m_used = mx;
      }
      // pass 2: p = exp2(s*scale - m_used), row sum, P_j (bf16) into the UMMA SW128 K-major layout
      float rs = 0.f;
#pragma unroll
      for (int c2 = 0; c2 < 2; ++c2) {  // 64 keys (one P tile) per TMEM wait
        float t[64];
        tmem_ld32(lane_addr + S_COL + c2 * 64, *reinterpret_cast<float(*)[32]>(t));
        tmem_ld32(lane_addr + S_COL + c2 * 64 + 32, *reinterpret_cast<float(*)[32]>(t + 32));
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 64; ++i) {
          t[i] = (c2 * 64 + i < kvalid) ? fast_exp2(fmaf(t[i], scale_log2, -m_used)) : 0.f;
          rs += t[i];
        }
        uint8_t* prow = prow0 + c2 * TILE;
#pragma unroll
        for (int k = 0; k < 8; ++k) {  // 16-byte chunk k of the 128-byte row, SW128 position
          uint4 u;
          u.x = pack_bf16(t[8 * k + 0], t[8 * k + 1]);
          u.y = pack_bf16(t[8 * k + 2], t[8 * k + 3]);
          u.z = pack_bf16(t[8 * k + 4], t[8 * k + 5]);
          u.w = pack_bf16(t[8 * k + 6], t[8 * k + 7]);
          *reinterpret_cast<uint4*>(prow + ((k ^ (r & 7)) << 4)) = u;
        }
      }
      l += rs;
      fence_async_smem();
      tc_fence_before();
      mbar_arrive(p_full);
    }
    mbar_wait(o_full, (nkv - 1) & 1);
    tc_fence_after();
    const int qi = q0 + r;
    const float inv = 1.f / l;
    float t[32], u[32];
    tmem_ld32(lane_addr + O_COL, t);
    tmem_ld32(lane_addr + O_COL + 32, u);
    tmem_ld_wait();
    if (qi < T) {
      uint4* dst = reinterpret_cast<uint4*>(out + (int64_t)(row_base + qi) * D + head * 64);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint4 w;
        w.x = pack_bf16(t[8 * c + 0] * inv, t[8 * c + 1] * inv);
        w.y = pack_bf16(t[8 * c + 2] * inv, t[8 * c + 3] * inv);
        w.z = pack_bf16(t[8 * c + 4] * inv, t[8 * c + 5] * inv);
        w.w = pack_bf16(t[8 * c + 6] * inv, t[8 * c + 7] * inv);
        dst[c] = w;
        uint4 x;
        x.x = pack_bf16(u[8 * c + 0] * inv, u[8 * c + 1] * inv);
        x.y = pack_bf16(u[8 * c + 2] * inv, u[8 * c + 3] * inv);
        x.z = pack_bf16(u[8 * c + 4] * inv, u[8 * c + 5] * inv);
        x.w = pack_bf16(u[8 * c + 6] * inv, u[8 * c + 7] * inv);
        dst[4 + c] = x;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, TMEM_COLS);
  }
}

int plan_attention(AttnPlan* a, const __nv_bfloat16* qkv, __nv_bfloat16* out, int B, int T, int D, int heads) {
  if (D != heads * 64) return VPE_E_SHAPE;
  uint64_t dims[2] = {(uint64_t)(3 * D), (uint64_t)B * T};
  uint64_t strides[1] = {(uint64_t)3 * D * 2};
  uint32_t box[2] = {64u, 128u};
  int rc = encode_tma(&a->tqkv, 2, qkv, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  a->out = out;
  a->B = B;
  a->T = T;
  a->D = D;
  a->heads = heads;
  return VPE_OK;
}

int launch_attention(const AttnPlan& a, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attention_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_ATT);
    attr = true;
  }
  dim3 grid((a.T + 127) / 128, a.heads, a.B);
  const float scale_log2 = 0.125f * 1.4426950408889634f;
  attention_tc_kernel<<<grid, 192, SMEM_ATT, s>>>(a.tqkv, a.out, a.T, a.D, scale_log2);
  return cudaGetLastError() == cudaSuccess ? VPE_OK : VPE_E_CUDA;
}

}  // namespace vpe
