// Ping-pong attention on tcgen05 (head_dim 64, non-causal): one CTA owns TWO 128-query tiles of a
// (image, head) and two softmax warpgroups, so while warpgroup 0 turns S0_j into P0_j the tensor
// core computes S1_j / PV1_{j-1} and vice versa (the FA4 structure, specialised to ViT shapes).
//
//   warp 0      TMA: Q0,Q1 once; K_j / V_j double-buffered
//   warp 1      tcgen05.mma issuer: S_g = Q_g K_j^T (TMEM), O_g += P_g V_j (TMEM, accumulate)
//   warps 2-5   softmax WG0 (rows of tile 0), warps 6-9 softmax WG1 (tile 1); one thread per row
//
// TMEM: S0 [0,128) S1 [128,256) O0 [256,320) O1 [320,384). O stays in TMEM across KV blocks; the
// running max used for the exponentials only moves when a block max exceeds it by > 8 (log2), and
// only then is O rescaled in place. Half of each row's exponentials run on the FMA pipe (degree-3
// polynomial 2^f, rel. err 1.7e-4, below P's bf16 rounding) to balance the MUFU (ncu: XU 41%).
// Oracle: transformers modeling_dinov2.py:153-178.
#include <cudaTypedefs.h>

#include "attention.cuh"
#include "tc.cuh"
#include "util.cuh"

namespace vpe {

namespace {
constexpr int TILE = 16 * 1024;  // one [128][64] bf16 SW128 tile
constexpr int SMEM_PP = 1024 + 2 * TILE /*Q0,Q1*/ + 2 * TILE /*K*/ + 2 * TILE /*V*/ + 4 * TILE /*P0,P1*/ + 512;
constexpr int PP_THREADS = 320;

// 2^x on the FMA/ALU pipes: 2^floor(x) * p(frac(x)), p(f) ~ 2^f (degree 3, max rel err 1.7e-4)
VPE_DEV float exp2_poly(float x) {
  x = fmaxf(x, -126.f);
  const float xi = floorf(x);
  const float f = x - xi;
  float p = fmaf(0.07632499f, f, 0.22830876f);
  p = fmaf(p, f, 0.69503605f);
  p = fmaf(p, f, 1.0f);
  return __int_as_float(__float_as_int(p) + (static_cast<int>(xi) << 23));
}
}  // namespace

__global__ void __launch_bounds__(PP_THREADS, 1)
    attention_pp_kernel(const __grid_constant__ CUtensorMap tqkv, __nv_bfloat16* __restrict__ out, int T, int D,
                        float scale_log2) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;              // [2] tiles
  uint8_t* sK = sQ + 2 * TILE;     // [2]
  uint8_t* sV = sK + 2 * TILE;     // [2]
  uint8_t* sP = sV + 2 * TILE;     // [2 groups][2 tiles]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + 4 * TILE);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;   // [2]
  uint64_t* k_empty = bars + 3;  // [2]
  uint64_t* v_full = bars + 5;   // [2]
  uint64_t* v_empty = bars + 7;  // [2]
  uint64_t* s_full = bars + 9;   // [2 groups]
  uint64_t* p_full = bars + 11;  // [2 groups]
  uint64_t* o_full = bars + 13;  // [2 groups]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 15);

  const int pair = blockIdx.x, head = blockIdx.y, b = blockIdx.z;
  const int q0 = pair * 256;
  const int row_base = b * T;
  const int nkv = (T + 127) / 128;
  const bool has1 = q0 + 128 < T;  // second tile holds at least one query
  const uint32_t warp = warp_id(), lane = lane_id();

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tqkv);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 128);
      mbar_init(&o_full[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(q_full, has1 ? 2 * TILE : TILE);
      tma_load_2d(sQ, &tqkv, q_full, head * 64, row_base + q0);
      if (has1) tma_load_2d(sQ + TILE, &tqkv, q_full, head * 64, row_base + q0 + 128);
      mbar_expect_tx(&k_full[0], TILE);
      tma_load_2d(sK, &tqkv, &k_full[0], D + head * 64, row_base);
      for (int j = 0; j < nkv; ++j) {
        if (j + 1 < nkv) {
          const int s = (j + 1) & 1;
          mbar_wait(&k_empty[s], (((j + 1) >> 1) & 1) ^ 1);
          mbar_expect_tx(&k_full[s], TILE);
          tma_load_2d(sK + s * TILE, &tqkv, &k_full[s], D + head * 64, row_base + (j + 1) * 128);
        }
        const int sv = j & 1;
        mbar_wait(&v_empty[sv], ((j >> 1) & 1) ^ 1);
        mbar_expect_tx(&v_full[sv], TILE);
        tma_load_2d(sV + sv * TILE, &tqkv, &v_full[sv], 2 * D + head * 64, row_base + j * 128);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_bf16(128, 128);
      constexpr uint32_t idesc_o = idesc_bf16(128, 64, /*b_mn_major=*/true);
      const int ng = has1 ? 2 : 1;
      auto issue_s = [&](int g, int ks) {
        const uint32_t qa = smem_u32(sQ + g * TILE), ka = smem_u32(sK + ks * TILE);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          umma_f16(tmem + g * 128, smem_desc(qa + k * 32, 16, 1024, 2), smem_desc(ka + k * 32, 16, 1024, 2), idesc_s,
                   k > 0);
        umma_commit(&s_full[g]);
      };
      auto issue_pv = [&](int g, int vs, int j) {
        const uint32_t va = smem_u32(sV + vs * TILE), pa0 = smem_u32(sP + g * 2 * TILE);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t pa = pa0 + (k >> 2) * TILE + (k & 3) * 32;
          umma_f16(tmem + 256 + g * 64, smem_desc(pa, 16, 1024, 2), smem_desc(va + k * 2048, 1024, 1024, 2), idesc_o,
                   (j | k) > 0);
        }
        umma_commit(&o_full[g]);
      };
      mbar_wait(q_full, 0);
      mbar_wait(&k_full[0], 0);
      tc_fence_after();
      for (int g = 0; g < ng; ++g) issue_s(g, 0);
      umma_commit(&k_empty[0]);
      for (int j = 0; j < nkv; ++j) {
        const int vs = j & 1, ks1 = (j + 1) & 1;
        mbar_wait(&v_full[vs], (j >> 1) & 1);
        if (j + 1 < nkv) mbar_wait(&k_full[ks1], ((j + 1) >> 1) & 1);
        for (int g = 0; g < ng; ++g) {
          mbar_wait(&p_full[g], j & 1);  // P_g,j written, S_g,j consumed, O_g stable
          tc_fence_after();
          issue_pv(g, vs, j);
          if (j + 1 < nkv) issue_s(g, ks1);
        }
        if (j + 1 < nkv) umma_commit(&k_empty[ks1]);
        umma_commit(&v_empty[vs]);
      }
    }
  } else {
    // softmax warpgroup g (warps 2-5 -> g=0, 6-9 -> g=1); TMEM lane quadrant = warp % 4
    const int g = (warp - 2) >> 2;
    if (g == 1 && !has1) goto done;
    {
      const int q = warp & 3;
      const int r = q * 32 + lane;
      const uint32_t lane_addr = tmem + ((uint32_t)(q * 32) << 16);
      const uint32_t S_COL = g * 128, O_COL = 256 + g * 64;
      float m_used = -INFINITY, l = 0.f;
      uint8_t* prow0 = sP + g * 2 * TILE + r * 128;
      for (int j = 0; j < nkv; ++j) {
        mbar_wait(&s_full[g], j & 1);
        tc_fence_after();
        const int kvalid = T - j * 128;
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
        if (j > 0) {
          mbar_wait(&o_full[g], (j - 1) & 1);
          tc_fence_after();
        }
        if (mx > m_used + 8.f) {
          const float alpha = fast_exp2(m_used - mx);
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
        float rs = 0.f;
#pragma unroll
        for (int c2 = 0; c2 < 2; ++c2) {
          float t[64];
          tmem_ld32(lane_addr + S_COL + c2 * 64, *reinterpret_cast<float(*)[32]>(t));
          tmem_ld32(lane_addr + S_COL + c2 * 64 + 32, *reinterpret_cast<float(*)[32]>(t + 32));
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 64; ++i) {
            const float x = fmaf(t[i], scale_log2, -m_used);
            const float e = (i < 32) ? fast_exp2(x) : exp2_poly(x);
            t[i] = (c2 * 64 + i < kvalid) ? e : 0.f;
            rs += t[i];
          }
          uint8_t* prow = prow0 + c2 * TILE;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
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
        mbar_arrive(&p_full[g]);
      }
      mbar_wait(&o_full[g], (nkv - 1) & 1);
      tc_fence_after();
      const int qi = q0 + g * 128 + r;
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
  }
done:
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

int launch_attention_pp(const AttnPlan& a, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attention_pp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_PP);
    attr = true;
  }
  dim3 grid((a.T + 255) / 256, a.heads, a.B);
  const float scale_log2 = 0.125f * 1.4426950408889634f;
  attention_pp_kernel<<<grid, PP_THREADS, SMEM_PP, s>>>(a.tqkv, a.out, a.T, a.D, scale_log2);
  return cudaGetLastError() == cudaSuccess ? VPE_OK : VPE_E_CUDA;
}

}  // namespace vpe
