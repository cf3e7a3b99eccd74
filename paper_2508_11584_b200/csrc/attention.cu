// Non-causal multi-head attention (head_dim 64) on tcgen05, one persistent CTA per SM.
//
// Oracle: transformers modeling_dinov2.py:153-178 (eager softmax(QK^T * 1/8) V).
// Q/K/V are read in place from the fused QKV GEMM output [B*T, 3D] through one 2D TMA map
// (box 64 cols x 128 rows), so no head re-layout pass is needed.
//
// Work unit = (image, head, pair of 128-row Q tiles). The two Q tiles share every K/V tile the
// producer brings in, and run ping-pong on the tensor core:
//   warp 0      TMA producer: Q_A, Q_B per unit (double-buffered across units), then K_j / V_j
//               through 3-stage rings
//   warps 1, 2  MMA issuers, one per Q slot X: S_X(j+1) = Q_X K_{j+1}^T as soon as softmax X has
//               pulled S_X(j) into registers; O_X += P_X(j) V_j with P read from TMEM (.kind::f16
//               A-from-TMEM), so P never touches shared memory
//   warps 3-10  softmax A, warps 11-18 softmax B: two warps per 32 query rows, one per 64-key
//               half of each S tile; the pair agrees on the row max through smem + a named
//               barrier (pass 1), then p = 2^(s*scale - m) is written to TMEM as bf16 pairs
//               (pass 2). The two slots' exponential passes alternate (mbarrier token
//               A(j) -> B(j) -> A(j+1)), so one slot's max pass runs under the other slot's MUFU
//               work. O is rescaled in TMEM only when the running max rises by > 8 (log2), i.e.
//               almost never after the first KV tile. (Holding the whole 64-key half in
//               registers to read S once needs ~110 registers; at 608 threads ptxas caps at 96
//               and spills the scores: 2x slower, measured.)
// TMEM (512 columns): S_A | S_B | P_A | P_B | O_A | O_B.
// Rows/keys past T (tail tiles) are computed on whatever the TMA brought (the next image's rows
// or zero fill) and masked: invalid keys get p = 0, invalid rows are never stored, and warps whose
// 32 rows are all past T skip the exponentials.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <utility>
#include <vector>

#include "attention.cuh"
#include "tc.cuh"
#include "util.cuh"

namespace vpe {

namespace {
constexpr int TILE = 16 * 1024;  // one [128][64] bf16 SW128 tile
constexpr int KS = 3, VS = 3;    // K / V ring depth
constexpr int ATT_THREADS = 608;  // 0 TMA, 1-2 MMA (slot A / B), 3-10 softmax A, 11-18 softmax B
constexpr int XCH_BYTES = 2 * 3 * 2 * 128 * 4;  // row max / sum exchange [slot][tile parity | epi][half][row]
constexpr int SMEM_ATT = 1024 + 4 * TILE /*Q_A,Q_B x 2 units*/ + KS * TILE + VS * TILE + XCH_BYTES + 512;
constexpr uint32_t S_COL = 0, P_COL = 256, O_COL = 384;
}  // namespace

VPE_DEV void tmem_st32u(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),
      "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),
      "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

VPE_DEV void tmem_st16u(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

VPE_DEV void tmem_st4u(uint32_t taddr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}

// O[tmem] (+)= A[tmem] * B[smem], kind::f16; A (M x K, K-major, 2 bf16 per 32-bit column)
VPE_DEV void umma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// ---- softmax arithmetic: f32x2 SIMD (FFMA2/FADD2), 3-input max, exp2 split between MUFU and an
// FMA-pipe polynomial, bf16 packing by byte permute (no F2FP on the XU pipe).
VPE_DEV float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// tcgen05.wait::ld that also ties the loaded registers, so no use of them can be scheduled
// above the wait
VPE_DEV void tmem_ld_wait_dep(float (&v)[32]) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                 "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),
                 "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
               :
               : "memory");
}

VPE_DEV float chunk_max_log2(const float (&v)[32], float scale_log2) {
  float m0 = fmax3(v[0], v[1], v[2]), m1 = fmax3(v[3], v[4], v[5]);
#pragma unroll
  for (int i = 6; i < 30; i += 4) {
    m0 = fmax3(m0, v[i], v[i + 1]);
    m1 = fmax3(m1, v[i + 2], v[i + 3]);
  }
  return fmax3(m0, m1, fmaxf(v[30], v[31])) * scale_log2;
}

// 2^x for a pair on the FMA pipe: x = n + f (n = rint(x), |f| <= 1/2), 2^f by a cubic (max rel.
// error 1.4e-4, far below the bf16 rounding of P), 2^n by adding n to the exponent field of each
// 32-bit half (two IMADs; a 64-bit shift/or cost six instructions). Valid for x < 128; x is
// clamped at -126 (p(f) may be just below 1, so n = -127 would borrow into the sign bit: NaN).
VPE_DEV uint64_t exp2_poly2(uint64_t x) {
  float x0, x1;
  f2_unpack(x, x0, x1);
  x = f2_pack(fmaxf(x0, -126.f), fmaxf(x1, -126.f));
  const float kMagic = 12582912.f;  // 1.5 * 2^23: x + kMagic holds rint(x) in its low mantissa bits
  const uint64_t j = fadd2(x, f2_pack(kMagic, kMagic));
  const uint64_t nf = fadd2(j, f2_pack(-kMagic, -kMagic));
  const uint64_t f = ffma2(nf, f2_pack(-1.f, -1.f), x);
  uint64_t p = ffma2(f, f2_pack(0.05502927f, 0.05502927f), f2_pack(0.24225698f, 0.24225698f));
  p = ffma2(p, f, f2_pack(0.69325305f, 0.69325305f));
  p = ffma2(p, f, f2_pack(0.99995134f, 0.99995134f));
  uint32_t jl, jh, pl, ph;
  asm("mov.b64 {%0, %1}, %2;" : "=r"(jl), "=r"(jh) : "l"(j));
  asm("mov.b64 {%0, %1}, %2;" : "=r"(pl), "=r"(ph) : "l"(p));
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(pl + (jl << 23)), "r"(ph + (jh << 23)));
  return r;
}

// P in bf16 by truncation (one PRMT per pair). The exponent offset carries +log2(1 + 0.00282),
// the mean relative truncation loss of bf16, so the kept P is unbiased; l is corrected by the
// same factor in the epilogue.
constexpr float kTruncBias = 0.0040625f;     // log2(1.00282)
constexpr float kTruncScale = 1.00282f;

// p = 2^(v*scale - m) for one 32-key chunk -> 16 bf16 pairs in TMEM at p_taddr; returns the
// chunk's f32x2 partial sums. poly_ok: chunk has no masked (-inf) keys.
template <int kPolyMask, bool kPolyOk>  // pairs (of 16 per chunk) whose exp2 runs on the FMA pipe
VPE_DEV uint64_t emit_chunk(const float (&v)[32], float scale_log2, float m_used, uint32_t p_taddr) {
  const uint64_t sc2 = f2_pack(scale_log2, scale_log2);
  const float mb = kTruncBias - m_used;
  const uint64_t mb2 = f2_pack(mb, mb);
  uint64_t acc0 = 0, acc1 = 0;
  // P leaves in groups of 4 pairs (x4 stores): 4 live packed registers instead of 16
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    uint32_t pk[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = 4 * g + q;
      const uint64_t xx = ffma2(f2_pack(v[2 * i], v[2 * i + 1]), sc2, mb2);
      uint64_t pp;
      if (kPolyOk && ((kPolyMask >> i) & 1)) {
        pp = exp2_poly2(xx);
      } else {
        float x0, x1;
        f2_unpack(xx, x0, x1);
        pp = f2_pack(fast_exp2(x0), fast_exp2(x1));
      }
      if (i & 1) acc1 = fadd2(acc1, pp); else acc0 = fadd2(acc0, pp);
      pk[q] = __byte_perm((uint32_t)pp, (uint32_t)(pp >> 32), 0x7632);
    }
    tmem_st4u(p_taddr + 4 * g, pk[0], pk[1], pk[2], pk[3]);
  }
  return fadd2(acc0, acc1);
}

// ---- optional timeline trace of CTA 0 (diagnostics only: VPE_ATT_TRACE=1, read back with
// vpe_debug_att_trace). Slots: [0,2048) MMA thread, [2048,3072) softmax A, [3072,4096) softmax B;
// each event = (code, clock64).
__device__ unsigned long long g_att_trace[4096];
static int g_att_trace_on = -1;
#ifdef VPE_TRACE_BUILD
#define ATT_TRACE(slot_base, idx, code)                                              \
  do {                                                                               \
    if ((trace & 1) && blockIdx.x == 0 && (idx) < 510) {                             \
      g_att_trace[(slot_base) + 2 * (idx)] = (unsigned long long)(code);             \
      g_att_trace[(slot_base) + 2 * (idx) + 1] = (unsigned long long)clock64();      \
      ++(idx);                                                                       \
    }                                                                                \
  } while (0)
#else
#define ATT_TRACE(slot_base, idx, code) \
  do {                                  \
  } while (0)
#endif

struct AttnUnit {
  int b, h, q0, has_b;
};

VPE_DEV AttnUnit unit_of(int u, int BH, int heads, int T, int single) {
  // pair-major ordering: every (image, head) pair-0 first, ..., so the (cheap) tail pairs run last.
  // single: a unit is one 128-row Q tile (slot B never used)
  AttnUnit r;
  const int pair = u / BH, bh = u - pair * BH;
  r.b = bh / heads;
  r.h = bh - r.b * heads;
  r.q0 = pair * (single ? 128 : 256);
  r.has_b = !single && (r.q0 + 128) < T;
  return r;
}

template <int POLY>
__global__ void __launch_bounds__(ATT_THREADS, 1)
    attention_tc_kernel(const __grid_constant__ CUtensorMap tqkv, __nv_bfloat16* __restrict__ out, int B, int T,
                        int D, int heads, float scale_log2, int trace, const int* __restrict__ sched,
                        int single) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;               // [2 units][2 slots]: the next unit's Q lands during this one
  uint8_t* sK = sQ + 4 * TILE;      // [KS]
  uint8_t* sV = sK + KS * TILE;     // [VS]
  float* xch = reinterpret_cast<float*>(sV + VS * TILE);  // [2 slots][3][2 halves][128 rows]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + VS * TILE + XCH_BYTES);
  uint64_t* q_full = bars;          // [2 units][2 slots]
  uint64_t* q_empty = bars + 4;     // [2 units][2 slots]
  uint64_t* k_full = bars + 8;      // [KS]
  uint64_t* k_empty = k_full + KS;  // [KS]  released by both MMA issuers
  uint64_t* v_full = k_empty + KS;  // [VS]
  uint64_t* v_empty = v_full + VS;  // [VS]  released by both MMA issuers
  uint64_t* s_full = v_empty + VS;  // [2]
  uint64_t* s_free = s_full + 2;    // [2] softmax x has pulled S_x into registers
  uint64_t* p_full = s_free + 2;    // [2 slots][2 key halves]
  uint64_t* o_done = p_full + 4;    // [2 slots][2 key halves]
  uint64_t* e_done = o_done + 4;    // [2 slots] exp pass of the slot's current tile finished
  uint32_t* tslot = reinterpret_cast<uint32_t*>(e_done + 2);

  const int BH = B * heads;
  const int nkv = (T + 127) / 128;
  // this CTA's units (host LPT schedule, heavy first, so units without a B tile come last)
  const int u_lo = __ldg(sched + blockIdx.x), u_hi = __ldg(sched + blockIdx.x + 1);
  const int* ulist = sched + gridDim.x + 1;
  const uint32_t warp = warp_id(), lane = lane_id();

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tqkv);
    for (int i = 0; i < 4; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 8);
      for (int h = 0; h < 2; ++h) {
        mbar_init(&p_full[i * 2 + h], 4);
        mbar_init(&o_done[i * 2 + h], 1);
      }
      mbar_init(&e_done[i], 8);
    }
    for (int i = 0; i < KS; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 2);
    }
    for (int i = 0; i < VS; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 2);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  pdl_wait();
  const bool pdl_late = (trace >> 8) & 1;  // signal dependents after the last K/V load
  if (!pdl_late) pdl_trigger();

  // Units are ordered pair-major, so a unit without a B tile (T <= q0 + 128) is followed only by
  // such units: the slot-B barriers are simply left alone from then on.
  if (warp == 0) {
    if (lane == 0) {
      int kit = 0, vit = 0, qn = 0;
      for (int ui = u_lo; ui < u_hi; ++ui, ++qn) {
        const AttnUnit w = unit_of(__ldg(ulist + ui), BH, heads, T, single);
        const int row0 = w.b * T;
        const int qb = qn & 1;
        for (int x = 0; x < 1 + w.has_b; ++x) {
          mbar_wait(&q_empty[qb * 2 + x], ((qn >> 1) & 1) ^ 1);
          mbar_expect_tx(&q_full[qb * 2 + x], TILE);
          tma_load_2d(sQ + (qb * 2 + x) * TILE, &tqkv, &q_full[qb * 2 + x], w.h * 64, row0 + w.q0 + x * 128);
        }
        for (int j = 0; j < nkv; ++j, ++kit, ++vit) {
          const int ks = kit % KS, vs = vit % VS;
          mbar_wait(&k_empty[ks], ((kit / KS) & 1) ^ 1);
          mbar_expect_tx(&k_full[ks], TILE);
          tma_load_2d(sK + ks * TILE, &tqkv, &k_full[ks], D + w.h * 64, row0 + j * 128);
          mbar_wait(&v_empty[vs], ((vit / VS) & 1) ^ 1);
          mbar_expect_tx(&v_full[vs], TILE);
          tma_load_2d(sV + vs * TILE, &tqkv, &v_full[vs], 2 * D + w.h * 64, row0 + j * 128);
        }
      }
      if (pdl_late) pdl_trigger();
    }
  } else if (warp == 1 || warp == 2) {
    // One MMA issuer warp per Q slot, so neither slot's PV/S issue queues behind the other's.
    // The whole warp runs the loop and one elected lane issues, with every operand computed by
    // all lanes before the election, so the descriptors stay in uniform registers (a lone lane-0
    // thread needed a ~16-instruction R2UR.BROADCAST waterfall per UTCHMMA).
    {
      const int x = __shfl_sync(0xffffffffu, (int)warp - 1, 0);
      int tn = 0;
      const int tbase = 1024 * x;
      constexpr uint32_t idesc_s = idesc_bf16(128, 128);
      constexpr uint32_t idesc_o = idesc_bf16(128, 64, /*b_mn_major=*/true);
      int kit = 0, vit = 0, qn = 0, np = 0;  // np: PV MMAs issued (= p_full / s_free phases consumed)
      const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem, 0);
      const uint32_t s_t = tmem_u + S_COL + x * 128, p_t = tmem_u + P_COL + x * 64, o_t = tmem_u + O_COL + x * 64;
      const uint32_t sQ_u = __shfl_sync(0xffffffffu, smem_u32(sQ), 0), sK_u = sQ_u + 4 * TILE, sV_u = sK_u + KS * TILE;
      auto commit = [&](uint64_t* bar) {
        if (elect_one()) umma_commit(bar);
        __syncwarp();
      };
      auto arrive = [&](uint64_t* bar) {
        if (elect_one()) mbar_arrive(bar);
        __syncwarp();
      };
      if (lane != 0) tn = 1 << 20;  // (trace build) lane 0 records
      for (int ui = u_lo; ui < u_hi; ++ui, ++qn) {
        const AttnUnit w = unit_of(__ldg(ulist + ui), BH, heads, T, single);
        const bool mine = (x == 0) || w.has_b;
        const int qi = (qn & 1) * 2 + x;
        if (mine) {
          mbar_wait(&q_full[qi], (qn >> 1) & 1);
          tc_fence_after();
        }
        const uint32_t q_addr = sQ_u + qi * TILE;
        // S_x = Q_x K^T. The previous S_x was released (s_free / p_full waited) before the
        // previous PV, so the S_x columns are free here.
        auto issue_s = [&](uint32_t k_addr) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t ad = smem_desc(q_addr + k * 32, 16, 1024, 2), bd = smem_desc(k_addr + k * 32, 16, 1024, 2);
            if (elect_one()) umma_f16(s_t, ad, bd, idesc_s, k > 0);
            __syncwarp();
          }
          commit(&s_full[x]);
        };
        for (int j = 0; j < nkv; ++j, ++vit) {
          if (j == 0) {  // S_x(0)
            const int ks = kit % KS;
            mbar_wait(&k_full[ks], (kit / KS) & 1);
            tc_fence_after();
            if (mine) issue_s(sK_u + ks * TILE);
            if (mine) ATT_TRACE(tbase, tn, 20);
            if (nkv > 1) {  // K_0 stays until S_x(0) is done; with nkv == 1 it is released below
              if (mine) commit(&k_empty[ks]); else arrive(&k_empty[ks]);
              ++kit;
            }
          }
          const bool next = j + 1 < nkv;
          const int ks = kit % KS, vs = vit % VS;
          if (next) mbar_wait(&k_full[ks], (kit / KS) & 1);
          mbar_wait(&v_full[vs], (vit / VS) & 1);
          tc_fence_after();
          if (mine) {
            if (next) {
              mbar_wait(&s_free[x], np & 1);  // S_x(j) is in softmax registers: S_x(j+1) may land
              tc_fence_after();
              issue_s(sK_u + ks * TILE);
              ATT_TRACE(tbase, tn, 20);
            }
            // O_x += P_x(j) V_j in two key halves, each as soon as its softmax warp pair has
            // written its half of P (and each half of P is released on its own)
            const uint64_t vd0 = smem_desc(sV_u + vs * TILE, 1024, 1024, 2);
            const uint32_t vlo = __shfl_sync(0xffffffffu, (uint32_t)vd0, 0), vhi = (uint32_t)(vd0 >> 32);
            for (int h = 0; h < 2; ++h) {
              mbar_wait(&p_full[x * 2 + h], np & 1);
              ATT_TRACE(tbase, tn, 21 + h);
              tc_fence_after();
#pragma unroll
              for (int k = 4 * h; k < 4 * h + 4; ++k) {
                const uint64_t bd = ((uint64_t)vhi << 32) | (vlo + (uint32_t)(k * (2048 >> 4)));
                if (elect_one()) umma_f16_ts(o_t, p_t + k * 8, bd, idesc_o, (j > 0 || k > 0) ? 1u : 0u);
                __syncwarp();
              }
              commit(&o_done[x * 2 + h]);
            }
            ++np;
            if (next || nkv == 1) commit(&k_empty[ks]);
            commit(&v_empty[vs]);
            if (!next) commit(&q_empty[qi]);  // every S_x of the unit issued
          } else {
            if (next || nkv == 1) arrive(&k_empty[ks]);
            arrive(&v_empty[vs]);
          }
          if (next || nkv == 1) ++kit;
        }
      }
    }
  } else {
    // softmax warps 3-18: Q slot x, column half hh (keys 64*hh .. 64*hh+63 of each tile), TMEM
    // lane quadrant = warp % 4 (hardware). The two warps of a (slot, quadrant) own the same 32
    // rows and agree on the row max through smem + a 64-thread named barrier.
    const int sw = (int)warp - 3;
    const int x = sw >> 3, hh = (sw >> 2) & 1;
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const int bar_id = 1 + x * 4 + quad;  // named barrier of the warp pair
    const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16);
    const uint32_t s_addr = lane_base + S_COL + x * 128 + hh * 64;
    const uint32_t p_addr = lane_base + P_COL + x * 64 + hh * 32;
    const uint32_t o_addr = lane_base + O_COL + x * 64;
    int ns = 0, npv = 0;  // S tiles consumed, P tiles produced (global counts)
    int na = 0, nb = 0;   // exp passes slot A / slot B completed before the current unit
    int tn = 0;
    const bool tr = (quad == 0 && lane == 0 && hh == 0);
    const int tbase = 2048 + 1024 * x;
    const int dbg = (trace >> 1) & 0x7f;  // diagnostics (VPE_ATT_DBG): 2 = no exp ping-pong
    const bool pp = !(dbg & 2);
    auto pair_sync = [&]() { asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory"); };
    for (int ui = u_lo; ui < u_hi; ++ui) {
      const AttnUnit w = unit_of(__ldg(ulist + ui), BH, heads, T, single);
      if (x == 1 && !w.has_b) continue;
      const int q0 = w.q0 + x * 128;
      const bool warp_active = (q0 + quad * 32) < T;
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < nkv; ++j, ++ns, ++npv) {
        if (tr) ATT_TRACE(tbase, tn, 10);
        mbar_wait(&s_full[x], ns & 1);
        tc_fence_after();
        if (tr) ATT_TRACE(tbase, tn, 11);
        auto release_s = [&]() {  // every load of this half of S_x(j) has landed in registers
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&s_free[x]);
        };
        // ping-pong on the exponential unit: slot A's pass j follows slot B's pass j-1 and slot
        // B's pass j follows slot A's pass j, so one slot's max pass (TMEM reads, 3-input max,
        // exchange) runs under the other slot's exponentials instead of both slots contending
        // for MUFU at once and leaving it idle during their max passes
        auto exp_token = [&]() {
          if (w.has_b && pp) {
            if (x == 0 && j > 0) mbar_wait(&e_done[1], (nb + j - 1) & 1);
            if (x == 1) mbar_wait(&e_done[0], (na + j) & 1);
          }
        };
        auto exp_done = [&]() {
          __syncwarp();
          if (w.has_b && pp && lane == 0) mbar_arrive(&e_done[x]);
        };
        if (warp_active) {
          const int kvalid = T - j * 128 - hh * 64;  // keys of this half >= kvalid are padding
          const int nch = kvalid >= 64 ? 2 : (kvalid <= 0 ? 0 : (kvalid + 31) >> 5);
          auto mask = [&](int c, float (&v)[32]) {
            if (c * 32 + 32 > kvalid) {
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (c * 32 + i >= kvalid) v[i] = -INFINITY;
            }
          };
          // pass 1: row max over this half (one 32-column chunk in registers at a time). Full
          // halves (every tile but the ragged last one) take a branch-free path.
          const bool full = kvalid >= 64;
          float mx = -INFINITY;
          if (full) {
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              float v[32];
              tmem_ld32(s_addr + c * 32, v);
              tmem_ld_wait_dep(v);
              mx = fmaxf(mx, chunk_max_log2(v, scale_log2));
            }
          } else {
#pragma unroll 1
            for (int c = 0; c < nch; ++c) {
              float v[32];
              tmem_ld32(s_addr + c * 32, v);
              tmem_ld_wait_dep(v);
              mask(c, v);
              mx = fmaxf(mx, chunk_max_log2(v, scale_log2));
            }
          }
          float* xrow = xch + ((x * 3 + (ns & 1)) * 2) * 128;
          xrow[hh * 128 + r] = mx;
          pair_sync();
          mx = fmaxf(mx, xrow[(hh ^ 1) * 128 + r]);
          // the exponent offset m_used only moves when a row max exceeds it by > 8 (p <= 256),
          // so O is rescaled in TMEM about once per row; both halves take identical decisions
          const bool raise = mx > m_used + 8.f;
          const bool rescale = __any_sync(0xffffffffu, raise);
          float alpha = 1.f;
          if (rescale) {
            const float m_new = fmaxf(m_used, mx);
            alpha = fast_exp2(m_used - m_new);  // 0 on the first tile (m_used = -inf)
            l *= alpha;
            m_used = m_new;
          }
          exp_token();
          // this half of P_x(j-1) must have been consumed before this half of P_x(j) is written
          if (npv > 0) {
            mbar_wait(&o_done[x * 2 + hh], (npv - 1) & 1);
            tc_fence_after();
          }
          if (tr) ATT_TRACE(tbase, tn, 12);
          // pass 2: p = 2^(s*scale - m_used) for this half's two chunks
          uint64_t lt = 0;  // f32x2 partial row sums
          if (full) {
            {
              float v[32];
              tmem_ld32(s_addr, v);
              tmem_ld_wait_dep(v);
              lt = emit_chunk<POLY, true>(v, scale_log2, m_used, p_addr);
            }
            float v[32];
            tmem_ld32(s_addr + 32, v);
            tmem_ld_wait_dep(v);
            release_s();
            lt = fadd2(lt, emit_chunk<POLY, true>(v, scale_log2, m_used, p_addr + 16));
          } else {
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              if (c < nch) {
                float v[32];
                tmem_ld32(s_addr + c * 32, v);
                tmem_ld_wait_dep(v);
                if (c + 1 >= nch) release_s();
                mask(c, v);
                lt = fadd2(lt, c * 32 + 32 <= kvalid ? emit_chunk<POLY, true>(v, scale_log2, m_used, p_addr + c * 16)
                                                     : emit_chunk<POLY, false>(v, scale_log2, m_used, p_addr + c * 16));
              } else {
                if (c == 0) release_s();
#pragma unroll
                for (int g = 0; g < 4; ++g) tmem_st4u(p_addr + c * 16 + 4 * g, 0u, 0u, 0u, 0u);
              }
            }
          }
          exp_done();
          if (rescale && j > 0) {
            // O_x *= alpha in TMEM, once per row (half 0), after both halves of PV_x(j-1) and
            // before either half of PV_x(j) may be issued (the pair syncs before p_full)
            mbar_wait(&o_done[x * 2 + (hh ^ 1)], (npv - 1) & 1);
            tc_fence_after();
            if (hh == 0) {
#pragma unroll 1
              for (int c = 0; c < 2; ++c) {
                float t[32];
                tmem_ld32(o_addr + c * 32, t);
                tmem_ld_wait_dep(t);
#pragma unroll
                for (int i = 0; i < 32; ++i) t[i] *= alpha;
                tmem_st32(o_addr + c * 32, t);
              }
              tmem_st_wait();
            }
            tc_fence_before();
            pair_sync();
            tc_fence_after();
          }
          float l0, l1;
          f2_unpack(lt, l0, l1);
          l += l0 + l1;
          tmem_st_wait();
        } else {
          release_s();
          // a warp whose rows are all past T must not run ahead: its p_full arrival for tile j
          // would otherwise count toward tile j-1's phase while the active warps of the tile are
          // still writing P_x(j-1), releasing PV_x(j-1) early (a latent race of round 1's kernel)
          if (npv > 0) mbar_wait(&o_done[x * 2 + hh], (npv - 1) & 1);
          exp_token();  // inactive rows still take part in the hand-off (arrive counts are per warp)
          exp_done();
        }
        tc_fence_before();
        __syncwarp();
        if (tr) ATT_TRACE(tbase, tn, 13);
        (void)dbg;
        if (lane == 0) mbar_arrive(&p_full[x * 2 + hh]);  // this half of P_x(j) in TMEM
      }
      // epilogue: l = l_half0 + l_half1; each half writes 32 of the 64 output columns
      mbar_wait(&o_done[x * 2], (npv - 1) & 1);
      mbar_wait(&o_done[x * 2 + 1], (npv - 1) & 1);
      tc_fence_after();
      if (warp_active) {
        float* xrow = xch + ((x * 3 + 2) * 2) * 128;  // own slot: the next tile's max exchange may start
        xrow[hh * 128 + r] = l;
        pair_sync();
        const float lsum = l + xrow[(hh ^ 1) * 128 + r];
        float t[32];
        tmem_ld32(o_addr + hh * 32, t);
        tmem_ld_wait();
        const int qi = q0 + r;
        if (qi < T) {
          const float inv = kTruncScale / lsum;
          uint4* dst = reinterpret_cast<uint4*>(out + (int64_t)(w.b * T + qi) * D + w.h * 64 + hh * 32);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint4 a;
            a.x = pack_bf16(t[8 * c + 0] * inv, t[8 * c + 1] * inv);
            a.y = pack_bf16(t[8 * c + 2] * inv, t[8 * c + 3] * inv);
            a.z = pack_bf16(t[8 * c + 4] * inv, t[8 * c + 5] * inv);
            a.w = pack_bf16(t[8 * c + 6] * inv, t[8 * c + 7] * inv);
            dst[c] = a;
          }
        }
      }
      tc_fence_before();
      na += nkv;
      if (w.has_b) nb += nkv;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
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
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int BH = B * heads, npairs = (T + 255) / 256;
  // small batches: pairs of Q tiles would leave most SMs idle, so run one tile per unit
  const char* es = getenv("VPE_ATT_SINGLE");
  a->single = es ? (es[0] == '1') : (2 * BH * npairs <= sms);
  const int per = a->single ? (T + 127) / 128 : npairs, units = BH * per;
  a->grid = units < sms ? units : sms;
  const char* e = getenv("VPE_ATT_GRID");  // experiment: "all" = one unit per CTA (no persistence)
  if (e && e[0] == 'a') a->grid = units;
  // Longest-processing-time-first static schedule: a unit costs ~ its Q tiles' valid rows plus a
  // fixed MMA/pipeline share; heavy units first, each to the least-loaded CTA. Round-robin left
  // T = 1025 at 3 full pairs + 1 tail unit on 36 CTAs (the tail pair holds one valid row).
  // (device, B*heads, T, grid, mode) -> device schedule; the schedule array lives on that device
  static std::map<std::tuple<int, int, int, int, int>, int*> cache;
  static std::mutex cache_mu;
  // fixed share of a Q tile: a tile with one valid row still runs the whole KV loop (S MMAs, the
  // pipeline, the softmax of its active warps). Calibrated with VPE_ATT_FIX over B = 4..24 at
  // T = 1025: 0.35 left batch 12 at 95 us (8 CTAs with one full pair + 6 tail units), 0.75 -> 60 us.
  static const double fix = getenv("VPE_ATT_FIX") ? atof(getenv("VPE_ATT_FIX")) : 0.75;
  const auto key = std::make_tuple(dev, BH, T, a->grid, (int)(fix * 1000) * 2 + a->single);
  std::lock_guard<std::mutex> lock(cache_mu);
  auto it = cache.find(key);
  if (it == cache.end()) {
    std::vector<std::pair<double, int>> cost(units);
    for (int u = 0; u < units; ++u) {
      const int q0 = (u / BH) * (a->single ? 128 : 256);
      double c = 0;
      for (int t = 0; t < (a->single ? 1 : 2); ++t) {
        const int rows = std::min(128, std::max(0, T - (q0 + 128 * t)));
        if (rows > 0) c += fix + (1.0 - fix) * rows / 128.0;
      }
      cost[u] = {c, u};
    }
    std::stable_sort(cost.begin(), cost.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
    std::vector<double> load(a->grid, 0.0);
    std::vector<std::vector<int>> lists(a->grid);
    for (const auto& cu : cost) {
      int best = 0;
      for (int c = 1; c < a->grid; ++c)
        if (load[c] < load[best]) best = c;
      load[best] += cu.first;
      lists[best].push_back(cu.second);
    }
    std::vector<int> host(a->grid + 1 + units);
    int off = 0;
    for (int c = 0; c < a->grid; ++c) {
      host[c] = off;
      for (int u : lists[c]) host[a->grid + 1 + off++] = u;
    }
    host[a->grid] = off;
    int* d = nullptr;
    if (cudaMalloc(&d, host.size() * sizeof(int)) != cudaSuccess) return VPE_E_RESOURCE;
    if (cudaMemcpy(d, host.data(), host.size() * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess)
      return VPE_E_CUDA;
    it = cache.emplace(key, d).first;
  }
  a->sched = it->second;
  return VPE_OK;
}

static int att_dbg() {
  static const int d = getenv("VPE_ATT_DBG") ? atoi(getenv("VPE_ATT_DBG")) : 0;
  return d;
}

int launch_attention(const AttnPlan& a, cudaStream_t s) {
  static int poly = -1;
  if (poly < 0) {
    const char* e = getenv("VPE_ATT_POLY");
    poly = e ? atoi(e) : 3;  // 4 of 16 pairs on the FMA pipe (tools/ubench/emit.cu: best MUFU/FMA balance)
  }
  static OncePerDevice attr;
  if (attr.first()) {
#define VPE_ATT_ATTR(P_)                                                                          \
  cudaFuncSetAttribute(attention_tc_kernel<P_>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_ATT); \
  max_smem_carveout(attention_tc_kernel<P_>);
    VPE_ATT_ATTR(0) VPE_ATT_ATTR(0x0303) VPE_ATT_ATTR(0x1111) VPE_ATT_ATTR(0x2525) VPE_ATT_ATTR(0x5555)
#undef VPE_ATT_ATTR
  }
  const float scale_log2 = 0.125f * 1.4426950408889634f;
  if (g_att_trace_on < 0) {
    const char* e = getenv("VPE_ATT_TRACE");
    g_att_trace_on = (e && e[0] == '1') ? 1 : 0;
  }
  // pairs of exponentials (of 16 per 32-key chunk) computed on the FMA pipe instead of MUFU
  auto k = poly == 0   ? attention_tc_kernel<0>
           : poly == 2 ? attention_tc_kernel<0x0303>
           : poly == 4 ? attention_tc_kernel<0x2525>
           : poly == 5 ? attention_tc_kernel<0x5555>
                       : attention_tc_kernel<0x1111>;
  // In the programmatic chain like every backbone kernel (VPE_ATT_PDL=0 takes it out). Round 1
  // kept it out: with it in, engine outputs varied bitwise run to run. The likely cause was this
  // kernel's own tail-tile race (inactive softmax warps ran ahead on p_full before PV(j-1) had
  // consumed P; since fixed in the softmax loop), which PDL's tighter overlap exposed more often:
  // after that fix tools/pdl_determinism.py finds 0 of 300 PDL replays differing bitwise
  // (batch 1; 0 of 100 at batch 4).
  static const int att_pdl = getenv("VPE_ATT_PDL") ? atoi(getenv("VPE_ATT_PDL")) : 1;
  const int saved_scope = pdl_scope();
  if (!att_pdl) pdl_scope() = 0;
  struct Restore {
    int v;
    ~Restore() { pdl_scope() = v; }
  } restore{saved_scope};
  return launch_k(k, dim3(a.grid), dim3(ATT_THREADS), SMEM_ATT, s, a.tqkv, a.out, a.B, a.T, a.D, a.heads, scale_log2,
                  g_att_trace_on | (att_dbg() << 1) | (pdl_late() << 8), a.sched, a.single) == cudaSuccess
             ? VPE_OK
             : VPE_E_CUDA;
}

}  // namespace vpe

extern "C" int vpe_debug_att_trace(unsigned long long* host, int n) {
  if (!host || n < 0 || n > 4096) return VPE_E_VALUE;
  VPE_CUDA_TRY(cudaMemcpyFromSymbol(host, vpe::g_att_trace, n * sizeof(unsigned long long)));
  return VPE_OK;
}
