// RPN-style detection head ("b200_det") on sm_100a.
//   1. 3x3 conv D->D + ReLU, read in place from the ring's `final` tap as an NHWC image; tcgen05
//      implicit GEMM with split-precision weights (W = hi + lo bf16; the ring features are exact
//      bf16 so A needs no split). Measured objectness error vs the fp32 oracle ~1e-5 relative,
//      set by the tensor core's fp32 accumulation (a third weight part makes it worse).
//   2. 1x1 cls (A) / bbox (4A) convs in fp32 FFMA (fp32-faithful objectness for identical top-k).
//   3. per image: radix-select top-k (k = pre_nms_top_n) of the objectness logits, bitonic sort,
//      anchor decode (BoxCoder(1,1,1,1), clip log(1000/16)), clip to image, remove-small, sigmoid.
//   4. NMS: parallel 64x64-tile IoU bitmask over many CTAs, then one warp's greedy scan.
// Oracle: oracle/det.py (torchvision rpn.py:15-79, 231-297; _utils.py:183-225;
// anchor_utils.py:58-113; ops/boxes.py:20-48).
#include <cuda_runtime.h>

#include <new>

#include "gemm.cuh"
#include "runtime.h"
#include "util.cuh"

using namespace vpe;

namespace {
constexpr int KMAX = 1024;  // candidate capacity (pre_nms_top_n <= 1024)
constexpr size_t TOPK_SMEM_MAX = 160 * 1024;  // det_topk_kernel order-key cache (n * 4 bytes)
constexpr int NMS_BLK = 64;
constexpr int NWORDS = KMAX / NMS_BLK;  // 16 x u64 per mask row
}  // namespace

struct vpe_det {
  vpe_det_config cfg;
  vpe_det_weights w;
  int h = 0, P = 0, A = 0, NO = 0;
  float* hidden = nullptr;   // [B*P, D] fp32
  float* wT = nullptr;       // [D, 5A] fp32 (cls | box transposed)
  float* bcat = nullptr;     // [5A]
  float* obj = nullptr;      // [B, P*A]
  float* deltas = nullptr;   // [B, P*A, 4]
  float* cbox = nullptr;     // [B, KMAX, 4]
  float* cscore = nullptr;   // [B, KMAX]
  int* cidx = nullptr;       // [B, KMAX]
  uint8_t* cvalid = nullptr; // [B, KMAX]
  unsigned long long* mask = nullptr;  // [B, KMAX, NWORDS]
  const void* bound = nullptr;
  GemmPlan g;
};

namespace {

__global__ void transpose_heads_kernel(const float* __restrict__ cls_w, const float* __restrict__ box_w,
                                       const float* __restrict__ cls_b, const float* __restrict__ box_b, int A, int D,
                                       float* __restrict__ wT, float* __restrict__ bcat) {
  const int NO = 5 * A;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < D * NO; i += gridDim.x * blockDim.x) {
    const int k = i / NO, o = i - k * NO;
    wT[i] = o < A ? cls_w[o * D + k] : box_w[(o - A) * D + k];
  }
  if (blockIdx.x == 0)
    for (int o = threadIdx.x; o < NO; o += blockDim.x) bcat[o] = o < A ? cls_b[o] : box_b[o - A];
}

// 1x1 cls (A) / bbox (4A) convs in fp32 FFMA, register-tiled SGEMM: a block computes 32 pixels
// x 48 outputs (45 used); each thread 4 pixels x 3 outputs; K = D streamed through SMEM in chunks.
// (64-pixel blocks of 256 threads: 256 blocks for 148 SMs, 51 vs 47 us at B = 16.)
constexpr int PX_PER_BLK = 32, KT = 32, SH_PITCH = 36, NO_PAD = 48, DET_THREADS = 128;
__global__ void __launch_bounds__(DET_THREADS) det_1x1_kernel(const float* __restrict__ hidden, int npix_total, int P,
                                                      int D, int A, const float* __restrict__ wT,
                                                      const float* __restrict__ bcat, float* __restrict__ obj,
                                                      float* __restrict__ deltas) {
  __shared__ __align__(16) float s_h[KT][SH_PITCH];  // transposed hidden chunk [k][pixel]
  __shared__ float s_w[KT][NO_PAD];
  const int NO = 5 * A;
  const int p0 = blockIdx.x * PX_PER_BLK;
  const int tid = threadIdx.x, pg = tid >> 4, og = tid & 15;
  float acc[4][3];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) acc[i][j] = 0.f;
  // the next K chunk's hidden / weight values are loaded into registers while this chunk's FMAs
  // run (one global round trip per chunk was the kernel's critical path: 12 chunks at D = 384)
  constexpr int HJ = (PX_PER_BLK * KT) / DET_THREADS, WJ = (KT * NO_PAD + DET_THREADS - 1) / DET_THREADS;
  float hn[HJ], wn[WJ];
  auto fetch = [&](int k0) {
#pragma unroll
    for (int j = 0; j < HJ; ++j) {
      const int i = tid + DET_THREADS * j;
      const int px = i / KT, kk = i - px * KT;
      const int gp = p0 + px;
      hn[j] = gp < npix_total ? hidden[(int64_t)gp * D + k0 + kk] : 0.f;
    }
#pragma unroll
    for (int j = 0; j < WJ; ++j) {
      const int i = tid + DET_THREADS * j;
      const int kk = i / NO_PAD, o = i - kk * NO_PAD;
      wn[j] = (i < KT * NO_PAD && o < NO) ? __ldg(wT + (int64_t)(k0 + kk) * NO + o) : 0.f;
    }
  };
  fetch(0);
  for (int k0 = 0; k0 < D; k0 += KT) {
#pragma unroll
    for (int j = 0; j < HJ; ++j) {
      const int i = tid + DET_THREADS * j;
      const int px = i / KT, kk = i - px * KT;
      s_h[kk][px] = hn[j];
    }
#pragma unroll
    for (int j = 0; j < WJ; ++j) {
      const int i = tid + DET_THREADS * j;
      if (i < KT * NO_PAD) s_w[i / NO_PAD][i % NO_PAD] = wn[j];
    }
    __syncthreads();
    if (k0 + KT < D) fetch(k0 + KT);
#pragma unroll 8
    for (int kk = 0; kk < KT; ++kk) {
      const float4 h = *reinterpret_cast<const float4*>(&s_h[kk][pg * 4]);
      const float w0 = s_w[kk][og], w1 = s_w[kk][og + 16], w2 = s_w[kk][og + 32];
      const float hv[4] = {h.x, h.y, h.z, h.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        acc[i][0] = fmaf(hv[i], w0, acc[i][0]);
        acc[i][1] = fmaf(hv[i], w1, acc[i][1]);
        acc[i][2] = fmaf(hv[i], w2, acc[i][2]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gp = p0 + pg * 4 + i;
    if (gp >= npix_total) continue;
    const int b = gp / P, p = gp - b * P;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int o = og + 16 * j;
      if (o >= NO) continue;
      const float v = acc[i][j] + bcat[o];
      if (o < A) {
        obj[(int64_t)b * P * A + (int64_t)p * A + o] = v;
      } else {
        const int q = o - A, a = q >> 2, c = q & 3;
        deltas[((int64_t)b * P * A + (int64_t)p * A + a) * 4 + c] = v;
      }
    }
  }
}

__device__ __forceinline__ uint32_t order_key(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// per image: top-k select + sort + decode
__global__ void __launch_bounds__(1024) det_topk_kernel(const float* __restrict__ obj, const float* __restrict__ deltas,
                                                        int n, int K, vpe_det_config cfg, int h, float* __restrict__ cbox,
                                                        float* __restrict__ cscore, int* __restrict__ cidx,
                                                        uint8_t* __restrict__ cvalid, int64_t* __restrict__ top_index) {
  __shared__ uint32_t hist[256];
  __shared__ uint32_t s_key[KMAX];
  __shared__ int s_idx[KMAX];
  __shared__ uint32_t s_prefix, s_krem, s_cnt, s_ties;
  __shared__ uint32_t s_wcount[32];
  extern __shared__ uint32_t s_okey[];  // [n] order keys: the 4 radix passes and the gathers read smem
  const int b = blockIdx.x, tid = threadIdx.x;
  const float* o = obj + (int64_t)b * n;
  for (int i = tid; i < n; i += blockDim.x) s_okey[i] = order_key(__ldg(o + i));
  __syncthreads();
  uint32_t prefix = 0, pmask = 0, krem = K;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int i = tid; i < n; i += blockDim.x) {
      const uint32_t k = s_okey[i];
      if ((k & pmask) == prefix) atomicAdd(&hist[(k >> shift) & 255], 1u);
    }
    __syncthreads();
    if (tid < 32) {
      // lane l owns bins [8*(31-l), 8*(31-l)+8): lane 0 the highest bins
      uint32_t local = 0;
      const int hi0 = 8 * (31 - tid);
      for (int q = 0; q < 8; ++q) local += hist[hi0 + q];
      uint32_t incl = local;  // inclusive prefix from the top
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, off);
        if (tid >= off) incl += v;
      }
      const uint32_t excl = incl - local;
      if (excl < krem && incl >= krem) {
        uint32_t above = excl;
        int digit = hi0;
        for (int q = 7; q >= 0; --q) {
          const uint32_t c = hist[hi0 + q];
          if (above + c >= krem) {
            digit = hi0 + q;
            break;
          }
          above += c;
        }
        s_prefix = prefix | ((uint32_t)digit << shift);
        s_krem = krem - above;
      }
    }
    __syncthreads();
    prefix = s_prefix;
    krem = s_krem;
    pmask |= 255u << shift;
    __syncthreads();
  }
  // prefix = threshold key; krem = how many ties (== threshold) to take, lowest index first
  if (tid == 0) {
    s_cnt = 0;
    s_ties = 0;
  }
  __syncthreads();
  for (int i = tid; i < n; i += blockDim.x) {
    const uint32_t k = s_okey[i];
    if (k > prefix) {
      const uint32_t pos = atomicAdd(&s_cnt, 1u);
      s_key[pos] = k;
      s_idx[pos] = i;
    }
  }
  __syncthreads();
  const uint32_t gcount = K - krem;
  for (int base = 0; base < n; base += blockDim.x) {
    const int i = base + tid;
    const bool tie = (i < n) && s_okey[i] == prefix;
    const uint32_t bal = __ballot_sync(0xffffffffu, tie);
    if ((tid & 31) == 0) s_wcount[tid >> 5] = __popc(bal);
    __syncthreads();
    uint32_t before = s_ties;
    for (int w = 0; w < (tid >> 5); ++w) before += s_wcount[w];
    before += __popc(bal & ((1u << (tid & 31)) - 1u));
    if (tie && before < krem) {
      s_key[gcount + before] = prefix;
      s_idx[gcount + before] = i;
    }
    __syncthreads();
    if (tid == 0) {
      uint32_t tot = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += s_wcount[w];
      s_ties += tot;
    }
    __syncthreads();
  }
  for (int i = K + tid; i < KMAX; i += blockDim.x) {
    s_key[i] = 0;
    s_idx[i] = 0x7fffffff;
  }
  __syncthreads();
  // bitonic sort, descending key, ascending index on ties. One element per thread (blockDim ==
  // KMAX); partners closer than a warp exchange by shuffle, the 15 wider stages through smem
  // (55 block-wide barriers -> 30)
  {
    uint32_t key = s_key[tid];
    int idx = s_idx[tid];
    for (int k = 2; k <= KMAX; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        uint32_t pk;
        int pi;
        if (j >= 32) {
          __syncthreads();
          s_key[tid] = key;
          s_idx[tid] = idx;
          __syncthreads();
          pk = s_key[tid ^ j];
          pi = s_idx[tid ^ j];
        } else {
          pk = __shfl_xor_sync(0xffffffffu, key, j);
          pi = __shfl_xor_sync(0xffffffffu, idx, j);
        }
        const bool up = (tid & k) == 0, lower = (tid & j) == 0;
        const bool self_first = (key > pk) || (key == pk && idx < pi);
        const bool take = (lower == up) ? !self_first : self_first;
        if (take) {
          key = pk;
          idx = pi;
        }
      }
    }
    __syncthreads();
    s_key[tid] = key;
    s_idx[tid] = idx;
    __syncthreads();
  }
  // decode (torchvision _utils.py:183-225) + clip + remove small + sigmoid
  const int A = cfg.num_anchors;
  const float stride = (float)(cfg.resolution / h);
  const float R = (float)cfg.resolution;
  for (int i = tid; i < KMAX; i += blockDim.x) {
    float* bx = cbox + ((int64_t)b * KMAX + i) * 4;
    if (i >= K) {
      cvalid[(int64_t)b * KMAX + i] = 0;
      cidx[(int64_t)b * KMAX + i] = -1;
      bx[0] = bx[1] = bx[2] = bx[3] = 0.f;
      cscore[(int64_t)b * KMAX + i] = 0.f;
      continue;
    }
    const int idx = s_idx[i];
    const int loc = idx / A, a = idx - loc * A;
    const int y = loc / h, x = loc - y * h;
    const float sx = (float)x * stride, sy = (float)y * stride;
    const float ax1 = sx + cfg.base_anchors[a][0], ay1 = sy + cfg.base_anchors[a][1];
    const float ax2 = sx + cfg.base_anchors[a][2], ay2 = sy + cfg.base_anchors[a][3];
    const float* d = deltas + ((int64_t)b * n + idx) * 4;
    const float wdt = __fsub_rn(ax2, ax1), hgt = __fsub_rn(ay2, ay1);
    const float cx = __fadd_rn(ax1, __fmul_rn(0.5f, wdt)), cy = __fadd_rn(ay1, __fmul_rn(0.5f, hgt));
    const float dw = fminf(d[2], cfg.bbox_clip), dh = fminf(d[3], cfg.bbox_clip);
    const float pcx = __fadd_rn(__fmul_rn(d[0], wdt), cx), pcy = __fadd_rn(__fmul_rn(d[1], hgt), cy);
    const float pw = __fmul_rn(expf(dw), wdt), ph = __fmul_rn(expf(dh), hgt);
    const float hw = __fmul_rn(0.5f, pw), hh = __fmul_rn(0.5f, ph);
    float x1 = __fsub_rn(pcx, hw), y1 = __fsub_rn(pcy, hh), x2 = __fadd_rn(pcx, hw), y2 = __fadd_rn(pcy, hh);
    x1 = fminf(fmaxf(x1, 0.f), R);
    x2 = fminf(fmaxf(x2, 0.f), R);
    y1 = fminf(fmaxf(y1, 0.f), R);
    y2 = fminf(fmaxf(y2, 0.f), R);
    const float logit = o[idx];
    const float score = 1.f / (1.f + expf(-logit));
    const bool ok = (x2 - x1 >= cfg.min_size) && (y2 - y1 >= cfg.min_size) && (score >= cfg.score_thresh);
    bx[0] = x1;
    bx[1] = y1;
    bx[2] = x2;
    bx[3] = y2;
    cscore[(int64_t)b * KMAX + i] = score;
    cidx[(int64_t)b * KMAX + i] = idx;
    cvalid[(int64_t)b * KMAX + i] = ok ? 1 : 0;
    if (top_index) top_index[(int64_t)b * K + i] = idx;
  }
}

// IoU > thresh bitmask, 64x64 tiles (upper triangle), one thread per row box
__global__ void __launch_bounds__(NMS_BLK) det_nms_mask_kernel(const float* __restrict__ cbox, int K, float thresh,
                                                               unsigned long long* __restrict__ mask) {
  const int cb = blockIdx.x, rb = blockIdx.y, b = blockIdx.z;
  if (cb < rb) return;
  __shared__ float4 s_box[NMS_BLK];  // one LDS.128 per candidate
  __shared__ float s_area[NMS_BLK];   // its area, computed once (same operations as per pair)
  const int j0 = cb * NMS_BLK;
  const int t = threadIdx.x;
  const float* base = cbox + (int64_t)b * KMAX * 4;
  if (j0 + t < K) {
    const float4 bx = *reinterpret_cast<const float4*>(base + (j0 + t) * 4);
    s_box[t] = bx;
    s_area[t] = (bx.z - bx.x) * (bx.w - bx.y);
  }
  __syncthreads();
  const int i = rb * NMS_BLK + t;
  if (i >= K) return;
  const float x1 = base[i * 4 + 0], y1 = base[i * 4 + 1], x2 = base[i * 4 + 2], y2 = base[i * 4 + 3];
  const float iarea = (x2 - x1) * (y2 - y1);
  unsigned long long bits = 0;
  const int jn = min(NMS_BLK, K - j0);
  for (int jj = 0; jj < jn; ++jj) {
    const int j = j0 + jj;
    if (j <= i) continue;
    const float4 bj = s_box[jj];
    const float xx1 = fmaxf(x1, bj.x), yy1 = fmaxf(y1, bj.y);
    const float xx2 = fminf(x2, bj.z), yy2 = fminf(y2, bj.w);
    const float w = fmaxf(0.f, xx2 - xx1), hh = fmaxf(0.f, yy2 - yy1);
    const float inter = w * hh;
    const float ovr = inter / ((iarea + s_area[jj]) - inter);
    if (ovr > thresh) bits |= 1ull << jj;
  }
  mask[((int64_t)b * KMAX + i) * NWORDS + cb] = bits;
}

// greedy scan: one CTA per image copies the mask into smem, warp 0 walks the sorted candidates
__global__ void __launch_bounds__(512) det_nms_scan_kernel(const unsigned long long* __restrict__ mask,
                                                           const uint8_t* __restrict__ cvalid,
                                                           const float* __restrict__ cbox,
                                                           const float* __restrict__ cscore,
                                                           const int* __restrict__ cidx, int K, int post,
                                                           float* __restrict__ boxes, float* __restrict__ scores,
                                                           int64_t* __restrict__ index, int32_t* __restrict__ count) {
  extern __shared__ unsigned long long s_mask[];  // [K][NWORDS]
  __shared__ uint8_t s_valid[KMAX];
  __shared__ int s_keep[KMAX];
  __shared__ int s_nk;
  const int b = blockIdx.x;
  const unsigned long long* m = mask + (int64_t)b * KMAX * NWORDS;
  for (int i = threadIdx.x; i < K * NWORDS; i += blockDim.x) {
    const int r = i / NWORDS, c = i - r * NWORDS;
    // only the upper-triangle words were written
    s_mask[i] = (c >= r / NMS_BLK) ? m[i] : 0ull;
  }
  for (int i = threadIdx.x; i < K; i += blockDim.x) s_valid[i] = cvalid[(int64_t)b * KMAX + i];
  __syncthreads();
  if (threadIdx.x < 32) {
    // Block by block (64 candidates): the warp resolves a block's keep bits from its own
    // removal word with the block's in-block mask words loaded up front (independent of the
    // chain), then lane w ORs the kept rows' word w into its removal word -- instead of one
    // dependent shuffle + LDS per candidate.
    const int lane = threadIdx.x;
    unsigned long long remv = 0;  // lane w < NWORDS: removal bits of block w
    int nk = 0;
    const int nblk = (K + NMS_BLK - 1) / NMS_BLK;
    for (int c = 0; c < nblk && nk < post; ++c) {
      const int i0 = c * NMS_BLK, n = min(NMS_BLK, K - i0);
      unsigned long long w = __shfl_sync(0xffffffffu, remv, c);
      const uint32_t vlo = __ballot_sync(0xffffffffu, lane < n && s_valid[i0 + lane]);
      const uint32_t vhi = __ballot_sync(0xffffffffu, lane + 32 < n && s_valid[i0 + 32 + lane]);
      const unsigned long long vb = ((unsigned long long)vhi << 32) | vlo;
      unsigned long long keep = 0;
#pragma unroll 8
      for (int ii = 0; ii < n; ++ii) {
        const unsigned long long mw = s_mask[(i0 + ii) * NWORDS + c];
        const bool k = !((w >> ii) & 1ull) && ((vb >> ii) & 1ull);
        keep |= (unsigned long long)k << ii;
        w |= k ? mw : 0ull;
      }
      int cnt = __popcll(keep);
      if (nk + cnt > post) {  // greedy order: keep only the first post - nk
        for (int drop = nk + cnt - post; drop > 0; --drop) keep &= ~(1ull << (63 - __clzll(keep)));
        cnt = post - nk;
      }
      if (lane < NWORDS) {
        unsigned long long kk = keep;
        while (kk) {
          const int ii = __ffsll(kk) - 1;
          kk &= kk - 1;
          remv |= s_mask[(i0 + ii) * NWORDS + lane];
        }
      }
      // kept candidates in order: lane l writes the positions of set bits l and l + 32
      const uint32_t klo = (uint32_t)keep, khi = (uint32_t)(keep >> 32);
      if ((klo >> lane) & 1u) s_keep[nk + __popc(klo & ((1u << lane) - 1u))] = i0 + lane;
      if ((khi >> lane) & 1u) s_keep[nk + __popc(klo) + __popc(khi & ((1u << lane) - 1u))] = i0 + 32 + lane;
      nk += cnt;
    }
    if (lane == 0) s_nk = nk;
  }
  __syncthreads();
  const int nk = s_nk;
  for (int k = threadIdx.x; k < post; k += blockDim.x) {
    float* ob = boxes + ((int64_t)b * post + k) * 4;
    if (k < nk) {
      const int i = s_keep[k];
      const float* cb = cbox + ((int64_t)b * KMAX + i) * 4;
      ob[0] = cb[0];
      ob[1] = cb[1];
      ob[2] = cb[2];
      ob[3] = cb[3];
      scores[(int64_t)b * post + k] = cscore[(int64_t)b * KMAX + i];
      index[(int64_t)b * post + k] = cidx[(int64_t)b * KMAX + i];
    } else {
      ob[0] = ob[1] = ob[2] = ob[3] = 0.f;
      scores[(int64_t)b * post + k] = 0.f;
      index[(int64_t)b * post + k] = -1;
    }
  }
  if (threadIdx.x == 0) count[b] = nk;
}

}  // namespace

extern "C" int vpe_det_destroy(vpe_det* d) {
  if (!d) return VPE_OK;
  cudaFree(d->hidden);
  cudaFree(d->wT);
  cudaFree(d->bcat);
  cudaFree(d->obj);
  cudaFree(d->deltas);
  cudaFree(d->cbox);
  cudaFree(d->cscore);
  cudaFree(d->cidx);
  cudaFree(d->cvalid);
  cudaFree(d->mask);
  delete d;
  return VPE_OK;
}

extern "C" int vpe_det_create(const vpe_det_config* cfg, const vpe_det_weights* w, vpe_det** out) {
  if (!cfg || !w || !out) return VPE_E_VALUE;
  if (cfg->resolution % 14 || cfg->dim % 64 || cfg->num_anchors < 1 || cfg->num_anchors > 9 ||
      cfg->pre_nms_top_n < 1 || cfg->pre_nms_top_n > KMAX || cfg->post_nms_top_n < 1)
    return VPE_E_CONFIG;
  {
    // the top-k kernel keeps one 4-byte order key per anchor in shared memory
    const int hh = cfg->resolution / 14;
    if ((size_t)hh * hh * cfg->num_anchors * 4 > TOPK_SMEM_MAX) return VPE_E_CONFIG;
  }
  vpe_det* d = new (std::nothrow) vpe_det();
  if (!d) return VPE_E_RESOURCE;
  d->cfg = *cfg;
  d->w = *w;
  d->h = cfg->resolution / 14;
  d->P = d->h * d->h;
  d->A = cfg->num_anchors;
  d->NO = 5 * d->A;
  const int B = cfg->batch, D = cfg->dim, n = d->P * d->A;
  bool ok = cudaMalloc(&d->hidden, (size_t)B * d->P * D * 4) == cudaSuccess &&
            cudaMalloc(&d->wT, (size_t)D * d->NO * 4) == cudaSuccess &&
            cudaMalloc(&d->bcat, (size_t)d->NO * 4) == cudaSuccess &&
            cudaMalloc(&d->obj, (size_t)B * n * 4) == cudaSuccess &&
            cudaMalloc(&d->deltas, (size_t)B * n * 16) == cudaSuccess &&
            cudaMalloc(&d->cbox, (size_t)B * KMAX * 16) == cudaSuccess &&
            cudaMalloc(&d->cscore, (size_t)B * KMAX * 4) == cudaSuccess &&
            cudaMalloc(&d->cidx, (size_t)B * KMAX * 4) == cudaSuccess &&
            cudaMalloc(&d->cvalid, (size_t)B * KMAX) == cudaSuccess &&
            cudaMalloc(&d->mask, (size_t)B * KMAX * NWORDS * 8) == cudaSuccess;
  if (!ok) {
    vpe_det_destroy(d);
    return VPE_E_RESOURCE;
  }
  transpose_heads_kernel<<<64, 256>>>(w->cls_w, w->box_w, w->cls_b, w->box_b, d->A, D, d->wT, d->bcat);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    vpe_det_destroy(d);
    return VPE_E_CUDA;
  }
  *out = d;
  return VPE_OK;
}

extern "C" int vpe_det_forward(vpe_det* d, const void* final_tap, const vpe_det_outputs* o, void* stream) {
  if (!d || !final_tap || !o || !o->boxes || !o->scores || !o->index || !o->count) return VPE_E_VALUE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int D = d->cfg.dim, h = d->h, B = d->cfg.batch, T = h * h + 1, A = d->A;
  const int n = d->P * A;
  const int K = d->cfg.pre_nms_top_n < n ? d->cfg.pre_nms_top_n : n;
  if (d->bound != final_tap) {
    EpiParams ep;
    ep.kind = EPI_F32;
    ep.act = ACT_RELU;
    ep.N = D;
    ep.bias = d->w.conv_b;
    ep.out = d->hidden;
    ep.ldo = D;
    const __nv_bfloat16* x = static_cast<const __nv_bfloat16*>(final_tap) + D;
    const int kb = 9 * D;
    if (plan_conv_halo(&d->g, x, B, h, h, D, D, (int64_t)h * D, (int64_t)T * D, 2,
                       static_cast<const __nv_bfloat16*>(d->w.conv_w_split), D, 2 * kb, ep, 128) != VPE_OK)
      VPE_TRY(plan_gemm_conv(&d->g, x, B, h, h, D, D, (int64_t)h * D, (int64_t)T * D, 3, 64,
                             static_cast<const __nv_bfloat16*>(d->w.conv_w_split), D, 2 * kb, 2 * kb, ep, 64));
    d->bound = final_tap;
  }
  VPE_TRY(launch_gemm(d->g, st));
  const int npix = B * d->P;
  det_1x1_kernel<<<(npix + PX_PER_BLK - 1) / PX_PER_BLK, DET_THREADS, 0, st>>>(d->hidden, npix, d->P, D, A, d->wT, d->bcat, d->obj,
                                                         d->deltas);
  VPE_CUDA_TRY(cudaGetLastError());
  const size_t topk_smem = (size_t)n * 4;
  static OncePerDevice topk_attr;
  if (topk_attr.first()) {
    VPE_CUDA_TRY(cudaFuncSetAttribute(det_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, TOPK_SMEM_MAX));
  }
  det_topk_kernel<<<B, 1024, topk_smem, st>>>(d->obj, d->deltas, n, K, d->cfg, h, d->cbox, d->cscore, d->cidx, d->cvalid,
                                      o->top_index);
  VPE_CUDA_TRY(cudaGetLastError());
  const int nb = (K + NMS_BLK - 1) / NMS_BLK;
  det_nms_mask_kernel<<<dim3(nb, nb, B), NMS_BLK, 0, st>>>(d->cbox, K, d->cfg.nms_thresh, d->mask);
  VPE_CUDA_TRY(cudaGetLastError());
  static OncePerDevice attr;
  const size_t smem = (size_t)K * NWORDS * 8;
  if (attr.first()) {
    cudaFuncSetAttribute(det_nms_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, KMAX * NWORDS * 8);
    max_smem_carveout(det_nms_scan_kernel);
    max_smem_carveout(det_1x1_kernel);
    max_smem_carveout(det_topk_kernel);
    max_smem_carveout(det_nms_mask_kernel);
  }
  det_nms_scan_kernel<<<B, 512, smem, st>>>(d->mask, d->cvalid, d->cbox, d->cscore, d->cidx, K,
                                            d->cfg.post_nms_top_n, o->boxes, o->scores, o->index, o->count);
  VPE_CUDA_TRY(cudaGetLastError());
  count_launches(5);
  if (o->objectness)
    VPE_CUDA_TRY(cudaMemcpyAsync(o->objectness, d->obj, (size_t)B * n * 4, cudaMemcpyDeviceToDevice, st));
  if (o->deltas)
    VPE_CUDA_TRY(cudaMemcpyAsync(o->deltas, d->deltas, (size_t)B * n * 16, cudaMemcpyDeviceToDevice, st));
  return VPE_OK;
}
