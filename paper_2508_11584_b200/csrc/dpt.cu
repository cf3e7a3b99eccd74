// DPT depth head ("b200_dpt") on sm_100a, NHWC bf16 end to end.
//
// Oracle: oracle/dpt.py (transformers modeling_depth_anything.py:31-308). Mapping:
//   reassemble 0/1  1x1 proj composed with ConvTranspose(k=s=4/2) into ONE GEMM read in place from
//                   the ring tap (cls row skipped by the TMA map), scatter epilogue -> NHWC
//   reassemble 2    1x1 proj GEMM;  reassemble 3: 1x1 proj GEMM, im2col, 3x3/s2 GEMM
//   neck convs      3x3 implicit GEMM (TMA 4D boxes, zero padding from OOB fill), epilogue also
//                   writes relu(x) for the following pre-activation residual unit
//   fusion          RCU convs with bias/residual/upsampled-skip adds fused into the epilogue;
//                   the 1x1 projection is applied BEFORE the align_corners=True x2 upsample
//                   (both linear, weights sum to 1 -> identical math, 4x fewer FLOPs)
//   head            conv1 3x3, bilinear to (14h,14w), conv2 3x3 with ReLU -> 1x1 -> ReLU*max_depth
//                   fused into conv2's epilogue (depth written directly, pre-ReLU map optional).
//                   Both head resizes are fused into the conv that consumes them (conv_up_kernel:
//                   the halo is interpolated in smem from a TMA-staged source box, so the 2x and
//                   14h-wide maps never reach HBM; bit-identical to resize + halo conv).
//                   VPE_DPT_UNFUSED=1 restores the resize kernels (A/B). Round 1's attempt
//                   interpolated from global memory inside the producer and lost to the resize
//                   kernel + halo conv (head1 290 vs 215 us, head2 373 vs 350 us at B=16).
#include <cuda_runtime.h>

#include <cstdlib>
#include <new>

#include "gemm.cuh"
#include "misc.cuh"
#include "runtime.h"
#include "util.cuh"

using namespace vpe;
typedef __nv_bfloat16 bf16;

static int pad_ch(int c) { return (c % 64 == 0) ? c : (c == 32 ? 32 : (c + 63) / 64 * 64); }
static int bk_for(int cp) { return cp % 64 == 0 ? 64 : 32; }
static int bn_for(int n) { return n <= 32 ? 32 : (n <= 64 ? 64 : 128); }

struct vpe_dpt {
  vpe_dpt_config cfg;
  vpe_dpt_weights w;
  int h = 0, S[4] = {0}, C[4] = {0}, Cp[4] = {0}, F = 0, Fh = 0, Hh = 0, R = 0, B = 0;
  bf16 *r[4] = {nullptr}, *r3a = nullptr, *r3col = nullptr;
  bf16 *f[4] = {nullptr}, *fr[4] = {nullptr};
  bf16 *t = nullptr, *hid = nullptr, *hidr = nullptr, *o = nullptr, *po = nullptr, *fused = nullptr;
  bf16 *head_in = nullptr, *h1 = nullptr, *h1up = nullptr;
  float *depth_pre_tmp = nullptr;
  const void* bound[4] = {nullptr};
  GemmPlan rs[4], rs3conv, neck[4], rcu[4][4], proj[4], head1;
  GemmPlan head2;  // epilogue pointers patched per call (depth outputs)
  bool fused_up = false;  // head1 / head2 read the un-resized maps (conv_up_kernel)
  bf16 *wpack1 = nullptr, *wpack2 = nullptr;  // their dy-stacked weights
  // Reassemble + neck branches 0..2 run on side streams beside branch 3 and the first fusion
  // stages (forked / joined with events, so graph capture records the same DAG).
  cudaStream_t side[3] = {nullptr};
  cudaEvent_t fork = nullptr, join[3] = {nullptr};
  int side_prio = 1 << 30;
  int nkern = 0;
};

// Default: on for small batches, where each branch kernel leaves most SMs idle (batch-1 depth
// p50 0.94 -> 0.88 ms); off at batch >= 8, where the branches already fill the GPU and the
// engine overlaps the head with the next batch's backbone anyway (C2 unchanged within noise).
// VPE_DPT_BRANCHES=0/1 forces it.
static int& dpt_branch_mode() {
  static int v = [] {
    const char* e = getenv("VPE_DPT_BRANCHES");
    return e ? (atoi(e) != 0 ? 1 : 0) : -1;
  }();
  return v;
}

static bool dpt_branches_enabled(int B) {
  const int v = dpt_branch_mode();
  return v < 0 ? B < 8 : v != 0;
}

extern "C" int vpe_set_dpt_branches(int32_t mode) {
  if (mode < -1 || mode > 1) return VPE_E_VALUE;
  dpt_branch_mode() = mode;
  return VPE_OK;
}

// Side streams carry the caller's priority (the engine runs heads above the producer).
static int dpt_side_streams(vpe_dpt* d, cudaStream_t s) {
  int prio = 0;
  if (cudaStreamGetPriority(s, &prio) != cudaSuccess) return VPE_E_CUDA;
  if (d->side[0] && prio == d->side_prio) return VPE_OK;
  for (int i = 0; i < 3; ++i) {
    if (d->side[i]) cudaStreamDestroy(d->side[i]);
    d->side[i] = nullptr;
  }
  for (int i = 0; i < 3; ++i)
    if (cudaStreamCreateWithPriority(&d->side[i], cudaStreamNonBlocking, prio) != cudaSuccess) return VPE_E_CUDA;
  if (!d->fork && cudaEventCreateWithFlags(&d->fork, cudaEventDisableTiming) != cudaSuccess) return VPE_E_CUDA;
  for (int i = 0; i < 3; ++i)
    if (!d->join[i] && cudaEventCreateWithFlags(&d->join[i], cudaEventDisableTiming) != cudaSuccess) return VPE_E_CUDA;
  d->side_prio = prio;
  return VPE_OK;
}

static int conv_plan(GemmPlan* g, const bf16* x, int B, int S, int Cp, const void* w, int N, const EpiParams& ep) {
  const int kb = 9 * Cp;
  if (plan_conv_halo(g, x, B, S, S, Cp, Cp, (int64_t)S * Cp, (int64_t)S * S * Cp, 1, static_cast<const bf16*>(w), N,
                     kb, ep, bn_for(N)) == VPE_OK)
    return VPE_OK;
  return plan_gemm_conv(g, x, B, S, S, Cp, Cp, (int64_t)S * Cp, (int64_t)S * S * Cp, 3, bk_for(Cp),
                        static_cast<const bf16*>(w), N, kb, kb, ep, bn_for(N));
}

static EpiParams conv_ep(int N, const float* bias, bf16* out, int ldo, int act, const bf16* add1, const bf16* add2,
                         bf16* out_relu) {
  EpiParams e;
  e.kind = EPI_CONV;
  e.act = act;
  e.N = N;
  e.bias = bias;
  e.out = out;
  e.ldo = ldo;
  e.add1 = add1;
  e.add2 = add2;
  e.out_relu = out_relu;
  return e;
}

extern "C" int vpe_dpt_destroy(vpe_dpt* d) {
  if (!d) return VPE_OK;
  for (int i = 0; i < 4; ++i) {
    cudaFree(d->r[i]);
    cudaFree(d->f[i]);
    cudaFree(d->fr[i]);
  }
  cudaFree(d->r3a);
  cudaFree(d->r3col);
  cudaFree(d->t);
  cudaFree(d->hid);
  cudaFree(d->hidr);
  cudaFree(d->o);
  cudaFree(d->po);
  cudaFree(d->fused);
  cudaFree(d->head_in);
  cudaFree(d->h1);
  cudaFree(d->h1up);
  cudaFree(d->depth_pre_tmp);
  cudaFree(d->wpack1);
  cudaFree(d->wpack2);
  for (int i = 0; i < 3; ++i) {
    if (d->side[i]) cudaStreamDestroy(d->side[i]);
    if (d->join[i]) cudaEventDestroy(d->join[i]);
  }
  if (d->fork) cudaEventDestroy(d->fork);
  delete d;
  return VPE_OK;
}

extern "C" int vpe_dpt_create(const vpe_dpt_config* cfg, const vpe_dpt_weights* w, vpe_dpt** out) {
  if (!cfg || !w || !out) return VPE_E_VALUE;
  if (cfg->resolution % 14 || cfg->dim % 64 || cfg->head_hidden != 32 || cfg->fusion % 64) return VPE_E_CONFIG;
  vpe_dpt* d = new (std::nothrow) vpe_dpt();
  if (!d) return VPE_E_RESOURCE;
  d->cfg = *cfg;
  d->w = *w;
  const int h = cfg->resolution / 14, B = cfg->batch, F = cfg->fusion;
  d->h = h;
  d->B = B;
  d->R = cfg->resolution;
  d->F = F;
  d->Fh = F / 2;
  d->Hh = cfg->head_hidden;
  d->S[0] = 4 * h;
  d->S[1] = 2 * h;
  d->S[2] = h;
  d->S[3] = (h + 1) / 2;
  for (int i = 0; i < 4; ++i) {
    d->C[i] = cfg->neck[i];
    d->Cp[i] = pad_ch(cfg->neck[i]);
  }
  auto fail = [&](int rc) {
    vpe_dpt_destroy(d);
    return rc;
  };
  auto alloc = [&](bf16** p, size_t elems) { return cudaMalloc(p, elems * 2) == cudaSuccess && cudaMemset(*p, 0, elems * 2) == cudaSuccess; };
  const size_t big = (size_t)B * d->S[0] * d->S[0] * F;
  bool ok = true;
  for (int i = 0; i < 4; ++i) {
    ok = ok && alloc(&d->r[i], (size_t)B * d->S[i] * d->S[i] * d->Cp[i]);
    ok = ok && alloc(&d->f[i], (size_t)B * d->S[i] * d->S[i] * F);
    ok = ok && alloc(&d->fr[i], (size_t)B * d->S[i] * d->S[i] * F);
  }
  ok = ok && alloc(&d->r3a, (size_t)B * h * h * d->Cp[3]);
  ok = ok && alloc(&d->r3col, (size_t)B * d->S[3] * d->S[3] * 9 * d->Cp[3]);
  ok = ok && alloc(&d->t, big) && alloc(&d->hid, big) && alloc(&d->hidr, big) && alloc(&d->o, big) &&
       alloc(&d->po, big) && alloc(&d->fused, big);
  const int S4 = 2 * d->S[0];
  ok = ok && alloc(&d->h1, (size_t)B * S4 * S4 * d->Fh);  // head_in / h1up: unfused path only
  ok = ok && cudaMalloc(&d->depth_pre_tmp, (size_t)B * d->R * d->R * 4) == cudaSuccess;
  if (!ok) return fail(VPE_E_RESOURCE);
  int rc;
  // reassemble 3: 3x3 stride-2 conv as im2col + GEMM
  {
    const int C3 = d->C[3], C3p = d->Cp[3], S3 = d->S[3];
    EpiParams e = conv_ep(C3, w->rs3_conv_b, d->r[3], C3p, ACT_NONE, nullptr, nullptr, nullptr);
    if ((rc = plan_gemm_rows(&d->rs3conv, d->r3col, B * S3 * S3, 9 * C3p, 9 * C3p,
                             static_cast<const bf16*>(w->rs3_conv_w), C3, 9 * C3p, 9 * C3p, e, bn_for(C3))))
      return fail(rc);
  }
  // neck 3x3 convs (no bias) -> f[i] and relu(f[i])
  for (int i = 0; i < 4; ++i) {
    EpiParams e = conv_ep(F, nullptr, d->f[i], F, ACT_NONE, nullptr, nullptr, d->fr[i]);
    if ((rc = conv_plan(&d->neck[i], d->r[i], B, d->S[i], d->Cp[i], w->neck_w[i], F, e))) return fail(rc);
  }
  // fusion layers (k = 0 deepest)
  for (int k = 0; k < 4; ++k) {
    const int fi = 3 - k, S = d->S[fi];
    if (k > 0) {
      EpiParams e0 = conv_ep(F, w->rcu_b[k][0], d->t, F, ACT_RELU, nullptr, nullptr, nullptr);
      if ((rc = conv_plan(&d->rcu[k][0], d->fr[fi], B, S, F, w->rcu_w[k][0], F, e0))) return fail(rc);
      EpiParams e1 = conv_ep(F, w->rcu_b[k][1], d->hid, F, ACT_NONE, d->f[fi], d->fused, d->hidr);
      if ((rc = conv_plan(&d->rcu[k][1], d->t, B, S, F, w->rcu_w[k][1], F, e1))) return fail(rc);
    }
    const bf16* in_relu = k > 0 ? d->hidr : d->fr[fi];
    const bf16* in_res = k > 0 ? d->hid : d->f[fi];
    EpiParams e2 = conv_ep(F, w->rcu_b[k][2], d->t, F, ACT_RELU, nullptr, nullptr, nullptr);
    if ((rc = conv_plan(&d->rcu[k][2], in_relu, B, S, F, w->rcu_w[k][2], F, e2))) return fail(rc);
    EpiParams e3 = conv_ep(F, w->rcu_b[k][3], d->o, F, ACT_NONE, in_res, nullptr, nullptr);
    if ((rc = conv_plan(&d->rcu[k][3], d->t, B, S, F, w->rcu_w[k][3], F, e3))) return fail(rc);
    EpiParams ep;
    ep.kind = EPI_BF16;
    ep.N = F;
    ep.bias = w->proj_b[k];
    ep.out = d->po;
    ep.ldo = F;
    if ((rc = plan_gemm_rows(&d->proj[k], d->o, B * S * S, F, F, static_cast<const bf16*>(w->proj_w[k]), F, F, F, ep,
                             bn_for(F))))
      return fail(rc);
  }
  {
    EpiParams e = conv_ep(d->Fh, w->head1_b, d->h1, d->Fh, ACT_NONE, nullptr, nullptr, nullptr);
    EpiParams e2;
    e2.kind = EPI_DEPTH;
    e2.N = d->Hh;
    e2.bias = w->head2_b;
    e2.w3 = w->head3_w;
    e2.b3 = w->head3_b;
    e2.max_depth = cfg->max_depth;
    e2.depth_pre = d->depth_pre_tmp;
    e2.depth = d->depth_pre_tmp;  // patched per call
    const char* uf = getenv("VPE_DPT_UNFUSED");
    d->fused_up = !(uf && uf[0] == '1') && F == 64 && d->Fh == 32 && d->Hh == 32 &&
                  alloc(&d->wpack1, (size_t)3 * 96 * F) && alloc(&d->wpack2, (size_t)3 * 96 * d->Fh) &&
                  plan_conv_up(&d->head1, d->po, B, d->S[0], d->S[0], F, S4, S4, static_cast<const bf16*>(w->head1_w),
                               d->Fh, e, d->wpack1, 0) == VPE_OK &&
                  plan_conv_up(&d->head2, d->h1, B, S4, S4, d->Fh, d->R, d->R, static_cast<const bf16*>(w->head2_w),
                               d->Hh, e2, d->wpack2, 0) == VPE_OK &&
                  cudaDeviceSynchronize() == cudaSuccess;
    if (d->fused_up) {
      *out = d;
      return VPE_OK;
    }
    if (!alloc(&d->head_in, (size_t)B * S4 * S4 * F) || !alloc(&d->h1up, (size_t)B * d->R * d->R * d->Fh))
      return fail(VPE_E_RESOURCE);
    if ((rc = conv_plan(&d->head1, d->head_in, B, S4, F, w->head1_w, d->Fh, e))) return fail(rc);
    if ((rc = conv_plan(&d->head2, d->h1up, B, d->R, d->Fh, w->head2_w, d->Hh, e2))) return fail(rc);
  }
  *out = d;
  return VPE_OK;
}

static int bind_taps(vpe_dpt* d, const void* const* taps) {
  const int D = d->cfg.dim, h = d->h, B = d->B, T = h * h + 1;
  for (int i = 0; i < 4; ++i) {
    if (d->bound[i] == taps[i]) continue;
    const bf16* x = static_cast<const bf16*>(taps[i]) + D;  // skip cls row: tap as NHWC [B,h,h,D]
    EpiParams e;
    int N;
    if (i < 2) {
      const int k = i == 0 ? 4 : 2;
      const int cout_p = (d->C[i] + 31) / 32 * 32;  // weights padded per sub-pixel (heads.py)
      N = k * k * cout_p;
      e.kind = EPI_CONVT;
      e.N = N;
      e.bias = d->w.rs_b[i];
      e.out = d->r[i];
      e.ldo = d->Cp[i];
      e.ct_k = k;
      e.ct_cout = cout_p;
      e.ct_H = h;
      e.ct_W = h;
    } else {
      N = d->C[i];
      e = conv_ep(N, d->w.rs_b[i], i == 2 ? d->r[2] : d->r3a, d->Cp[i], ACT_NONE, nullptr, nullptr, nullptr);
    }
    VPE_TRY(plan_gemm_conv(&d->rs[i], x, B, h, h, D, D, (int64_t)h * D, (int64_t)T * D, 1, 64,
                           static_cast<const bf16*>(d->w.rs_w[i]), N, D, D, e, bn_for(N)));
    d->bound[i] = taps[i];
  }
  return VPE_OK;
}

extern "C" int vpe_dpt_forward(vpe_dpt* d, const void* const* taps, float* depth, float* depth_pre, void* stream) {
  if (!d || !taps || !depth) return VPE_E_VALUE;
  for (int i = 0; i < 4; ++i)
    if (!taps[i]) return VPE_E_VALUE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  VPE_TRY(bind_taps(d, taps));
  const int B = d->B, F = d->F;
  int n = 0;
  const bool br = dpt_branches_enabled(B);
  if (br) {
    VPE_TRY(dpt_side_streams(d, s));
    VPE_CUDA_TRY(cudaEventRecord(d->fork, s));
    for (int i = 0; i < 3; ++i) {
      VPE_CUDA_TRY(cudaStreamWaitEvent(d->side[i], d->fork, 0));
      VPE_TRY(launch_gemm(d->rs[i], d->side[i]));
      VPE_TRY(launch_gemm(d->neck[i], d->side[i]));
      VPE_CUDA_TRY(cudaEventRecord(d->join[i], d->side[i]));
    }
    VPE_TRY(launch_gemm(d->rs[3], s));
    VPE_TRY(launch_im2col_s2(d->r3a, B, d->h, d->h, d->Cp[3], d->r3col, s));
    VPE_TRY(launch_gemm(d->rs3conv, s));
    VPE_TRY(launch_gemm(d->neck[3], s));
    n += 9;
  } else {
    for (int i = 0; i < 4; ++i) {
      VPE_TRY(launch_gemm(d->rs[i], s));
      ++n;
    }
    VPE_TRY(launch_im2col_s2(d->r3a, B, d->h, d->h, d->Cp[3], d->r3col, s));
    VPE_TRY(launch_gemm(d->rs3conv, s));
    n += 2;
    for (int i = 0; i < 4; ++i) {
      VPE_TRY(launch_gemm(d->neck[i], s));
      ++n;
    }
  }
  for (int k = 0; k < 4; ++k) {
    const int fi = 3 - k, S = d->S[fi];
    if (br && k > 0) VPE_CUDA_TRY(cudaStreamWaitEvent(s, d->join[fi], 0));
    for (int j = (k > 0 ? 0 : 2); j < 4; ++j) {
      VPE_TRY(launch_gemm(d->rcu[k][j], s));
      ++n;
    }
    VPE_TRY(launch_gemm(d->proj[k], s));
    ++n;
    if (k == 3 && d->fused_up) break;  // the x2 resize happens inside head1
    const int So = k < 3 ? d->S[fi - 1] : 2 * d->S[0];
    VPE_TRY(launch_bilinear_ac(d->po, B, S, S, F, k < 3 ? d->fused : d->head_in, So, So, F, s));
    ++n;
  }
  VPE_TRY(launch_gemm(d->head1, s));
  if (!d->fused_up) {
    VPE_TRY(launch_bilinear_ac(d->h1, B, 2 * d->S[0], 2 * d->S[0], d->Fh, d->h1up, d->R, d->R, d->Fh, s));
    ++n;
  }
  GemmPlan g2 = d->head2;
  g2.p.ep.depth = depth;
  g2.p.ep.depth_pre = depth_pre ? depth_pre : d->depth_pre_tmp;
  VPE_TRY(launch_gemm(g2, s));
  n += 2;
  count_launches(n);
  return VPE_OK;
}
