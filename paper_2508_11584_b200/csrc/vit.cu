// DINOv2 ViT backbone forward on sm_100a: plan once (TMA maps, workspaces), enqueue per frame.
//
// Per block (modeling_dinov2.py:348-386):  LN1 -> QKV GEMM(+bias) -> tcgen05 attention ->
// out-proj GEMM with fused bias*LayerScale+residual into the fp32 stream -> LN2 -> FC1 GEMM with
// fused bias+erf-GELU -> FC2 GEMM with fused bias*LayerScale+residual. Tap LayerNorms
// (modeling_dinov2.py:605-618) are fused into the next block's LN1 pass and written straight
// into the ring slot the caller passes (zero-copy publish).
#include <cstdlib>
#include <cstring>
#include <new>

#include "attention.cuh"
#include "gemm.cuh"
#include "misc.cuh"
#include "runtime.h"
#include "util.cuh"

using namespace vpe;

struct vpe_vit {
  vpe_vit_config cfg;
  vpe_vit_weights w;
  int T = 0, Np = 0, M = 0;
  float* resid = nullptr;
  __nv_bfloat16 *xln = nullptr, *qkv = nullptr, *ctx = nullptr, *hid = nullptr, *im2col = nullptr;
  GemmPlan patch;
  GemmPlan qkv_g[VPE_MAX_LAYERS], proj_g[VPE_MAX_LAYERS], fc1_g[VPE_MAX_LAYERS], fc2_g[VPE_MAX_LAYERS];
  AttnPlan attn;
  // proj / FC2 with the following LayerNorm in their epilogue (gemm_resid_ln_kernel): D = 384 at
  // large M only (the kernel owns whole rows: one CTA per 128-row block)
  GemmPlan proj_rl[VPE_MAX_LAYERS], fc2_rl[VPE_MAX_LAYERS];
  bool resid_ln = false;
};

static constexpr int KPATCH = 640;

// BN per GEMM: wide tiles amortise the A re-read (the K=384 GEMMs are L2-bandwidth bound at
// BN=128: FC1+GELU 32.7 -> 28.9 us at BN=256, tools/microbench.py); at small M fall back to
// narrower tiles so the persistent grid still covers the SMs.
static int pick_bn(int N, int M) {
  const int m_tiles = (M + 127) / 128;
  // 256-wide tiles. (BN = 192 for the N = 384 proj / FC2 wins alone -- FC2 with the residual
  // epilogue 25.4 -> 22.8 us, graph-timed microbench -- but made the backbone step slower,
  // 2.15 -> 2.23 ms, in the pipelined engine; measured twice this round.)
  static const int bn384 = getenv("VPE_BN384") ? atoi(getenv("VPE_BN384")) : 256;  // A/B experiments
  int bn = N == 384 ? bn384 : 256;
  while (bn > 64 && m_tiles * ((N + bn - 1) / bn) < 148) bn = bn == 192 ? 128 : bn >> 1;
  return bn;
}

extern "C" int vpe_vit_create(const vpe_vit_config* cfg, const vpe_vit_weights* w, vpe_vit** out) {
  if (!cfg || !w || !out) return VPE_E_VALUE;
  const int D = cfg->dim, L = cfg->depth, R = cfg->resolution, B = cfg->batch;
  if (L < 1 || L > VPE_MAX_LAYERS || D % 128 || D != cfg->heads * 64 || R % 14 || B < 1) return VPE_E_CONFIG;
  if (cfg->taps[3] != L) return VPE_E_CONFIG;
  vpe_vit* v = new (std::nothrow) vpe_vit();
  if (!v) return VPE_E_RESOURCE;
  v->cfg = *cfg;
  v->w = *w;
  const int h = R / 14;
  v->Np = h * h;
  v->T = v->Np + 1;
  v->M = B * v->T;
  const int M = v->M, Hd = cfg->mlp_hidden;
  auto fail = [&](int rc) {
    vpe_vit_destroy(v);
    return rc;
  };
  if (cudaMalloc(&v->resid, (size_t)M * D * 4) != cudaSuccess) return fail(VPE_E_RESOURCE);
  if (cudaMalloc(&v->xln, (size_t)M * D * 2) != cudaSuccess) return fail(VPE_E_RESOURCE);
  if (cudaMalloc(&v->qkv, (size_t)M * 3 * D * 2) != cudaSuccess) return fail(VPE_E_RESOURCE);
  if (cudaMalloc(&v->ctx, (size_t)M * D * 2) != cudaSuccess) return fail(VPE_E_RESOURCE);
  if (cudaMalloc(&v->hid, (size_t)M * Hd * 2) != cudaSuccess) return fail(VPE_E_RESOURCE);
  if (cudaMalloc(&v->im2col, (size_t)B * v->Np * KPATCH * 2) != cudaSuccess) return fail(VPE_E_RESOURCE);
  int rc;
  {
    EpiParams ep;
    ep.kind = EPI_PATCH;
    ep.N = D;
    ep.bias = w->patch_b;
    ep.resid = v->resid;
    ep.ldr = D;
    ep.pos = w->pos;
    ep.rows_per_img = v->Np;
    rc = plan_gemm_rows(&v->patch, v->im2col, B * v->Np, KPATCH, KPATCH,
                        static_cast<const __nv_bfloat16*>(w->patch_w), D, KPATCH, KPATCH, ep, pick_bn(D, M));
    if (rc) return fail(rc);
  }
  for (int l = 0; l < L; ++l) {
    EpiParams e;
    e.kind = EPI_BF16;
    e.N = 3 * D;
    e.bias = w->qkv_b[l];
    e.out = v->qkv;
    e.ldo = 3 * D;
    if ((rc = plan_gemm_rows(&v->qkv_g[l], v->xln, M, D, D, static_cast<const __nv_bfloat16*>(w->qkv_w[l]), 3 * D, D,
                             D, e, pick_bn(3 * D, M))))
      return fail(rc);
    EpiParams p;
    p.kind = EPI_RESID;
    p.N = D;
    p.bias = w->proj_b[l];
    p.scale = w->ls1[l];
    p.resid = v->resid;
    p.ldr = D;
    if ((rc = plan_gemm_rows(&v->proj_g[l], v->ctx, M, D, D, static_cast<const __nv_bfloat16*>(w->proj_w[l]), D, D, D,
                             p, pick_bn(D, M))))
      return fail(rc);
    EpiParams f1;
    f1.kind = EPI_BF16;
    f1.act = ACT_GELU;
    f1.N = Hd;
    f1.bias = w->fc1_b[l];
    f1.out = v->hid;
    f1.ldo = Hd;
    if ((rc = plan_gemm_rows(&v->fc1_g[l], v->xln, M, D, D, static_cast<const __nv_bfloat16*>(w->fc1_w[l]), Hd, D, D,
                             f1, pick_bn(Hd, M))))
      return fail(rc);
    EpiParams f2;
    f2.kind = EPI_RESID;
    f2.N = D;
    f2.bias = w->fc2_b[l];
    f2.scale = w->ls2[l];
    f2.resid = v->resid;
    f2.ldr = D;
    if ((rc = plan_gemm_rows(&v->fc2_g[l], v->hid, M, Hd, Hd, static_cast<const __nv_bfloat16*>(w->fc2_w[l]), D, Hd,
                             Hd, f2, pick_bn(D, M))))
      return fail(rc);
  }
  if ((rc = plan_attention(&v->attn, v->qkv, v->ctx, B, v->T, D, cfg->heads))) return fail(rc);
  {
    // Measured (tools/microbench.py --only rln, M = 16400): proj + LN2 20.0 -> 18.9 us, FC2 + LN1
    // 32.9 -> 29.5 us. VPE_RESID_LN=0 keeps the separate LayerNorm kernels.
    const char* e = getenv("VPE_RESID_LN");
    v->resid_ln = D == 384 && (M + 127) / 128 >= 100 && !(e && e[0] == '0');
    for (int l = 0; v->resid_ln && l < L; ++l) {
      if ((rc = plan_gemm_resid_ln(&v->proj_rl[l], v->ctx, M, D, static_cast<const __nv_bfloat16*>(w->proj_w[l]),
                                   w->proj_b[l], w->ls1[l], v->resid, w->ln2_w[l], w->ln2_b[l], cfg->ln_eps, v->xln,
                                   nullptr, nullptr)))
        return fail(rc);
      const bool last = l + 1 == L;
      if ((rc = plan_gemm_resid_ln(&v->fc2_rl[l], v->hid, M, Hd, static_cast<const __nv_bfloat16*>(w->fc2_w[l]),
                                   w->fc2_b[l], w->ls2[l], v->resid, last ? w->norm_w : w->ln1_w[l + 1],
                                   last ? w->norm_b : w->ln1_b[l + 1], cfg->ln_eps, last ? nullptr : v->xln,
                                   last ? nullptr : w->norm_w, last ? nullptr : w->norm_b)))
        return fail(rc);
    }
  }
  *out = v;
  return VPE_OK;
}

extern "C" int vpe_vit_destroy(vpe_vit* v) {
  if (!v) return VPE_OK;
  cudaFree(v->resid);
  cudaFree(v->xln);
  cudaFree(v->qkv);
  cudaFree(v->ctx);
  cudaFree(v->hid);
  cudaFree(v->im2col);
  delete v;
  return VPE_OK;
}

extern "C" int vpe_vit_residual(vpe_vit* v, const float** resid) {
  if (!v || !resid) return VPE_E_VALUE;
  *resid = v->resid;
  return VPE_OK;
}

// Shared tail of both entry points: patch GEMM, the L blocks, final LN into taps[3].
static int vit_blocks_impl(vpe_vit* v, void* const* taps, cudaStream_t s);
static int vit_blocks(vpe_vit* v, void* const* taps, cudaStream_t s) {
  pdl_scope() = 1;  // kernels after the patch im2col may overlap their predecessor's drain
  const int rc = vit_blocks_impl(v, taps, s);
  pdl_scope() = 0;
  return rc;
}
static int vit_blocks_impl(vpe_vit* v, void* const* taps, cudaStream_t s) {
  const vpe_vit_config& c = v->cfg;
  const vpe_vit_weights& w = v->w;
  const int D = c.dim, M = v->M;
  VPE_TRY(launch_gemm(v->patch, s));
  count_launches(1);
  int tap = 0;
  if (v->resid_ln) {
    __nv_bfloat16* t0 = (c.taps[0] == 0) ? static_cast<__nv_bfloat16*>(taps[tap++]) : nullptr;
    VPE_TRY(launch_layernorm(v->resid, M, D, w.ln1_w[0], w.ln1_b[0], c.ln_eps, v->xln, w.norm_w, w.norm_b, t0, s));
    for (int l = 0; l < c.depth; ++l) {
      VPE_TRY(launch_gemm(v->qkv_g[l], s));
      VPE_TRY(launch_attention(v->attn, s));
      VPE_TRY(launch_gemm_resid_ln(v->proj_rl[l], nullptr, nullptr, s));
      VPE_TRY(launch_gemm(v->fc1_g[l], s));
      if (l + 1 < c.depth) {
        __nv_bfloat16* t = (tap < 3 && c.taps[tap] == l + 1) ? static_cast<__nv_bfloat16*>(taps[tap++]) : nullptr;
        VPE_TRY(launch_gemm_resid_ln(v->fc2_rl[l], nullptr, t, s));
      } else {
        VPE_TRY(launch_gemm_resid_ln(v->fc2_rl[l], static_cast<__nv_bfloat16*>(taps[3]), nullptr, s));
      }
      count_launches(5);
    }
    count_launches(1);
    return VPE_OK;
  }
  for (int l = 0; l < c.depth; ++l) {
    // LN1 of block l; if block l-1 was a tap, the same pass writes the tap LN into the ring slot
    __nv_bfloat16* tap_out = nullptr;
    if (tap < 3 && c.taps[tap] == l) tap_out = static_cast<__nv_bfloat16*>(taps[tap++]);
    VPE_TRY(launch_layernorm(v->resid, M, D, w.ln1_w[l], w.ln1_b[l], c.ln_eps, v->xln, w.norm_w, w.norm_b, tap_out,
                             s));
    VPE_TRY(launch_gemm(v->qkv_g[l], s));
    VPE_TRY(launch_attention(v->attn, s));
    VPE_TRY(launch_gemm(v->proj_g[l], s));
    VPE_TRY(launch_layernorm(v->resid, M, D, w.ln2_w[l], w.ln2_b[l], c.ln_eps, v->xln, nullptr, nullptr, nullptr, s));
    VPE_TRY(launch_gemm(v->fc1_g[l], s));
    VPE_TRY(launch_gemm(v->fc2_g[l], s));
    count_launches(7);
  }
  VPE_TRY(launch_layernorm(v->resid, M, D, w.norm_w, w.norm_b, c.ln_eps, static_cast<__nv_bfloat16*>(taps[3]),
                           nullptr, nullptr, nullptr, s));
  count_launches(1);
  return VPE_OK;
}

extern "C" int vpe_vit_forward(vpe_vit* v, const void* pixels_u8, void* const* taps, void* stream) {
  if (!v || !pixels_u8 || !taps) return VPE_E_VALUE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const vpe_vit_config& c = v->cfg;
  VPE_TRY(launch_patch_im2col(static_cast<const uint8_t*>(pixels_u8), v->im2col, c.batch, c.resolution, KPATCH,
                              v->resid, v->w.cls_pos0, c.dim, s));
  count_launches(1);
  return vit_blocks(v, taps, s);
}

extern "C" int vpe_vit_forward_camera(vpe_vit* v, const void* frames_hwc_u8, int32_t height, int32_t width,
                                      void* const* taps, void* stream) {
  if (!v || !frames_hwc_u8 || !taps) return VPE_E_VALUE;
  if (height < 1 || width < 1) return VPE_E_SHAPE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const vpe_vit_config& c = v->cfg;
  VPE_TRY(launch_camera_im2col(static_cast<const uint8_t*>(frames_hwc_u8), height, width, v->im2col, c.batch,
                               c.resolution, KPATCH, v->resid, v->w.cls_pos0, c.dim, s));
  count_launches(1);
  return vit_blocks(v, taps, s);
}

extern "C" int vpe_op_camera_im2col(const void* frames_hwc_u8, int32_t B, int32_t height, int32_t width,
                                    int32_t resolution, void* out_bf16, void* stream) {
  if (!frames_hwc_u8 || !out_bf16 || B < 1 || resolution % 14) return VPE_E_VALUE;
  // im2col rows only: a scratch cls/residual target is not needed (D = 0 writes nothing)
  VPE_TRY(launch_camera_im2col(static_cast<const uint8_t*>(frames_hwc_u8), height, width,
                               static_cast<__nv_bfloat16*>(out_bf16), B, resolution, KPATCH, nullptr, nullptr, 0,
                               static_cast<cudaStream_t>(stream)));
  count_launches(1);
  return VPE_OK;
}
