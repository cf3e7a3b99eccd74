// tcgen05/TMEM/TMA GEMM engine for sm_100a: D[M,N] = A[M,K] * B[N,K]^T with fused epilogues.
//
// A is either a row-major activation matrix (mode ROWS) or an NHWC bf16 image read as an
// implicit-GEMM convolution (mode CONV, kernel 1x1 or 3x3, stride 1, zero padding supplied by
// TMA out-of-bounds fill). B is a K-major bf16 weight matrix. One CTA computes a 128 x BN tile:
// warp 0 issues TMA, warp 1 issues tcgen05.mma (accumulator in TMEM), warps 2-5 run the epilogue.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace vpe {

enum EpiKind : int {
  EPI_BF16 = 0,   // out_bf16 = act(acc + bias)            [+ optional relu copy]
  EPI_RESID = 1,  // resid_f32 += scale * (acc + bias)     (LayerScale + residual)
  EPI_PATCH = 2,  // resid_f32[row remapped past cls] = acc + bias + pos
  EPI_F32 = 3,    // out_f32 = acc + bias
  EPI_CONV = 4,   // out_bf16 = act(acc + bias + add1 + add2) [+ relu copy]  (NHWC)
  EPI_CONVT = 5,  // ConvTranspose(k=s) scatter into NHWC: col = (ky*k+kx)*cout + co
  EPI_DEPTH = 6,  // depth = relu(b3 + sum_c relu(acc_c + bias_c) * w3_c) * max_depth
};
enum Act : int { ACT_NONE = 0, ACT_GELU = 1, ACT_RELU = 2 };

struct EpiParams {
  int kind = EPI_BF16;
  int act = ACT_NONE;
  int N = 0;                       // valid output columns
  const float* bias = nullptr;     // [N]
  const float* scale = nullptr;    // [N] (EPI_RESID)
  void* out = nullptr;             // bf16 / f32 output
  int64_t ldo = 0;                 // output row (pixel) pitch, elements
  __nv_bfloat16* out_relu = nullptr;  // optional relu(out) copy, same pitch as out
  float* resid = nullptr;          // fp32 residual stream
  int64_t ldr = 0;
  const __nv_bfloat16* add1 = nullptr;  // NHWC adds (pitch ldo)
  const __nv_bfloat16* add2 = nullptr;
  const float* pos = nullptr;      // EPI_PATCH: [T, N] position embedding
  int rows_per_img = 0;            // EPI_PATCH: Np
  int ct_k = 0, ct_cout = 0;       // EPI_CONVT: factor, real out channels
  int ct_H = 0, ct_W = 0;          // EPI_CONVT: input grid (output grid = k*H x k*W)
  const float* w3 = nullptr;       // EPI_DEPTH: [32]
  float b3 = 0.f, max_depth = 1.f;
  float* depth_pre = nullptr;      // EPI_DEPTH outputs [pixels]
  float* depth = nullptr;
};

// LayerNorm fused into the residual GEMM's epilogue (gemm_resid_ln_kernel)
struct LnParams {
  const float* x = nullptr;  // fp32 residual stream [M, D]
  const float* w = nullptr;
  const float* b = nullptr;
  float eps = 0.f;
  const float* tw = nullptr;  // optional second affine written to `tap` (the ring's tap LN)
  const float* tb = nullptr;
  __nv_bfloat16* tap = nullptr;
};

struct GemmParams {
  int kblocks = 0;     // K blocks on the B side
  int kblocks_a = 0;   // A-side K blocks before wrap-around (split-precision weights repeat A)
  int mode = 0;        // 0 rows, 1 conv
  int M = 0;           // mode 0: valid rows
  int ks = 1;          // conv kernel size
  int cchunks = 1;     // channel chunks (of BK) per tap
  int H = 0, W = 0, bw = 0, bh = 0, tiles_x = 0, tiles_per_img = 0;
  int m_tiles = 0, n_tiles = 0;  // persistent tile space
  int tma_out = 0;               // 1: epilogue leaves through TMA store / reduce-add (tout)
  int hp = 0, rows_box = 0;      // halo conv: virtual row pitch P, halo rows per stage
  int flat = 0;                  // halo conv, W < 128: tiles are 128 consecutive positions of the
                                 // image's P-pitched layout (rows straddle tiles), see plan_conv_halo
  int parts = 1, kcp = 0;        // halo conv: split-precision weight parts, K extent per tap (Cpad)
  // upsample-fused conv (conv_up_kernel): source map Hs x Ws, align_corners scales, source box
  int up_hs = 0, up_ws = 0, up_rows = 0, up_cols = 0, up_stages = 0, up_src_bytes = 0, up_box_bytes = 0;
  float up_sh = 0.f, up_sw = 0.f;
  int pdl_late = 0;              // 1: signal programmatic dependents after the last TMA load, not at start
  int trace = 0;                 // diagnostics: record the MMA timeline of CTA 0
  int dbg = 0;                   // diagnostics (halo conv, VPE_HALO_DBG): 1 no stores, 2 no A reloads, 4 no MMA
  EpiParams ep;
  LnParams ln;
};

struct GemmPlan {
  CUtensorMap ta;
  CUtensorMap tb;
  CUtensorMap tout;
  GemmParams p;
  dim3 grid;
  int bn = 0, bk = 0;
  int halo_kc = 0;  // > 0: conv_halo_kernel<bn, halo_kc, halo_rt>
  int halo_rt = 1;
  int halo_wres = 0;  // 1: conv_halo_kernel<.., WRES> (all weight tiles resident in smem)
  int up_kc = 0;      // > 0: conv_up_kernel<bn, up_kc, halo_rt> (resize fused into the halo builder)
  int resid_ln = 0; // 1: gemm_resid_ln_kernel (residual GEMM + the next LayerNorm in the epilogue)
  CUtensorMap tx;   // resid_ln: bf16 LayerNorm output map
  size_t smem = 0;
};

// 3x3 / stride 1 / pad 1 conv with a shared halo tile (see gemm.cu). X: NHWC with Cp channels
// (multiple of 32), pitches in elements; weights [N, parts*9*Cp] tap-major. Returns VPE_E_SHAPE
// when the halo tiling would waste too much of the 128-row MMA (caller falls back to
// plan_gemm_conv).
int plan_conv_halo(GemmPlan* g, const __nv_bfloat16* X, int nimg, int H, int W, int Cp, int64_t pitch_px,
                   int64_t pitch_row, int64_t pitch_img, int parts, const __nv_bfloat16* B, int N, int64_t ldb,
                   const EpiParams& ep, int bn);

// 3x3 / stride 1 / pad 1 conv of the align_corners=True bilinear resize of X (NHWC [nimg, Hs, Ws,
// Cp], Cp = 32 or 64, dense) to Ho x Wo (Wo >= 128), without materialising the resized map: the
// halo tiles are interpolated in shared memory from TMA-staged source boxes. Bit-identical to
// launch_bilinear_ac followed by the same conv. Weights [N = 32, 9*Cp] tap-major, repacked
// (stream-ordered) into wpack (3 * 96 * Cp bf16, caller-owned, kept for the plan's lifetime);
// B null: wpack was packed already (pack_conv_up_weights).
int pack_conv_up_weights(const __nv_bfloat16* B, int Cp, __nv_bfloat16* wpack, cudaStream_t stream);
int plan_conv_up(GemmPlan* g, const __nv_bfloat16* X, int nimg, int Hs, int Ws, int Cp, int Ho, int Wo,
                 const __nv_bfloat16* B, int N, const EpiParams& ep, __nv_bfloat16* wpack, cudaStream_t stream);

// --- host-side builders (gemm.cu) ---
bool tma_available();
// Row-major A [M, K] (pitch lda elements) times K-major weights B [N, Kb] (pitch ldb).
// Kb may be a multiple of K (split-precision weights concatenated along K; A repeats).
int plan_gemm_rows(GemmPlan* g, const __nv_bfloat16* A, int M, int K, int64_t lda,
                   const __nv_bfloat16* B, int N, int Kb, int64_t ldb, const EpiParams& ep, int bn);
// NHWC image X (channels C real, pitches in elements: pixel, row, image) as implicit-GEMM conv
// input; weights B [N, Kb] with Kb = ks*ks*Cpad (+ repeats), tap-major then channel.
int plan_gemm_conv(GemmPlan* g, const __nv_bfloat16* X, int nimg, int H, int W, int C,
                   int64_t pitch_px, int64_t pitch_row, int64_t pitch_img, int ks, int bk,
                   const __nv_bfloat16* B, int N, int Kb, int64_t ldb, const EpiParams& ep, int bn);
int launch_gemm(const GemmPlan& g, cudaStream_t stream);
// resid [M, 384] fp32 += ls * (A W^T + bias) (A bf16 [M, K], W [384, K]); then xln = LN(resid)
// with (ln_w, ln_b) in bf16 and optionally tap = LN(resid) with (tw, tb). xln / tap pointers may
// be given at launch (ring slots); a null xln at plan and launch skips that output.
int plan_gemm_resid_ln(GemmPlan* g, const __nv_bfloat16* A, int M, int K, const __nv_bfloat16* W, const float* bias,
                       const float* ls, float* resid, const float* ln_w, const float* ln_b, float eps,
                       __nv_bfloat16* xln, const float* tw, const float* tb);
int launch_gemm_resid_ln(const GemmPlan& g, __nv_bfloat16* xln, __nv_bfloat16* tap, cudaStream_t stream);

}  // namespace vpe

namespace vpe {
// cuTensorMapEncodeTiled wrapper (bf16, zero OOB fill); dims/strides innermost first.
int encode_tma(CUtensorMap* m, int rank, const void* ptr, const uint64_t* dims, const uint64_t* strides_bytes,
               const uint32_t* box, CUtensorMapSwizzle swz);
}  // namespace vpe
