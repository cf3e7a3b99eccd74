// C ABI: single-op entry points, streams, events, CUDA graphs, launch accounting.
#include <atomic>
#include <chrono>
#include <new>

#include "attention.cuh"
#include "gemm.cuh"
#include "misc.cuh"
#include "runtime.h"
#include "util.cuh"

using namespace vpe;

namespace {
std::atomic<int64_t> g_launches{0};
thread_local bool t_capturing = false;
thread_local int64_t t_captured = 0;
}  // namespace

namespace vpe {
void count_launches(int64_t n) {
  if (t_capturing)
    t_captured += n;
  else
    g_launches.fetch_add(n, std::memory_order_relaxed);
}
}  // namespace vpe

struct vpe_graph {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int64_t kernels = 0;
};

extern "C" {

int64_t vpe_kernel_launches(void) { return g_launches.load(); }

const char* vpe_status_str(int s) {
  switch (s) {
    case VPE_OK: return "ok";
    case VPE_E_ENGINE: return "EngineError";
    case VPE_E_ALREADY_EXISTS: return "AlreadyExists";
    case VPE_E_NOT_FOUND: return "NotFound";
    case VPE_E_RESOURCE: return "ResourceError";
    case VPE_E_CORRUPT_HANDLE: return "CorruptHandle";
    case VPE_E_SHAPE: return "ShapeError";
    case VPE_E_LABEL: return "LabelError";
    case VPE_E_USE_AFTER_CONSUME: return "UseAfterConsume";
    case VPE_E_WRITER: return "WriterError";
    case VPE_E_CONFIG: return "ConfigError";
    case VPE_E_PROTOCOL: return "ProtocolError";
    case VPE_E_STARTUP: return "StartupError";
    case VPE_E_CORRUPT_CARD: return "CorruptCard";
    case VPE_E_VALUE: return "ValueError";
    case VPE_E_RUNTIME: return "RuntimeError";
    case VPE_E_CUDA: return "CudaError";
    case VPE_OVERFLOW_REJECTED: return "OverflowRejected";
    case VPE_NO_NEW_DATA: return "NoNewData";
    default: return "unknown";
  }
}

int vpe_op_linear(const void* A, int32_t M, int32_t K, const void* W, int32_t N, int32_t Kw, const float* bias,
                  const float* scale, void* out, int32_t kind, int32_t act, int32_t bn, void* stream) {
  EpiParams ep;
  ep.kind = kind;
  ep.act = act;
  ep.N = N;
  ep.bias = bias;
  ep.scale = scale;
  if (kind == EPI_RESID) {
    ep.resid = static_cast<float*>(out);
    ep.ldr = N;
  } else if (kind == EPI_BF16 || kind == EPI_F32) {
    ep.out = out;
    ep.ldo = N;
  } else {
    return VPE_E_CONFIG;
  }
  GemmPlan g;
  VPE_TRY(plan_gemm_rows(&g, static_cast<const __nv_bfloat16*>(A), M, K, K, static_cast<const __nv_bfloat16*>(W), N,
                         Kw, Kw, ep, bn));
  VPE_TRY(launch_gemm(g, static_cast<cudaStream_t>(stream)));
  count_launches(1);
  return VPE_OK;
}

int vpe_op_linear_resid_ln(const void* A, int32_t M, int32_t K, const void* W, const float* bias, const float* ls,
                           float* resid, const float* ln_w, const float* ln_b, float eps, void* xln, const float* tap_w,
                           const float* tap_b, void* tap_out, void* stream) {
  GemmPlan g;
  VPE_TRY(plan_gemm_resid_ln(&g, static_cast<const __nv_bfloat16*>(A), M, K, static_cast<const __nv_bfloat16*>(W), bias,
                             ls, resid, ln_w, ln_b, eps, static_cast<__nv_bfloat16*>(xln), tap_w, tap_b));
  VPE_TRY(launch_gemm_resid_ln(g, static_cast<__nv_bfloat16*>(xln), static_cast<__nv_bfloat16*>(tap_out),
                               static_cast<cudaStream_t>(stream)));
  count_launches(1);
  return VPE_OK;
}

int vpe_op_conv(const void* x, int32_t B, int32_t H, int32_t W, int32_t C, int32_t Cp, int32_t ks, const void* w,
                int32_t N, const float* bias, const void* add1, const void* add2, void* out, void* out_relu,
                int32_t ldo, int32_t act, void* stream) {
  EpiParams ep;
  ep.kind = EPI_CONV;
  ep.act = act;
  ep.N = N;
  ep.bias = bias;
  ep.out = out;
  ep.ldo = ldo;
  ep.add1 = static_cast<const __nv_bfloat16*>(add1);
  ep.add2 = static_cast<const __nv_bfloat16*>(add2);
  ep.out_relu = static_cast<__nv_bfloat16*>(out_relu);
  const int bk = (Cp % 64 == 0) ? 64 : 32;
  const int kb = ks * ks * Cp;
  const int bn = N <= 32 ? 32 : (N <= 64 ? 64 : 128);
  GemmPlan g;
  const bool halo = ks == 3 && plan_conv_halo(&g, static_cast<const __nv_bfloat16*>(x), B, H, W, Cp, Cp,
                                              (int64_t)W * Cp, (int64_t)H * W * Cp, 1,
                                              static_cast<const __nv_bfloat16*>(w), N, kb, ep, bn) == VPE_OK;
  if (!halo)
    VPE_TRY(plan_gemm_conv(&g, static_cast<const __nv_bfloat16*>(x), B, H, W, C, Cp, (int64_t)W * Cp,
                           (int64_t)H * W * Cp, ks, bk, static_cast<const __nv_bfloat16*>(w), N, kb, kb, ep, bn));
  VPE_TRY(launch_gemm(g, static_cast<cudaStream_t>(stream)));
  count_launches(1);
  return VPE_OK;
}

int vpe_op_conv_up_pack(const void* w, int32_t Cp, void* wpack, void* stream) {
  if (!w || !wpack || (Cp != 32 && Cp != 64)) return VPE_E_VALUE;
  VPE_TRY(pack_conv_up_weights(static_cast<const __nv_bfloat16*>(w), Cp, static_cast<__nv_bfloat16*>(wpack),
                               static_cast<cudaStream_t>(stream)));
  return VPE_OK;
}

int vpe_op_conv_up(const void* x, int32_t B, int32_t Hs, int32_t Ws, int32_t Cp, int32_t Ho, int32_t Wo,
                   const void* wpack, int32_t N, const float* bias, void* out, int32_t ldo, int32_t act,
                   const float* w3, float b3, float* depth, void* stream) {
  if (!x || !wpack || B < 1 || (w3 ? (!depth || N != 32) : !out)) return VPE_E_VALUE;
  EpiParams ep;
  ep.kind = w3 ? EPI_DEPTH : EPI_CONV;
  ep.act = act;
  ep.N = N;
  ep.bias = bias;
  ep.out = out;
  ep.ldo = ldo;
  ep.w3 = w3;
  ep.b3 = b3;
  ep.max_depth = 1.f;
  ep.depth = depth;
  ep.depth_pre = depth;
  GemmPlan g;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  VPE_TRY(plan_conv_up(&g, static_cast<const __nv_bfloat16*>(x), B, Hs, Ws, Cp, Ho, Wo, nullptr, N, ep,
                       static_cast<__nv_bfloat16*>(const_cast<void*>(wpack)), s));
  VPE_TRY(launch_gemm(g, s));
  count_launches(1);
  return VPE_OK;
}

int vpe_set_pdl(int32_t on) {
  if (on < 0 || on > 2) return VPE_E_VALUE;
  pdl_flag() = on;
  return VPE_OK;
}

int vpe_op_attention(const void* qkv, void* out, int32_t B, int32_t T, int32_t D, int32_t heads, void* stream) {
  AttnPlan a;
  VPE_TRY(plan_attention(&a, static_cast<const __nv_bfloat16*>(qkv), static_cast<__nv_bfloat16*>(out), B, T, D,
                         heads));
  static const int op_pdl = getenv("VPE_OP_PDL") ? atoi(getenv("VPE_OP_PDL")) : 0;  // diagnostics
  const int saved = pdl_scope();
  if (op_pdl) pdl_scope() = 1;
  const int rc = launch_attention(a, static_cast<cudaStream_t>(stream));
  pdl_scope() = saved;
  VPE_TRY(rc);
  count_launches(1);
  return VPE_OK;
}

int vpe_op_bilinear(const void* in, int32_t B, int32_t Hi, int32_t Wi, int32_t cp, int32_t C, void* out, int32_t Ho,
                    int32_t Wo, void* stream) {
  if (!in || !out) return VPE_E_VALUE;
  VPE_TRY(launch_bilinear_ac(static_cast<const __nv_bfloat16*>(in), B, Hi, Wi, cp, static_cast<__nv_bfloat16*>(out),
                             Ho, Wo, C, static_cast<cudaStream_t>(stream)));
  count_launches(1);
  return VPE_OK;
}

int vpe_op_layernorm(const float* x, int32_t M, int32_t D, const float* w, const float* b, float eps, void* out,
                     const float* w2, const float* b2, void* out2, void* stream) {
  VPE_TRY(launch_layernorm(x, M, D, w, b, eps, static_cast<__nv_bfloat16*>(out), w2, b2,
                           static_cast<__nv_bfloat16*>(out2), static_cast<cudaStream_t>(stream)));
  count_launches(1);
  return VPE_OK;
}

int vpe_stream_create(int32_t priority, void** stream) {
  cudaStream_t s;
  VPE_CUDA_TRY(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, priority));
  *stream = s;
  return VPE_OK;
}
int vpe_stream_destroy(void* stream) {
  VPE_CUDA_TRY(cudaStreamDestroy(static_cast<cudaStream_t>(stream)));
  return VPE_OK;
}
int vpe_stream_sync(void* stream) {
  VPE_CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  return VPE_OK;
}
int vpe_graph_begin(void* stream) {
  VPE_CUDA_TRY(cudaStreamBeginCapture(static_cast<cudaStream_t>(stream), cudaStreamCaptureModeThreadLocal));
  t_capturing = true;
  t_captured = 0;
  return VPE_OK;
}
int vpe_graph_end(void* stream, vpe_graph** out) {
  t_capturing = false;
  vpe_graph* g = new (std::nothrow) vpe_graph();
  if (!g) return VPE_E_RESOURCE;
  g->kernels = t_captured;
  if (cudaStreamEndCapture(static_cast<cudaStream_t>(stream), &g->graph) != cudaSuccess ||
      cudaGraphInstantiate(&g->exec, g->graph, 0) != cudaSuccess) {
    fprintf(stderr, "[vpe] graph capture failed: %s\n", cudaGetErrorString(cudaGetLastError()));
    delete g;
    return VPE_E_CUDA;
  }
  *out = g;
  return VPE_OK;
}
int vpe_graph_launch(vpe_graph* g, void* stream) {
  if (!g) return VPE_E_VALUE;
  VPE_CUDA_TRY(cudaGraphLaunch(g->exec, static_cast<cudaStream_t>(stream)));
  g_launches.fetch_add(g->kernels, std::memory_order_relaxed);
  return VPE_OK;
}
int vpe_graph_destroy(vpe_graph* g) {
  if (!g) return VPE_OK;
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->graph) cudaGraphDestroy(g->graph);
  delete g;
  return VPE_OK;
}
int vpe_event_create(void** ev) {
  cudaEvent_t e;
  VPE_CUDA_TRY(cudaEventCreate(&e));
  *ev = e;
  return VPE_OK;
}
int vpe_event_record(void* ev, void* stream) {
  VPE_CUDA_TRY(cudaEventRecord(static_cast<cudaEvent_t>(ev), static_cast<cudaStream_t>(stream)));
  return VPE_OK;
}
int vpe_event_sync(void* ev) {
  VPE_CUDA_TRY(cudaEventSynchronize(static_cast<cudaEvent_t>(ev)));
  return VPE_OK;
}
int vpe_event_elapsed_ms(void* a, void* b, float* ms) {
  VPE_CUDA_TRY(cudaEventElapsedTime(ms, static_cast<cudaEvent_t>(a), static_cast<cudaEvent_t>(b)));
  return VPE_OK;
}
int vpe_event_destroy(void* ev) {
  VPE_CUDA_TRY(cudaEventDestroy(static_cast<cudaEvent_t>(ev)));
  return VPE_OK;
}
int vpe_stream_wait_event(void* stream, void* ev) {
  VPE_CUDA_TRY(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), static_cast<cudaEvent_t>(ev), 0));
  return VPE_OK;
}
int vpe_memcpy_async(void* dst, const void* src, size_t bytes, void* stream) {
  VPE_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, static_cast<cudaStream_t>(stream)));
  return VPE_OK;
}

}  // extern "C"
