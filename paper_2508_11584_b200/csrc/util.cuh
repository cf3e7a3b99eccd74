#pragma once
#include <cuda_runtime.h>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <utility>

#include "../../include/vpe.h"

#define VPE_CUDA_TRY(expr)                                                                       \
  do {                                                                                           \
    cudaError_t _e = (expr);                                                                     \
    if (_e != cudaSuccess) {                                                                     \
      fprintf(stderr, "[vpe] CUDA error %s at %s:%d: %s\n", cudaGetErrorName(_e), __FILE__, __LINE__, \
              cudaGetErrorString(_e));                                                           \
      return VPE_E_CUDA;                                                                         \
    }                                                                                            \
  } while (0)

#define VPE_TRY(expr)          \
  do {                         \
    int _rc = (expr);          \
    if (_rc != VPE_OK) return _rc; \
  } while (0)

namespace vpe {
// "first call on the current device": kernel attributes (max dynamic smem, carveout) are set per
// device, so a process driving several GPUs must set them once on each of them
struct OncePerDevice {
  std::atomic<uint64_t> done{0};
  bool first() {
    int d = 0;
    cudaGetDevice(&d);
    const uint64_t bit = 1ull << (d & 63);
    return !(done.fetch_or(bit, std::memory_order_acq_rel) & bit);
  }
};
// Programmatic dependent launch: a process-wide switch set per engine before it captures its
// graphs (vpe_set_pdl; VPE_PDL=0/1 overrides). Engines turn it on for small batches (latency
// mode: batch-1 p50 depth 1.01 -> 0.94 ms, seg 0.73 -> 0.66, det 0.83 -> 0.77) and leave it off
// for throughput batches (C2 batch 16: 5285 -> 5194 fps with it, early-scheduled dependents hold
// SM slots the concurrent head kernels could use). Bit-identical over 300 replays
// (tools/pdl_determinism.py) since the attention kernel's tail-tile race was fixed.
inline int& pdl_flag() {
  static int on = 0;
  return on;
}
// Scope: only the backbone's kernel chain after its first kernel is launched with PDL (vit.cu
// sets the scope); head kernels keep full stream serialization. A PDL kernel whose stream
// predecessor is an event wait (the head graphs start by waiting on the ring's ready event) was
// measured to break graph-replay determinism (tests/test_gpu_engine.py), so the first kernel
// after any non-kernel dependency is never launched with PDL.
inline int& pdl_scope() {
  static thread_local int s = 0;
  return s;
}
inline bool pdl_enabled() {
  static int env = -2;
  if (env == -2) {
    const char* e = getenv("VPE_PDL");
    env = e ? (e[0] == '1' ? 1 : 0) : -1;
  }
  if (!pdl_scope()) return false;
  return env >= 0 ? env == 1 : pdl_flag() == 1;
}
// diagnostics: VPE_PDL_MASK limits PDL to kernel kinds (1 GEMM, 2 attention, 4 LayerNorm,
// 8 halo conv, 16 im2col); a guard drops the scope for kinds outside the mask
struct PdlKind {
  int saved;
  explicit PdlKind(int bit) : saved(pdl_scope()) {
    static int mask = -2;
    if (mask == -2) {
      const char* e = getenv("VPE_PDL_MASK");
      mask = e ? atoi(e) : 0xFF;
    }
    if (!(mask & bit)) pdl_scope() = 0;
  }
  ~PdlKind() { pdl_scope() = saved; }
};
// Shared-memory carveout: kernels that need little smem (LayerNorm, im2col) otherwise prefer a
// large L1 split, and every switch between them and the ~200 KB tcgen05 kernels reconfigures
// the SM's L1/smem split at the kernel boundary. VPE_CARVEOUT=0 disables (A/B experiments).
inline bool carveout_on() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("VPE_CARVEOUT");
    on = e ? (e[0] != '0') : 1;
  }
  return on == 1;
}
template <typename K>
inline void max_smem_carveout(K kernel) {
  if (carveout_on()) cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}
// <<<grid, block, smem, stream>>> with programmatic stream serialization (see tc.cuh pdl_wait)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                            Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
  if (e != cudaSuccess)
    fprintf(stderr, "[vpe] launch failed: %s (grid %u, block %u, smem %zu)\n", cudaGetErrorString(e), grid.x, block.x,
            smem);
  return e;
}
}  // namespace vpe
