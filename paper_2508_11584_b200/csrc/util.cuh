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
// Programmatic dependent launch: a process-wide mode set per engine before it captures its
// graphs (vpe_set_pdl: 0 off, 1 early release, 2 late release; VPE_PDL=0/1 overrides on/off).
// Early release (dependents launched as soon as each kernel passed its own griddepcontrol.wait)
// helped batch 1 but cost throughput batches (C2 batch 16: 5285 -> 5194 fps: dependents parked on
// SMs for a whole kernel, SMs the concurrent head kernels could have used). Late release (see
// pdl_late) wins both: batch-1 p50 depth 1.01 -> 0.94 ms, batch 16 5272 -> 5380 fps. Outputs are
// bit-identical over 300 replays (tools/pdl_determinism.py) since the attention kernel's tail-tile
// race was fixed.
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
  return env >= 0 ? env == 1 : pdl_flag() != 0;
}
// Trigger placement: early (each kernel lets its dependents launch right after its own
// griddepcontrol.wait) or late (the persistent GEMM / attention kernels signal after their last
// TMA load, so the dependent grid occupies SMs only for the final tiles' drain). vpe_set_pdl(2)
// selects late, vpe_set_pdl(1) early; VPE_PDL_LATE=0/1 overrides.
inline int pdl_late() {
  static int env = -2;
  if (env == -2) {
    const char* e = getenv("VPE_PDL_LATE");
    env = e ? atoi(e) : -1;
  }
  return env >= 0 ? env : (pdl_flag() == 2 ? 1 : 0);
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
