#pragma once
#include <cuda_runtime.h>
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
// PDL off by default (VPE_PDL=1 enables): measured neutral on the backbone alone (2.184 ->
// 2.175 ms) and slightly negative on the pipelined step with concurrent head streams (3.58 ->
// 3.63 ms), where early-scheduled dependents hold SM slots the head kernels could use.
inline bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("VPE_PDL");
    on = (e && e[0] == '1') ? 1 : 0;
  }
  return on == 1;
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
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
}  // namespace vpe
