#pragma once
#include <cuda_runtime.h>
#include <cstdio>

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
