// Where does a cta_group::1 M=64 tcgen05.mma put its accumulator rows in TMEM, and may the D
// address carry a lane offset? A[m][0] = m + 1, A[m][1] = 256, B[n][1] = n, B[n][0] = 1, all
// other K zero, so D[m][n] = m + 1 + 256 n. Prints, per TMEM lane, the row m it holds (or -).
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I../../include tmem_m64.cu -o tmem_m64
#include <cuda_bf16.h>
#include <cstdio>

#include "../../paper_2508_11584_b200/csrc/tc.cuh"

using namespace vpe;

__global__ void k(float* out, int lane_off) {
  __shared__ __align__(1024) uint8_t sA[64 * 128];
  __shared__ __align__(1024) uint8_t sB[32 * 128];
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  const int t = threadIdx.x;
  for (int i = t; i < 64 * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sA)[i] = 0;
  for (int i = t; i < 32 * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sB)[i] = 0;
  __syncthreads();
  if (t < 64) {  // row m: chunk 0 -> physical chunk (m & 7) under SWIZZLE_128B
    __nv_bfloat16* a = reinterpret_cast<__nv_bfloat16*>(sA + t * 128 + (t & 7) * 16);
    a[0] = __float2bfloat16((float)(t + 1));
    a[1] = __float2bfloat16(256.f);
  }
  if (t < 32) {
    __nv_bfloat16* b = reinterpret_cast<__nv_bfloat16*>(sB + t * 128 + (t & 7) * 16);
    b[0] = __float2bfloat16(1.f);
    b[1] = __float2bfloat16((float)t);
  }
  fence_async_smem();
  if (t == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (t < 32) tmem_alloc(&tslot, 64);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  // zero the 64 columns of every lane first
  {
    float z[32];
    for (int i = 0; i < 32; ++i) z[i] = -1.f;
    tmem_st32(tmem + ((uint32_t)((t >> 5) * 32) << 16), z);
    tmem_st32(tmem + ((uint32_t)((t >> 5) * 32) << 16) + 32, z);
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (t == 0) {
    const uint64_t ad = smem_desc(smem_u32(sA), 16, 1024, 2), bd = smem_desc(smem_u32(sB), 16, 1024, 2);
    umma_f16(tmem + ((uint32_t)lane_off << 16), ad, bd, idesc_bf16(64, 32), 0u);
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  float v[32];
  tmem_ld32(tmem + ((uint32_t)((t >> 5) * 32) << 16), v);
  tmem_ld_wait();
  for (int c = 0; c < 32; ++c) out[t * 32 + c] = v[c];
  tc_fence_before();
  __syncthreads();
  if (t < 32) tmem_dealloc(tmem, 64);
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * 32 * 4);
  float h[128 * 32];
  for (int off : {0, 16, 32, 64}) {
    cudaMemset(d, 0, 128 * 32 * 4);
    k<<<1, 128>>>(d, off);
    const cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("lane_off %d: %s\n", off, cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("lane_off %2d:", off);
    for (int L = 0; L < 128; ++L) {
      const float x = h[L * 32 + 1];  // column n = 1: m + 1 + 256
      if (x < 0)
        printf(" -");
      else
        printf(" %d", (int)(x - 257));
    }
    printf("\n");
  }
  return 0;
}
