// Microbenchmark (diagnostics only): does TMA streaming into smem slow concurrent tcgen05.mma?
// One CTA per SM: thread 0 issues MMAs (M128 N256 K16, operands in smem) back to back while
// warp 1 lane 0 streams 2D TMA tiles from a large global buffer into another smem region.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(layout & 0x7) << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n\t.reg .pred P1;\nW%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W%=;\n\t}" ::"r"(smem_u32(b)), "r"(ph) : "memory");
}

__global__ void k(const __grid_constant__ CUtensorMap tm, unsigned long long* out, int iters, int tma_on) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar, tbar[4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    for (int i = 0; i < 4; ++i) mbar_init(&tbar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  volatile __shared__ int done;
  if (threadIdx.x == 0) done = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t a0 = smem_u32(s), b0 = smem_u32(s + 16384);
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t ad = desc(a0 + kk * 32, 16, 1024, 2), bd = desc(b0 + kk * 32, 16, 1024, 2);
        const uint32_t id = idesc(128, 256), acc = (it | kk) ? 1u : 0u;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tslot), "l"(ad), "l"(bd), "r"(id), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    mbar_wait(&bar, 0);
    out[blockIdx.x * 2] = clock64() - t0;
    done = 1;
  } else if (warp == 1 && lane == 0 && tma_on) {
    // stream 32 KB TMA tiles (box 64 x 256 bf16, SW128) into a 4-slot ring at s + 64 KB
    unsigned long long bytes = 0;
    int n = 0;
    const unsigned long long t0 = clock64();
    while (!done) {
      const int slot = n & 3;
      if (n >= 4) mbar_wait(&tbar[slot], ((n >> 2) - 1) & 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&tbar[slot])), "r"(32768) : "memory");
      const int row = ((blockIdx.x * 64 + n) * 256) % (1 << 16);
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                   ::"r"(smem_u32(s + 65536 + slot * 32768)), "l"((uint64_t)&tm), "r"(smem_u32(&tbar[slot])), "r"(0), "r"(row) : "memory");
      bytes += 32768;
      ++n;
    }
    for (int i = 0; i < 4 && i < n; ++i) { const int m = n - 1 - i; mbar_wait(&tbar[m & 3], (m >> 2) & 1); }
    out[blockIdx.x * 2 + 1] = (bytes * 1000ull) / (clock64() - t0);  // milli-bytes per clk
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tslot));
}

int main() {
  void* buf;
  const size_t rows = 1 << 16;  // 64K rows x 128 B = 8 MB (L2 resident)
  cudaMalloc(&buf, rows * 128);
  cudaMemset(buf, 0, rows * 128);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap tm;
  uint64_t dims[2] = {64, rows};
  uint64_t strides[1] = {128};
  uint32_t box[2] = {64, 256}, es[2] = {1, 1};
  enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  unsigned long long* d;
  cudaMalloc(&d, 148 * 16);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  unsigned long long h[296];
  for (int on = 0; on < 2; ++on) {
    for (int rep = 0; rep < 2; ++rep) k<<<148, 128, 200 * 1024>>>(tm, d, 4000, on);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    const double mma_clk = (double)h[0] / 4000;  // per K64 block of M128 N256 (ideal 512)
    printf("tma_on=%d  mma clk/kblock=%.1f (ideal 512)  tma B/clk=%.1f  (%s)\n", on, mma_clk, h[1] / 1000.0,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
