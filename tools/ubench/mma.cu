// Microbenchmark (diagnostics only): tcgen05.mma issue/throughput for the attention shapes.
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
__host__ __device__ constexpr uint32_t idesc(int M, int N, bool bmn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((bmn ? 1u : 0u) << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a), "l"(b), "r"(id), "r"(acc));
}

template <int MODE>
__global__ void k(unsigned long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((uint32_t*)s)[i] = 0x3c003c00u;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t a0 = smem_u32(s), b0 = smem_u32(s + 32768);
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (MODE == 0) {  // S: M128 N128 K64 (4 x K16), SS, B K-major
#pragma unroll
        for (int k = 0; k < 4; ++k) mma_ss(tmem, desc(a0 + k * 32, 16, 1024, 2), desc(b0 + k * 32, 16, 1024, 2), idesc(128, 128, false), k > 0);
      } else if (MODE == 1) {  // PV: M128 N64 K128, TS (A in TMEM), B MN-major
#pragma unroll
        for (int k = 0; k < 8; ++k) mma_ts(tmem + 256, tmem + 128 + k * 8, desc(b0 + k * 2048, 1024, 1024, 2), idesc(128, 64, true), k > 0);
      } else if (MODE == 2) {  // PV: SS, B MN-major
#pragma unroll
        for (int k = 0; k < 8; ++k) mma_ss(tmem + 256, desc(a0 + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024, 2), desc(b0 + k * 2048, 1024, 1024, 2), idesc(128, 64, true), k > 0);
      } else if (MODE == 3) {  // PV-shaped SS with K-major B (V^T)
#pragma unroll
        for (int k = 0; k < 8; ++k) mma_ss(tmem + 256, desc(a0 + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024, 2), desc(b0 + (k >> 2) * 8192 + (k & 3) * 32, 16, 1024, 2), idesc(128, 64, false), k > 0);
      } else if (MODE == 4) {  // TS with K-major B
#pragma unroll
        for (int k = 0; k < 8; ++k) mma_ts(tmem + 256, tmem + 128 + k * 8, desc(b0 + (k >> 2) * 8192 + (k & 3) * 32, 16, 1024, 2), idesc(128, 64, false), k > 0);
      } else if (MODE == 5) {  // GEMM-like: M128 N256 K64 SS
#pragma unroll
        for (int k = 0; k < 4; ++k) mma_ss(tmem, desc(a0 + k * 32, 16, 1024, 2), desc(b0 + k * 32, 16, 1024, 2), idesc(128, 256, false), k > 0);
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
    unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int M>
void run(const char* name, unsigned long long* d, double flop_per_iter) {
  unsigned long long h[148];
  const int iters = 2000;
  cudaFuncSetAttribute(k<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
  k<M><<<148, 128, 66 * 1024>>>(d, iters);
  k<M><<<148, 128, 66 * 1024>>>(d, iters);
  cudaDeviceSynchronize();
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%-34s clk/iter=%.1f  flop/clk/SM=%.0f (%s)\n", name, (double)h[0] / iters, flop_per_iter * iters / h[0],
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  run<0>("S  M128 N128 K64 SS Kmaj", d, 2.0 * 128 * 128 * 64);
  run<1>("PV M128 N64 K128 TS MNmaj", d, 2.0 * 128 * 64 * 128);
  run<2>("PV M128 N64 K128 SS MNmaj", d, 2.0 * 128 * 64 * 128);
  run<3>("PV M128 N64 K128 SS Kmaj", d, 2.0 * 128 * 64 * 128);
  run<4>("PV M128 N64 K128 TS Kmaj", d, 2.0 * 128 * 64 * 128);
  run<5>("GEMM M128 N256 K64 SS", d, 2.0 * 128 * 256 * 64);
  return 0;
}
