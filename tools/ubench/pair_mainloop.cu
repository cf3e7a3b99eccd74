// Microbenchmark (diagnostics only): bare cta_group::2 TMA -> MMA mainloop, M256 x N256 x K64
// k-blocks (each CTA stages 128 A rows + 128 B rows), STAGES ring, no epilogue.
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
__device__ __forceinline__ void tma2_pair(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
               ::"r"(smem_u32(dst)), "l"((uint64_t)m), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1) : "memory");
}

template <int STAGES>
__global__ void __cluster_dims__(2, 1, 1) k(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                                            unsigned long long* out, int iters) {
  constexpr int AB = 128 * 128, BB = 128 * 128, SB = AB + BB;
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], done;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (threadIdx.x == 32) {
    for (int i = 0; i < STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    mbar_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 1 && lane == 0) {
    for (int it = 0; it < iters; ++it) {
      const int st = it % STAGES;
      mbar_wait(&empty[st], ((it / STAGES) & 1) ^ 1);
      if (rank == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[st])), "r"(2 * SB) : "memory");
      const int kb = it % 6, mt = ((blockIdx.x >> 1) + (it / 6) * 74) % 64;
      tma2_pair(s + st * SB, &ta, &full[st], kb * 64, mt * 256 + rank * 128);
      tma2_pair(s + st * SB + AB, &tb, &full[st], kb * 64, ((it / 6) % 6) * 256 + rank * 128);
    }
  } else if (warp == 2 && lane == 0 && rank == 0) {
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int st = it % STAGES;
      mbar_wait(&full[st], (it / STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t a0 = smem_u32(s + st * SB), b0 = a0 + AB;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t ad = desc(a0 + kk * 32, 16, 1024, 2), bd = desc(b0 + kk * 32, 16, 1024, 2);
        const uint32_t id = idesc(256, 256), acc = ((it % 6) | kk) ? 1u : 0u;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tslot), "l"(ad), "l"(bd), "r"(id), "r"(acc));
      }
      asm volatile("{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\ttcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(smem_u32(&empty[st])) : "memory");
    }
    asm volatile("{\n\t.reg .b16 m;\n\tmov.b16 m, 1;\n\ttcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(smem_u32(&done)) : "memory");
    mbar_wait(&done, 0);
    out[blockIdx.x >> 1] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tslot));
}

static PFN_cuTensorMapEncodeTiled_v12000 enc;
static CUtensorMap mk(void* p, uint64_t rows) {
  CUtensorMap tm;
  uint64_t dims[2] = {384, rows};
  uint64_t strides[1] = {768};
  uint32_t box[2] = {64, 128}, es[2] = {1, 1};
  enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return tm;
}

template <int S>
void run(unsigned long long* d, CUtensorMap ta, CUtensorMap tb) {
  constexpr int smem = S * 32768 + 2048;
  cudaFuncSetAttribute(k<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 3000;
  unsigned long long h[74];
  k<S><<<148, 96, smem>>>(ta, tb, d, iters);
  k<S><<<148, 96, smem>>>(ta, tb, d, iters);
  cudaDeviceSynchronize();
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  unsigned long long mx = 0, sum = 0;
  for (int i = 0; i < 74; ++i) { mx = h[i] > mx ? h[i] : mx; sum += h[i]; }
  printf("pair stages=%d  clk/kblock mean=%.1f max=%.1f (ideal 512)  (%s)\n", S, (double)sum / 74 / iters,
         (double)mx / iters, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  void *A, *B;
  cudaMalloc(&A, 16384ull * 768);
  cudaMalloc(&B, 1536ull * 768);
  cudaMemset(A, 0, 16384ull * 768);
  cudaMemset(B, 0, 1536ull * 768);
  unsigned long long* d;
  cudaMalloc(&d, 74 * 8);
  CUtensorMap ta = mk(A, 16384), tb = mk(B, 1536);
  run<3>(d, ta, tb);
  run<4>(d, ta, tb);
  run<6>(d, ta, tb);
  return 0;
}
