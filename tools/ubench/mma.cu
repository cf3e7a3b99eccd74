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

#ifndef RANDOM_DATA
#define RANDOM_DATA 0
#endif
template <int MODE>
__global__ void k(unsigned long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t done;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 100 * 1024 / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u;  // pseudo-random bf16 pairs, exponents kept sane
    h ^= h >> 13;
    ((uint32_t*)s)[i] = (RANDOM_DATA ? ((h & 0x807f807fu) | 0x3e003e00u) : 0x3c003c00u);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&done)));
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
      } else if (MODE >= 6 && MODE <= 9) {  // conv-halo-like: K64 as 4 x K16, N = 32 (6,7) / 64 (8,9)
        constexpr int N = MODE <= 7 ? 32 : 64;
        constexpr bool nosw = (MODE == 6 || MODE == 8);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint64_t ad = nosw ? desc(a0 + k * 2 * 8192, 8192, 128, 0) : desc(a0 + k * 32, 16, 1024, 2);
          mma_ss(tmem, ad, desc(b0 + k * 32, 16, 1024, 2), idesc(128, N, false), k > 0);
        }
      } else if (MODE >= 10 && MODE <= 13) {  // misaligned starts: 10 no-swz +16 B, 11 no-swz +32 B,
                                               // 12 SW128 +128 B (base offset 1), 13 SW128 +384 B (3)
        const uint32_t off = MODE == 10 ? 16 : (MODE == 11 ? 32 : (MODE == 12 ? 128 : 384));
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          uint64_t ad = MODE <= 11 ? desc(a0 + off + k * 2 * 8192, 8192, 128, 0) : desc(a0 + off + k * 32, 16, 1024, 2);
          if (MODE >= 12) ad |= (uint64_t)((off >> 7) & 7) << 49;
          mma_ss(tmem, ad, desc(b0 + k * 32, 16, 1024, 2), idesc(128, 32, false), k > 0);
        }
      } else if (MODE == 14 || MODE == 15 || MODE == 16 || MODE == 17) {  // the halo conv's loop: 9 taps x RT=2 x 4 K16, P=130,
                                              // LBO 8320 (14) or 8192 (15), 2 accumulators, B per tap
        const int P = 130;
        const uint32_t lbo = MODE == 15 ? 8192 : 8320;
        for (int j = 0; j < 9; ++j) {
          const int dy = j / 3, dx = j % 3;
#pragma unroll
          for (int rt = 0; rt < 2; ++rt) {
            const uint32_t at = a0 + (uint32_t)(((rt + dy) * P + dx) * 16);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              mma_ss(tmem + rt * 32, desc(at + 2 * k * lbo, lbo, 128, 0), desc(b0 + (j & 3) * 4096 + k * 32, 16, 1024, 2),
                     idesc(128, 32, false), (j | k) != 0);
          }
        }
      } else if (MODE == 5) {  // GEMM-like: M128 N256 K64 SS
#pragma unroll
        for (int k = 0; k < 4; ++k) mma_ss(tmem, desc(a0 + k * 32, 16, 1024, 2), desc(b0 + k * 32, 16, 1024, 2), idesc(128, 256, false), k > 0);
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
    unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&done)) : "memory");
  } else if ((MODE == 16 || MODE == 17) && warp >= 2) {  // 16 "epilogue" warps waiting meanwhile
    if (MODE == 16)
      asm volatile("{\n\t.reg .pred P1;\nW2:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W2;\n\t}" ::"r"(smem_u32(&done)) : "memory");
    else
      asm volatile("{\n\t.reg .pred P1;\nW3:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0, 1000000;\n\t@!P1 bra W3;\n\t}" ::"r"(smem_u32(&done)) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int M>
void run(const char* name, unsigned long long* d, double flop_per_iter) {
  unsigned long long h[148];
  const int iters = M >= 14 ? 200 : 2000;
  cudaFuncSetAttribute(k<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 101 * 1024);
  const int threads = M >= 16 ? 576 : 128;
  k<M><<<148, threads, 101 * 1024>>>(d, iters);
  k<M><<<148, threads, 101 * 1024>>>(d, iters);
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
  run<6>("conv N32 K64 A no-swizzle", d, 2.0 * 128 * 32 * 64);
  run<7>("conv N32 K64 A SW128", d, 2.0 * 128 * 32 * 64);
  run<8>("conv N64 K64 A no-swizzle", d, 2.0 * 128 * 64 * 64);
  run<9>("conv N64 K64 A SW128", d, 2.0 * 128 * 64 * 64);
  run<14>("halo loop N32 LBO8320 (72 MMA)", d, 2.0 * 128 * 32 * 16 * 72);
  run<15>("halo loop N32 LBO8192 (72 MMA)", d, 2.0 * 128 * 32 * 16 * 72);
  run<16>("halo loop + 16 spinning warps", d, 2.0 * 128 * 32 * 16 * 72);
  run<17>("halo loop + 16 sleeping warps", d, 2.0 * 128 * 32 * 16 * 72);
  run<10>("conv N32 no-swz A +16B", d, 2.0 * 128 * 32 * 64);
  run<11>("conv N32 no-swz A +32B", d, 2.0 * 128 * 32 * 64);
  run<12>("conv N32 SW128 A +128B bo1", d, 2.0 * 128 * 32 * 64);
  run<13>("conv N32 SW128 A +384B bo3", d, 2.0 * 128 * 32 * 64);
  return 0;
}
