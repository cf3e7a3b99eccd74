// Microbenchmark (diagnostics only): which concurrent warp activity slows tcgen05.mma?
// Warp 16 issues S-shaped MMAs (SS M128 N128 K16 x4 per group) from a converged warp with
// uniform operands; warps 0..7 run one kind of load: FFMA2 chains, MUFU ex2, LDTM, STTM, LDS.
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
__device__ __forceinline__ bool elect1() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mb_try(uint64_t* b, uint32_t par) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.b32 %0, 1, 0, P1;\n\t}" : "=r"(ok) : "r"(smem_u32(b)), "r"(par) : "memory");
  return ok != 0;
}

template <int LOAD, int MMA>  // LOAD: 0 none, 1 FFMA2, 2 MUFU, 3 LDTM, 4 STTM, 5 LDS, 6 IADD; MMA: 0 S, 1 PV
__global__ void __launch_bounds__(544, 1) k(unsigned long long* out, int iters, float* sink, int lw) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t done[2];
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) ((uint32_t*)s)[i] = 0x3c003c00u;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&done[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&done[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    stop = 0;
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (warp == 16) {
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    const uint32_t base = __shfl_sync(0xffffffffu, smem_u32(s), 0);
    int g = 0;
    unsigned long long t0 = clock64();
    while (!__all_sync(0xffffffffu, stop != 0)) {
      if (g >= 2) while (!__all_sync(0xffffffffu, mb_try(&done[g & 1], ((g >> 1) - 1) & 1))) {}
      if (MMA == 0) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint64_t ad = desc(base + k * 32, 16, 1024, 2), bd = desc(base + 32768 + k * 32, 16, 1024, 2);
          if (elect1()) mma_ss(tm + 384, ad, bd, idesc(128, 128, false), k > 0);
          __syncwarp();
        }
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint64_t bd = desc(base + 65536 + k * 2048, 1024, 1024, 2);
          if (elect1()) mma_ts(tm + 448, tm + 256 + k * 8, bd, idesc(128, 64, true), k > 0);
          __syncwarp();
        }
      }
      if (elect1()) commit(&done[g & 1]);
      __syncwarp();
      ++g;
    }
    unsigned long long t1 = clock64();
    if (lane == 0) { out[148 * 16 + blockIdx.x] = g; out[148 * 17 + blockIdx.x] = t1 - t0; }
  } else if (warp < lw) {
    const int quad = warp & 3;
    const uint32_t lb = tmem + ((uint32_t)(quad * 32) << 16) + (warp >> 2) * 32;
    float a[8];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
    uint32_t acc = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        if (LOAD == 1) {
#pragma unroll
          for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], 1.0001f, 0.5f);
        } else if (LOAD == 2) {
#pragma unroll
          for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        } else if (LOAD == 3) {
          uint32_t r0, r1, r2, r3;
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(lb + (u & 7) * 4));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          acc += r0 ^ r1 ^ r2 ^ r3;
        } else if (LOAD == 4) {
          asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(lb + (u & 7) * 4), "r"(acc), "r"(u), "r"(it), "r"(acc) : "memory");
        } else if (LOAD == 5) {
          acc += *(volatile uint32_t*)(s + 96 * 1024 - 4096 + ((threadIdx.x * 4 + u * 128) & 4095));
        } else if (LOAD == 6) {
#pragma unroll
          for (int i = 0; i < 8; ++i) acc = acc * 3 + i;
        } else if (LOAD == 7) {  // FMNMX3
#pragma unroll
          for (int i = 0; i < 8; ++i) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(a[(i + 1) & 7]), "f"(a[(i + 2) & 7]));
        } else if (LOAD == 8) {  // FFMA2
#pragma unroll
          for (int i = 0; i < 8; i += 2) {
            uint64_t v; asm("mov.b64 %0, {%1, %2};" : "=l"(v) : "f"(a[i]), "f"(a[i + 1]));
            asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(v) : "l"(v));
            asm("mov.b64 {%0, %1}, %2;" : "=f"(a[i]), "=f"(a[i + 1]) : "l"(v));
          }
        } else if (LOAD == 9) {  // PRMT
#pragma unroll
          for (int i = 0; i < 8; ++i) acc = __byte_perm(acc, acc + i, 0x7632);
        } else if (LOAD == 10) {  // half of the warps FFMA, FFMA at 1/4 density (3 IMAD per FFMA)
#pragma unroll
          for (int i = 0; i < 8; ++i) { a[i] = fmaf(a[i], 1.0001f, 0.5f); acc = acc * 3 + i; acc ^= acc >> 3; acc += i; }
        }
      }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    float t = 0;
    for (int i = 0; i < 8; ++i) t += a[i];
    if (t + acc == 1.2345f) *sink = t;
    asm volatile("bar.sync 1, %0;" ::"r"(lw * 32) : "memory");
    if (threadIdx.x == 0) stop = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tslot));
}

template <int L, int M>
void run(const char* name, unsigned long long* d, float* sink, int iters) {
  static unsigned long long h[148 * 18];
  cudaFuncSetAttribute(k<L, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  printf("%-10s %s", name, M ? "PV" : "S ");
  for (int lw : {4, 8, 16}) {
    k<L, M><<<148, 544, 100 * 1024>>>(d, iters, sink, lw);
    k<L, M><<<148, 544, 100 * 1024>>>(d, iters, sink, lw);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("   w%-2d %6.0f clk/group", lw, (double)h[148 * 17] / (h[148 * 16] + 1e-9));
  }
  printf("  (ideal %d) %s\n", M ? 364 : 256, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  unsigned long long* d;
  float* sink;
  cudaMalloc(&d, 148 * 18 * 8);
  cudaMalloc(&sink, 4);
  const int it = 4000;
  run<0, 0>("none", d, sink, it); run<0, 1>("none", d, sink, it);
  run<1, 0>("FFMA", d, sink, it); run<1, 1>("FFMA", d, sink, it);
  run<2, 0>("MUFU", d, sink, it / 4); run<2, 1>("MUFU", d, sink, it / 4);
  run<3, 0>("LDTM", d, sink, it / 4); run<3, 1>("LDTM", d, sink, it / 4);
  run<4, 0>("STTM", d, sink, it); run<4, 1>("STTM", d, sink, it);
  run<5, 0>("LDS", d, sink, it); run<5, 1>("LDS", d, sink, it);
  run<6, 0>("IMAD", d, sink, it); run<6, 1>("IMAD", d, sink, it);
  run<7, 0>("FMNMX3", d, sink, it); run<7, 1>("FMNMX3", d, sink, it);
  run<8, 0>("FFMA2", d, sink, it); run<8, 1>("FFMA2", d, sink, it);
  run<9, 0>("PRMT", d, sink, it); run<9, 1>("PRMT", d, sink, it);
  run<10, 0>("FFMA 1/4", d, sink, it / 2); run<10, 1>("FFMA 1/4", d, sink, it / 2);
  return 0;
}
