// Microbenchmark (diagnostics only): softmax emit-chunk throughput variants on sm_100a.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t f2_pack(float a, float b) { uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ void f2_unpack(uint64_t r, float& a, float& b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); }
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) { uint64_t d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) { uint64_t d; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ void st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]) : "memory");
}

__device__ __forceinline__ uint64_t exp2_poly2(uint64_t x) {
  float x0, x1;
  f2_unpack(x, x0, x1);
  x = f2_pack(fmaxf(x0, -127.f), fmaxf(x1, -127.f));
  const float kMagic = 12582912.f;
  const uint64_t j = fadd2(x, f2_pack(kMagic, kMagic));
  const uint64_t nf = fadd2(j, f2_pack(-kMagic, -kMagic));
  const uint64_t f = ffma2(nf, f2_pack(-1.f, -1.f), x);
  uint64_t p = ffma2(f, f2_pack(0.05502927f, 0.05502927f), f2_pack(0.24225698f, 0.24225698f));
  p = ffma2(p, f, f2_pack(0.69325305f, 0.69325305f));
  p = ffma2(p, f, f2_pack(0.99995134f, 0.99995134f));
  const uint32_t jl = (uint32_t)j, jh = (uint32_t)(j >> 32);
  const uint32_t pl = (uint32_t)p, ph = (uint32_t)(p >> 32);
  return ((uint64_t)(ph + (jh << 23)) << 32) | (uint64_t)(pl + (jl << 23));
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) k(unsigned long long* out, int iters, float* sink, float m) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 64;
  float v[32];
  for (int i = 0; i < 32; ++i) v[i] = (threadIdx.x + i) * 1e-3f;
  uint64_t acc = 0;
  const uint64_t sc2 = f2_pack(0.18f, 0.18f);
  float mm = -m;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t pk[16];
    uint64_t a0 = 0, a1 = 0;
    mm -= 1e-7f;
    const uint64_t mb2 = f2_pack(mm, mm);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const uint64_t xx = ffma2(f2_pack(v[2 * i], v[2 * i + 1]), sc2, mb2);
      float x0, x1;
      f2_unpack(xx, x0, x1);
      uint64_t pp;
      if (MODE == 2) pp = xx;
      else if (MODE >= 4 && ((MODE >> 4) >> i) & 1) pp = exp2_poly2(xx);
      else pp = f2_pack(ex2(x0), ex2(x1));
      if (i & 1) a1 = fadd2(a1, pp); else a0 = fadd2(a0, pp);
      pk[i] = (MODE == 3) ? 0u : __byte_perm((uint32_t)pp, (uint32_t)(pp >> 32), 0x7632);
    }
    acc = fadd2(acc, fadd2(a0, a1));
    if (MODE != 1) st16(tmem + (it & 3) * 16, pk);
    else {
      uint32_t s = 0;
      for (int i = 0; i < 16; ++i) s ^= pk[i];
      acc += s;
    }
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  unsigned long long t1 = clock64();
  float a, b;
  f2_unpack(acc, a, b);
  if (a + b == 12345.f) *sink = a;
  if ((threadIdx.x & 31) == 0) out[blockIdx.x * 16 + warp] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tslot));
}

template <int M>
void run(const char* name, unsigned long long* d, float* sink) {
  unsigned long long h[148 * 16];
  const int iters = 2000;
  for (int warps : {4, 8, 16}) {
    k<M><<<148, warps * 32>>>(d, iters, sink, 1.f);
    k<M><<<148, warps * 32>>>(d, iters, sink, 1.f);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    unsigned long long mx = 0;
    for (int w = 0; w < warps; ++w) mx = h[w] > mx ? h[w] : mx;
    printf("%-26s warps=%2d  clk/chunk/warp=%.1f  elems/clk/SM=%.1f (%s)\n", name, warps, (double)mx / iters,
           (double)warps * iters * 32 * 32 / mx, cudaGetErrorString(cudaGetLastError()));
  }
}

int main() {
  unsigned long long* d;
  float* sink;
  cudaMalloc(&d, 148 * 16 * 8);
  cudaMalloc(&sink, 4);
  run<0>("emit (mufu+prmt+sttm)", d, sink);
  run<1>("emit no sttm", d, sink);
  run<2>("emit no mufu", d, sink);
  run<3>("emit no prmt", d, sink);
  run<(0x0707 << 4) | 4>("poly 6/16", d, sink);
  run<(0x1111 << 4) | 4>("poly 4/16", d, sink);
  run<(0x5555 << 4) | 4>("poly 8/16", d, sink);
  run<(0x0101 << 4) | 4>("poly 2/16", d, sink);
  return 0;
}
