// Microbenchmark (diagnostics only): attention exp-pass variants on sm_100a, per warp count.
// Each iteration: LDTM x32 of one S chunk (optional) -> 16 pairs x = s*scale - m -> exp2 (MUFU or
// FMA-pipe cubic) -> bf16 pack -> STTM x4; optional f32x2 row-sum accumulation.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t f2_pack(float a, float b) { uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ void f2_unpack(uint64_t r, float& a, float& b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); }
__device__ __forceinline__ void u2_unpack(uint64_t r, uint32_t& a, uint32_t& b) { asm("mov.b64 {%0, %1}, %2;" : "=r"(a), "=r"(b) : "l"(r)); }
__device__ __forceinline__ uint64_t u2_pack(uint32_t a, uint32_t b) { uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(a), "r"(b)); return r; }
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) { uint64_t d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) { uint64_t d; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ void st4(uint32_t taddr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ void ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]), "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]), "+r"(r[30]), "+r"(r[31]) :: "memory");
}

// 64-bit exponent insert (the kernel's current form)
__device__ __forceinline__ uint64_t poly_a(uint64_t x) {
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
// 32-bit halves through mov.b64 unpack, exponent by one IMAD-shift per lane
__device__ __forceinline__ uint64_t poly_b(uint64_t x) {
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
  uint32_t jl, jh, pl, ph;
  u2_unpack(j, jl, jh);
  u2_unpack(p, pl, ph);
  return u2_pack(pl + (jl << 23), ph + (jh << 23));
}

template <int MODE, int POLY>  // MODE bit0: row sum, bit1: LDTM per chunk, bit2: 32-bit exponent insert
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
    if (MODE & 2) ld32(tmem + 32 * ((it >> 1) & 1), v);
    uint64_t a0 = 0, a1 = 0;
    mm -= 1e-7f;
    const uint64_t mb2 = f2_pack(mm, mm);
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      uint32_t pk[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int i = 4 * g + q;
        const uint64_t xx = ffma2(f2_pack(v[2 * i], v[2 * i + 1]), sc2, mb2);
        uint64_t pp;
        if ((POLY >> i) & 1) pp = (MODE & 4) ? poly_b(xx) : poly_a(xx);
        else {
          float x0, x1;
          f2_unpack(xx, x0, x1);
          pp = f2_pack(ex2(x0), ex2(x1));
        }
        if (MODE & 1) { if (i & 1) a1 = fadd2(a1, pp); else a0 = fadd2(a0, pp); }
        else a0 ^= pp;
        pk[q] = __byte_perm((uint32_t)pp, (uint32_t)(pp >> 32), 0x7632);
      }
      st4(tmem + 128 + (warp >> 2) * 0 + ((it & 1) * 16 + 4 * g), pk[0], pk[1], pk[2], pk[3]);
    }
    acc = fadd2(acc, (MODE & 1) ? fadd2(a0, a1) : a0);
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


__device__ __forceinline__ float fmax3(float a, float b, float c) { float d; asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d; }
__device__ __forceinline__ void ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]) : "r"(taddr));
}
__device__ __forceinline__ void wait16(float (&v)[16]) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]) :: "memory");
}
template <int PM, bool TRACK>
__device__ __forceinline__ uint64_t e16(const float (&v)[16], uint64_t sc2, uint64_t mb2, uint32_t p, float& mx) {
  uint64_t a0 = 0, a1 = 0;
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    uint32_t pk[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = 4 * g + q;
      const uint64_t xx = ffma2(f2_pack(v[2 * i], v[2 * i + 1]), sc2, mb2);
      uint64_t pp;
      if ((PM >> i) & 1) pp = poly_b(xx);
      else { float x0, x1; f2_unpack(xx, x0, x1); pp = f2_pack(ex2(x0), ex2(x1)); }
      if (i & 1) a1 = fadd2(a1, pp); else a0 = fadd2(a0, pp);
      pk[q] = __byte_perm((uint32_t)pp, (uint32_t)(pp >> 32), 0x7632);
    }
    st4(p + 4 * g, pk[0], pk[1], pk[2], pk[3]);
  }
  if (TRACK) {
    mx = fmax3(mx, fmax3(v[0], v[1], v[2]), fmax3(v[3], v[4], v[5]));
    mx = fmax3(mx, fmax3(v[6], v[7], v[8]), fmax3(v[9], v[10], v[11]));
    mx = fmax3(mx, fmax3(v[12], v[13], v[14]), v[15]);
  }
  return fadd2(a0, a1);
}
// the attention kernel's one-pass half tile: 4 x (16 keys), next load in flight
template <bool TRACK>
__global__ void __launch_bounds__(512, 1) k2(unsigned long long* out, int iters, float* sink, float m) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t s_addr = tslot + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 64;
  const uint32_t p_addr = tslot + ((uint32_t)((warp & 3) * 32) << 16) + 256 + (warp >> 2) * 32;
  uint64_t acc = 0;
  const uint64_t sc2 = f2_pack(0.18f, 0.18f);
  float mm = -m, mx = -1e30f;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    mm -= 1e-7f;
    const uint64_t mb2 = f2_pack(mm, mm);
    float va[16], vb[16];
    uint64_t lt;
    ld16(s_addr, va); wait16(va);
    ld16(s_addr + 16, vb);
    lt = e16<0x11, TRACK>(va, sc2, mb2, p_addr, mx);
    wait16(vb); ld16(s_addr + 32, va);
    lt = fadd2(lt, e16<0x11, TRACK>(vb, sc2, mb2, p_addr + 8, mx));
    wait16(va); ld16(s_addr + 48, vb);
    lt = fadd2(lt, e16<0x11, TRACK>(va, sc2, mb2, p_addr + 16, mx));
    wait16(vb);
    lt = fadd2(lt, e16<0x11, TRACK>(vb, sc2, mb2, p_addr + 24, mx));
    acc = fadd2(acc, lt);
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  unsigned long long t1 = clock64();
  float a, b;
  f2_unpack(acc, a, b);
  if (a + b + mx == 12345.f) *sink = a;
  if ((threadIdx.x & 31) == 0) out[blockIdx.x * 16 + warp] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tslot));
}
template <bool TR>
void run2(const char* name, unsigned long long* d, float* sink) {
  unsigned long long h[148 * 16];
  const int iters = 1000;
  printf("%-40s", name);
  for (int warps : {4, 8, 16}) {
    k2<TR><<<148, warps * 32>>>(d, iters, sink, 1.f);
    k2<TR><<<148, warps * 32>>>(d, iters, sink, 1.f);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    unsigned long long mx = 0;
    for (int w = 0; w < warps; ++w) mx = h[w] > mx ? h[w] : mx;
    printf("  w%-2d %5.1f/clk", warps, (double)warps * iters * 32 * 64 / mx);
  }
  printf("  (%s)\n", cudaGetErrorString(cudaGetLastError()));
}


__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c)); }
__device__ __forceinline__ void mb_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory"); }
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t par) {
  asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}" ::"r"(smem_u32(b)), "r"(par) : "memory");
}
// MODE 0: ping-pong, warps 0-7 (slot A) / 8-15 (slot B) alternate half-tile passes (4 x 16 keys)
//         through mbarrier tokens, as in the attention kernel
// MODE 1: all 16 warps on one slot's tile at a time: 2 x 16 keys each, then a 128-thread named
//         barrier per TMEM lane quadrant (the max exchange)
// MODE 2: as 0 with a 64-thread pair barrier after each pass (the kernel's max exchange)
template <int MODE>
__global__ void __launch_bounds__(512, 1) k3(unsigned long long* out, int iters, float* sink, float m) {
  __shared__ uint32_t tslot;
  __shared__ uint64_t tok[2];
  __shared__ float xch[4 * 128];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) { mb_init(&tok[0], 8); mb_init(&tok[1], 8); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int quad = warp & 3;
  const uint32_t lb = tslot + ((uint32_t)(quad * 32) << 16);
  const int x = warp >> 3, hh = (warp >> 2) & 1, qt = warp >> 2;
  uint32_t s_addr, p_addr;
  if (MODE == 1) { s_addr = lb + qt * 32; p_addr = lb + 256 + qt * 16; }
  else { s_addr = lb + x * 128 + hh * 64; p_addr = lb + 256 + x * 64 + hh * 32; }
  uint64_t acc = 0;
  const uint64_t sc2 = f2_pack(0.18f, 0.18f);
  float mm = -m, mx = -1e30f;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    mm -= 1e-7f;
    const uint64_t mb2 = f2_pack(mm, mm);
    float va[16], vb[16];
    uint64_t lt;
    if (MODE == 1) {
      for (int xs = 0; xs < 2; ++xs) {
        ld16(s_addr + xs * 128, va); wait16(va);
        ld16(s_addr + xs * 128 + 16, vb);
        lt = e16<0x11, true>(va, sc2, mb2, p_addr + xs * 64, mx);
        wait16(vb);
        lt = fadd2(lt, e16<0x11, true>(vb, sc2, mb2, p_addr + xs * 64 + 8, mx));
        acc = fadd2(acc, lt);
        xch[qt * 128 + quad * 32 + lane] = mx;
        asm volatile("bar.sync %0, 128;" ::"r"(1 + quad) : "memory");
        mx = fmaxf(fmaxf(xch[quad * 32 + lane], xch[128 + quad * 32 + lane]), fmaxf(xch[256 + quad * 32 + lane], xch[384 + quad * 32 + lane])) - 1e-3f;
      }
    } else {
      if (x == 0 && it > 0) mb_wait(&tok[1], (it - 1) & 1);
      if (x == 1) mb_wait(&tok[0], it & 1);
      ld16(s_addr, va); wait16(va);
      ld16(s_addr + 16, vb);
      lt = e16<0x11, true>(va, sc2, mb2, p_addr, mx);
      wait16(vb); ld16(s_addr + 32, va);
      lt = fadd2(lt, e16<0x11, true>(vb, sc2, mb2, p_addr + 8, mx));
      wait16(va); ld16(s_addr + 48, vb);
      lt = fadd2(lt, e16<0x11, true>(va, sc2, mb2, p_addr + 16, mx));
      wait16(vb);
      lt = fadd2(lt, e16<0x11, true>(vb, sc2, mb2, p_addr + 24, mx));
      __syncwarp();
      if (lane == 0) mb_arrive(&tok[x]);
      acc = fadd2(acc, lt);
      if (MODE == 2) {
        xch[x * 256 + hh * 128 + quad * 32 + lane] = mx;
        asm volatile("bar.sync %0, 64;" ::"r"(1 + x * 4 + quad) : "memory");
        mx = fmaxf(mx, xch[x * 256 + (hh ^ 1) * 128 + quad * 32 + lane]) - 1e-3f;
      }
    }
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  unsigned long long t1 = clock64();
  float a, b;
  f2_unpack(acc, a, b);
  if (a + b + mx == 12345.f) *sink = a;
  if ((threadIdx.x & 31) == 0) out[blockIdx.x * 16 + warp] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tslot));
}
template <int MODE>
void run3(const char* name, unsigned long long* d, float* sink) {
  unsigned long long h[148 * 16];
  const int iters = 1000;
  k3<MODE><<<148, 512>>>(d, iters, sink, 1.f);
  k3<MODE><<<148, 512>>>(d, iters, sink, 1.f);
  cudaDeviceSynchronize();
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int w = 0; w < 16; ++w) mx = h[w] > mx ? h[w] : mx;
  // one iteration = one 128x128 tile for both slots (32768 exponentials)
  printf("%-48s clk per tile pair %7.1f  %5.1f/clk (%s)\n", name, (double)mx / iters, 32768.0 * iters / mx,
         cudaGetErrorString(cudaGetLastError()));
}

template <int M, int P>
void run(const char* name, unsigned long long* d, float* sink) {
  unsigned long long h[148 * 16];
  const int iters = 2000;
  printf("%-40s", name);
  for (int warps : {4, 8, 16}) {
    k<M, P><<<148, warps * 32>>>(d, iters, sink, 1.f);
    k<M, P><<<148, warps * 32>>>(d, iters, sink, 1.f);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    unsigned long long mx = 0;
    for (int w = 0; w < warps; ++w) mx = h[w] > mx ? h[w] : mx;
    printf("  w%-2d %5.1f/clk", warps, (double)warps * iters * 32 * 32 / mx);
  }
  printf("  (%s)\n", cudaGetErrorString(cudaGetLastError()));
}

int main() {
  unsigned long long* d;
  float* sink;
  cudaMalloc(&d, 148 * 16 * 8);
  cudaMalloc(&sink, 4);
  run3<0>("ping-pong 8+8 warps, token per pass", d, sink);
  run3<2>("ping-pong 8+8 + pair max exchange", d, sink);
  run3<1>("16 warps per slot, quad barrier", d, sink);
  run2<true>("kernel one-pass half tile (x16 pipelined, max)", d, sink);
  run2<false>("same without max tracking", d, sink);
  run<3, 0x1111>("cur: ld+sum, poly4 64b", d, sink);
  run<7, 0x1111>("ld+sum, poly4 32b", d, sink);
  run<6, 0x1111>("ld, nosum, poly4 32b", d, sink);
  run<6, 0x0000>("ld, nosum, mufu only", d, sink);
  run<7, 0x0000>("ld+sum, mufu only", d, sink);
  run<6, 0x2525>("ld, nosum, poly6 32b", d, sink);
  run<6, 0x5555>("ld, nosum, poly8 32b", d, sink);
  run<7, 0x2525>("ld+sum, poly6 32b", d, sink);
  run<5, 0x1111>("noload+sum, poly4 32b", d, sink);
  run<4, 0x1111>("noload nosum, poly4 32b", d, sink);
  return 0;
}
