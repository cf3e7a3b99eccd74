// Microbenchmark (diagnostics only): tcgen05.ld throughput by shape on sm_100a.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

#define R32 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}"
#define O32(r) "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), \
            "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), \
            "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), \
            "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])

template <int SHAPE, int NLD>
__global__ void __launch_bounds__(512, 1) k(unsigned long long* out, int iters, float* sink) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 128;
  float acc = 0.f;
  uint32_t r[32];
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < NLD; ++q) {
      const uint32_t a = tmem + ((it * NLD + q) & 3) * 32;
      if (SHAPE == 0)
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 " R32 ", [%32];" : O32(r) : "r"(a));
      else if (SHAPE == 1)
        asm volatile("tcgen05.ld.sync.aligned.16x256b.x8.b32 " R32 ", [%32];" : O32(r) : "r"(a));
      else if (SHAPE == 2)
        asm volatile("tcgen05.ld.sync.aligned.16x128b.x16.b32 " R32 ", [%32];" : O32(r) : "r"(a));
      else if (SHAPE == 3)
        asm volatile("tcgen05.ld.sync.aligned.16x64b.x32.b32 " R32 ", [%32];" : O32(r) : "r"(a));
      else if (SHAPE == 4)
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.pack::16b.b32 " R32 ", [%32];" : O32(r) : "r"(a));
#pragma unroll
      for (int i = 0; i < 32; i += 8) acc += __uint_as_float(r[i]);
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  }
  unsigned long long t1 = clock64();
  if (acc == 12345.f) *sink = acc;
  if ((threadIdx.x & 31) == 0) out[blockIdx.x * 16 + warp] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tslot));
}

template <int S, int N>
void run(const char* name, unsigned long long* d, float* sink) {
  unsigned long long h[148 * 16];
  const int iters = 1000;
  for (int warps : {4, 8, 16}) {
    k<S, N><<<148, warps * 32>>>(d, iters, sink);
    k<S, N><<<148, warps * 32>>>(d, iters, sink);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    unsigned long long mx = 0;
    for (int w = 0; w < warps; ++w) mx = h[w] > mx ? h[w] : mx;
    const double bytes = (double)warps * iters * N * 32 * 32 * 4;
    printf("%-22s nld=%d warps=%2d  B/clk/SM=%.1f (%s)\n", name, N, warps, bytes / mx,
           cudaGetErrorString(cudaGetLastError()));
  }
}

int main() {
  unsigned long long* d;
  float* sink;
  cudaMalloc(&d, 148 * 16 * 8);
  cudaMalloc(&sink, 4);
  run<0, 1>("32x32b.x32", d, sink);
  run<0, 4>("32x32b.x32", d, sink);
  run<1, 4>("16x256b.x8", d, sink);
  run<2, 4>("16x128b.x16", d, sink);
  run<3, 4>("16x64b.x32", d, sink);
  run<4, 4>("32x32b.x32.pack16", d, sink);
  return 0;
}
