// tmem_bench.cu — microbenchmark: tcgen05.ld (TMEM -> registers) throughput per SM on
// sm_100a, for 4/8/16 warps per CTA and x8/x32/x64 column loads.  Used to size the
// matcher epilogue (bytes of accumulator it can read per clock).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bench tools/tmem_bench.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int X>
__device__ __forceinline__ void ld(uint32_t taddr, uint32_t* v);

template <>
__device__ __forceinline__ void ld<8>(uint32_t taddr, uint32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}
template <>
__device__ __forceinline__ void ld<32>(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}

// 64 columns of 16-bit values (an fp16 accumulator) packed pairwise into 32 registers.
template <>
__device__ __forceinline__ void ld<-64>(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}

// X > 0: X columns into X registers; X = -64: 64 columns packed into 32 registers.
template <int X, int LOADS_IN_FLIGHT>
__global__ void bench(int iters, unsigned long long* cycles, uint32_t* sink) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = tbase + ((uint32_t)((warp & 3) * 32) << 16);
  uint32_t acc = 0;
  constexpr int R = X > 0 ? X : -X / 2;  // registers per load
  constexpr int C = X > 0 ? X : -X;      // columns per load
  uint32_t v[R * LOADS_IN_FLIGHT];
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int l = 0; l < LOADS_IN_FLIGHT; ++l) ld<X>(base + ((it * LOADS_IN_FLIGHT + l) * C) % 512, v + l * R);
    asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
    for (int k = 0; k < R * LOADS_IN_FLIGHT; ++k) acc ^= v[k];
  }
  const unsigned long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

template <int X, int L>
void run(int warps) {
  const int iters = 4096, blocks = 148;
  unsigned long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, blocks * 8);
  cudaMalloc(&sink, blocks * warps * 32 * 4);
  bench<X, L><<<blocks, warps * 32>>>(iters, cyc, sink);
  bench<X, L><<<blocks, warps * 32>>>(iters, cyc, sink);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < blocks; ++i) avg += h[i];
  avg /= blocks;
  const int C = X > 0 ? X : -X;
  const double cols = (double)iters * L * C * 32 * warps;  // lane-columns per CTA (= per SM)
  printf("x%-3d%s in-flight %d warps %2d: %8.1f cycles/iter  %7.1f lane-columns/clk/SM  (%s)\n", C,
         X > 0 ? "      " : " pack16", L, warps, avg / iters, cols / avg, cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc);
  cudaFree(sink);
}

int main() {
  for (int w : {4, 8, 16}) {
    run<8, 1>(w);
    run<32, 1>(w);
    run<32, 2>(w);
    run<-64, 1>(w);
    run<-64, 2>(w);
  }
  return 0;
}
