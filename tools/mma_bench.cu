// mma_bench.cu — microbenchmark: tcgen05.mma (kind::f16, cta_group::1, M=128, K=16 steps)
// issue throughput on sm_100a with both operands in shared memory (SS), K-major,
// SWIZZLE_NONE vs SWIZZLE_128B, for N = 64 / 128 / 256.  One CTA per SM, one thread issues
// `iters` groups of (subtiles x K/16) MMAs, committing each group to an mbarrier and waiting
// for the group `depth` groups back (like a TMEM ring of `depth` buffers).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_bench tools/mma_bench.cu
#include <cstdio>
#include <cstdint>

#include "../paper_1404_0774_b200/csrc/tc_ptx.cuh"

using namespace ficb;

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;                 // LBO (unused for swizzled K-major), 16 B
  d |= (uint64_t)(1024 >> 4) << 32;       // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                 // version
  d |= (uint64_t)2 << 61;                 // SWIZZLE_128B
  return d;
}

template <int N, bool SW>
__global__ void bench(int iters, int depth, unsigned long long* cycles) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bars[8];
  constexpr int K = 64;
  unsigned char* sA = smem;                    // 256 rows x K fp16 = 32 KB
  unsigned char* sB = smem + 256 * K * 2;      // N rows x K fp16
  for (int i = threadIdx.x; i < (256 + N) * K * 2 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    for (int b = 0; b < 8; ++b) ptx::mbar_init(&bars[b], 1);
    ptx::fence_mbar_init();
  }
  if (threadIdx.x < 32) ptx::tmem_alloc<512>(&tbase);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tb = tbase;
  const int nbuf = 512 / (2 * N) > 0 ? 512 / (2 * N) : 1;
  if (threadIdx.x == 0) {
    const uint32_t idesc = ptx::idesc_f16_f32(128, N);
    const uint32_t a0 = ptx::smem_addr(sA), b0 = ptx::smem_addr(sB);
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int buf = it % nbuf;
      if (it >= depth) ptx::mbar_wait(&bars[(it - depth) % 8], ((it - depth) / 8) & 1);
      for (int m = 0; m < 2; ++m) {
        for (int kk = 0; kk < K / 16; ++kk) {
          uint64_t ad, bd;
          if (SW) {
            ad = desc_sw128(a0 + m * 128 * 128 + kk * 32);
            bd = desc_sw128(b0 + kk * 32);
          } else {
            ad = ptx::smem_desc(a0 + m * 128 * K * 2 + kk * 256, 128, K * 16);
            bd = ptx::smem_desc(b0 + kk * 256, 128, K * 16);
          }
          ptx::mma_f16_ss(tb + ((buf * 2 + m) * N) % 512, ad, bd, idesc, kk > 0 ? 1u : 0u);
        }
      }
      ptx::tc_commit(&bars[it % 8]);
    }
    for (int it = iters - depth > 0 ? iters - depth : 0; it < iters; ++it) ptx::mbar_wait(&bars[it % 8], (it / 8) & 1);
    const unsigned long long t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tb);
  }
}

template <int N, bool SW>
void run(int depth) {
  const int iters = 20000, blocks = 148;
  unsigned long long* cyc;
  cudaMalloc(&cyc, blocks * 8);
  const int smem = (256 + N) * 64 * 2 + 1024;
  cudaFuncSetAttribute(bench<N, SW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  bench<N, SW><<<blocks, 128, smem>>>(iters, depth, cyc);
  bench<N, SW><<<blocks, 128, smem>>>(iters, depth, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < blocks; ++i) avg += h[i];
  avg /= blocks;
  const double per = avg / iters;                  // cycles per group of 2 x 4 MMAs
  const double floor_c = 2 * 4 * 128.0 * N / 256;  // guide's issue floor
  printf("N=%3d %s depth %d: %7.1f cycles per 2x(128x%dx64) tile, floor %6.1f -> %5.1f%% (%s)\n", N,
         SW ? "SW128" : "NOSW ", depth, per, N, floor_c, 100.0 * floor_c / per, cudaGetErrorString(e));
  cudaFree(cyc);
}

int main() {
  for (int d : {2, 4}) {
    run<64, false>(d);
    run<64, true>(d);
    run<128, false>(d);
    run<128, true>(d);
    run<256, false>(d);
    run<256, true>(d);
  }
  return 0;
}
