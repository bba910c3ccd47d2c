// pipe_bench.cu — does bulk-copy streaming into shared memory overlap with tcgen05 MMAs that
// read shared memory?  One CTA per SM: a producer thread streams `tile` bytes per step from an
// L2-resident global buffer into a ring of shared-memory stages (cp.async.bulk + mbarrier);
// an MMA thread issues, per step, 4 x tcgen05.mma.cta_group::1.kind::f16 M=128 x N x K=16
// with A = the streamed stage (128 rows x 64 fp16) and B = a resident N x 64 operand.
// Modes: 0 = both, 1 = copies only (MMA thread just recycles stages), 2 = MMAs only (stages
// reused without copies).  Reports cycles per step.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pipe_bench tools/pipe_bench.cu
#include <cstdio>
#include <cstdint>

#include "../paper_1404_0774_b200/csrc/tc_ptx.cuh"

using namespace ficb;

constexpr int K = 64, STAGE_BYTES = 128 * K * 2, STAGES = 8;

template <int N>
__global__ void __launch_bounds__(128, 1) pipe(const unsigned char* src, long long src_tiles, int steps, int mode,
                                                unsigned long long* cycles) {
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* sB = smem;                          // resident N x K
  unsigned char* sA = smem + N * K * 2;              // ring
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], done;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (N * K * 2 + STAGES * STAGE_BYTES) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(&done, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<512>(&tbase);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tb = tbase;
  unsigned long long t0 = clock64();
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < steps; ++i) {
      const int s = i % STAGES;
      ptx::mbar_wait(&empty[s], ((i / STAGES) & 1) ^ 1);
      if (mode == 2) {
        ptx::mbar_arrive(&full[s]);
      } else {
        ptx::mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
        const long long t = ((long long)blockIdx.x * 977 + i) % src_tiles;
        ptx::bulk_g2s(sA + s * STAGE_BYTES, src + t * STAGE_BYTES, STAGE_BYTES, &full[s]);
      }
    }
  } else if (warp == 1 && lane == 0) {
    const uint32_t idesc = ptx::idesc_f16_f32(128, N);
    for (int i = 0; i < steps; ++i) {
      const int s = i % STAGES;
      ptx::mbar_wait(&full[s], (i / STAGES) & 1);
      ptx::tc_fence_after();
      if (mode != 1) {
        const uint32_t a0 = ptx::smem_addr(sA + s * STAGE_BYTES), b0 = ptx::smem_addr(sB);
        for (int kk = 0; kk < K / 16; ++kk)
          ptx::mma_f16_ss(tb + (i & 1) * N, ptx::smem_desc(a0 + kk * 256, 128, K * 16),
                          ptx::smem_desc(b0 + kk * 256, 128, K * 16), idesc, kk > 0 ? 1u : 0u);
      }
      ptx::tc_commit(&empty[s]);
    }
    ptx::tc_commit(&done);
    ptx::mbar_wait(&done, 0);
    cycles[blockIdx.x] = clock64() - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tb);
  }
}

template <int N>
void run(const unsigned char* src, long long tiles, int mode) {
  const int steps = 20000, blocks = 148;
  unsigned long long* cyc;
  cudaMalloc(&cyc, blocks * 8);
  const int smem = N * K * 2 + STAGES * STAGE_BYTES + 1024;
  cudaFuncSetAttribute(pipe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  pipe<N><<<blocks, 128, smem>>>(src, tiles, steps, mode, cyc);
  pipe<N><<<blocks, 128, smem>>>(src, tiles, steps, mode, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < blocks; ++i) avg += h[i];
  avg /= blocks;
  const char* names[] = {"copy+MMA", "copy only", "MMA only"};
  printf("N=%3d %-9s: %7.1f cycles/step (MMA floor %5d, %s)\n", N, names[mode], avg / steps, 4 * 128 * N / 256,
         cudaGetErrorString(e));
  cudaFree(cyc);
}

int main() {
  const long long tiles = 2048;  // 32 MB: L2-resident
  unsigned char* src;
  cudaMalloc(&src, tiles * STAGE_BYTES);
  cudaMemset(src, 0, tiles * STAGE_BYTES);
  for (int mode : {0, 1, 2}) run<256>(src, tiles, mode);
  for (int mode : {0, 1, 2}) run<128>(src, tiles, mode);
  return 0;
}
