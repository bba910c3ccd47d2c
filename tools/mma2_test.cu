// mma2_test.cu — checks the CTA-pair tcgen05 MMA conventions the pair scan relies on:
// kind::f16, cta_group::2, M=256 (A from TMEM: 128 rows per CTA, lane = row, two fp16 K
// elements per 32-bit column), N=224 (B from shared memory, 112 rows per CTA at the same
// offset, K-major no-swizzle core matrices), K=64 as 4 MMAs, D in each CTA's TMEM (its 128
// rows x 224 columns, column j = B row j with rows 0..111 from CTA 0 and 112..223 from CTA 1).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma2_test tools/mma2_test.cu
#include <cuda_fp16.h>

#include <cstdio>
#include <cstdint>
#include <vector>

#include "../paper_1404_0774_b200/csrc/tc2_ptx.cuh"

using namespace ficb;

constexpr int K = 64, N = 224, NH = 112, ACOL = 448;

__device__ __host__ inline int aval(int row, int k) { return ((row * 7 + k * 3) % 9) - 4; }
__device__ __host__ inline int bval(int n, int k) { return ((n * 5 + k * 11) % 7) - 3; }

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) mma2_test(float* out, int* flag) {
  __shared__ __align__(1024) unsigned char sB[NH * K * 2];
  __shared__ __align__(8) uint64_t done_bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  if (threadIdx.x == 0) {
    ptx::mbar_init(&done_bar, 1);
    ptx::fence_mbar_init();
  }
  // B half: rows n = rank*112 + r, core-matrix layout (r/8)*K*16 + (k/8)*128 + (r%8)*16 + (k%8)*2
  for (int c = threadIdx.x; c < NH * K / 8; c += blockDim.x) {
    const int r = c / (K / 8), kc = c % (K / 8);
    uint32_t w[4];
    for (int h = 0; h < 4; ++h) {
      const int k0 = kc * 8 + 2 * h;
      const uint32_t lo = __half_as_ushort(__int2half_rn(bval(rank * NH + r, k0)));
      const uint32_t hi = __half_as_ushort(__int2half_rn(bval(rank * NH + r, k0 + 1)));
      w[h] = lo | (hi << 16);
    }
    *reinterpret_cast<uint4*>(sB + (r >> 3) * K * 16 + kc * 128 + (r & 7) * 16) = make_uint4(w[0], w[1], w[2], w[3]);
  }
  ptx::fence_proxy_async_smem();
  if (warp == 1) ptx::tmem_alloc_2sm<512>(&tbase);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tb = tbase;
  // A rows into TMEM: lane = row (rank*128 + warp*32 + lane), column ACOL + k/2
  {
    const int row = rank * 128 + warp * 32 + lane;
    uint32_t v[32];
    for (int c = 0; c < 32; ++c) {
      const uint32_t lo = __half_as_ushort(__int2half_rn(aval(row, 2 * c)));
      const uint32_t hi = __half_as_ushort(__int2half_rn(aval(row, 2 * c + 1)));
      v[c] = lo | (hi << 16);
    }
    ptx::tmem_st_32x32b_x32(tb + ((uint32_t)(warp * 32) << 16) + ACOL, v);
    ptx::tmem_st_wait();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  if (rank == 0 && threadIdx.x == 0) {
    const uint32_t idesc = ptx::idesc_f16_f32(256, N);
    const uint32_t b_base = ptx::smem_addr(sB);
    for (int kk = 0; kk < K / 16; ++kk) {
      const uint64_t bd = ptx::smem_desc(b_base + kk * 256, 128, K * 16);
      ptx::mma_f16_ts_2sm(tb, tb + ACOL + kk * 8, bd, idesc, kk > 0 ? 1u : 0u);
    }
    ptx::tc_commit_2sm_mc(&done_bar, 0x3);
  }
  ptx::mbar_wait_cluster(&done_bar, 0);
  ptx::tc_fence_after();
  {
    const int row = rank * 128 + warp * 32 + lane;
    for (int c0 = 0; c0 < N; c0 += 16) {
      uint32_t v[16];
      ptx::tmem_ld_32x32b_x16(tb + ((uint32_t)(warp * 32) << 16) + c0, v);
      ptx::tmem_ld_wait();
      for (int j = 0; j < 16; ++j) out[row * N + c0 + j] = __uint_as_float(v[j]);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_2sm<512>(tb);
  }
  if (threadIdx.x == 0 && rank == 0) *flag = 1;
}

int main() {
  float* d_out;
  int* d_flag;
  cudaMalloc(&d_out, 256 * N * 4);
  cudaMalloc(&d_flag, 4);
  cudaMemset(d_out, 0, 256 * N * 4);
  cudaMemset(d_flag, 0, 4);
  mma2_test<<<2, 128>>>(d_out, d_flag);
  cudaError_t e = cudaDeviceSynchronize();
  printf("launch: %s\n", cudaGetErrorString(e));
  std::vector<float> h(256 * N);
  int flag = 0;
  cudaMemcpy(h.data(), d_out, h.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(&flag, d_flag, 4, cudaMemcpyDeviceToHost);
  long bad = 0;
  for (int m = 0; m < 256; ++m)
    for (int n = 0; n < N; ++n) {
      int ref = 0;
      for (int k = 0; k < K; ++k) ref += aval(m, k) * bval(n, k);
      if (h[m * N + n] != (float)ref) {
        if (bad < 8) printf("mismatch m=%d n=%d got %g want %d\n", m, n, h[m * N + n], ref);
        ++bad;
      }
    }
  printf("flag %d, mismatches %ld of %d\n", flag, bad, 256 * N);
  return bad ? 1 : 0;
}
