// f16acc_probe.cu — how precisely does tcgen05.mma kind::f16 accumulate into an fp16 D?
// (Groundwork for halving the scan's TMEM read volume: the pruning bound needs a proven error
// bound for the accumulator.)  One CTA: A = 128 x 64 fp16 (domain-like values in [-8, 8]),
// B = 256 x 64 fp16 (centred-range-like values in [-128, 128] scaled by 1/T ~ 1/300), four K=16
// MMAs into an fp32 D and into an fp16 D; the fp16 D is read back both as one element per
// 32-bit column and as two packed elements per column, whichever matches the fp32 result.
// Reports max |D16 - exact| / sum|a b| and / |exact| against an fp64 reference.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/f16acc_probe tools/f16acc_probe.cu
#include <cuda_fp16.h>

#include <cmath>
#include <cstdio>
#include <cstdint>
#include <random>
#include <vector>

#include "../paper_1404_0774_b200/csrc/tc_ptx.cuh"

using namespace ficb;

constexpr int M = 128, N = 256, K = 64;

// no-swizzle K-major core-matrix layout of an R x K operand: [row/8][k/8][row%8][8 halves]
__host__ __device__ inline int core_off(int row, int k) { return ((row >> 3) * (K / 8) + (k >> 3)) * 64 + (row & 7) * 8 + (k & 7); }

__device__ __forceinline__ void ld_pack16(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}

__global__ void probe(const __half* A, const __half* B, float* d32, uint32_t* d16raw, uint32_t* d16pack) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  __half* sA = reinterpret_cast<__half*>(smem);
  __half* sB = sA + M * K;
  for (int i = threadIdx.x; i < M * K; i += blockDim.x) sA[i] = A[i];
  for (int i = threadIdx.x; i < N * K; i += blockDim.x) sB[i] = B[i];
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  if (threadIdx.x < 32) ptx::tmem_alloc<512>(&tbase);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tb = tbase;
  if (threadIdx.x == 0) {
    const uint32_t id32 = ptx::idesc_f16_f32(M, N);
    const uint32_t id16 = id32 & ~(3u << 4);  // D format F16
    const uint32_t a0 = ptx::smem_addr(sA), b0 = ptx::smem_addr(sB);
    for (int kk = 0; kk < K / 16; ++kk) {
      const uint64_t ad = ptx::smem_desc(a0 + kk * 256, 128, K * 16);
      const uint64_t bd = ptx::smem_desc(b0 + kk * 256, 128, K * 16);
      ptx::mma_f16_ss(tb, ad, bd, id32, kk > 0 ? 1u : 0u);         // fp32 D: columns 0..255
      ptx::mma_f16_ss(tb + 256, ad, bd, id16, kk > 0 ? 1u : 0u);   // fp16 D: columns 256..
    }
    ptx::tc_commit(&bar);
  }
  ptx::mbar_wait(&bar, 0);
  ptx::tc_fence_after();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = warp * 32 + lane;
  uint32_t v[32];
  for (int c = 0; c < 256; c += 32) {
    ptx::tmem_ld_32x32b_x32(tb + ((uint32_t)(warp * 32) << 16) + c, v);
    ptx::tmem_ld_wait();
    for (int j = 0; j < 32; ++j) d32[row * N + c + j] = __uint_as_float(v[j]);
    ptx::tmem_ld_32x32b_x32(tb + ((uint32_t)(warp * 32) << 16) + 256 + c, v);
    ptx::tmem_ld_wait();
    for (int j = 0; j < 32; ++j) d16raw[row * N + c + j] = v[j];
  }
  // .pack::16b: 32 registers from the fp16 D; register j should hold columns (2j, 2j+1) if the
  // load covers 64 columns
  for (int c = 0; c < 256; c += 64) {
    ld_pack16(tb + ((uint32_t)(warp * 32) << 16) + 256 + c, v);
    ptx::tmem_ld_wait();
    for (int j = 0; j < 32; ++j) d16pack[row * (N / 2) + c / 2 + j] = v[j];
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tb);
  }
}

int main() {
  std::mt19937 rng(1404);
  std::uniform_real_distribution<float> ua(-8.f, 8.f), ub(-128.f / 300.f, 128.f / 300.f);
  std::vector<__half> hA(M * K), hB(N * K);
  std::vector<double> a(M * K), b(N * K);
  for (int r = 0; r < M; ++r)
    for (int k = 0; k < K; ++k) {
      const __half h = __float2half(ua(rng));
      hA[core_off(r, k)] = h;
      a[r * K + k] = __half2float(h);
    }
  for (int r = 0; r < N; ++r)
    for (int k = 0; k < K; ++k) {
      const __half h = __float2half(ub(rng));
      hB[core_off(r, k)] = h;
      b[r * K + k] = __half2float(h);
    }
  __half *dA, *dB;
  float* d32;
  uint32_t *d16, *d16p;
  cudaMalloc(&dA, M * K * 2);
  cudaMalloc(&dB, N * K * 2);
  cudaMalloc(&d32, M * N * 4);
  cudaMalloc(&d16, M * N * 4);
  cudaMalloc(&d16p, M * N * 2);
  cudaMemcpy(dA, hA.data(), M * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), N * K * 2, cudaMemcpyHostToDevice);
  const int smem = (M + N) * K * 2;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<<<1, 128, smem>>>(dA, dB, d32, d16, d16p);
  const cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> h32(M * N);
  std::vector<uint32_t> h16(M * N);
  cudaMemcpy(h32.data(), d32, M * N * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(h16.data(), d16, M * N * 4, cudaMemcpyDeviceToHost);
  std::vector<uint32_t> h16p(M * N / 2);
  cudaMemcpy(h16p.data(), d16p, M * N * 2, cudaMemcpyDeviceToHost);
  int pack_match = 0, pack_match32 = 0;
  for (int m = 0; m < M; ++m)
    for (int j = 0; j < N / 2; ++j) {
      const uint32_t w = h16p[m * (N / 2) + j];
      // hypothesis A: register j of a 64-column load = columns (2j, 2j+1)
      pack_match += (w & 0xFFFF) == (h16[m * N + 2 * j] & 0xFFFF) && (w >> 16) == (h16[m * N + 2 * j + 1] & 0xFFFF);
      // hypothesis B: the load covers 32 columns, register j = column j of that load window
      const int c = (j / 32) * 64 + (j % 32);
      pack_match32 += (w & 0xFFFF) == (h16[m * N + c] & 0xFFFF);
    }
  double e32 = 0, e16lo = 0, e16pk = 0, e16lo_rel = 0, e16pk_rel = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double ex = 0, ab = 0;
      for (int k = 0; k < K; ++k) {
        ex += a[m * K + k] * b[n * K + k];
        ab += std::fabs(a[m * K + k] * b[n * K + k]);
      }
      e32 = std::fmax(e32, std::fabs(h32[m * N + n] - ex) / ab);
      __half_raw lo;
      lo.x = (unsigned short)(h16[m * N + n] & 0xFFFF);
      const double vlo = __half2float(__half(lo));
      __half_raw pk;
      pk.x = (unsigned short)((h16[m * N + n / 2] >> (16 * (n & 1))) & 0xFFFF);
      const double vpk = __half2float(__half(pk));
      e16lo = std::fmax(e16lo, std::fabs(vlo - ex) / ab);
      e16pk = std::fmax(e16pk, std::fabs(vpk - ex) / ab);
      if (std::fabs(ex) > 0.05 * ab) {
        e16lo_rel = std::fmax(e16lo_rel, std::fabs(vlo - ex) / std::fabs(ex));
        e16pk_rel = std::fmax(e16pk_rel, std::fabs(vpk - ex) / std::fabs(ex));
      }
    }
  int hi_nonzero = 0;
  for (int i = 0; i < M * N; ++i) hi_nonzero += (h16[i] >> 16) != 0;
  std::printf("status %s\n", cudaGetErrorString(e));
  std::printf("fp16 D cells with a non-zero upper half: %d of %d\n", hi_nonzero, M * N);
  std::printf("pack::16b load: register j == columns (2j, 2j+1): %d of %d; low half == column j: %d\n",
              pack_match, M * N / 2, pack_match32);
  std::printf("fp32 D: max |D - exact| / sum|ab| = %.3e\n", e32);
  std::printf("fp16 D, one element per column: max err / sum|ab| = %.3e, / |exact| = %.3e\n", e16lo, e16lo_rel);
  std::printf("fp16 D, two packed per column:  max err / sum|ab| = %.3e, / |exact| = %.3e\n", e16pk, e16pk_rel);
  // rounding mode of the fp16 D: row m adds x_m = (m - 64) * 2^-13 to 1.0, either inside the
  // first K=16 step (k = 1) or as the second step (k = 16, the running sum 1.0 read back first);
  // predictions for round-to-nearest-even, toward zero and truncation-away
  for (int k2 : {1, 16}) {
    for (auto& h : hA) h = __float2half(0.f);
    for (auto& h : hB) h = __float2half(0.f);
    for (int m = 0; m < M; ++m) {
      hA[core_off(m, 0)] = __float2half(1.f);
      hA[core_off(m, k2)] = __float2half((float)(m - 64) * 0x1p-13f);
    }
    hB[core_off(0, 0)] = __float2half(1.f);
    hB[core_off(0, k2)] = __float2half(1.f);
    cudaMemcpy(dA, hA.data(), M * K * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB.data(), N * K * 2, cudaMemcpyHostToDevice);
    probe<<<1, 128, smem>>>(dA, dB, d32, d16, d16p);
    cudaDeviceSynchronize();
    cudaMemcpy(h16.data(), d16, M * N * 4, cudaMemcpyDeviceToHost);
    int rn = 0, rz = 0, other = 0;
    for (int m = 0; m < M; ++m) {
      const double ex = 1.0 + (double)(m - 64) * 0x1p-13;
      __half_raw hr;
      hr.x = (unsigned short)(h16[m * N] & 0xFFFF);
      const double got = __half2float(__half(hr));
      const double rne = __half2float(__float2half_rn((float)ex));
      const double rtz = __half2float(__float2half_rz((float)ex));
      rn += got == rne;
      rz += got == rtz;
      other += got != rne && got != rtz;
    }
    std::printf("rounding probe (second term at k=%d): matches RNE %d, RZ %d, neither %d of %d\n", k2, rn, rz, other, M);
  }
  // many terms inside ONE K=16 step: row m sums 1.0 and 15 copies of c_m = (m+1) 2^-16, each
  // below half an fp16 ulp of the running sum for small m.  Exact-then-round (what the pruning
  // bound assumes: one rounding per step, relative to the result, plus a K 2^-21 allowance)
  // gives fl16(1 + 15 c_m); rounding after every product would leave 1.0.
  {
    for (auto& h : hA) h = __float2half(0.f);
    for (auto& h : hB) h = __float2half(0.f);
    for (int m = 0; m < M; ++m) {
      hA[core_off(m, 0)] = __float2half(1.f);
      for (int k = 1; k < 16; ++k) hA[core_off(m, k)] = __float2half((float)(m + 1) * 0x1p-16f);
    }
    for (int k = 0; k < 16; ++k) hB[core_off(0, k)] = __float2half(1.f);
    cudaMemcpy(dA, hA.data(), M * K * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB.data(), N * K * 2, cudaMemcpyHostToDevice);
    probe<<<1, 128, smem>>>(dA, dB, d32, d16, d16p);
    cudaDeviceSynchronize();
    cudaMemcpy(h16.data(), d16, M * N * 4, cudaMemcpyDeviceToHost);
    int exact_round = 0, per_product = 0, within_bound = 0;
    for (int m = 0; m < M; ++m) {
      const double c = (double)(m + 1) * 0x1p-16, ex = 1.0 + 15.0 * c;
      __half_raw hr;
      hr.x = (unsigned short)(h16[m * N] & 0xFFFF);
      const double got = __half2float(__half(hr));
      exact_round += got == (double)__half2float(__float2half_rn((float)ex));
      float seq = 1.f;
      for (int k = 1; k < 16; ++k) seq = __half2float(__float2half_rn(seq + (float)c));
      per_product += got == (double)seq;
      within_bound += std::fabs(got - ex) <= std::ldexp(1.0, -11) * std::fabs(ex) + 16 * std::ldexp(1.0, -21) * ex;
    }
    std::printf("many-term step: exact-then-round %d, per-product rounding %d, within the bound %d of %d\n",
                exact_round, per_product, within_bound, M);
  }
  std::printf("reference: 2^-11 = %.3e, 4 * 2^-11 = %.3e, 64 * 2^-11 = %.3e\n", std::ldexp(1.0, -11),
              4 * std::ldexp(1.0, -11), 64 * std::ldexp(1.0, -11));
  return 0;
}
