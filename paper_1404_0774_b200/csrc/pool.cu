// pool.cu — K1, the domain-pool builder, and the per-range pass.
//
// K1 replaces the per-(range, domain) contraction the reference recomputes inside its
// search loop (proj/src/encoder.cpp:205-234): every domain is contracted ONCE per
// image into 2x2 group sums q (integers <= 1020, exact in fp16), its integer moments
// Sq, Sqq, den = N*Sqq - Sq^2 are formed exactly in int64, and the 8 isometries
// (proj/src/transforms.cpp:13-26) are materialised as the 8 rows of a K-major
// UMMA operand block.  One warp per domain; each lane stores 16-byte chunks so a warp
// writes 512 contiguous bytes per step (coalesced, HBM-bound).
#include "common.cuh"

namespace ficb {

// Domains handled per block (one warp each).
constexpr int kPoolWarps = 8;

__global__ void __launch_bounds__(kPoolWarps * 32)
pool_build_kernel(const unsigned char* __restrict__ img, Geometry g, unsigned char* __restrict__ pool,
                  DomainMetaF* __restrict__ meta_f, DomainMetaI* __restrict__ meta_i,
                  unsigned long long* __restrict__ flat_count) {
  extern __shared__ unsigned short q_smem[];  // kPoolWarps * N
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int d = blockIdx.x * kPoolWarps + warp;
  if (d >= g.D_pad) return;
  const int N = g.N, n = g.n, K = g.K;
  unsigned short* q = q_smem + warp * N;
  uint4* out = reinterpret_cast<uint4*>(pool + (long long)d * K * 16);
  const int chunks = K;  // 16-byte chunks per domain block: (K/8 core matrices) x 8 isometries

  if (d >= g.D) {  // padding domain: zero operand, never a candidate
    for (int c = lane; c < chunks; c += 32) out[c] = make_uint4(0, 0, 0, 0);
    if (lane == 0) {
      meta_f[d] = DomainMetaF{0.f, kNeverRadius};
      meta_i[d] = DomainMetaI{0, -1};
    }
    return;
  }
  // canonical order: x outer, y inner (proj/src/codebook.cpp:17-18)
  int x, y;
  domain_origin(g, d, x, y);
  long long s = 0, ss = 0;
  for (int j = lane; j < N; j += 32) {
    const int r = j / n, c = j % n;
    const unsigned char* row0 = img + (long long)(y + 2 * r) * g.W + x + 2 * c;
    const unsigned char* row1 = row0 + g.W;
    const int v = row0[0] + row0[1] + row1[0] + row1[1];  // encoder.cpp:213-215
    q[j] = (unsigned short)v;
    s += v;
    ss += (long long)v * v;
  }
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
  }
  const long long den = (long long)N * ss - s * s;
  const bool flat = (double)den <= 16.0 * g.shadow_eps;  // encoder.cpp:223
  __syncwarp();
  for (int c = lane; c < chunks; c += 32) {
    const int kc = c >> 3, sym = c & 7;  // chunk c = (core matrix kc, isometry row sym)
    unsigned int w[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      unsigned int h2 = 0;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int k = kc * 8 + t * 2 + u;
        unsigned short hv = 0;
        if (k < N && !flat) {
          int sr, sc;
          symmetry_source(sym, k / n, k % n, n, sr, sc);
          hv = __half_as_ushort(__ushort2half_rn(q[sr * n + sc]));  // exact: q <= 1020 < 2048
        }
        h2 |= (unsigned int)hv << (16 * u);
      }
      w[t] = h2;
    }
    out[c] = make_uint4(w[0], w[1], w[2], w[3]);
  }
  if (lane == 0) {
    if (flat) {
      meta_f[d] = DomainMetaF{0.f, kNeverRadius};
      meta_i[d] = DomainMetaI{s, -1};
      atomicAdd(flat_count, 1ull);
    } else {
      meta_f[d] = DomainMetaF{(float)s / (float)N,
                              __double2float_rd(sqrt((double)den) * (1.0 - 1e-12) / (double)N)};
      meta_i[d] = DomainMetaI{s, den};
    }
  }
}

// Per-range sums and the shadow test (proj/src/encoder.cpp:165-181).
__global__ void range_pass_kernel(const unsigned char* __restrict__ img, Geometry g,
                                  RangeMeta* __restrict__ meta, unsigned long long* __restrict__ shadow_count) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= g.R) return;
  int x0, y0;
  range_origin(g, r, x0, y0);
  const int n = g.n;
  long long sb = 0, sbb = 0;
  for (int i = 0; i < n; ++i) {
    const unsigned char* row = img + (long long)(y0 + i) * g.W + x0;
    for (int j = 0; j < n; ++j) {
      const int v = row[j];
      sb += v;
      sbb += v * v;
    }
  }
  const long long var = (long long)g.N * sbb - sb * sb;
  const int shadow = (double)var <= g.shadow_eps;
  meta[r] = RangeMeta{(int)sb, shadow, var};
  if (shadow) atomicAdd(shadow_count + range_slice(g, r), 1ull);  // per slice of a batch
}

void launch_pool_build(const unsigned char* img, const Geometry& g, unsigned char* pool, DomainMetaF* meta_f,
                       DomainMetaI* meta_i, unsigned long long* flat_count, cudaStream_t st) {
  const int blocks = (g.D_pad + kPoolWarps - 1) / kPoolWarps;
  pool_build_kernel<<<blocks, kPoolWarps * 32, kPoolWarps * g.N * sizeof(unsigned short), st>>>(
      img, g, pool, meta_f, meta_i, flat_count);
}

void launch_range_pass(const unsigned char* img, const Geometry& g, RangeMeta* meta,
                       unsigned long long* shadow_count, cudaStream_t st) {
  range_pass_kernel<<<(g.R + 127) / 128, 128, 0, st>>>(img, g, meta, shadow_count);
}

}  // namespace ficb
