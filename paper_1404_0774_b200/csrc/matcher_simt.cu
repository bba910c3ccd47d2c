// matcher_simt.cu — the CUDA-core matcher (exact integer correlations on FP32/FP64
// pipes).  It is the parity anchor for the tensor-core matcher (same pool, same
// epilogue, same partial-result format) and the path for range sides the tcgen05
// matcher does not cover exactly (n >= 16, where a 64-term fp32 sum can exceed 2^24).
//
// One thread owns one range and scans a contiguous chunk of domain tiles in canonical
// order, exactly as Searcher::search_impl does (proj/src/encoder.cpp:205-288).
#include "common.cuh"

namespace ficb {

constexpr int kSimtThreads = 128;
constexpr int kStageBytes = 16384;

// n <= 8: acc in fp32 is exact (64 * 1020 * 255 < 2^24); b lives in registers and the
// 8-isometry group test runs before any exact work.
template <int NN>
__global__ void __launch_bounds__(kSimtThreads)
matcher_simt_small(const unsigned char* __restrict__ img, Geometry g, const unsigned char* __restrict__ pool,
                   const DomainMetaF* __restrict__ meta_f, const DomainMetaI* __restrict__ meta_i,
                   const RangeMeta* __restrict__ rmeta, int tiles_per_chunk, Partial* __restrict__ partials,
                   unsigned long long* __restrict__ gbest, unsigned long long* __restrict__ counters) {
  constexpr int K = NN < 16 ? 16 : NN;
  __shared__ __align__(16) unsigned char stage[kStageBytes];
  constexpr int kDomBytes = K * 16;
  constexpr int kStageDomains = kStageBytes / kDomBytes;
  const int tid = threadIdx.x;
  const int r = blockIdx.x * kSimtThreads + tid;
  RangeState st;
  st.r = r;
  st.active = false;
  st.best = st.thr = __longlong_as_double(0x7ff0000000000000ll);
  st.bd = -1;
  st.bs = 0;
  st.bqs = st.bqo = 0;
  st.sqrtT = -1e30f;
  st.x0 = st.y0 = 0;
  st.sb = 0;
  st.ssb = 0.0;
  if (r < g.R) {
    const RangeMeta m = rmeta[r];
    range_origin(g, r, st.x0, st.y0);
    st.sb = m.sb;
    st.ssb = (double)m.var / (double)g.N;
    st.active = !m.shadow;
  }
  uint32_t bpk[NN / 4];
  load_range_packed<NN>(img, g, st.x0, st.y0, bpk);
  float b[K];
#pragma unroll
  for (int k = 0; k < K; ++k) b[k] = k < NN ? (float)((bpk[k >> 2] >> (8 * (k & 3))) & 0xFFu) : 0.f;
  const float sb_f = (float)st.sb;
  const int t0 = blockIdx.y * tiles_per_chunk;
  const int d_begin = t0 * kDomainsPerTile;
  const int d_end = min(g.D, (t0 + tiles_per_chunk) * kDomainsPerTile);
  for (int d0 = d_begin; d0 < d_end; d0 += kStageDomains) {
    const int nd = min(kStageDomains, d_end - d0);
    __syncthreads();
    {
      const uint4* src = reinterpret_cast<const uint4*>(pool + (long long)d0 * kDomBytes);
      uint4* dst = reinterpret_cast<uint4*>(stage);
      for (int i = tid; i < nd * kDomBytes / 16; i += kSimtThreads) dst[i] = src[i];
    }
    __syncthreads();
    if (!st.active) continue;
    refresh_thr(st, gbest, NN);
    for (int j = 0; j < nd; ++j) {
      const int d = d0 + j;
      const unsigned char* blk = stage + j * kDomBytes;
      float acc[kSyms];
#pragma unroll
      for (int s = 0; s < kSyms; ++s) acc[s] = 0.f;
#pragma unroll
      for (int kc = 0; kc < K / 8; ++kc) {
#pragma unroll
        for (int s = 0; s < kSyms; ++s) {
          const uint4 v = *reinterpret_cast<const uint4*>(blk + kc * 128 + s * 16);
          const __half2* h = reinterpret_cast<const __half2*>(&v);
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const float2 f = __half22float2(h[t]);
            acc[s] = __fmaf_rn(f.x, b[kc * 8 + 2 * t], acc[s]);
            acc[s] = __fmaf_rn(f.y, b[kc * 8 + 2 * t + 1], acc[s]);
          }
        }
      }
      const DomainMetaF mf = meta_f[d];
      uint32_t bits[kSyms];
#pragma unroll
      for (int s = 0; s < kSyms; ++s) bits[s] = __float_as_uint(acc[s]);
      count(counters, 0, g);
      if (!(g.flags & 1) && group_pruned(bits, mf.a, mf.e, sb_f, st.sqrtT)) continue;
      count(counters, 1, g);
      long long acc_ll[kSyms];
#pragma unroll
      for (int s = 0; s < kSyms; ++s) acc_ll[s] = (long long)acc[s];
      evaluate_domain<NN>(st, g, d, acc_ll, meta_i, pool, img, bpk, gbest, counters);
    }
  }
  if (r < g.R) partials[(long long)blockIdx.y * g.R + r] = Partial{st.best, st.bd, st.bs, st.bqs, st.bqo};
}

// Any n: exact integer correlations read straight from the pool and the image
// (fp32 partial sums over <= 64 terms are exact; they are folded into int64).
__device__ __forceinline__ void exact_acc_generic(const Geometry& g, const unsigned char* __restrict__ pool,
                                                  const unsigned char* __restrict__ img, int x0, int y0, int d,
                                                  long long* acc) {
  for (int s = 0; s < kSyms; ++s) {
    long long total = 0;
    for (int k0 = 0; k0 < g.N; k0 += 64) {
      float part = 0.f;
      for (int k = k0; k < min(g.N, k0 + 64); ++k) {
        const float q = __half2float(*reinterpret_cast<const __half*>(pool + pool_offset(d, s, k, g.K)));
        const float bv = (float)img[(long long)(y0 + k / g.n) * g.W + x0 + k % g.n];
        part = __fmaf_rn(q, bv, part);
      }
      total += (long long)part;
    }
    acc[s] = total;
  }
}

__global__ void __launch_bounds__(kSimtThreads)
matcher_simt_generic(const unsigned char* __restrict__ img, Geometry g, const unsigned char* __restrict__ pool,
                     const DomainMetaI* __restrict__ meta_i, const RangeMeta* __restrict__ rmeta,
                     int tiles_per_chunk, Partial* __restrict__ partials, unsigned long long* __restrict__ gbest,
                     unsigned long long* __restrict__ counters) {
  const int r = blockIdx.x * kSimtThreads + threadIdx.x;
  if (r >= g.R) return;
  RangeState st;
  const RangeMeta m = rmeta[r];
  st.r = r;
  range_origin(g, r, st.x0, st.y0);
  st.sb = m.sb;
  st.ssb = (double)m.var / (double)g.N;
  st.active = !m.shadow;
  st.best = st.thr = __longlong_as_double(0x7ff0000000000000ll);
  st.bd = -1;
  st.bs = 0;
  st.bqs = st.bqo = 0;
  st.sqrtT = -1e30f;
  const int t0 = blockIdx.y * tiles_per_chunk;
  const int d_begin = t0 * kDomainsPerTile;
  const int d_end = min(g.D, (t0 + tiles_per_chunk) * kDomainsPerTile);
  if (st.active) {
    for (int d = d_begin; d < d_end; ++d) {
      if (meta_i[d].den < 0) continue;
      if ((d & 31) == 0) refresh_thr(st, gbest, g.N);
      long long acc[kSyms];
      exact_acc_generic(g, pool, img, st.x0, st.y0, d, acc);
      count(counters, 1, g);
      evaluate_domain<0>(st, g, d, acc, meta_i, pool, img, nullptr, gbest, counters);
    }
  }
  partials[(long long)blockIdx.y * g.R + r] = Partial{st.best, st.bd, st.bs, st.bqs, st.bqo};
}

void launch_matcher_simt(const unsigned char* img, const Geometry& g, const unsigned char* pool,
                         const DomainMetaF* meta_f, const DomainMetaI* meta_i, const RangeMeta* rmeta,
                         int n_chunks, int tiles_per_chunk, Partial* partials, unsigned long long* gbest,
                         unsigned long long* counters, cudaStream_t st) {
  dim3 grid((g.R + kSimtThreads - 1) / kSimtThreads, n_chunks);
  if (g.N == 4)
    matcher_simt_small<4><<<grid, kSimtThreads, 0, st>>>(img, g, pool, meta_f, meta_i, rmeta, tiles_per_chunk,
                                                         partials, gbest, counters);
  else if (g.N == 16)
    matcher_simt_small<16><<<grid, kSimtThreads, 0, st>>>(img, g, pool, meta_f, meta_i, rmeta, tiles_per_chunk,
                                                          partials, gbest, counters);
  else if (g.N == 64)
    matcher_simt_small<64><<<grid, kSimtThreads, 0, st>>>(img, g, pool, meta_f, meta_i, rmeta, tiles_per_chunk,
                                                          partials, gbest, counters);
  else
    matcher_simt_generic<<<grid, kSimtThreads, 0, st>>>(img, g, pool, meta_i, rmeta, tiles_per_chunk, partials,
                                                        gbest, counters);
}

// Seeds the shared pruning bar of every range with the best residual among the 8
// isometries of the domains on the grid points around the range's own 2x-scaled
// neighbourhood (the self-similar candidates that usually fit well).  Only the bar is
// seeded — the matcher re-finds and records these candidates itself — so the emitted
// codes do not depend on the seed, only how much the first tiles prune.
template <int NN>
__global__ void seed_kernel(const unsigned char* __restrict__ img, Geometry g, const unsigned char* __restrict__ pool,
                            const DomainMetaI* __restrict__ meta_i, const RangeMeta* __restrict__ rmeta,
                            unsigned long long* __restrict__ gbest) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= g.R) return;
  RangeState st;
  const RangeMeta m = rmeta[r];
  st.r = r;
  range_origin(g, r, st.x0, st.y0);
  st.sb = m.sb;
  st.ssb = (double)m.var / (double)g.N;
  st.active = !m.shadow;
  st.best = st.thr = __longlong_as_double(0x7ff0000000000000ll);
  st.bd = -1;
  st.bs = 0;
  st.bqs = st.bqo = 0;
  st.sqrtT = -1e30f;
  if (st.active && g.D > 0) {
    constexpr int NW = NN > 0 ? NN / 4 : 1;
    uint32_t bpk[NW];
    if constexpr (NN > 0) load_range_packed<NN>(img, g, st.x0, st.y0, bpk);
    const int cx = st.x0 - g.n / 2, cy = st.y0 - g.n / 2;
    const int xi0 = min(max(cx / g.step, 0), g.PX - 1), yi0 = min(max(cy / g.step, 0), g.PY - 1);
    for (int dx = -1; dx <= 1; ++dx) {
      for (int dy = -1; dy <= 1; ++dy) {
        const int xi = xi0 + dx, yi = yi0 + dy;
        if (xi < 0 || yi < 0 || xi >= g.PX || yi >= g.PY) continue;
        const int d = xi * g.PY + yi;
        long long acc[kSyms];
        exact_acc_generic(g, pool, img, st.x0, st.y0, d, acc);
        evaluate_domain<NN>(st, g, d, acc, meta_i, pool, img, bpk, nullptr, nullptr);
      }
    }
  }
  gbest[r] = (unsigned long long)__double_as_longlong(st.best);
}

void launch_seed(const unsigned char* img, const Geometry& g, const unsigned char* pool, const DomainMetaI* meta_i,
                 const RangeMeta* rmeta, unsigned long long* gbest, cudaStream_t st) {
  const int blocks = (g.R + 127) / 128;
  if (g.N == 4)
    seed_kernel<4><<<blocks, 128, 0, st>>>(img, g, pool, meta_i, rmeta, gbest);
  else if (g.N == 16)
    seed_kernel<16><<<blocks, 128, 0, st>>>(img, g, pool, meta_i, rmeta, gbest);
  else if (g.N == 64)
    seed_kernel<64><<<blocks, 128, 0, st>>>(img, g, pool, meta_i, rmeta, gbest);
  else
    seed_kernel<0><<<blocks, 128, 0, st>>>(img, g, pool, meta_i, rmeta, gbest);
}

// Merge the per-scanner partial results of every range (lexicographic (R, domain,
// isometry) — the reference's strict-< scan order) and emit RangeMapping records.
// Shadow ranges and ranges without any non-flat candidate get flat_mapping
// (proj/src/encoder.cpp:176-181, 291-308).
__global__ void finalize_kernel(const unsigned char* __restrict__ img, Geometry g, const RangeMeta* __restrict__ rmeta,
                                const Partial* __restrict__ partials, int n_slots, fic_mapping* __restrict__ out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= g.R) return;
  const RangeMeta m = rmeta[r];
  double br = __longlong_as_double(0x7ff0000000000000ll);
  int bd = -1, bs = 0;
  unsigned bqs = 0, bqo = 0;
  if (!m.shadow) {
    for (int k = 0; k < n_slots; ++k) {
      const Partial p = partials[(long long)k * g.R + r];
      if (p.d >= 0 && better(p.r, p.d, p.sym, br, bd, bs)) {
        br = p.r;
        bd = p.d;
        bs = p.sym;
        bqs = p.qs;
        bqo = p.qo;
      }
    }
  }
  fic_mapping o;
  o.reserved = 0;
  if (bd >= 0) {
    domain_origin(g, bd, o.x, o.y);
    o.sym = bs;
    o.qs = bqs;
    o.qo = bqo;
    o.residual = br;
  } else {
    // flat_mapping (encoder.cpp:298-308)
    int x0, y0;
    range_origin(g, r, x0, y0);
    const double count_d = (double)g.N;
    const double ov = (double)m.sb / count_d;
    const unsigned qo = quantize(ov, 255.0, g.o_bits);
    const double o_deq = dequantize(qo, 255.0, g.o_bits);
    double rv = 0.0;
    for (int i = 0; i < g.N; ++i) {
      const double dd = __dsub_rn(o_deq, (double)img[(long long)(y0 + i / g.n) * g.W + x0 + i % g.n]);
      rv = __dadd_rn(rv, __dmul_rn(dd, dd));
    }
    o.x = 0;
    o.y = 0;
    o.sym = 0;
    o.qs = 0;
    o.qo = qo;
    o.residual = rv;
  }
  out[r] = o;
}

void launch_finalize(const unsigned char* img, const Geometry& g, const RangeMeta* rmeta, const Partial* partials,
                     int n_slots, fic_mapping* out, cudaStream_t st) {
  finalize_kernel<<<(g.R + 127) / 128, 128, 0, st>>>(img, g, rmeta, partials, n_slots, out);
}

}  // namespace ficb
