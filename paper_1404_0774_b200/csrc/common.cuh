// common.cuh — device-side pieces shared by the pool builder, both matchers, the
// finalize pass and the decoder.
//
// Exactness contract: every fp64 expression that feeds an emitted code or residual is
// written with explicit round-to-nearest intrinsics (__dmul_rn/__dadd_rn/__dsub_rn,
// IEEE `/`), in the reference's operation order, and the library is compiled with
// --fmad=false, matching the reference's -ffp-contract=off (proj/CMakeLists.txt:29-31).
#pragma once

#include <cuda_fp16.h>
#include <cstdint>

#include "../../include/fic_b200.h"

namespace ficb {

constexpr int kSyms = 8;
constexpr int kRangesPerTile = 128;   // M of one matcher tile (TMEM lanes)
constexpr int kDomainsPerTile = 32;   // 32 domains x 8 isometries = 256 MMA columns

// Normalised parameters plus the derived geometry every kernel needs.
struct Geometry {
  int W, H;       // image width (row stride) and height
  int n, N;       // range side, pixels per range
  int K;          // MMA K: N rounded up to a multiple of 16 (fp16 K atom)
  int step;
  int PX, PY;     // domain positions along x and y
  int D;          // domains (PX*PY), canonical index d = xi*PY + yi
  int D_pad;      // D rounded up to a multiple of kDomainsPerTile
  int RX;         // ranges per range-grid row (W/n)
  int R;          // ranges in the encoded region
  int row_begin;  // first range row encoded (range sharding)
  int single_x0;  // >= 0: encode exactly one range at (single_x0, single_y0) (encode_range)
  int single_y0;
  int flags;      // debug: bit0 = no group bound, bit1 = no per-candidate screens (exhaustive)
  int s_bits, o_bits;
  double s_max;
  double shadow_eps;
  // batched encodes (volumes): `batch` equal slices stacked vertically (H = H1 * batch); ranges
  // are numbered across the stack (R = R1 * batch), domains per slice (D), and slice b's pool
  // entries start at domain b * Dt.  batch == 1 for single images.
  int batch;
  int H1;
  int R1;
  int Dt;
};

// Per-domain metadata written by the pool builder.
struct DomainMetaF {  // bound evaluation (fp32)
  float a;            // Sq / N                (0 for flat / padding domains)
  float e;            // sqrt(den) / N, rounded down (kNeverRadius for flat / padding)
};
// Flat and padding domains have all-zero operand columns (acc == 0) and a huge radius,
// so the group test drops them as soon as any candidate has been found; before that
// (sqrtT < 0) they reach evaluate_domain, which skips them on den < 0.
constexpr float kNeverRadius = 1e30f;
struct DomainMetaI {  // exact values for survivors
  long long sq;       // sum of 2x2 group sums
  long long den;      // N*Sqq - Sq^2 ; < 0 marks a flat or padding domain
};

// Per-range metadata written by the range pass.
struct RangeMeta {
  int sb;             // sum of pixels
  int shadow;         // range_var <= shadow_eps (encoder.cpp:176-181)
  long long var;      // N*Sbb - Sb^2
};

// One matcher's best candidate for a range over the domains it scanned.
struct Partial {
  double r;           // residual (+inf when nothing was found)
  int d;              // canonical domain index, -1 when none
  int sym;
  unsigned qs, qo;
};

// Pixel origin of the r-th encoded range (row-major over the range grid).
__host__ __device__ __forceinline__ void range_origin(const Geometry& g, int r, int& x0, int& y0) {
  if (g.single_x0 >= 0) {
    x0 = g.single_x0;
    y0 = g.single_y0;
  } else {
    x0 = (r % g.RX) * g.n;
    y0 = (g.row_begin + r / g.RX) * g.n;
  }
}

// Slice-local position of canonical domain d: x outer, y inner (proj/src/codebook.cpp:17-18)
// (d is a pool index; in a batch, slice b's domains are b * Dt + local index).
__host__ __device__ __forceinline__ void domain_origin(const Geometry& g, int d, int& x, int& y) {
  const int dl = g.batch > 1 ? d % g.Dt : d;
  x = (dl / g.PY) * g.step;
  y = (dl % g.PY) * g.step;
}

// Pixel origin of pool domain d in the (stacked) image, and its slice.
__host__ __device__ __forceinline__ int domain_origin_px(const Geometry& g, int d, int& x, int& y) {
  const int b = g.batch > 1 ? d / g.Dt : 0;
  domain_origin(g, d, x, y);
  y += b * g.H1;
  return b;
}

// Slice of encoded range r.
__host__ __device__ __forceinline__ int range_slice(const Geometry& g, int r) { return g.batch > 1 ? r / g.R1 : 0; }

// ------------------------------------------------------------------ quantiser
// UniformQuantizer::quantize / dequantize (proj/include/fic/format.hpp:26-40).
__host__ __device__ __forceinline__ unsigned quantize(double v, double maxv, int bits) {
  const unsigned mc = (1u << bits) - 1u;
  if (v == 0.0) return 0u;
  const double m = (double)mc;
#ifdef __CUDA_ARCH__
  const double scaled = __dmul_rn(__ddiv_rn(__dadd_rn(v, maxv), __dmul_rn(2.0, maxv)), m);
  const unsigned code = __double2uint_rz(__dadd_rn(scaled, 0.5));
#else
  const double scaled = (v + maxv) / (2.0 * maxv) * m;
  const unsigned code = (unsigned)(scaled + 0.5);
#endif
  return code < 1u ? 1u : (code > mc ? mc : code);
}

__host__ __device__ __forceinline__ double dequantize(unsigned code, double maxv, int bits) {
  const unsigned mc = (1u << bits) - 1u;
  if (code == 0u) return 0.0;
#ifdef __CUDA_ARCH__
  return __dadd_rn(-maxv, __dmul_rn(__dmul_rn(2.0, maxv), __ddiv_rn((double)code, (double)mc)));
#else
  return -maxv + (2.0 * maxv) * ((double)code / (double)mc);
#endif
}

__host__ __device__ __forceinline__ double clampd(double v, double lo, double hi) {
  return v < lo ? lo : (hi < v ? hi : v);  // std::clamp
}

// symmetry_source (proj/src/transforms.cpp:13-26): output cell (r, c) reads (sr, sc).
__host__ __device__ __forceinline__ void symmetry_source(int s, int r, int c, int side, int& sr, int& sc) {
  const int m = side - 1;
  switch (s) {
    case 0: sr = r; sc = c; break;
    case 1: sr = m - c; sc = r; break;
    case 2: sr = m - r; sc = m - c; break;
    case 3: sr = c; sc = m - r; break;
    case 4: sr = r; sc = m - c; break;
    case 5: sr = m - r; sc = c; break;
    case 6: sr = c; sc = r; break;
    default: sr = m - c; sc = m - r; break;
  }
}

// symmetry_source as an affine map: sr = R_r r + R_c c + R_m m, sc = C_r r + C_c c + C_m m with
// m = side - 1 and coefficients in {-1, 0, 1} packed 2 bits each (value + 1) per isometry:
// bits [0,2) R_r, [2,4) R_c, [4,6) R_m, [6,8) C_r, [8,10) C_c, [10,12) C_m.  No branches: one
// table word per isometry (warp-uniform in the decoder's whole-tile blocks).
__host__ __device__ __forceinline__ unsigned symmetry_affine_word(int s) {
  // (R_r, R_c, R_m; C_r, C_c, C_m) of transforms.cpp:13-26
  constexpr unsigned k[8] = {
      (2u << 0) | (1u << 2) | (1u << 4) | (1u << 6) | (2u << 8) | (1u << 10),  // 0 (r, c)
      (1u << 0) | (0u << 2) | (2u << 4) | (2u << 6) | (1u << 8) | (1u << 10),  // 1 (m - c, r)
      (0u << 0) | (1u << 2) | (2u << 4) | (1u << 6) | (0u << 8) | (2u << 10),  // 2 (m - r, m - c)
      (1u << 0) | (2u << 2) | (1u << 4) | (0u << 6) | (1u << 8) | (2u << 10),  // 3 (c, m - r)
      (2u << 0) | (1u << 2) | (1u << 4) | (1u << 6) | (0u << 8) | (2u << 10),  // 4 (r, m - c)
      (0u << 0) | (1u << 2) | (2u << 4) | (1u << 6) | (2u << 8) | (1u << 10),  // 5 (m - r, c)
      (1u << 0) | (2u << 2) | (1u << 4) | (2u << 6) | (1u << 8) | (1u << 10),  // 6 (c, r)
      (1u << 0) | (0u << 2) | (2u << 4) | (0u << 6) | (1u << 8) | (2u << 10),  // 7 (m - c, m - r)
  };
  return k[s & 7];
}
__host__ __device__ __forceinline__ int affine_coef(unsigned w, int field) { return (int)((w >> (2 * field)) & 3u) - 1; }

// Byte offset of element (sym s, k) of domain d inside the fp16 operand pool.  Each
// domain is one K-major, no-swizzle UMMA block of 8 rows (its isometries) by K
// columns: [K/8 core matrices][8 rows][8 fp16] = K*16 bytes, so a tile of
// kDomainsPerTile domains is a contiguous canonical B operand.
__host__ __device__ __forceinline__ long long pool_offset(long long d, int s, int k, int K) {
  return d * (long long)K * 16 + (long long)(k >> 3) * 128 + s * 16 + (k & 7) * 2;
}

#ifdef __CUDACC__

// ------------------------------------------------------------------ bound
// Pruning radius factor for a range whose current best residual is `best`:
// a candidate is dropped iff its unconstrained least-squares residual
// R* = ssb - num^2/(N*den) is >= best + delta (R of any quantised candidate is
// >= R*), i.e. iff |acc - Sq*Sb/N| <= sqrt(den)/N * sqrtT with
// sqrtT = sqrt(N*(ssb - best - delta)).  The float is rounded down and shrunk, and the
// caller subtracts an absolute slack, so fp32 evaluation only ever prunes less.
__device__ __forceinline__ float prune_sqrtT(double ssb, double best, int N) {
  const double delta = 1e-6 * (1.0 + best);
  const double t = (ssb - best) - delta;
  if (!(t > 0.0)) return -1e30f;  // also catches best == +inf
  return __double2float_rd(sqrt((double)N * t) * (1.0 - 1e-6));
}

// Absolute slack (in accumulator units) absorbing the fp32 rounding of the center
// Sq*Sb/N and of the interval ends.
constexpr float kBoundSlack = 4.0f;

// Range-side state held by one epilogue thread.
struct RangeState {
  int x0, y0;         // range origin in pixels
  int r;              // encoded-range index (row into the global best array)
  int sb;             // sum of pixels
  double ssb;         // range_var / N
  double best;        // best residual so far (own candidates)
  double thr;         // min(best, best any scanner has published) used for pruning
  float sqrtT;
  int bd, bs;         // best domain / isometry (-1 = none)
  unsigned bqs, bqo;
  bool active;        // non-shadow range inside the image
};

// Shared pruning bar: every scanner publishes the residuals it achieves per range
// (atomicMin on the IEEE bits: non-negative doubles order like unsigned integers), so
// all CTAs and epilogue groups working on a range prune against the best value any of
// them has reached.  Any achieved residual is a valid bar: a candidate whose lower
// bound exceeds it cannot be the (R, domain, isometry)-lexicographic minimum.
__device__ __forceinline__ void publish_best(unsigned long long* gbest, int r, double v) {
  if (gbest) atomicMin(gbest + r, (unsigned long long)__double_as_longlong(v));
}

__device__ __forceinline__ void refresh_thr(RangeState& st, const unsigned long long* gbest, int N) {
  if (!gbest || !st.active) return;
  const double gb = __longlong_as_double((long long)__ldcg(gbest + st.r));
  if (gb < st.thr) {
    st.thr = gb;
    st.sqrtT = prune_sqrtT(st.ssb, st.thr, N);
  }
}

// Diagnostic counters (Geometry::flags bit 2): [0] domain groups tested, [1] groups
// surviving the 8-isometry bound, [2] isometries passing the tight bound, [3] exact
// residual evaluations.
__device__ __forceinline__ void count(unsigned long long* c, int i, const Geometry& g) {
  if ((g.flags & 4) && c) atomicAdd(c + i, 1ull);
}

// Range pixels of (x0, y0) packed 4 per word (NN pixels, NN % 4 == 0).
template <int NN>
__device__ __forceinline__ void load_range_packed(const unsigned char* __restrict__ img, const Geometry& g, int x0,
                                                  int y0, uint32_t* bpk) {
#pragma unroll
  for (int w = 0; w < NN / 4; ++w) {
    uint32_t v = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = w * 4 + b;
      v |= (uint32_t)img[(long long)(y0 + i / g.n) * g.W + x0 + i % g.n] << (8 * b);
    }
    bpk[w] = v;
  }
}

// Same packing with 32/16-bit loads: 4 consecutive pixels of a range row per word
// (n >= 4: range rows are 4-byte aligned since x0 is a multiple of n), or two 2-pixel
// rows per word (n == 2).
template <int NN>
__device__ __forceinline__ void load_range_words(const unsigned char* __restrict__ img, const Geometry& g, int x0,
                                                 int y0, uint32_t* bpk) {
  constexpr int n = NN == 4 ? 2 : (NN == 16 ? 4 : 8);
#pragma unroll
  for (int w = 0; w < NN / 4; ++w) {
    if constexpr (n >= 4) {
      const int i = 4 * w;
      bpk[w] = *reinterpret_cast<const uint32_t*>(img + (long long)(y0 + i / n) * g.W + x0 + i % n);
    } else {
      const uint32_t lo = *reinterpret_cast<const unsigned short*>(img + (long long)(y0 + 2 * w) * g.W + x0);
      const uint32_t hi = *reinterpret_cast<const unsigned short*>(img + (long long)(y0 + 2 * w + 1) * g.W + x0);
      bpk[w] = lo | (hi << 16);
    }
  }
}

// Reference-exact evaluation of one candidate (domain d, isometry s) for a range with
// pixel sum sb and ssb = range_var/N, following Searcher::search_impl
// (proj/src/encoder.cpp:236-280) operation by operation.  Returns its residual, or +inf
// when a bound shows it cannot beat `thr` (an achieved residual; the screens are the
// reference's own, with its +1e-3 margins, plus the unconstrained-LS bound).
// NN > 0: N == NN and the range pixels come packed in `bpk` (pixel i in byte i%4 of
// word i/4) so the residual loop is unrolled over 16-byte pool loads; NN == 0: any N,
// pixels read from the image at (x0, y0).
template <int NN>
__device__ __forceinline__ double eval_candidate(const Geometry& g, int d, int s, long long acc, const DomainMetaI& mi,
                                                 int sb, double ssb, double thr, const uint32_t* bpk,
                                                 const unsigned char* __restrict__ pool,
                                                 const unsigned char* __restrict__ img, int x0, int y0, unsigned& qs_out,
                                                 unsigned& qo_out, unsigned long long* counters) {
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  const int N = NN > 0 ? NN : g.N;
  const double count_d = (double)N;
  const double inv_count = 1.0 / count_d;
  const double den_d = (double)mi.den;
  const double sa_d = __dmul_rn((double)mi.sq, 0.25);
  const double sb_d = (double)sb;
  const double smax = g.s_max;
  const long long num_q = (long long)N * acc - mi.sq * (long long)sb;
  const double num_d = (double)num_q;
  if (!(g.flags & 2)) {  // tight unconstrained-LS bound
    const double rstar = ssb - (num_d * num_d) / (count_d * den_d);
    if (rstar >= thr + 1e-6 * (1.0 + thr)) return inf;
  }
  count(counters, 2, g);
  const double s_raw = __ddiv_rn(__dmul_rn(4.0, num_d), den_d);
  const double sc = clampd(s_raw, -smax, smax);
  const unsigned qs = quantize(sc, smax, g.s_bits);
  const double s_deq = dequantize(qs, smax, g.s_bits);
  const double cov = __dmul_rn(__dmul_rn(num_d, 0.25), inv_count);
  const double var_a = __dmul_rn(__dmul_rn(den_d, 0.0625), inv_count);
  const double parabola =
      __dadd_rn(__dsub_rn(ssb, __dmul_rn(__dmul_rn(2.0, s_deq), cov)), __dmul_rn(__dmul_rn(s_deq, s_deq), var_a));
  if (!(g.flags & 2) && parabola >= thr + 1e-3) return inf;  // encoder.cpp:263
  const double o = clampd(__dmul_rn(__dsub_rn(sb_d, __dmul_rn(sc, sa_d)), inv_count), -255.0, 255.0);
  const unsigned qo = quantize(o, 255.0, g.o_bits);
  const double o_deq = dequantize(qo, 255.0, g.o_bits);
  const double o_gap = __dsub_rn(o_deq, __dmul_rn(__dsub_rn(sb_d, __dmul_rn(s_deq, sa_d)), inv_count));
  const double screen = __dadd_rn(parabola, __dmul_rn(__dmul_rn(count_d, o_gap), o_gap));
  if (!(g.flags & 2) && screen >= thr + 1e-3) return inf;  // encoder.cpp:272
  count(counters, 3, g);
  // Exact residual in range-pixel order (encoder.cpp:274-280).
  double r_val = 0.0;
  if constexpr (NN > 0) {
    uint32_t lb[NN / 4];
    if (bpk == nullptr) {  // range pixels fetched only when a candidate reaches the exact loop
      load_range_words<NN>(img, g, x0, y0, lb);
      bpk = lb;
    }
    const unsigned char* col = pool + (long long)d * (NN < 16 ? 16 : NN) * 16 + s * 16;
#pragma unroll
    for (int kc = 0; kc < (NN + 7) / 8; ++kc) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(col + kc * 128));
      const __half* h = reinterpret_cast<const __half*>(&v);
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int i = kc * 8 + t;
        if (i < NN) {
          const double ai = __dmul_rn((double)__half2float(h[t]), 0.25);
          const double bi = (double)((bpk[i >> 2] >> (8 * (i & 3))) & 0xFFu);
          const double dd = __dsub_rn(__dadd_rn(__dmul_rn(s_deq, ai), o_deq), bi);
          r_val = __dadd_rn(r_val, __dmul_rn(dd, dd));
        }
      }
    }
  } else {
    const int n = g.n;
    for (int i = 0; i < N; ++i) {
      const __half qh = *reinterpret_cast<const __half*>(pool + pool_offset(d, s, i, g.K));
      const double ai = __dmul_rn((double)__half2float(qh), 0.25);
      const double bi = (double)img[(long long)(y0 + i / n) * g.W + x0 + (i % n)];
      const double dd = __dsub_rn(__dadd_rn(__dmul_rn(s_deq, ai), o_deq), bi);
      r_val = __dadd_rn(r_val, __dmul_rn(dd, dd));
    }
  }
  qs_out = qs;
  qo_out = qo;
  return r_val;
}

// The 8 isometries of domain d for the range held in `st`, in isometry order, each
// replacing the best only on strict `<` (encoder.cpp:281).
template <int NN>
static __device__ __noinline__ void evaluate_domain(RangeState& st, const Geometry& g, int d, const long long* acc,
                                                    const DomainMetaI* __restrict__ meta_i,
                                                    const unsigned char* __restrict__ pool,
                                                    const unsigned char* __restrict__ img, const uint32_t* bpk,
                                                    unsigned long long* gbest, unsigned long long* counters) {
  const DomainMetaI mi = meta_i[d];
  if (mi.den < 0) return;  // flat code block: never a candidate (encoder.cpp:223-229)
  for (int s = 0; s < kSyms; ++s) {
    unsigned qs = 0, qo = 0;
    const double r_val =
        eval_candidate<NN>(g, d, s, acc[s], mi, st.sb, st.ssb, st.thr, bpk, pool, img, st.x0, st.y0, qs, qo, counters);
    if (r_val < st.best) {
      st.best = r_val;
      st.bd = d;
      st.bs = s;
      st.bqs = qs;
      st.bqo = qo;
      if (r_val < st.thr) {
        st.thr = r_val;
        st.sqrtT = prune_sqrtT(st.ssb, st.thr, NN > 0 ? NN : g.N);
        publish_best(gbest, st.r, r_val);
      }
    }
  }
}

// Group test for one domain: the 8 isometry correlations (raw fp32 bits; all are
// non-negative exact integers, so their bit patterns order like the values) are all
// inside [center - radius, center + radius].  Negative interval ends compare below
// every non-negative pattern as signed ints, which keeps the test conservative.
__device__ __forceinline__ bool group_pruned(const uint32_t* v, float a, float e, float sb_f, float sqrtT) {
  int mx = max(max(max((int)v[0], (int)v[1]), max((int)v[2], (int)v[3])),
               max(max((int)v[4], (int)v[5]), max((int)v[6], (int)v[7])));
  int mn = min(min(min((int)v[0], (int)v[1]), min((int)v[2], (int)v[3])),
               min(min((int)v[4], (int)v[5]), min((int)v[6], (int)v[7])));
  const float center = a * sb_f;
  const float rad = __fmaf_rn(e, sqrtT, -kBoundSlack);
  const float hi = center + rad;
  const float lo = center - rad;
  return (mx <= __float_as_int(hi)) & (mn >= __float_as_int(lo));
}

__device__ __forceinline__ bool better(double r1, int d1, int s1, double r2, int d2, int s2) {
  // lexicographic (R, canonical domain index, isometry): the reference's scan order
  // with strict `<` (encoder.cpp:281, codebook.cpp:17-18)
  if (r1 != r2) return r1 < r2;
  if (d1 != d2) return (unsigned)d1 < (unsigned)d2;  // -1 (none) sorts last
  return s1 < s2;
}

#endif  // __CUDACC__

}  // namespace ficb
