// scan.cu — the tcgen05 encoder path for n in {2, 4, 8}: normalised domain pool (K1),
// the range x domain scan on the tensor cores (K2), the exact survivor evaluation and the
// lexicographic winner / record pass.
//
// What the reference computes (Searcher::search_impl, proj/src/encoder.cpp:159-296) is,
// for every range, the lexicographic minimum of (R, canonical domain index, isometry)
// over all non-flat candidates, R being the exact quantised residual (encoder.cpp:236-287).
// Its pruning stages never drop that minimum.  This path computes the same minimum with
// a different, equally output-neutral pruning:
//
//  * K1 writes every domain once as a NORMALISED operand u_j = (N q_j - Sq) / sqrt(den)
//    (fp16, |u_j| <= sqrt(N), sum u_j^2 = N), and the range side is the CENTRED range
//    b_i - Sb/N (fp16), one operand row per isometry (the reference's pre-permuted range
//    bv[s], encoder.cpp:183-190).  Their dot product is X = num / sqrt(den) with
//    num = N*acc - Sq*Sb the reference's integer correlation (encoder.cpp:241), so the
//    unconstrained least-squares lower bound of any quantised residual of the candidate,
//    R* = ssb - num^2 / (N den), is ssb - X^2/N.
//  * A candidate is dropped iff |X~| <= sqrt(N (ssb - bar - delta)) - err, where bar is an
//    ACHIEVED residual of the same range and err bounds |X~ - X| (fp16 rounding of both
//    operands, fp32 accumulation): then R >= R* > bar, so it cannot be the minimum.  The
//    test needs only the range's own threshold: per accumulator column it is one 3-input
//    |max| (FMNMX3) per two columns.
//  * Survivors (range, isometry, domain) go to a global list (full level: 40-byte mask
//    records expanded by expand_kernel; sparse levels: one selected entry per warp and tile
//    or per lane and segment); eval_kernel recomputes the exact integer correlation and runs
//    the reference's fp64 arithmetic operation by operation, lowering the range's bar
//    (atomicMin on the IEEE bits).  The scan runs as sparse levels (every s-th tile, see
//    scan_levels in fic_api.cu) and then in full, each level pruning with the bar the
//    previous ones achieved.  Every candidate whose residual equals the final bar is in the
//    full level's list; winner_kernel takes the smallest (domain, isometry) among them and
//    record_kernel re-evaluates it into the RangeMapping record.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace ficb {

constexpr int kScanRows = 256;                  // range-operand rows per CTA: 32 ranges x 8 isometries (MMA N)
constexpr int kScanRanges = kScanRows / kSyms;  // 32
constexpr int kPoolBlock = 128;                 // domains per pool-builder CTA (pool padding)
constexpr int kScanTileDom = 128;               // domains per pool tile (MMA M = TMEM lanes)
constexpr int kScanMaxStages = 16;
#ifndef FIC_EPI_WARPS
#define FIC_EPI_WARPS 16
#endif
constexpr int kScanEpiWarps = FIC_EPI_WARPS;            // 4 lane quarters x kEpiParts column parts
constexpr int kEpiParts = kScanEpiWarps / 4;
constexpr int kEpiRanges = kScanRanges / kEpiParts;    // ranges per epilogue thread
constexpr int kEpiCols = kEpiRanges * kSyms;           // TMEM columns per epilogue thread
constexpr int kScanThreads = (2 + kScanEpiWarps) * 32;
// fused scan (scan + exact evaluation in one kernel): kEvalWarps consumer warps evaluate the
// epilogue's survivors while the tensor core runs; every other warp joins them once its own
// role is done
constexpr int kEvalWarps = 2;
constexpr int kFusedThreads = (2 + kScanEpiWarps + kEvalWarps) * 32;
// Scan CTAs per SM (FIC_SCAN_CTAS, 1 or 2).  Two CTAs per SM each own ONE 256-column TMEM
// accumulator (instead of one CTA with two) and half the shared memory: twice the epilogue warps
// per SM to hide the epilogue's latency, at a 56-register budget (fp32 accumulators are then
// read 32 columns at a time).
#ifndef FIC_SCAN_CTAS
#define FIC_SCAN_CTAS 1
#endif
constexpr int kScanCtas = FIC_SCAN_CTAS;
constexpr int kTBufs = 2 / kScanCtas;  // TMEM accumulator buffers per CTA
constexpr uint32_t kScanTmemCols = 256 * kTBufs;
constexpr int kSmemBudget = kScanCtas == 1 ? 226 * 1024 : 112 * 1024;

// Survivor list entry: (encoded range r * 8 + isometry, canonical domain).
typedef uint2 SurvEntry;

// ------------------------------------------------------------------ K1: normalised pool
// One CTA per 128 domains.  Phase 1: one thread per domain contracts its 2n x 2n window
// into 2x2 group sums q (encoder.cpp:205-219) and forms Sq, Sqq and den = N*Sqq - Sq^2
// exactly; flat iff (double)den <= 16*shadow_eps (encoder.cpp:223).  Phase 2: all threads
// write the tile's fp16 operand (UMMA K-major no-swizzle core matrices, 16-byte coalesced
// chunks: [domain/8][k/8][domain%8][8 halves]) and the exact u16 q rows.
constexpr int kPoolThreads = 512;
static_assert(kPoolThreads == 4 * kPoolBlock, "pool moments: four threads per domain");

// The encode's other per-range / per-code preparations ride in the same launch (blocks past
// the pool's): the range pass (sums, variance, shadow test; encoder.cpp:165-181), the bar and
// winner-key initialisation and the dequantised code tables (one launch instead of five).
struct PrepAux {
  RangeMeta* rmeta;
  unsigned long long* shadow_count;
  unsigned long long* gbest;
  unsigned long long* win;  // 2 words per range
  double* deq;              // 2^s_bits s values, then 2^o_bits o values
  int pool_blocks;
  int aux_blocks;
  // first scan level's range operands (no bar yet: every range allpass), built by the blocks
  // past the aux ones when the encode starts with a sparse level and no seed (else nullptr)
  float* thr;
  unsigned char* ropnd;
  unsigned long long* pend_count;
};
__device__ void range_op_first_level(const unsigned char* __restrict__ img, const Geometry& g, const PrepAux& a,
                                     int mt);

__device__ void prep_aux(const unsigned char* __restrict__ img, const Geometry& g, const PrepAux& a) {
  const int tid = (blockIdx.x - a.pool_blocks) * blockDim.x + threadIdx.x;
  const int nthreads = a.aux_blocks * blockDim.x;
  for (int r = tid; r < g.R; r += nthreads) {
    int x0, y0;
    range_origin(g, r, x0, y0);
    long long sb = 0, sbb = 0;
    for (int i = 0; i < g.n; ++i) {
      const unsigned char* row = img + (long long)(y0 + i) * g.W + x0;
      for (int j = 0; j < g.n; ++j) {
        const int v = row[j];
        sb += v;
        sbb += v * v;
      }
    }
    const long long var = (long long)g.N * sbb - sb * sb;
    const int shadow = (double)var <= g.shadow_eps;
    a.rmeta[r] = RangeMeta{(int)sb, shadow, var};
    if (shadow) atomicAdd(a.shadow_count + range_slice(g, r), 1ull);  // per slice of a batch
    a.gbest[r] = 0x7ff0000000000000ull;  // +inf: no bar yet
    a.win[2 * r] = ~0ull;                // no winner yet
    a.win[2 * r + 1] = ~0ull;
  }
  const int ns = 1 << g.s_bits, no = 1 << g.o_bits;
  for (int c = tid; c < ns + no; c += nthreads) {  // UniformQuantizer::dequantize (format.hpp:34-40)
    if (c < ns) a.deq[c] = dequantize((unsigned)c, g.s_max, g.s_bits);
    else a.deq[c] = dequantize((unsigned)(c - ns), 255.0, g.o_bits);
  }
}

__global__ void __launch_bounds__(kPoolThreads)
pool_v3_kernel(const unsigned char* __restrict__ img, Geometry g, __half* __restrict__ upool,
               unsigned short* __restrict__ qpool, DomainMetaI* __restrict__ meta_i,
               unsigned long long* __restrict__ flat_count, PrepAux aux) {
  if ((int)blockIdx.x >= aux.pool_blocks + aux.aux_blocks) {
    range_op_first_level(img, g, aux, (int)blockIdx.x - aux.pool_blocks - aux.aux_blocks);
    return;
  }
  if ((int)blockIdx.x >= aux.pool_blocks) {
    prep_aux(img, g, aux);
    return;
  }
  extern __shared__ __align__(16) unsigned short sq_tile[];  // 128 x N contracted cells, then their transposes
  unsigned short* sq_tileT = sq_tile + kPoolBlock * g.N;      // per domain: TT[c][r] = q[r][c]
  __shared__ double s_inv[kPoolBlock];
  __shared__ long long s_sum[kPoolBlock];
  __shared__ long long s_sqq[kPoolBlock];
  __shared__ int s_org[kPoolBlock];  // pixel offset of each domain's window (-1: padding)
  __shared__ unsigned char s_perm[kSyms * 64];
  __shared__ unsigned s_flat;
  const int t = threadIdx.x;
  const int N = g.N, n = g.n, K = g.K;
  // N, n and K / 8 are powers of two: index arithmetic by shifts and masks (the kernel is
  // issue-bound on large pools otherwise)
  const int lgN = __ffs(N) - 1, lgn = __ffs(n) - 1, lgkc = __ffs(K >> 3) - 1;
  const long long dbase = (long long)blockIdx.x * kPoolBlock;
  if (t == 0) s_flat = 0;
  for (int k = t; k < kSyms * N; k += kPoolThreads) {  // perm_s(i) (transforms.cpp:13-26)
    const int s = k >> lgN, i = k & (N - 1);
    int sr, sc;
    symmetry_source(s, i >> lgn, i & (n - 1), n, sr, sc);
    s_perm[k] = (unsigned char)(sr * n + sc);
  }
  // a block never straddles slices of a batch (Dt is a multiple of the block)
  const int slice = g.batch > 1 ? (int)(dbase / g.Dt) : 0;
  const long long lbase = dbase - (long long)slice * (g.batch > 1 ? g.Dt : 0);  // slice-local index
  if (t < kPoolBlock) {  // domain origins once per domain (the divisions by PY and Dt)
    int o = -1;
    if (lbase + t < g.D) {
      int x, y;
      domain_origin_px(g, (int)(dbase + t), x, y);
      o = y * g.W + x;
    }
    s_org[t] = o;
  }
  __syncthreads();
  // phase 1: 2x2 group sums (encoder.cpp:213-215), one (domain, cell) per thread and step; with
  // an even step (and row stride) every cell's pixel pairs are 2-byte aligned: two 16-bit loads
  // per cell instead of four byte loads (the kernel is L1-bound on large pools)
  const bool pairs = ((g.step | g.W) & 1) == 0 && ((uintptr_t)img & 1) == 0;
  for (int idx = t; idx < (kPoolBlock << lgN); idx += kPoolThreads) {
    const int dl = idx >> lgN, j = idx & (N - 1);
    const int o = s_org[dl];
    int v = 0;
    if (o >= 0) {
      const unsigned char* row0 = img + (long long)o + (long long)(2 * (j >> lgn)) * g.W + 2 * (j & (n - 1));
      const unsigned char* row1 = row0 + g.W;
      if (pairs) {
        const unsigned a0 = *reinterpret_cast<const unsigned short*>(row0);
        const unsigned a1 = *reinterpret_cast<const unsigned short*>(row1);
        v = (int)((a0 & 0xFFu) + (a0 >> 8) + (a1 & 0xFFu) + (a1 >> 8));
      } else {
        v = row0[0] + row0[1] + row1[0] + row1[1];
      }
    }
    sq_tile[idx] = (unsigned short)v;
    sq_tileT[(dl << lgN) + ((j & (n - 1)) << lgn) + (j >> lgn)] = (unsigned short)v;
  }
  __syncthreads();
  // moments of domain t: Sq, Sqq, den = N*Sqq - Sq^2 (exact), flat iff (double)den <= 16*shadow_eps (encoder.cpp:223)
  // (kPoolThreads / kPoolBlock = 4 threads per domain, partial sums combined by shuffles)
  {
    const int dl = t >> 2, part = t & 3;
    long long s = 0, ss = 0;
    for (int j = part; j < N; j += 4) {
      const int v = sq_tile[(dl << lgN) + ((j + dl) & (N - 1))];  // rotated start: fewer bank conflicts
      s += v;
      ss += (long long)v * v;
    }
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    ss += __shfl_xor_sync(0xffffffffu, ss, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    ss += __shfl_xor_sync(0xffffffffu, ss, 2);
    if (part == 0) {
      s_sum[dl] = s;
      s_sqq[dl] = ss;
    }
  }
  __syncthreads();
  if (t < kPoolBlock) {
    const long long d = dbase + t;
    const long long s = s_sum[t], ss = s_sqq[t];
    if (s_org[t] >= 0) {
      const long long den = (long long)N * ss - s * s;
      const bool flat = (double)den <= 16.0 * g.shadow_eps;
      meta_i[d] = DomainMetaI{s, flat ? -1 : den};
      s_inv[t] = flat ? 0.0 : 1.0 / sqrt((double)den);
      if (flat) atomicAdd(&s_flat, 1u);
    } else {
      meta_i[d] = DomainMetaI{0, -1};
      s_inv[t] = 0.0;
    }
    s_sum[t] = s;
  }
  __syncthreads();
  if (t == 0 && s_flat) atomicAdd(flat_count + slice, (unsigned long long)s_flat);  // per slice
  // phase 2a: fp16 normalised operand u = (N q - Sq) / sqrt(den), UMMA K-major no-swizzle
  // core matrices, chunk c = ((dl/8) * (K/8) + k/8) * 8 + dl%8 (16-byte coalesced stores)
  uint4* out = reinterpret_cast<uint4*>(upool + dbase * K);
  for (int c = t; c < (kPoolBlock << lgkc); c += kPoolThreads) {
    const int d8 = c & 7, kc = (c >> 3) & ((1 << lgkc) - 1), dg = (c >> 3) >> lgkc;
    const int dl = dg * 8 + d8;
    const double inv = s_inv[dl];
    const double sN = (double)s_sum[dl];
    uint32_t w[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      uint32_t pair = 0;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int k = kc * 8 + 2 * h + u;
        float v = 0.f;
        if (k < N) v = (float)(((double)N * (double)sq_tile[(dl << lgN) + k] - sN) * inv);
        pair |= (uint32_t)__half_as_ushort(__float2half_rn(v)) << (16 * u);
      }
      w[h] = pair;
    }
    out[c] = make_uint4(w[0], w[1], w[2], w[3]);
  }
  // phase 2b: exact contracted cells per isometry, row (d, s)[i] = q[perm_s(i)] (u16): the
  // survivor evaluation reads one contiguous row instead of gathering through the isometry.
  // Pixel row r of isometry s is one source row or column of the block, forward or reversed
  // (symmetry_source): s 0 row r, 1 column r reversed, 2 row m-r reversed, 3 column m-r,
  // 4 row r reversed, 5 row m-r, 6 column r, 7 column m-r reversed (m = n - 1) — one aligned
  // shared-memory vector load from the tile or its transpose plus a half-word reversal.
  if (n == 8) {
    uint4* qdst = reinterpret_cast<uint4*>(qpool + dbase * kSyms * 64);
    for (int c = t; c < kPoolBlock * kSyms * 8; c += kPoolThreads) {
      const int r = c & 7, sym = (c >> 3) & 7, dl = c >> 6;
      const bool col = (0xCAu >> sym) & 1u, rev = (0x96u >> sym) & 1u, mir = (0xACu >> sym) & 1u;
      const int idx = mir ? 7 - r : r;
      const uint4 v = reinterpret_cast<const uint4*>((col ? sq_tileT : sq_tile) + (dl << 6))[idx];
      qdst[c] = rev ? make_uint4(__byte_perm(v.w, 0, 0x1032), __byte_perm(v.z, 0, 0x1032), __byte_perm(v.y, 0, 0x1032),
                                 __byte_perm(v.x, 0, 0x1032))
                    : v;
    }
  } else if (n == 4) {
    uint2* qdst = reinterpret_cast<uint2*>(qpool + dbase * kSyms * 16);
    for (int c = t; c < kPoolBlock * kSyms * 4; c += kPoolThreads) {
      const int r = c & 3, sym = (c >> 2) & 7, dl = c >> 5;
      const bool col = (0xCAu >> sym) & 1u, rev = (0x96u >> sym) & 1u, mir = (0xACu >> sym) & 1u;
      const int idx = mir ? 3 - r : r;
      const uint2 v = reinterpret_cast<const uint2*>((col ? sq_tileT : sq_tile) + (dl << 4))[idx];
      qdst[c] = rev ? make_uint2(__byte_perm(v.y, 0, 0x1032), __byte_perm(v.x, 0, 0x1032)) : v;
    }
  } else {  // N == 4: one 8-byte row per (domain, isometry)
    uint2* qdst = reinterpret_cast<uint2*>(qpool + dbase * kSyms * N);
    for (int row = t; row < kPoolBlock * kSyms; row += kPoolThreads) {
      const int sym = row & 7, dl = row >> 3;
      const unsigned char* pr = s_perm + sym * N;
      const unsigned short* qs = sq_tile + dl * N;
      qdst[row] = make_uint2((uint32_t)qs[pr[0]] | ((uint32_t)qs[pr[1]] << 16),
                             (uint32_t)qs[pr[2]] | ((uint32_t)qs[pr[3]] << 16));
    }
  }
}

// ------------------------------------------------------------------ bound threshold
// |X~| <= T  =>  R* >= bar + delta  (see the header).  err covers the fp16 rounding of both
// operands (relative 2^-11 each, |sum u b| <= |u| |b| = sqrt(N * ssb)), the fp32
// accumulation of K products (2^-21 relative each, generous) and fp16 subnormals.
// f16acc (the full level with an fp16 accumulator, flags & 256): each of the K/16 MMAs rounds
// the running sum to fp16, to nearest even (pinned on the B200 by tools/f16acc_probe.cu: ties
// and quarter points, inside a K=16 step and across steps); every intermediate partial sum is
// bounded by sum |u_i b_i| <= |u| |b|, so the first K/16 - 1 roundings add at most
// (K/16 - 1) 2^-11 |u| |b|, while the last one is relative to the result the test compares:
// |y| <= |fl(y)| / (1 - 2^-11), so a column passing the test at T (1 - 2^-11) has |y| <= T
// (K = 16: the only rounding is that last one, ~T instead of ~|u| |b| wide).
// Invariant: no scaled operand (fp16) and no fp16 partial sum may overflow, because the
// epilogue's tests do not agree on non-finite values (the fp16 bit-pattern test counts inf and
// NaN as hits, while __hmax2 in the whole-tile vote and the per-range max drops NaN operands).
// The guard below keeps them unreachable: a range whose scaled bound |u| |b| / T (>= every
// |b_i - mean| / T) exceeds 60000 gets no bar (all its columns pass).
__device__ __forceinline__ float scan_threshold(double ssb, double bar, int N, int K, bool f16acc = false) {
  const double t = (ssb - bar) - 1e-6 * (1.0 + bar);
  if (!(t > 0.0)) return -1.f;  // no usable bar (also bar == +inf): everything survives
  const double sqrtT = sqrt((double)N * t) * (1.0 - 1e-6);
  const double ub = sqrt((double)N * ssb);
  double err = (9.765625e-4 * 1.0005 + (double)K * 4.76837158203125e-7) * 1.05 * ub + 0.01;
  if (f16acc) err += (double)(K / 16 - 1) * 4.8828125e-4 * 1.05 * ub;
  const double T = (sqrtT - err) * (f16acc ? 1.0 - 4.8828125e-4 * 1.05 : 1.0);
  if (T * 60000.0 < ub * 1.01) return -1.f;
  return T > 0.0 ? __double2float_rd(T) : -1.f;
}

// ------------------------------------------------------------------ exact evaluation
// One candidate of a range, given a_i = q[perm_s(i)] (its domain's contracted cells in the
// isometry's order, i.e. range-pixel order, encoder.cpp:236-240) packed two u16 per word,
// following encoder.cpp:241-280 operation by operation (round-to-nearest intrinsics, no
// FMA).  Returns the residual, or +inf when a bound shows it cannot reach `thr` (tight LS
// bound, then the reference's own screens with their +1e-3 margins).  Control flow does
// not depend on the isometry.
__device__ __forceinline__ int q_at(const uint32_t* qw, int i) { return (int)((qw[i >> 1] >> (16 * (i & 1))) & 0xFFFFu); }

// sum_i q_i b_i for q packed two u16 per word and b four u8 per word: two DP2A per four
// pixels (exact: every partial sum < 2^24).
template <int NN>
__device__ __forceinline__ int dot_q_b(const uint32_t* qw, const uint32_t* bpk) {
  unsigned acc = 0;
#pragma unroll
  for (int w = 0; w < NN / 4; ++w) {
    acc = __dp2a_lo(qw[2 * w], bpk[w], acc);
    acc = __dp2a_hi(qw[2 * w + 1], bpk[w], acc);
  }
  return (int)acc;
}

template <int NN>
__device__ __forceinline__ double eval_exact(const Geometry& g, const uint32_t* qw, const uint32_t* bpk, int sb,
                                             double ssb, long long sqv, long long denv, double thr, bool screens,
                                             unsigned& qs_out, unsigned& qo_out) {
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  int acc = 0;
#pragma unroll
  for (int i = 0; i < NN; ++i) acc += q_at(qw, i) * (int)((bpk[i >> 2] >> (8 * (i & 3))) & 0xFFu);
  const double count_d = (double)NN;
  const double inv_count = 1.0 / count_d;
  const double den_d = (double)denv;
  const double sa_d = __dmul_rn((double)sqv, 0.25);
  const double sb_d = (double)sb;
  const double smax = g.s_max;
  const long long num_q = (long long)NN * acc - sqv * (long long)sb;
  const double num_d = (double)num_q;
  if (screens) {
    const double rstar = ssb - (num_d * num_d) / (count_d * den_d);
    if (rstar >= thr + 1e-6 * (1.0 + thr)) return inf;
  }
  const double s_raw = __ddiv_rn(__dmul_rn(4.0, num_d), den_d);       // encoder.cpp:248
  const double sc = clampd(s_raw, -smax, smax);                       // :249
  const unsigned qs = quantize(sc, smax, g.s_bits);                   // :250
  const double s_deq = dequantize(qs, smax, g.s_bits);                // :251
  const double cov = __dmul_rn(__dmul_rn(num_d, 0.25), inv_count);    // :253-263
  const double var_a = __dmul_rn(__dmul_rn(den_d, 0.0625), inv_count);
  const double parabola =
      __dadd_rn(__dsub_rn(ssb, __dmul_rn(__dmul_rn(2.0, s_deq), cov)), __dmul_rn(__dmul_rn(s_deq, s_deq), var_a));
  if (screens && parabola >= thr + 1e-3) return inf;
  const double o = clampd(__dmul_rn(__dsub_rn(sb_d, __dmul_rn(sc, sa_d)), inv_count), -255.0, 255.0);  // :265-267
  const unsigned qo = quantize(o, 255.0, g.o_bits);
  const double o_deq = dequantize(qo, 255.0, g.o_bits);
  const double o_gap = __dsub_rn(o_deq, __dmul_rn(__dsub_rn(sb_d, __dmul_rn(s_deq, sa_d)), inv_count));
  const double screen = __dadd_rn(parabola, __dmul_rn(__dmul_rn(count_d, o_gap), o_gap));
  if (screens && screen >= thr + 1e-3) return inf;  // :272
  double r_val = 0.0;                                 // :274-280, pixel order
#pragma unroll
  for (int i = 0; i < NN; ++i) {
    const double ai = __dmul_rn((double)q_at(qw, i), 0.25);
    const double bi = (double)((bpk[i >> 2] >> (8 * (i & 3))) & 0xFFu);
    const double dd = __dsub_rn(__dadd_rn(__dmul_rn(s_deq, ai), o_deq), bi);
    r_val = __dadd_rn(r_val, __dmul_rn(dd, dd));
  }
  qs_out = qs;
  qo_out = qo;
  return r_val;
}

// Dequantised values of every code (UniformQuantizer::dequantize, format.hpp:34-40), computed
// once per encode with the same device function, so table lookups are bit-identical to it.
struct DeqTables {
  const double* s;  // 2^s_bits entries
  const double* o;  // 2^o_bits entries
};

// The exact residual of encoder.cpp:274-280 (pixel order, each operation rounded) for given
// dequantised s and o, operands read from memory in a rolled loop (out of line and light on
// registers: only candidates that pass every screen get here).
template <int NN>
__device__ __noinline__ double residual_reload(const Geometry g, const unsigned short* __restrict__ qpool,
                                               const unsigned char* __restrict__ img, int d, int s, int x0, int y0,
                                               double s_deq, double o_deq) {
  constexpr int n = NN == 4 ? 2 : (NN == 16 ? 4 : 8);
  const unsigned short* qrow = qpool + ((long long)d * kSyms + s) * NN;
  double r_val = 0.0;
#pragma unroll 1
  for (int i = 0; i < NN; ++i) {
    const double ai = __dmul_rn((double)qrow[i], 0.25);
    const double bi = (double)img[(long long)(y0 + i / n) * g.W + x0 + i % n];
    const double dd = __dsub_rn(__dadd_rn(__dmul_rn(s_deq, ai), o_deq), bi);
    r_val = __dadd_rn(r_val, __dmul_rn(dd, dd));
  }
  return r_val;
}

// eval_exact for the rare boundary cases of eval_fast, operands read from memory in rolled
// loops (out of line, light on registers).  Same arithmetic as eval_exact.
template <int NN>
__device__ __noinline__ double eval_exact_reload(const Geometry g, const unsigned short* __restrict__ qpool,
                                                 const unsigned char* __restrict__ img, int d, int s, int x0, int y0,
                                                 int sb, double ssb, long long sqv, long long denv, double thr,
                                                 bool screens, unsigned* qs_out, unsigned* qo_out) {
  constexpr int n = NN == 4 ? 2 : (NN == 16 ? 4 : 8);
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  const unsigned short* qrow = qpool + ((long long)d * kSyms + s) * NN;
  int acc = 0;
#pragma unroll 1
  for (int i = 0; i < NN; ++i) acc += (int)qrow[i] * (int)img[(long long)(y0 + i / n) * g.W + x0 + i % n];
  const double count_d = (double)NN;
  const double inv_count = 1.0 / count_d;
  const double den_d = (double)denv;
  const double sa_d = __dmul_rn((double)sqv, 0.25);
  const double sb_d = (double)sb;
  const double smax = g.s_max;
  const long long num_q = (long long)NN * acc - sqv * (long long)sb;
  const double num_d = (double)num_q;
  if (screens) {
    const double rstar = ssb - (num_d * num_d) / (count_d * den_d);
    if (rstar >= thr + 1e-6 * (1.0 + thr)) return inf;
  }
  const double s_raw = __ddiv_rn(__dmul_rn(4.0, num_d), den_d);
  const double sc = clampd(s_raw, -smax, smax);
  const unsigned qs = quantize(sc, smax, g.s_bits);
  const double s_deq = dequantize(qs, smax, g.s_bits);
  const double cov = __dmul_rn(__dmul_rn(num_d, 0.25), inv_count);
  const double var_a = __dmul_rn(__dmul_rn(den_d, 0.0625), inv_count);
  const double parabola =
      __dadd_rn(__dsub_rn(ssb, __dmul_rn(__dmul_rn(2.0, s_deq), cov)), __dmul_rn(__dmul_rn(s_deq, s_deq), var_a));
  if (screens && parabola >= thr + 1e-3) return inf;
  const double o = clampd(__dmul_rn(__dsub_rn(sb_d, __dmul_rn(sc, sa_d)), inv_count), -255.0, 255.0);
  const unsigned qo = quantize(o, 255.0, g.o_bits);
  const double o_deq = dequantize(qo, 255.0, g.o_bits);
  const double o_gap = __dsub_rn(o_deq, __dmul_rn(__dsub_rn(sb_d, __dmul_rn(s_deq, sa_d)), inv_count));
  const double screen = __dadd_rn(parabola, __dmul_rn(__dmul_rn(count_d, o_gap), o_gap));
  if (screens && screen >= thr + 1e-3) return inf;
  *qs_out = qs;
  *qo_out = qo;
  return residual_reload<NN>(g, qpool, img, d, s, x0, y0, s_deq, o_deq);
}

// floor(t + 0.5) of a scaled quantiser argument known to within ~1e-12, or -1 when it is
// within 1e-9 of a rounding boundary (the caller then takes the exact path).
__device__ __forceinline__ int safe_code(double scaled) {
  const double t = scaled + 0.5;
  const double f = floor(t);
  const double fr = t - f;
  return (fr < 1e-9 || fr > 1.0 - 1e-9) ? -1 : (int)f;
}

// Same result as eval_exact (bit-identical residual and codes, same +inf cases up to the
// screens, which only ever reject candidates whose residual exceeds thr + 1e-3 - 1e-9),
// but without IEEE divisions on the common path: s and o are quantised from reciprocal
// products and the codes are checked to lie away from rounding boundaries (else the
// exact operation-by-operation path is taken); the dequantised values come from tables.
// upper_only: return an upper bound of the exact residual from the closed form
// parabola(s_deq) + N*o_gap^2 (seeding the bar; no residual loop).
template <int NN>
__device__ __forceinline__ double eval_fast_acc(const Geometry& g, int acc, const uint32_t* qw, const uint32_t* bpk,
                                                int sb, double ssb, long long sqv, long long denv, double thr,
                                                bool screens, bool upper_only, const DeqTables& tab,
                                                const unsigned short* qpool, const unsigned char* img, int d, int s,
                                                int x0, int y0, unsigned& qs_out, unsigned& qo_out,
                                                bool* pending = nullptr) {
  // (acc: the exact correlation sum_i q[perm_s(i)] b_i; qw / bpk are only read by the inline
  // residual, i.e. never when upper_only)
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  const long long num_q = (long long)NN * acc - sqv * (long long)sb;
  const double num_d = (double)num_q, den_d = (double)denv, sb_d = (double)sb;
  const double smax = g.s_max;
  const unsigned ms = (1u << g.s_bits) - 1u, mo = (1u << g.o_bits) - 1u;
  // s_raw = 4 num / den, clamped; quantised away from boundaries
  const double s_raw = 4.0 * num_d * (1.0 / den_d);
  const double sc = fmin(fmax(s_raw, -smax), smax);
  int qs;
  if (num_q == 0) {
    qs = 0;
  } else {
    const int c = safe_code((sc + smax) * (1.0 / (2.0 * smax)) * (double)ms);
    if (c < 0 || fabs(fabs(s_raw) - smax) < 1e-12 * smax) goto exact;
    qs = c < 1 ? 1 : (c > (int)ms ? (int)ms : c);
  }
  {
    const double s_deq = tab.s[qs];
    const double sa_d = (double)sqv * 0.25;
    const double inv_count = 1.0 / (double)NN;
    const double cov = num_d * 0.25 * inv_count;
    const double var_a = den_d * 0.0625 * inv_count;
    const double parabola = ssb - 2.0 * s_deq * cov + s_deq * s_deq * var_a;
    if (screens && parabola >= thr + (1e-3 - 1e-9)) return inf;
    // o = clamp((Sb - s Sa) / N): the same rounded operations as the reference (the division by
    // N = 2^k is exact), so the clamp decides identically; a clamped o = +-255 quantises to the
    // top code / code 1 away from any rounding boundary (safe_code checks every other case)
    const double o = fmin(fmax((sb_d - sc * sa_d) * inv_count, -255.0), 255.0);
    if (fabs(o) < 1e-9) goto exact;  // quantize(0) is the special code 0
    const int c = safe_code((o + 255.0) * (1.0 / 510.0) * (double)mo);
    if (c < 0) goto exact;
    const unsigned qo = c < 1 ? 1u : (c > (int)mo ? mo : (unsigned)c);
    const double o_deq = tab.o[qo];
    const double o_gap = o_deq - (sb_d - s_deq * sa_d) * inv_count;
    const double screen = parabola + (double)NN * o_gap * o_gap;
    if (upper_only) {
      qs_out = qs;
      qo_out = qo;
      return screen * (1.0 + 1e-9) + 1e-6;
    }
    if (screens && screen >= thr + (1e-3 - 1e-9)) return inf;
    qs_out = qs;
    qo_out = qo;
    if (pending) {  // the caller computes the residual in a separate, convergent pass
      *pending = true;
      return inf;
    }
    // the exact residual (encoder.cpp:274-280, pixel order, each operation rounded) from the
    // operands already in registers
    double r_val = 0.0;
#pragma unroll
    for (int i = 0; i < NN; ++i) {
      const double ai = __dmul_rn((double)q_at(qw, i), 0.25);
      const double bi = (double)((bpk[i >> 2] >> (8 * (i & 3))) & 0xFFu);
      const double dd = __dsub_rn(__dadd_rn(__dmul_rn(s_deq, ai), o_deq), bi);
      r_val = __dadd_rn(r_val, __dmul_rn(dd, dd));
    }
    return r_val;
  }
exact:
  return eval_exact_reload<NN>(g, qpool, img, d, s, x0, y0, sb, ssb, sqv, denv, upper_only ? inf : thr,
                               screens && !upper_only, &qs_out, &qo_out);
}

template <int NN>
__device__ __forceinline__ double eval_fast(const Geometry& g, const uint32_t* qw, const uint32_t* bpk, int sb,
                                            double ssb, long long sqv, long long denv, double thr, bool screens,
                                            bool upper_only, const DeqTables& tab, const unsigned short* qpool,
                                            const unsigned char* img, int d, int s, int x0, int y0,
                                            unsigned& qs_out, unsigned& qo_out, bool* pending = nullptr) {
  return eval_fast_acc<NN>(g, dot_q_b<NN>(qw, bpk), qw, bpk, sb, ssb, sqv, denv, thr, screens, upper_only, tab, qpool,
                           img, d, s, x0, y0, qs_out, qo_out, pending);
}

__device__ __forceinline__ double load_bar(const unsigned long long* gbest, int r) {
  return __longlong_as_double((long long)__ldcg(gbest + r));
}

// Operands of the survivor evaluation (scan epilogue bounds, fused consumers).
struct EvalCtx {
  const unsigned char* img;
  const unsigned short* qpool;
  const DomainMetaI* meta_i;
  const RangeMeta* rmeta;
  unsigned long long* gbest;
  unsigned __int128* win;
  DeqTables tab;
};



__global__ void deq_tables_kernel(Geometry g, double* ts, double* to) {
  const int ns = 1 << g.s_bits, no = 1 << g.o_bits;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ns + no; c += gridDim.x * blockDim.x) {
    if (c < ns) ts[c] = dequantize((unsigned)c, g.s_max, g.s_bits);
    else to[c - ns] = dequantize((unsigned)(c - ns), 255.0, g.o_bits);
  }
}

// The (domain d, isometry s) row of the q8 pool into registers.
template <int NN>
__device__ __forceinline__ void load_q8_row(const unsigned short* __restrict__ qpool, int d, int s, uint32_t* qw) {
  const unsigned short* row = qpool + ((long long)d * kSyms + s) * NN;
  if constexpr (NN >= 8) {
#pragma unroll
    for (int w = 0; w < NN / 8; ++w) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(row) + w);
      qw[4 * w] = v.x;
      qw[4 * w + 1] = v.y;
      qw[4 * w + 2] = v.z;
      qw[4 * w + 3] = v.w;
    }
  } else {
    const uint2 v = __ldg(reinterpret_cast<const uint2*>(row));
    qw[0] = v.x;
    qw[1] = v.y;
  }
}


// ------------------------------------------------------------------ seed
// Exact evaluation of the 8 isometries of the (2h+1)^2 grid domains around each range's own
// 2x-scaled neighbourhood (self-similar candidates that usually fit well) to give the
// first scan level a bar.  One thread per (range, local domain, isometry).


// HALF: the (2 HALF + 1)^2 local domains (small pools: HALF = 0, only the range's own 2x-scaled
// neighbourhood; large pools: HALF = 1).
template <int NN, int HALF>
__global__ void __launch_bounds__(128)
seed_v3_kernel(const unsigned char* __restrict__ img, Geometry g, const unsigned short* __restrict__ qpool,
               const DomainMetaI* __restrict__ meta_i, const RangeMeta* __restrict__ rmeta,
               unsigned long long* __restrict__ gbest, DeqTables tab) {
  constexpr int kSeedHalf = HALF, kSeedSide = 2 * HALF + 1, kSeedPerRange = kSeedSide * kSeedSide * kSyms;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const bool in = tid < (long long)g.R * kSeedPerRange && g.D > 0;
  const int r = in ? (int)(tid / kSeedPerRange) : -1, k = (int)(tid % kSeedPerRange);
  const int s = k % kSyms, w = k / kSyms;
  unsigned long long key = 0x7ff0000000000000ull;  // +inf
  if (in) {
    int x0, y0;
    range_origin(g, r, x0, y0);
    const int b = range_slice(g, r);
    const int cx = x0 - g.n / 2, cy = y0 - b * g.H1 - g.n / 2;  // slice-local
    const int xi0 = min(max(cx / g.step, 0), g.PX - 1), yi0 = min(max(cy / g.step, 0), g.PY - 1);
    const int xi = xi0 + w / kSeedSide - kSeedHalf, yi = yi0 + w % kSeedSide - kSeedHalf;
    if (xi >= 0 && yi >= 0 && xi < g.PX && yi < g.PY) {
      const int d = b * g.Dt + xi * g.PY + yi;
      // all operand loads depend only on (r, d, s): issued together, one memory round trip
      const RangeMeta m = rmeta[r];
      const DomainMetaI mi = meta_i[d];
      uint32_t qw[NN / 2], bpk[NN / 4];
      load_q8_row<NN>(qpool, d, s, qw);
      load_range_words<NN>(img, g, x0, y0, bpk);
      if (!m.shadow && mi.den >= 0) {
        unsigned qs, qo;
        // an upper bound of the candidate's exact residual is a valid pruning bar
        const double v = eval_fast<NN>(g, qw, bpk, m.sb, (double)m.var / (double)NN, mi.sq, mi.den,
                                       __longlong_as_double(0x7ff0000000000000ll), false, true, tab, qpool, img, d,
                                       s, x0, y0, qs, qo);
        key = (unsigned long long)__double_as_longlong(v);
      }
    }
  }
  // minimum over the warp's lanes of the same range (consecutive lanes: contiguous segments),
  // one atomic per (warp, range) instead of one per candidate
  const unsigned lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long ok = __shfl_down_sync(0xffffffffu, key, o);
    const int orr = __shfl_down_sync(0xffffffffu, r, o);
    if (lane + o < 32 && orr == r && ok < key) key = ok;
  }
  const int prev_r = __shfl_up_sync(0xffffffffu, r, 1);
  if (in && (lane == 0 || prev_r != r) && key < 0x7ff0000000000000ull) atomicMin(gbest + r, key);
}

// ------------------------------------------------------------------ pipeline trace
// FIC_DEBUG bit 5 (32), trace builds: scan CTA 0 records clock64() stamps of its first kTraceTiles tiles:
// [tile][0..2] the MMA issuer before / after waiting for the TMEM buffer and after the pool tile
// landed, [tile][3 + e] epilogue warp e releasing the tile, [tile][19 + e] warp e done with it,
// [tile][35 + e] warp e past the per-range test (full level).
// Read with fic_debug_trace (tools/trace.py).
constexpr int kTraceTiles = 256;
constexpr int kTraceSlots = 51;
__device__ long long g_trace[kTraceTiles * kTraceSlots];

// Compiled in only with -DFIC_TRACE (FIC_TRACE=1 python -m paper_1404_0774_b200.build): the
// stamps cost ~10% of the scan even when disabled at run time.
// The scan's decomposition switches (FIC_DEBUG 8 / 16 / 128: no test, no MMAs, no TMEM reads;
// DESIGN.md section 5).  Compiling them out (-DFIC_SCAN_DEBUG=0) removes a few instructions per
// tile but measured SLOWER (cfg2 full level 96.4 -> 101.5 us, cfg3 1071 -> 1127 us: the
// schedule of the epilogue loop changes), so they stay in.
#ifndef FIC_SCAN_DEBUG
#define FIC_SCAN_DEBUG 1
#endif
constexpr bool kScanDebug = FIC_SCAN_DEBUG != 0;
__device__ __forceinline__ void trace_stamp(const Geometry& g, int tile, int slot) {
#ifdef FIC_TRACE
  if ((g.flags & 32) && blockIdx.x == 0 && tile < kTraceTiles) g_trace[tile * kTraceSlots + slot] = clock64();
#else
  (void)g;
  (void)tile;
  (void)slot;
#endif
}

int scan_trace_copy(long long* out, int n) {
  const int m = n < kTraceTiles * kTraceSlots ? n : kTraceTiles * kTraceSlots;
  return cudaMemcpyFromSymbol(out, g_trace, (size_t)m * sizeof(long long)) == cudaSuccess ? m : -1;
}

// ------------------------------------------------------------------ K2: tensor-core scan
struct ScanSmem {
  uint32_t r_bytes, p_bytes, stages, r_off, p_off, bar_off, wbuf_off, total;
};

// ------------------------------------------------------------------ fused evaluation
// The epilogue warps publish finished chunks of survivors (16 mask records at the full level,
// 32 direct entries at sparse levels) into a CTA-local bounded queue (Vyukov: seq[i] == t: slot
// free for ticket t, == t + 1: filled by ticket t); consumer warps take chunks in ticket order,
// expand records into a per-warp buffer of entries and evaluate 32 at a time with the exact
// arithmetic of eval_fast (encoder.cpp:236-287), lowering the range's bar and keeping the
// lexicographic (residual, domain * 8 + isometry) minimum of every evaluated candidate in a
// 128-bit key per range — so no survivor list round trip, expand / eval / residual / winner pass.
constexpr uint32_t kRing = 512;
constexpr int kEvalBuf = 64;
constexpr uint32_t kChunkEntries = 0x80000000u;  // chunk id flag: an entry chunk (sparse levels)
constexpr uint32_t kRingEmpty = 0xFFFFFFFFu;

struct EvalRing {
  uint32_t seq[kRing];
  uint32_t ids[kRing];
  unsigned head, tail, done, entries;
};
constexpr uint32_t kEvalConsumers = kScanEpiWarps + 2 + kEvalWarps;  // every warp consumes eventually
constexpr uint32_t kEvalSmem = (uint32_t)sizeof(EvalRing) + kEvalConsumers * kEvalBuf * 8;

// Shared memory: two range operands (256 rows x K fp16 each), a ring of pool tiles
// (128 domains x K fp16), barriers, (fused) the evaluation queue and per-warp entry buffers.
__host__ __device__ inline ScanSmem scan_smem_layout(int K, bool fused = false) {
  ScanSmem L;
  L.r_bytes = kScanRows * K * 2;
  L.p_bytes = kScanTileDom * K * 2;
  L.r_off = 0;
  L.p_off = 2 * L.r_bytes;
  const uint32_t fixed = L.p_off + 512 + (fused ? kEvalSmem : 0u);
  uint32_t st = (kSmemBudget - fixed) / L.p_bytes;
  L.stages = st > kScanMaxStages ? kScanMaxStages : st;
  L.bar_off = L.p_off + L.stages * L.p_bytes;
  L.wbuf_off = L.bar_off + 512;
  L.total = L.wbuf_off + (fused ? kEvalSmem : 0u);
  return L;
}

// Work of one scan level.  A "segment" is (m-tile, level-tile range): the CTA keeps the
// m-tile's range operand resident and streams the pool tiles of the range.  Full rounds:
// CTA c takes m-tile r*G + c over all level tiles (all CTAs sweep the pool in step, so each
// pool tile is read from L2 by every CTA within a short window).  The m-tiles left over
// (M' < G) are split into k chunks of the tile range, ordered chunk-major, and the M'*k
// units are shared out contiguously.
struct ScanLevel {
  int stride;     // tile stride of this level (1 = full scan)
  int n_lvl;      // tiles in the level: ceil(n_tiles / stride)
  int m_tiles;    // 256-row range tiles: ceil(R / 32)
  int rounds;     // full rounds: m_tiles / G
  int rem;        // m-tiles of the last round: m_tiles % G
  int k;          // chunks per leftover m-tile
  int select;     // sparse levels: 1, 2 each range's best column per warp and tile (2: small pools), 3 per lane and segment
  int coarse;     // 1: whole-tile |max| vote before the per-range test (large pools: rare hits)
  int lanes_per_best;  // select == 3: lanes sharing one best entry per range (1, 2 or 4)
  int rotate;          // epilogue column parts rotate over the warps tile by tile (select != 3)
};

struct Segment {
  int m, j0, j1;  // m-tile, level tiles [j0, j1)
};

// (32-bit arithmetic: rem < G <= 256 CTAs, k <= 16, level tiles < 2^20, so every product fits)
__host__ __device__ inline int seg_count(const ScanLevel& lv, int c, int G) {
  if (lv.rem == 0) return lv.rounds;
  const unsigned U = (unsigned)lv.rem * (unsigned)lv.k;
  return lv.rounds + (int)(U * (unsigned)(c + 1) / (unsigned)G - U * (unsigned)c / (unsigned)G);
}

__host__ __device__ inline Segment seg_at(const ScanLevel& lv, int c, int G, int s) {
  Segment sg;
  if (s < lv.rounds) {
    sg.m = s * G + c;
    sg.j0 = 0;
    sg.j1 = lv.n_lvl;
    return sg;
  }
  const unsigned U = (unsigned)lv.rem * (unsigned)lv.k;
  const unsigned u = U * (unsigned)c / (unsigned)G + (unsigned)(s - lv.rounds);
  const unsigned chunk = u / (unsigned)lv.rem, mr = u % (unsigned)lv.rem;
  sg.m = lv.rounds * G + (int)mr;
  sg.j0 = (int)((unsigned)lv.n_lvl * chunk / (unsigned)lv.k);
  sg.j1 = (int)((unsigned)lv.n_lvl * (chunk + 1) / (unsigned)lv.k);
  return sg;
}

// Operand scale of a range with scan threshold T: rows are divided by T so every column's
// test is |X~/T| > 1.  Thresholds below 1e-3 (no usable bar, exhaustive mode) and shadow or
// padding ranges get scale 0; the former are flagged to the epilogue (all columns pass).
// (1 + 1e-6) / T >= 1/T even after rounding, so |X~ * scale| <= 1 implies |X~| <= T.
__device__ __forceinline__ float range_scale(float T) { return T > 1e-3f && T < 1e29f ? (1.0f + 1e-6f) / T : 0.f; }
__device__ __forceinline__ bool range_allpass(float T) { return !(T > 1e-3f); }
// The full level accumulates in fp16 (flags & 256, FIC_F16ACC=1): halves the epilogue's TMEM
// read (two columns per register, tcgen05.ld .pack::16b) and its |max| test (half2 VHMNMX).
__host__ __device__ __forceinline__ bool scan_f16acc(const Geometry& g) { return (g.flags & 256) != 0; }

// Range operand of m-tile `mt` into `sR` (threads [tid, tid + nthreads)): row
// rl * 8 + s holds the centred range rl permuted by isometry s's inverse and scaled,
// R[row][j] = (b[i] - Sb/N) / T_r with perm_s(i) = j, so sum_j u_j R[row][j] = X / T_r.
__device__ void build_ranges(unsigned char* sR, const unsigned char* __restrict__ img, const Geometry& g,
                             const RangeMeta* __restrict__ rmeta, const float* __restrict__ thr, int mt, int tid,
                             int nthreads, int chunks) {
  const int K = g.K, N = g.N, n = g.n;
  for (int c = tid; c < chunks; c += nthreads) {
    const int row = c / (K / 8), kc = c % (K / 8);
    const int rl = row >> 3, s = row & 7;
    const int r = mt * kScanRanges + rl;
    const int sinv = s == 1 ? 3 : (s == 3 ? 1 : s);  // inverse isometries: 1 <-> 3, the others are involutions
    uint32_t w[4] = {0, 0, 0, 0};
    if (r < g.R) {
      int x0, y0;
      range_origin(g, r, x0, y0);
      const float mean = (float)rmeta[r].sb / (float)N;  // exact: N is a power of two
      float scale = range_scale(thr[r]);
      // a range without a usable bar keeps every column at the full level; at sparse levels its
      // columns are the normalised correlations, so the selection there still picks the best
      if (range_allpass(thr[r])) scale = rsqrtf((float)rmeta[r].var / (float)N + 1.0f);
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        const int j = kc * 8 + h;
        if (j < N) {
          int ir, ic;
          symmetry_source(sinv, j / n, j % n, n, ir, ic);  // i with perm_s(i) = j
          const float v = ((float)img[(long long)(y0 + ir) * g.W + x0 + ic] - mean) * scale;
          w[h >> 1] |= (uint32_t)__half_as_ushort(__float2half_rn(v)) << (16 * (h & 1));
        }
      }
    }
    *reinterpret_cast<uint4*>(sR + (row >> 3) * K * 16 + kc * 128 + (row & 7) * 16) =
        make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// build_ranges for a compile-time range size NN = n * n (4, 16, 64): shifts instead of
// divisions, and the inverse isometry's source cell from three bitmasks instead of a switch
// (the rows of one warp carry different isometries): swap (0xCA), first flipped (0xA6),
// second flipped (0x9C), the same map as symmetry_source (transforms.cpp:13-26).
template <int NN>
__device__ void build_ranges_n(unsigned char* sR, const unsigned char* __restrict__ img, const Geometry& g,
                               const RangeMeta* __restrict__ rmeta, const float* __restrict__ thr, int mt, int tid,
                               int nthreads, int chunks) {
  constexpr int n = NN == 4 ? 2 : (NN == 16 ? 4 : 8);
  constexpr int K = NN < 16 ? 16 : NN;
  constexpr int KC = K / 8;
  constexpr int m = n - 1;
  for (int c = tid; c < chunks; c += nthreads) {
    const int row = c / KC, kc = c % KC;
    const int rl = row >> 3, s = row & 7;
    const int r = mt * kScanRanges + rl;
    const int sinv = s == 1 ? 3 : (s == 3 ? 1 : s);  // inverse isometries: 1 <-> 3, the others are involutions
    const bool swap = (0xCAu >> sinv) & 1u, f0 = (0xA6u >> sinv) & 1u, f1 = (0x9Cu >> sinv) & 1u;
    uint32_t w[4] = {0, 0, 0, 0};
    if (r < g.R) {
      int x0, y0;
      range_origin(g, r, x0, y0);
      const float mean = (float)rmeta[r].sb / (float)NN;  // exact: NN is a power of two
      float scale = range_scale(thr[r]);
      if (range_allpass(thr[r])) scale = rsqrtf((float)rmeta[r].var / (float)NN + 1.0f);
      const unsigned char* base = img + (long long)y0 * g.W + x0;
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        const int j = kc * 8 + h;
        if (j < NN) {
          const int jr = j / n, jc = j % n;
          const int a = swap ? jc : jr, b = swap ? jr : jc;
          const int ir = f0 ? m - a : a, ic = f1 ? m - b : b;  // i with perm_s(i) = j
          const float v = ((float)base[(long long)ir * g.W + ic] - mean) * scale;
          w[h >> 1] |= (uint32_t)__half_as_ushort(__float2half_rn(v)) << (16 * (h & 1));
        }
      }
    }
    *reinterpret_cast<uint4*>(sR + (row >> 3) * K * 16 + kc * 128 + (row & 7) * 16) =
        make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// After the level's padded thresholds: one bit mask per 32-range m-tile of its ranges without a
// usable bar (range_allpass), written by range_op_kernel, read once per scan segment.
__host__ __device__ __forceinline__ uint32_t* scan_allpass_masks(float* thr, const Geometry& g) {
  return reinterpret_cast<uint32_t*>(thr + (size_t)((g.R + kScanRanges - 1) / kScanRanges) * kScanRanges);
}
__host__ __device__ __forceinline__ const uint32_t* scan_allpass_masks(const float* thr, const Geometry& g) {
  return reinterpret_cast<const uint32_t*>(thr + (size_t)((g.R + kScanRanges - 1) / kScanRanges) * kScanRanges);
}

// Per-range scan thresholds of a level (scan_threshold against the range's current bar);
// padded to whole m-tiles.  Invalid and shadow ranges get +1e30 (never survive), flags & 1
// (exhaustive debug mode) -1 (everything survives).
__device__ __forceinline__ float range_threshold(const Geometry& g, const RangeMeta* __restrict__ rmeta,
                                                 const unsigned long long* __restrict__ gbest, int r,
                                                 bool f16acc = false) {
  float t = 1e30f;
  if (r < g.R) {
    const RangeMeta rm = rmeta[r];
    if (!rm.shadow)
      t = (g.flags & 1) ? -1.f
                        : scan_threshold((double)rm.var / (double)g.N, load_bar(gbest, r), g.N, g.K, f16acc);
  }
  return t;
}

__global__ void threshold_kernel(Geometry g, const RangeMeta* __restrict__ rmeta,
                                 const unsigned long long* __restrict__ gbest, float* __restrict__ thr, int padded) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= padded) return;
  thr[r] = range_threshold(g, rmeta, gbest, r);
}

// Range operands of every m-tile, built per level into global memory (one CTA per m-tile,
// r_bytes each) so the scan loads them with one bulk copy per segment.
// The level's per-range thresholds are computed here too (each CTA for its m-tile's 32
// ranges, the blockIdx.y == 0 CTA writes them out for the scan epilogue), one launch per level.
// It also resets the level's pending-residual counter and, for the full level, the record
// self-check counter (instead of separate memsets).
template <int NN>
__global__ void __launch_bounds__(256)
range_op_kernel(const unsigned char* __restrict__ img, Geometry g, const RangeMeta* __restrict__ rmeta,
                const unsigned long long* __restrict__ gbest, float* __restrict__ thr,
                unsigned char* __restrict__ ropnd, unsigned long long* __restrict__ pend_count, int full_level,
                unsigned long long* __restrict__ selfcheck) {
  __shared__ float s_thr[kScanRanges];
  if (threadIdx.x < kScanRanges) {
    const int r = blockIdx.x * kScanRanges + threadIdx.x;
    const float t = range_threshold(g, rmeta, gbest, r, full_level && scan_f16acc(g));
    s_thr[threadIdx.x] = t;
    if (blockIdx.y == 0) thr[r] = t;
    // the m-tile's ranges without a usable bar as one bit mask (the scan epilogue's allpass)
    const unsigned ap = __ballot_sync(0xffffffffu, range_allpass(t));
    if (blockIdx.y == 0 && threadIdx.x == 0) scan_allpass_masks(thr, g)[blockIdx.x] = ap;
  }
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
    *pend_count = 0;
    if (selfcheck) *selfcheck = 0;
  }
  __syncthreads();
  // blockIdx.y splits the m-tile's 256 x K/8 chunks over several CTAs
  const int per = kScanRows * (g.K / 8) / gridDim.y;
  unsigned char* dst = ropnd + (long long)blockIdx.x * kScanRows * g.K * 2;
  const float* t = s_thr - blockIdx.x * kScanRanges;
  if constexpr (NN == 0)
    build_ranges(dst, img, g, rmeta, t, blockIdx.x, blockIdx.y * per + threadIdx.x, blockDim.x, blockIdx.y * per + per);
  else
    build_ranges_n<NN>(dst, img, g, rmeta, t, blockIdx.x, blockIdx.y * per + threadIdx.x, blockDim.x,
                       blockIdx.y * per + per);
}

// range_op_kernel for the first scan level of an encode that starts without a bar (no seed),
// riding in the pool launch: every range is allpass (scan_threshold against +inf is -1) or
// shadow / padding (1e30), so the level's operands only need the range's own sums, computed
// here from its pixels as the range pass does (RangeMeta is written by other blocks of the same
// launch).  One block per m-tile, all K/8 chunks.
__device__ void range_op_first_level(const unsigned char* __restrict__ img, const Geometry& g, const PrepAux& a,
                                     int mt) {
  __shared__ float s_thr[kScanRanges];
  __shared__ RangeMeta s_rm[kScanRanges];
  if (threadIdx.x < kScanRanges) {
    const int r = mt * kScanRanges + threadIdx.x;
    float t = 1e30f;
    RangeMeta rm{0, 1, 0};
    if (r < g.R) {
      int x0, y0;
      range_origin(g, r, x0, y0);
      long long sb = 0, sbb = 0;
      for (int i = 0; i < g.n; ++i) {
        const unsigned char* row = img + (long long)(y0 + i) * g.W + x0;
        for (int j = 0; j < g.n; ++j) {
          const int v = row[j];
          sb += v;
          sbb += v * v;
        }
      }
      const long long var = (long long)g.N * sbb - sb * sb;
      rm = RangeMeta{(int)sb, (double)var <= g.shadow_eps, var};
      if (!rm.shadow) t = -1.f;  // range_threshold with the bar at +inf (and the flags & 1 mode)
    }
    s_rm[threadIdx.x] = rm;
    s_thr[threadIdx.x] = t;
    a.thr[r] = t;
    const unsigned ap = __ballot_sync(0xffffffffu, range_allpass(t));
    if (threadIdx.x == 0) scan_allpass_masks(a.thr, g)[mt] = ap;
  }
  if (mt == 0 && threadIdx.x == 0) *a.pend_count = 0;
  __syncthreads();
  unsigned char* dst = a.ropnd + (long long)mt * kScanRows * g.K * 2;
  const float* t = s_thr - mt * kScanRanges;
  const RangeMeta* rm = s_rm - mt * kScanRanges;
  const int chunks = kScanRows * (g.K / 8);
  if (g.N == 4 && g.K == 16)
    build_ranges_n<4>(dst, img, g, rm, t, mt, threadIdx.x, blockDim.x, chunks);
  else if (g.N == 16 && g.K == 16)
    build_ranges_n<16>(dst, img, g, rm, t, mt, threadIdx.x, blockDim.x, chunks);
  else if (g.N == 64 && g.K == 64)
    build_ranges_n<64>(dst, img, g, rm, t, mt, threadIdx.x, blockDim.x, chunks);
  else
    build_ranges(dst, img, g, rm, t, mt, threadIdx.x, blockDim.x, chunks);
}

// Survivor appender of one warp: entries go straight to the CTA's list partition, into
// 64-entry chunks the warp reserves with one 32-bit shared-memory atomic.  Slots a warp
// leaves unused at a chunk switch or at exit hold kSentinel (skipped by the consumers);
// entries past the partition size are dropped (the reserved count still reports them).
constexpr uint32_t kSentinel = 0xFFFFFFFFu;
constexpr uint32_t kChunk = 64;

struct WarpAppender {
  SurvEntry* list;
  unsigned* count;   // CTA's reserved slots (shared memory)
  uint32_t cap;      // partition size
  uint32_t base;     // next slot of the warp's chunk
  uint32_t left;     // slots left in it

  __device__ __forceinline__ void put(SurvEntry e, uint32_t pos) {
    if (pos < cap) list[pos] = e;
  }
  // Pad the current chunk with sentinels (lanes of the warp cooperatively).
  __device__ __forceinline__ void close() {
    const uint32_t lane = threadIdx.x & 31;
    for (uint32_t k = lane; k < left; k += 32) put(make_uint2(kSentinel, kSentinel), base + k);
    left = 0;
  }
  // Appends (rowbase + b, d) for every set bit b of this lane's mask.
  __device__ __forceinline__ void bits(uint32_t mask, uint32_t rowbase, uint32_t d) {
    const uint32_t lane = threadIdx.x & 31, lt = (1u << lane) - 1u;
    while (true) {
      const bool has = mask != 0;
      const uint32_t bal = __ballot_sync(0xffffffffu, has);
      if (!bal) break;
      const uint32_t n = __popc(bal);
      if (n > left) {
        close();
        uint32_t nb = 0;
        if (lane == 0) nb = atomicAdd(count, kChunk);
        base = __shfl_sync(0xffffffffu, nb, 0);
        left = kChunk;
      }
      if (has) {
        const int b = __ffs(mask) - 1;
        mask &= mask - 1;
        put(make_uint2(rowbase + (uint32_t)b, d), base + __popc(bal & lt));
      }
      base += n;
      left -= n;
    }
  }
  // Appends (rowid, d0 + b) for every set bit b of this lane's column mask.
  __device__ __forceinline__ void cols(uint32_t mask, uint32_t rowid, uint32_t d0) {
    const uint32_t lane = threadIdx.x & 31, lt = (1u << lane) - 1u;
    while (true) {
      const bool has = mask != 0;
      const uint32_t bal = __ballot_sync(0xffffffffu, has);
      if (!bal) break;
      const uint32_t n = __popc(bal);
      if (n > left) {
        close();
        uint32_t nb = 0;
        if (lane == 0) nb = atomicAdd(count, kChunk);
        base = __shfl_sync(0xffffffffu, nb, 0);
        left = kChunk;
      }
      if (has) {
        const int b = __ffs(mask) - 1;
        mask &= mask - 1;
        put(make_uint2(rowid, d0 + (uint32_t)b), base + __popc(bal & lt));
      }
      base += n;
      left -= n;
    }
  }
};

// ---- fused evaluation: producer side ----
// One lane publishes chunk `id` (the warp's writes to it fenced first by the caller).
__device__ __forceinline__ void ring_publish(EvalRing* rg, uint32_t id) {
  const unsigned t = atomicAdd(&rg->tail, 1u);
  volatile uint32_t* seq = rg->seq;
  while (seq[t % kRing] != t) __nanosleep(64);  // full: wait for the consumer of ticket t - kRing
  reinterpret_cast<volatile uint32_t*>(rg->ids)[t % kRing] = id;
  __threadfence_block();
  seq[t % kRing] = t + 1;
}

// Warp-uniform: publish the warp's finished chunk `cur` (no-op when none / not fused).
__device__ __forceinline__ void publish_chunk(EvalRing* rg, uint32_t cur) {
  if (!rg || cur == kSentinel) return;
  __threadfence_block();
  __syncwarp();
  if ((threadIdx.x & 31) == 0) ring_publish(rg, cur);
  __syncwarp();
}

// Mask records: the scan epilogue writes one record per (warp, tile, range) with a hit: the
// range's encoded index r * 8, the pool index of the warp's first domain and, per lane (one
// domain each), the 8-bit mask of its isometry columns above the threshold.  One 8-byte
// header store and one coalesced 32-byte store per record instead of a ballot loop per
// survivor; expand_kernel turns the records into SurvEntry lists for the evaluation.
struct MaskRec {
  uint32_t r8;      // r * 8 (kSentinel: unused slot)
  uint32_t d0;      // pool index of lane 0's domain
  uint8_t m[32];    // lane l: isometry mask of domain d0 + l
};
constexpr uint32_t kRecChunk = 16;
#ifndef FIC_REC_GROUP
#define FIC_REC_GROUP 1  // full-level fp16 epilogue: one record reservation per tile (0: per record)
#endif
static_assert((kRecChunk & (kRecChunk - 1)) == 0, "record chunks: a power of two");
static_assert(kEpiRanges <= (int)kRecChunk, "one tile's records of a warp fit one chunk");

struct WarpRecAppender {
  MaskRec* recs;
  unsigned* count;   // CTA's reserved record slots (shared memory)
  uint32_t cap;      // partition size (records)
  uint32_t base;
  uint32_t left;
  uint32_t cur;      // first record of the warp's current chunk (kSentinel: none)
  EvalRing* ring;    // fused scan: finished chunks are published to the consumers
  MaskRec* next = nullptr;  // record `base` (valid while base < cap): advanced by one per put,
                            // so a put is two stores and no 64-bit index arithmetic
  MaskRec* trash = nullptr;  // this CTA's scratch chunk past every partition (group() of an
                             // overflowed partition: the stores need no branch)

  // Warp-uniform: every lane passes its mask (0 for none).
  __device__ __forceinline__ void put(uint32_t bits, uint32_t r8, uint32_t d0) {
    const uint32_t lane = threadIdx.x & 31;
    if (left == 0) {
      if (cur < cap) publish_chunk(ring, cur);
      uint32_t nb = 0;
      if (lane == 0) nb = atomicAdd(count, kRecChunk);
      base = __shfl_sync(0xffffffffu, nb, 0);
      cur = base;
      left = kRecChunk;
      next = recs + base;
    }
    if (base < cap) {
      if (lane == 0) *reinterpret_cast<uint2*>(next) = make_uint2(r8, d0);
      next->m[lane] = (uint8_t)bits;
    }
    ++next;
    ++base;
    --left;
  }
  // Room for `nh` (<= kRecChunk) more records of one tile in the warp's chunk, written by the
  // caller at the returned record and the nh - 1 after it (the chunk lies wholly inside the
  // partition, whose size is a multiple of kRecChunk, or the scratch chunk is returned); a chunk
  // too short for the group is padded with sentinels and a new one reserved.  Separate scan only (a fused scan publishes chunks to its consumers as they
  // fill).  Returns the group's first record.
  __device__ __forceinline__ MaskRec* group(uint32_t nh) {
    if (nh > left) {
      const uint32_t lane = threadIdx.x & 31;
      if (lane < left && base + lane < cap) next[lane].r8 = kSentinel;
      uint32_t nb = 0;
      if (lane == 0) nb = atomicAdd(count, kRecChunk);
      base = __shfl_sync(0xffffffffu, nb, 0);
      cur = base;
      left = kRecChunk;
      next = recs + base;
    }
    // an overflowed partition (the host re-runs the level) writes to the scratch chunk
    MaskRec* at = base < cap ? next : trash;
    next += nh;
    base += nh;
    left -= nh;
    return at;
  }
  __device__ __forceinline__ void close() {
    const uint32_t lane = threadIdx.x & 31;
    for (uint32_t k = lane; k < left; k += 32)
      if (base + k < cap) recs[base + k].r8 = kSentinel;
    left = 0;
    if (cur < cap) publish_chunk(ring, cur);
    cur = kSentinel;
  }
};

// Lexicographic minimum of (residual, domain * 8 + isometry) per range: one 128-bit CAS loop on
// (IEEE bits of the residual, candidate index) — non-negative doubles order like their bits.
__device__ __forceinline__ void win_min(unsigned __int128* w, double R, uint32_t idx) {
  const unsigned __int128 key = ((unsigned __int128)(unsigned long long)__double_as_longlong(R) << 64) | idx;
  const volatile unsigned long long* h = reinterpret_cast<const volatile unsigned long long*>(w);
  unsigned __int128 old = ((unsigned __int128)h[1] << 64) | h[0];
  while (key < old) {
    const unsigned __int128 prev = atomicCAS(w, old, key);
    if (prev == old) break;
    old = prev;
  }
}

// Sparse levels: a warp's 32-slot chunks of direct entries in its CTA's list partition.
struct EntryChunks {
  SurvEntry* list;
  unsigned* count;
  uint32_t cap, base, left, cur;
  EvalRing* ring;
  // Room for `need` more entries: pads and publishes the current chunk if it is too short.
  __device__ __forceinline__ void reserve(uint32_t need) {
    if (left >= need) return;
    const uint32_t lane = threadIdx.x & 31;
    for (uint32_t q = lane; q < left; q += 32)
      if (base + q < cap) list[base + q] = make_uint2(kSentinel, kSentinel);
    if (cur < cap) publish_chunk(ring, kChunkEntries | cur);
    uint32_t nb = 0;
    if (lane == 0) nb = atomicAdd(count, 32u);
    base = __shfl_sync(0xffffffffu, nb, 0);
    cur = base;
    left = 32;
  }
  __device__ __forceinline__ void close() {
    const uint32_t lane = threadIdx.x & 31;
    for (uint32_t q = lane; q < left; q += 32)
      if (base + q < cap) list[base + q] = make_uint2(kSentinel, kSentinel);
    left = 0;
    if (cur < cap) publish_chunk(ring, kChunkEntries | cur);
    cur = kSentinel;
  }
};

// ---- fused evaluation: consumer side ----

// One lane's survivor, evaluated exactly (eval_kernel's body with the residual inline).
template <int NN>
__device__ __forceinline__ void eval_entry(const Geometry& g, const EvalCtx& c, uint2 en) {
  if (en.x == kSentinel) return;
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  const int r = (int)(en.x >> 3), s = (int)(en.x & 7), d = (int)(en.y & 0x7FFFFFFFu);
  const DomainMetaI mi = c.meta_i[d];
  const RangeMeta rm = c.rmeta[r];
  const double bar = load_bar(c.gbest, r);
  int x0, y0;
  range_origin(g, r, x0, y0);
  uint32_t qw[NN / 2], bpk[NN / 4];
  load_q8_row<NN>(c.qpool, d, s, qw);
  load_range_words<NN>(c.img, g, x0, y0, bpk);
  if (mi.den < 0) return;  // flat code blocks are never candidates (encoder.cpp:223-229)
  unsigned qs = 0, qo = 0;
  const double R = eval_fast<NN>(g, qw, bpk, rm.sb, (double)rm.var / (double)NN, mi.sq, mi.den, bar,
                                 !(g.flags & 2), false, c.tab, c.qpool, c.img, d, s, x0, y0, qs, qo);
  if (R < inf) {
    publish_best(c.gbest, r, R);
    win_min(c.win + r, R, (uint32_t)d * 8u + (uint32_t)s);
  }
}

// Consumer loop of one warp: takes published chunks until every producer is done and the
// queue is empty.  `buf`: this warp's kEvalBuf-entry staging buffer (shared memory).
template <int NN>
__device__ void consume(const Geometry& g, const EvalCtx& c, EvalRing* rg, uint2* buf, const MaskRec* recs,
                        uint32_t rcap, const SurvEntry* elist, uint32_t ecap, unsigned producers) {
  const uint32_t lane = threadIdx.x & 31, lt = (1u << lane) - 1u;
  uint32_t nb = 0;        // warp-uniform: entries staged in buf
  unsigned taken = 0;     // entries this warp evaluated
  auto drain = [&]() {    // evaluate buf[0..31], keep the rest
    eval_entry<NN>(g, c, buf[lane]);
    __syncwarp();
    uint2 mv = make_uint2(0, 0);
    if (lane + 32 < nb) mv = buf[32 + lane];
    __syncwarp();
    if (lane + 32 < nb) buf[lane] = mv;
    __syncwarp();
    nb -= 32;
  };
  auto append = [&](bool has, uint2 e) {  // warp-uniform call; nb < 32 on entry
    const uint32_t bal = __ballot_sync(0xffffffffu, has);
    if (has) buf[nb + __popc(bal & lt)] = e;
    nb += __popc(bal);
    taken += __popc(bal);
    __syncwarp();
    if (nb >= 32) drain();
  };
  volatile uint32_t* seq = rg->seq;
  volatile unsigned* vdone = &rg->done;
  volatile unsigned* vtail = &rg->tail;
  while (true) {
    uint32_t id = kRingEmpty;
    if (lane == 0) {
      const unsigned t = atomicAdd(&rg->head, 1u);
      while (true) {
        if (seq[t % kRing] == t + 1) {
          id = reinterpret_cast<volatile uint32_t*>(rg->ids)[t % kRing];
          __threadfence_block();
          seq[t % kRing] = t + kRing;  // free for ticket t + kRing
          break;
        }
        if (*vdone == producers && t >= *vtail) break;  // every chunk published and taken
        __nanosleep(128);
      }
    }
    id = __shfl_sync(0xffffffffu, id, 0);
    if (id == kRingEmpty) break;
    __syncwarp();
    __threadfence_block();
    if (id & kChunkEntries) {
      const uint32_t pos = (id & ~kChunkEntries) + lane;
      uint2 e = make_uint2(kSentinel, kSentinel);
      if (pos < ecap) e = __ldcg(elist + pos);
      append(e.x != kSentinel, e);
    } else {
      // the chunk's 16 headers (lanes 0-15) and every record's mask byte of this lane, all
      // loaded up front (one L2 round trip), then the records in order from registers
      uint2 hq = make_uint2(kSentinel, 0);
      if (lane < kRecChunk && id + lane < rcap) hq = __ldcg(reinterpret_cast<const uint2*>(recs + id + lane));
      uint32_t mk[kRecChunk];
#pragma unroll
      for (uint32_t q = 0; q < kRecChunk; ++q) mk[q] = id + q < rcap ? (uint32_t)__ldcg(recs[id + q].m + lane) : 0u;
#pragma unroll 1
      for (uint32_t q = 0; q < kRecChunk; ++q) {
        uint2 h;
        h.x = __shfl_sync(0xffffffffu, hq.x, q);
        h.y = __shfl_sync(0xffffffffu, hq.y, q);
        if (h.x == kSentinel) continue;
        uint32_t m = 0;
#pragma unroll
        for (uint32_t k = 0; k < kRecChunk; ++k)
          if (k == q) m = mk[k];
        while (__any_sync(0xffffffffu, m != 0)) {
          const bool has = m != 0;
          const uint32_t b = has ? (uint32_t)(__ffs(m) - 1) : 0u;
          m &= m - 1;
          append(has, make_uint2(h.x + b, h.y + lane));
        }
      }
    }
  }
  if (nb > 0) eval_entry<NN>(g, c, lane < nb ? buf[lane] : make_uint2(kSentinel, kSentinel));
  if (lane == 0) atomicAdd(&rg->entries, taken);
}

__device__ __forceinline__ float absmax8(const uint32_t* v) {
  const float* f = reinterpret_cast<const float*>(v);
  return fmaxf(fmaxf(fmaxf(fmaxf(fabsf(f[0]), fabsf(f[1])), fmaxf(fabsf(f[2]), fabsf(f[3]))),
                     fmaxf(fabsf(f[4]), fabsf(f[5]))),
               fmaxf(fabsf(f[6]), fabsf(f[7])));
}

// Persistent scan over the segments of ScanLevel (see there); 18 warps:
//   warp 0        lane 0: bulk-copy producer, 128-domain pool tiles (contiguous 128*K*2 bytes) ->
//                 smem ring; lane 1: range-operand loader, the segment's 256 x K operand (built
//                 per level by range_op_kernel) -> one of two smem buffers
//   warp 1        TMEM allocation; MMA issuer (the whole warp runs the loop, an elected lane
//                 issues): K/16 x tcgen05.mma M=128 (domains) x N=256 (32 ranges x 8
//                 isometries) x K=16 per tile into one of two 256-column TMEM accumulators
//   warps 2-17    epilogue: 16 warps (lane quarter x column part); for every tile a thread owns
//                 one domain (TMEM lane) and kEpiRanges ranges x 8 isometries (kEpiCols columns,
//                 scaled so the pruning test is |X~/T_r| > 1 for every column), tests each
//                 range's 8-isometry |max| against 1 and records the columns above it (MODE)
// MODE: 0 full level, 1 full level with the whole-tile vote (lv.coarse), 2 sparse level with
// the per-range test before the selection (lv.select == 1), 3 sparse level selecting from the
// packed maxima of every range (lv.select == 2: most ranges hit in most tiles), 4 sparse level
// keeping each lane's best per range over the whole segment (lv.select == 3: short levels of
// small pools, one segment per m-tile); 5, 6, 7 and 9: modes 0, 1, 2 and 4 with an fp16
// accumulator (full level: scan_f16acc; sparse level: scan_f16sel).  One instantiation per mode keeps each epilogue's registers to its own path.
// EV: 0 = survivors to the global list (expand / eval / residual / winner kernels follow);
// NN (4, 16, 64) = fused: kEvalWarps consumer warps evaluate them in this kernel (EvalCtx).
template <int MODE, int EV>
__global__ void __launch_bounds__(EV ? kFusedThreads : kScanThreads, EV ? 1 : kScanCtas)
scan_kernel(const unsigned char* __restrict__ img, Geometry g, ScanLevel lv, const __half* __restrict__ upool,
            const RangeMeta* __restrict__ rmeta, const unsigned char* __restrict__ ropnd,
            const float* __restrict__ thr, MaskRec* __restrict__ recs_all,
            unsigned long long* __restrict__ rcounts, unsigned long long rcap,
            SurvEntry* __restrict__ list_all, unsigned long long cap,
            unsigned long long* __restrict__ counts, EvalCtx ev) {
  extern __shared__ __align__(1024) unsigned char smem[];
  constexpr bool F16 = MODE >= 5;            // fp16 accumulator (full level only)
  constexpr int MB = F16 ? MODE - 5 : MODE;  // the epilogue mode proper
  constexpr bool FUSED = EV != 0;
  const ScanSmem L = scan_smem_layout(g.K, FUSED);
  const int K = g.K;
  unsigned char* sR = smem + L.r_off;
  unsigned char* sP = smem + L.p_off;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + L.bar_off);
  uint64_t* empty_bar = full_bar + kScanMaxStages;
  uint64_t* tfull_bar = empty_bar + kScanMaxStages;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* rfull_bar = tempty_bar + 2;
  uint64_t* rempty_bar = rfull_bar + 2;
  uint32_t* tmem_base_smem = reinterpret_cast<uint32_t*>(rempty_bar + 2);
  unsigned* count = reinterpret_cast<unsigned*>(smem + L.bar_off + 448);  // CTA's reserved record slots
  unsigned* ecount = count + 1;  // CTA's reserved entry slots (sparse levels)
  MaskRec* recs = recs_all + (unsigned long long)blockIdx.x * rcap;  // this CTA's partition of `rcap` records
  EvalRing* ring = FUSED ? reinterpret_cast<EvalRing*>(smem + L.wbuf_off) : nullptr;
  uint2* ebufs = FUSED ? reinterpret_cast<uint2*>(smem + L.wbuf_off + sizeof(EvalRing)) : nullptr;
  SurvEntry* elist_cta = list_all + (unsigned long long)blockIdx.x * cap;  // sparse levels: direct entries

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x, cta = blockIdx.x;
  const int nseg = seg_count(lv, cta, G);
  const int stages = (int)L.stages;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < stages; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull_bar[b], 1);
      ptx::mbar_init(&tempty_bar[b], kScanEpiWarps);  // every epilogue warp reads every tile
      ptx::mbar_init(&rfull_bar[b], 1);    // arrive.expect_tx of the range-operand loader
      ptx::mbar_init(&rempty_bar[b], 1);   // tcgen05.commit after a segment's last MMA
    }
    ptx::fence_mbar_init();
    *count = 0;
    *ecount = 0;
  }
  if constexpr (FUSED) {
    for (uint32_t k = threadIdx.x; k < kRing; k += blockDim.x) ring->seq[k] = k;
    if (threadIdx.x == 0) ring->head = ring->tail = ring->done = ring->entries = 0;
  }
  if (warp == 1) ptx::tmem_alloc<kScanTmemCols>(tmem_base_smem);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_base_smem;

  if (warp == 0) {
    // ================= producer (lane 0) and range-operand loader (lane 1) =================
    if (lane == 1) {
      for (int sg = 0; sg < nseg; ++sg) {
        if (sg >= 2) ptx::mbar_wait(&rempty_bar[sg & 1], ((sg >> 1) - 1) & 1);
        ptx::mbar_arrive_expect_tx(&rfull_bar[sg & 1], L.r_bytes);
        ptx::bulk_g2s(sR + (sg & 1) * L.r_bytes, ropnd + (long long)seg_at(lv, cta, G, sg).m * L.r_bytes, L.r_bytes,
                      &rfull_bar[sg & 1]);
      }
    }
    if (lane == 0) {
      int s = 0;
      uint32_t ring_phase = 0;
      for (int sg = 0; sg < nseg; ++sg) {
        const Segment S = seg_at(lv, cta, G, sg);
        // the segment's slice pool (batched encodes: slice b's domains start at b * Dt)
        const unsigned char* src = reinterpret_cast<const unsigned char*>(upool) +
                                   (long long)range_slice(g, S.m * kScanRanges) * g.Dt * K * 2;
        const long long step_bytes = (long long)lv.stride * L.p_bytes;
        for (int j = S.j0; j < S.j1; ++j) {
          ptx::mbar_wait(&empty_bar[s], ring_phase ^ 1u);
          ptx::mbar_arrive_expect_tx(&full_bar[s], L.p_bytes);
          ptx::bulk_g2s(sP + s * L.p_bytes, src + (long long)j * step_bytes, L.p_bytes, &full_bar[s]);
          if (++s == stages) {
            s = 0;
            ring_phase ^= 1u;
          }
        }
      }
    }
    if constexpr (FUSED) {  // the producer warp joins the consumers once every tile is issued
      __syncwarp();
      consume<EV>(g, ev, ring, ebufs + (warp * kEvalBuf), recs, (uint32_t)rcap, elist_cta, (uint32_t)cap,
                  kScanEpiWarps);
    }
  } else if (warp == 1) {
    // ================= MMA issuer =================
    // The whole warp runs the loop (all its values warp-uniform); one elected lane issues the
    // MMAs and commits.  The issuing thread is on the scan's critical path.
    {
      const uint32_t idesc = F16 ? ptx::idesc_f16_f16(128, kScanRows) : ptx::idesc_f16_f32(128, kScanRows);
      const bool do_mma = !(kScanDebug && (g.flags & 16));  // debug: flags & 16 skips the MMAs
      // descriptors: the start address field (bits 0-13, 16-byte units) advances by 16 per
      // K=16 step (256 bytes) and by p_bytes/16 per ring stage; everything else is constant
      const uint64_t p_desc0 = ptx::smem_desc(ptx::smem_addr(sP), 128, K * 16);
      const uint32_t p_stage = L.p_bytes >> 4;
      int i = 0, s = 0;
      uint32_t ring_phase = 0;  // phase of full_bar[s] for the current pass over the ring
      for (int sg = 0; sg < nseg; ++sg) {
        const Segment S = seg_at(lv, cta, G, sg);
        ptx::mbar_wait(&rfull_bar[sg & 1], (sg >> 1) & 1);
        const uint64_t r_desc = ptx::smem_desc(ptx::smem_addr(sR + (sg & 1) * L.r_bytes), 128, K * 16);
        for (int j = S.j0; j < S.j1; ++j, ++i) {
          const int buf = kTBufs == 2 ? (i & 1) : 0;
          trace_stamp(g, i, 0);
          ptx::mbar_wait(&tempty_bar[buf], (kTBufs == 2 ? ((i >> 1) & 1) : (i & 1)) ^ 1);
          trace_stamp(g, i, 1);
          ptx::mbar_wait(&full_bar[s], ring_phase);
          trace_stamp(g, i, 2);
          ptx::tc_fence_after();
          if (ptx::elect_one()) {
            if (do_mma) {
              const uint64_t ad0 = p_desc0 + (uint64_t)(s * p_stage);
              const uint32_t d_tmem = tmem_base + buf * kScanRows;
              ptx::mma_f16_ss(d_tmem, ad0, r_desc, idesc, 0u);
              if (K == 64) {  // n = 8: four K=16 steps, unrolled (K is 16 otherwise)
                ptx::mma_f16_ss(d_tmem, ad0 + 16u, r_desc + 16u, idesc, 1u);
                ptx::mma_f16_ss(d_tmem, ad0 + 32u, r_desc + 32u, idesc, 1u);
                ptx::mma_f16_ss(d_tmem, ad0 + 48u, r_desc + 48u, idesc, 1u);
              }
            }
            ptx::tc_commit(&empty_bar[s]);
            ptx::tc_commit(&tfull_bar[buf]);
          }
          __syncwarp();
          if (++s == stages) {
            s = 0;
            ring_phase ^= 1u;
          }
        }
        if (ptx::elect_one()) ptx::tc_commit(&rempty_bar[sg & 1]);
        __syncwarp();
      }
    }
    if constexpr (FUSED) {  // the MMA warp joins the consumers once every MMA is issued
      consume<EV>(g, ev, ring, ebufs + (warp * kEvalBuf), recs, (uint32_t)rcap, elist_cta, (uint32_t)cap,
                  kScanEpiWarps);
    }
  } else if (warp < 2 + kScanEpiWarps) {
    // ================= epilogue =================
    const int e = warp - 2;
    const int part0 = e >> 2;       // column part: ranges part*kEpiRanges .. +kEpiRanges-1 of the m-tile
    const int quarter = warp & 3;   // TMEM lane quarter: domains quarter*32 .. +31 of the tile
    // lv.rotate: the column part advances by one per tile, so the warps of a part with a hot
    // range (many hits) take turns instead of pacing every tile
    const bool rotate = MB != 4 && lv.rotate;
    WarpRecAppender app{recs, count, (uint32_t)rcap, 0u, 0u, kSentinel, ring};
    app.trash = recs_all + (unsigned long long)G * rcap + (unsigned long long)cta * kRecChunk;
    constexpr bool sel = MB >= 2;
    SurvEntry* elist = elist_cta;
    const uint32_t ecap = (uint32_t)cap;
    EntryChunks ech{elist, ecount, ecap, 0u, 0u, kSentinel, ring};
    const uint32_t tlane = tmem_base + ((uint32_t)(quarter * 32) << 16);
    // fp16 selection tags (7 - isometry in each half's low 3 bits) held in registers: with the
    // mask an immediate, (v & mask) | tag is ONE LOP3 (two immediates would take two); the
    // runtime zero keeps the compiler from folding them back into immediates
    const uint32_t t1 = 1u + ((uint32_t)lv.stride >> 30);  // 1 (strides < 2^30)
    const uint32_t tagr[4] = {0x00060007u * t1, 0x00040005u * t1, 0x00020003u * t1, 0x00000001u * t1};
    // (the fp32 selection's tags 7 - isometry likewise, for the hit ranges of sparse levels)
    uint32_t tagf[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) tagf[c] = (uint32_t)(7 - c) * t1;
    int i = 0;
    for (int sg = 0; sg < nseg; ++sg) {
      const Segment S = seg_at(lv, cta, G, sg);
      const int m0 = S.m * kScanRanges;  // the m-tile's first range (one slice per m-tile)
      const uint32_t dslice = (uint32_t)(range_slice(g, m0) * g.Dt);  // pool index of the slice's domain 0
      // ranges of the m-tile without a usable threshold (range_op_kernel's bit mask)
      const uint32_t allpass_all = __ldg(scan_allpass_masks(thr, g) + S.m);
      uint32_t allpass = (allpass_all >> (part0 * kEpiRanges)) & ((1u << kEpiRanges) - 1u);
      uint32_t rowbase = (uint32_t)(m0 + part0 * kEpiRanges) * 8u;  // this thread's ranges x 8
      uint32_t tcol = tlane + part0 * kEpiCols;
      // MODE 4: each lane's running best column per range over the segment's tiles, packed as
      // (|x| truncated to 7 mantissa bits | 7 - isometry | level tile index), flushed below
      uint32_t lbest[MB == 4 ? kEpiRanges : 1];
#pragma unroll
      for (int k = 0; k < (MB == 4 ? kEpiRanges : 1); ++k) lbest[k] = 0u;
      for (int j = S.j0; j < S.j1; ++j, ++i) {
        const int buf = kTBufs == 2 ? (i & 1) : 0;
        if (rotate) {
          const int part = (part0 + i) & (kEpiParts - 1);
          allpass = (allpass_all >> (part * kEpiRanges)) & ((1u << kEpiRanges) - 1u);
          rowbase = (uint32_t)(m0 + part * kEpiRanges) * 8u;
          tcol = tlane + part * kEpiCols;
        }
        if (lane == 0 && i > 0) trace_stamp(g, i - 1, 19 + e);  // done with the previous tile
        const uint32_t d = dslice + (uint32_t)(j * lv.stride * kScanTileDom + quarter * 32 + lane);
        ptx::mbar_wait_sleep(&tfull_bar[buf], kTBufs == 2 ? ((i >> 1) & 1) : (i & 1));
        ptx::tc_fence_after();
        if (kScanDebug && (g.flags & 128)) {  // debug: no TMEM reads at all (MMA + producer throughput)
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&tempty_bar[buf]);
          continue;
        }
        const uint32_t ta = tcol + buf * kScanRows;
        // fp32 accumulators at two CTAs per SM: kLoadCols = 32 columns (kCR ranges) per TMEM
        // load, the buffer released after the last chunk's load
        constexpr int kLoadCols = (F16 || kScanCtas == 1) ? kEpiCols : 32;
        constexpr int kChunks = F16 ? 1 : kEpiCols / kLoadCols;
        constexpr int kCR = kEpiRanges / kChunks;  // ranges per chunk
#pragma unroll
        for (int hc = 0; hc < kChunks; ++hc) {
        uint32_t v[F16 ? kEpiCols : kLoadCols];  // F16: the first kEpiCols / 2
        __syncwarp();
        if constexpr (F16) {
          if constexpr (kEpiCols == 64) ptx::tmem_ld_32x32b_x64_pack16(ta, v);  // register j: columns 2j, 2j + 1
          else ptx::tmem_ld_32x32b_x32_pack16(ta, v);
        } else {
#pragma unroll
          for (int c = 0; c < kLoadCols; c += 32) ptx::tmem_ld_32x32b_x32(ta + hc * kLoadCols + c, v + c);
        }
        ptx::tmem_ld_wait();
        if (hc == kChunks - 1) {
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            ptx::mbar_arrive(&tempty_bar[buf]);  // all columns read: release the buffer
            trace_stamp(g, i, 3 + e);
          }
        }
        if (kScanDebug && (g.flags & 8)) continue;          // debug: skip the test
        const uint32_t ap = (allpass >> (hc * kCR)) & ((1u << kCR) - 1u);  // the chunk's ranges
        const uint32_t rb = rowbase + 8u * (uint32_t)(hc * kCR);
        if constexpr (F16) {
          // fp16 pairs: range k's 8 isometry columns are registers 4k .. 4k + 3; the |max| test
          // runs on half2 (3-input VHMNMX with |.| modifiers: four columns per instruction).
          // |x| > 1 on the bit patterns: (h & 0x7FFF) > 0x3C00 (no inf / NaN: scan_threshold)
          const __half2* h = reinterpret_cast<const __half2*>(v);
          const __half2 one2 = __float2half2_rn(1.0f);
          if constexpr (MB == 4) {
            // per-lane best per range over the segment: the isometry-tagged half2 |max| tree
            // (as the fp16 hit-first selection) and the tile index below it
            const uint32_t jtag = (uint32_t)j;  // < 8192 tiles (small pools only)
#pragma unroll
            for (int k = 0; k < kEpiRanges; ++k) {
              __half2 t[4];
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const uint32_t u = (v[4 * k + q] & 0x7FF87FF8u) | tagr[q];
                t[q] = *reinterpret_cast<const __half2*>(&u);
              }
              const __half2 m2 = __hmax2(__hmax2(__hmax2(t[0], t[1]), t[2]), t[3]);
              const uint32_t m = __half_as_ushort(__hmax(__low2half(m2), __high2half(m2)));
              lbest[k] = max(lbest[k], (m << 16) | jtag);
            }
            continue;
          }
          // per range: one 3-input and one 2-input half2 |max|
          __half2 mxr[kEpiRanges];
#pragma unroll
          for (int k = 0; k < kEpiRanges; ++k)
            mxr[k] = __hmax2(__hmax2(__hmax2(__habs2(h[4 * k]), __habs2(h[4 * k + 1])), __habs2(h[4 * k + 2])),
                             __habs2(h[4 * k + 3]));
          if (MB == 1 && !allpass) {
            // whole-tile vote on the ranges' maxima (a 3-input tree: kEpiRanges / 2 more
            // instructions); the per-range compares only for tiles where some lane hits
            __half2 t[kEpiRanges];
#pragma unroll
            for (int k = 0; k < kEpiRanges; ++k) t[k] = mxr[k];
#pragma unroll
            for (int w = kEpiRanges; w > 1; w = (w + 1) / 2) {
#pragma unroll
              for (int k = 0; k < w / 2; ++k) t[k] = __hmax2(t[2 * k], t[2 * k + 1]);
              if (w & 1) t[w / 2] = t[w - 1];
            }
            if (!__any_sync(0xffffffffu, __hgt2_mask(t[0], one2) != 0u)) continue;
          }
          // per range one half2 compare (a 0xFFFF mask per half) and one masked OR; both halves
          // folded once at the end
          uint32_t g2 = 0u;
#pragma unroll
          for (int k = 0; k < kEpiRanges; ++k) g2 |= __hgt2_mask(mxr[k], one2) & (0x00010001u << k);
          const uint32_t gmask = ((g2 | (g2 >> 16)) & ((1u << kEpiRanges) - 1u)) | allpass;
          const uint32_t groups = __reduce_or_sync(0xffffffffu, gmask);
          if constexpr (MB == 2) {
            // sparse level (it only lowers the bar, so fp16 accuracy is enough): per hit range the
            // warp's best column.  Each half's low 3 mantissa bits are replaced by 7 - isometry
            // (one LOP3 per register; the magnitude order is kept to 2^-7), so the half2 |max|
            // tree yields the best column AND its isometry; key = that half << 5 | 31 - lane,
            // one warp max per range, one chunk reservation per tile, lane k writes range k's
            // entry (as the fp32 selection)
            // every range of `groups` has a lane above the threshold (or is allpass), so its warp
            // maximum is that range's entry: hits == groups, no per-lane threshold in the key (a
            // best |x| within 2^-7 of the threshold still yields an entry: a sparse level only
            // lowers the bar, any evaluated candidate is a valid one)
            if (!groups) continue;
            uint32_t wm[kEpiRanges];
#pragma unroll
            for (int k = 0; k < kEpiRanges; ++k) {
              uint32_t key = 0u;
              if ((groups >> k) & 1u) {
                __half2 t[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const uint32_t u = (v[4 * k + j] & 0x7FF87FF8u) | tagr[j];
                  t[j] = *reinterpret_cast<const __half2*>(&u);
                }
                const __half2 m2 = __hmax2(__hmax2(__hmax2(t[0], t[1]), t[2]), t[3]);
                const uint32_t m = __half_as_ushort(__hmax(__low2half(m2), __high2half(m2)));
                key = (m << 5) | (31u - (uint32_t)lane) | 0x200000u;  // nonzero even for lane 31 at |x| = 0
              }
              wm[k] = __reduce_max_sync(0xffffffffu, key);
            }
            const uint32_t hits = groups;
            uint32_t mine = 0u;
#pragma unroll
            for (int k = 0; k < kEpiRanges; ++k)
              if (lane == k) mine = (groups >> k) & 1u ? wm[k] : 0u;
            const uint32_t nh = (uint32_t)__popc(hits);
            ech.reserve(nh);
            if (mine != 0u) {
              const uint32_t pos = ech.base + (uint32_t)__popc(hits & ((1u << lane) - 1u));
              const uint32_t wl = 31u - (mine & 31u), ws = 7u - ((mine >> 5) & 7u);
              if (pos < ecap) elist[pos] = make_uint2(rowbase + 8u * (uint32_t)lane + ws, d - (uint32_t)lane + wl);
            }
            ech.base += nh;
            ech.left -= nh;
            continue;
          }
          if (groups) {
            // one slot reservation for the tile's records (no per-record chunk bookkeeping)
            constexpr bool kPut = FUSED || !FIC_REC_GROUP;
            MaskRec* rc = kPut ? nullptr : app.group((uint32_t)__popc(groups));
#pragma unroll
            for (int k = 0; k < kEpiRanges; ++k) {
              if ((groups >> k) & 1u) {
                // column c = 2j + half of register j: half2 compares give 0xFFFF masks, bit 2j of
                // the low half and bit 2j + 1 of the high half are kept, then folded; an allpass
                // range keeps every column (no branch: the low byte is what is stored)
                uint32_t x = 0u;
#pragma unroll
                for (int j = 0; j < 4; ++j) x |= __hgt2_mask(__habs2(h[4 * k + j]), one2) & (0x00020001u << (2 * j));
                const uint32_t bits = (x | (x >> 16) | (0u - ((allpass >> k) & 1u))) & 0xFFu;
                if constexpr (kPut) {
                  app.put(bits, rowbase + 8u * (uint32_t)k, d - (uint32_t)lane);
                } else {
                  if (lane == 0) *reinterpret_cast<uint2*>(rc) = make_uint2(rowbase + 8u * (uint32_t)k, d);
                  rc->m[lane] = (uint8_t)bits;
                  ++rc;
                }
              }
            }
          }
          continue;
        } else if constexpr (MB == 4) {
          // small pools, short sparse level: per lane and range keep the best column seen in the
          // segment (one per tile slot, like the warp's best per tile but without any cross-lane
          // work per tile); the threshold test is applied once, when the segment is flushed
          const uint32_t jtag = (uint32_t)j;  // < 8192 tiles (small pools only)
#pragma unroll
          for (int k = 0; k < kCR; ++k) {
            float m = 0.f;
#pragma unroll
            for (int c = 0; c < 8; ++c)
              m = fmaxf(m, __uint_as_float((v[8 * k + c] & 0x7FFF0000u) | ((uint32_t)(7 - c) << 13) | jtag));
            lbest[hc * kCR + k] = max(lbest[hc * kCR + k], __float_as_uint(m));
          }
          continue;
        }
        if constexpr (sel) {
          // sparse level: it only has to lower the bar, so of this warp's 32 domains x 8
          // isometries of each range only the column with the largest |X~| (the smallest
          // unconstrained bound R*) is evaluated, written straight to the entry list.  For the
          // ranges that hit, the isometry rides in the low 3 bits of the packed |x| (7 - s: ties
          // within 2^-20 go to the lower isometry, then the lower lane), so one max tree and one
          // warp max yield the winning lane and isometry.
          // MODE 3: packed maxima of every range up front (most ranges hit); MODE 2: plain
          // maxima for the hit test, packed ones only for the ranges that hit
          uint32_t pk[kCR];
          uint32_t gmask = ap;
#pragma unroll
          for (int k = 0; k < kCR; ++k) {
            if constexpr (MB == 3) {
              float m = 0.f;
#pragma unroll
              for (int c = 0; c < 8; ++c)
                m = fmaxf(m, __uint_as_float((v[8 * k + c] & 0x7FFFFFF8u) | tagf[c]));
              pk[k] = __float_as_uint(m);
              gmask |= (uint32_t)(m > 1.0f) << k;
            } else {
              const float* f = reinterpret_cast<const float*>(v + 8 * k);
              const float gm = fmaxf(fmaxf(fmaxf(fmaxf(fabsf(f[0]), fabsf(f[1])), fmaxf(fabsf(f[2]), fabsf(f[3]))),
                                           fmaxf(fabsf(f[4]), fabsf(f[5]))),
                                     fmaxf(fabsf(f[6]), fabsf(f[7])));
              gmask |= (uint32_t)(gm > 1.0f) << k;
            }
          }
          const uint32_t groups = __reduce_or_sync(0xffffffffu, gmask);
          if (!groups) continue;
          // one key per range, (|x| truncated to 15 mantissa bits | 7 - isometry | 31 - lane), so
          // one warp max yields the winning isometry AND lane; the hit ranges' maxima are
          // independent (issued back to back), then one chunk reservation covers all entries of
          // the tile and lane k writes range k's entry
          uint32_t wm[kCR];
#pragma unroll
          for (int k = 0; k < kCR; ++k) {
            uint32_t key = 0u;
            if ((groups >> k) & 1u) {
              float m = 0.f;
              if constexpr (MB == 3) {
                m = __uint_as_float(pk[k]);
              } else {
#pragma unroll
                for (int c = 0; c < 8; ++c)
                  m = fmaxf(m, __uint_as_float((v[8 * k + c] & 0x7FFFFFF8u) | tagf[c]));
              }
              // (hits == groups, as in the fp16 selection; bit 8 keeps the key nonzero)
              key = (__float_as_uint(m) & 0x7FFFFE00u) | 0x100u | ((__float_as_uint(m) & 7u) << 5) |
                    (31u - (uint32_t)lane);
            }
            wm[k] = __reduce_max_sync(0xffffffffu, key);
          }
          const uint32_t hits = groups;
          uint32_t mine = 0u;
#pragma unroll
          for (int k = 0; k < kCR; ++k)
            if (lane == k) mine = (groups >> k) & 1u ? wm[k] : 0u;
          const uint32_t nh = (uint32_t)__popc(hits);
          ech.reserve(nh);  // pads the rest of the chunk and takes a new one when it is short
          if (mine != 0u) {
            const uint32_t pos = ech.base + (uint32_t)__popc(hits & ((1u << lane) - 1u));
            const uint32_t wl = 31u - (mine & 31u), ws = 7u - ((mine >> 5) & 7u);
            if (pos < ecap) elist[pos] = make_uint2(rb + 8u * (uint32_t)lane + ws, d - (uint32_t)lane + wl);
          }
          ech.base += nh;
          ech.left -= nh;
          continue;
        }
        if (MB == 1 && !ap) {
          // large pools, hits in ~2% of warp-tiles: one |max| over all 64 columns (32 FMNMX3)
          // and a warp vote first; the per-range breakdown only for the rare tiles with a hit
          // four independent FMNMX3 chains (8 deep instead of 16: the test's latency, not its
          // instruction count, is what the MMA waits on)
          float m0 = 0.f, m1 = 0.f, m2 = 0.f, m3 = 0.f;
#pragma unroll
          for (int c = 0; c < kLoadCols; c += 8) {
            m0 = fmaxf(m0, fmaxf(fabsf(__uint_as_float(v[c])), fabsf(__uint_as_float(v[c + 1]))));
            m1 = fmaxf(m1, fmaxf(fabsf(__uint_as_float(v[c + 2])), fabsf(__uint_as_float(v[c + 3]))));
            m2 = fmaxf(m2, fmaxf(fabsf(__uint_as_float(v[c + 4])), fabsf(__uint_as_float(v[c + 5]))));
            m3 = fmaxf(m3, fmaxf(fabsf(__uint_as_float(v[c + 6])), fabsf(__uint_as_float(v[c + 7]))));
          }
          if (!__any_sync(0xffffffffu, fmaxf(fmaxf(m0, m1), fmaxf(m2, m3)) > 1.0f)) continue;
        }
        // |max| of each range's 8 isometry columns (4 FMNMX3 each); mask of ranges above 1
        uint32_t gmask = ap;
#pragma unroll
        for (int k = 0; k < kCR; ++k) {
          const float* f = reinterpret_cast<const float*>(v + 8 * k);
          const float gm = fmaxf(fmaxf(fmaxf(fmaxf(fabsf(f[0]), fabsf(f[1])), fmaxf(fabsf(f[2]), fabsf(f[3]))),
                                       fmaxf(fabsf(f[4]), fabsf(f[5]))),
                                 fmaxf(fabsf(f[6]), fabsf(f[7])));
          gmask |= (uint32_t)(gm > 1.0f) << k;
        }
        const uint32_t groups = __reduce_or_sync(0xffffffffu, gmask);
        if (lane == 0) trace_stamp(g, i, 35 + e);
        if (groups) {
          // ranges with a hit in some lane of the warp, one warp-uniform branch per range, so
          // only the hit ranges' column bits are formed (8 compares each)
#pragma unroll
          for (int k = 0; k < kCR; ++k) {
            if ((groups >> k) & 1u) {
              uint32_t bits = 0;
              if ((ap >> k) & 1u) {
                bits = 0xFFu;
              } else {
#pragma unroll
                for (int c = 0; c < 8; ++c) bits |= (uint32_t)(fabsf(__uint_as_float(v[8 * k + c])) > 1.0f) << c;
              }
              app.put(bits, rb + 8u * (uint32_t)k, d - (uint32_t)lane);
            }
          }
        }
        }  // chunk
      }
      if constexpr (MB == 4) {  // flush the segment's per-lane bests: one entry per lane group and range
        // lv.lanes_per_best consecutive lanes (1, 2, 4) share one entry: the group's largest key
        // (ties: the lowest lane) — fewer exact evaluations for a slightly weaker bar
#pragma unroll
        for (int k = 0; k < kEpiRanges; ++k) {
          const uint32_t b = lbest[k];
          bool win_lane = true;
          for (int o = 1; o < lv.lanes_per_best; o <<= 1) {
            const uint32_t ob = __shfl_xor_sync(0xffffffffu, b, o);
            const bool lower = (lane & o) == 0;
            if (ob > b || (ob == b && !lower)) win_lane = false;
          }
          // fp32 key: the float bits (|x| to 7 mantissa bits | 7 - isometry | tile); fp16 key:
          // (half |x| with 7 - isometry in its low 3 bits) << 16 | tile
          const bool above = F16 ? (b >> 16) > 0x3C07u : __uint_as_float(b) > 1.0f;
          const bool keep = win_lane && b != 0u && (above || ((allpass >> k) & 1u));
          const uint32_t bal = __ballot_sync(0xffffffffu, keep);
          if (!bal) continue;
          ech.reserve((uint32_t)__popc(bal));
          const uint32_t pos = ech.base + __popc(bal & ((1u << lane) - 1u));
          if (keep && pos < ecap) {
            const uint32_t jt = b & 0x1FFFu, s_iso = 7u - ((b >> (F16 ? 16 : 13)) & 7u);
            const uint32_t dd = dslice + (uint32_t)(jt * lv.stride * kScanTileDom + quarter * 32 + lane);
            elist[pos] = make_uint2(rowbase + 8u * (uint32_t)k + s_iso, dd);
          }
          ech.base += __popc(bal);
          ech.left -= __popc(bal);
        }
      }
    }
    // pad the warp's unused entry slots (sparse levels), publish the last chunks
    ech.close();
    app.close();
    if constexpr (FUSED) {
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        atomicAdd(&ring->done, 1u);
      }
      consume<EV>(g, ev, ring, ebufs + (warp * kEvalBuf), recs, (uint32_t)rcap, elist, ecap, kScanEpiWarps);
    }
  } else if constexpr (FUSED) {
    // ================= consumers (evaluation warps) =================
    consume<EV>(g, ev, ring, ebufs + (warp * kEvalBuf), recs, (uint32_t)rcap, elist_cta, (uint32_t)cap,
                kScanEpiWarps);
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    rcounts[blockIdx.x] = *count;
    if (FUSED && MB <= 1) {
      // full level, fused: the entries were evaluated here (none are stored); a record partition
      // that overflowed reports at least twice its record count so that the host re-runs the
      // level with a larger partition (as expand_kernel does)
      const unsigned long long ent = ring->entries;
      counts[blockIdx.x] = *count > rcap ? 2ull * *count : (ent < cap ? ent : cap);
    } else {
      counts[blockIdx.x] = *ecount;  // direct entries (sparse levels); expand_kernel adds the records' entries
    }
  }
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<kScanTmemCols>(tmem_base);
  }
}

// Mask records of partition c -> SurvEntry list partition c (counts[c] entries; entries past
// the partition size are dropped but counted, as with direct appends).  A record partition
// that overflowed reports at least twice its record count as the entry count, which makes
// the host re-run the level with lists large enough for it (records take half an entry
// partition's slot count).  One thread per record (its 32 mask bytes in registers), one warp
// prefix sum and one global atomic per 32 records.
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, uint32_t lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= (uint32_t)o) v += t;
  }
  return v;
}

__global__ void __launch_bounds__(256)
expand_kernel(const MaskRec* __restrict__ recs_all, const unsigned long long* __restrict__ rcounts,
              unsigned long long rcap, SurvEntry* __restrict__ list_all, unsigned long long* __restrict__ counts,
              unsigned long long part, int per) {
  const int c = blockIdx.x / per, sub = blockIdx.x % per;
  const uint32_t lane = threadIdx.x & 31;
  const unsigned long long nr = rcounts[c];
  if (nr > rcap) {
    if (sub == 0 && threadIdx.x == 0) atomicAdd(counts + c, 2ull * nr);
    return;
  }
  const MaskRec* recs = recs_all + (unsigned long long)c * rcap;
  SurvEntry* list = list_all + (unsigned long long)c * part;
  const unsigned long long wpb = blockDim.x / 32;
  const unsigned long long nw = (unsigned long long)per * wpb;
  for (unsigned long long i0 = ((unsigned long long)sub * wpb + threadIdx.x / 32) * 32; i0 < nr; i0 += nw * 32) {
    const unsigned long long i = i0 + lane;
    uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    uint2 h = make_uint2(kSentinel, 0);
    if (i < nr) {
      const uint2* rp = reinterpret_cast<const uint2*>(recs + i);  // records are 8-byte aligned
      h = rp[0];
#pragma unroll
      for (int q = 0; q < 4; ++q) {  // loaded with the header (no dependent round trip)
        const uint2 t = rp[1 + q];
        w[2 * q] = t.x;
        w[2 * q + 1] = t.y;
      }
      if (h.x == kSentinel) {
#pragma unroll
        for (int q = 0; q < 8; ++q) w[q] = 0;
      }
    }
    uint32_t cnt = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) cnt += __popc(w[q]);
    const uint32_t incl = warp_incl_scan(cnt, lane);
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    if (total == 0) continue;
    unsigned long long b0 = 0;
    if (lane == 0) b0 = atomicAdd(counts + c, (unsigned long long)total);
    unsigned long long pos = __shfl_sync(0xffffffffu, b0, 0) + incl - cnt;
    // byte l of the mask words is domain d0 + l, bit k of a byte isometry k
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      uint32_t x = w[q];
      while (x) {
        const int b = __ffs(x) - 1;
        x &= x - 1;
        if (pos < part) list[pos] = make_uint2(h.x + (uint32_t)(b & 7), h.y + (uint32_t)(4 * q + (b >> 3)));
        ++pos;
      }
    }
  }
}

// ------------------------------------------------------------------ survivor evaluation
// The scan's list is partitioned per scan CTA: partition c holds counts[c] entries (those
// beyond the partition size `part` were dropped and are detected by the host).
__device__ __forceinline__ bool list_slot(unsigned long long i, unsigned long long part,
                                          const unsigned long long* __restrict__ counts) {
  const unsigned long long c = i / part, j = i - c * part;
  return j < counts[c];
}

// One thread per list entry: exact correlation from the q8 row and the range pixels, then
// the reference's fp64 arithmetic (eval_exact) against the range's current bar; an achieved
// residual lowers the bar.  res[i] = residual (+inf when pruned or flat).
#ifndef FIC_EVAL_MINB_FULL
#define FIC_EVAL_MINB_FULL 3  // blocks per SM the register budget targets (full level: 85 registers, no spills)
#endif
#ifndef FIC_EVAL_MINB_BAR
#define FIC_EVAL_MINB_BAR 4  // (sparse levels, bar only: 64 registers)
#endif
template <int NN, int BAR_ONLY>
__global__ void __launch_bounds__(256, BAR_ONLY ? FIC_EVAL_MINB_BAR : FIC_EVAL_MINB_FULL)
eval_kernel(const unsigned char* __restrict__ img, Geometry g, const unsigned short* __restrict__ qpool,
            const DomainMetaI* __restrict__ meta_i, const RangeMeta* __restrict__ rmeta,
            const SurvEntry* __restrict__ list, const unsigned long long* __restrict__ counts, int parts,
            unsigned long long part, double* __restrict__ res, unsigned long long* __restrict__ gbest, DeqTables tab,
            uint2* __restrict__ pend, unsigned* __restrict__ pend_counts, unsigned long long seg,
            unsigned __int128* __restrict__ win) {
  constexpr bool bar_only = BAR_ONLY != 0;
  // pend == nullptr: every candidate's residual is computed here from the operands in registers
  // and the (residual, domain * 8 + isometry) minimum is kept per range in `win` (no residual
  // and winner passes); else the candidates that pass every screen go to the pending list.
  // bar_only (sparse levels, which only have to lower the bar): a rigorous closed-form upper
  // bound of each candidate's exact residual is published instead of the residual itself (no
  // residual loop); the full level evaluates every candidate below that bar exactly
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  const bool screens = !(g.flags & 2);
  const int lane = threadIdx.x & 31;
  // pending candidates go to this block's own segment of the pending list (a shared-memory
  // counter instead of one global counter every warp of the grid contends for)
  __shared__ unsigned s_pend;
  if (threadIdx.x == 0) s_pend = 0;
  __syncthreads();
  uint2* my_pend = pend + (unsigned long long)blockIdx.x * seg;
  const int per = gridDim.x / parts;  // blocks per partition (launch: a multiple of parts)
  const int c = blockIdx.x / per, sub = blockIdx.x % per;
  const unsigned long long n = min(counts[c], part);
  const unsigned long long base = (unsigned long long)c * part;
  // warp-uniform trip count so the pending pushes below can use warp collectives; the next
  // iteration's entry is loaded one iteration ahead
  const unsigned long long jstep = (unsigned long long)per * blockDim.x;
  unsigned long long j0 = (unsigned long long)sub * blockDim.x + (threadIdx.x & ~31u);
  SurvEntry en_next = j0 + lane < n ? list[base + j0 + lane] : make_uint2(kSentinel, 0);
  for (; j0 < n; j0 += jstep) {
    const unsigned long long j = j0 + lane, i = base + j;
    const SurvEntry en = en_next;
    if (j + jstep < n) en_next = list[i + jstep];
    bool pending = false;
    unsigned qs = 0, qo = 0;
    if (j < n) {
      double R = inf;
      if (en.x != kSentinel) {
        const int r = (int)(en.x >> 3), s = (int)(en.x & 7), d = (int)(en.y & 0x7FFFFFFFu);
        // every operand load depends only on the entry: issued together, one L2 round trip
        const DomainMetaI mi = meta_i[d];
        const RangeMeta rm = rmeta[r];
        const double bar = load_bar(gbest, r);
        int x0, y0;
        range_origin(g, r, x0, y0);
        uint32_t qw[NN / 2], bpk[NN / 4];
        load_q8_row<NN>(qpool, d, s, qw);
        load_range_words<NN>(img, g, x0, y0, bpk);
        if (mi.den >= 0) {  // flat code blocks are never candidates (encoder.cpp:223-229)
          R = eval_fast<NN>(g, qw, bpk, rm.sb, (double)rm.var / (double)NN, mi.sq, mi.den, bar, screens,
                            bar_only, tab, qpool, img, d, s, x0, y0, qs, qo, pend ? &pending : nullptr);
          if (R < inf) {
            if (pend || bar_only) {
              publish_best(gbest, r, R);
            } else if (R <= bar) {
              // only a residual at or below the bar read above can lower it or be the final
              // (residual, index) minimum: the bar never drops below the final minimum (seed
              // values are upper bounds of candidates the full level evaluates exactly)
              const unsigned long long rb = (unsigned long long)__double_as_longlong(R);
              if (rb <= atomicMin(gbest + r, rb)) win_min(win + r, R, (uint32_t)d * 8u + (uint32_t)s);
            }
          }
        }
      }
      if (pend) res[i] = R;
    }
    if (!pend) continue;
    // candidates that passed every screen: (entry, codes) to the residual pass
    const unsigned bal = __ballot_sync(0xffffffffu, pending);
    if (bal) {
      unsigned b = 0;
      if (lane == 0) b = atomicAdd(&s_pend, (unsigned)__popc(bal));
      b = __shfl_sync(0xffffffffu, b, 0);
      if (pending) my_pend[b + __popc(bal & ((1u << lane) - 1u))] = make_uint2((uint32_t)i, qs | (qo << 16));
    }
  }
  if (!pend) return;
  __syncthreads();
  if (threadIdx.x == 0) pend_counts[blockIdx.x] = s_pend;
}

// Exact residuals (encoder.cpp:274-280, pixel order, each operation rounded) of the
// candidates eval_kernel left pending, with their dequantised codes from the tables.
template <int NN>
__global__ void __launch_bounds__(256)
residual_kernel(const unsigned char* __restrict__ img, Geometry g, const unsigned short* __restrict__ qpool,
                const SurvEntry* __restrict__ list, const uint2* __restrict__ pend,
                const unsigned* __restrict__ pend_counts, unsigned long long seg, double* __restrict__ res,
                unsigned long long* __restrict__ gbest, DeqTables tab) {
  // one block per eval block: its segment of the pending list
  const unsigned n = pend_counts[blockIdx.x];
  const uint2* my_pend = pend + (unsigned long long)blockIdx.x * seg;
  for (unsigned k = threadIdx.x; k < n; k += blockDim.x) {
    const uint2 p = my_pend[k];
    const SurvEntry en = list[p.x];
    const int r = (int)(en.x >> 3), s = (int)(en.x & 7), d = (int)en.y;
    int x0, y0;
    range_origin(g, r, x0, y0);
    uint32_t qw[NN / 2], bpk[NN / 4];
    load_q8_row<NN>(qpool, d, s, qw);
    load_range_words<NN>(img, g, x0, y0, bpk);
    const double s_deq = tab.s[p.y & 0xFFFFu], o_deq = tab.o[p.y >> 16];
    double r_val = 0.0;
#pragma unroll
    for (int i = 0; i < NN; ++i) {
      const double ai = __dmul_rn((double)q_at(qw, i), 0.25);
      const double bi = (double)((bpk[i >> 2] >> (8 * (i & 3))) & 0xFFu);
      const double dd = __dsub_rn(__dadd_rn(__dmul_rn(s_deq, ai), o_deq), bi);
      r_val = __dadd_rn(r_val, __dmul_rn(dd, dd));
    }
    publish_best(gbest, r, r_val);
    res[p.x] = r_val;
  }
}

// Among the final level's entries whose residual equals the range's final bar, the
// smallest (domain, isometry): the reference's first strict minimum (encoder.cpp:281).
__global__ void winner_kernel(const SurvEntry* __restrict__ list, const unsigned long long* __restrict__ counts,
                              int parts, unsigned long long part, const double* __restrict__ res,
                              const unsigned long long* __restrict__ gbest, unsigned __int128* __restrict__ win) {
  const int per = gridDim.x / parts;
  const int c = blockIdx.x / per, sub = blockIdx.x % per;
  const unsigned long long n = min(counts[c], part);
  for (unsigned long long j = (unsigned long long)sub * blockDim.x + threadIdx.x; j < n;
       j += (unsigned long long)per * blockDim.x) {
    const unsigned long long i = (unsigned long long)c * part + j;
    const double R = res[i];  // +inf for screened-out entries and sentinels (most of them)
    if (!(R < __longlong_as_double(0x7ff0000000000000ll))) continue;
    const SurvEntry en = list[i];
    const int r = (int)(en.x >> 3);
    if ((unsigned long long)__double_as_longlong(R) == gbest[r]) win_min(win + r, R, en.y * 8u + (en.x & 7u));
  }
}

// RangeMapping records: the winner re-evaluated without screens (its quantised codes and
// residual), or flat_mapping for shadow ranges / ranges without any non-flat candidate
// (encoder.cpp:176-181, 291-308).  A winner whose residual differs from the bar it was
// selected by would be an internal error; it is counted in `selfcheck`.
template <int NN>
__global__ void __launch_bounds__(128)
record_kernel(const unsigned char* __restrict__ img, Geometry g, const unsigned short* __restrict__ qpool,
              const DomainMetaI* __restrict__ meta_i, const RangeMeta* __restrict__ rmeta,
              const unsigned __int128* __restrict__ win, const unsigned long long* __restrict__ gbest,
              fic_mapping* __restrict__ out, unsigned long long* __restrict__ selfcheck,
              const unsigned long long* __restrict__ full_counts, int parts, unsigned long long* __restrict__ need,
              unsigned long long* __restrict__ accum, unsigned long long* __restrict__ snap,
              unsigned long long* __restrict__ ticket, int nslots, int snapshot,
              volatile unsigned long long* __restrict__ hstat, int need_off, int cnt_off) {
  // the largest full-level list partition, for the host's overflow check (one status read-back):
  // one warp, its loads in flight together
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    unsigned long long m = 0;
    for (int c = threadIdx.x; c < parts; c += 32) m = max(m, full_counts[c]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) *need = m;
  }
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < g.R) {
  const RangeMeta m = rmeta[r];
  int x0, y0;
  range_origin(g, r, x0, y0);
  uint32_t bpk[NN / 4];
  load_range_words<NN>(img, g, x0, y0, bpk);
  fic_mapping o;
  o.reserved = 0;
  // the (residual, domain * 8 + isometry) minimum; all ones: no non-flat candidate
  const unsigned __int128 wk = win[r];
  const unsigned w = (m.shadow || (unsigned long long)(wk >> 64) == ~0ull) ? 0xFFFFFFFFu : (unsigned)wk;
  if (w != 0xFFFFFFFFu) {
    const int d = (int)(w >> 3), s = (int)(w & 7);
    const DomainMetaI mi = meta_i[d];
    uint32_t qw[NN / 2];
    load_q8_row<NN>(qpool, d, s, qw);
    unsigned qs = 0, qo = 0;
    const double R = eval_exact<NN>(g, qw, bpk, m.sb, (double)m.var / (double)NN, mi.sq, mi.den,
                                    __longlong_as_double(0x7ff0000000000000ll), false, qs, qo);
    if ((unsigned long long)__double_as_longlong(R) != gbest[r]) atomicAdd(selfcheck, 1ull);
    domain_origin(g, d, o.x, o.y);
    o.sym = s;
    o.qs = qs;
    o.qo = qo;
    o.residual = R;
  } else {
    // flat_mapping (encoder.cpp:298-308)
    const double count_d = (double)NN;
    const double ov = (double)m.sb / count_d;
    const unsigned qo = quantize(ov, 255.0, g.o_bits);
    const double o_deq = dequantize(qo, 255.0, g.o_bits);
    double rv = 0.0;
#pragma unroll
    for (int i = 0; i < NN; ++i) {
      const double dd = __dsub_rn(o_deq, (double)((bpk[i >> 2] >> (8 * (i & 3))) & 0xFFu));
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
  // The encode's flat / shadow counters accumulate (pool launch atomics) in `accum`, zero at
  // the start of every encode: the last record block moves them to `snap` (the status slots the
  // host reads; not on a re-run of the full level, which must keep the first snapshot) and
  // clears them and the ticket, so no memset node has to start the next encode.
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(ticket, 1ull) == (unsigned long long)gridDim.x - 1ull;
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    for (int i = threadIdx.x; i < nslots; i += blockDim.x) {
      const unsigned long long v = accum[i];
      accum[i] = 0ull;
      if (snapshot) {
        snap[i] = v;
        if (hstat) hstat[cnt_off + i] = v;
      }
    }
    if (threadIdx.x == 0) {
      *ticket = 0ull;
      // the status the host checks, written straight into its page-locked copy (no read-back
      // copy): self-check count and the largest full-level partition
      if (hstat) {
        hstat[0] = *(volatile unsigned long long*)selfcheck;
        hstat[need_off] = *(volatile unsigned long long*)need;
      }
    }
    if (hstat) __threadfence_system();
  }
}

// (test support, fic_debug_correlations) the exact integer correlation sum_i q_{perm_s(i)} b_i of
// given (range, domain, isometry) triples, through the same q8-row / packed-range loads and
// DP2A dot product the survivor evaluation uses (eval_fast -> dot_q_b).
template <int NN>
__global__ void probe_corr_kernel(const unsigned char* __restrict__ img, Geometry g,
                                  const unsigned short* __restrict__ qpool, int count, const int* __restrict__ rr,
                                  const int* __restrict__ dd, const int* __restrict__ ss, long long* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  int x0, y0;
  range_origin(g, rr[i], x0, y0);
  uint32_t qw[NN / 2], bpk[NN / 4];
  load_q8_row<NN>(qpool, dd[i], ss[i], qw);
  load_range_words<NN>(img, g, x0, y0, bpk);
  out[i] = dot_q_b<NN>(qw, bpk);
}

void launch_probe_corr(const unsigned char* img, const Geometry& g, const unsigned short* qpool, int count,
                       const int* r, const int* d, const int* s, long long* out, cudaStream_t st) {
  const int blocks = (count + 127) / 128;
  if (blocks == 0) return;
  if (g.N == 4) probe_corr_kernel<4><<<blocks, 128, 0, st>>>(img, g, qpool, count, r, d, s, out);
  else if (g.N == 16) probe_corr_kernel<16><<<blocks, 128, 0, st>>>(img, g, qpool, count, r, d, s, out);
  else probe_corr_kernel<64><<<blocks, 128, 0, st>>>(img, g, qpool, count, r, d, s, out);
}

__global__ void fill_u64_kernel(unsigned long long* p, long long n, unsigned long long v) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = v;
}

// ------------------------------------------------------------------ host launchers
bool scan_supported(const Geometry& g) { return g.N == 4 || g.N == 16 || g.N == 64; }

int scan_tiles(const Geometry& g) {
  return (g.D + kScanTileDom - 1) / kScanTileDom;
}

// Padded domain count of the pools (a multiple of the pool-builder block).
long long scan_pool_domains(const Geometry& g) {
  const long long q = kPoolBlock;
  return (g.D + q - 1) / q * q;
}

int scan_rows_per_cta() { return kScanRanges; }

// K1 plus the encode's preparations (PrepAux): counters[b] = flat domains, counters[batch + b]
// = shadow ranges of slice b (zeroed by the caller).  rmeta / gbest / win / deq may be null
// (pool only: the read-back probe).
void launch_pool_v3(const unsigned char* img, const Geometry& g, __half* upool, unsigned short* qpool,
                    DomainMetaI* meta_i, unsigned long long* counters, RangeMeta* rmeta, unsigned long long* gbest,
                    void* win, double* deq, cudaStream_t st, float* thr, unsigned char* ropnd,
                    unsigned long long* pend_count) {
  const int blocks = (int)((long long)g.Dt * g.batch / kPoolBlock);
  const int aux_blocks = rmeta ? (g.R + kPoolThreads - 1) / kPoolThreads : 0;
  const int ro_blocks = rmeta && ropnd ? (g.R + kScanRanges - 1) / kScanRanges : 0;
  const PrepAux aux{rmeta, counters + g.batch, gbest, static_cast<unsigned long long*>(win), deq, blocks,
                    aux_blocks, thr, ropnd, pend_count};
  pool_v3_kernel<<<blocks + aux_blocks + ro_blocks, kPoolThreads, 2 * kPoolBlock * g.N * sizeof(unsigned short),
                   st>>>(img, g, upool, qpool, meta_i, counters, aux);
}

void launch_fill_u64(unsigned long long* p, long long n, unsigned long long v, cudaStream_t st) {
  const int blocks = (int)std::min<long long>((n + 255) / 256, 4096);
  fill_u64_kernel<<<blocks > 0 ? blocks : 1, 256, 0, st>>>(p, n, v);
}

size_t deq_table_entries(const Geometry& g) { return (size_t)(1 << g.s_bits) + (size_t)(1 << g.o_bits); }

void launch_deq_tables(const Geometry& g, double* deq, cudaStream_t st) {
  deq_tables_kernel<<<64, 256, 0, st>>>(g, deq, deq + (1 << g.s_bits));
}

void launch_seed_v3(const unsigned char* img, const Geometry& g, const unsigned short* qpool,
                    const DomainMetaI* meta_i, const RangeMeta* rmeta, unsigned long long* gbest, const double* deq,
                    int half, cudaStream_t st) {
  const int per = (2 * half + 1) * (2 * half + 1) * kSyms;
  const long long threads = (long long)g.R * per;
  const int blocks = (int)((threads + 127) / 128);
  const DeqTables tab{deq, deq + (1 << g.s_bits)};
#define FIC_SEED(NN, H) seed_v3_kernel<NN, H><<<blocks, 128, 0, st>>>(img, g, qpool, meta_i, rmeta, gbest, tab)
  if (g.N == 4) {
    if (half) FIC_SEED(4, 1); else FIC_SEED(4, 0);
  } else if (g.N == 16) {
    if (half) FIC_SEED(16, 1); else FIC_SEED(16, 0);
  } else {
    if (half) FIC_SEED(64, 1); else FIC_SEED(64, 0);
  }
#undef FIC_SEED
}

// Scan CTAs (= list partitions) of a level: kScanCtas per SM.
int scan_grid(const Geometry& g, int stride, int sms) {
  (void)g;
  (void)stride;
  return sms * kScanCtas;
}

static ScanLevel make_level(const Geometry& g, int stride, int G) {
  ScanLevel lv;
  const int n_tiles = scan_tiles(g);
  lv.stride = stride;
  {
    const char* e = std::getenv("FIC_SELECT");  // "0": sparse levels keep every survivor (A/B)
    const int n_lvl = (n_tiles + stride - 1) / stride;
    const char* lb = std::getenv("FIC_LANEBEST_MAX");  // longest level (tiles) using per-lane bests
    const int lane_best_max = lb ? std::atoi(lb) : 48;
    // per-lane bests only for a short last sparse level of a small pool (cfg2: stride 4, 31
    // tiles); every other sparse level selects hit-first (cfg3, levels {32, 4}: 2.343 ms vs
    // 2.411 with per-lane bests at stride 32 and the all-packed selection at stride 4)
    lv.select = stride > 1 && !(e && std::strcmp(e, "0") == 0)
                    ? (n_tiles <= 1024 && stride <= 4 && n_lvl <= lane_best_max ? 3 : 1)
                    : 0;
    if (stride > 1 && e && e[0] >= '1' && e[0] <= '3' && (e[0] != '3' || n_lvl < 8192))
      lv.select = e[0] - '0';  // "1" / "2" / "3": force a selection mode (A/B)
  }
  {
    const char* e = std::getenv("FIC_COARSE");  // "0" / "1": force the whole-tile vote off / on (A/B)
    lv.coarse = e ? (std::strcmp(e, "0") != 0) : (n_tiles > 1024 ? 1 : 0);
  }
  {
    const char* e = std::getenv("FIC_LANE_GROUP");  // lanes per best entry at per-lane-best levels
    const int lg = e ? std::atoi(e) : 1;
    lv.lanes_per_best = lg >= 4 ? 4 : (lg >= 2 ? 2 : 1);
  }
  {
    // rotate the epilogue's column parts over the warps tile by tile (cfg3 full level 1.42 ->
    // 1.31 ms, cfg4 -1 %, cfg2 neutral); FIC_ROTATE=0 / 1 forces it off / on (A/B)
    const char* e = std::getenv("FIC_ROTATE");
    lv.rotate = e ? (std::strcmp(e, "0") != 0) : 1;
  }
  lv.n_lvl = (n_tiles + stride - 1) / stride;
  lv.m_tiles = (g.R + kScanRanges - 1) / kScanRanges;
  lv.rounds = lv.m_tiles / G;
  lv.rem = lv.m_tiles % G;
  lv.k = 1;
  // (select == 3 keeps per-lane bests over a segment: whole m-tiles, one segment each)
  if (lv.rem && lv.select != 3) {  // chunks per leftover m-tile: minimise ceil(rem * k / G) / k, prefer small k
    double best = 1e30;
    for (int k = 1; k <= 16 && k <= lv.n_lvl; ++k) {
      const double t = (double)((lv.rem * k + G - 1) / G) / k;
      if (t < best - 1e-9) {
        best = t;
        lv.k = k;
      }
    }
  }
  return lv;
}

// counts[c] = survivors of scan CTA c; its entries are list[c * part, c * part + min(counts[c], part)).
// Record partition size for entry partitions of `part` entries (see expand_kernel).
// a multiple of kRecChunk: every reserved chunk lies wholly inside or wholly outside its partition
// (and partitions stay 16-byte aligned)
unsigned long long scan_rec_part(unsigned long long part) { return (part / 2 + kRecChunk) & ~(unsigned long long)(kRecChunk - 1); }
size_t scan_rec_bytes(unsigned long long list_cap, int parts) {
  // the partitions, then one scratch chunk per scan CTA
  return ((size_t)scan_rec_part(list_cap / (unsigned long long)parts) + kRecChunk) * parts * sizeof(MaskRec);
}

// Hit-first sparse levels with an fp16 accumulator (scan mode 7): a sparse level only lowers
// the bar, so neither its test nor its selection needs a bound.  The fp16 selection tags each
// half with its isometry (one LOP3 per register) and takes the half2 |max| tree: on by default
// for small pools (cfg3: stride-32 / stride-4 levels 112 -> 88 / 512 -> 421 us, encode 2.04 ->
// 1.92 ms); large pools keep fp32 (cfg4: its stride-16 level got slower and its 2^-7 magnitude
// resolution a weaker bar, 63.1 -> 64.9 ms).  FIC_F16SEL=0 / 1 forces it off / on.
bool scan_f16sel(const Geometry& g) {
  const char* e = std::getenv("FIC_F16SEL");
  if (e) return e[0] == '1';
  return scan_tiles(g) <= 1024;
}

typedef void (*ScanKern)(const unsigned char*, Geometry, ScanLevel, const __half*, const RangeMeta*,
                         const unsigned char*, const float*, MaskRec*, unsigned long long*, unsigned long long,
                         SurvEntry*, unsigned long long, unsigned long long*, EvalCtx);

template <int EV>
ScanKern scan_fn(int mode) {
  switch (mode) {
    case 0: return scan_kernel<0, EV>;
    case 1: return scan_kernel<1, EV>;
    case 2: return scan_kernel<2, EV>;
    case 3: return scan_kernel<3, EV>;
    case 4: return scan_kernel<4, EV>;
    case 5: return scan_kernel<5, EV>;
    case 6: return scan_kernel<6, EV>;
    case 7: return scan_kernel<7, EV>;
    default: return scan_kernel<9, EV>;
  }
}

// The fused scan (survivors evaluated inside the scan kernel): opt-in, FIC_FUSED=1 (measured
// slower than the separate evaluation pass on every configuration).
bool scan_fused() {
  const char* e = std::getenv("FIC_FUSED");
  return e && e[0] == '1';
}

cudaError_t launch_scan(const unsigned char* img, const Geometry& g, int stride, int sms, const __half* upool,
                        const RangeMeta* rmeta, const unsigned char* ropnd, const float* thr, SurvEntry* list,
                        unsigned long long* counts, unsigned long long part, void* recs, unsigned long long* rcounts,
                        const unsigned short* qpool, const DomainMetaI* meta_i, unsigned long long* gbest,
                        void* win, const double* deq, bool fused, cudaStream_t st, cudaEvent_t after_scan) {
  const int grid = scan_grid(g, stride, sms);
  const ScanLevel lv = make_level(g, stride, grid);
  const ScanSmem L = scan_smem_layout(g.K, fused);
  int mode = lv.select == 3 ? 4 : (lv.select == 2 ? 3 : (lv.select == 1 ? 2 : (lv.coarse ? 1 : 0)));
  // fp16 accumulator: the full level only (its thresholds carry the fp16 bound, range_op_kernel)
  if (scan_f16acc(g) && stride == 1 && mode <= 1) mode += 5;
  if ((mode == 2 || mode == 4) && scan_f16sel(g)) mode += 5;  // 7 / 9: fp16 selection
  const ScanKern kern = !fused ? scan_fn<0>(mode)
                        : g.N == 4 ? scan_fn<4>(mode) : (g.N == 16 ? scan_fn<16>(mode) : scan_fn<64>(mode));
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
  if (e != cudaSuccess) return e;
  const unsigned long long rcap = scan_rec_part(part);
  MaskRec* R = static_cast<MaskRec*>(recs);
  const EvalCtx ev{img, qpool, meta_i, rmeta, gbest, static_cast<unsigned __int128*>(win),
                   DeqTables{deq, deq + (1 << g.s_bits)}};
  kern<<<grid, fused ? kFusedThreads : kScanThreads, L.total, st>>>(img, g, lv, upool, rmeta, ropnd, thr, R, rcounts,
                                                                    rcap, list, part, counts, ev);
  e = cudaGetLastError();
  if (e == cudaSuccess && after_scan) e = cudaEventRecord(after_scan, st);  // timing: the scan kernel alone
  // sparse levels append their selected entries directly (no mask records to expand)
  if (e != cudaSuccess || fused || lv.select != 0) return e;
  expand_kernel<<<grid * 8, 256, 0, st>>>(R, rcounts, rcap, list, counts, part, 8);
  return cudaGetLastError();
}

// Kernels launch_scan enqueues for a level: the scan, plus expand_kernel where the level writes
// mask records (full level, separate evaluation).
int scan_level_launches(const Geometry& g, int stride, int sms, bool fused) {
  return 1 + (!fused && make_level(g, stride, scan_grid(g, stride, sms)).select == 0 ? 1 : 0);
}

// Full level with an fp16 accumulator whenever sparse levels ran before it (their bar keeps the
// wider fp16 bound's extra survivors few) or the pool is large (whole-tile vote).  The fp16
// epilogue tests 4 columns per |max| instruction and one half2 compare per range, so it beats
// fp32 wherever the survivors stay few: cfg2 full level 121 -> 102 us, cfg3 1.31 -> 1.09 ms,
// cfg4 56.5 -> 51.6 ms; cfg1 (no sparse level: hit-dominated) keeps fp32 (0.226 vs 0.223 ms).
// FIC_F16ACC=1 / 0 forces it on / off.
bool scan_use_f16acc(const Geometry& g, int stride, int sms, bool sparse_levels) {
  if (stride != 1) return false;
  const char* e = std::getenv("FIC_F16ACC");
  if (e) return e[0] == '1';
  const ScanLevel lv = make_level(g, 1, scan_grid(g, 1, sms));
  return lv.select == 0 && (lv.coarse || sparse_levels);
}

int scan_padded_ranges(const Geometry& g) { return ((g.R + kScanRanges - 1) / kScanRanges) * kScanRanges; }

void launch_threshold(const Geometry& g, const RangeMeta* rmeta, const unsigned long long* gbest, float* thr,
                      cudaStream_t st) {
  const int padded = scan_padded_ranges(g);
  threshold_kernel<<<(padded + 255) / 256, 256, 0, st>>>(g, rmeta, gbest, thr, padded);
}

size_t range_op_bytes(const Geometry& g) {
  return (size_t)((g.R + kScanRanges - 1) / kScanRanges) * kScanRows * g.K * 2;
}

// Thresholds of a level (thr, padded to whole m-tiles) and, when the scan needs new ones, the
// range operands.
void launch_level_ops(const unsigned char* img, const Geometry& g, const RangeMeta* rmeta,
                      const unsigned long long* gbest, float* thr, unsigned char* ropnd,
                      unsigned long long* pend_count, bool full_level, unsigned long long* selfcheck,
                      cudaStream_t st) {
  const dim3 grid((g.R + kScanRanges - 1) / kScanRanges, g.K / 8);
  const int fl = full_level ? 1 : 0;
  if (g.N == 4 && g.K == 16)
    range_op_kernel<4><<<grid, 256, 0, st>>>(img, g, rmeta, gbest, thr, ropnd, pend_count, fl, selfcheck);
  else if (g.N == 16 && g.K == 16)
    range_op_kernel<16><<<grid, 256, 0, st>>>(img, g, rmeta, gbest, thr, ropnd, pend_count, fl, selfcheck);
  else if (g.N == 64 && g.K == 64)
    range_op_kernel<64><<<grid, 256, 0, st>>>(img, g, rmeta, gbest, thr, ropnd, pend_count, fl, selfcheck);
  else
    range_op_kernel<0><<<grid, 256, 0, st>>>(img, g, rmeta, gbest, thr, ropnd, pend_count, fl, selfcheck);
}

// Pending-list segment per eval block: the most entries one block can take (eval_kernel's
// warp-strided loop over its partition).
constexpr int kEvalPer = 8;  // eval blocks per partition
unsigned long long eval_pend_seg(unsigned long long part) {
  const unsigned long long stride = (unsigned long long)kEvalPer * 256;
  return (part + stride - 1) / stride * 256;
}

// inline_res: residuals and the per-range winner key in eval_kernel itself (no residual pass;
// the final level needs no winner pass either); else eval + residual kernels (pending list).
void launch_eval(const unsigned char* img, const Geometry& g, const unsigned short* qpool, const DomainMetaI* meta_i,
                 const RangeMeta* rmeta, const SurvEntry* list, const unsigned long long* counts, int parts,
                 unsigned long long part, double* res, unsigned long long* gbest, const double* deq, uint2* pend,
                 unsigned* pend_counts, void* win_, bool inline_res, bool bar_only, int sms, cudaStream_t st) {
  (void)sms;
  int per = kEvalPer;  // blocks per list partition (the pending-list path needs kEvalPer)
  if (inline_res || bar_only) per = std::max(1, kEvalPer / kScanCtas);  // the same grid for 2 CTAs per SM
  if (const char* e = std::getenv("FIC_EVAL_PER"); e && (inline_res || bar_only)) per = std::max(1, std::atoi(e));
  const int blocks = parts * per;
  const unsigned long long seg = eval_pend_seg(part);
  const DeqTables tab{deq, deq + (1 << g.s_bits)};
  unsigned __int128* win = static_cast<unsigned __int128*>(win_);
  uint2* pd = inline_res || bar_only ? nullptr : pend;
#define FIC_EVAL(NN)                                                                                                 \
  if (bar_only)                                                                                                      \
    eval_kernel<NN, 1><<<blocks, 256, 0, st>>>(img, g, qpool, meta_i, rmeta, list, counts, parts, part, res, gbest,  \
                                               tab, pd, pend_counts, seg, win);                                      \
  else                                                                                                               \
    eval_kernel<NN, 0><<<blocks, 256, 0, st>>>(img, g, qpool, meta_i, rmeta, list, counts, parts, part, res, gbest,  \
                                               tab, pd, pend_counts, seg, win);                                      \
  if (pd)                                                                                                            \
    residual_kernel<NN><<<blocks, 256, 0, st>>>(img, g, qpool, list, pend, pend_counts, seg, res, gbest, tab);
  if (g.N == 4) {
    FIC_EVAL(4)
  } else if (g.N == 16) {
    FIC_EVAL(16)
  } else {
    FIC_EVAL(64)
  }
#undef FIC_EVAL
}

// Inline residuals in eval_kernel (FIC_EVAL_SPLIT=1: separate pending-list residual pass).
bool eval_inline() {
  const char* e = std::getenv("FIC_EVAL_SPLIT");
  return !(e && e[0] == '1');
}

void launch_winner(const SurvEntry* list, const unsigned long long* counts, int parts, unsigned long long part,
                   const double* res, const unsigned long long* gbest, void* win, int sms, cudaStream_t st) {
  winner_kernel<<<parts * 16, 256, 0, st>>>(list, counts, parts, part, res, gbest,
                                            static_cast<unsigned __int128*>(win));
}

void launch_record(const unsigned char* img, const Geometry& g, const unsigned short* qpool,
                   const DomainMetaI* meta_i, const RangeMeta* rmeta, const void* win_,
                   const unsigned long long* gbest, fic_mapping* out, unsigned long long* selfcheck,
                   const unsigned long long* full_counts, int parts, unsigned long long* need,
                   unsigned long long* accum, unsigned long long* snap, unsigned long long* ticket, int nslots,
                   bool snapshot, unsigned long long* hstat, int need_off, int cnt_off, cudaStream_t st) {
  // small blocks: the per-range exact evaluations (a latency chain each) spread over more SMs
  constexpr int kRecThreads = 32;
  const int blocks = (g.R + kRecThreads - 1) / kRecThreads;
  const unsigned __int128* win = static_cast<const unsigned __int128*>(win_);
#define FIC_REC(NN) \
  record_kernel<NN><<<blocks, kRecThreads, 0, st>>>(img, g, qpool, meta_i, rmeta, win, gbest, out, selfcheck, full_counts, parts, \
                                           need, accum, snap, ticket, nslots, snapshot ? 1 : 0, hstat, need_off, cnt_off)
  if (g.N == 4) FIC_REC(4);
  else if (g.N == 16) FIC_REC(16);
  else FIC_REC(64);
#undef FIC_REC
}

}  // namespace ficb
