// decoder.cu — K3, the iterated PIFS decoder (proj/src/decoder.cpp:39-128).
//
// One thread per OUTPUT pixel: the write stream is perfectly coalesced, and the four
// source reads of neighbouring threads fall in the same few rows of the domain window,
// so each iteration moves ~16 B/px of algorithmic traffic (8 B read through L2, 8 B
// written).  The step RMSE of decode_traced (decoder.cpp:28-37) is fused: each block
// reduces its (current - next)^2 terms into one fp64 partial, and a second tiny kernel
// sums the partials in a fixed order (deterministic run to run; the reference's
// sequential sum order is not reproduced, so step_rmse agrees to ~1e-15 relative,
// while every raster value is bit-exact).
#include <cstdlib>

#include "common.cuh"

namespace ficb {

// Dequantised per-range transform, prepared once per decode.
struct RangeXform {
  double s, o;
  int dx, dy;  // domain origin at magnification (pixels)
  int sym;
  int pad;
};

__global__ void xform_kernel(const fic_mapping* __restrict__ maps, int count, int scale, int s_bits, double s_max,
                             int o_bits, RangeXform* __restrict__ xf) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const fic_mapping m = maps[i];
  RangeXform t;
  t.s = dequantize(m.qs, s_max, s_bits);
  t.o = dequantize(m.qo, 255.0, o_bits);
  t.dx = m.x * scale;
  t.dy = m.y * scale;
  t.sym = m.sym;
  t.pad = 0;
  xf[i] = t;
}

constexpr int kDecodeThreads = 256;

__global__ void __launch_bounds__(kDecodeThreads)
decode_step_kernel(const double* __restrict__ cur, double* __restrict__ nxt, const RangeXform* __restrict__ xf,
                   int out_w, int out_h, int kn, int ranges_x, int ranges_y, double* __restrict__ partial) {
  const long long idx = (long long)blockIdx.x * kDecodeThreads + threadIdx.x;
  const long long total = (long long)out_w * out_h;
  double sq = 0.0;
  if (idx < total) {
    const int Y = (int)(idx / out_w), X = (int)(idx % out_w);
    const int ry = Y / kn, rx = X / kn;
    double v = 0.0;  // pixels outside the range grid keep constant_raster's 0 (decoder.cpp:56)
    if (rx < ranges_x && ry < ranges_y) {
      const int r = Y - ry * kn, c = X - rx * kn;
      const RangeXform t = xf[ry * ranges_x + rx];
      int sr, sc;
      symmetry_source(t.sym, r, c, kn, sr, sc);
      const double* row0 = cur + (long long)(t.dy + 2 * sr) * out_w + t.dx + 2 * sc;
      const double* row1 = row0 + out_w;
      // ((p00 + p01) + p10 + p11) / 4.0 then s*z + o, each op rounded (decoder.cpp:71-75); the
      // division by 4 is an exact power-of-two scaling, identical to the multiplication by 0.25
      const double z =
          __dmul_rn(__dadd_rn(__dadd_rn(__dadd_rn(__ldg(row0), __ldg(row0 + 1)), __ldg(row1)), __ldg(row1 + 1)), 0.25);
      v = __dadd_rn(__dmul_rn(t.s, z), t.o);
    }
    nxt[idx] = v;
    const double dlt = __dsub_rn(cur[idx], v);
    sq = __dmul_rn(dlt, dlt);
  }
  if (partial) {
    __shared__ double red[kDecodeThreads / 32];
    for (int o = 16; o > 0; o >>= 1) sq = __dadd_rn(sq, __shfl_xor_sync(0xffffffffu, sq, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < kDecodeThreads / 32; ++w) s = __dadd_rn(s, red[w]);
      partial[blockIdx.x] = s;
    }
  }
}

// Tiled variant of decode_step_kernel for the common geometries (kn a multiple of 32, or a
// divisor of 32 with the raster a whole number of 32 x 32 tiles, ranges covering it).  One CTA per 32 x 32 output
// tile, i.e. (32/T)^2 blocks of T x T output pixels (T = min(kn, 32)), each block the whole
// range (kn <= 32) or a sub-square of one (kn > 32).  An isometry maps an aligned T x T
// sub-square of the range onto an aligned T x T sub-square of its source, so phase 1 loads
// the 2T x 2T source windows of the tile's blocks row by row (coalesced for every isometry)
// and forms their 2x2 means z in shared memory; phase 2 writes the tile's outputs
// row-coalesced, reading z through the isometry (the transposing isometries, half of them,
// no longer turn every warp's gather into 32 separate raster rows).  Same per-pixel
// arithmetic as decode_step_kernel, so the rasters are bit-identical.
constexpr int kTile = 32;
constexpr int kTileThreads = 256;

bool decode_tiled(int out_w, int out_h, int kn) {
  if (out_w % kTile != 0 || out_h % kTile != 0) return false;
  return kn >= kTile ? kn % kTile == 0 : (kTile % kn == 0 && kn >= 2);
}

__global__ void __launch_bounds__(kTileThreads)
decode_tile_kernel(const double* __restrict__ cur, double* __restrict__ nxt, const RangeXform* __restrict__ xf,
                   int out_w, int kn, int ranges_x, double* __restrict__ partial) {
  __shared__ double zs[kTile][kTile + 1];
  struct Blk {
    double s, o;
    int row0, col0;  // raster origin of the block's source window (2T x 2T)
    int sym, sr0, sc0;
  };
  __shared__ Blk blk[(kTile / 2) * (kTile / 2)];
  const int T = kn < kTile ? kn : kTile;
  const int bpr = kTile / T;  // blocks per tile row
  const int tiles_x = out_w / kTile;
  const int ty = blockIdx.x / tiles_x, tx = blockIdx.x % tiles_x;
  const int Y0 = ty * kTile, X0 = tx * kTile;
  for (int b = threadIdx.x; b < bpr * bpr; b += kTileThreads) {
    const int bi = b / bpr, bj = b % bpr;
    const int Yb = Y0 + bi * T, Xb = X0 + bj * T;  // the block's first output pixel
    const int ry = Yb / kn, rx = Xb / kn;
    const int a = Yb - ry * kn, c = Xb - rx * kn;  // its offset inside the range
    const RangeXform t = xf[ry * ranges_x + rx];
    int r0, c0, r1, c1;
    symmetry_source(t.sym, a, c, kn, r0, c0);
    symmetry_source(t.sym, a + T - 1, c + T - 1, kn, r1, c1);
    Blk B;
    B.s = t.s;
    B.o = t.o;
    B.sym = t.sym;
    B.sr0 = min(r0, r1);
    B.sc0 = min(c0, c1);
    B.row0 = t.dy + 2 * B.sr0;
    B.col0 = t.dx + 2 * B.sc0;
    blk[b] = B;
  }
  __syncthreads();
  // phase 1: z of every block's source sub-square, stored at the block's place in the tile
  // (all 16 loads of a thread issued before the first use)
  constexpr int kPer = kTile * kTile / kTileThreads;
  double p[kPer][4];
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int e = threadIdx.x + k * kTileThreads;
    const int zr = e / kTile, zc = e % kTile;
    const Blk& B = blk[(zr / T) * bpr + zc / T];
    const double* row0 = cur + (long long)(B.row0 + 2 * (zr % T)) * out_w + B.col0 + 2 * (zc % T);
    p[k][0] = __ldg(row0);
    p[k][1] = __ldg(row0 + 1);
    p[k][2] = __ldg(row0 + out_w);
    p[k][3] = __ldg(row0 + out_w + 1);
  }
  double cv[kPer];  // the tile's own current values, for the step RMSE
  if (partial) {
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int e = threadIdx.x + k * kTileThreads;
      cv[k] = __ldg(cur + (long long)(Y0 + e / kTile) * out_w + X0 + e % kTile);
    }
  }
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int e = threadIdx.x + k * kTileThreads;
    zs[e / kTile][e % kTile] = __dmul_rn(__dadd_rn(__dadd_rn(__dadd_rn(p[k][0], p[k][1]), p[k][2]), p[k][3]), 0.25);
  }
  __syncthreads();
  // phase 2: outputs, row-coalesced.  The next raster is written with evict-first stores so
  // the current one (re-read by the overlapping domain windows) keeps the L2.
  double sq = 0.0;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int e = threadIdx.x + k * kTileThreads;
    const int orow = e / kTile, ocol = e % kTile;
    const int bi = orow / T, bj = ocol / T;
    const Blk& B = blk[bi * bpr + bj];
    const int Y = Y0 + orow, X = X0 + ocol;
    int sr, sc;
    symmetry_source(B.sym, Y % kn, X % kn, kn, sr, sc);
    const double z = zs[bi * T + sr - B.sr0][bj * T + sc - B.sc0];
    const double v = __dadd_rn(__dmul_rn(B.s, z), B.o);
    __stcs(nxt + (long long)Y * out_w + X, v);
    if (partial) {
      const double dlt = __dsub_rn(cv[k], v);
      sq = __dadd_rn(sq, __dmul_rn(dlt, dlt));
    }
  }
  if (partial) {
    __shared__ double red[kTileThreads / 32];
    for (int o = 16; o > 0; o >>= 1) sq = __dadd_rn(sq, __shfl_xor_sync(0xffffffffu, sq, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < kTileThreads / 32; ++w) s = __dadd_rn(s, red[w]);
      partial[blockIdx.x] = s;
    }
  }
}

// ------------------------------------------------------------------ mean-raster decoder
// Every 2x2 mean the decoder reads, z = ((p00 + p01) + p10 + p11) / 4 at (dy + 2 sr, dx + 2 sc),
// lies on the even grid whenever every magnified domain origin (dx, dy) is even (checked on
// the host against the actual mappings: scale even, or every x and y even).  Then iteration i
// needs only the half-resolution MEAN raster m_i (m_i(a, b) = z at (2a, 2b) of raster i): output
// pixel P of iteration i + 1 is v_{i+1}(P) = s_P * m_i(src(P)) + o_P, with src and (s, o) fixed
// by P's range.  So the full-resolution raster never has to exist between iterations:
//   * the step RMSE's current value v_i(P) = s_P * m_{i-1}(src(P)) + o_P is recomputed from the
//     previous mean raster (the same operations on the same operands, so the same bits as the
//     stored raster value), the initial raster being read only in iteration 0;
//   * each 32 x 32 output tile forms its own 2 x 2 means m_{i+1} (quarter size);
//   * the last iteration writes the quantised output image directly (decoder.cpp:99-109).
// Per iteration and output pixel that is 8 B of m_i + 8 B of m_{i-1} read and 2 B of m_{i+1}
// written — three quarter-size rasters, L2-resident up to 4096^2 outputs (3 x 33.5 MB) — instead
// of an 8 B raster write and an 8 B raster read in HBM.  Every raster value, the output image
// and each step's sum of squared differences are those of the per-pixel kernel.
constexpr int kMeanThreads = 128;  // 8 output pixels per thread: the per-tile setup amortised over more work

bool decode_mean_ok(int out_w, int out_h, int kn, bool even_origins) {
  return decode_tiled(out_w, out_h, kn) && even_origins;
}

// m_0: the initial raster's 2 x 2 means (constant kinds: the constant).
__global__ void mean_init_kernel(double* __restrict__ m, int out_w, int out_h, int kind,
                                 const unsigned char* __restrict__ sup) {
  const int hw = out_w / 2;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)hw * (out_h / 2)) return;
  if (kind != FIC_INITIAL_SUPPLIED) {
    m[i] = kind == FIC_INITIAL_MID_GRAY ? 128.0 : 0.0;  // (c + c + c + c) / 4 == c exactly
    return;
  }
  const int y = (int)(i / hw), x = (int)(i % hw);
  const unsigned char* p = sup + (long long)(2 * y) * out_w + 2 * x;
  m[i] = __dmul_rn(__dadd_rn(__dadd_rn(__dadd_rn((double)p[0], (double)p[1]), (double)p[out_w]), (double)p[out_w + 1]),
                   0.25);
}

// LT = log2 of the block side T: 5 = the tile lies inside one range (kn a multiple of 32), else
// T = kn = 2^LT < 32 and the tile holds (32/T)^2 whole ranges.  Index arithmetic is shifts and
// masks.  mprev == nullptr: iteration 0, the current values come from the initial raster
// (init_kind, sup); out_u8 != nullptr: also write the quantised image of this iteration's output.
template <int LT>
__global__ void __launch_bounds__(kMeanThreads)
decode_means_kernel(const double* __restrict__ mcur, const double* __restrict__ mprev, int init_kind,
                    const unsigned char* __restrict__ sup, double* __restrict__ mnxt,
                    const RangeXform* __restrict__ xf, int out_w, int kn, int ranges_x,
                    double* __restrict__ partial, unsigned char* __restrict__ out_u8) {
  constexpr bool kWhole = LT == 5;
  constexpr int T = 1 << LT, bpr = kTile / T, nb = bpr * bpr;
  __shared__ double zs[kTile][kTile + 1];  // m_i at the tile's sources
  __shared__ double ps[kTile][kTile + 1];  // m_{i-1} at the same places (i >= 1)
  __shared__ double vs[kTile][kTile + 1];  // the tile's new values (its 2 x 2 means)
  struct Blk {
    double s, o;
    int mrow0, mcol0;  // mean-raster origin of the block's source sub-square (T x T)
    int sym, sr0, sc0;
  };
  __shared__ Blk blk[kWhole ? 1 : nb];
  const int hw = out_w / 2;
  const int Y0 = blockIdx.y * kTile, X0 = blockIdx.x * kTile;  // 2-D grid of tiles
  const int lane_c = threadIdx.x & (kTile - 1), row0 = threadIdx.x >> 5;  // element e = threadIdx.x + 256 k
  constexpr int kPer = kTile * kTile / kMeanThreads;
  constexpr int kRowStep = kMeanThreads / kTile;
  const bool first = mprev == nullptr;
  double zv[kPer], pv[kPer];
  Blk B;
  unsigned aw = 0;     // kWhole: the isometry as an affine map (symmetry_affine_word)
  int a0 = 0, c0 = 0;  // kWhole: the tile's offset inside its range
  if (kWhole) {
    // the tile's block (one range): thread 0 does the divisions, the code load and the corner
    // sources once, every thread reads them from shared memory
    __shared__ int s_blk[6];
    __shared__ double s_so[2];
    if (threadIdx.x == 0) {
      const int ry = Y0 / kn, rx = X0 / kn;
      const int ta0 = Y0 - ry * kn, tc0 = X0 - rx * kn;
      const RangeXform t = xf[ry * ranges_x + rx];
      int r0, cc0, r1, c1;
      symmetry_source(t.sym, ta0, tc0, kn, r0, cc0);
      symmetry_source(t.sym, ta0 + T - 1, tc0 + T - 1, kn, r1, c1);
      s_blk[0] = ta0;
      s_blk[1] = tc0;
      s_blk[2] = t.sym;
      s_blk[3] = min(r0, r1);
      s_blk[4] = min(cc0, c1);
      s_blk[5] = 0;
      s_so[0] = t.s;
      s_so[1] = t.o;
      blk[0].mrow0 = t.dy / 2 + min(r0, r1);
      blk[0].mcol0 = t.dx / 2 + min(cc0, c1);
    }
    __syncthreads();
    a0 = s_blk[0];
    c0 = s_blk[1];
    B.sym = s_blk[2];
    B.sr0 = s_blk[3];
    B.sc0 = s_blk[4];
    B.s = s_so[0];
    B.o = s_so[1];
    B.mrow0 = blk[0].mrow0;
    B.mcol0 = blk[0].mcol0;
    aw = symmetry_affine_word(B.sym);
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const long long off = (long long)(B.mrow0 + row0 + k * kRowStep) * hw + B.mcol0 + lane_c;
      zv[k] = __ldg(mcur + off);
      pv[k] = first ? 0.0 : __ldg(mprev + off);
    }
  } else {
    for (int b = threadIdx.x; b < nb; b += kMeanThreads) {
      const int ry = (Y0 >> LT) + b / bpr, rx = (X0 >> LT) + b % bpr;
      const RangeXform t = xf[ry * ranges_x + rx];
      Blk Q;
      Q.s = t.s;
      Q.o = t.o;
      Q.sym = t.sym;
      Q.sr0 = Q.sc0 = 0;
      Q.mrow0 = t.dy / 2;
      Q.mcol0 = t.dx / 2;
      blk[b] = Q;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int zr = row0 + k * kRowStep, zc = lane_c;
      const Blk& Q = blk[(zr >> LT) * bpr + (zc >> LT)];
      const long long off = (long long)(Q.mrow0 + (zr & (T - 1))) * hw + Q.mcol0 + (zc & (T - 1));
      zv[k] = __ldg(mcur + off);
      pv[k] = first ? 0.0 : __ldg(mprev + off);
    }
  }
  // iteration 0: the tile's initial values (constant, or the supplied image at the output pixel)
  double cv[kPer];
  if (first) {
#pragma unroll
    for (int k = 0; k < kPer; ++k)
      cv[k] = init_kind == FIC_INITIAL_MID_GRAY ? 128.0
              : init_kind == FIC_INITIAL_BLACK  ? 0.0
                                                : (double)sup[(long long)(Y0 + row0 + k * kRowStep) * out_w + X0 + lane_c];
  }
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    zs[row0 + k * kRowStep][lane_c] = zv[k];
    ps[row0 + k * kRowStep][lane_c] = pv[k];
  }
  __syncthreads();
  double sq = 0.0;
  int zoff0 = 0, zstep = 0;
  if (kWhole) {  // the isometry is affine in (row, col): one base and one stride per thread
    const int m = kn - 1, r = a0 + row0, c = c0 + lane_c;
    const int sr = affine_coef(aw, 0) * r + affine_coef(aw, 1) * c + affine_coef(aw, 2) * m;
    const int sc = affine_coef(aw, 3) * r + affine_coef(aw, 4) * c + affine_coef(aw, 5) * m;
    zoff0 = (sr - B.sr0) * (kTile + 1) + (sc - B.sc0);
    zstep = kRowStep * (affine_coef(aw, 0) * (kTile + 1) + affine_coef(aw, 3));
  }
  const double* zflat = &zs[0][0];
  const double* pflat = &ps[0][0];
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int orow = row0 + k * kRowStep, ocol = lane_c;
    double z, p, s, o;
    if (kWhole) {
      z = zflat[zoff0 + k * zstep];
      p = pflat[zoff0 + k * zstep];
      s = B.s;
      o = B.o;
    } else {
      const int bi = orow >> LT, bj = ocol >> LT;
      const Blk& Q = blk[bi * bpr + bj];
      int sr, sc;
      symmetry_source(Q.sym, orow & (T - 1), ocol & (T - 1), T, sr, sc);
      z = zs[(bi << LT) + sr][(bj << LT) + sc];
      p = ps[(bi << LT) + sr][(bj << LT) + sc];
      s = Q.s;
      o = Q.o;
    }
    const double v = __dadd_rn(__dmul_rn(s, z), o);  // decoder.cpp:71-75
    const double c = first ? cv[k] : __dadd_rn(__dmul_rn(s, p), o);
    vs[orow][ocol] = v;
    if (out_u8) out_u8[(long long)(Y0 + orow) * out_w + X0 + ocol] = (unsigned char)lround(clampd(v, 0.0, 255.0));
    const double dlt = __dsub_rn(c, v);
    sq = __dadd_rn(sq, __dmul_rn(dlt, dlt));
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 256; e += kMeanThreads) {  // the next iteration's 16 x 16 means of the tile
    const int i = e >> 4, j = e & 15;
    const double m = __dmul_rn(
        __dadd_rn(__dadd_rn(__dadd_rn(vs[2 * i][2 * j], vs[2 * i][2 * j + 1]), vs[2 * i + 1][2 * j]), vs[2 * i + 1][2 * j + 1]),
        0.25);
    mnxt[(long long)(Y0 / 2 + i) * hw + X0 / 2 + j] = m;
  }
  __shared__ double red[kMeanThreads / 32];
  for (int off = 16; off > 0; off >>= 1) sq = __dadd_rn(sq, __shfl_xor_sync(0xffffffffu, sq, off));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kMeanThreads / 32; ++w) t = __dadd_rn(t, red[w]);
    partial[blockIdx.y * gridDim.x + blockIdx.x] = t;
  }
}

void launch_mean_init(double* m, int out_w, int out_h, int kind, const unsigned char* sup, cudaStream_t st) {
  const long long n = (long long)(out_w / 2) * (out_h / 2);
  mean_init_kernel<<<(int)((n + 255) / 256), 256, 0, st>>>(m, out_w, out_h, kind, sup);
}

// One iteration on the mean rasters (decode_mean_ok); partials as decode_partials.
void launch_decode_means(const double* mcur, const double* mprev, int init_kind, const unsigned char* sup,
                         double* mnxt, const RangeXform* xf, int out_w, int out_h, int kn, int ranges_x,
                         double* partial, unsigned char* out_u8, cudaStream_t st) {
  const dim3 grid(out_w / kTile, out_h / kTile);
#define FIC_MEANS(LT)                                                                                   \
  decode_means_kernel<LT><<<grid, kMeanThreads, 0, st>>>(mcur, mprev, init_kind, sup, mnxt, xf, out_w, kn, \
                                                         ranges_x, partial, out_u8)
  switch (kn >= kTile ? 5 : __builtin_ctz((unsigned)kn)) {
    case 1: FIC_MEANS(1); break;
    case 2: FIC_MEANS(2); break;
    case 3: FIC_MEANS(3); break;
    case 4: FIC_MEANS(4); break;
    default: FIC_MEANS(5); break;
  }
#undef FIC_MEANS
}

// Sums the per-block partials in index order and writes rmse = sqrt(sum / count); block k
// finishes iteration k (partials partial[k * blocks ...], result out[k]), so a decode without
// a convergence test reduces every iteration's partials in one launch at the end.
__global__ void rmse_finish_kernel(const double* __restrict__ partial, int blocks, long long count,
                                   double* __restrict__ out) {
  __shared__ double red[1024];
  partial += (long long)blockIdx.x * blocks;
  out += blockIdx.x;
  double s = 0.0;
  for (int i = threadIdx.x; i < blocks; i += blockDim.x) s = __dadd_rn(s, partial[i]);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] = __dadd_rn(red[threadIdx.x], red[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sqrt(__ddiv_rn(red[0], (double)count));
}

__global__ void raster_init_kernel(double* __restrict__ r, long long count, int kind,
                                   const unsigned char* __restrict__ supplied) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  r[i] = kind == FIC_INITIAL_MID_GRAY ? 128.0 : (kind == FIC_INITIAL_BLACK ? 0.0 : (double)supplied[i]);
}

// quantize_raster (decoder.cpp:99-109): clamp to [0, 255] and round half away from zero.
__global__ void quantize_raster_kernel(const double* __restrict__ r, long long count, unsigned char* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  out[i] = (unsigned char)lround(clampd(r[i], 0.0, 255.0));
}

int decode_blocks(long long count) { return (int)((count + kDecodeThreads - 1) / kDecodeThreads); }

// Partials one decode step writes.
int decode_partials(int out_w, int out_h, int kn, bool covers) {
  if (covers && decode_tiled(out_w, out_h, kn) && !std::getenv("FIC_DECODE_FLAT"))
    return (out_w / kTile) * (out_h / kTile);
  return decode_blocks((long long)out_w * out_h);
}

void launch_xform(const fic_mapping* maps, int count, int scale, const Geometry& g, RangeXform* xf, cudaStream_t st) {
  xform_kernel<<<(count + 255) / 256, 256, 0, st>>>(maps, count, scale, g.s_bits, g.s_max, g.o_bits, xf);
}

// ranges_x x ranges_y ranges of kn x kn pixels; the tiled kernel needs them to cover the raster
// (fic_decode passes covers = width % n == 0 && height % n == 0).
void launch_decode_step(const double* cur, double* nxt, const RangeXform* xf, int out_w, int out_h, int kn,
                        int ranges_x, int ranges_y, double* partial, cudaStream_t st) {
  const long long count = (long long)out_w * out_h;
  const bool covers = (long long)ranges_x * kn == out_w && (long long)ranges_y * kn == out_h;
  if (covers && decode_tiled(out_w, out_h, kn) && !std::getenv("FIC_DECODE_FLAT")) {
    decode_tile_kernel<<<(out_w / kTile) * (out_h / kTile), kTileThreads, 0, st>>>(cur, nxt, xf, out_w, kn, ranges_x,
                                                                                   partial);
    return;
  }
  decode_step_kernel<<<decode_blocks(count), kDecodeThreads, 0, st>>>(cur, nxt, xf, out_w, out_h, kn, ranges_x,
                                                                      ranges_y, partial);
}

// `iterations` reductions of `blocks` partials each (consecutive), one block per iteration.
void launch_rmse_finish(const double* partial, int blocks, long long count, double* out, int iterations,
                        cudaStream_t st) {
  rmse_finish_kernel<<<iterations, 1024, 0, st>>>(partial, blocks, count, out);
}

void launch_raster_init(double* r, long long count, int kind, const unsigned char* supplied, cudaStream_t st) {
  raster_init_kernel<<<(int)((count + 255) / 256), 256, 0, st>>>(r, count, kind, supplied);
}

void launch_quantize_raster(const double* r, long long count, unsigned char* out, cudaStream_t st) {
  quantize_raster_kernel<<<(int)((count + 255) / 256), 256, 0, st>>>(r, count, out);
}

}  // namespace ficb
