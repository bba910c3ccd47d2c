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
                   int out_w, int kn, int ranges_x, double* __restrict__ partial) {
  const long long idx = (long long)blockIdx.x * kDecodeThreads + threadIdx.x;
  const long long total = (long long)out_w * out_w;
  double sq = 0.0;
  if (idx < total) {
    const int Y = (int)(idx / out_w), X = (int)(idx % out_w);
    const int ry = Y / kn, rx = X / kn;
    const int r = Y - ry * kn, c = X - rx * kn;
    const RangeXform t = xf[ry * ranges_x + rx];
    int sr, sc;
    symmetry_source(t.sym, r, c, kn, sr, sc);
    const double* row0 = cur + (long long)(t.dy + 2 * sr) * out_w + t.dx + 2 * sc;
    const double* row1 = row0 + out_w;
    // ((p00 + p01) + p10 + p11) / 4.0 then s*z + o, each op rounded (decoder.cpp:71-75); the
    // division by 4 is an exact power-of-two scaling, identical to the multiplication by 0.25
    const double z = __dmul_rn(__dadd_rn(__dadd_rn(__dadd_rn(__ldg(row0), __ldg(row0 + 1)), __ldg(row1)), __ldg(row1 + 1)),
                               0.25);
    const double v = __dadd_rn(__dmul_rn(t.s, z), t.o);
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

// Sums the per-block partials in index order and writes rmse = sqrt(sum / count).
__global__ void rmse_finish_kernel(const double* __restrict__ partial, int blocks, long long count,
                                   double* __restrict__ out) {
  __shared__ double red[1024];
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
int decode_partials(int out_w, int kn) {
  (void)kn;
  return decode_blocks((long long)out_w * out_w);
}

void launch_xform(const fic_mapping* maps, int count, int scale, const Geometry& g, RangeXform* xf, cudaStream_t st) {
  xform_kernel<<<(count + 255) / 256, 256, 0, st>>>(maps, count, scale, g.s_bits, g.s_max, g.o_bits, xf);
}

void launch_decode_step(const double* cur, double* nxt, const RangeXform* xf, int out_w, int kn, int ranges_x,
                        double* partial, cudaStream_t st) {
  const long long count = (long long)out_w * out_w;
  decode_step_kernel<<<decode_blocks(count), kDecodeThreads, 0, st>>>(cur, nxt, xf, out_w, kn, ranges_x, partial);
}

void launch_rmse_finish(const double* partial, int blocks, long long count, double* out, cudaStream_t st) {
  rmse_finish_kernel<<<1, 1024, 0, st>>>(partial, blocks, count, out);
}

void launch_raster_init(double* r, long long count, int kind, const unsigned char* supplied, cudaStream_t st) {
  raster_init_kernel<<<(int)((count + 255) / 256), 256, 0, st>>>(r, count, kind, supplied);
}

void launch_quantize_raster(const double* r, long long count, unsigned char* out, cudaStream_t st) {
  quantize_raster_kernel<<<(int)((count + 255) / 256), 256, 0, st>>>(r, count, out);
}

}  // namespace ficb
