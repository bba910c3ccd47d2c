/*
 * fic_oracle.c — TEST INFRASTRUCTURE ONLY.  CPU restatement of the reference's
 * encode/decode path (arxiv/paper_1404_0774 `fic`, /root/reference/proj), used as the
 * parity checker by tests/, by __graft_entry__.smoke() and by bench.py's cpu_baseline
 * leg.  The product path (paper_1404_0774_b200/) never links or calls this file.
 *
 * Parity pinning: tests/test_oracle.py checks this restatement against the
 * reference's own known answers (test_encoder.cpp, test_decoder.cpp, test_format.cpp,
 * test_transforms.cpp, test_codebook.cpp) and against the reference library itself,
 * compiled from its sources by oracle/Makefile into oracle/_ref/ (golden vectors
 * under tests/golden/ were produced by tests/golden/make_golden.py from that build).
 *
 * Compile with -ffp-contract=off: the reference builds with it PUBLIC
 * (proj/CMakeLists.txt:29-31) and its residual sums are bit-exact only without FMA.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/fic_b200.h"

/* ------------------------------------------------------------------ mt19937
 * std::mt19937 raw draws (the C++ standard pins them; proj/tests/testimg.hpp:11-12). */
typedef struct {
  uint32_t mt[624];
  int idx;
} mt19937;

static void mt_seed(mt19937* m, uint32_t seed) {
  m->mt[0] = seed;
  for (int i = 1; i < 624; ++i)
    m->mt[i] = 1812433253u * (m->mt[i - 1] ^ (m->mt[i - 1] >> 30)) + (uint32_t)i;
  m->idx = 624;
}

static uint32_t mt_next(mt19937* m) {
  if (m->idx >= 624) {
    for (int i = 0; i < 624; ++i) {
      uint32_t y = (m->mt[i] & 0x80000000u) | (m->mt[(i + 1) % 624] & 0x7fffffffu);
      uint32_t v = m->mt[(i + 397) % 624] ^ (y >> 1);
      if (y & 1u) v ^= 0x9908b0dfu;
      m->mt[i] = v;
    }
    m->idx = 0;
  }
  uint32_t y = m->mt[m->idx++];
  y ^= y >> 11;
  y ^= (y << 7) & 0x9d2c5680u;
  y ^= (y << 15) & 0xefc60000u;
  y ^= y >> 18;
  return y;
}

void oracle_mt19937(uint32_t seed, int64_t count, uint32_t* out) {
  mt19937 m;
  mt_seed(&m, seed);
  for (int64_t i = 0; i < count; ++i) out[i] = mt_next(&m);
}

/* noise_image (proj/tests/testimg.hpp:13-21). */
void oracle_noise_image(int side, uint32_t seed, uint8_t* out) {
  mt19937 m;
  mt_seed(&m, seed);
  for (int64_t i = 0; i < (int64_t)side * side; ++i) out[i] = (uint8_t)(mt_next(&m) & 0xffu);
}

/* smooth_image (proj/tests/testimg.hpp:26-59). */
void oracle_smooth_image(int side, uint32_t seed, uint8_t* out) {
  mt19937 m;
  mt_seed(&m, seed);
  double fx[4], fy[4], ph[4], amp[4];
  for (int b = 0; b < 4; ++b) {
    fx[b] = 1.0 + (double)mt_next(&m) / 4294967296.0 * 3.0;
    fy[b] = 1.0 + (double)mt_next(&m) / 4294967296.0 * 3.0;
    ph[b] = (double)mt_next(&m) / 4294967296.0 * 6.283185307179586;
    amp[b] = 20.0 + (double)mt_next(&m) / 4294967296.0 * 25.0;
  }
  const double gx = (double)mt_next(&m) / 4294967296.0 * 60.0 - 30.0;
  const double gy = (double)mt_next(&m) / 4294967296.0 * 60.0 - 30.0;
  for (int y = 0; y < side; ++y) {
    for (int x = 0; x < side; ++x) {
      const double u = (double)x / side;
      const double v = (double)y / side;
      double z = 128.0 + gx * (u - 0.5) + gy * (v - 0.5);
      for (int b = 0; b < 4; ++b) z += amp[b] * cos(6.283185307179586 * (fx[b] * u + fy[b] * v) + ph[b]);
      const double c = z < 0.0 ? 0.0 : (z > 255.0 ? 255.0 : z);
      out[(int64_t)y * side + x] = (uint8_t)lround(c);
    }
  }
}

/* ------------------------------------------------------------------ params
 * CodecParams::normalized (proj/src/params.cpp:9-23). */
static int is_pow2(unsigned v) { return v != 0 && (v & (v - 1)) == 0; }

int32_t oracle_normalize_params(const fic_params* in, fic_params* out) {
  fic_params p = *in;
  if (p.n < 2 || !is_pow2((unsigned)p.n)) return FIC_ERR_BAD_PARAMS;
  if (p.step == 0) p.step = p.n;
  if (p.step < 1) return FIC_ERR_BAD_PARAMS;
  if (p.s_bits < 1 || p.s_bits > 16) return FIC_ERR_BAD_PARAMS;
  if (p.o_bits < 1 || p.o_bits > 16) return FIC_ERR_BAD_PARAMS;
  if (!(p.s_max > 0.0)) return FIC_ERR_BAD_PARAMS;
  if (p.s_max > 65.535) return FIC_ERR_BAD_PARAMS;
  p.s_max = (double)lround(p.s_max * 1000.0) / 1000.0;
  if (!(p.s_max > 0.0)) return FIC_ERR_BAD_PARAMS;
  if (p.shadow_eps < 0.0) return FIC_ERR_BAD_PARAMS;
  *out = p;
  return FIC_OK;
}

/* validate_geometry (proj/src/image.cpp:138-149). */
int32_t oracle_validate_geometry(int w, int h, const fic_params* p) {
  if (w != h) return FIC_ERR_NOT_SQUARE;
  if (w <= 0 || !is_pow2((unsigned)w)) return FIC_ERR_NOT_POWER_OF_TWO;
  if (w % p->n != 0) return FIC_ERR_INDIVISIBLE_BY_RANGE;
  if (w < 2 * p->n) return FIC_ERR_TOO_SMALL_FOR_DOMAIN;
  return FIC_OK;
}

/* ------------------------------------------------------------------ quantiser
 * UniformQuantizer (proj/include/fic/format.hpp:17-49). */
uint32_t oracle_quantize(double v, double maxv, int bits) {
  const uint32_t mc = (1u << bits) - 1u;
  if (v == 0.0) return 0;
  const double m = (double)mc;
  const double scaled = (v + maxv) / (2.0 * maxv) * m;
  const uint32_t code = (uint32_t)(scaled + 0.5);
  return code < 1 ? 1 : (code > mc ? mc : code);
}

double oracle_dequantize(uint32_t code, double maxv, int bits) {
  const uint32_t mc = (1u << bits) - 1u;
  if (code == 0) return 0.0;
  return -maxv + (2.0 * maxv) * ((double)code / (double)mc);
}

static double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

/* ------------------------------------------------------------------ isometries
 * symmetry_source (proj/src/transforms.cpp:13-26): output (r, c) reads source (sr, sc). */
void oracle_symmetry_source(int s, int r, int c, int side, int* sr, int* sc) {
  const int m = side - 1;
  switch (s) {
    case 0: *sr = r; *sc = c; break;
    case 1: *sr = m - c; *sc = r; break;
    case 2: *sr = m - r; *sc = m - c; break;
    case 3: *sr = c; *sc = m - r; break;
    case 4: *sr = r; *sc = m - c; break;
    case 5: *sr = m - r; *sc = c; break;
    case 6: *sr = c; *sc = r; break;
    default: *sr = m - c; *sc = m - r; break;
  }
}

/* ------------------------------------------------------------------ domain pool
 * Per-domain 2x2 group sums and integer moments in canonical order, x outer / y inner
 * (proj/src/codebook.cpp:13-20, proj/src/encoder.cpp:205-222).
 * q: D*N int16 (may be NULL), sq/sqq: D int64, flat: D bytes (den <= 16*eps). */
int64_t oracle_domain_count(int w, const fic_params* p) {
  const int per = (w - 2 * p->n) / p->step + 1;
  return (int64_t)per * per;
}

void oracle_domain_pool(const uint8_t* img, int w, const fic_params* p, int16_t* q, int64_t* sq,
                        int64_t* sqq, uint8_t* flat) {
  const int n = p->n, N = n * n;
  int64_t d = 0;
  for (int x = 0; x + 2 * n <= w; x += p->step) {
    for (int y = 0; y + 2 * n <= w; y += p->step, ++d) {
      int64_t s = 0, ss = 0;
      for (int r = 0; r < n; ++r) {
        const uint8_t* row0 = img + (int64_t)(y + 2 * r) * w + x;
        const uint8_t* row1 = row0 + w;
        for (int c = 0; c < n; ++c) {
          const int v = row0[2 * c] + row0[2 * c + 1] + row1[2 * c] + row1[2 * c + 1];
          if (q) q[d * N + r * n + c] = (int16_t)v;
          s += v;
          ss += (int64_t)v * v;
        }
      }
      const int64_t den = (int64_t)N * ss - s * s;
      if (sq) sq[d] = s;
      if (sqq) sqq[d] = ss;
      if (flat) flat[d] = (double)den <= 16.0 * p->shadow_eps;
    }
  }
}

/* ------------------------------------------------------------------ encoder
 * Restatement of Searcher::search_impl (proj/src/encoder.cpp:159-296) including its
 * pruning stages, plus flat_mapping (encoder.cpp:298-308). */
typedef struct {
  const uint8_t* img;
  int w;
  fic_params p;
  int n, N;
  int64_t D;
  int* perm;     /* 8*N: perm[s*N + i] = source index of output cell i */
  int* inv_perm; /* 8*N */
  int16_t* q;    /* D*N pool */
  int64_t* sq;
  int64_t* sqq;
  uint8_t* flat;
  int* pos_x;
  int* pos_y;
} searcher;

static int searcher_init(searcher* S, const uint8_t* img, int w, const fic_params* p) {
  memset(S, 0, sizeof *S);
  S->img = img;
  S->w = w;
  S->p = *p;
  S->n = p->n;
  S->N = p->n * p->n;
  S->D = oracle_domain_count(w, p);
  const int N = S->N, n = S->n;
  S->perm = (int*)malloc(sizeof(int) * 8 * N);
  S->inv_perm = (int*)malloc(sizeof(int) * 8 * N);
  S->q = (int16_t*)malloc(sizeof(int16_t) * (size_t)S->D * N);
  S->sq = (int64_t*)malloc(sizeof(int64_t) * (size_t)S->D);
  S->sqq = (int64_t*)malloc(sizeof(int64_t) * (size_t)S->D);
  S->flat = (uint8_t*)malloc((size_t)S->D);
  S->pos_x = (int*)malloc(sizeof(int) * (size_t)S->D);
  S->pos_y = (int*)malloc(sizeof(int) * (size_t)S->D);
  if (!S->perm || !S->inv_perm || !S->q || !S->sq || !S->sqq || !S->flat || !S->pos_x || !S->pos_y)
    return FIC_ERR_INTERNAL;
  for (int s = 0; s < 8; ++s) {
    for (int r = 0; r < n; ++r)
      for (int c = 0; c < n; ++c) {
        int sr, sc;
        oracle_symmetry_source(s, r, c, n, &sr, &sc);
        S->perm[s * N + r * n + c] = sr * n + sc;
      }
    for (int i = 0; i < N; ++i) S->inv_perm[s * N + S->perm[s * N + i]] = i;
  }
  int64_t d = 0;
  for (int x = 0; x + 2 * n <= w; x += p->step)
    for (int y = 0; y + 2 * n <= w; y += p->step, ++d) {
      S->pos_x[d] = x;
      S->pos_y[d] = y;
    }
  oracle_domain_pool(img, w, p, S->q, S->sq, S->sqq, S->flat);
  return FIC_OK;
}

static void searcher_free(searcher* S) {
  free(S->perm);
  free(S->inv_perm);
  free(S->q);
  free(S->sq);
  free(S->sqq);
  free(S->flat);
  free(S->pos_x);
  free(S->pos_y);
}

static void flat_mapping(const searcher* S, const int* rb, int64_t sum_b, fic_mapping* out) {
  const double count_d = (double)S->N;
  const double o = (double)sum_b / count_d;
  const uint32_t qo = oracle_quantize(o, 255.0, S->p.o_bits);
  const double o_deq = oracle_dequantize(qo, 255.0, S->p.o_bits);
  double r = 0.0;
  for (int i = 0; i < S->N; ++i) {
    const double d = o_deq - (double)rb[i];
    r += d * d;
  }
  memset(out, 0, sizeof *out);
  out->qo = qo;
  out->residual = r;
}

static void search_range(const searcher* S, int x0, int y0, fic_mapping* out, fic_stats* st,
                         int brute) {
  const int n = S->n, N = S->N, w = S->w;
  const fic_params* p = &S->p;
  int rb[4096 * 4];
  int* rbuf = N <= 4096 * 4 ? rb : (int*)malloc(sizeof(int) * N);
  int64_t sum_b = 0, sum_bb = 0;
  for (int r = 0; r < n; ++r)
    for (int c = 0; c < n; ++c) {
      const int v = S->img[(int64_t)(y0 + r) * w + x0 + c];
      rbuf[r * n + c] = v;
      sum_b += v;
      sum_bb += (int64_t)v * v;
    }
  const int64_t range_var = (int64_t)N * sum_bb - sum_b * sum_b;
  if ((double)range_var <= p->shadow_eps) {
    st->shadow_ranges += 1;
    flat_mapping(S, rbuf, sum_b, out);
    if (rbuf != rb) free(rbuf);
    return;
  }
  const double count_d = (double)N;
  const double inv_count = 1.0 / count_d;
  const double ssb = (double)range_var / count_d;
  const double sb_d = (double)sum_b;
  const double smax = p->s_max;
  double best_r = INFINITY;
  int found = 0;
  fic_mapping best;
  memset(&best, 0, sizeof best);
  double gate = -INFINITY;
  for (int64_t d = 0; d < S->D; ++d) {
    const int16_t* q = S->q + d * N;
    const int64_t sum_q = S->sq[d];
    const int64_t den_q = (int64_t)N * S->sqq[d] - sum_q * sum_q;
    if (S->flat[d]) {
      st->shadow_codeblocks += 8;
      continue;
    }
    const double den_d = (double)den_q;
    const double sa_d = (double)sum_q * 0.25;
    const int64_t sqsb = sum_q * sum_b;
    double gate_den = gate * den_d;
    st->candidates_tested += 8;
    for (int s = 0; s < 8; ++s) {
      const int* pm = S->perm + s * N;
      int64_t acc = 0;
      for (int i = 0; i < N; ++i) acc += (int64_t)q[pm[i]] * rbuf[i];
      const int64_t num_q = (int64_t)N * acc - sqsb;
      const double num_d = (double)num_q;
      if (!brute && num_d * num_d <= gate_den) continue; /* encoder.cpp:246 */
      const double s_raw = 4.0 * num_d / den_d;
      const double sc = clampd(s_raw, -smax, smax);
      const uint32_t qs = oracle_quantize(sc, smax, p->s_bits);
      const double s_deq = oracle_dequantize(qs, smax, p->s_bits);
      const double cov = num_d * 0.25 * inv_count;
      const double var_a = den_d * 0.0625 * inv_count;
      const double parabola = ssb - 2.0 * s_deq * cov + s_deq * s_deq * var_a;
      if (!brute && parabola >= best_r + 1e-3) continue; /* encoder.cpp:263 */
      const double o = clampd((sb_d - sc * sa_d) * inv_count, -255.0, 255.0);
      const uint32_t qo = oracle_quantize(o, 255.0, p->o_bits);
      const double o_deq = oracle_dequantize(qo, 255.0, p->o_bits);
      const double o_gap = o_deq - (sb_d - s_deq * sa_d) * inv_count;
      const double screen = parabola + count_d * o_gap * o_gap;
      if (!brute && screen >= best_r + 1e-3) continue; /* encoder.cpp:272 */
      double r_val = 0.0;
      for (int i = 0; i < N; ++i) {
        const double ai = (double)q[pm[i]] * 0.25;
        const double dd = s_deq * ai + o_deq - (double)rbuf[i];
        r_val += dd * dd;
      }
      if (r_val < best_r) {
        best_r = r_val;
        best.x = S->pos_x[d];
        best.y = S->pos_y[d];
        best.sym = s;
        best.qs = qs;
        best.qo = qo;
        best.reserved = 0;
        best.residual = r_val;
        found = 1;
        gate = ssb - best_r;
        gate_den = gate * den_d;
      }
    }
  }
  if (!found)
    flat_mapping(S, rbuf, sum_b, out);
  else
    *out = best;
  if (rbuf != rb) free(rbuf);
}

static int32_t check_encode_args(const uint8_t* img, int w, int h, const fic_params* in,
                                 fic_params* p) {
  if (!img || !in) return FIC_ERR_BAD_PARAMS;
  int32_t e = oracle_normalize_params(in, p);
  if (e) return e;
  return oracle_validate_geometry(w, h, p);
}

/* encode_sequential (proj/src/encoder.cpp:344-366); brute != 0 disables the three pruning
 * stages (an exhaustive scan, the structure of proj/tests/oracle.hpp:102-138). */
int32_t oracle_encode(const uint8_t* img, int w, int h, const fic_params* params, int brute,
                      fic_mapping* out, fic_stats* stats) {
  fic_params p;
  int32_t e = check_encode_args(img, w, h, params, &p);
  if (e) return e;
  searcher S;
  if ((e = searcher_init(&S, img, w, &p))) {
    searcher_free(&S);
    return e;
  }
  fic_stats st = {0, 0, 0};
  const int R = w / p.n;
  for (int ry = 0; ry < R; ++ry)
    for (int rx = 0; rx < R; ++rx) search_range(&S, rx * p.n, ry * p.n, out + (int64_t)ry * R + rx, &st, brute);
  searcher_free(&S);
  if (stats) *stats = st;
  return FIC_OK;
}

/* encode_range (proj/src/encoder.cpp:332-342) without the per-call Searcher rebuild cost
 * mattering: used for sampled parity on large configurations. */
int32_t oracle_encode_ranges(const uint8_t* img, int w, int h, const fic_params* params,
                             int count, const int32_t* xs, const int32_t* ys, fic_mapping* out,
                             fic_stats* stats) {
  fic_params p;
  int32_t e = check_encode_args(img, w, h, params, &p);
  if (e) return e;
  for (int i = 0; i < count; ++i) /* check_range_origin, encoder.cpp:323-328 */
    if (xs[i] % p.n || ys[i] % p.n || xs[i] < 0 || ys[i] < 0 || xs[i] + p.n > w || ys[i] + p.n > h)
      return FIC_ERR_GEOMETRY;
  searcher S;
  if ((e = searcher_init(&S, img, w, &p))) {
    searcher_free(&S);
    return e;
  }
  fic_stats st = {0, 0, 0};
  for (int i = 0; i < count; ++i) search_range(&S, xs[i], ys[i], out + i, &st, 0);
  searcher_free(&S);
  if (stats) *stats = st;
  return FIC_OK;
}

/* ------------------------------------------------------------------ decoder
 * decode_step (proj/src/decoder.cpp:39-79). */
int32_t oracle_decode_step(const double* cur, const fic_mapping* maps, int w, const fic_params* params,
                           int scale, double* next) {
  fic_params p;
  int32_t e = oracle_normalize_params(params, &p);
  if (e) return e;
  if (scale < 1) return FIC_ERR_BAD_PARAMS;
  const int out_w = w * scale;
  const int kn = p.n * scale;
  const int R = w / p.n;
  for (int ry = 0; ry < R; ++ry)
    for (int rx = 0; rx < R; ++rx) {
      const fic_mapping* m = maps + (int64_t)ry * R + rx;
      const double s = oracle_dequantize(m->qs, p.s_max, p.s_bits);
      const double o = oracle_dequantize(m->qo, 255.0, p.o_bits);
      const int dx = m->x * scale, dy = m->y * scale;
      for (int r = 0; r < kn; ++r) {
        double* orow = next + (int64_t)(ry * kn + r) * out_w + (int64_t)rx * kn;
        for (int c = 0; c < kn; ++c) {
          int sr, sc;
          oracle_symmetry_source(m->sym, r, c, kn, &sr, &sc);
          const double* row0 = cur + (int64_t)(dy + 2 * sr) * out_w + dx;
          const double* row1 = row0 + out_w;
          const double z = (row0[2 * sc] + row0[2 * sc + 1] + row1[2 * sc] + row1[2 * sc + 1]) / 4.0;
          orow[c] = s * z + o;
        }
      }
    }
  return FIC_OK;
}

/* raster_rmse (proj/src/decoder.cpp:28-37). */
double oracle_raster_rmse(const double* a, const double* b, int64_t count) {
  double acc = 0.0;
  for (int64_t i = 0; i < count; ++i) {
    const double d = a[i] - b[i];
    acc += d * d;
  }
  return sqrt(acc / (double)count);
}

/* decode_traced (proj/src/decoder.cpp:83-128). */
int32_t oracle_decode(const fic_mapping* maps, int w, const fic_params* params, int scale,
                      int iterations, int initial_kind, const uint8_t* supplied, int has_eps,
                      double eps, uint8_t* out, double* step_rmse, int32_t* iterations_run) {
  if (scale < 1 || iterations < 1) return FIC_ERR_BAD_PARAMS;
  const int out_w = w * scale;
  const int64_t cnt = (int64_t)out_w * out_w;
  double* cur = (double*)malloc(sizeof(double) * cnt);
  double* nxt = (double*)malloc(sizeof(double) * cnt);
  if (!cur || !nxt) {
    free(cur);
    free(nxt);
    return FIC_ERR_INTERNAL;
  }
  for (int64_t i = 0; i < cnt; ++i)
    cur[i] = initial_kind == 0 ? 128.0 : (initial_kind == 1 ? 0.0 : (double)supplied[i]);
  int runs = 0;
  for (int it = 0; it < iterations; ++it) {
    int32_t e = oracle_decode_step(cur, maps, w, params, scale, nxt);
    if (e) {
      free(cur);
      free(nxt);
      return e;
    }
    const double r = oracle_raster_rmse(cur, nxt, cnt);
    if (step_rmse) step_rmse[it] = r;
    double* t = cur;
    cur = nxt;
    nxt = t;
    ++runs;
    if (has_eps && r < eps) break;
  }
  for (int64_t i = 0; i < cnt; ++i) out[i] = (uint8_t)lround(clampd(cur[i], 0.0, 255.0));
  if (iterations_run) *iterations_run = runs;
  free(cur);
  free(nxt);
  return FIC_OK;
}

/* collage_error (proj/src/decoder.cpp:134-140). */
int32_t oracle_collage_error(const uint8_t* img, const fic_mapping* maps, int w, const fic_params* params,
                             double* out) {
  const int64_t cnt = (int64_t)w * w;
  double* a = (double*)malloc(sizeof(double) * cnt);
  double* b = (double*)malloc(sizeof(double) * cnt);
  for (int64_t i = 0; i < cnt; ++i) a[i] = img[i];
  int32_t e = oracle_decode_step(a, maps, w, params, 1, b);
  if (!e) *out = oracle_raster_rmse(a, b, cnt);
  free(a);
  free(b);
  return e;
}

/* rmse / psnr (proj/src/metrics.cpp:8-23). */
double oracle_rmse(const uint8_t* a, const uint8_t* b, int64_t count) {
  int64_t acc = 0;
  for (int64_t i = 0; i < count; ++i) {
    const int d = (int)a[i] - (int)b[i];
    acc += (int64_t)d * d;
  }
  return sqrt((double)acc / (double)count);
}

double oracle_psnr(const uint8_t* a, const uint8_t* b, int64_t count) {
  const double e = oracle_rmse(a, b, count);
  if (e == 0.0) return INFINITY;
  return 20.0 * log10(255.0 / e);
}
