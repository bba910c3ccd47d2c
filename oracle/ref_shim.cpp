// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.  A C shim over the UNMODIFIED reference
// library (/root/reference/proj/src/*.cpp, compiled from where the sources lie by
// oracle/Makefile into oracle/_ref/libfic_ref.so).  It lets tests and bench.py's
// reference arm call the reference's own encode/decode entry points through ctypes.
// Nothing here is on the product path.
#include <cstring>
#include <optional>
#include <string>
#include <thread>
#include <vector>

#include "fic/decoder.hpp"
#include "fic/encoder.hpp"
#include "fic/format.hpp"
#include "fic/metrics.hpp"
#include "oracle.hpp"   // proj/tests/oracle.hpp (reference brute force)
#include "testimg.hpp"  // proj/tests/testimg.hpp (reference fixtures)

#include "../include/fic_b200.h"

namespace {

thread_local std::string g_err;

fic::CodecParams to_params(const fic_params* p) {
  fic::CodecParams c;
  c.n = p->n;
  c.step = p->step;
  c.s_bits = p->s_bits;
  c.o_bits = p->o_bits;
  c.s_max = p->s_max;
  c.shadow_eps = p->shadow_eps;
  return c;
}

fic::GrayImage to_image(const uint8_t* img, int w, int h) {
  fic::GrayImage g;
  g.width = w;
  g.height = h;
  g.data.assign(img, img + static_cast<size_t>(w) * h);
  return g;
}

void put(const fic::RangeMapping& m, fic_mapping* o) {
  o->x = m.domain.x;
  o->y = m.domain.y;
  o->sym = static_cast<int32_t>(m.symmetry);
  o->qs = m.qs;
  o->qo = m.qo;
  o->reserved = 0;
  o->residual = m.residual;
}

fic::RangeMapping get(const fic_mapping& o) {
  fic::RangeMapping m;
  m.domain = {o.x, o.y};
  m.symmetry = static_cast<fic::Symmetry>(o.sym);
  m.qs = o.qs;
  m.qo = o.qo;
  m.residual = o.residual;
  return m;
}

fic::EncodedImage to_encoded(const fic_mapping* maps, int w, int h, const fic_params* p) {
  fic::EncodedImage e;
  e.width = w;
  e.height = h;
  e.params = to_params(p).normalized();
  e.mappings.resize(e.range_count());
  for (size_t i = 0; i < e.mappings.size(); ++i) e.mappings[i] = get(maps[i]);
  return e;
}

template <class F>
int32_t guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const fic::CodecError& e) {
    g_err = e.what();
    return static_cast<int32_t>(e.code()) + 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 101;
  }
}

void put_stats(const fic::EncodeStats& s, fic_stats* o) {
  if (!o) return;
  o->candidates_tested = s.candidates_tested;
  o->shadow_ranges = s.shadow_ranges;
  o->shadow_codeblocks = s.shadow_codeblocks;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int32_t ref_hardware_concurrency() { return static_cast<int32_t>(std::thread::hardware_concurrency()); }

int32_t ref_encode(const uint8_t* img, int32_t w, int32_t h, const fic_params* p, int32_t workers,
                   int32_t chunk_w, int32_t chunk_h, fic_mapping* out, fic_stats* stats) {
  return guard([&] {
    const fic::GrayImage g = to_image(img, w, h);
    fic::EncodeStats st;
    const fic::EncodedImage e =
        workers > 1 ? fic::encode_parallel(g, to_params(p), workers, {chunk_w, chunk_h}, &st)
                    : fic::encode_sequential(g, to_params(p), &st);
    for (size_t i = 0; i < e.mappings.size(); ++i) put(e.mappings[i], out + i);
    put_stats(st, stats);
  });
}

int32_t ref_encode_range(const uint8_t* img, int32_t w, int32_t h, int32_t x, int32_t y,
                         const fic_params* p, fic_mapping* out, fic_stats* stats) {
  return guard([&] {
    fic::EncodeStats st;
    put(fic::encode_range(to_image(img, w, h), x, y, to_params(p), &st), out);
    put_stats(st, stats);
  });
}

// The reference's exhaustive brute force (proj/tests/oracle.hpp:102-138).
int32_t ref_oracle_encode(const uint8_t* img, int32_t w, int32_t h, const fic_params* p,
                          fic_mapping* out) {
  return guard([&] {
    const auto r = fic::testing::oracle_encode(to_image(img, w, h), to_params(p));
    for (size_t i = 0; i < r.size(); ++i) {
      const auto& c = r[i].best;
      out[i].x = c.domain.x;
      out[i].y = c.domain.y;
      out[i].sym = static_cast<int32_t>(c.symmetry);
      out[i].qs = c.qs;
      out[i].qo = c.qo;
      out[i].reserved = 0;
      out[i].residual = c.residual;
    }
  });
}

int32_t ref_decode_step(const double* cur, const fic_mapping* maps, int32_t w, int32_t h,
                        const fic_params* p, int32_t scale, double* next) {
  return guard([&] {
    const fic::EncodedImage e = to_encoded(maps, w, h, p);
    fic::RealRaster r;
    r.width = w * scale;
    r.height = h * scale;
    r.v.assign(cur, cur + static_cast<size_t>(r.width) * r.height);
    const fic::RealRaster o = fic::decode_step(r, e, scale);
    std::memcpy(next, o.v.data(), o.v.size() * sizeof(double));
  });
}

int32_t ref_decode(const fic_mapping* maps, int32_t w, int32_t h, const fic_params* p, int32_t scale,
                   int32_t iterations, int32_t initial_kind, const uint8_t* supplied, int32_t has_eps,
                   double eps, uint8_t* out, double* step_rmse, int32_t* iterations_run) {
  return guard([&] {
    const fic::EncodedImage e = to_encoded(maps, w, h, p);
    fic::DecodeParams dp;
    dp.scale = scale;
    dp.iterations = iterations;
    dp.initial = initial_kind == 0 ? fic::InitialRaster::MidGray
                                   : (initial_kind == 1 ? fic::InitialRaster::Black
                                                        : fic::InitialRaster::Supplied);
    fic::GrayImage sup;
    if (initial_kind == 2) {
      sup = to_image(supplied, w * scale, h * scale);
      dp.supplied = &sup;
    }
    if (has_eps) dp.convergence_eps = eps;
    const fic::DecodeResult r = fic::decode_traced(e, dp);
    std::memcpy(out, r.image.data.data(), r.image.data.size());
    if (step_rmse)
      for (size_t i = 0; i < r.step_rmse.size(); ++i) step_rmse[i] = r.step_rmse[i];
    if (iterations_run) *iterations_run = r.iterations_run;
  });
}

int32_t ref_collage_error(const uint8_t* img, const fic_mapping* maps, int32_t w, int32_t h,
                          const fic_params* p, double* out) {
  return guard([&] { *out = fic::collage_error(to_image(img, w, h), to_encoded(maps, w, h, p)); });
}

// FIC1 container (proj/src/format.cpp:105-185): returns the byte count; copies into
// `buf` when it is large enough.
int64_t ref_serialize(const fic_mapping* maps, int32_t w, int32_t h, const fic_params* p, uint8_t* buf,
                      int64_t cap) {
  int64_t n = -1;
  const int32_t rc = guard([&] {
    const auto bytes = fic::serialize(to_encoded(maps, w, h, p));
    n = static_cast<int64_t>(bytes.size());
    if (buf && cap >= n) std::memcpy(buf, bytes.data(), bytes.size());
  });
  return rc ? -static_cast<int64_t>(rc) : n;
}

// The public per-candidate fit pipeline (proj/src/encoder.cpp:60-102).  kind 0:
// least_squares_fit(shadow_eps), 1: least_squares_clamped, 2: least_squares; out = {s, o,
// residual, qs, qo}.
int32_t ref_least_squares(int32_t kind, const double* a, int32_t side_a, const double* b, int32_t side_b,
                          const fic_params* p, double shadow_eps, double* out) {
  return guard([&] {
    const fic::Block A(side_a, std::vector<double>(a, a + static_cast<size_t>(side_a) * side_a));
    const fic::Block B(side_b, std::vector<double>(b, b + static_cast<size_t>(side_b) * side_b));
    if (kind == 2) {
      const fic::QuantizedFit q = fic::least_squares(A, B, to_params(p));
      out[0] = q.s, out[1] = q.o, out[2] = q.residual, out[3] = q.qs, out[4] = q.qo;
    } else {
      const fic::LinearFit f =
          kind == 0 ? fic::least_squares_fit(A, B, shadow_eps) : fic::least_squares_clamped(A, B, to_params(p));
      out[0] = f.s, out[1] = f.o, out[2] = f.residual, out[3] = out[4] = 0;
    }
  });
}

int32_t ref_is_shadow(const double* b, int32_t side, double eps) {
  return fic::is_shadow(fic::Block(side, std::vector<double>(b, b + static_cast<size_t>(side) * side)), eps) ? 1 : 0;
}

void ref_noise_image(int32_t side, uint32_t seed, uint8_t* out) {
  const auto g = fic::testing::noise_image(side, seed);
  std::memcpy(out, g.data.data(), g.data.size());
}

void ref_smooth_image(int32_t side, uint32_t seed, uint8_t* out) {
  const auto g = fic::testing::smooth_image(side, seed);
  std::memcpy(out, g.data.data(), g.data.size());
}

double ref_psnr(const uint8_t* a, const uint8_t* b, int32_t w, int32_t h) {
  return fic::psnr(to_image(a, w, h), to_image(b, w, h));
}

}  // extern "C"
