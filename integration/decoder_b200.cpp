// decoder_b200.cpp — the reference's decoder API (proj/include/fic/decoder.hpp) with the
// iterated decode, decode_step and collage_error bodies swapped for the B200 C-ABI
// (include/fic_b200.h): compiled by integration/Makefile in place of proj/src/decoder.cpp.
// Validation order and error texts follow proj/src/decoder.cpp:39-146; the small raster
// helpers the header also declares (raster_from_image, constant_raster, raster_rmse) keep
// their host definitions (decoder.cpp:12-37).
#include <cmath>
#include <stdexcept>
#include <string>
#include <vector>

#include "fic/decoder.hpp"
#include "fic_b200.h"

namespace fic {
namespace {

fic_params to_c(const CodecParams& p) { return fic_params{p.n, p.step, p.s_bits, p.o_bits, p.s_max, p.shadow_eps}; }

void check(int32_t rc) {
  if (rc == FIC_OK) return;
  if (rc >= 1 && rc <= 18) raise(static_cast<Errc>(rc - 1), fic_last_error());
  throw std::runtime_error(std::string("fic_b200 ") + fic_errc_name(rc) + ": " + fic_last_error());
}

std::vector<fic_mapping> to_c_maps(const EncodedImage& enc) {
  std::vector<fic_mapping> m(enc.mappings.size());
  for (size_t i = 0; i < m.size(); ++i) {
    const RangeMapping& r = enc.mappings[i];
    m[i] = fic_mapping{r.domain.x, r.domain.y, static_cast<int32_t>(r.symmetry), r.qs, r.qo, 0, r.residual};
  }
  return m;
}

// decode_step's mapping-count check (decoder.cpp:49-50): the C-ABI derives the count from
// the geometry, so the wrapper checks the vector first.
void check_count(const EncodedImage& enc) {
  if (enc.mappings.size() != enc.range_count()) raise(Errc::BadParams, "mapping count does not cover the range grid");
}

}  // namespace

RealRaster raster_from_image(const GrayImage& img) {
  RealRaster r;
  r.width = img.width;
  r.height = img.height;
  r.v.assign(img.data.begin(), img.data.end());
  return r;
}

RealRaster constant_raster(int width, int height, double value) {
  RealRaster r;
  r.width = width;
  r.height = height;
  r.v.assign(static_cast<std::size_t>(width) * height, value);
  return r;
}

double raster_rmse(const RealRaster& a, const RealRaster& b) {
  if (a.width != b.width || a.height != b.height) raise(Errc::DimensionMismatch, "raster geometry differs");
  double acc = 0.0;
  for (std::size_t i = 0; i < a.v.size(); ++i) {
    const double d = a.v[i] - b.v[i];
    acc += d * d;
  }
  return std::sqrt(acc / static_cast<double>(a.v.size()));
}

// decode_step (decoder.cpp:39-79)
RealRaster decode_step(const RealRaster& current, const EncodedImage& enc, int scale) {
  if (scale < 1) raise(Errc::BadParams, "scale must be >= 1");
  const CodecParams p = enc.params.normalized();
  const int out_w = enc.width * scale, out_h = enc.height * scale;
  if (current.width != out_w || current.height != out_h)
    raise(Errc::ScaleMismatch, "raster is " + std::to_string(current.width) + "x" + std::to_string(current.height) +
                                   ", expected " + std::to_string(out_w) + "x" + std::to_string(out_h));
  check_count(enc);
  const fic_params cp = to_c(p);
  const std::vector<fic_mapping> maps = to_c_maps(enc);
  RealRaster next;
  next.width = out_w;
  next.height = out_h;
  next.v.resize(current.v.size());
  check(fic_decode_step(current.v.data(), current.width, current.height, maps.data(), enc.width, enc.height, &cp,
                        scale, next.v.data()));
  return next;
}

// decode_traced (decoder.cpp:113-128)
DecodeResult decode_traced(const EncodedImage& enc, const DecodeParams& params) {
  if (params.scale < 1) raise(Errc::BadParams, "scale must be >= 1");
  if (params.iterations < 1) raise(Errc::BadParams, "iterations must be >= 1");
  const int out_w = enc.width * params.scale, out_h = enc.height * params.scale;
  int kind = FIC_INITIAL_MID_GRAY;
  const uint8_t* sup = nullptr;
  int sw = 0, sh = 0;
  switch (params.initial) {  // initial_raster (decoder.cpp:83-97)
    case InitialRaster::MidGray: kind = FIC_INITIAL_MID_GRAY; break;
    case InitialRaster::Black: kind = FIC_INITIAL_BLACK; break;
    case InitialRaster::Supplied:
      if (params.supplied == nullptr) raise(Errc::BadParams, "no supplied initial image");
      if (params.supplied->width != out_w || params.supplied->height != out_h)
        raise(Errc::ScaleMismatch, "supplied initial image has the wrong geometry");
      kind = FIC_INITIAL_SUPPLIED;
      sup = params.supplied->data.data();
      sw = params.supplied->width;
      sh = params.supplied->height;
      break;
  }
  const CodecParams p = enc.params.normalized();
  check_count(enc);
  const fic_params cp = to_c(p);
  const std::vector<fic_mapping> maps = to_c_maps(enc);
  DecodeResult result;
  result.image.width = out_w;
  result.image.height = out_h;
  result.image.data.resize(static_cast<std::size_t>(out_w) * out_h);
  std::vector<double> rmse(static_cast<std::size_t>(params.iterations));
  int32_t runs = 0;
  check(fic_decode(maps.data(), enc.width, enc.height, &cp, params.scale, params.iterations, kind, sup, sw, sh,
                   params.convergence_eps ? 1 : 0, params.convergence_eps.value_or(0.0), result.image.data.data(),
                   rmse.data(), &runs));
  result.iterations_run = runs;
  result.step_rmse.assign(rmse.begin(), rmse.begin() + runs);
  return result;
}

GrayImage decode(const EncodedImage& enc, const DecodeParams& params) { return decode_traced(enc, params).image; }

// collage_error (decoder.cpp:134-140)
double collage_error(const GrayImage& img, const EncodedImage& enc) {
  if (img.width != enc.width || img.height != enc.height)
    raise(Errc::DimensionMismatch, "image does not match the encoding's geometry");
  const CodecParams p = enc.params.normalized();
  check_count(enc);
  const fic_params cp = to_c(p);
  const std::vector<fic_mapping> maps = to_c_maps(enc);
  double out = 0.0;
  check(fic_collage_error(img.data.data(), img.width, img.height, maps.data(), enc.width, enc.height, &cp, &out));
  return out;
}

// decoded_error_bound (decoder.cpp:142-146)
double decoded_error_bound(double collage_rmse, double s_max) {
  double out = 0.0;
  check(fic_decoded_error_bound(collage_rmse, s_max, &out));
  return out;
}

}  // namespace fic
