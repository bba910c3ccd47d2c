// encoder_b200.cpp — the reference's encoder API (proj/include/fic/encoder.hpp) with its
// bodies swapped for the B200 C-ABI (include/fic_b200.h, libfic_b200.so).
//
// This is the "keep the signatures, swap the bodies" binding of INTEGRATION.md §2, compiled
// for real by integration/Makefile in place of proj/src/encoder.cpp: the reference's own
// pybind module (proj/python/bindings/module.cpp) and every other caller link against it
// unchanged.  Each function keeps the reference's validation order and error texts; all
// compute runs on the device behind the C-ABI.
#include <stdexcept>
#include <string>
#include <vector>

#include "fic/encoder.hpp"
#include "fic_b200.h"

namespace fic {
namespace {

fic_params to_c(const CodecParams& p) { return fic_params{p.n, p.step, p.s_bits, p.o_bits, p.s_max, p.shadow_eps}; }

RangeMapping from_c(const fic_mapping& m) {
  return RangeMapping{DomainPosition{m.x, m.y}, static_cast<Symmetry>(m.sym), m.qs, m.qo, m.residual};
}

// C-ABI code -> the reference's CodecError (codes 1..18 are Errc ordinal + 1).
void check(int32_t rc) {
  if (rc == FIC_OK) return;
  if (rc >= 1 && rc <= 18) raise(static_cast<Errc>(rc - 1), fic_last_error());
  throw std::runtime_error(std::string("fic_b200 ") + fic_errc_name(rc) + ": " + fic_last_error());
}

void put_stats(const fic_stats& st, EncodeStats* stats) {
  if (stats) *stats = EncodeStats{st.candidates_tested, st.shadow_ranges, st.shadow_codeblocks};
}

}  // namespace

// is_shadow (encoder.cpp:60-67)
bool is_shadow(const Block& b, double eps) {
  int32_t out = 0;
  check(fic_is_shadow(b.samples.data(), b.side, eps, &out));
  return out != 0;
}

// least_squares_fit (encoder.cpp:69-76)
LinearFit least_squares_fit(const Block& a, const Block& b, double shadow_eps) {
  fic_linear_fit f{};
  check(fic_least_squares_fit(a.samples.data(), a.side, b.samples.data(), b.side, shadow_eps, &f));
  return LinearFit{f.s, f.o, f.residual};
}

// least_squares_clamped (encoder.cpp:78-88)
LinearFit least_squares_clamped(const Block& a, const Block& b, const CodecParams& params) {
  const fic_params p = to_c(params);
  fic_linear_fit f{};
  check(fic_least_squares_clamped(a.samples.data(), a.side, b.samples.data(), b.side, &p, &f));
  return LinearFit{f.s, f.o, f.residual};
}

// least_squares (encoder.cpp:90-102)
QuantizedFit least_squares(const Block& a, const Block& b, const CodecParams& params) {
  const fic_params p = to_c(params);
  fic_quantized_fit f{};
  check(fic_least_squares(a.samples.data(), a.side, b.samples.data(), b.side, &p, &f));
  return QuantizedFit{f.qs, f.qo, f.s, f.o, f.residual};
}

// encode_range (encoder.cpp:332-342)
RangeMapping encode_range(const GrayImage& img, int x, int y, const CodecParams& params, EncodeStats* stats) {
  const fic_params p = to_c(params);
  fic_mapping m{};
  fic_stats st{};
  check(fic_encode_range(img.data.data(), img.width, img.height, x, y, &p, &m, &st));
  put_stats(st, stats);
  return from_c(m);
}

// encode_sequential (encoder.cpp:344-366)
EncodedImage encode_sequential(const GrayImage& img, const CodecParams& params, EncodeStats* stats) {
  const CodecParams p = params.normalized();
  validate_geometry(img, p);
  const fic_params cp = to_c(p);
  std::vector<fic_mapping> out(static_cast<size_t>(img.width / p.n) * (img.height / p.n));
  fic_stats st{};
  check(fic_encode(img.data.data(), img.width, img.height, &cp, out.data(), &st));
  EncodedImage enc{img.width, img.height, p, {}};
  enc.mappings.reserve(out.size());
  for (const fic_mapping& m : out) enc.mappings.push_back(from_c(m));
  put_stats(st, stats);
  return enc;
}

// encode_parallel (encoder.cpp:368-427): same validation; one device call gives the same
// bytes for every worker count and chunk geometry.
EncodedImage encode_parallel(const GrayImage& img, const CodecParams& params, int workers, ChunkGeometry chunk,
                             EncodeStats* stats) {
  const CodecParams p = params.normalized();
  validate_geometry(img, p);
  const fic_params cp = to_c(p);
  std::vector<fic_mapping> out(static_cast<size_t>(img.width / p.n) * (img.height / p.n));
  fic_stats st{};
  check(fic_encode_parallel(img.data.data(), img.width, img.height, &cp, workers, chunk.w, chunk.h, out.data(),
                            &st));
  EncodedImage enc{img.width, img.height, p, {}};
  enc.mappings.reserve(out.size());
  for (const fic_mapping& m : out) enc.mappings.push_back(from_c(m));
  put_stats(st, stats);
  return enc;
}

}  // namespace fic
