// fit.cu — the reference's public per-candidate fit pipeline behind the
// C-ABI: is_shadow, least_squares_fit, least_squares_clamped and least_squares
// (proj/src/encoder.cpp:60-102, declared at proj/include/fic/encoder.hpp:32-45).
//
// These are single-candidate host helpers (the reference checks its search against them,
// proj/tests/test_encoder.cpp:15-60,169-202); the encoder's own evaluation of the same
// arithmetic runs on the device (scan.cu: eval_exact / eval_fast).  Host fp64 in the
// reference's operation order; the library's host code is compiled with
// -ffp-contract=off like the reference (proj/CMakeLists.txt:29-31), so no FMA contraction.
#include <algorithm>
#include <cmath>
#include <string>
#include <utility>

#include "common.cuh"

namespace ficb {
int32_t api_fail(int32_t code, const std::string& detail);  // fic_api.cu: sets fic_last_error()
}

namespace {

int32_t fit_fail(int32_t code, const std::string& detail) { return ficb::api_fail(code, detail); }

// FitSums / gather_sums (encoder.cpp:22-44): sums in index order.
struct FitSums {
  double n, sa, sb, saa, sab, den, num;
};

FitSums gather(const double* a, const double* b, long count) {
  FitSums f{};
  f.n = (double)count;
  for (long i = 0; i < count; ++i) {
    const double av = a[i];
    const double bv = b[i];
    f.sa += av;
    f.sb += bv;
    f.saa += av * av;
    f.sab += av * bv;
  }
  f.den = f.n * f.saa - f.sa * f.sa;
  f.num = f.n * f.sab - f.sa * f.sb;
  return f;
}

// score_residual (encoder.cpp:49-56): term by term in index order.
double score(const double* a, const double* b, long count, double s, double o) {
  double r = 0.0;
  for (long i = 0; i < count; ++i) {
    const double d = s * a[i] + o - b[i];
    r += d * d;
  }
  return r;
}

int32_t check_blocks(const double* a, int32_t side_a, const double* b, int32_t side_b) {
  if (side_a != side_b)  // gather_sums (encoder.cpp:30-31)
    return fit_fail(FIC_ERR_SIDE_MISMATCH, std::to_string(side_a) + " vs " + std::to_string(side_b));
  if (side_a < 0) return fit_fail(FIC_ERR_BAD_PARAMS, "negative block side");
  if (side_a > 0 && (!a || !b)) return fit_fail(FIC_ERR_BAD_PARAMS, "null block");
  return FIC_OK;
}

}  // namespace

extern "C" {

int32_t fic_is_shadow(const double* samples, int32_t side, double eps, int32_t* out) {
  if (side < 0) return fit_fail(FIC_ERR_BAD_PARAMS, "negative block side");
  if (side > 0 && !samples) return fit_fail(FIC_ERR_BAD_PARAMS, "null block");
  const long count = (long)side * side;
  double sum = 0.0, sum_sq = 0.0;
  for (long i = 0; i < count; ++i) {
    sum += samples[i];
    sum_sq += samples[i] * samples[i];
  }
  if (out) *out = (double)count * sum_sq - sum * sum <= eps ? 1 : 0;
  return FIC_OK;
}

int32_t fic_least_squares_fit(const double* a, int32_t side_a, const double* b, int32_t side_b, double shadow_eps,
                              fic_linear_fit* out) {
  if (int32_t e = check_blocks(a, side_a, b, side_b)) return e;
  const long count = (long)side_a * side_a;
  const FitSums f = gather(a, b, count);
  fic_linear_fit fit;
  fit.s = f.den <= shadow_eps ? 0.0 : f.num / f.den;
  fit.o = (f.sb - fit.s * f.sa) / f.n;
  fit.residual = score(a, b, count, fit.s, fit.o);
  if (out) *out = fit;
  return FIC_OK;
}

int32_t fic_least_squares_clamped(const double* a, int32_t side_a, const double* b, int32_t side_b,
                                  const fic_params* params, fic_linear_fit* out) {
  fic_params p;
  if (int32_t e = fic_normalize_params(params, &p)) return e;
  if (int32_t e = check_blocks(a, side_a, b, side_b)) return e;
  const long count = (long)side_a * side_a;
  const FitSums f = gather(a, b, count);
  fic_linear_fit fit;
  fit.s = f.den <= p.shadow_eps ? 0.0 : std::clamp(f.num / f.den, -p.s_max, p.s_max);
  fit.o = std::clamp((f.sb - fit.s * f.sa) / f.n, -255.0, 255.0);
  fit.residual = score(a, b, count, fit.s, fit.o);
  if (out) *out = fit;
  return FIC_OK;
}

int32_t fic_least_squares(const double* a, int32_t side_a, const double* b, int32_t side_b,
                          const fic_params* params, fic_quantized_fit* out) {
  fic_params p;
  if (int32_t e = fic_normalize_params(params, &p)) return e;
  fic_linear_fit fit;
  if (int32_t e = fic_least_squares_clamped(a, side_a, b, side_b, &p, &fit)) return e;
  const long count = (long)side_a * side_a;
  // UniformQuantizer::quantize's range check (format.hpp:27, format.cpp:12-15): only a NaN
  // sample can get past the clamps
  for (const auto& [v, mx] : {std::pair<double, double>{fit.s, p.s_max}, {fit.o, 255.0}})
    if (!(v >= -mx && v <= mx))
      return fit_fail(FIC_ERR_OUT_OF_RANGE,
                      std::to_string(v) + " outside [-" + std::to_string(mx) + ", " + std::to_string(mx) + "]");
  fic_quantized_fit q;
  q.qs = ficb::quantize(fit.s, p.s_max, p.s_bits);  // UniformQuantizer (format.hpp:26-40)
  q.qo = ficb::quantize(fit.o, 255.0, p.o_bits);
  q.s = ficb::dequantize(q.qs, p.s_max, p.s_bits);
  q.o = ficb::dequantize(q.qo, 255.0, p.o_bits);
  q.residual = score(a, b, count, q.s, q.o);
  if (out) *out = q;
  return FIC_OK;
}

}  // extern "C"
