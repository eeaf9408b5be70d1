// Host-side lattice configuration: QuantizerConfig.from_params /
// __post_init__ (quantizer.py:89-135) and tune_eps (quantizer.py:154-214).
// Pure scalar logic, no GPU; exported through the C ABI so non-Python hosts
// get the exact same configuration the reference computes.
#include <math.h>
#include <string.h>

#include <string>

#include "fgc_internal.h"

namespace {

constexpr double kMinEps = 1.1754943508222875e-38;   // 2^-126 (quantizer.py:48)
constexpr uint32_t kTopPattern = 0x7F7FFFFFu;        // quantizer.py:52
constexpr int kTuneIters = 64;                       // quantizer.py:54

uint32_t f32_bits(double x) {
  const float f = (float)x;
  uint32_t u;
  memcpy(&u, &f, 4);
  return u;
}

double bits_f32(uint32_t p) {
  float f;
  memcpy(&f, &p, 4);
  return (double)f;
}

fgc_status invalid(const std::string& m) {
  fgc::set_error(m);
  return FGC_ERR_INVALID;
}

}  // namespace

extern "C" fgc_status fgc_quantizer_from_params(double min, double max, int n_bits, int mantissa_bits, double eps,
                                                fgc_quantizer* out) {
  if (!out) return invalid("null output");
  if (n_bits < 2 || n_bits > 16) return invalid("n_bits must be in [2, 16], got " + std::to_string(n_bits));
  if (mantissa_bits < 1 || mantissa_bits >= n_bits)
    return invalid("mantissa_bits must satisfy 1 <= m < n_bits, got m=" + std::to_string(mantissa_bits) +
                   ", N=" + std::to_string(n_bits));
  const int shift = 23 - mantissa_bits;
  const double eps_l = bits_f32((f32_bits(eps) >> shift) << shift);
  const uint32_t pbase = f32_bits(eps_l) >> shift;
  const int64_t top = (int64_t)(f32_bits(max) >> shift);
  const int64_t pos = top - (int64_t)pbase + 1;
  const double fmin_ = (double)(float)min, fmax_ = (double)(float)max;
  // __post_init__ order (quantizer.py:89-106)
  if (!(isfinite(fmin_) && isfinite(fmax_))) return invalid("min/max must be finite");
  if (!(fmin_ < 0.0 && 0.0 < fmax_)) return invalid("range must straddle zero");
  if (!(0.0 < eps_l && eps_l < fmax_)) return invalid("eps must be in (0, max)");
  const int64_t codes = (int64_t)1 << n_bits;
  if (!(1 <= pos && pos <= codes - 2)) return invalid("config leaves no room for positive or negative codes");
  const int64_t neg = codes - 1 - pos;
  if ((int64_t)pbase + neg - 1 > (int64_t)(kTopPattern >> shift))
    return invalid("negative lattice runs past the float32 range");
  out->min = (float)fmin_;
  out->max = (float)fmax_;
  out->eps = (float)eps_l;
  out->n_bits = n_bits;
  out->mantissa_bits = mantissa_bits;
  out->pbase = pbase;
  out->pos_count = (uint32_t)pos;
  out->neg_count = (uint32_t)neg;
  out->actual_min = (float)-bits_f32((uint32_t)((pbase + neg - 1) << shift));
  out->actual_max = (float)bits_f32((uint32_t)((pbase + pos - 1) << shift));
  return FGC_OK;
}

extern "C" fgc_status fgc_quantizer_validate(fgc_quantizer* q) {
  if (!q) return invalid("null quantizer");
  const int n = q->n_bits, m = q->mantissa_bits;
  if (n < 2 || n > 16) return invalid("n_bits must be in [2, 16], got " + std::to_string(n));
  if (m < 1 || m >= n)
    return invalid("mantissa_bits must satisfy 1 <= m < n_bits, got m=" + std::to_string(m) + ", N=" + std::to_string(n));
  if (!(isfinite(q->min) && isfinite(q->max))) return invalid("min/max must be finite");
  if (!(q->min < 0.0f && 0.0f < q->max)) return invalid("range must straddle zero");
  if (!(0.0f < q->eps && q->eps < q->max)) return invalid("eps must be in (0, max)");
  const int shift = 23 - m;
  if (q->pbase != (f32_bits(q->eps) >> shift)) return invalid("pbase inconsistent with eps");
  const int64_t codes = (int64_t)1 << n;
  if (!(1 <= (int64_t)q->pos_count && (int64_t)q->pos_count <= codes - 2))
    return invalid("config leaves no room for positive or negative codes");
  const int64_t neg = codes - 1 - (int64_t)q->pos_count;
  if ((int64_t)q->pbase + neg - 1 > (int64_t)(kTopPattern >> shift))
    return invalid("negative lattice runs past the float32 range");
  q->neg_count = (uint32_t)neg;
  q->actual_min = (float)-bits_f32((uint32_t)((q->pbase + neg - 1) << shift));
  q->actual_max = (float)bits_f32((uint32_t)(((int64_t)q->pbase + q->pos_count - 1) << shift));
  return FGC_OK;
}

extern "C" fgc_status fgc_tune_eps(double min, double max, int n_bits, int mantissa_bits, double eps_init,
                                   fgc_quantizer* out) {
  if (!out) return invalid("null output");
  if (!(isfinite(min) && isfinite(max) && min < 0.0 && 0.0 < max))
    return invalid("bounds must be finite with min < 0 < max");
  if (n_bits < 2 || n_bits > 16) return invalid("n_bits must be in [2, 16]");
  if (mantissa_bits < 1 || mantissa_bits >= n_bits) return invalid("mantissa_bits must satisfy 1 <= m < N");
  if (!(isfinite(eps_init) && eps_init > 0.0)) return invalid("eps_init must be positive and finite");
  const int shift = 23 - mantissa_bits;
  const int64_t top = (int64_t)(f32_bits(max) >> shift);
  const int64_t max_pattern = (int64_t)(kTopPattern >> shift);
  // np.clip(eps_init, MIN_EPS, nextafter(float32(max), 0)) in float64 (quantizer.py:183)
  const double upper = (double)nextafterf((float)max, 0.0f);
  double start = eps_init < kMinEps ? kMinEps : eps_init;
  if (start > upper) start = upper;
  double eps = bits_f32((f32_bits(start) >> shift) << shift);
  bool have_best = false, have_prev = false;
  fgc_quantizer best{};
  double best_gap = INFINITY, prev = 0.0;
  const int64_t codes = (int64_t)1 << n_bits;
  for (int it = 0; it < kTuneIters; ++it) {
    const int64_t pbase = (int64_t)(f32_bits(eps) >> shift);
    const int64_t neg = codes - 2 - (top - pbase);
    if (neg < 1) {
      eps *= 2.0;
      have_prev = false;
      continue;
    }
    if (pbase + neg - 1 > max_pattern) {
      eps /= 2.0;
      have_prev = false;
      continue;
    }
    fgc_quantizer cand;
    fgc_status st = fgc_quantizer_from_params(min, max, n_bits, mantissa_bits, eps, &cand);
    if (st != FGC_OK) return st;
    const double diff = (double)cand.actual_min - min;
    if (fabs(diff) < best_gap) {
      best = cand;
      best_gap = fabs(diff);
      have_best = true;
    }
    if (diff == 0.0) {
      *out = cand;
      return FGC_OK;
    }
    if (have_prev && ((diff > 0.0) != (prev > 0.0))) break;
    prev = diff;
    have_prev = true;
    eps = diff < 0.0 ? eps / 2.0 : eps * 2.0;
    if (!(kMinEps < eps && eps < max)) break;
  }
  if (!have_best) {
    fgc::set_error("eps tuning found no valid configuration");
    return FGC_ERR_NO_CONFIG;
  }
  *out = best;
  return FGC_OK;
}
