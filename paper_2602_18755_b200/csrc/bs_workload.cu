// bs_workload.cu — host-side workload synthesis and window plumbing of the
// C ABI: gen_gamma_trace (workload.hpp:95-116) with the reference's own
// samplers (rng.hpp:22-70: Box-Muller normal, Marsaglia-Tsang gamma,
// lognormal, rejection-sampled uniform_index), split_windows
// (workload.hpp:184-201) and peak_rps (placement.hpp:513-527).
// Input generation, not decisions: plain host C++ on the same libm the
// reference links, so traces are bit-identical to the reference's.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "bs_internal.h"
#include "bs_rng.cuh"

using namespace bs;

namespace {

struct HostRng {  // pdsim::Rng (rng.hpp:15-75)
  Mt64 e;
  explicit HostRng(unsigned long long seed) { e.seed(seed); }
  unsigned long long next() { return e.next(); }
  double uniform01() { return e.uniform01(); }
  double uniform_open01() {
    for (;;) {
      const double u = uniform01();
      if (u > 0.0) return u;
    }
  }
  unsigned long long uniform_index(unsigned long long n) {
    const unsigned long long limit = UINT64_MAX - UINT64_MAX % n;
    for (;;) {
      const unsigned long long x = next();
      if (x < limit) return x % n;
    }
  }
  double normal() {
    const double u1 = uniform_open01();
    const double u2 = uniform01();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
  }
  double gamma(double shape, double scale) {
    if (shape < 1.0) {
      const double u = uniform_open01();
      return gamma(shape + 1.0, scale) * std::pow(u, 1.0 / shape);
    }
    const double d = shape - 1.0 / 3.0;
    const double c = 1.0 / std::sqrt(9.0 * d);
    for (;;) {
      const double x = normal();
      double v = 1.0 + c * x;
      if (v <= 0.0) continue;
      v = v * v * v;
      const double u = uniform_open01();
      if (std::log(u) < 0.5 * x * x + d - d * v + d * std::log(v)) return d * v * scale;
    }
  }
  double lognormal(double mu, double sigma) { return std::exp(mu + sigma * normal()); }
};

}  // namespace

extern "C" {

int bs_gen_gamma_trace(double mean_rps, double shape, double duration_ms, const bs_length_dist* lengths,
                       uint64_t seed, bs_request* out, int64_t capacity, int64_t* n_out) {
  if (!lengths || !n_out) return BS_PARAMETER_ERROR;
  if (mean_rps <= 0.0) return BS_PARAMETER_ERROR;  // gen_gamma_trace: mean_rps must be > 0
  if (shape <= 0.0) return BS_PARAMETER_ERROR;
  if (duration_ms <= 0.0) return BS_PARAMETER_ERROR;
  if (lengths->n_samples <= 0 && !lengths->lognormal) return BS_PARAMETER_ERROR;
  HostRng rng(seed);
  const double scale_s = 1.0 / (shape * mean_rps);
  double now_ms = 0.0;
  int64_t n = 0;
  for (;;) {
    now_ms += rng.gamma(shape, scale_s) * 1000.0;
    if (now_ms >= duration_ms) break;
    int64_t in_len, out_len;
    if (lengths->n_samples > 0) {  // LengthDistribution::sample (workload.hpp:71-84)
      const unsigned long long i = rng.uniform_index(static_cast<unsigned long long>(lengths->n_samples));
      in_len = lengths->sample_input[i];
      out_len = lengths->sample_output[i];
    } else {
      double v = std::round(rng.lognormal(lengths->input_mu, lengths->input_sigma));
      in_len = std::max<int64_t>(1, static_cast<int64_t>(v));
      v = std::round(rng.lognormal(lengths->output_mu, lengths->output_sigma));
      out_len = std::max<int64_t>(1, static_cast<int64_t>(v));
    }
    if (out && n < capacity) out[n] = bs_request{n, now_ms, in_len, out_len};
    ++n;
  }
  *n_out = n;
  return n <= capacity || !out ? BS_OK : BS_PARAMETER_ERROR;
}

}  // extern "C"
