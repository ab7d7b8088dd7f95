// host_rng.cpp -- host-side randomness of the path, restating rng.hpp:11-61 and the RNG
// consumption order of sample_prior (sampling.cpp:14-35) and build_sample_rhs (:56-64).
// Draws stay on the host (F*(d+5) normals per prior, B indices per SGD step); only the
// results are uploaded, so device results are reproducible against the reference streams.
#include <cmath>
#include <cstdint>

#include "../../include/warmgp_capi.h"
#include "rng.h"

using wgp::Rng;

extern "C" {

uint64_t wgp_derive_seed(uint64_t seed, uint64_t stream) {  // rng.hpp:11-16
  return wgp::derive_seed(seed, stream);
}

uint64_t wgp_rng_next_u64(uint64_t* state) { Rng r{*state}; uint64_t v = r.next_u64(); *state = r.state; return v; }
double wgp_rng_uniform(uint64_t* state) { Rng r{*state}; double v = r.uniform(); *state = r.state; return v; }
double wgp_rng_normal(uint64_t* state) { Rng r{*state}; double v = r.normal(); *state = r.state; return v; }
double wgp_rng_chi_square3(uint64_t* state) { Rng r{*state}; double v = r.chi_square3(); *state = r.state; return v; }
uint64_t wgp_rng_uniform_index(uint64_t* state, uint64_t n) {
  Rng r{*state};
  uint64_t v = r.uniform_index(n);
  *state = r.state;
  return v;
}

void wgp_rng_normal_fill(uint64_t* state, int64_t n, double scale, double* out) {
  Rng r{*state};
  for (int64_t i = 0; i < n; ++i) out[i] = scale * r.normal();
  *state = r.state;
}

void wgp_normal_fill(uint64_t seed, int64_t n, double scale, double* out) {
  Rng r{seed};  // build_sample_rhs noise order, sampling.cpp:58-62
  for (int64_t i = 0; i < n; ++i) out[i] = scale * r.normal();
}

wgp_status wgp_sample_prior(int kernel, double lengthscale, int64_t dim, int64_t F, uint64_t seed,
                            double* Omega, double* phases, double* amps) {
  // sample_prior, sampling.cpp:14-35.  Omega: F x dim column-major (RffPrior::frequencies).
  if (!(lengthscale > 0.0) || dim < 1 || F < 1 || !Omega || !phases || !amps)
    return WGP_INVALID_ARGUMENT;
  if (kernel != WGP_MATERN32 && kernel != WGP_RBF) return WGP_INVALID_ARGUMENT;
  Rng rng{seed};
  for (int64_t i = 0; i < F; ++i) {
    double t_scale;
    if (kernel == WGP_MATERN32) {  // Student-t(3) rows
      const double u = rng.chi_square3();
      t_scale = std::sqrt(3.0 / u) / lengthscale;
    } else {  // RBF extension: N(0, l^-2 I)
      t_scale = 1.0 / lengthscale;
    }
    for (int64_t d = 0; d < dim; ++d) Omega[d * F + i] = rng.normal() * t_scale;
    phases[i] = rng.uniform(0.0, 6.283185307179586476925287);
    amps[i] = rng.normal();
  }
  return WGP_OK;
}

}  // extern "C"
