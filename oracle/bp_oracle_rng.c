/* TEST INFRASTRUCTURE ONLY (oracle). Plain-C restatement of the reference's
 * random source, used by tests/ to check the GPU noise kernel bit-for-bit at
 * Wan pool sizes where a pure-Python loop would be slow.
 *
 *   next_u64      rng.cpp:12-18   splitmix64 (state += phi; two xor-shift-multiplies)
 *   next_normal   rng.cpp:24-31   Box-Muller, two raw draws, glibc log/cos/sqrt
 *   normal_tensor rng.cpp:35-39   row-major fill, * sigma
 *   derive_seed   rng.cpp:51-60   s ^ ((tag+1)*phi), one splitmix step per tag
 *
 * Compiled with -ffp-contract=off so no FMA sneaks into the Box-Muller
 * arithmetic (the reference's default x86-64 build has none there). */
#include <math.h>
#include <stdint.h>

#define PHI 0x9E3779B97F4A7C15ULL

static inline uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

uint64_t bpo_derive_seed(uint64_t base, const uint64_t* tags, int n) {
  uint64_t s = base;
  for (int i = 0; i < n; ++i) s = mix((s ^ ((tags[i] + 1) * PHI)) + PHI);
  return s;
}

/* Fills out[0..n) with normal_tensor values of RandomSource(seed) and returns
 * the final state, so callers can continue the stream. */
uint64_t bpo_normals(uint64_t state, int64_t n, double sigma, double* out) {
  const double two_pow_m53 = 1.0 / 9007199254740992.0;
  const double two_pi = 2.0 * M_PI;
  for (int64_t i = 0; i < n; ++i) {
    state += PHI;
    const uint64_t a = mix(state);
    state += PHI;
    const uint64_t b = mix(state);
    const double u1 = (double)((a >> 11) + 1) * two_pow_m53;
    const double u2 = (double)(b >> 11) * two_pow_m53;
    const double r = sqrt(-2.0 * log(u1));
    out[i] = (r * cos(two_pi * u2)) * sigma;
  }
  return state;
}

double bpo_log(double x) { return log(x); }
double bpo_cos(double x) { return cos(x); }
