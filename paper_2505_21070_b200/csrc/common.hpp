// Internal helpers shared by the host and device translation units.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "bp_cuda.h"

namespace bp {

// Internal exception carrying a bp_status; the C-ABI wrappers translate it
// into the return code + thread-local message (the reference throws the
// matching blockpipe::*Error, errors.hpp:11-41).
struct Error : std::runtime_error {
  bp_status status;
  Error(bp_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] inline void fail(bp_status s, const std::string& m) { throw Error(s, m); }

void set_last_error(const std::string& m);

template <class F>
bp_status guarded(F&& f) {
  try {
    f();
    return BP_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.status;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return BP_ERR_INTERNAL;
  }
}

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// Host RandomSource integer stream (rng.cpp:12-18, 41-49): the noise ids and
// permutations live on the host; the normals they would draw are produced on
// the device from the same counter (state advances by 2*phi per normal).
struct HostRng {
  uint64_t state;
  explicit HostRng(uint64_t s) : state(s) {}
  uint64_t next_u64() {
    state += kGolden;
    return mix64(state);
  }
  uint64_t next_below(uint64_t n) { return next_u64() % n; }
  std::vector<int> permutation(int n) {
    std::vector<int> p(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) p[static_cast<size_t>(i)] = i;
    for (int i = n - 1; i > 0; --i) {
      const int j = static_cast<int>(next_below(static_cast<uint64_t>(i) + 1));
      std::swap(p[static_cast<size_t>(i)], p[static_cast<size_t>(j)]);
    }
    return p;
  }
  // Skips the 2*n raw draws of normal_tensor with n elements.
  void skip_normals(int64_t n) { state += kGolden * static_cast<uint64_t>(2 * n); }
};

inline uint64_t derive_seed(uint64_t base, const uint64_t* tags, int n) {
  uint64_t s = base;
  for (int i = 0; i < n; ++i) s = mix64((s ^ ((tags[i] + 1) * kGolden)) + kGolden);
  return s;
}
inline uint64_t derive_seed2(uint64_t base, uint64_t a, uint64_t b) {
  const uint64_t t[2] = {a, b};
  return derive_seed(base, t, 2);
}

}  // namespace bp
