// gofmm_rng.h — the reference's random number streams (common.hpp:40-98), restated so the product
// draws the same streams as the reference: splitmix64, Rng(seed, stream) with next / uniform /
// uniform01 / Box-Muller gauss (cached spare) / sorted rejection sample without replacement.
// Host code shared by the C-ABI (error_eps2 draws) and the compress pipeline (tree pivots,
// skeleton column samples, ANN seeds).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

namespace gofmm {

inline uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

struct RefRng {
  uint64_t state;
  bool have_spare = false;
  double spare = 0.0;
  static uint64_t mix(uint64_t x) { return splitmix64(x); }
  RefRng(uint64_t seed, uint64_t stream) : state(mix(seed ^ mix(stream + 0x632be59bd9b4e019ULL))) {}
  uint64_t next() { return state = mix(state); }
  int uniform(int n) { return int(next() % uint64_t(n)); }
  double uniform01() { return double(next() >> 11) * 0x1.0p-53; }
  double gauss() {
    if (have_spare) {
      have_spare = false;
      return spare;
    }
    double u1 = uniform01(), u2 = uniform01();
    while (u1 <= 1e-300) u1 = uniform01();
    double rr = std::sqrt(-2.0 * std::log(u1));
    double a = 2.0 * M_PI * u2;
    spare = rr * std::sin(a);
    have_spare = true;
    return rr * std::cos(a);
  }
  // k distinct values of [0, n), ascending (common.hpp:80-98)
  std::vector<int> sample_without_replacement(int n, int k) {
    std::vector<int> out;
    if (k >= n) {
      out.resize(n);
      for (int i = 0; i < n; ++i) out[i] = i;
      return out;
    }
    std::vector<char> taken(n, 0);
    out.reserve(k);
    while (int(out.size()) < k) {
      const int v = uniform(n);
      if (!taken[v]) {
        taken[v] = 1;
        out.push_back(v);
      }
    }
    std::sort(out.begin(), out.end());
    return out;
  }
};

}  // namespace gofmm
