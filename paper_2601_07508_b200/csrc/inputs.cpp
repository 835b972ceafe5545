// inputs.cpp -- the seeded synthetic inputs of the reference benchmark
// (mat.hpp:92-120 random_mat with std::mt19937_64 and rejection sampling).
#include <cstdint>
#include <limits>
#include <random>

#include "fpmm_b200.h"

extern "C" int fpmm_b200_random_mat(int64_t rows, int64_t cols, uint64_t p, uint64_t seed,
                                    double* out) {
  if (rows < 0 || cols < 0 || p == 0) return FPMM_B200_EERROR;
  std::mt19937_64 rng(seed);
  constexpr uint64_t kMax = std::numeric_limits<uint64_t>::max();
  const uint64_t reject_at = kMax - kMax % p;  // unbiased: reject the partial top bucket
  const int64_t count = rows * cols;
  for (int64_t e = 0; e < count; ++e) {
    uint64_t r = rng();
    while (r >= reject_at) r = rng();
    out[e] = static_cast<double>(r % p);
  }
  return FPMM_B200_OK;
}
