// SeqRng::bounded (csrc/domain.hpp) with its power-of-two and cached-remainder fast paths
// against the plain rejection rule of Rng::bounded (rng.hpp: reject r < 2^64 mod n, r % n).
#include "domain.hpp"
#include <cstdio>
#include <random>
int main() {
  using lann::SeqRng;
  long bad = 0, total = 0;
  for (std::uint64_t n = 1; n <= 5000; ++n) {
    SeqRng a(n * 7919 + 1);
    std::mt19937_64 b(n * 7919 + 1);
    for (int k = 0; k < 2000; ++k) {
      const std::uint64_t got = a.bounded(n);
      const std::uint64_t thr = (0 - n) % n;
      std::uint64_t r;
      do r = b(); while (r < thr);
      bad += got != r % n;
      ++total;
    }
  }
  for (std::uint64_t n : {4097ull, 1000003ull, (1ull << 40) + 7, ~0ull / 3}) {
    SeqRng a(n); std::mt19937_64 b(n);
    for (int k = 0; k < 10000; ++k) { const std::uint64_t thr = (0 - n) % n; std::uint64_t r; do r = b(); while (r < thr); bad += a.bounded(n) != r % n; ++total; }
  }
  std::printf("checked %ld draws, %ld mismatches\n", total, bad);
  return bad != 0;
}
