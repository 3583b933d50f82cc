// oracle/_ref driver: links the REFERENCE's own rng.hpp (kernid::Rng, derive_seed)
// unmodified, and prints its streams as JSON so tests/golden/make_rng_golden.py can
// pin oracle/kernid_oracle.c's restatement bit-for-bit. The gen_normal loop below is
// datagen.hpp:35-43 verbatim in behaviour (point-major draws, col-major store).
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <vector>
#include "kernid/rng.hpp"

static void hexd(double v) { unsigned long long u; std::memcpy(&u, &v, 8); std::printf("\"%016llx\"", u); }

int main(int argc, char** argv) {
  const unsigned long long seed = argc > 1 ? std::strtoull(argv[1], nullptr, 0) : 1ull;
  const int n = argc > 2 ? std::atoi(argv[2]) : 16;
  std::printf("{\"seed\": %llu,\n", seed);
  std::printf("\"derive_seed\": [");
  for (int a = 0; a < 4; ++a) for (int b = 0; b < 3; ++b)
    std::printf("%s[%d, %d, %llu]", (a || b) ? ", " : "", a, b, (unsigned long long)kernid::derive_seed(seed, a, b));
  std::printf("],\n\"derive_special\": [%llu, %llu],\n",
              (unsigned long long)kernid::derive_seed(seed, 0xDA7A), (unsigned long long)kernid::derive_seed(seed, 0xCE));
  { kernid::Rng r(seed); std::printf("\"u64\": ["); for (int i = 0; i < n; ++i) std::printf("%s%llu", i ? ", " : "", (unsigned long long)r.next_u64()); std::printf("],\n"); }
  { kernid::Rng r(seed); std::printf("\"uniform01\": ["); for (int i = 0; i < n; ++i) { if (i) std::printf(", "); hexd(r.uniform01()); } std::printf("],\n"); }
  { kernid::Rng r(seed); std::printf("\"normal\": ["); for (int i = 0; i < n; ++i) { if (i) std::printf(", "); hexd(r.normal()); } std::printf("],\n"); }
  { kernid::Rng r(seed); std::printf("\"below_1000003\": ["); for (int i = 0; i < n; ++i) std::printf("%s%llu", i ? ", " : "", (unsigned long long)r.below(1000003)); std::printf("],\n"); }
  { // gen_normal(d=3, N=n) in col-major order (datagen.hpp:35-43)
    const int d = 3; kernid::Rng r(kernid::derive_seed(seed, 0xDA7A));
    std::vector<double> ps(static_cast<size_t>(n) * d);
    for (int i = 0; i < n; ++i) for (int j = 0; j < d; ++j) ps[i + static_cast<size_t>(j) * n] = r.normal();
    std::printf("\"gen_normal_d3\": ["); for (size_t i = 0; i < ps.size(); ++i) { if (i) std::printf(", "); hexd(ps[i]); } std::printf("]}\n");
  }
  return 0;
}
