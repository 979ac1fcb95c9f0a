// Golden-vector generator for the RNG restatement in
// paper_2307_08606_b200/rng.py.  Built and run with g++ 13 / libstdc++ in
// the build container:
//
//   g++ -O2 -std=c++17 tests/golden/gen_rng_golden.cpp -o /tmp/gen && /tmp/gen > tests/golden/rng_golden.json
//
// It uses the real std::mt19937_64 and std::normal_distribution the
// reference's generators and tests are built on (scene.hpp:103-116,
// tests/fixtures.hpp:42-47, tests/acceptance.cpp:70-84), and an independent
// restatement of the splitmix64 seed mixer and the hand Box-Muller sampler.
// Printed with %.17g so every double round-trips.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <random>

static std::uint64_t splitmix(std::uint64_t base, std::uint64_t stream) {
  std::uint64_t z = base + stream * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

int main() {
  std::printf("{\n");
  // Raw engine outputs for a few seeds, including draws past one twist.
  std::printf("  \"mt19937_64\": {\n");
  const std::uint64_t seeds[3] = {5489ull, 1ull, 0x123456789abcdefull};
  for (int s = 0; s < 3; ++s) {
    std::mt19937_64 rng(seeds[s]);
    std::printf("    \"%llu\": [", static_cast<unsigned long long>(seeds[s]));
    for (int i = 0; i < 700; ++i) {
      const std::uint64_t v = rng();
      if (i < 8 || i >= 620)
        std::printf("%s\"%llu\"", (i == 0 ? "" : ", "),
                    static_cast<unsigned long long>(v));
    }
    std::printf("]%s\n", s == 2 ? "" : ",");
  }
  std::printf("  },\n");

  std::printf("  \"mix_seed\": [");
  for (int i = 0; i < 6; ++i)
    std::printf("%s\"%llu\"", i ? ", " : "",
                static_cast<unsigned long long>(splitmix(1 + 7 * i, i)));
  std::printf("],\n");

  // Hand Box-Muller on mt19937_64 (unit complex variance).
  {
    std::mt19937_64 rng(splitmix(1, 3));
    std::printf("  \"complex_gaussian_seed_mix_1_3\": [");
    for (int i = 0; i < 16; ++i) {
      const double u1 = (static_cast<double>(rng() >> 11) + 1.0) * 0x1p-53;
      const double u2 = static_cast<double>(rng() >> 11) * 0x1p-53;
      const double rad = std::sqrt(-std::log(u1));
      const double th = 2.0 * 3.141592653589793238462643383279502884 * u2;
      std::printf("%s[%.17g, %.17g]", i ? ", " : "", rad * std::cos(th),
                  rad * std::sin(th));
    }
    std::printf("],\n");
  }

  // libstdc++ normal_distribution: persistent distribution (cached pair).
  {
    std::mt19937_64 rng(9);
    std::normal_distribution<double> dist(0.0, 1.0);
    std::printf("  \"std_normal_seed_9\": [");
    for (int i = 0; i < 41; ++i)
      std::printf("%s%.17g", i ? ", " : "", dist(rng));
    std::printf("],\n");
  }
  // Fresh distribution per vector (discards the cached second sample).
  {
    std::mt19937_64 rng(4);
    std::printf("  \"std_normal_fresh_per_vector_seed_4\": [");
    for (int v = 0; v < 3; ++v) {
      std::normal_distribution<double> dist(0.0, 1.0);
      for (int i = 0; i < 3; ++i) {
        const double re = dist(rng);
        const double im = dist(rng);
        std::printf("%s[%.17g, %.17g]", (v || i) ? ", " : "", re, im);
      }
    }
    std::printf("]\n");
  }
  std::printf("}\n");
  return 0;
}
