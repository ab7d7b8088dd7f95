// Golden-stream generator built against the REFERENCE's own rng.hpp
// (/root/reference/proj/core/include/warmgp/rng.hpp, compiled unchanged via -I).
// TEST INFRASTRUCTURE ONLY: output goes to oracle/_ref/ and is frozen into
// tests/golden/rng_golden.json by tests/golden/make_golden.py.
#include <cstdio>
#include <cinttypes>
#include <initializer_list>
#include "warmgp/rng.hpp"

using warmgp::Rng;

static void emit_stream(std::uint64_t seed, bool first) {
  Rng r(seed);
  std::printf("%s{\"seed\": %" PRIu64 ", \"u64\": [", first ? "" : ",\n", seed);
  for (int i = 0; i < 8; ++i) std::printf("%s\"%" PRIu64 "\"", i ? ", " : "", r.next_u64());
  std::printf("], \"uniform\": [");
  for (int i = 0; i < 8; ++i) std::printf("%s%.17g", i ? ", " : "", r.uniform());
  std::printf("], \"normal\": [");
  for (int i = 0; i < 8; ++i) std::printf("%s%.17g", i ? ", " : "", r.normal());
  std::printf("], \"chi_square3\": [");
  for (int i = 0; i < 4; ++i) std::printf("%s%.17g", i ? ", " : "", r.chi_square3());
  std::printf("], \"uniform_index_1000\": [");
  for (int i = 0; i < 8; ++i) std::printf("%s%zu", i ? ", " : "", r.uniform_index(1000));
  std::printf("], \"uniform_index_7\": [");
  for (int i = 0; i < 8; ++i) std::printf("%s%zu", i ? ", " : "", r.uniform_index(7));
  std::printf("], \"uniform_range\": [");
  for (int i = 0; i < 4; ++i) std::printf("%s%.17g", i ? ", " : "", r.uniform(0.0, 6.283185307179586476925287));
  std::printf("], \"derive_17\": \"%" PRIu64 "\"}", r.derive(17).next_u64());
}

int main() {
  std::printf("{\"streams\": [\n");
  const std::uint64_t seeds[] = {0ull, 1ull, 42ull, 1234ull, 0xc0ffeeull, 18446744073709551615ull};
  bool first = true;
  for (auto s : seeds) { emit_stream(s, first); first = false; }
  std::printf("],\n\"derive_seed\": [");
  first = true;
  for (std::uint64_t s : {0ull, 1ull, 42ull, 7ull}) {
    for (std::uint64_t t : {0ull, 1ull, 2ull, 0xc0000ull + 3, 0x0b1ec7ull}) {
      std::printf("%s[\"%" PRIu64 "\", \"%" PRIu64 "\", \"%" PRIu64 "\"]", first ? "" : ", ", s, t,
                  warmgp::derive_seed(s, t));
      first = false;
    }
  }
  std::printf("]}\n");
  return 0;
}
