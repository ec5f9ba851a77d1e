// ref_rng_dump.cpp -- driver compiled AGAINST THE REFERENCE'S OWN rng.hpp
// (/root/reference/proj/include/lmra/rng.hpp, the only Eigen-free file on the hot path).
// TEST INFRASTRUCTURE ONLY: it produces the golden RNG vectors under tests/golden/
// (see tests/golden/make_golden.py).  Output: one JSON object on stdout.
#include <cstdio>
#include <cstdint>
#include "lmra/rng.hpp"

static void dump(std::uint64_t seed, std::uint64_t stream, int n_u32, int n_dbl, int n_nrm, bool last) {
  std::printf("  {\"seed\": %llu, \"stream\": %llu,\n   \"u32\": [", (unsigned long long)seed,
              (unsigned long long)stream);
  lmra::RandomStream a(lmra::RngStream{seed, stream});
  for (int i = 0; i < n_u32; ++i) std::printf("%s%u", i ? ", " : "", a.next_u32());
  std::printf("],\n   \"double_hex\": [");
  lmra::RandomStream b(lmra::RngStream{seed, stream});
  for (int i = 0; i < n_dbl; ++i) std::printf("%s\"%a\"", i ? ", " : "", b.next_double());
  std::printf("],\n   \"normal_hex\": [");
  lmra::RandomStream c(lmra::RngStream{seed, stream});
  for (int i = 0; i < n_nrm; ++i) std::printf("%s\"%a\"", i ? ", " : "", c.next_normal());
  std::printf("]}%s\n", last ? "" : ",");
}

int main() {
  std::printf("{\"source\": \"reference proj/include/lmra/rng.hpp compiled by oracle/Makefile (ref target)\",\n \"streams\": [\n");
  dump(42, 54, 64, 32, 33, false);   // test_sketching.cpp:16-23 KAT pair
  dump(0, 1, 64, 32, 65, false);     // gaussian_stream(seed=0, mode 0)
  dump(1, 1, 64, 32, 65, false);     // BASELINE seed 1, mode 0 Omega
  dump(1, 4, 64, 32, 65, false);     // sampling stream N+n+1 (N=3, n=0)
  dump(5, 0, 64, 32, 65, false);     // test_sketching.cpp:114 point-mass stream
  dump(99, 7, 64, 32, 65, false);
  dump(1ull << 40, 123456789ull, 64, 32, 65, true);
  std::printf(" ]\n}\n");
  return 0;
}
