// neighbor_dump.cpp -- TEST INFRASTRUCTURE ONLY.  Built twice by
// oracle/Makefile (target `neighbor`): against the reference sources
// (_ref/neighbor_on_reference) and against this repo's drop-in library
// (_ref/neighbor_on_b200).  Both apply `neighbor` (solver.hpp:44-47) along
// seeded std::mt19937_64 streams and print the orders; the outputs must be
// identical (tests/test_host_logic.py).
#include <cstdio>
#include <random>

#include "rankweave/solver.hpp"
#include "rankweave/types.hpp"

int main() {
  const int sizes[] = {1, 2, 3, 5, 8, 13, 64, 1000};
  for (int n : sizes)
    for (unsigned seed = 0; seed < 6; ++seed) {
      std::mt19937_64 rng(1000003ull * seed + (unsigned)n);
      rankweave::RankOrder o = rankweave::RankOrder::identity(n);
      for (int step = 0; step < 300; ++step) o = rankweave::neighbor(o, rng);
      std::printf("n=%d seed=%u:", n, seed);
      for (int v : o.perm) std::printf(" %d", v);
      std::printf(" | next=%llu\n", (unsigned long long)rng());
    }
  return 0;
}
