// latency.cpp -- TEST INFRASTRUCTURE / MEASUREMENT.  Built twice by
// oracle/Makefile (target `latency`): against the reference sources
// (_ref/latency_on_reference) and against this repo's drop-in library
// (_ref/latency_on_b200, -DRW_B200).  Times single evaluate() calls
// (cost_model.hpp:28, cost_model.cpp:140-148) -- the per-call latency a
// reference user sees -- on generated hierarchical matrices, and prints one
// JSON object per case: the median and 10th/90th percentile in microseconds.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "rankweave/cost_model.hpp"
#include "rankweave/topology.hpp"
#include "rankweave/types.hpp"

using namespace rankweave;

static CostMatrix matrix_for(int n) {
  TopologySpec t;
  const int racks = n >= 64 ? 8 : 2;
  t.levels.push_back({racks, 5.0, 1000.0, 1.0});
  t.levels.push_back({n / racks, 25.0, 1000.0, 4.0});
  t.jitter = 0.1;
  t.seed = 2105;
  CostMatrix m = generate_matrix(t);
  for (double& v : m.rtt_us) v = std::floor(v * 16.0 + 0.5) / 16.0;  // fixed point, as the C4 fixture
  return m;
}

int main(int argc, char** argv) {
#ifdef RW_B200
  // modes: (none) content-keyed matrix cache; "immutable": address-keyed;
  // "resident": address-keyed + resident evaluator (rw_problem_set_resident)
  GpuOptions o = gpu_options();
  const std::string mode = argc > 1 ? argv[1] : "";
  o.immutable_matrices = mode == "immutable" || mode == "resident";
  o.resident_idle_us = mode == "resident" ? 2000 : 0;
  set_gpu_options(o);
#else
  (void)argc;
  (void)argv;
#endif
  struct Case {
    int n;
    Algorithm a;
    HdPairing pair;
  };
  const Case cases[] = {{64, Algorithm::Ring, HdPairing::PaperFormula},
                        {256, Algorithm::Ring, HdPairing::PaperFormula},
                        {1024, Algorithm::Ring, HdPairing::PaperFormula},
                        {4096, Algorithm::Ring, HdPairing::PaperFormula},
                        {1024, Algorithm::HalvingDoubling, HdPairing::XorPairing},
                        {4096, Algorithm::HalvingDoubling, HdPairing::XorPairing},
                        {1024, Algorithm::DoubleBinaryTree, HdPairing::PaperFormula}};
  for (const Case& c : cases) {
    const CostMatrix m = matrix_for(c.n);
    CollectiveSpec spec;
    spec.algorithm = c.a;
    spec.n = c.n;
    spec.size_bytes = 134217728.0;
    spec.hd_pairing = c.pair;
    std::mt19937_64 rng(7);
    std::vector<RankOrder> orders(64, RankOrder::identity(c.n));
    for (auto& o : orders) std::shuffle(o.perm.begin(), o.perm.end(), rng);
    double sink = 0.0;
    for (int k = 0; k < 20; ++k) sink += evaluate(m, orders[k % orders.size()], spec);  // warm (upload, plans)
    std::vector<double> us;
    const int reps = c.n >= 4096 ? 200 : 1000;
    for (int k = 0; k < reps; ++k) {
      const auto t0 = std::chrono::steady_clock::now();
      sink += evaluate(m, orders[k % orders.size()], spec);
      us.push_back(std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
    }
    std::sort(us.begin(), us.end());
    std::printf("{\"n\": %d, \"model\": \"%s\", \"median_us\": %.2f, \"p10_us\": %.2f, \"p90_us\": %.2f, "
                "\"calls\": %d, \"checksum\": %.17g}\n",
                c.n, to_string(c.a), us[us.size() / 2], us[us.size() / 10], us[us.size() * 9 / 10], reps, sink);
  }
  return 0;
}
