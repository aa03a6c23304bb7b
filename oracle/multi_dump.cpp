// multi_dump.cpp -- TEST INFRASTRUCTURE.  Built against this repo's drop-in
// (oracle/Makefile target `multi`): runs the reference C++ API --
// brute_force, anneal, two_stage_solve, evaluate_batch -- with
// GpuOptions::num_devices = argv[1] (a device set with in-process NCCL when
// > 1) and prints every result.  tests/test_multi_device.py runs it at 1, 2
// and 4 devices and requires identical output.
#include <cstdio>
#include <cstdlib>
#include <random>

#include "rankweave/rankweave.hpp"

using namespace rankweave;

static CostMatrix hier(int racks, int per, unsigned seed) {
  TopologySpec t;
  t.levels.push_back({per, 5.0, 1000.0, 1.0});
  t.levels.push_back({racks, 25.0, 1000.0, 4.0});
  t.jitter = 0.1;
  t.seed = seed;
  CostMatrix m = generate_matrix(t);
  for (double& v : m.rtt_us) v = static_cast<double>(static_cast<long long>(v * 16.0 + 0.5)) / 16.0;
  return m;
}

int main(int argc, char** argv) {
  GpuOptions o = gpu_options();
  o.num_devices = argc > 1 ? std::atoi(argv[1]) : 1;
  o.chains = 96;  // fixed chain count: results independent of the device count
  set_gpu_options(o);
  const CostMatrix m11 = hier(4, 3, 7);  // 12 hosts -> take 11
  CostMatrix m;
  for (int i = 0; i < 11; ++i) m.hosts.push_back("h" + std::to_string(i));
  for (int i = 0; i < 11; ++i)
    for (int j = 0; j < 11; ++j) m.rtt_us.push_back(m11.at(i, j));
  for (Algorithm a : {Algorithm::Ring}) {
    CollectiveSpec s;
    s.algorithm = a;
    s.n = 11;
    s.size_bytes = 1.0;
    const Solution b = brute_force(m, s, 11);
    std::printf("brute %s cost=%.17g evals=%llu order=", to_string(a), b.cost, (unsigned long long)b.evaluations);
    for (int v : b.order.perm) std::printf("%d ", v);
    std::printf("\n");
  }
  const CostMatrix m64 = hier(8, 8, 2105);
  for (Algorithm a : {Algorithm::Ring, Algorithm::DoubleBinaryTree}) {
    CollectiveSpec s;
    s.algorithm = a;
    s.n = 64;
    s.size_bytes = 134217728.0;
    SolverConfig cfg;
    cfg.seed = 11;
    cfg.budget = std::chrono::duration<double>(1e6);
    cfg.steps_per_temperature = 32;
    const Solution sa = anneal(m64, s, cfg);
    std::printf("anneal %s cost=%.17g evals=%llu order=", to_string(a), sa.cost, (unsigned long long)sa.evaluations);
    for (int v : sa.order.perm) std::printf("%d ", v);
    std::printf("\n");
    const Solution ts = two_stage_solve(m64, s, cfg);
    std::printf("two_stage %s cost=%.17g method=%s\n", to_string(a), ts.cost, to_string(ts.method));
  }
  std::mt19937_64 rng(5);
  std::vector<RankOrder> orders(5000, RankOrder::identity(64));
  for (auto& ord : orders) std::shuffle(ord.perm.begin(), ord.perm.end(), rng);
  CollectiveSpec s;
  s.n = 64;
  s.size_bytes = 134217728.0;
  double sum = 0.0;
  for (double c : evaluate_batch(m64, orders, s)) sum += c;
  std::printf("evaluate_batch sum=%.17g\n", sum);
  return 0;
}
