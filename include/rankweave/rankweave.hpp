// rankweave/rankweave.hpp -- C++ drop-in API of the B200-native solver.
//
// Source-compatible with the reference's public headers
// (proj/include/rankweave/{types,cost_model,solver,stats,smtlib}.hpp): the
// same namespace, types, enumerators, signatures, defaults and exception
// types, so code written against the reference -- including its own test
// suites, see oracle/Makefile `suites` -- compiles unchanged and links against
// librankweave_b200.so instead.  The per-name headers next to this file just
// include it.
//
// Every cost computation (evaluate, the four closed forms, schedule_cost,
// brute_force, anneal, sample_costs) runs on the GPU through the C ABI in
// rankweave_c.h; validation, string conversion and the schedule *structure*
// stay on the host.  The cost matrix is uploaded once and cached by content.
#pragma once

#include <chrono>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace rankweave {

// ------------------------------------------------------------------ errors --
// CLI exit-code mapping as in the reference: io_error 2, domain_error 3, net_error 4.
class domain_error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class io_error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class net_error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

// ------------------------------------------------------------------- enums --
enum class Algorithm { Ring, HalvingDoubling, DoubleBinaryTree, BCube };
enum class CostMode { LatencyOnly, LatencyTimesSize };
enum class HdPairing { PaperFormula, XorPairing };
enum class ScheduleSemantics { SequentialHops, BulkSynchronousRounds, CriticalPath };
enum class SolveMethod { BruteForce, Anneal, External };

const char* to_string(Algorithm a);
const char* to_string(CostMode m);
const char* to_string(HdPairing p);
const char* to_string(SolveMethod m);
Algorithm algorithm_from_string(const std::string& s);  // ring|hd|dbt|bcube
CostMode cost_mode_from_string(const std::string& s);   // latency|latency-size
HdPairing hd_pairing_from_string(const std::string& s); // paper|xor
SolveMethod solve_method_from_string(const std::string& s);

// ------------------------------------------------------------- value types --
// N x N pairwise cost in microseconds, row-major: at(i, j) is host i -> host j.
struct CostMatrix {
  std::vector<std::string> hosts;
  std::vector<double> rtt_us;

  CostMatrix() = default;
  CostMatrix(std::vector<std::string> host_ids, std::vector<std::vector<double>> rows);

  int n() const { return static_cast<int>(hosts.size()); }
  double at(int i, int j) const { return rtt_us[static_cast<std::size_t>(i) * hosts.size() + static_cast<std::size_t>(j)]; }
  double& at(int i, int j) { return rtt_us[static_cast<std::size_t>(i) * hosts.size() + static_cast<std::size_t>(j)]; }
  std::vector<std::vector<double>> rows() const;
};

// perm[rank] = index of the host that holds `rank`; a bijection on [0, n).
struct RankOrder {
  std::vector<int> perm;
  static RankOrder identity(int n);
  int size() const { return static_cast<int>(perm.size()); }
};

struct CollectiveSpec {
  Algorithm algorithm = Algorithm::Ring;
  int n = 0;
  double size_bytes = 0.0;
  int bcube_b = 2;
  CostMode cost_mode = CostMode::LatencyTimesSize;
  HdPairing hd_pairing = HdPairing::PaperFormula;
};

struct Transfer {
  int src = 0;
  int dst = 0;
  double bytes = 0.0;
  int parent = -1;
};

struct Schedule {
  Algorithm algorithm = Algorithm::Ring;
  int node_count = 0;
  ScheduleSemantics semantics = ScheduleSemantics::SequentialHops;
  std::vector<std::vector<Transfer>> rounds;
};

struct DistributionStats {
  double min = 0.0;
  double max = 0.0;
  double mean = 0.0;
  double stddev = 0.0;
  int count = 0;
};

// --------------------------------------------------------------- validation --
void validate(const CostMatrix& m);
bool is_symmetric(const CostMatrix& m);
void validate(const RankOrder& order, int n);
void validate(const CollectiveSpec& spec);
RankOrder rotated(const RankOrder& order, int k);
RankOrder inverse(const RankOrder& order);
bool is_power_of(long long n, long long base);
int ilog(long long n, long long base);
double total_wire_bytes(const Schedule& s);

// --------------------------------------------------------------- cost model --
inline int alias_rank(int r, int n) { return ((r % n) + n) % n; }
double round_bytes(double size_bytes, int base, int round);
double transfer_cost(const CostMatrix& m, int i, int j, double bytes, CostMode mode);
double ring_cost(const CostMatrix& m, const RankOrder& order, const CollectiveSpec& spec);
double halving_doubling_cost(const CostMatrix& m, const RankOrder& order, const CollectiveSpec& spec);
double double_binary_tree_cost(const CostMatrix& m, const RankOrder& order, const CollectiveSpec& spec);
double bcube_cost(const CostMatrix& m, const RankOrder& order, const CollectiveSpec& spec);
double evaluate(const CostMatrix& m, const RankOrder& order, const CollectiveSpec& spec);
Schedule expand_schedule(const CollectiveSpec& spec);
double schedule_cost(const Schedule& s, const CostMatrix& m, const RankOrder& order, CostMode mode);

// ------------------------------------------------------------------- solver --
struct SolverConfig {
  std::chrono::duration<double> budget{10.0};
  std::uint64_t seed = 0;
  double initial_temperature = 0.0;
  double cooling = 0.995;
  int steps_per_temperature = 0;
  int restarts = 4;
  int brute_force_threshold = 10;
};
void validate(const SolverConfig& cfg);

struct Solution {
  RankOrder order;
  double cost = 0.0;
  SolveMethod method = SolveMethod::BruteForce;
  std::uint64_t evaluations = 0;
};

Solution brute_force(const CostMatrix& m, const CollectiveSpec& spec,
                     int threshold = SolverConfig{}.brute_force_threshold);
RankOrder neighbor(const RankOrder& order, std::mt19937_64& rng);
Solution anneal(const CostMatrix& m, const CollectiveSpec& spec, const SolverConfig& cfg);

struct TwoStageOptions {
  std::string emit_smt_path;
  std::string external_model_path;
  std::function<void(const std::string&)> log;
};
Solution two_stage_solve(const CostMatrix& m, const CollectiveSpec& spec, const SolverConfig& cfg,
                         const TwoStageOptions& opts = {});

// -------------------------------------------------------------------- stats --
double spearman(const std::vector<double>& xs, const std::vector<double>& ys);
DistributionStats distribution_stats(const std::vector<double>& values);
DistributionStats sample_cost_distribution(const CostMatrix& m, const CollectiveSpec& spec, int n_samples,
                                           std::uint64_t seed);
std::vector<double> sample_costs(const CostMatrix& m, const CollectiveSpec& spec, int n_samples, std::uint64_t seed);
std::vector<RankOrder> sample_orders(int n, int n_samples, std::uint64_t seed);

// ------------------------------------------------------------------- smtlib --
std::string emit_smtlib(const CostMatrix& m, const CollectiveSpec& spec,
                        std::optional<double> upper_bound = std::nullopt, int emission_cap = 64);
RankOrder parse_model_file(const std::string& text, int n);
bool balanced_sexpr(const std::string& text);

// ------------------------------------------- topology / flow simulator -----
// (topology.hpp / simulate.hpp: synthetic inputs and the validation ground
// truth; not on the solver path, kept for the SPEC's validate workflow)
struct TopologyLevel {
  int fanout = 0;
  double latency_us = 0.0;
  double bandwidth_Bpus = 0.0;
  double oversub = 1.0;
};
struct TopologySpec {
  std::vector<TopologyLevel> levels;
  double jitter = 0.0;
  std::uint64_t seed = 0;
  int host_count() const;
};
void validate(const TopologySpec& topo);
int lca_level(const TopologySpec& topo, int i, int j);
CostMatrix generate_matrix(const TopologySpec& topo);
double simulate_collective(const TopologySpec& topo, const RankOrder& order, const CollectiveSpec& spec);
double simulate_collective(const TopologySpec& topo, const CostMatrix& m, const RankOrder& order,
                           const CollectiveSpec& spec);

// ------------------------------------------------- GPU extensions (new) -----
// Batched simulate_collective on the GPU.
std::vector<double> simulate_batch(const TopologySpec& topo, const CostMatrix& m, const std::vector<RankOrder>& orders,
                                   const CollectiveSpec& spec);
// Process-wide defaults applied by anneal() / two_stage_solve().
struct GpuOptions {
  int device = -1;      // -1: current CUDA device
  int chains = 0;       // SA chains; <= 0: 4 per SM (at least cfg.restarts)
  bool exact_batch = false;
  // Device copies of CostMatrix are cached by exact content (a byte compare
  // against a host shadow on every call).  true: key the cache by the matrix
  // storage address and size instead -- the caller promises not to mutate a
  // CostMatrix it has passed before (O(1) per call instead of O(N^2)).
  bool immutable_matrices = false;
  // > 1: brute_force, anneal, two_stage_solve and evaluate_batch run over that
  // many devices of this process (the first num_devices visible ones, or all
  // of them when the count exceeds the visible devices) through an
  // in-process NCCL communicator; 0: every visible device.  Results do not
  // depend on the device count for a fixed `chains`.
  int num_devices = 1;
  // > 0: evaluate() is served by a resident evaluator on the device (one CTA
  // that polls a mapped mailbox; no kernel launch per call), which leaves
  // after this many microseconds without a call.  See rw_problem_set_resident.
  int resident_idle_us = 0;
};
void set_gpu_options(const GpuOptions& opts);
GpuOptions gpu_options();

// Batched evaluate(): one GPU launch for many orders.
std::vector<double> evaluate_batch(const CostMatrix& m, const std::vector<RankOrder>& orders,
                                   const CollectiveSpec& spec);

}  // namespace rankweave
