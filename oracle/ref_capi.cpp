// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the UNMODIFIED reference library, compiled by
// oracle/Makefile together with the reference sources read in place from
// /root/reference/proj/src (nothing is copied into this repository).  The
// result, oracle/_ref/librankweave_ref.so, is the "reference arm" of bench.py
// and a cross-check for the C restatement in oracle/rw_oracle.c.  It links no
// product code.
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "rankweave/cost_model.hpp"
#include "rankweave/simulate.hpp"
#include "rankweave/smtlib.hpp"
#include "rankweave/solver.hpp"
#include "rankweave/stats.hpp"
#include "rankweave/topology.hpp"
#include "rankweave/types.hpp"

using namespace rankweave;

namespace {

thread_local std::string g_err;

struct RefSpec {  // same layout as rwo_spec / rw_spec
  int32_t algorithm;
  int32_t n;
  double size_bytes;
  int32_t bcube_b;
  int32_t cost_mode;
  int32_t hd_pairing;
};

CollectiveSpec to_spec(const RefSpec* s) {
  CollectiveSpec c;
  c.algorithm = static_cast<Algorithm>(s->algorithm);
  c.n = s->n;
  c.size_bytes = s->size_bytes;
  c.bcube_b = s->bcube_b;
  c.cost_mode = static_cast<CostMode>(s->cost_mode);
  c.hd_pairing = static_cast<HdPairing>(s->hd_pairing);
  return c;
}

CostMatrix to_matrix(const double* m, int n) {
  CostMatrix cm;
  cm.hosts.reserve(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) cm.hosts.push_back("h" + std::to_string(i));
  cm.rtt_us.assign(m, m + static_cast<size_t>(n) * static_cast<size_t>(n));
  return cm;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const domain_error& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// evaluate() over a batch of int32 permutations using `threads` host threads,
// each calling the reference evaluate() on disjoint slices (evaluate is pure
// and reentrant).
int ref_evaluate_batch(const double* m, int32_t n, const RefSpec* s, const int32_t* perms, int64_t batch,
                       double* costs, int32_t threads) {
  return guarded([&] {
    const CostMatrix cm = to_matrix(m, n);
    const CollectiveSpec spec = to_spec(s);
    if (threads < 1) threads = 1;
    std::vector<std::thread> pool;
    std::atomic<int> failed{0};
    std::string first_err;
    const int64_t per = (batch + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
      const int64_t lo = t * per, hi = std::min<int64_t>(batch, lo + per);
      if (lo >= hi) break;
      pool.emplace_back([&, lo, hi] {
        RankOrder o;
        o.perm.resize(static_cast<size_t>(spec.n));
        try {
          for (int64_t b = lo; b < hi; ++b) {
            std::memcpy(o.perm.data(), perms + b * spec.n, sizeof(int32_t) * static_cast<size_t>(spec.n));
            costs[b] = evaluate(cm, o, spec);
          }
        } catch (const std::exception& e) {
          if (failed.fetch_add(1) == 0) first_err = e.what();
        }
      });
    }
    for (auto& th : pool) th.join();
    if (failed.load()) throw domain_error(first_err);
  });
}

int ref_brute_force(const double* m, const RefSpec* s, int32_t threshold, int32_t* perm_out, double* cost_out,
                    uint64_t* evals_out) {
  return guarded([&] {
    const Solution sol = brute_force(to_matrix(m, s->n), to_spec(s), threshold);
    std::memcpy(perm_out, sol.order.perm.data(), sizeof(int32_t) * sol.order.perm.size());
    *cost_out = sol.cost;
    *evals_out = sol.evaluations;
  });
}

int ref_anneal(const double* m, const RefSpec* s, double budget_s, uint64_t seed, double t0, double cooling,
               int32_t steps, int32_t restarts, int32_t* perm_out, double* cost_out, uint64_t* evals_out) {
  return guarded([&] {
    SolverConfig cfg;
    cfg.budget = std::chrono::duration<double>(budget_s);
    cfg.seed = seed;
    cfg.initial_temperature = t0;
    cfg.cooling = cooling;
    cfg.steps_per_temperature = steps;
    cfg.restarts = restarts;
    const Solution sol = anneal(to_matrix(m, s->n), to_spec(s), cfg);
    std::memcpy(perm_out, sol.order.perm.data(), sizeof(int32_t) * sol.order.perm.size());
    *cost_out = sol.cost;
    *evals_out = sol.evaluations;
  });
}

// Synthetic hierarchical matrix from the reference generator (topology.cpp:40-64).
int ref_generate_matrix(int32_t nlevels, const int32_t* fanout, const double* latency_us, const double* bw,
                        const double* oversub, double jitter, uint64_t seed, double* out, int32_t out_cap) {
  return guarded([&] {
    TopologySpec t;
    for (int l = 0; l < nlevels; ++l) t.levels.push_back({fanout[l], latency_us[l], bw[l], oversub[l]});
    t.jitter = jitter;
    t.seed = seed;
    const CostMatrix cm = generate_matrix(t);
    if (cm.n() > out_cap) throw domain_error("output capacity too small");
    std::memcpy(out, cm.rtt_us.data(), sizeof(double) * cm.rtt_us.size());
  });
}

// Expanded schedule, flattened: per transfer {round, src, dst, parent}, bytes separately.
int ref_expand_schedule(const RefSpec* s, int32_t* semantics, int32_t* quad_out, double* bytes_out, int64_t cap,
                        int64_t* count_out) {
  return guarded([&] {
    const Schedule sch = expand_schedule(to_spec(s));
    *semantics = static_cast<int32_t>(sch.semantics);
    int64_t k = 0;
    for (size_t r = 0; r < sch.rounds.size(); ++r)
      for (const auto& t : sch.rounds[r]) {
        if (k < cap) {
          quad_out[4 * k + 0] = static_cast<int32_t>(r);
          quad_out[4 * k + 1] = t.src;
          quad_out[4 * k + 2] = t.dst;
          quad_out[4 * k + 3] = t.parent;
          bytes_out[k] = t.bytes;
        }
        ++k;
      }
    *count_out = k;
  });
}

int ref_sample_costs(const double* m, const RefSpec* s, int32_t samples, uint64_t seed, double* out) {
  return guarded([&] {
    const auto v = sample_costs(to_matrix(m, s->n), to_spec(s), samples, seed);
    std::memcpy(out, v.data(), sizeof(double) * v.size());
  });
}

// simulate_collective (simulate.cpp:81-138) for a batch of orders on the
// topology's generated matrix.
int ref_simulate_batch(int32_t nlevels, const int32_t* fanout, const double* latency_us, const double* bw,
                       const double* oversub, double jitter, uint64_t seed, const RefSpec* s, const int32_t* perms,
                       int64_t batch, double* out) {
  return guarded([&] {
    TopologySpec t;
    for (int l = 0; l < nlevels; ++l) t.levels.push_back({fanout[l], latency_us[l], bw[l], oversub[l]});
    t.jitter = jitter;
    t.seed = seed;
    const CostMatrix m = generate_matrix(t);
    const CollectiveSpec spec = to_spec(s);
    RankOrder o;
    o.perm.resize(static_cast<size_t>(spec.n));
    for (int64_t b = 0; b < batch; ++b) {
      std::memcpy(o.perm.data(), perms + b * spec.n, sizeof(int32_t) * static_cast<size_t>(spec.n));
      out[b] = simulate_collective(t, m, o, spec);
    }
  });
}

int ref_spearman(const double* x, const double* y, int64_t count, double* out) {
  return guarded([&] { *out = spearman(std::vector<double>(x, x + count), std::vector<double>(y, y + count)); });
}

int ref_distribution_stats(const double* v, int32_t count, double* out4) {
  return guarded([&] {
    const DistributionStats st = distribution_stats(std::vector<double>(v, v + count));
    out4[0] = st.min;
    out4[1] = st.max;
    out4[2] = st.mean;
    out4[3] = st.stddev;
  });
}

// sample_orders (stats.cpp:83-94): the seeded orders themselves.
int ref_sample_orders(int32_t n, int32_t samples, uint64_t seed, int32_t* out) {
  return guarded([&] {
    const auto v = sample_orders(n, samples, seed);
    for (size_t k = 0; k < v.size(); ++k)
      std::memcpy(out + k * static_cast<size_t>(n), v[k].perm.data(), sizeof(int32_t) * static_cast<size_t>(n));
  });
}

// emit_smtlib (smtlib.cpp:104-158): text into a caller buffer (length first).
int ref_emit_smtlib(const double* m, const RefSpec* s, int32_t has_bound, double bound, int32_t cap, char* out,
                    int64_t capacity, int64_t* length_out) {
  return guarded([&] {
    const std::string text = emit_smtlib(to_matrix(m, s->n), to_spec(s),
                                         has_bound ? std::optional<double>(bound) : std::nullopt, cap);
    *length_out = static_cast<int64_t>(text.size());
    if (out && capacity > 0) {
      const size_t k = std::min<size_t>(text.size(), static_cast<size_t>(capacity - 1));
      std::memcpy(out, text.data(), k);
      out[k] = '\0';
    }
  });
}

}  // extern "C"
