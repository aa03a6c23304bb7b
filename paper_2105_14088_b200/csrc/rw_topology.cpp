// rw_topology.cpp -- synthetic hierarchical-datacenter cost matrices for
// fixtures and benchmarks (generate_matrix, proj/src/topology.cpp:40-64;
// validation wording from topology.cpp:20-29).  Host code: input generation,
// not part of the scoring path.  Uses the standard library's mt19937_64 and
// uniform_real_distribution, as the reference does, so a build against the
// same libstdc++ produces the same matrices (checked by tests/test_oracle.py
// against oracle/_ref when it is present).
#include <algorithm>
#include <cmath>
#include <random>
#include <string>
#include <vector>

#include "rw_internal.h"

namespace rwb {

rw_status generate_matrix(int nlevels, const int32_t* fanout, const double* latency, const double* bw,
                          const double* oversub, double jitter, uint64_t seed, double* out, int64_t cap,
                          int32_t* n_out) {
  if (nlevels < 1) fail_domain("topology needs at least one level");
  long long hosts = 1;
  for (int l = 0; l < nlevels; ++l) {
    if (fanout[l] < 1) fail_domain("topology level fanout must be >= 1");
    if (!(latency[l] > 0.0)) fail_domain("topology level latency must be > 0");
    if (!(bw[l] > 0.0)) fail_domain("topology level bandwidth must be > 0");
    if (!(oversub[l] >= 1.0)) fail_domain("topology oversubscription must be >= 1");
    hosts *= fanout[l];
    if (hosts > 1000000) fail_domain("topology host count exceeds 1e6");
  }
  if (hosts < 2) fail_domain("topology fanout product must be >= 2 hosts, got " + std::to_string(hosts));
  if (jitter < 0.0 || jitter >= 1.0) fail_domain("jitter must be in [0, 1)");
  const int n = static_cast<int>(hosts);
  *n_out = n;
  if (!out) return RW_OK;  // size query
  if (cap < static_cast<int64_t>(n) * n) fail_domain("output buffer too small for an n x n matrix");

  // group size below each level: lowest common ancestor = first level whose
  // group contains both hosts
  std::vector<long long> group(static_cast<size_t>(nlevels));
  long long gsz = 1;
  for (int l = 0; l < nlevels; ++l) group[static_cast<size_t>(l)] = (gsz *= fanout[l]);
  auto lca = [&](int i, int j) {
    for (int l = 0; l < nlevels; ++l)
      if (i / group[static_cast<size_t>(l)] == j / group[static_cast<size_t>(l)]) return l;
    return nlevels - 1;
  };

  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> noise(0.0, jitter > 0.0 ? jitter : 1.0);
  for (int i = 0; i < n; ++i) out[static_cast<size_t>(i) * n + i] = 0.0;
  for (int i = 0; i < n; ++i) {
    for (int j = i + 1; j < n; ++j) {
      const int top = lca(i, j);
      double one_way = 0.0;
      for (int l = 0; l <= top; ++l) {
        const double u = jitter > 0.0 ? noise(rng) : 0.0;
        one_way += latency[l] * (1.0 + u);
      }
      const double rtt = 2.0 * one_way;
      out[static_cast<size_t>(i) * n + j] = rtt;
      out[static_cast<size_t>(j) * n + i] = rtt;
    }
  }
  return RW_OK;
}

// Host relabeling used to build benchmark fixtures:
// rl = std::shuffle(iota(n), mt19937_64(seed)); m'[i][j] = m[rl[i]][rl[j]].
void relabel_matrix(double* m, int n, uint64_t seed) {
  std::vector<int> rl(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) rl[static_cast<size_t>(i)] = i;
  std::mt19937_64 rng(seed);
  std::shuffle(rl.begin(), rl.end(), rng);
  std::vector<double> src(m, m + static_cast<size_t>(n) * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      m[static_cast<size_t>(i) * n + j] =
          src[static_cast<size_t>(rl[static_cast<size_t>(i)]) * n + rl[static_cast<size_t>(j)]];
}

}  // namespace rwb
