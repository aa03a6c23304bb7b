/*
 * rw_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference hot path (rankweave cost models,
 * exhaustive search and distribution statistics).  It is the CHECKER used by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg.  Nothing
 * in the product (paper_2105_14088_b200/) links, loads or calls it.
 *
 * Parity pinning: tests/test_oracle.py checks every function here against
 * (1) the reference's own known-answer tests transcribed from
 *     proj/tests/test_cost_model.cpp / test_solver.cpp / test_stats.cpp,
 * (2) golden vectors in tests/golden/ produced by the reference itself
 *     (oracle/_ref, built from /root/reference sources by oracle/Makefile,
 *     script tests/golden/make_golden.py), and
 * (3) live cross-checks against oracle/_ref on random inputs when present.
 */
#ifndef RW_ORACLE_H
#define RW_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mirrors rankweave::CollectiveSpec (types.hpp:73-80). */
typedef struct {
  int32_t algorithm;  /* 0 ring, 1 halving-doubling, 2 double binary tree, 3 bcube */
  int32_t n;
  double size_bytes;
  int32_t bcube_b;
  int32_t cost_mode;  /* 0 latency-only, 1 latency*size */
  int32_t hd_pairing; /* 0 paper formula, 1 xor */
} rwo_spec;

/* Returns 0 on success, -1 on a domain violation (reference throws). */
int rwo_validate_spec(const rwo_spec* s);
int rwo_validate_order(const int32_t* perm, int32_t n);

double rwo_round_bytes(double size_bytes, int32_t base, int32_t round);
double rwo_ring_cost(const double* m, const int32_t* perm, const rwo_spec* s);
double rwo_hd_cost(const double* m, const int32_t* perm, const rwo_spec* s);
double rwo_dbt_cost(const double* m, const int32_t* perm, const rwo_spec* s);
double rwo_bcube_cost(const double* m, const int32_t* perm, const rwo_spec* s);
/* evaluate(): returns 0 and writes *cost, or -1 on invalid inputs. */
int rwo_evaluate(const double* m, int32_t mat_n, const int32_t* perm, const rwo_spec* s, double* cost);
int rwo_evaluate_batch(const double* m, int32_t mat_n, const int32_t* perms, int64_t batch,
                       const rwo_spec* s, double* costs);

/* brute_force(): lexicographic enumeration, ring pins perm[0] = 0. */
int rwo_brute_force(const double* m, const rwo_spec* s, int32_t threshold, int32_t* perm_out,
                    double* cost_out, uint64_t* evals_out);

/* distribution_stats(): out = {min, max, mean, stddev}; returns count or -1. */
int rwo_distribution_stats(const double* v, int32_t count, double* out4);

uint64_t rwo_splitmix64(uint64_t x);
uint64_t rwo_substream(uint64_t seed, uint64_t k);

/* Number of matrix lookups one evaluation makes (SURVEY 8(d) L(model, N)). */
int64_t rwo_lookups(const rwo_spec* s);

#ifdef __cplusplus
}
#endif
#endif
