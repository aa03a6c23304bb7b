/*
 * rw_oracle.c -- TEST INFRASTRUCTURE ONLY (see rw_oracle.h).
 *
 * A deliberately naive, scalar C restatement of the reference algorithms.
 * Each function names the reference lines it follows (paths relative to the
 * reference root).  Built with plain gcc -O2 (no -ffast-math, no FMA
 * contraction on x86-64 baseline) so the FP64 operation sequence matches the
 * reference's Release build, which also contains no FMA instructions.
 */
#include "rw_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- validation: proj/src/types.cpp:100-110 (order), 127-163 (spec) ---- */

static int is_power_of(long long n, long long base) {
  if (base < 2 || n < 1) return 0;
  while (n % base == 0) n /= base;
  return n == 1;
}

static int ilog_exact(long long n, long long base) {
  int k = 0;
  while (n > 1) {
    n /= base;
    ++k;
  }
  return k;
}

int rwo_validate_spec(const rwo_spec* s) {
  if (s->n < 1) return -1;
  if (!(s->size_bytes > 0.0)) return -1;
  if (s->n == 1) return 0;
  switch (s->algorithm) {
    case 0: return 0;
    case 1:
    case 2: return is_power_of(s->n, 2) ? 0 : -1;
    case 3:
      if (s->bcube_b < 2) return -1;
      return is_power_of(s->n, s->bcube_b) ? 0 : -1;
    default: return -1;
  }
}

int rwo_validate_order(const int32_t* perm, int32_t n) {
  char* seen = (char*)calloc((size_t)n + 1, 1);
  int ok = 0;
  for (int32_t i = 0; i < n; ++i) {
    int32_t v = perm[i];
    if (v < 0 || v >= n || seen[v]) {
      ok = -1;
      break;
    }
    seen[v] = 1;
  }
  free(seen);
  return ok;
}

/* ---- helpers: cost_model.hpp:9 (alias_rank), cost_model.cpp:22-34 ---- */

static int alias(int r, int n) { return ((r % n) + n) % n; }

/* OrderedCost::operator() -- cost_model.cpp:28-33 */
static double hop(const double* m, const int32_t* perm, int n, int mode, int i, int j, double bytes) {
  const int a = perm[alias(i, n)];
  const int b = perm[alias(j, n)];
  const double rtt = m[(size_t)a * (size_t)n + (size_t)b];
  return mode == 0 ? rtt : rtt * bytes;
}

static int cmp_double(const void* x, const void* y) {
  const double a = *(const double*)x, b = *(const double*)y;
  return (a < b) ? -1 : (a > b) ? 1 : 0;
}

/* sorted_sum -- cost_model.cpp:38-43: sort ascending, then a plain serial sum. */
static double sorted_sum(double* v, int count) {
  qsort(v, (size_t)count, sizeof(double), cmp_double);
  double total = 0.0;
  for (int k = 0; k < count; ++k) total += v[k];
  return total;
}

/* round_bytes -- cost_model.cpp:47-51: divisor built by repeated multiplication. */
double rwo_round_bytes(double size_bytes, int32_t base, int32_t round) {
  double divisor = 1.0;
  for (int k = 0; k <= round; ++k) divisor *= (double)base;
  return size_bytes / divisor;
}

/* ring_cost -- cost_model.cpp:59-69: hop i is rtt[perm[i]][perm[i-1]] (wraps). */
double rwo_ring_cost(const double* m, const int32_t* perm, const rwo_spec* s) {
  const int n = s->n;
  if (n == 1) return 0.0;
  double* hops = (double*)malloc(sizeof(double) * (size_t)n);
  for (int i = 0; i < n; ++i) hops[i] = hop(m, perm, n, s->cost_mode, i, i - 1, s->size_bytes);
  const double total = sorted_sum(hops, n);
  free(hops);
  return total;
}

/* halving_doubling_cost -- cost_model.cpp:71-92 */
double rwo_hd_cost(const double* m, const int32_t* perm, const rwo_spec* s) {
  const int n = s->n;
  if (n == 1) return 0.0;
  const int rounds = ilog_exact(n, 2);
  double total = 0.0;
  for (int r = 0; r < rounds; ++r) {
    const double bytes = rwo_round_bytes(s->size_bytes, 2, r);
    const int stride = 1 << r;
    double round_max = 0.0;
    if (s->hd_pairing == 0) {
      for (int j = 0; j < n / 2; ++j) {
        const double c = hop(m, perm, n, s->cost_mode, j, j + stride, bytes);
        if (round_max < c) round_max = c;
      }
    } else {
      for (int j = 0; j < n; ++j) {
        const double c = hop(m, perm, n, s->cost_mode, j, j ^ stride, bytes);
        if (round_max < c) round_max = c;
      }
    }
    total += round_max;
  }
  return total;
}

/* double_binary_tree_cost -- cost_model.cpp:94-116 (recursive T(i, j, shift)). */
static double dbt_tree(const double* m, const int32_t* perm, const rwo_spec* s, double half, int i, int j,
                       int shift) {
  if (i >= j) return 0.0;
  const int n = s->n;
  const int mid = (i + j) / 2;
  const int left_peer = (3 * i + j) / 2 - 1;
  const int right_peer = (i + 3 * j) / 2 + 1;
  const double left = hop(m, perm, n, s->cost_mode, mid + shift, left_peer + shift, half) +
                      dbt_tree(m, perm, s, half, i, mid - 1, shift);
  const double right = hop(m, perm, n, s->cost_mode, mid + shift, right_peer + shift, half) +
                       dbt_tree(m, perm, s, half, mid + 1, j, shift);
  return left < right ? right : left; /* std::max(left, right) */
}

double rwo_dbt_cost(const double* m, const int32_t* perm, const rwo_spec* s) {
  const int n = s->n;
  if (n == 1) return 0.0;
  const double half = s->size_bytes / 2.0;
  const double a = dbt_tree(m, perm, s, half, 0, n - 1, 0);
  const double b = dbt_tree(m, perm, s, half, 0, n - 1, -1);
  return a < b ? b : a;
}

/* bcube_cost -- cost_model.cpp:118-138 */
double rwo_bcube_cost(const double* m, const int32_t* perm, const rwo_spec* s) {
  const int n = s->n;
  if (n == 1) return 0.0;
  const int b = s->bcube_b;
  const int rounds = ilog_exact(n, b);
  double total = 0.0;
  long long stride = 1;
  for (int r = 0; r < rounds; ++r) {
    const double bytes = rwo_round_bytes(s->size_bytes, b, r);
    double round_max = 0.0;
    for (int j = 0; j < n / b; ++j)
      for (int k = 1; k < b; ++k) {
        const double c = hop(m, perm, n, s->cost_mode, j, (int)((j + k * stride) % n), bytes);
        if (round_max < c) round_max = c;
      }
    total += round_max;
    stride *= b;
  }
  return total;
}

/* evaluate -- cost_model.cpp:140-148, with check_inputs (cost_model.cpp:13-19). */
int rwo_evaluate(const double* m, int32_t mat_n, const int32_t* perm, const rwo_spec* s, double* cost) {
  if (rwo_validate_spec(s) != 0) return -1;
  if (mat_n != s->n) return -1;
  if (rwo_validate_order(perm, s->n) != 0) return -1;
  switch (s->algorithm) {
    case 0: *cost = rwo_ring_cost(m, perm, s); return 0;
    case 1: *cost = rwo_hd_cost(m, perm, s); return 0;
    case 2: *cost = rwo_dbt_cost(m, perm, s); return 0;
    case 3: *cost = rwo_bcube_cost(m, perm, s); return 0;
  }
  return -1;
}

int rwo_evaluate_batch(const double* m, int32_t mat_n, const int32_t* perms, int64_t batch,
                       const rwo_spec* s, double* costs) {
  for (int64_t b = 0; b < batch; ++b)
    if (rwo_evaluate(m, mat_n, perms + b * s->n, s, costs + b) != 0) return -1;
  return 0;
}

/* std::next_permutation restated for int arrays. */
static int next_perm(int32_t* a, int n) {
  int i = n - 2;
  while (i >= 0 && a[i] >= a[i + 1]) --i;
  if (i < 0) return 0;
  int j = n - 1;
  while (a[j] <= a[i]) --j;
  int32_t t = a[i];
  a[i] = a[j];
  a[j] = t;
  for (int l = i + 1, r = n - 1; l < r; ++l, --r) {
    t = a[l];
    a[l] = a[r];
    a[r] = t;
  }
  return 1;
}

/* brute_force -- solver.cpp:73-105: strict '<' keeps the first (lex-smallest) minimum. */
int rwo_brute_force(const double* m, const rwo_spec* s, int32_t threshold, int32_t* perm_out,
                    double* cost_out, uint64_t* evals_out) {
  if (rwo_validate_spec(s) != 0) return -1;
  if (s->n > threshold) return -2;
  const int n = s->n;
  int32_t* o = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  for (int i = 0; i < n; ++i) o[i] = i;
  const int pinned = (s->algorithm == 0 && n >= 2) ? 1 : 0;
  uint64_t evals = 0;
  int have = 0;
  double best = 0.0;
  do {
    double c = 0.0;
    rwo_evaluate(m, n, o, s, &c);
    ++evals;
    if (!have || c < best) {
      best = c;
      memcpy(perm_out, o, sizeof(int32_t) * (size_t)n);
      have = 1;
    }
  } while (next_perm(o + pinned, n - pinned));
  free(o);
  *cost_out = best;
  *evals_out = evals;
  return 0;
}

/* distribution_stats -- stats.cpp:64-81 (population stddev, serial sums). */
int rwo_distribution_stats(const double* v, int32_t count, double* out4) {
  if (count < 1) return -1;
  double mn = v[0], mx = v[0], sum = 0.0;
  for (int i = 0; i < count; ++i) {
    if (v[i] < mn) mn = v[i];
    if (mx < v[i]) mx = v[i];
    sum += v[i];
  }
  const double mean = sum / (double)count;
  double sq = 0.0;
  for (int i = 0; i < count; ++i) sq += (v[i] - mean) * (v[i] - mean);
  out4[0] = mn;
  out4[1] = mx;
  out4[2] = mean;
  out4[3] = sqrt(sq / (double)count);
  return count;
}

/* splitmix64 / substream -- solver.cpp:20-28 */
uint64_t rwo_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

uint64_t rwo_substream(uint64_t seed, uint64_t k) { return rwo_splitmix64(seed ^ rwo_splitmix64(k)); }

/* Lookups per evaluation: ring N, hd-paper N/2 log2 N,
 * hd-xor N log2 N, dbt 2N (both trees, self-edges included), bcube (N/B)(B-1) log_B N. */
int64_t rwo_lookups(const rwo_spec* s) {
  const int64_t n = s->n;
  if (n <= 1) return 0;
  switch (s->algorithm) {
    case 0: return n;
    case 1: return (s->hd_pairing == 0 ? n / 2 : n) * ilog_exact(n, 2);
    case 2: return 2 * n;
    case 3: return (n / s->bcube_b) * (s->bcube_b - 1) * ilog_exact(n, s->bcube_b);
  }
  return 0;
}
