/*
 * rankweave_c.h -- C ABI of the B200-native rank-reordering solver
 * (librankweave_b200.so).  Plain pointers and sizes only; no C++ or torch
 * types cross this boundary.
 *
 * The reference (arxiv/paper_2105_14088, "rankweave") exposes its hot path as
 * C++ free functions in proj/include/rankweave/ headers and has no C ABI, FFI or
 * Python binding (proj/python/CMakeLists.txt:1 is a placeholder).  Each entry
 * point below names the reference interface it replaces; the C++ drop-in
 * headers in include/rankweave/ are implemented on top of these calls, and
 * the Python package paper_2105_14088_b200 binds them with ctypes
 * (INTEGRATION.md shows the bindings).
 *
 * Conventions
 *  - Every call returns rw_status.  On failure rw_last_error() returns the
 *    message of the failing call on the calling thread.  RW_ERR_DOMAIN carries
 *    the reference's domain_error text (types.hpp:12-27, exit code 3).
 *  - All buffers are caller-owned.  The only library-owned object is the
 *    opaque rw_problem: one cost matrix resident in device memory.
 *  - Host-buffer entry points are synchronous.  *_device entry points take
 *    device pointers and a cudaStream_t passed as void* and are asynchronous.
 *  - Thread safety: distinct threads may call concurrently; every host-buffer
 *    call runs on a per-thread stream of the problem's device.
 */
#ifndef RANKWEAVE_C_H
#define RANKWEAVE_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RW_ABI_VERSION 3  /* 2: uint16 / packed host orders, device sets (NCCL), host logic, GPU options, Philox samplers;
                             3: resident evaluator (rw_problem_set_resident, rw_gpu_options.resident_idle_us) */

typedef enum rw_status {
  RW_OK = 0,
  RW_ERR_IO = 2,       /* rankweave::io_error      (types.hpp:21-24) */
  RW_ERR_DOMAIN = 3,   /* rankweave::domain_error  (types.hpp:14-17) */
  RW_ERR_CUDA = 5,     /* CUDA runtime failure (no device, OOM, fault) */
  RW_ERR_NCCL = 6,     /* collective failure (multi-GPU helpers) */
  RW_ERR_INTERNAL = 7
} rw_status;

/* rankweave::Algorithm / CostMode / HdPairing (types.hpp:29-31). */
enum { RW_RING = 0, RW_HALVING_DOUBLING = 1, RW_DOUBLE_BINARY_TREE = 2, RW_BCUBE = 3 };
enum { RW_LATENCY_ONLY = 0, RW_LATENCY_TIMES_SIZE = 1 };
enum { RW_PAIRING_PAPER = 0, RW_PAIRING_XOR = 1 };
/* rankweave::ScheduleSemantics (types.hpp:99-103). */
enum { RW_SEQUENTIAL_HOPS = 0, RW_BULK_SYNCHRONOUS_ROUNDS = 1, RW_CRITICAL_PATH = 2 };
/* rankweave::SolveMethod (solver.hpp:26). */
enum { RW_METHOD_BRUTE_FORCE = 0, RW_METHOD_ANNEAL = 1, RW_METHOD_EXTERNAL = 2 };

/* Device storage of the matrix (chosen at rw_problem_create). */
enum {
  RW_STORAGE_AUTO = 0, /* u16 fixed point if exact, else f32 if exact, else f64 */
  RW_STORAGE_U16 = 1,  /* value = q * 2^-frac_bits, q < 65536 */
  RW_STORAGE_F32 = 2,
  RW_STORAGE_F64 = 3
};

/* rw_evaluate_batch* flags. */
enum {
  RW_EVAL_EXACT = 1u << 0,       /* reference-identical ring summation (sorted) */
  RW_EVAL_NO_VALIDATE = 1u << 1  /* skip the per-order bijection check */
};

/* rankweave::CollectiveSpec (types.hpp:73-80). */
typedef struct rw_spec {
  int32_t algorithm;
  int32_t n;
  double size_bytes;
  int32_t bcube_b;
  int32_t cost_mode;
  int32_t hd_pairing;
} rw_spec;

/* rankweave::SolverConfig (solver.hpp:14-22); budget in seconds. */
typedef struct rw_solver_config {
  double budget_s;
  uint64_t seed;
  double initial_temperature;
  double cooling;
  int32_t steps_per_temperature;
  int32_t restarts;
  int32_t brute_force_threshold;
  int32_t reserved;
} rw_solver_config;

/* GPU extension of the search configuration (not in the reference). */
typedef struct rw_gpu_config {
  int32_t chains;       /* SA chains on this call; <= 0: max(restarts, 4 x SMs) */
  int32_t chain_begin;  /* global id of the first chain (multi-GPU sharding) */
  int32_t chain_total;  /* total chains across all ranks (<= 0: chains) */
  int32_t schedule;     /* temperatures when initial_temperature <= 0:
                           0 = reference rule (T0 = stddev of 100 random-order
                               costs, floor T0 * 1e-6; solver.cpp:152-167);
                           1 = calibrated (ring): T0 = 0.1 x mean uphill 2-opt
                               delta of random orders, floor = 5th-percentile
                               uphill delta / 20; the calibration samples are
                               counted as evaluations */
  int64_t max_proposals;/* total evaluation budget of the call (T0/calibration
                           samples + chain starts + proposals); the steps per
                           temperature level are derived from it (0: use
                           steps_per_temperature) */
} rw_gpu_config;

typedef struct rw_problem rw_problem;

typedef struct rw_problem_info {
  int32_t n;
  int32_t device;
  int32_t storage;      /* RW_STORAGE_U16 / F32 / F64 */
  int32_t frac_bits;    /* u16 only */
  int32_t symmetric;
  int32_t zero_diagonal;
  int64_t device_bytes; /* matrix bytes resident on the device */
  double max_value;
} rw_problem_info;

/* Per-call search report (optional out-parameter of rw_anneal). */
typedef struct rw_search_report {
  int64_t winner_chain;   /* global id of the chain that produced the result */
  int64_t chains;         /* chains run by this call */
  int64_t proposals;      /* Metropolis proposals (sequential-equivalent) */
  int32_t levels;         /* temperature levels in the schedule */
  int32_t levels_run;     /* levels completed before the budget expired */
  double initial_temperature;
  double seconds;         /* wall time of the call */
} rw_search_report;

/* Per-call evaluation report (optional out-parameter). */
typedef struct rw_eval_report {
  int32_t bit_exact;    /* 1: every cost equals the reference's bits */
  int32_t kernel;       /* internal kernel id */
  float kernel_ms;      /* device time of the scoring kernels */
  int64_t lookups;      /* matrix lookups performed */
} rw_eval_report;

/* ---- library ---------------------------------------------------------- */
const char* rw_last_error(void);
int32_t rw_abi_version(void);
/* Number of visible CUDA devices (0 when none). */
int32_t rw_device_count(void);

/* validate(CollectiveSpec) (types.cpp:143-163): RW_ERR_DOMAIN with the
 * reference's message when the spec is invalid. */
rw_status rw_validate_spec(const rw_spec* spec);

/* ---- problem: the device-resident CostMatrix (types.hpp:42-53) --------- */
/* Validates like the reference evaluate path (square, n >= 1); the matrix
 * itself is NOT validated (evaluate() does not call validate(CostMatrix)). */
rw_status rw_problem_create(const double* rtt_us, int32_t n, int32_t storage_hint, int32_t device,
                            rw_problem** out);
rw_status rw_problem_destroy(rw_problem* p);
rw_status rw_problem_get_info(const rw_problem* p, rw_problem_info* out);
/* Kernel-path override for A/B measurements and tests, used when the matrix
 * exceeds one CTA's shared memory (results are identical on every path):
 *   RW_PATH_AUTO       default: the transpose path for ring up to N = 1536, for
 *                      halving-doubling (512 <= N <= 16384, power of 2) and for
 *                      BCube with B = 2 or 4 (B = 8: FP64 matrices from N = 2048),
 *                      the L2-gather kernels otherwise
 *   RW_PATH_L2_GATHER  one warp per order, random gathers from the L2-resident matrix
 *   RW_PATH_CLUSTER    ring only: row-partitioned thread-block cluster, DSMEM hop
 *                      routing (u16 matrices, N = 64*C, C <= 16)
 *   RW_PATH_TRANSPOSE  two passes through an HBM exchange buffer (predecessor /
 *                      partner by host, grouped by matrix row block; paper pairing
 *                      and BCube: only each block's sources); lookups from a
 *                      shared-memory row block (ring: N % 8 == 0, 256 <= N <= 8192) */
enum { RW_PATH_AUTO = 0, RW_PATH_L2_GATHER = 1, RW_PATH_CLUSTER = 2, RW_PATH_TRANSPOSE = 3 };
rw_status rw_problem_set_path(rw_problem* p, int32_t path);

/* Resident evaluator for single-order rw_evaluate calls (N <= 4096): one CTA
 * stays resident on the problem's device and serves them through a mailbox in
 * mapped pinned host memory, so a call costs no kernel launch (B200, N=64:
 * ~6 us instead of ~13 us).  The CTA leaves after idle_us without a call (at
 * most 100000; and after 5 ms of continuous use, relaunched transparently), so
 * a device-wide synchronisation elsewhere waits at most that long.
 * idle_us <= 0 stops it.  Results are bit-identical to the launched path; a
 * call made while another thread holds the server takes the launched path. */
rw_status rw_problem_set_resident(rw_problem* p, int32_t idle_us);

/* ---- cost model (cost_model.hpp:28-36) --------------------------------- */
/* evaluate(m, order, spec): reference-identical bits for every matrix. */
rw_status rw_evaluate(const rw_problem* p, const rw_spec* spec, const int32_t* perm, double* cost);
/* B orders (row-major B x n int32, host) -> B costs (host). */
rw_status rw_evaluate_batch(const rw_problem* p, const rw_spec* spec, const int32_t* perms, int64_t batch,
                            double* costs, uint32_t flags, rw_eval_report* report);
/* Host orders as uint16 (n <= 65536): half the host-to-device bytes of int32. */
rw_status rw_evaluate_batch_u16(const rw_problem* p, const rw_spec* spec, const uint16_t* perms, int64_t batch,
                                double* costs, uint32_t flags, rw_eval_report* report);
/* Packed host orders: `bits` per element (1..16, 2^bits >= n); element i of
 * an order occupies bits [i*bits, (i+1)*bits) of the order's little-endian
 * 32-bit word stream, and every order starts on a 16-byte boundary:
 * rw_packed_row_bytes(n, bits) bytes per order (-1 for invalid arguments).
 * At n = 1024 and 10 bits an order is 1280 bytes, 5/16 of int32.  The
 * orders are unpacked on the device; costs and errors as rw_evaluate_batch. */
int64_t rw_packed_row_bytes(int32_t n, int32_t bits);
rw_status rw_pack_orders(const int32_t* perms, int32_t n, int64_t batch, int32_t bits, void* out);
rw_status rw_evaluate_batch_packed(const rw_problem* p, const rw_spec* spec, const void* packed, int32_t bits,
                                   int64_t batch, double* costs, uint32_t flags, rw_eval_report* report);
/* Same with device buffers; perm_bytes is 2 (uint16) or 4 (int32). Async on
 * `stream`.  Validation failures are reported by the next rw_sync_errors(). */
rw_status rw_evaluate_batch_device(const rw_problem* p, const rw_spec* spec, const void* d_perms,
                                   int32_t perm_bytes, int64_t batch, double* d_costs, void* stream,
                                   uint32_t flags);
/* Collect asynchronous validation errors raised by *_device calls on p. */
rw_status rw_sync_errors(const rw_problem* p, void* stream);
/* schedule_cost(expand_schedule(spec), m, order, mode) (cost_model.hpp:31-36):
 * transfers are flattened round by round; round_offsets has nrounds+1 entries. */
rw_status rw_schedule_cost(const rw_problem* p, int32_t semantics, int32_t nrounds, const int32_t* round_offsets,
                           const int32_t* src, const int32_t* dst, const double* bytes, const int32_t* parent,
                           int32_t cost_mode, const int32_t* perm, double* cost);

/* ---- exhaustive search (solver.hpp:37-42, solver.cpp:73-105) ----------- */
rw_status rw_brute_force(const rw_problem* p, const rw_spec* spec, int32_t threshold, int32_t* perm_out,
                         double* cost_out, uint64_t* evals_out);
/* Size of the enumerated space ((n-1)! for ring, n! otherwise). */
rw_status rw_brute_force_space(const rw_spec* spec, uint64_t* count_out);
/* One shard [first, first+count) of the lexicographic space: (min cost, min
 * lex index).  Used by the multi-GPU driver; rw_unrank maps an index back. */
rw_status rw_brute_force_range(const rw_problem* p, const rw_spec* spec, uint64_t first, uint64_t count,
                               double* cost_out, uint64_t* index_out);
rw_status rw_unrank(const rw_spec* spec, uint64_t index, int32_t* perm_out);

/* ---- heuristic search (solver.hpp:44-53, solver.cpp:141-202) ----------- */
rw_status rw_anneal(const rw_problem* p, const rw_spec* spec, const rw_solver_config* cfg,
                    const rw_gpu_config* gpu, int32_t* perm_out, double* cost_out, uint64_t* evals_out,
                    rw_search_report* report);
/* Batched best-improvement local search (ring: 2-opt + swap + or-opt with O(1)
 * deltas; tree / halving-doubling / BCube: swap + 2-opt by full evaluation):
 * orders are improved in place; costs_out receives reference-exact costs. */
rw_status rw_local_search(const rw_problem* p, const rw_spec* spec, int32_t* perms_inout, int64_t batch,
                          int32_t max_rounds, double* costs_out, uint64_t* evals_out);

/* ---- statistics (stats.hpp:18-28) -------------------------------------- */
/* sample_orders (stats.cpp:83-94): the reference's orders bit for bit -- one
 * std::mt19937_64(seed) stream, identity std::shuffle'd per sample (host). */
rw_status rw_sample_orders(int32_t n, int32_t samples, uint64_t seed, int32_t* perms_out);
/* sample_costs (stats.cpp:96-103): those orders, scored on the GPU with the
 * reference-identical summation (costs equal the reference's bits). */
rw_status rw_sample_costs(const rw_problem* p, const rw_spec* spec, int32_t samples, uint64_t seed,
                          double* costs_out);
/* GPU extension: uniform random orders from a counter-based Philox stream
 * generated on the device (deterministic per seed; NOT the reference's
 * sequence), and their reference-exact costs. */
rw_status rw_sample_orders_philox(int32_t n, int32_t samples, uint64_t seed, int32_t* perms_out);
rw_status rw_sample_costs_philox(const rw_problem* p, const rw_spec* spec, int32_t samples, uint64_t seed,
                                 double* costs_out);

/* ---- schedules and the flow simulator ---------------------------------- */
/* expand_schedule (cost_model.hpp:33): call once with NULL arrays to get
 * *nrounds_out and *count_out, then with round_offsets[nrounds+1] and
 * src/dst/parent/bytes[count]. */
rw_status rw_expand_schedule(const rw_spec* spec, int32_t* semantics_out, int32_t* nrounds_out, int64_t* count_out,
                             int32_t* round_offsets, int32_t* src, int32_t* dst, int32_t* parent, double* bytes);
/* simulate_collective(topo, m, order, spec) (simulate.hpp:24-25) for a batch
 * of host orders; p must hold generate_matrix(topo).  bandwidth/oversub per
 * level give the link capacities (bandwidth / oversub). */
rw_status rw_simulate_batch(const rw_problem* p, int32_t nlevels, const int32_t* fanout, const double* bandwidth,
                            const double* oversub, const rw_spec* spec, const int32_t* perms, int64_t batch,
                            double* out);

/* ---- synthetic inputs (topology.hpp:40, out of scope for kernels) ------ */
/* generate_matrix(TopologySpec): writes n*n doubles; returns n in *n_out. */
rw_status rw_generate_matrix(int32_t nlevels, const int32_t* fanout, const double* latency_us,
                             const double* bandwidth, const double* oversub, double jitter, uint64_t seed,
                             double* out, int64_t out_capacity, int32_t* n_out);
/* Fixture relabeling: rl = std::shuffle(iota(n), mt19937_64(seed)),
 * m'[i][j] = m[rl[i]][rl[j]] (in place). */
rw_status rw_relabel_matrix(double* m, int32_t n, uint64_t seed);

/* ---- multi-GPU in one process (north star (4)) ------------- */
/* A cost matrix replicated on a set of this process's devices (devices =
 * NULL or ndevices <= 0: every visible device), with an in-process NCCL
 * communicator over them (ncclCommInitAll; libnccl.so.2 is loaded on first
 * use).  The matrix is analysed and uploaded once and ncclBroadcast from the
 * first member.  Calls on one set are serialised. */
typedef struct rw_problem_set rw_problem_set;
enum { RW_LAYOUT_PACKED = 0, RW_LAYOUT_U16 = 2, RW_LAYOUT_INT32 = 4 };
rw_status rw_problem_set_create(const double* rtt_us, int32_t n, int32_t storage_hint, const int32_t* devices,
                                int32_t ndevices, rw_problem_set** out);
rw_status rw_problem_set_destroy(rw_problem_set* s);
rw_status rw_problem_set_devices(const rw_problem_set* s, int32_t* ndevices_out, int32_t* devices_out);
/* Borrowed handle of member `index` (valid while the set lives). */
rw_status rw_problem_set_member(const rw_problem_set* s, int32_t index, rw_problem** out);
/* One host batch (layout RW_LAYOUT_*; `bits` for packed) split into
 * contiguous slices, one per device, each over its own PCIe link. */
rw_status rw_evaluate_batch_set(const rw_problem_set* s, const rw_spec* spec, const void* perms, int32_t layout,
                                int32_t bits, int64_t batch, double* costs, uint32_t flags);
/* brute_force over the set: the lexicographic range split evenly; winner by
 * ncclAllReduce MIN on the cost, then MIN on the lex index at that cost --
 * the same order, cost and evaluation count as one device. */
rw_status rw_brute_force_set(const rw_problem_set* s, const rw_spec* spec, int32_t threshold, int32_t* perm_out,
                             double* cost_out, uint64_t* evals_out);
/* anneal over the set: global chain ids [0, chains) split over the members
 * (gpu->chains <= 0: the single-device default per member); winner by
 * ncclAllReduce MIN on the cost, MIN on the chain id, ncclBroadcast of the
 * order from its owner.  For a fixed chain count the result does not depend
 * on the number of devices. */
rw_status rw_anneal_set(const rw_problem_set* s, const rw_spec* spec, const rw_solver_config* cfg,
                        const rw_gpu_config* gpu, int32_t* perm_out, double* cost_out, uint64_t* evals_out,
                        rw_search_report* report);

/* rankweave::GpuOptions of the C++ drop-in (rankweave.hpp), process-wide:
 * what evaluate / brute_force / anneal / two_stage_solve use when called
 * through the reference's C++ API or rw_two_stage_solve. */
typedef struct rw_gpu_options {
  int32_t device;              /* -1: current CUDA device */
  int32_t chains;              /* SA chains; <= 0: max(restarts, 4 x SMs) per device */
  int32_t exact_batch;         /* evaluate_batch with the reference's summation order */
  int32_t immutable_matrices;  /* cache device matrices by address, not content */
  int32_t num_devices;         /* > 1 (0: all visible): device sets with in-process NCCL */
  int32_t resident_idle_us;    /* > 0: evaluate() through a resident evaluator (rw_problem_set_resident) */
} rw_gpu_options;
rw_status rw_set_gpu_options(const rw_gpu_options* opts);
rw_status rw_get_gpu_options(rw_gpu_options* out);

/* ---- host logic (one implementation, shared with the C++ drop-in) ------ */
/* distribution_stats (stats.cpp:64-81): out4 = {min, max, mean, stddev}. */
rw_status rw_distribution_stats(const double* values, int64_t count, double* out4);
/* spearman (stats.cpp:56-62); the lengths are passed separately so the
 * reference's length-mismatch error is reproduced. */
rw_status rw_spearman(const double* xs, const double* ys, int64_t count_x, int64_t count_y, double* out);
/* parse_model_file (smtlib.cpp:160-186): NUL-terminated text -> perm_out[n]. */
rw_status rw_parse_model_file(const char* text, int32_t n, int32_t* perm_out);
/* balanced_sexpr (smtlib.cpp:188-203): *out = 1 when balanced. */
rw_status rw_balanced_sexpr(const char* text, int32_t* out);
/* emit_smtlib (smtlib.cpp:104-158), byte-identical text.  Call with
 * out = NULL to get *length_out; then with capacity >= length + 1. */
rw_status rw_emit_smtlib(const double* rtt_us, int32_t n, const rw_spec* spec, int32_t has_bound, double bound,
                         int32_t emission_cap, char* out, int64_t capacity, int64_t* length_out);
/* two_stage_solve (solver.cpp:204-261): routing, SMT side file, external
 * model; `log` (optional) receives each log line.  method_out: RW_METHOD_*. */
typedef void (*rw_log_fn)(const char* message, void* user);
rw_status rw_two_stage_solve(const double* rtt_us, int32_t n, const rw_spec* spec, const rw_solver_config* cfg,
                             const char* emit_smt_path, const char* external_model_path, rw_log_fn log, void* user,
                             int32_t* perm_out, double* cost_out, int32_t* method_out, uint64_t* evals_out);

#ifdef __cplusplus
}
#endif
#endif /* RANKWEAVE_C_H */
