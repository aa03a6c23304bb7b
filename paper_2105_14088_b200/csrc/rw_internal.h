// rw_internal.h -- private declarations shared by the librankweave_b200
// translation units (host C++ and CUDA).  Nothing here is part of the ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "rankweave_c.h"

namespace rwb {

// NVTX range around a host-side phase (K1 scoring launches, K2 exhaustive
// search, K3 local search, K4 annealing, and every C ABI entry point), so an
// nsys / ncu --nvtx timeline shows which call issued which kernels.  Header-
// only NVTX v3: a no-op unless a tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// ---------------------------------------------------------------- errors ----
struct Failure : std::runtime_error {
  rw_status status;
  Failure(rw_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};
[[noreturn]] inline void fail_domain(const std::string& m) { throw Failure(RW_ERR_DOMAIN, m); }
[[noreturn]] inline void fail_internal(const std::string& m) { throw Failure(RW_ERR_INTERNAL, m); }
void cuda_check(cudaError_t e, const char* expr, const char* file, int line);
#define RW_CUDA(x) ::rwb::cuda_check((x), #x, __FILE__, __LINE__)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev);
  ~DeviceGuard();
};

// Model ids (= rw_spec.algorithm).
enum Model : int { kRing = 0, kHalvingDoubling = 1, kDoubleBinaryTree = 2, kBCube = 3 };

// ----------------------------------------------------------------- problem --
// Critical-path form of the double binary tree for one n: the transfers of
// expand_schedule (cost_model.cpp:194-222) in depth order, each with the two
// transfers of its sub-interval as children.  Device resident.
struct DbtPlan {
  int n = 0;
  int edges = 0;
  int depths = 0;
  std::vector<int32_t> h_src, h_dst, h_c0, h_c1, h_depth_off;
  // [edge records {src | dst << 16, c0} (one 8-byte load per edge; the second
  // child is c0 + 1, see build_dbt_plan) | depth_off]
  int32_t* d_all = nullptr;
  const uint2* d_rec() const { return reinterpret_cast<const uint2*>(d_all); }
  const int32_t* d_depth_off() const { return d_all + 2 * edges; }
  // [per edge (parent << 8) | depth | per position 8 incident edges, -1 padded]
  int32_t* d_aux = nullptr;
  const int32_t* d_pd() const { return d_aux; }
  const int32_t* d_posedges() const { return d_aux + edges; }
};

struct ResidentServer;  // rw_resident.cu

struct Problem {
  int n = 0;
  int device = 0;
  int storage = RW_STORAGE_F64;
  int frac_bits = 0;
  double scale = 1.0;  // u16: value = q * scale
  bool symmetric = false;
  bool zero_diag = false;
  double max_value = 0.0;
  uint32_t max_q = 0;
  void* d_mat = nullptr;
  size_t mat_bytes = 0;
  int* d_err = nullptr;  // async error slot for *_device calls: {flag, min index}
  int path = RW_PATH_AUTO;   // kernel-path override (rw_problem_set_path)
  uint16_t* d_nb = nullptr;      // candidate lists: K nearest hosts per host (lazy)
  int nb_k = 0;
  std::mutex mu;
  std::unique_ptr<DbtPlan> dbt;
  // Max-based models on FP64 storage: the order-preserving rank of every
  // entry among the matrix's distinct values (u32, half the bytes of FP64)
  // and the rank -> value table; built lazily on the device (rw_rounds_transpose.cu).
  uint32_t* d_rank = nullptr;
  double* d_rank_vals = nullptr;
  uint32_t zero_rank = 0;
  // Resident evaluator for single-order calls (rw_problem_set_resident);
  // read and replaced with std::atomic_load / atomic_store, so a call in
  // flight keeps the server it took alive across a reconfiguration.
  std::shared_ptr<ResidentServer> resident;
  size_t elem_bytes() const { return storage == RW_STORAGE_U16 ? 2 : storage == RW_STORAGE_F32 ? 4 : 8; }
};

// ---------------------------------------------------------------- planning --
constexpr int kMaxRounds = 64;

// Everything a scoring kernel needs for one (problem, spec), computed on the
// host: per-round byte counts exactly as round_bytes() forms them
// (cost_model.cpp:47-51), the ring multiplier, and exactness facts.
struct EvalPlan {
  int model = kRing;
  int n = 0;
  int mode = RW_LATENCY_TIMES_SIZE;
  int pairing = RW_PAIRING_PAPER;
  int bcube_b = 2;
  int rounds = 0;
  double size_bytes = 0.0;
  double half = 0.0;                   // dbt: S / 2
  double round_bytes[kMaxRounds] = {}; // hd / bcube
  double ring_mul = 1.0;               // ring: cost = sum(raw) * ring_mul
  bool ring_int = false;               // ring sums raw u16 codes as integers
  bool bit_exact = false;              // fast path reproduces reference bits
  const DbtPlan* dbt = nullptr;
  bool dbt_int = false;                // dbt on u16: exact integer critical path (see make_plan)
  double dbt_w = 0.0;                  //   value = (sum of codes on the path) * dbt_w
};

// expand_schedule (cost_model.cpp:150-236): rounds of transfers in rank space.
struct Expanded {
  int semantics = RW_SEQUENTIAL_HOPS;
  std::vector<int32_t> off{0};  // round offsets (nrounds + 1)
  std::vector<int32_t> src, dst, parent;
  std::vector<double> bytes;
  int nrounds() const { return static_cast<int>(off.size()) - 1; }
};
Expanded expand_schedule_core(const rw_spec& s);

// Batched simulate_collective (simulate.cpp:52-138) on the device.
struct TopologyDesc {
  std::vector<int32_t> fanout;
  std::vector<double> capacity;  // bandwidth / oversub per level
};
void simulate_batch_device(Problem& p, const TopologyDesc& topo, const Expanded& sch, const int32_t* perms,
                           int64_t batch, double* out);

void validate_spec(const rw_spec& s);                  // types.cpp:143-163 wording
EvalPlan make_plan(Problem& p, const rw_spec& s);       // + n / matrix checks
int64_t lookups_per_eval(const EvalPlan& plan);

// Per-thread, per-device execution context for host-buffer calls.
struct ThreadCtx {
  int device = -1;
  cudaStream_t stream[2] = {nullptr, nullptr};
  cudaEvent_t ev[4] = {};
  int* d_err = nullptr;
  int* h_err = nullptr;  // pinned
  void* d_buf[8] = {};
  size_t d_cap[8] = {};
  void* h_pin = nullptr;  // pinned, mapped host staging for small synchronous calls
  void* d_pin = nullptr;  // its device alias
  size_t h_cap = 0;
  void* scratch(int slot, size_t bytes);
  void* pinned(size_t bytes);
};
ThreadCtx& thread_ctx(int device);
// Frees the calling thread's contexts (streams, scratch, pinned staging);
// for threads the library owns (rw_multi.cpp member workers) before they exit.
void thread_ctx_release();

// Scope of one asynchronous *_device call on a caller's stream: every scratch
// buffer the launch code asks for (ThreadCtx::scratch) comes from the
// stream-ordered allocator on that stream and is freed, stream-ordered, when
// the scope ends.  So concurrent device calls on different streams, or a
// device call followed by a host-buffer call before the stream drains, never
// share buffers; and the allocation is capturable into a CUDA graph.
struct StreamScratch {
  int device;
  cudaStream_t stream;
  StreamScratch* prev;
  void* buf[8] = {};
  size_t cap[8] = {};
  StreamScratch(int device, cudaStream_t stream);
  ~StreamScratch();
  StreamScratch(const StreamScratch&) = delete;
  StreamScratch& operator=(const StreamScratch&) = delete;
  void* get(int slot, size_t bytes);
};

// Reads and clears an error slot; throws the reference's domain_error text.
void raise_order_errors(int* d_err, int* h_err, cudaStream_t st);

// ----------------------------------------------------------------- kernels --
// Batch scoring (K1) of `batch` orders stored row-major (perm_bytes 2 or 4).
// exact: reference-identical ring summation (K0).  validate: bijection check,
// failures recorded in err_slot.
// scratch_slot: first of two ThreadCtx scratch slots this launch may use.
void launch_evaluate(const Problem& p, const EvalPlan& plan, const void* d_perms, int perm_bytes, int64_t batch,
                     double* d_costs, bool exact, bool validate, int* err_slot, cudaStream_t st,
                     int scratch_slot = 2);

// Two-pass ring scoring through an L2-resident predecessor buffer
// (rw_ring_transpose.cu); false when the shape is not supported.
bool launch_ring_transpose(const Problem& p, const EvalPlan& plan, const void* d_perms, int perm_bytes, int64_t batch,
                           double* d_costs, bool validate, int* err_slot, cudaStream_t st, int slot);

// Halving-doubling (paper / xor pairing) through per-round partner-by-host
// slices (rw_rounds_transpose.cu); false when the shape is not supported.
bool launch_rounds_transpose(const Problem& p, const EvalPlan& plan, const void* d_perms, int perm_bytes,
                             int64_t batch, double* d_costs, bool validate, int* err_slot, cudaStream_t st, int slot);

// Generic schedule re-costing (schedule_cost, cost_model.cpp:238-285), one order.
double schedule_cost_device(const Problem& p, int semantics, int nrounds, const int32_t* round_offsets,
                            const int32_t* src, const int32_t* dst, const double* bytes, const int32_t* parent,
                            int cost_mode, const int32_t* perm);

// Exhaustive search over lexicographic indices [first, first+count).
void brute_force_range(const Problem& p, const EvalPlan& plan, uint64_t first, uint64_t count, double* cost_out,
                       uint64_t* index_out);
uint64_t brute_force_space(const rw_spec& s);
void unrank(const rw_spec& s, uint64_t index, int32_t* perm_out);
// Best::offer (solver.cpp:34-46, 73-105): the first order of the enumeration is
// taken unconditionally and later ones only when c < best.  So when its cost is
// NaN, or no order costs less than +inf (argmin index ~0), it is the answer.
// `index` is the argmin over the whole space; returns the reference's index.
uint64_t brute_force_resolve(Problem& p, const EvalPlan& plan, const rw_spec& s, uint64_t index);

// Simulated annealing and local search.
struct AnnealResult {
  std::vector<int32_t> order;
  double cost = 0.0;
  uint64_t evaluations = 0;
  int64_t chain = 0;     // global id of the winning chain
  int64_t chains = 0;
  uint64_t proposals = 0;
  int levels = 0;
  int levels_run = 0;    // temperature levels completed within the budget
  double t0 = 0.0;
  uint64_t setup_evaluations = 0;  // T0 / calibration samples (identical on every shard)
};
AnnealResult anneal_device(Problem& p, const EvalPlan& plan, const rw_solver_config& cfg, const rw_gpu_config& gpu);
void local_search_device(Problem& p, const EvalPlan& plan, int32_t* perms, int64_t batch, int max_rounds,
                         double* costs, uint64_t* evals);

// Random orders (Philox), device side.
void sample_orders_device(int n, int64_t samples, uint64_t seed, uint16_t* d_out, cudaStream_t st);

// ---------------------------------------------------- multi-GPU (rw_multi) --
// Per-member reduction record of a sharded search (device memory): the
// member's best (cost, tie key) and evaluation count, and the all-reduced
// results.
struct alignas(16) SetReduce {
  double cost;
  double min_cost;                // NCCL all-reduce MIN of cost
  unsigned long long key;         // member's tie key (lex index / chain id)
  unsigned long long min_key;     // MIN of the keys of members at min_cost
  unsigned long long evals;
  unsigned long long evals_sum;   // NCCL all-reduce SUM of evals
};
// min_key = (cost == min_cost) ? key : ~0, on the device (one thread).
void launch_select_key(SetReduce* d, cudaStream_t st);

struct ProblemSet;
ProblemSet* problem_set_create(const double* rtt, int n, int hint, const int* devices, int ndev);
void problem_set_destroy(ProblemSet* s);
int problem_set_size(const ProblemSet& s);
Problem& problem_set_member(ProblemSet& s, int i);
int problem_set_device(const ProblemSet& s, int i);
void evaluate_host_orders_set(ProblemSet& s, const rw_spec& spec, const void* perms, int fmt, int bits, int64_t batch,
                              double* costs, bool exact, bool validate);
void brute_force_set(ProblemSet& s, const rw_spec& spec, int32_t* perm_out, double* cost_out, uint64_t* evals_out);
struct AnnealResult;
AnnealResult anneal_set(ProblemSet& s, const rw_spec& spec, const rw_solver_config& cfg, const rw_gpu_config& gpu);

// Host orders of any accepted layout (fmt 4: int32, 2: uint16, 0: packed with
// `bits` per element) through the chunked H2D / score / D2H pipeline.
// index_base: batch index of perms[0] in the caller's batch (error messages).
void evaluate_host_orders_fmt(Problem& p, const EvalPlan& plan, const void* perms, int fmt, int bits, int64_t batch,
                              double* costs, bool exact, bool validate, rw_eval_report* report,
                              int64_t index_base = 0);
int64_t packed_row_bytes(int n, int bits);

// Scores host orders and returns reference-exact costs (used by search code).
// Resident evaluator (rw_resident.cu): idle_us <= 0 stops and frees it.
constexpr int kResidentMaxN = 4096;
void resident_configure(Problem& p, int idle_us);
void resident_release(Problem& p);
// false: not configured, or busy with another thread (use the launched path)
bool resident_evaluate(Problem& p, const EvalPlan& plan, const int32_t* perm, double* cost);

void evaluate_host_orders(Problem& p, const EvalPlan& plan, const int32_t* perms, int64_t batch, double* costs,
                          bool exact, bool validate, rw_eval_report* report);

}  // namespace rwb
