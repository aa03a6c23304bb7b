// rw_capi.cpp -- the extern "C" boundary (include/rankweave_c.h).  Every
// entry point validates its arguments with the reference's wording, maps C++
// exceptions onto rw_status and records the message for rw_last_error().
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <numeric>
#include <random>
#include <string>
#include <vector>

#include "rankweave/rankweave.hpp"
#include "rw_internal.h"

namespace rwb {
Problem* problem_create(const double* rtt, int n, int hint, int device);
void problem_destroy(Problem* p);
rw_status generate_matrix(int nlevels, const int32_t* fanout, const double* latency, const double* bw,
                          const double* oversub, double jitter, uint64_t seed, double* out, int64_t cap, int32_t* n_out);
void relabel_matrix(double* m, int n, uint64_t seed);
}  // namespace rwb

struct rw_problem {
  rwb::Problem* impl;
};

struct rw_problem_set {
  rwb::ProblemSet* impl;
  std::vector<rw_problem> members;  // borrowed handles of the member problems
};

namespace {

thread_local std::string g_last_error;

template <class F>
rw_status guarded(F&& f) {
  try {
    f();
    g_last_error.clear();
    return RW_OK;
  } catch (const rwb::Failure& e) {
    g_last_error = e.what();
    return e.status;
  } catch (const rankweave::domain_error& e) {  // host logic shared with the C++ drop-in
    g_last_error = e.what();
    return RW_ERR_DOMAIN;
  } catch (const rankweave::io_error& e) {
    g_last_error = e.what();
    return RW_ERR_IO;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return RW_ERR_INTERNAL;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return RW_ERR_INTERNAL;
  }
}

rwb::Problem& get(const rw_problem* p) {
  if (!p || !p->impl) rwb::fail_domain("null rw_problem");
  return *p->impl;
}

void need(const void* ptr, const char* what) {
  if (!ptr) rwb::fail_domain(std::string("null pointer argument: ") + what);
}

// validate(order, n) (types.cpp:100-110) for one host order.
void validate_host_order(const int32_t* perm, int32_t size, int n) {
  if (size != n)
    rwb::fail_domain("rank order has " + std::to_string(size) + " entries, expected " + std::to_string(n));
  std::vector<char> seen(static_cast<size_t>(n), 0);
  for (int i = 0; i < n; ++i) {
    const int v = perm[i];
    if (v < 0 || v >= n || seen[static_cast<size_t>(v)])
      rwb::fail_domain("rank order is not a permutation of [0, " + std::to_string(n) + ")");
    seen[static_cast<size_t>(v)] = 1;
  }
}

}  // namespace

extern "C" {

const char* rw_last_error(void) { return g_last_error.c_str(); }
int32_t rw_abi_version(void) { return RW_ABI_VERSION; }

int32_t rw_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

rw_status rw_validate_spec(const rw_spec* spec) {
  return guarded([&] {
    need(spec, "spec");
    rwb::validate_spec(*spec);
  });
}

rw_status rw_problem_create(const double* rtt_us, int32_t n, int32_t storage_hint, int32_t device, rw_problem** out) {
  return guarded([&] {
    rwb::NvtxRange nvtx_("rw_problem_create");
    need(out, "out");
    *out = nullptr;
    need(rtt_us, "rtt_us");
    auto* h = new rw_problem{nullptr};
    try {
      h->impl = rwb::problem_create(rtt_us, n, storage_hint, device);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

rw_status rw_problem_destroy(rw_problem* p) {
  return guarded([&] {
    if (!p) return;
    rwb::problem_destroy(p->impl);
    delete p;
  });
}

rw_status rw_problem_get_info(const rw_problem* p, rw_problem_info* out) {
  return guarded([&] {
    need(out, "out");
    const rwb::Problem& q = get(p);
    out->n = q.n;
    out->device = q.device;
    out->storage = q.storage;
    out->frac_bits = q.frac_bits;
    out->symmetric = q.symmetric ? 1 : 0;
    out->zero_diagonal = q.zero_diag ? 1 : 0;
    out->device_bytes = static_cast<int64_t>(q.mat_bytes);
    out->max_value = q.max_value;
  });
}

rw_status rw_problem_set_path(rw_problem* p, int32_t path) {
  return guarded([&] {
    rwb::Problem& q = get(p);
    if (path != RW_PATH_AUTO && path != RW_PATH_L2_GATHER && path != RW_PATH_CLUSTER && path != RW_PATH_TRANSPOSE)
      rwb::fail_domain("unknown kernel path");
    q.path = path;
  });
}

rw_status rw_evaluate(const rw_problem* p, const rw_spec* spec, const int32_t* perm, double* cost) {
  return guarded([&] {
    rwb::NvtxRange nvtx_("rw_evaluate");
    need(spec, "spec");
    need(perm, "perm");
    need(cost, "cost");
    rwb::Problem& q = get(p);
    const rwb::EvalPlan plan = rwb::make_plan(q, *spec);
    validate_host_order(perm, spec->n, spec->n);  // host check done: no device error read-back
    if (!rwb::resident_evaluate(q, plan, perm, cost))
      rwb::evaluate_host_orders(q, plan, perm, 1, cost, /*exact=*/true, /*validate=*/false, nullptr);
  });
}

rw_status rw_problem_set_resident(rw_problem* p, int32_t idle_us) {
  return guarded([&] {
    rwb::Problem& q = get(p);
    rwb::resident_configure(q, idle_us);
  });
}

rw_status rw_evaluate_batch(const rw_problem* p, const rw_spec* spec, const int32_t* perms, int64_t batch,
                            double* costs, uint32_t flags, rw_eval_report* report) {
  return guarded([&] {
    rwb::NvtxRange nvtx_("rw_evaluate_batch");
    need(spec, "spec");
    if (batch < 0) rwb::fail_domain("batch must be >= 0");
    if (batch > 0) {
      need(perms, "perms");
      need(costs, "costs");
    }
    rwb::Problem& q = get(p);
    const rwb::EvalPlan plan = rwb::make_plan(q, *spec);
    rwb::evaluate_host_orders(q, plan, perms, batch, costs, (flags & RW_EVAL_EXACT) != 0,
                              (flags & RW_EVAL_NO_VALIDATE) == 0, report);
  });
}

rw_status rw_evaluate_batch_u16(const rw_problem* p, const rw_spec* spec, const uint16_t* perms, int64_t batch,
                                double* costs, uint32_t flags, rw_eval_report* report) {
  return guarded([&] {
    rwb::NvtxRange nvtx_("rw_evaluate_batch_u16");
    need(spec, "spec");
    if (batch < 0) rwb::fail_domain("batch must be >= 0");
    if (batch > 0) {
      need(perms, "perms");
      need(costs, "costs");
    }
    rwb::Problem& q = get(p);
    const rwb::EvalPlan plan = rwb::make_plan(q, *spec);
    rwb::evaluate_host_orders_fmt(q, plan, perms, 2, 0, batch, costs, (flags & RW_EVAL_EXACT) != 0,
                                  (flags & RW_EVAL_NO_VALIDATE) == 0, report);
  });
}

int64_t rw_packed_row_bytes(int32_t n, int32_t bits) {
  if (n < 1 || bits < 1 || bits > 16) return -1;
  return rwb::packed_row_bytes(n, bits);
}

rw_status rw_pack_orders(const int32_t* perms, int32_t n, int64_t batch, int32_t bits, void* out) {
  return guarded([&] {
    if (n < 1) rwb::fail_domain("n must be >= 1");
    if (bits < 1 || bits > 16 || (n > 1 && (1ll << bits) < n))
      rwb::fail_domain("packed orders need 1 <= bits <= 16 and 2^bits >= n");
    if (batch < 0) rwb::fail_domain("batch must be >= 0");
    if (batch == 0) return;
    need(perms, "perms");
    need(out, "out");
    const int64_t row = rwb::packed_row_bytes(n, bits);
    auto* w = static_cast<uint32_t*>(out);
    std::memset(out, 0, static_cast<size_t>(row * batch));
    for (int64_t b = 0; b < batch; ++b) {
      uint32_t* r = w + b * (row / 4);
      const int32_t* o = perms + b * n;
      for (int i = 0; i < n; ++i) {
        const uint32_t v = static_cast<uint32_t>(o[i]) & ((1u << bits) - 1u);
        if (static_cast<uint32_t>(o[i]) != v) rwb::fail_domain("rank order value does not fit the packed width");
        const uint64_t bit = static_cast<uint64_t>(i) * static_cast<uint64_t>(bits);
        const uint32_t q = static_cast<uint32_t>(bit >> 5), sh = static_cast<uint32_t>(bit & 31);
        r[q] |= v << sh;
        if (sh + static_cast<uint32_t>(bits) > 32u) r[q + 1] |= v >> (32u - sh);
      }
    }
  });
}

rw_status rw_evaluate_batch_packed(const rw_problem* p, const rw_spec* spec, const void* packed, int32_t bits,
                                   int64_t batch, double* costs, uint32_t flags, rw_eval_report* report) {
  return guarded([&] {
    rwb::NvtxRange nvtx_("rw_evaluate_batch_packed");
    need(spec, "spec");
    if (batch < 0) rwb::fail_domain("batch must be >= 0");
    if (batch > 0) {
      need(packed, "packed");
      need(costs, "costs");
    }
    rwb::Problem& q = get(p);
    const rwb::EvalPlan plan = rwb::make_plan(q, *spec);
    if (bits < 1 || bits > 16 || (spec->n > 1 && (1ll << bits) < spec->n))
      rwb::fail_domain("packed orders need 1 <= bits <= 16 and 2^bits >= n");
    rwb::evaluate_host_orders_fmt(q, plan, packed, 0, bits, batch, costs, (flags & RW_EVAL_EXACT) != 0,
                                  (flags & RW_EVAL_NO_VALIDATE) == 0, report);
  });
}

rw_status rw_evaluate_batch_device(const rw_problem* p, const rw_spec* spec, const void* d_perms, int32_t perm_bytes,
                                   int64_t batch, double* d_costs, void* stream, uint32_t flags) {
  return guarded([&] {
    rwb::NvtxRange nvtx_("rw_evaluate_batch_device");
    need(spec, "spec");
    if (batch < 0) rwb::fail_domain("batch must be >= 0");
    if (batch > 0) {
      need(d_perms, "d_perms");
      need(d_costs, "d_costs");
    }
    rwb::Problem& q = get(p);
    const rwb::EvalPlan plan = rwb::make_plan(q, *spec);
    rwb::DeviceGuard g(q.device);
    rwb::StreamScratch scope(q.device, static_cast<cudaStream_t>(stream));
    rwb::launch_evaluate(q, plan, d_perms, perm_bytes, batch, d_costs, (flags & RW_EVAL_EXACT) != 0,
                         (flags & RW_EVAL_NO_VALIDATE) == 0, q.d_err, static_cast<cudaStream_t>(stream));
  });
}

rw_status rw_sync_errors(const rw_problem* p, void* stream) {
  return guarded([&] {
    rwb::Problem& q = get(p);
    rwb::DeviceGuard g(q.device);
    rwb::ThreadCtx& c = rwb::thread_ctx(q.device);
    rwb::raise_order_errors(q.d_err, c.h_err, static_cast<cudaStream_t>(stream));
  });
}

rw_status rw_schedule_cost(const rw_problem* p, int32_t semantics, int32_t nrounds, const int32_t* round_offsets,
                           const int32_t* src, const int32_t* dst, const double* bytes, const int32_t* parent,
                           int32_t cost_mode, const int32_t* perm, double* cost) {
  return guarded([&] {
    need(round_offsets, "round_offsets");
    need(perm, "perm");
    need(cost, "cost");
    rwb::Problem& q = get(p);
    if (nrounds < 0) rwb::fail_domain("nrounds must be >= 0");
    if (semantics < RW_SEQUENTIAL_HOPS || semantics > RW_CRITICAL_PATH) rwb::fail_domain("schedule_cost: unknown semantics");
    const int edges = round_offsets[nrounds];
    if (edges > 0) {
      need(src, "src");
      need(dst, "dst");
      need(bytes, "bytes");
    }
    validate_host_order(perm, q.n, q.n);
    *cost = rwb::schedule_cost_device(q, semantics, nrounds, round_offsets, src, dst, bytes, parent, cost_mode, perm);
  });
}

rw_status rw_brute_force_space(const rw_spec* spec, uint64_t* count_out) {
  return guarded([&] {
    need(spec, "spec");
    need(count_out, "count_out");
    rwb::validate_spec(*spec);
    *count_out = rwb::brute_force_space(*spec);
  });
}

rw_status rw_brute_force(const rw_problem* p, const rw_spec* spec, int32_t threshold, int32_t* perm_out,
                         double* cost_out, uint64_t* evals_out) {
  return guarded([&] {
    rwb::NvtxRange nvtx_("rw_brute_force");
    need(spec, "spec");
    need(perm_out, "perm_out");
    need(cost_out, "cost_out");
    rwb::validate_spec(*spec);
    if (spec->n > threshold)
      rwb::fail_domain("N=" + std::to_string(spec->n) + " exceeds the brute-force threshold " +
                       std::to_string(threshold) + "; use anneal");
    rwb::Problem& q = get(p);
    const rwb::EvalPlan plan = rwb::make_plan(q, *spec);
    const uint64_t space = rwb::brute_force_space(*spec);
    double cost = 0.0;
    uint64_t index = 0;
    rwb::brute_force_range(q, plan, 0, space, &cost, &index);
    index = rwb::brute_force_resolve(q, plan, *spec, index);
    rwb::unrank(*spec, index, perm_out);
    // Reported cost is the reference-identical evaluation of the winner.
    rwb::evaluate_host_orders(q, plan, perm_out, 1, cost_out, true, true, nullptr);
    if (evals_out) *evals_out = space;
  });
}

rw_status rw_brute_force_range(const rw_problem* p, const rw_spec* spec, uint64_t first, uint64_t count,
                               double* cost_out, uint64_t* index_out) {
  return guarded([&] {
    rwb::NvtxRange nvtx_("rw_brute_force_range");
    need(spec, "spec");
    need(cost_out, "cost_out");
    need(index_out, "index_out");
    rwb::Problem& q = get(p);
    const rwb::EvalPlan plan = rwb::make_plan(q, *spec);
    const uint64_t space = rwb::brute_force_space(*spec);
    if (first > space) first = space;
    if (count > space - first) count = space - first;
    rwb::brute_force_range(q, plan, first, count, cost_out, index_out);
  });
}

rw_status rw_unrank(const rw_spec* spec, uint64_t index, int32_t* perm_out) {
  return guarded([&] {
    need(spec, "spec");
    need(perm_out, "perm_out");
    rwb::validate_spec(*spec);
    if (index >= rwb::brute_force_space(*spec)) rwb::fail_domain("lexicographic index out of range");
    rwb::unrank(*spec, index, perm_out);
  });
}

rw_status rw_anneal(const rw_problem* p, const rw_spec* spec, const rw_solver_config* cfg, const rw_gpu_config* gpu,
                    int32_t* perm_out, double* cost_out, uint64_t* evals_out, rw_search_report* report) {
  return guarded([&] {
    rwb::NvtxRange nvtx_("rw_anneal");
    const auto t_start = std::chrono::steady_clock::now();
    need(spec, "spec");
    need(cfg, "cfg");
    need(perm_out, "perm_out");
    need(cost_out, "cost_out");
    rwb::validate_spec(*spec);
    // validate(SolverConfig) -- solver.cpp:50-55
    if (!(cfg->budget_s > 0.0)) rwb::fail_domain("solver budget must be > 0");
    if (!(cfg->cooling > 0.0 && cfg->cooling < 1.0)) rwb::fail_domain("cooling factor must be in (0, 1)");
    if (cfg->restarts < 1) rwb::fail_domain("restarts must be >= 1");
    if (cfg->brute_force_threshold < 2) rwb::fail_domain("brute-force threshold must be >= 2");
    rwb::Problem& q = get(p);
    if (q.n != spec->n) rwb::fail_domain("matrix dimension does not match spec.n");
    const rwb::EvalPlan plan = rwb::make_plan(q, *spec);
    rw_gpu_config g{};
    if (gpu) g = *gpu;
    const rwb::AnnealResult r = rwb::anneal_device(q, plan, *cfg, g);
    std::copy(r.order.begin(), r.order.end(), perm_out);
    *cost_out = r.cost;
    if (evals_out) *evals_out = r.evaluations;
    if (report) {
      report->winner_chain = r.chain;
      report->chains = r.chains;
      report->proposals = static_cast<int64_t>(r.proposals);
      report->levels = r.levels;
      report->levels_run = r.levels_run;
      report->initial_temperature = r.t0;
      report->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    }
  });
}

rw_status rw_local_search(const rw_problem* p, const rw_spec* spec, int32_t* perms_inout, int64_t batch,
                          int32_t max_rounds, double* costs_out, uint64_t* evals_out) {
  return guarded([&] {
    rwb::NvtxRange nvtx_("rw_local_search");
    need(spec, "spec");
    if (batch < 0) rwb::fail_domain("batch must be >= 0");
    if (batch > 0) {
      need(perms_inout, "perms_inout");
      need(costs_out, "costs_out");
    }
    rwb::Problem& q = get(p);
    const rwb::EvalPlan plan = rwb::make_plan(q, *spec);
    for (int64_t b = 0; b < batch; ++b) validate_host_order(perms_inout + b * spec->n, spec->n, spec->n);
    uint64_t ev = 0;
    rwb::local_search_device(q, plan, perms_inout, batch, max_rounds, costs_out, &ev);
    if (evals_out) *evals_out = ev;
  });
}

// sample_orders (stats.cpp:83-94): one std::mt19937_64(seed) stream, an
// identity order std::shuffle'd per sample.  Host side: the draws are the
// libstdc++ algorithm itself, so the orders are the reference's bit for bit.
rw_status rw_sample_orders(int32_t n, int32_t samples, uint64_t seed, int32_t* perms_out) {
  return guarded([&] {
    if (samples < 1) rwb::fail_domain("sample_orders: need at least 1 sample");
    if (n < 0) rwb::fail_domain("sample_orders: n must be >= 0");
    if (n > 0) need(perms_out, "perms_out");
    std::mt19937_64 rng(seed);
    for (int32_t k = 0; k < samples; ++k) {
      int32_t* o = perms_out + static_cast<size_t>(k) * static_cast<size_t>(n);
      std::iota(o, o + n, 0);
      std::shuffle(o, o + n, rng);
    }
  });
}

// sample_costs (stats.cpp:96-103): the reference's orders, scored on the GPU
// in one batch with the reference-identical (sorted, serial) ring summation.
rw_status rw_sample_costs(const rw_problem* p, const rw_spec* spec, int32_t samples, uint64_t seed, double* costs_out) {
  return guarded([&] {
    rwb::NvtxRange nvtx_("rw_sample_costs");
    need(spec, "spec");
    if (samples < 1) rwb::fail_domain("sample_orders: need at least 1 sample");
    need(costs_out, "costs_out");
    rwb::Problem& q = get(p);
    const rwb::EvalPlan plan = rwb::make_plan(q, *spec);
    std::vector<int32_t> orders(static_cast<size_t>(spec->n) * static_cast<size_t>(samples));
    std::mt19937_64 rng(seed);
    for (int32_t k = 0; k < samples; ++k) {
      int32_t* o = orders.data() + static_cast<size_t>(k) * static_cast<size_t>(spec->n);
      std::iota(o, o + spec->n, 0);
      std::shuffle(o, o + spec->n, rng);
    }
    rwb::evaluate_host_orders(q, plan, orders.data(), samples, costs_out, /*exact=*/true, /*validate=*/false, nullptr);
  });
}

// GPU extension: counter-based (Philox) uniform orders, generated on the
// device.  Deterministic per seed, but NOT the reference's sequence.
rw_status rw_sample_orders_philox(int32_t n, int32_t samples, uint64_t seed, int32_t* perms_out) {
  return guarded([&] {
    if (samples < 1) rwb::fail_domain("sample_orders: need at least 1 sample");
    if (n < 1 || n > 65536) rwb::fail_domain("sample_orders: n out of range");
    need(perms_out, "perms_out");
    int dev = 0;
    RW_CUDA(cudaGetDevice(&dev));
    rwb::ThreadCtx& c = rwb::thread_ctx(dev);
    const size_t count = static_cast<size_t>(n) * static_cast<size_t>(samples);
    auto* d = static_cast<uint16_t*>(c.scratch(0, count * 2));
    rwb::sample_orders_device(n, samples, seed, d, c.stream[0]);
    std::vector<uint16_t> h(count);
    RW_CUDA(cudaMemcpyAsync(h.data(), d, count * 2, cudaMemcpyDeviceToHost, c.stream[0]));
    RW_CUDA(cudaStreamSynchronize(c.stream[0]));
    for (size_t k = 0; k < count; ++k) perms_out[k] = h[k];
  });
}

rw_status rw_sample_costs_philox(const rw_problem* p, const rw_spec* spec, int32_t samples, uint64_t seed,
                                 double* costs_out) {
  return guarded([&] {
    need(spec, "spec");
    need(costs_out, "costs_out");
    if (samples < 1) rwb::fail_domain("sample_orders: need at least 1 sample");
    rwb::Problem& q = get(p);
    const rwb::EvalPlan plan = rwb::make_plan(q, *spec);
    rwb::DeviceGuard g(q.device);
    rwb::ThreadCtx& c = rwb::thread_ctx(q.device);
    const size_t count = static_cast<size_t>(spec->n) * static_cast<size_t>(samples);
    auto* d = static_cast<uint16_t*>(c.scratch(0, count * 2));
    auto* dc = static_cast<double*>(c.scratch(1, static_cast<size_t>(samples) * 8));
    rwb::sample_orders_device(spec->n, samples, seed, d, c.stream[0]);
    rwb::launch_evaluate(q, plan, d, 2, samples, dc, /*exact=*/true, /*validate=*/false, c.d_err, c.stream[0]);
    RW_CUDA(cudaMemcpyAsync(costs_out, dc, static_cast<size_t>(samples) * 8, cudaMemcpyDeviceToHost, c.stream[0]));
    RW_CUDA(cudaStreamSynchronize(c.stream[0]));
  });
}

rw_status rw_generate_matrix(int32_t nlevels, const int32_t* fanout, const double* latency_us, const double* bandwidth,
                             const double* oversub, double jitter, uint64_t seed, double* out, int64_t out_capacity,
                             int32_t* n_out) {
  rw_status st = RW_OK;
  const rw_status g = guarded([&] {
    need(fanout, "fanout");
    need(latency_us, "latency_us");
    need(bandwidth, "bandwidth");
    need(oversub, "oversub");
    need(n_out, "n_out");
    st = rwb::generate_matrix(nlevels, fanout, latency_us, bandwidth, oversub, jitter, seed, out, out_capacity, n_out);
  });
  return g != RW_OK ? g : st;
}

rw_status rw_expand_schedule(const rw_spec* spec, int32_t* semantics_out, int32_t* nrounds_out, int64_t* count_out,
                             int32_t* round_offsets, int32_t* src, int32_t* dst, int32_t* parent, double* bytes) {
  return guarded([&] {
    need(spec, "spec");
    const rwb::Expanded e = rwb::expand_schedule_core(*spec);
    if (semantics_out) *semantics_out = e.semantics;
    if (nrounds_out) *nrounds_out = e.nrounds();
    if (count_out) *count_out = static_cast<int64_t>(e.src.size());
    if (round_offsets) std::copy(e.off.begin(), e.off.end(), round_offsets);
    if (src) std::copy(e.src.begin(), e.src.end(), src);
    if (dst) std::copy(e.dst.begin(), e.dst.end(), dst);
    if (parent) std::copy(e.parent.begin(), e.parent.end(), parent);
    if (bytes) std::copy(e.bytes.begin(), e.bytes.end(), bytes);
  });
}

rw_status rw_simulate_batch(const rw_problem* p, int32_t nlevels, const int32_t* fanout, const double* bandwidth,
                            const double* oversub, const rw_spec* spec, const int32_t* perms, int64_t batch,
                            double* out) {
  return guarded([&] {
    rwb::NvtxRange nvtx_("rw_simulate_batch");
    need(fanout, "fanout");
    need(bandwidth, "bandwidth");
    need(oversub, "oversub");
    need(spec, "spec");
    rwb::Problem& q = get(p);
    rwb::validate_spec(*spec);
    long long hosts = 1;
    rwb::TopologyDesc topo;
    for (int l = 0; l < nlevels; ++l) {
      if (fanout[l] < 1) rwb::fail_domain("topology level fanout must be >= 1");
      if (!(bandwidth[l] > 0.0)) rwb::fail_domain("topology level bandwidth must be > 0");
      if (!(oversub[l] >= 1.0)) rwb::fail_domain("topology oversubscription must be >= 1");
      hosts *= fanout[l];
      topo.fanout.push_back(fanout[l]);
      topo.capacity.push_back(bandwidth[l] / oversub[l]);  // simulate.cpp:45-48
    }
    if (hosts != spec->n)
      rwb::fail_domain("topology has " + std::to_string(hosts) + " hosts but spec.n=" + std::to_string(spec->n));
    if (q.n != spec->n) rwb::fail_domain("matrix dimension does not match spec.n");
    if (batch < 0) rwb::fail_domain("batch must be >= 0");
    if (batch > 0) {
      need(perms, "perms");
      need(out, "out");
    }
    for (int64_t b = 0; b < batch; ++b) validate_host_order(perms + b * spec->n, spec->n, spec->n);
    const rwb::Expanded e = rwb::expand_schedule_core(*spec);
    rwb::simulate_batch_device(q, topo, e, perms, batch, out);
  });
}

rw_status rw_relabel_matrix(double* m, int32_t n, uint64_t seed) {
  return guarded([&] {
    need(m, "m");
    if (n < 1) rwb::fail_domain("n must be >= 1");
    rwb::relabel_matrix(m, n, seed);
  });
}

// ---- host logic shared with the C++ drop-in (one implementation) ----------
// These forward to the rankweave:: functions in rankweave_api.cpp so that the
// C++ drop-in, the Python binding and any other FFI run the same code.

rw_status rw_distribution_stats(const double* values, int64_t count, double* out4) {
  return guarded([&] {
    need(out4, "out4");
    if (count > 0) need(values, "values");
    const rankweave::DistributionStats st =
        rankweave::distribution_stats(std::vector<double>(values, values + std::max<int64_t>(0, count)));
    out4[0] = st.min;
    out4[1] = st.max;
    out4[2] = st.mean;
    out4[3] = st.stddev;
  });
}

rw_status rw_spearman(const double* xs, const double* ys, int64_t count_x, int64_t count_y, double* out) {
  return guarded([&] {
    need(out, "out");
    if (count_x > 0) need(xs, "xs");
    if (count_y > 0) need(ys, "ys");
    *out = rankweave::spearman(std::vector<double>(xs, xs + std::max<int64_t>(0, count_x)),
                               std::vector<double>(ys, ys + std::max<int64_t>(0, count_y)));
  });
}

rw_status rw_parse_model_file(const char* text, int32_t n, int32_t* perm_out) {
  return guarded([&] {
    need(text, "text");
    if (n > 0) need(perm_out, "perm_out");
    const rankweave::RankOrder o = rankweave::parse_model_file(text, n);
    std::copy(o.perm.begin(), o.perm.end(), perm_out);
  });
}

rw_status rw_balanced_sexpr(const char* text, int32_t* out) {
  return guarded([&] {
    need(text, "text");
    need(out, "out");
    *out = rankweave::balanced_sexpr(text) ? 1 : 0;
  });
}

namespace {
rankweave::CostMatrix host_matrix(const double* rtt_us, int32_t n) {
  if (n < 0) rwb::fail_domain("n must be >= 0");
  if (n > 0) need(rtt_us, "rtt_us");
  rankweave::CostMatrix m;
  m.hosts.reserve(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) m.hosts.push_back("h" + std::to_string(i));
  m.rtt_us.assign(rtt_us, rtt_us + static_cast<size_t>(n) * static_cast<size_t>(n));
  return m;
}
rankweave::CollectiveSpec cxx_spec(const rw_spec& c) {
  rankweave::CollectiveSpec s;
  s.algorithm = static_cast<rankweave::Algorithm>(c.algorithm);
  s.n = c.n;
  s.size_bytes = c.size_bytes;
  s.bcube_b = c.bcube_b;
  s.cost_mode = static_cast<rankweave::CostMode>(c.cost_mode);
  s.hd_pairing = static_cast<rankweave::HdPairing>(c.hd_pairing);
  return s;
}
}  // namespace

rw_status rw_emit_smtlib(const double* rtt_us, int32_t n, const rw_spec* spec, int32_t has_bound, double bound,
                         int32_t emission_cap, char* out, int64_t capacity, int64_t* length_out) {
  return guarded([&] {
    need(spec, "spec");
    need(length_out, "length_out");
    const std::string text = rankweave::emit_smtlib(host_matrix(rtt_us, n), cxx_spec(*spec),
                                                    has_bound ? std::optional<double>(bound) : std::nullopt,
                                                    emission_cap);
    *length_out = static_cast<int64_t>(text.size());
    if (out && capacity > 0) {
      const size_t k = std::min<size_t>(text.size(), static_cast<size_t>(capacity - 1));
      std::memcpy(out, text.data(), k);
      out[k] = '\0';
    }
  });
}

rw_status rw_set_gpu_options(const rw_gpu_options* opts) {
  return guarded([&] {
    need(opts, "opts");
    if (opts->num_devices < 0) rwb::fail_domain("num_devices must be >= 0");
    rankweave::GpuOptions o;
    o.device = opts->device;
    o.chains = opts->chains;
    o.exact_batch = opts->exact_batch != 0;
    o.immutable_matrices = opts->immutable_matrices != 0;
    o.num_devices = opts->num_devices;
    o.resident_idle_us = opts->resident_idle_us;
    rankweave::set_gpu_options(o);
  });
}

rw_status rw_get_gpu_options(rw_gpu_options* out) {
  return guarded([&] {
    need(out, "out");
    const rankweave::GpuOptions o = rankweave::gpu_options();
    out->device = o.device;
    out->chains = o.chains;
    out->exact_batch = o.exact_batch ? 1 : 0;
    out->immutable_matrices = o.immutable_matrices ? 1 : 0;
    out->num_devices = o.num_devices;
    out->resident_idle_us = o.resident_idle_us;
  });
}

rw_status rw_two_stage_solve(const double* rtt_us, int32_t n, const rw_spec* spec, const rw_solver_config* cfg,
                             const char* emit_smt_path, const char* external_model_path, rw_log_fn log, void* user,
                             int32_t* perm_out, double* cost_out, int32_t* method_out, uint64_t* evals_out) {
  return guarded([&] {
    need(spec, "spec");
    need(cfg, "cfg");
    need(cost_out, "cost_out");
    if (spec->n > 0) need(perm_out, "perm_out");
    rankweave::SolverConfig c;
    c.budget = std::chrono::duration<double>(cfg->budget_s);
    c.seed = cfg->seed;
    c.initial_temperature = cfg->initial_temperature;
    c.cooling = cfg->cooling;
    c.steps_per_temperature = cfg->steps_per_temperature;
    c.restarts = cfg->restarts;
    c.brute_force_threshold = cfg->brute_force_threshold;
    rankweave::TwoStageOptions opts;
    if (emit_smt_path) opts.emit_smt_path = emit_smt_path;
    if (external_model_path) opts.external_model_path = external_model_path;
    if (log) opts.log = [log, user](const std::string& msg) { log(msg.c_str(), user); };
    const rankweave::Solution sol = rankweave::two_stage_solve(host_matrix(rtt_us, n), cxx_spec(*spec), c, opts);
    if (static_cast<int32_t>(sol.order.perm.size()) != spec->n) rwb::fail_internal("solution size mismatch");
    std::copy(sol.order.perm.begin(), sol.order.perm.end(), perm_out);
    *cost_out = sol.cost;
    if (method_out) *method_out = static_cast<int32_t>(sol.method);
    if (evals_out) *evals_out = sol.evaluations;
  });
}

// ---- multi-GPU: one process, a device set, in-process NCCL -----------------

rw_status rw_problem_set_create(const double* rtt_us, int32_t n, int32_t storage_hint, const int32_t* devices,
                                int32_t ndevices, rw_problem_set** out) {
  return guarded([&] {
    rwb::NvtxRange nvtx_("rw_problem_set_create");
    need(out, "out");
    *out = nullptr;
    need(rtt_us, "rtt_us");
    auto* h = new rw_problem_set{nullptr, {}};
    try {
      h->impl = rwb::problem_set_create(rtt_us, n, storage_hint, devices, ndevices);
      for (int i = 0; i < rwb::problem_set_size(*h->impl); ++i)
        h->members.push_back(rw_problem{&rwb::problem_set_member(*h->impl, i)});
    } catch (...) {
      if (h->impl) rwb::problem_set_destroy(h->impl);
      delete h;
      throw;
    }
    *out = h;
  });
}

rw_status rw_problem_set_destroy(rw_problem_set* s) {
  return guarded([&] {
    if (!s) return;
    rwb::problem_set_destroy(s->impl);
    delete s;
  });
}

namespace {
rwb::ProblemSet& get_set(const rw_problem_set* s) {
  if (!s || !s->impl) rwb::fail_domain("null rw_problem_set");
  return *s->impl;
}
}  // namespace

rw_status rw_problem_set_devices(const rw_problem_set* s, int32_t* ndevices_out, int32_t* devices_out) {
  return guarded([&] {
    need(ndevices_out, "ndevices_out");
    rwb::ProblemSet& q = get_set(s);
    *ndevices_out = rwb::problem_set_size(q);
    if (devices_out)
      for (int i = 0; i < *ndevices_out; ++i) devices_out[i] = rwb::problem_set_device(q, i);
  });
}

rw_status rw_problem_set_member(const rw_problem_set* s, int32_t index, rw_problem** out) {
  return guarded([&] {
    need(out, "out");
    get_set(s);
    if (index < 0 || index >= static_cast<int32_t>(s->members.size())) rwb::fail_domain("member index out of range");
    *out = const_cast<rw_problem*>(&s->members[static_cast<size_t>(index)]);
  });
}

rw_status rw_evaluate_batch_set(const rw_problem_set* s, const rw_spec* spec, const void* perms, int32_t layout,
                                int32_t bits, int64_t batch, double* costs, uint32_t flags) {
  return guarded([&] {
    rwb::NvtxRange nvtx_("rw_evaluate_batch_set");
    need(spec, "spec");
    if (batch < 0) rwb::fail_domain("batch must be >= 0");
    if (batch > 0) {
      need(perms, "perms");
      need(costs, "costs");
    }
    rwb::ProblemSet& q = get_set(s);
    rwb::make_plan(rwb::problem_set_member(q, 0), *spec);  // validates spec and n
    if (layout != RW_LAYOUT_INT32 && layout != RW_LAYOUT_U16 && layout != RW_LAYOUT_PACKED)
      rwb::fail_domain("unknown order layout");
    if (layout == RW_LAYOUT_PACKED && (bits < 1 || bits > 16 || (spec->n > 1 && (1ll << bits) < spec->n)))
      rwb::fail_domain("packed orders need 1 <= bits <= 16 and 2^bits >= n");
    rwb::evaluate_host_orders_set(q, *spec, perms, layout, bits, batch, costs, (flags & RW_EVAL_EXACT) != 0,
                                  (flags & RW_EVAL_NO_VALIDATE) == 0);
  });
}

rw_status rw_brute_force_set(const rw_problem_set* s, const rw_spec* spec, int32_t threshold, int32_t* perm_out,
                             double* cost_out, uint64_t* evals_out) {
  return guarded([&] {
    rwb::NvtxRange nvtx_("rw_brute_force_set");
    need(spec, "spec");
    need(perm_out, "perm_out");
    need(cost_out, "cost_out");
    rwb::validate_spec(*spec);
    if (spec->n > threshold)
      rwb::fail_domain("N=" + std::to_string(spec->n) + " exceeds the brute-force threshold " +
                       std::to_string(threshold) + "; use anneal");
    rwb::ProblemSet& q = get_set(s);
    rwb::make_plan(rwb::problem_set_member(q, 0), *spec);
    rwb::brute_force_set(q, *spec, perm_out, cost_out, evals_out);
  });
}

rw_status rw_anneal_set(const rw_problem_set* s, const rw_spec* spec, const rw_solver_config* cfg,
                        const rw_gpu_config* gpu, int32_t* perm_out, double* cost_out, uint64_t* evals_out,
                        rw_search_report* report) {
  return guarded([&] {
    rwb::NvtxRange nvtx_("rw_anneal_set");
    const auto t_start = std::chrono::steady_clock::now();
    need(spec, "spec");
    need(cfg, "cfg");
    need(perm_out, "perm_out");
    need(cost_out, "cost_out");
    rwb::validate_spec(*spec);
    if (!(cfg->budget_s > 0.0)) rwb::fail_domain("solver budget must be > 0");
    if (!(cfg->cooling > 0.0 && cfg->cooling < 1.0)) rwb::fail_domain("cooling factor must be in (0, 1)");
    if (cfg->restarts < 1) rwb::fail_domain("restarts must be >= 1");
    if (cfg->brute_force_threshold < 2) rwb::fail_domain("brute-force threshold must be >= 2");
    rwb::ProblemSet& q = get_set(s);
    if (rwb::problem_set_member(q, 0).n != spec->n) rwb::fail_domain("matrix dimension does not match spec.n");
    rwb::make_plan(rwb::problem_set_member(q, 0), *spec);
    rw_gpu_config g{};
    if (gpu) g = *gpu;
    const rwb::AnnealResult r = rwb::anneal_set(q, *spec, *cfg, g);
    std::copy(r.order.begin(), r.order.end(), perm_out);
    *cost_out = r.cost;
    if (evals_out) *evals_out = r.evaluations;
    if (report) {
      report->winner_chain = r.chain;
      report->chains = r.chains;
      report->proposals = static_cast<int64_t>(r.proposals);
      report->levels = r.levels;
      report->levels_run = r.levels_run;
      report->initial_temperature = r.t0;
      report->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    }
  });
}

}  // extern "C"
