// rw_multi.cpp -- one process, several GPUs: a cost matrix replicated on a
// device set with an in-process NCCL communicator (ncclCommInitAll), and the
// sharded entry points of the C ABI (rw_*_set).
//
// SURVEY 8(e) / north star (4):
//   * replication: the matrix is analysed and uploaded once (device 0) and
//     ncclBroadcast over NVLink to the other members;
//   * batch scoring: contiguous slices of one host batch per device, each on
//     its own host thread, so every GPU's PCIe link carries its own slice;
//   * exhaustive search (solver.cpp:73-105): the lexicographic range is cut
//     into contiguous slices; ncclAllReduce(MIN) on the cost, then MIN on the
//     index among members at that cost (ties resolve to the lex-smallest
//     order, as the reference's strict '<' does);
//   * annealing (solver.cpp:141-202): global chain ids are split over the
//     members (Philox keyed by (seed, chain id): trajectories do not depend on
//     the device count); ncclAllReduce(MIN) on the cost, MIN on the chain id,
//     ncclBroadcast of the winning order from its owner.
//
// NCCL is loaded at run time (dlopen "libnccl.so.2"): a process that already
// holds torch's NCCL reuses it, and single-device users never need it.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <functional>
#include <cstring>
#include <exception>
#include <limits>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "rw_internal.h"

namespace rwb {

Problem* problem_create(const double* rtt, int n, int hint, int device);
void problem_destroy(Problem* p);
Problem* problem_replica(const Problem& src, int device);

namespace {

struct NcclApi {
  ncclResult_t (*commInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
  std::string error;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.error = std::string("cannot load libnccl.so.2: ") + dlerror();
      return a;
    }
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn && a.error.empty()) a.error = std::string("libnccl.so.2 lacks ") + name;
    };
    sym(a.commInitAll, "ncclCommInitAll");
    sym(a.commDestroy, "ncclCommDestroy");
    sym(a.allReduce, "ncclAllReduce");
    sym(a.broadcast, "ncclBroadcast");
    sym(a.groupStart, "ncclGroupStart");
    sym(a.groupEnd, "ncclGroupEnd");
    sym(a.errorString, "ncclGetErrorString");
    return a;
  }();
  if (!api.error.empty()) throw Failure(RW_ERR_NCCL, api.error);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return;
  const NcclApi& a = nccl();
  throw Failure(RW_ERR_NCCL, std::string("NCCL ") + what + ": " + (a.errorString ? a.errorString(r) : "error"));
}

using Reduce = SetReduce;
constexpr unsigned long long kNoKey = ~0ull;

}  // namespace

// One persistent host thread per member: the library's per-(thread, device)
// contexts (streams, scratch, pinned staging) are reused across calls instead
// of being created by a fresh thread every time.
class MemberWorker {
 public:
  explicit MemberWorker(int device) : device_(device), th_([this] { loop(); }) {}
  ~MemberWorker() {
    {
      std::lock_guard<std::mutex> l(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    th_.join();
  }
  void post(std::function<void()> f) {
    {
      std::lock_guard<std::mutex> l(mu_);
      task_ = std::move(f);
      done_ = false;
      err_ = nullptr;
    }
    cv_.notify_all();
  }
  void wait() {
    std::unique_lock<std::mutex> l(mu_);
    cv_.wait(l, [this] { return done_; });
    if (err_) std::rethrow_exception(err_);
  }

 private:
  void loop() {
    for (;;) {
      std::function<void()> f;
      {
        std::unique_lock<std::mutex> l(mu_);
        cv_.wait(l, [this] { return stop_ || task_; });
        if (stop_) {
          l.unlock();
          thread_ctx_release();  // this thread's streams and scratch die with the set
          return;
        }
        f = std::move(task_);
        task_ = nullptr;
      }
      std::exception_ptr e;
      try {
        DeviceGuard g(device_);
        f();
      } catch (...) {
        e = std::current_exception();
      }
      {
        std::lock_guard<std::mutex> l(mu_);
        err_ = e;
        done_ = true;
      }
      cv_.notify_all();
    }
  }
  int device_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::function<void()> task_;
  bool done_ = true, stop_ = false;
  std::exception_ptr err_;
  std::thread th_;
};

struct ProblemSet {
  std::vector<std::unique_ptr<MemberWorker>> workers;
  std::vector<int> devices;
  std::vector<Problem*> members;
  std::vector<ncclComm_t> comms;
  std::vector<cudaStream_t> streams;
  std::vector<Reduce*> d_red;
  std::vector<int32_t*> d_order;  // winner broadcast buffers (n int32)
  std::mutex mu;                  // one sharded call at a time per set
};

namespace {

// Runs f(i) for every member on its own host thread (device selected);
// rethrows the first failure in member order.
template <class F>
void for_each_member(ProblemSet& s, F&& f) {
  const int k = static_cast<int>(s.members.size());
  for (int i = 0; i < k; ++i) s.workers[static_cast<size_t>(i)]->post([&f, i] { f(i); });
  std::exception_ptr first;
  for (int i = 0; i < k; ++i) {
    try {
      s.workers[static_cast<size_t>(i)]->wait();
    } catch (...) {
      if (!first) first = std::current_exception();
    }
  }
  if (first) std::rethrow_exception(first);
}

// MIN cost, then MIN key among members at that cost, and the evaluation sum:
// three collectives on the members' streams (rw_multi.cu selects the keys).
void reduce_best(ProblemSet& s) {
  const NcclApi& api = nccl();
  const int k = static_cast<int>(s.members.size());
  nccl_check(api.groupStart(), "group start");
  for (int i = 0; i < k; ++i) {
    Reduce* r = s.d_red[static_cast<size_t>(i)];
    nccl_check(api.allReduce(&r->cost, &r->min_cost, 1, ncclFloat64, ncclMin, s.comms[static_cast<size_t>(i)],
                             s.streams[static_cast<size_t>(i)]),
               "all-reduce MIN cost");
    nccl_check(api.allReduce(&r->evals, &r->evals_sum, 1, ncclUint64, ncclSum, s.comms[static_cast<size_t>(i)],
                             s.streams[static_cast<size_t>(i)]),
               "all-reduce SUM evaluations");
  }
  nccl_check(api.groupEnd(), "group end");
  for (int i = 0; i < k; ++i) {
    DeviceGuard g(s.devices[static_cast<size_t>(i)]);
    launch_select_key(s.d_red[static_cast<size_t>(i)], s.streams[static_cast<size_t>(i)]);
  }
  nccl_check(api.groupStart(), "group start");
  for (int i = 0; i < k; ++i) {
    Reduce* r = s.d_red[static_cast<size_t>(i)];
    nccl_check(api.allReduce(&r->min_key, &r->min_key, 1, ncclUint64, ncclMin, s.comms[static_cast<size_t>(i)],
                             s.streams[static_cast<size_t>(i)]),
               "all-reduce MIN key");
  }
  nccl_check(api.groupEnd(), "group end");
}

Reduce read_reduce(ProblemSet& s, int i) {
  Reduce h{};
  DeviceGuard g(s.devices[static_cast<size_t>(i)]);
  RW_CUDA(cudaMemcpyAsync(&h, s.d_red[static_cast<size_t>(i)], sizeof(Reduce), cudaMemcpyDeviceToHost,
                          s.streams[static_cast<size_t>(i)]));
  RW_CUDA(cudaStreamSynchronize(s.streams[static_cast<size_t>(i)]));
  return h;
}

void write_reduce(ProblemSet& s, int i, double cost, unsigned long long key, unsigned long long evals) {
  Reduce h{cost, 0.0, key, 0ull, evals, 0ull};
  DeviceGuard g(s.devices[static_cast<size_t>(i)]);
  RW_CUDA(cudaMemcpyAsync(s.d_red[static_cast<size_t>(i)], &h, sizeof(Reduce), cudaMemcpyHostToDevice,
                          s.streams[static_cast<size_t>(i)]));
  RW_CUDA(cudaStreamSynchronize(s.streams[static_cast<size_t>(i)]));
}

void sync_all(ProblemSet& s) {
  for (size_t i = 0; i < s.members.size(); ++i) {
    DeviceGuard g(s.devices[i]);
    RW_CUDA(cudaStreamSynchronize(s.streams[i]));
  }
}

}  // namespace

ProblemSet* problem_set_create(const double* rtt, int n, int hint, const int* devices, int ndev) {
  int visible = 0;
  RW_CUDA(cudaGetDeviceCount(&visible));
  std::vector<int> devs;
  if (ndev <= 0) {
    for (int d = 0; d < visible; ++d) devs.push_back(d);
  } else {
    if (!devices) fail_domain("null pointer argument: devices");
    devs.assign(devices, devices + ndev);
  }
  if (devs.empty()) fail_domain("no CUDA device for the problem set");
  for (size_t i = 0; i < devs.size(); ++i) {
    if (devs[i] < 0 || devs[i] >= visible) fail_domain("device " + std::to_string(devs[i]) + " does not exist");
    for (size_t j = 0; j < i; ++j)
      if (devs[j] == devs[i]) fail_domain("device " + std::to_string(devs[i]) + " listed twice");
  }
  auto s = std::make_unique<ProblemSet>();
  s->devices = devs;
  const int k = static_cast<int>(devs.size());
  try {
    s->members.push_back(problem_create(rtt, n, hint, devs[0]));
    for (int i = 1; i < k; ++i) s->members.push_back(problem_replica(*s->members[0], devs[static_cast<size_t>(i)]));
    for (int i = 0; i < k; ++i) {
      DeviceGuard g(devs[static_cast<size_t>(i)]);
      cudaStream_t st;
      RW_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
      s->streams.push_back(st);
      void* r = nullptr;
      RW_CUDA(cudaMalloc(&r, sizeof(Reduce)));
      s->d_red.push_back(static_cast<Reduce*>(r));
      void* o = nullptr;
      RW_CUDA(cudaMalloc(&o, static_cast<size_t>(n) * 4 + 16));
      s->d_order.push_back(static_cast<int32_t*>(o));
    }
    for (int i = 0; i < k; ++i) s->workers.push_back(std::make_unique<MemberWorker>(devs[static_cast<size_t>(i)]));
    if (k > 1) {
      const NcclApi& api = nccl();
      std::vector<ncclComm_t> comms(static_cast<size_t>(k));
      nccl_check(api.commInitAll(comms.data(), k, devs.data()), "comm init");
      s->comms = std::move(comms);  // only initialised communicators are ever destroyed
      // replicate the device matrix from member 0 over NVLink
      nccl_check(api.groupStart(), "group start");
      for (int i = 0; i < k; ++i) {
        Problem* m = s->members[static_cast<size_t>(i)];
        nccl_check(api.broadcast(i == 0 ? m->d_mat : nullptr, m->d_mat, m->mat_bytes, ncclUint8, 0,
                                 s->comms[static_cast<size_t>(i)], s->streams[static_cast<size_t>(i)]),
                   "broadcast matrix");
      }
      nccl_check(api.groupEnd(), "group end");
      sync_all(*s);
    }
  } catch (...) {
    problem_set_destroy(s.release());  // workers, communicators, streams, buffers, members
    throw;
  }
  return s.release();
}

void problem_set_destroy(ProblemSet* s) {
  if (!s) return;
  s->workers.clear();
  if (!s->comms.empty()) {
    try {
      const NcclApi& api = nccl();
      for (ncclComm_t c : s->comms) api.commDestroy(c);
    } catch (...) {
    }
  }
  for (size_t i = 0; i < s->members.size(); ++i) {
    DeviceGuard g(s->devices[i]);
    if (i < s->streams.size()) cudaStreamDestroy(s->streams[i]);
    if (i < s->d_red.size()) cudaFree(s->d_red[i]);
    if (i < s->d_order.size()) cudaFree(s->d_order[i]);
  }
  for (Problem* m : s->members) problem_destroy(m);
  delete s;
}

int problem_set_size(const ProblemSet& s) { return static_cast<int>(s.members.size()); }
Problem& problem_set_member(ProblemSet& s, int i) { return *s.members.at(static_cast<size_t>(i)); }
int problem_set_device(const ProblemSet& s, int i) { return s.devices.at(static_cast<size_t>(i)); }

void evaluate_host_orders_set(ProblemSet& s, const rw_spec& spec, const void* perms, int fmt, int bits, int64_t batch,
                              double* costs, bool exact, bool validate) {
  std::lock_guard<std::mutex> lock(s.mu);
  const int k = static_cast<int>(s.members.size());
  const int64_t row = fmt == 0 ? packed_row_bytes(spec.n, bits) : static_cast<int64_t>(spec.n) * fmt;
  const auto* hp = static_cast<const char*>(perms);
  for_each_member(s, [&](int i) {
    const int64_t lo = batch * i / k, hi = batch * (i + 1) / k;
    if (lo >= hi) return;
    Problem& m = *s.members[static_cast<size_t>(i)];
    const EvalPlan plan = make_plan(m, spec);
    evaluate_host_orders_fmt(m, plan, hp + lo * row, fmt, bits, hi - lo, costs + lo, exact, validate, nullptr, lo);
  });
}

void brute_force_set(ProblemSet& s, const rw_spec& spec, int32_t* perm_out, double* cost_out, uint64_t* evals_out) {
  std::lock_guard<std::mutex> lock(s.mu);
  const int k = static_cast<int>(s.members.size());
  const uint64_t space = brute_force_space(spec);
  for_each_member(s, [&](int i) {
    const uint64_t lo = space / k * i + std::min<uint64_t>(i, space % k);
    const uint64_t hi = lo + space / k + (static_cast<uint64_t>(i) < space % k ? 1 : 0);
    Problem& m = *s.members[static_cast<size_t>(i)];
    const EvalPlan plan = make_plan(m, spec);
    double c = std::numeric_limits<double>::infinity();
    uint64_t idx = ~0ull;
    if (hi > lo) brute_force_range(m, plan, lo, hi - lo, &c, &idx);
    write_reduce(s, i, c, idx, hi - lo);
  });
  uint64_t index = 0, evals = space;
  if (k > 1) {
    reduce_best(s);
    const Reduce r = read_reduce(s, 0);
    index = r.min_key;
    evals = r.evals_sum;
  } else {
    const Reduce r = read_reduce(s, 0);
    index = r.key;
  }
  Problem& m0 = *s.members[0];
  const EvalPlan plan = make_plan(m0, spec);
  index = brute_force_resolve(m0, plan, spec, index);
  unrank(spec, index, perm_out);
  evaluate_host_orders(m0, plan, perm_out, 1, cost_out, true, true, nullptr);
  if (evals_out) *evals_out = evals;
}

AnnealResult anneal_set(ProblemSet& s, const rw_spec& spec, const rw_solver_config& cfg, const rw_gpu_config& gpu) {
  std::lock_guard<std::mutex> lock(s.mu);
  const int k = static_cast<int>(s.members.size());
  int sms = 148;
  RW_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s.devices[0]));
  const int64_t total = gpu.chains > 0 ? gpu.chains : static_cast<int64_t>(k) * std::max(cfg.restarts, 4 * sms);
  std::vector<AnnealResult> res(static_cast<size_t>(k));
  for_each_member(s, [&](int i) {
    const int64_t lo = total * i / k, hi = total * (i + 1) / k;
    Problem& m = *s.members[static_cast<size_t>(i)];
    if (hi > lo) {
      rw_gpu_config g = gpu;
      g.chains = static_cast<int32_t>(hi - lo);
      g.chain_begin = static_cast<int32_t>(lo);
      g.chain_total = static_cast<int32_t>(total);
      if (gpu.max_proposals > 0) g.max_proposals = gpu.max_proposals * (hi - lo) / total;
      const EvalPlan plan = make_plan(m, spec);
      res[static_cast<size_t>(i)] = anneal_device(m, plan, cfg, g);
    }
    const AnnealResult& r = res[static_cast<size_t>(i)];
    write_reduce(s, i, hi > lo ? r.cost : std::numeric_limits<double>::infinity(),
                 hi > lo ? static_cast<unsigned long long>(r.chain) : kNoKey, r.evaluations);
  });
  AnnealResult out;
  int owner = 0;
  if (k > 1) {
    reduce_best(s);
    const Reduce r = read_reduce(s, 0);
    for (int i = 0; i < k; ++i)
      if (!res[static_cast<size_t>(i)].order.empty() &&
          static_cast<unsigned long long>(res[static_cast<size_t>(i)].chain) == r.min_key &&
          res[static_cast<size_t>(i)].cost == r.min_cost)
        owner = i;
    // the owner broadcasts its order over NVLink; every member holds the winner
    const NcclApi& api = nccl();
    {
      DeviceGuard g(s.devices[static_cast<size_t>(owner)]);
      RW_CUDA(cudaMemcpyAsync(s.d_order[static_cast<size_t>(owner)], res[static_cast<size_t>(owner)].order.data(),
                              static_cast<size_t>(spec.n) * 4, cudaMemcpyHostToDevice,
                              s.streams[static_cast<size_t>(owner)]));
    }
    nccl_check(api.groupStart(), "group start");
    for (int i = 0; i < k; ++i)
      nccl_check(api.broadcast(s.d_order[static_cast<size_t>(i)], s.d_order[static_cast<size_t>(i)],
                               static_cast<size_t>(spec.n), ncclInt32, owner, s.comms[static_cast<size_t>(i)],
                               s.streams[static_cast<size_t>(i)]),
                 "broadcast winner");
    nccl_check(api.groupEnd(), "group end");
    out.order.resize(static_cast<size_t>(spec.n));
    {
      DeviceGuard g(s.devices[0]);
      RW_CUDA(cudaMemcpyAsync(out.order.data(), s.d_order[0], static_cast<size_t>(spec.n) * 4, cudaMemcpyDeviceToHost,
                              s.streams[0]));
      RW_CUDA(cudaStreamSynchronize(s.streams[0]));
    }
    sync_all(s);
    out.cost = r.min_cost;
    out.chain = static_cast<int64_t>(r.min_key);
    // every shard draws the same T0 / calibration samples (seeded by the
    // solver seed alone); count them once, as one device does
    uint64_t dup = 0;
    int active = 0;
    for (const auto& x : res)
      if (!x.order.empty()) {
        dup = x.setup_evaluations;
        ++active;
      }
    out.evaluations = r.evals_sum - (active > 1 ? dup * static_cast<uint64_t>(active - 1) : 0);
  } else {
    out = res[0];
  }
  const AnnealResult& w = res[static_cast<size_t>(owner)];
  out.chains = total;
  out.levels = w.levels;
  out.t0 = w.t0;
  out.levels_run = w.levels_run;
  for (const auto& r : res) {
    out.proposals += r.proposals;
    out.levels_run = std::min(out.levels_run, r.levels_run);
  }
  return out;
}

}  // namespace rwb
