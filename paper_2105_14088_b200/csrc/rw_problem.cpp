// rw_problem.cpp -- host side of the device problem object: storage choice,
// upload, spec validation and evaluation planning.
//
// Reference correspondences:
//   CostMatrix (types.hpp:42-53)          -> rwb::Problem (matrix resident in HBM)
//   validate(CollectiveSpec) (types.cpp:143-163) -> validate_spec (same wording)
//   check_inputs (cost_model.cpp:13-19)   -> make_plan (same wording)
//   round_bytes (cost_model.cpp:47-51)    -> EvalPlan::round_bytes (same FP64 ops)
//   expand_dbt (cost_model.cpp:194-222)   -> build_dbt_plan (critical-path tree)
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>

#include "rw_internal.h"

namespace rwb {

void cuda_check(cudaError_t e, const char* expr, const char* file, int line) {
  if (e == cudaSuccess) return;
  throw Failure(RW_ERR_CUDA, std::string("CUDA error ") + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) +
                                 ") at " + file + ":" + std::to_string(line) + ": " + expr);
}

DeviceGuard::DeviceGuard(int dev) {
  RW_CUDA(cudaGetDevice(&prev));
  if (prev != dev) RW_CUDA(cudaSetDevice(dev));
}
DeviceGuard::~DeviceGuard() {
  int cur = -1;
  if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
}

// ------------------------------------------------------------ thread ctx --
namespace {
thread_local StreamScratch* t_stream_scratch = nullptr;
}

StreamScratch::StreamScratch(int dev, cudaStream_t s) : device(dev), stream(s), prev(t_stream_scratch) {
  // Keep freed blocks in the device's default pool: a call's scratch is then
  // a pool hit (microseconds), not a fresh cudaMalloc.
  static thread_local int configured = -1;
  if (configured != dev) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
    configured = dev;
  }
  t_stream_scratch = this;
}

StreamScratch::~StreamScratch() {
  for (int i = 0; i < 8; ++i)
    if (buf[i]) cudaFreeAsync(buf[i], stream);  // stream-ordered: after this call's kernels
  t_stream_scratch = prev;
}

void* StreamScratch::get(int slot, size_t bytes) {
  if (cap[slot] < bytes) {
    if (buf[slot]) RW_CUDA(cudaFreeAsync(buf[slot], stream));
    buf[slot] = nullptr;
    RW_CUDA(cudaMallocAsync(&buf[slot], bytes, stream));
    cap[slot] = bytes;
  }
  return buf[slot];
}

void* ThreadCtx::scratch(int slot, size_t bytes) {
  // Inside an asynchronous *_device call the scratch is stream-ordered on the
  // caller's stream (StreamScratch), never the per-thread buffers that the
  // host-buffer calls use on the internal streams.
  if (t_stream_scratch && t_stream_scratch->device == device) return t_stream_scratch->get(slot, bytes);
  if (d_cap[slot] < bytes) {
    if (d_buf[slot]) {
      RW_CUDA(cudaStreamSynchronize(stream[0]));
      RW_CUDA(cudaStreamSynchronize(stream[1]));
      RW_CUDA(cudaFree(d_buf[slot]));
      d_buf[slot] = nullptr;
    }
    size_t cap = bytes + bytes / 2 + 256;
    RW_CUDA(cudaMalloc(&d_buf[slot], cap));
    d_cap[slot] = cap;
  }
  return d_buf[slot];
}

void* ThreadCtx::pinned(size_t bytes) {
  if (h_cap < bytes) {
    if (h_pin) {
      RW_CUDA(cudaStreamSynchronize(stream[0]));
      RW_CUDA(cudaStreamSynchronize(stream[1]));
      RW_CUDA(cudaFreeHost(h_pin));
      h_pin = nullptr;
    }
    const size_t cap = std::max<size_t>(bytes + bytes / 2, 64 * 1024);
    // mapped: small calls let the kernel read the orders and write the costs
    // here directly (zero-copy), without separate copy operations
    RW_CUDA(cudaHostAlloc(&h_pin, cap, cudaHostAllocMapped | cudaHostAllocPortable));
    RW_CUDA(cudaHostGetDevicePointer(&d_pin, h_pin, 0));
    h_cap = cap;
  }
  return h_pin;
}

namespace {
// One context per (thread, device).  Not torn down by thread-exit handlers
// (CUDA objects must not be destroyed during process shutdown); threads the
// library owns release theirs explicitly (thread_ctx_release).
thread_local std::map<int, ThreadCtx*> t_ctxs;
}  // namespace

void thread_ctx_release() {
  for (auto& kv : t_ctxs) {
    ThreadCtx* c = kv.second;
    if (cudaSetDevice(c->device) == cudaSuccess) {
      for (auto& s : c->stream) cudaStreamSynchronize(s);
      for (void* b : c->d_buf)
        if (b) cudaFree(b);
      if (c->d_err) cudaFree(c->d_err);
      if (c->h_err) cudaFreeHost(c->h_err);
      if (c->h_pin) cudaFreeHost(c->h_pin);
      for (auto& e : c->ev) cudaEventDestroy(e);
      for (auto& s : c->stream) cudaStreamDestroy(s);
    }
    cudaGetLastError();
    delete c;
  }
  t_ctxs.clear();
}

ThreadCtx& thread_ctx(int device) {
  auto& ctxs = t_ctxs;
  auto it = ctxs.find(device);
  if (it != ctxs.end()) return *it->second;
  auto* c = new ThreadCtx();
  c->device = device;
  for (auto& s : c->stream) RW_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  for (auto& e : c->ev) RW_CUDA(cudaEventCreate(&e));
  RW_CUDA(cudaMalloc(&c->d_err, 2 * sizeof(unsigned long long)));
  const unsigned long long init[2] = {0ull, ~0ull};
  RW_CUDA(cudaMemcpy(c->d_err, init, sizeof(init), cudaMemcpyHostToDevice));
  RW_CUDA(cudaMallocHost(&c->h_err, 2 * sizeof(unsigned long long)));
  ctxs[device] = c;
  return *c;
}

void raise_order_errors(int* d_err, int* h_err, cudaStream_t st) {
  RW_CUDA(cudaMemcpyAsync(h_err, d_err, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  RW_CUDA(cudaStreamSynchronize(st));
  auto* h = reinterpret_cast<unsigned long long*>(h_err);
  if (h[0] != 0) {
    const unsigned long long bad = h[1];
    const unsigned long long init[2] = {0ull, ~0ull};
    RW_CUDA(cudaMemcpyAsync(d_err, init, sizeof(init), cudaMemcpyHostToDevice, st));
    RW_CUDA(cudaStreamSynchronize(st));
    throw Failure(RW_ERR_DOMAIN, "rank order is not a permutation of [0, " + std::to_string(h[0] >> 32) +
                                     ") (batch entry " + std::to_string(bad) + ")");
  }
}

// ---------------------------------------------------------- validation ----
static bool is_power_of(long long n, long long base) {
  if (base < 2 || n < 1) return false;
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

static const char* algo_name(int a) {
  switch (a) {
    case kRing: return "ring";
    case kHalvingDoubling: return "hd";
    case kDoubleBinaryTree: return "dbt";
    case kBCube: return "bcube";
  }
  return "?";
}

void validate_spec(const rw_spec& s) {
  if (s.n < 1) fail_domain("node count must be >= 1");
  if (!(s.size_bytes > 0.0)) fail_domain("data size must be > 0");
  if (s.algorithm < kRing || s.algorithm > kBCube) fail_domain("evaluate: unknown algorithm");
  if (s.cost_mode != RW_LATENCY_ONLY && s.cost_mode != RW_LATENCY_TIMES_SIZE) fail_domain("unknown cost mode");
  if (s.hd_pairing != RW_PAIRING_PAPER && s.hd_pairing != RW_PAIRING_XOR) fail_domain("unknown pairing");
  if (s.n == 1) return;  // degenerate single-node collective
  switch (s.algorithm) {
    case kHalvingDoubling:
    case kDoubleBinaryTree:
      if (!is_power_of(s.n, 2))
        fail_domain(std::string(algo_name(s.algorithm)) + " requires N a power of 2, got " + std::to_string(s.n));
      break;
    case kBCube:
      if (s.bcube_b < 2) fail_domain("BCube group size B must be >= 2");
      if (!is_power_of(s.n, s.bcube_b))
        fail_domain("BCube requires N a power of B=" + std::to_string(s.bcube_b) + ", got " + std::to_string(s.n));
      break;
    default: break;
  }
}

// ------------------------------------------------------------- dbt plan ---
// Emits the transfers of both trees in the same order as the reference's
// expansion: per depth, left edge then its subtree, then right edge.
static void build_dbt_plan(DbtPlan& plan, int n) {
  struct E {
    int src, dst, parent;
  };
  std::vector<std::vector<E>> rounds;
  auto alias = [n](int r) { return ((r % n) + n) % n; };
  // explicit recursion on a small stack (depth <= log2 n + 1)
  struct Frame {
    int i, j, shift, depth, parent, stage, mid;
  };
  for (int shift : {0, -1}) {
    std::vector<Frame> st;
    st.push_back({0, n - 1, shift, 0, -1, 0, 0});
    while (!st.empty()) {
      Frame& f = st.back();
      if (f.stage == 0) {
        if (f.i >= f.j) {
          st.pop_back();
          continue;
        }
        if (static_cast<int>(rounds.size()) <= f.depth) rounds.resize(f.depth + 1);
        f.mid = (f.i + f.j) / 2;
        const int left_peer = (3 * f.i + f.j) / 2 - 1;
        const int idx = static_cast<int>(rounds[f.depth].size());
        rounds[f.depth].push_back({alias(f.mid + f.shift), alias(left_peer + f.shift), f.parent});
        f.stage = 1;
        const Frame child{f.i, f.mid - 1, f.shift, f.depth + 1, idx, 0, 0};
        st.push_back(child);
      } else if (f.stage == 1) {
        const int right_peer = (f.i + 3 * f.j) / 2 + 1;
        const int idx = static_cast<int>(rounds[f.depth].size());
        rounds[f.depth].push_back({alias(f.mid + f.shift), alias(right_peer + f.shift), f.parent});
        f.stage = 2;
        const Frame child{f.mid + 1, f.j, f.shift, f.depth + 1, idx, 0, 0};
        st.push_back(child);
      } else {
        st.pop_back();
      }
    }
  }
  plan.n = n;
  plan.depths = static_cast<int>(rounds.size());
  plan.h_depth_off.assign(plan.depths + 1, 0);
  for (int d = 0; d < plan.depths; ++d)
    plan.h_depth_off[d + 1] = plan.h_depth_off[d] + static_cast<int>(rounds[d].size());
  plan.edges = plan.h_depth_off[plan.depths];
  plan.h_src.resize(plan.edges);
  plan.h_dst.resize(plan.edges);
  plan.h_c0.assign(plan.edges, -1);
  plan.h_c1.assign(plan.edges, -1);
  for (int d = 0; d < plan.depths; ++d) {
    for (size_t t = 0; t < rounds[d].size(); ++t) {
      const int g = plan.h_depth_off[d] + static_cast<int>(t);
      plan.h_src[g] = rounds[d][t].src;
      plan.h_dst[g] = rounds[d][t].dst;
      if (d > 0) {
        const int parent = plan.h_depth_off[d - 1] + rounds[d][t].parent;
        if (plan.h_c0[parent] < 0) plan.h_c0[parent] = g;
        else plan.h_c1[parent] = g;
      }
    }
  }
  // Packed records: positions fit 16 bits (n <= 65536), and the two children of
  // an edge are adjacent in their depth list (the left edge of the child node
  // is pushed, then only deeper edges, then its right edge), so c1 = c0 + 1.
  std::vector<int32_t> all;
  all.reserve(2 * static_cast<size_t>(plan.edges) + plan.depths + 1);
  for (int e = 0; e < plan.edges; ++e) {
    const size_t k = static_cast<size_t>(e);
    if ((plan.h_c0[k] < 0) != (plan.h_c1[k] < 0) || (plan.h_c0[k] >= 0 && plan.h_c1[k] != plan.h_c0[k] + 1))
      throw Failure(RW_ERR_INTERNAL, "dbt plan: children of an edge are not adjacent");
    all.push_back(static_cast<int32_t>(static_cast<uint32_t>(plan.h_src[k]) | (static_cast<uint32_t>(plan.h_dst[k]) << 16)));
    all.push_back(plan.h_c0[k]);
  }
  all.insert(all.end(), plan.h_depth_off.begin(), plan.h_depth_off.end());
  RW_CUDA(cudaMalloc(&plan.d_all, all.size() * sizeof(int32_t)));
  RW_CUDA(cudaMemcpy(plan.d_all, all.data(), all.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  // Delta-evaluation tables (swap moves in the tree-model anneal): per edge
  // (parent << 8) | depth, parent 0xFFFFFF at the roots; per position the (at
  // most 6) edges with that position as an endpoint, -1 padded to 8.
  std::vector<int32_t> aux(static_cast<size_t>(plan.edges) + 8 * static_cast<size_t>(n), -1);
  for (int d = 0; d < plan.depths; ++d)
    for (int e = plan.h_depth_off[d]; e < plan.h_depth_off[d + 1]; ++e) aux[static_cast<size_t>(e)] = (0xFFFFFF << 8) | d;
  for (int e = 0; e < plan.edges; ++e) {
    const int d = aux[static_cast<size_t>(e)] & 0xFF;
    for (int c : {plan.h_c0[static_cast<size_t>(e)], plan.h_c1[static_cast<size_t>(e)]})
      if (c >= 0) aux[static_cast<size_t>(c)] = (e << 8) | (d + 1);
  }
  for (int e = 0; e < plan.edges; ++e) {
    for (int x : {plan.h_src[static_cast<size_t>(e)], plan.h_dst[static_cast<size_t>(e)]}) {
      int32_t* slot = aux.data() + plan.edges + 8 * static_cast<size_t>(x);
      int k = 0;
      while (k < 8 && slot[k] >= 0 && slot[k] != e) ++k;
      if (k == 8) fail_internal("double binary tree: more than 8 edges at one position");
      slot[k] = e;
    }
  }
  RW_CUDA(cudaMalloc(&plan.d_aux, aux.size() * sizeof(int32_t)));
  RW_CUDA(cudaMemcpy(plan.d_aux, aux.data(), aux.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
}

// ------------------------------------------------------------- planning ---
static double round_bytes(double size_bytes, int base, int round) {
  double divisor = 1.0;
  for (int k = 0; k <= round; ++k) divisor *= static_cast<double>(base);
  return size_bytes / divisor;
}

// Rounds of transfers in rank space; the double binary tree reuses the
// critical-path plan builder's emission order (left edge, its subtree, right
// edge, its subtree; primary tree then mirrored tree).
Expanded expand_schedule_core(const rw_spec& s) {
  validate_spec(s);
  Expanded e;
  const int n = s.n;
  auto alias = [n](int r) { return ((r % n) + n) % n; };
  auto close_round = [&] { e.off.push_back(static_cast<int32_t>(e.src.size())); };
  auto add = [&](int a, int b, double by, int parent) {
    e.src.push_back(a);
    e.dst.push_back(b);
    e.bytes.push_back(by);
    e.parent.push_back(parent);
  };
  if (n == 1) return e;  // no rounds
  switch (s.algorithm) {
    case kRing:
      e.semantics = RW_SEQUENTIAL_HOPS;
      for (int i = 0; i < n; ++i) {
        add(i, alias(i - 1), s.size_bytes, -1);
        close_round();
      }
      break;
    case kHalvingDoubling:
    case kBCube: {
      e.semantics = RW_BULK_SYNCHRONOUS_ROUNDS;
      const bool hd = s.algorithm == kHalvingDoubling;
      const int base = hd ? 2 : s.bcube_b;
      const int rounds = ilog_exact(n, base);
      long long stride = 1;
      for (int r = 0; r < rounds; ++r, stride *= base) {
        const double by = round_bytes(s.size_bytes, base, r);
        if (hd && s.hd_pairing == RW_PAIRING_XOR) {
          for (int j = 0; j < n; ++j) add(j, j ^ static_cast<int>(stride), by, -1);
        } else if (hd) {
          for (int j = 0; j < n / 2; ++j) add(j, alias(j + static_cast<int>(stride)), by, -1);
        } else {
          for (int j = 0; j < n / base; ++j)
            for (int k = 1; k < base; ++k) add(j, static_cast<int>((j + k * stride) % n), by, -1);
        }
        close_round();
      }
      break;
    }
    case kDoubleBinaryTree: {
      e.semantics = RW_CRITICAL_PATH;
      struct Edge {
        int src, dst, parent;
      };
      std::vector<std::vector<Edge>> rounds;
      struct Frame {
        int i, j, shift, depth, parent, stage, mid;
      };
      for (int shift : {0, -1}) {
        std::vector<Frame> st;
        st.push_back({0, n - 1, shift, 0, -1, 0, 0});
        while (!st.empty()) {
          Frame& f = st.back();
          if (f.stage == 0) {
            if (f.i >= f.j) {
              st.pop_back();
              continue;
            }
            if (static_cast<int>(rounds.size()) <= f.depth) rounds.resize(f.depth + 1);
            f.mid = (f.i + f.j) / 2;
            const int idx = static_cast<int>(rounds[f.depth].size());
            rounds[f.depth].push_back({alias(f.mid + f.shift), alias((3 * f.i + f.j) / 2 - 1 + f.shift), f.parent});
            f.stage = 1;
            const Frame child{f.i, f.mid - 1, f.shift, f.depth + 1, idx, 0, 0};
            st.push_back(child);
          } else if (f.stage == 1) {
            const int idx = static_cast<int>(rounds[f.depth].size());
            rounds[f.depth].push_back({alias(f.mid + f.shift), alias((f.i + 3 * f.j) / 2 + 1 + f.shift), f.parent});
            f.stage = 2;
            const Frame child{f.mid + 1, f.j, f.shift, f.depth + 1, idx, 0, 0};
            st.push_back(child);
          } else {
            st.pop_back();
          }
        }
      }
      const double half = s.size_bytes / 2.0;
      for (const auto& r : rounds) {
        for (const auto& ed : r) add(ed.src, ed.dst, half, ed.parent);
        close_round();
      }
      break;
    }
  }
  return e;
}

// Odd integer mantissa of a positive finite double (x = m * 2^e, m odd).
static double odd_mantissa(double x) {
  int e = 0;
  double m = std::frexp(x, &e);  // x = m * 2^e, m in [0.5, 1)
  double mi = std::ldexp(m, 53);  // exact integer < 2^53
  while (mi != 0.0 && std::fmod(mi, 2.0) == 0.0) mi /= 2.0;
  return mi;
}

EvalPlan make_plan(Problem& p, const rw_spec& s) {
  validate_spec(s);
  if (p.n != s.n)
    fail_domain("matrix is " + std::to_string(p.n) + "x" + std::to_string(p.n) + " but spec has N=" +
                std::to_string(s.n));
  EvalPlan plan;
  plan.model = s.algorithm;
  plan.n = s.n;
  plan.mode = s.cost_mode;
  plan.pairing = s.hd_pairing;
  plan.bcube_b = s.bcube_b;
  plan.size_bytes = s.size_bytes;
  plan.half = s.size_bytes / 2.0;
  plan.bit_exact = true;
  if (s.n == 1) return plan;
  switch (s.algorithm) {
    case kRing: {
      const bool times = s.cost_mode == RW_LATENCY_TIMES_SIZE;
      if (p.storage == RW_STORAGE_U16) {
        plan.ring_int = true;
        plan.ring_mul = times ? p.scale * s.size_bytes : p.scale;
        // Every product and partial sum of the reference is exact when
        // n * max_q * odd(S) < 2^53; then sum(q) * scale * S is its value.
        const double odd = times ? odd_mantissa(s.size_bytes) : 1.0;
        const double bound = static_cast<double>(s.n) * static_cast<double>(p.max_q) * odd;
        plan.bit_exact = std::isfinite(plan.ring_mul) && bound < 9007199254740992.0;
      } else {
        plan.ring_int = false;
        plan.ring_mul = times ? s.size_bytes : 1.0;
        plan.bit_exact = false;
      }
      break;
    }
    case kHalvingDoubling: {
      plan.rounds = ilog_exact(s.n, 2);
      for (int r = 0; r < plan.rounds; ++r) plan.round_bytes[r] = round_bytes(s.size_bytes, 2, r);
      break;
    }
    case kBCube: {
      plan.rounds = ilog_exact(s.n, s.bcube_b);
      if (plan.rounds > kMaxRounds) fail_domain("BCube round count exceeds the supported maximum");
      for (int r = 0; r < plan.rounds; ++r) plan.round_bytes[r] = round_bytes(s.size_bytes, s.bcube_b, r);
      break;
    }
    case kDoubleBinaryTree: {
      std::lock_guard<std::mutex> lock(p.mu);
      if (!p.dbt) {
        DeviceGuard g(p.device);
        auto d = std::make_unique<DbtPlan>();
        build_dbt_plan(*d, s.n);
        p.dbt = std::move(d);
      }
      plan.dbt = p.dbt.get();
      if (p.storage == RW_STORAGE_U16) {
        // Each edge term is fl(q * 2^-f * half) (or q * 2^-f); with
        // (depths + 2) * max_q * odd(half) < 2^53 every term, sum and max
        // of the recursion (cost_model.cpp:94-116) is exact, so the result is
        // (max path sum of codes) * w, w = 2^-f * half, bit for bit.
        const bool times = s.cost_mode == RW_LATENCY_TIMES_SIZE;
        const double w = times ? p.scale * plan.half : p.scale;
        const double odd = times ? (plan.half > 0.0 ? odd_mantissa(plan.half) : 0.0) : 1.0;
        const double terms = static_cast<double>(plan.dbt->depths + 2) * static_cast<double>(p.max_q);
        plan.dbt_int = std::isfinite(w) && w > 0.0 && odd > 0.0 && terms * odd < 9007199254740992.0 &&
                       terms < 4294967295.0;
        plan.dbt_w = w;
      }
      break;
    }
  }
  return plan;
}

int64_t lookups_per_eval(const EvalPlan& plan) {
  const int64_t n = plan.n;
  if (n <= 1) return 0;
  switch (plan.model) {
    case kRing: return n;
    case kHalvingDoubling: return (plan.pairing == RW_PAIRING_PAPER ? n / 2 : n) * plan.rounds;
    case kBCube: return (n / plan.bcube_b) * (plan.bcube_b - 1) * plan.rounds;
    case kDoubleBinaryTree: return plan.dbt ? plan.dbt->edges : 2 * n;
  }
  return 0;
}

// ------------------------------------------------------------ creation ----
// Smallest f such that every entry is q * 2^-f with integer q (or -1).
static int needed_frac_bits(double v) {
  if (v == 0.0) return 0;
  int e = 0;
  const double m = std::frexp(v, &e);
  double mi = std::ldexp(m, 53);
  int tz = 0;
  while (std::fmod(mi, 2.0) == 0.0) {
    mi /= 2.0;
    ++tz;
  }
  const int f = 53 - e - tz;
  return f < 0 ? 0 : f;
}

static Problem* create_problem(const double* rtt, int n, int hint, int device) {
  if (n < 1) fail_domain("cost matrix is empty");
  if (n > 65536) fail_domain("n > 65536 is not supported (orders are stored as uint16 on the device)");
  int ndev = 0;
  RW_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0) RW_CUDA(cudaGetDevice(&device));
  if (device >= ndev) fail_domain("device " + std::to_string(device) + " does not exist");
  auto p = std::make_unique<Problem>();
  p->n = n;
  p->device = device;
  const size_t nn = static_cast<size_t>(n) * static_cast<size_t>(n);

  bool finite_nonneg = true, f32_exact = true, sym = true, zdiag = true;
  int frac = 0;
  double vmax = 0.0;
  for (size_t k = 0; k < nn; ++k) {
    const double v = rtt[k];
    if (!(std::isfinite(v) && v >= 0.0) || std::signbit(v)) finite_nonneg = false;
    if (static_cast<double>(static_cast<float>(v)) != v) f32_exact = false;
    if (finite_nonneg) {
      const int f = needed_frac_bits(v);
      if (f > frac) frac = f;
      if (v > vmax) vmax = v;
    }
  }
  for (int i = 0; i < n && (sym || zdiag); ++i) {
    if (rtt[static_cast<size_t>(i) * n + i] != 0.0) zdiag = false;
    for (int j = i + 1; j < n && sym; ++j)
      if (rtt[static_cast<size_t>(i) * n + j] != rtt[static_cast<size_t>(j) * n + i]) sym = false;
  }
  const bool u16_ok = finite_nonneg && frac <= 30 && std::ldexp(vmax, frac) <= 65535.0;
  int storage = RW_STORAGE_F64;
  switch (hint) {
    case RW_STORAGE_AUTO: storage = u16_ok ? RW_STORAGE_U16 : f32_exact ? RW_STORAGE_F32 : RW_STORAGE_F64; break;
    case RW_STORAGE_U16:
      if (!u16_ok) fail_domain("matrix is not representable as 16-bit fixed point");
      storage = RW_STORAGE_U16;
      break;
    case RW_STORAGE_F32:
      if (!f32_exact) fail_domain("matrix is not exactly representable in FP32");
      storage = RW_STORAGE_F32;
      break;
    case RW_STORAGE_F64: storage = RW_STORAGE_F64; break;
    default: fail_domain("unknown storage hint");
  }
  p->storage = storage;
  p->symmetric = sym;
  p->zero_diag = zdiag;
  p->max_value = vmax;
  if (storage == RW_STORAGE_U16) {
    p->frac_bits = frac;
    p->scale = std::ldexp(1.0, -frac);
  }

  DeviceGuard g(device);
  p->mat_bytes = nn * p->elem_bytes();
  RW_CUDA(cudaMalloc(&p->d_mat, p->mat_bytes));
  std::vector<unsigned char> staged(p->mat_bytes);
  if (storage == RW_STORAGE_U16) {
    auto* q = reinterpret_cast<uint16_t*>(staged.data());
    uint32_t mq = 0;
    for (size_t k = 0; k < nn; ++k) {
      q[k] = static_cast<uint16_t>(std::ldexp(rtt[k], frac));
      if (q[k] > mq) mq = q[k];
    }
    p->max_q = mq;
  } else if (storage == RW_STORAGE_F32) {
    auto* f = reinterpret_cast<float*>(staged.data());
    for (size_t k = 0; k < nn; ++k) f[k] = static_cast<float>(rtt[k]);
  } else {
    std::memcpy(staged.data(), rtt, p->mat_bytes);
  }
  RW_CUDA(cudaMemcpy(p->d_mat, staged.data(), p->mat_bytes, cudaMemcpyHostToDevice));
  RW_CUDA(cudaMalloc(&p->d_err, 2 * sizeof(unsigned long long)));
  const unsigned long long init[2] = {0ull, ~0ull};
  RW_CUDA(cudaMemcpy(p->d_err, init, sizeof(init), cudaMemcpyHostToDevice));
  return p.release();
}

// A replica of `src` on another device: the host-side analysis and metadata
// are copied, the device matrix is allocated but NOT filled (the problem set
// broadcasts it from the first member over NVLink, rw_multi.cpp).
static Problem* replica_problem(const Problem& src, int device) {
  auto p = std::make_unique<Problem>();
  p->n = src.n;
  p->device = device;
  p->storage = src.storage;
  p->frac_bits = src.frac_bits;
  p->scale = src.scale;
  p->symmetric = src.symmetric;
  p->zero_diag = src.zero_diag;
  p->max_value = src.max_value;
  p->max_q = src.max_q;
  p->mat_bytes = src.mat_bytes;
  p->path = src.path;
  DeviceGuard g(device);
  RW_CUDA(cudaMalloc(&p->d_mat, p->mat_bytes));
  RW_CUDA(cudaMalloc(&p->d_err, 2 * sizeof(unsigned long long)));
  const unsigned long long init[2] = {0ull, ~0ull};
  RW_CUDA(cudaMemcpy(p->d_err, init, sizeof(init), cudaMemcpyHostToDevice));
  return p.release();
}

static void destroy_problem(Problem* p) {
  if (!p) return;
  resident_release(*p);
  {
    DeviceGuard g(p->device);
    cudaDeviceSynchronize();
    if (p->d_mat) cudaFree(p->d_mat);
    if (p->d_err) cudaFree(p->d_err);
    if (p->dbt && p->dbt->d_all) cudaFree(p->dbt->d_all);
    if (p->dbt && p->dbt->d_aux) cudaFree(p->dbt->d_aux);
    if (p->d_nb) cudaFree(p->d_nb);
    if (p->d_rank) cudaFree(p->d_rank);
    if (p->d_rank_vals) cudaFree(p->d_rank_vals);
  }
  delete p;
}

}  // namespace rwb

// Exposed to rw_capi.cpp
namespace rwb {
Problem* problem_create(const double* rtt, int n, int hint, int device) { return create_problem(rtt, n, hint, device); }
void problem_destroy(Problem* p) { destroy_problem(p); }
Problem* problem_replica(const Problem& src, int device) { return replica_problem(src, device); }
}  // namespace rwb
