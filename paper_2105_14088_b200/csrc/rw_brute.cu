// rw_brute.cu -- exhaustive search (K2), replacing brute_force
// (proj/src/solver.cpp:73-105).
//
// The enumeration space is the lexicographic order of std::next_permutation:
// ring pins perm[0] = 0 and permutes positions 1..n-1 ((n-1)! orders), every
// other model permutes all n positions (n! orders).  The reference keeps the
// first strict minimum it meets, i.e. the lexicographically smallest optimal
// order; here every candidate carries its lexicographic index and the device
// reduces (cost, index) pairs, so ties resolve identically.
//
// Two kernels:
//  * k_brute_ring_int -- ring on u16 fixed-point matrices whose reference
//    arithmetic is exact (EvalPlan::bit_exact).  Threads own a prefix of the
//    order (unranked from the thread index); the last K positions are walked
//    by a depth-first search whose control flow is identical in every lane
//    (only the host ids differ), with integer partial sums -- about three
//    shared-memory lookups per enumerated order.
//  * k_brute_generic -- any model / storage, n <= 16: each thread walks a
//    contiguous run of lexicographic indices with next_permutation and
//    evaluates every order with the reference's exact FP64 sequence (ring:
//    sorted hops, serial sum).
#include <algorithm>
#include <cmath>
#include <vector>
#include <cstring>

#include "rw_device.cuh"
#include "rw_internal.h"

namespace rwb {

using namespace dev;

namespace {

__constant__ unsigned long long c_fact[21];

struct BestPair {
  double cost;
  unsigned long long index;
};

__device__ __forceinline__ bool better(double c, unsigned long long i, double bc, unsigned long long bi) {
  return c < bc || (c == bc && i < bi);
}

// Block-level (cost, index) argmin; thread 0 writes the block's pair.
__device__ void block_argmin(double cost, unsigned long long idx, BestPair* out) {
  __shared__ double s_c[32];
  __shared__ unsigned long long s_i[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double oc = __shfl_down_sync(kFull, cost, o);
    const unsigned long long oi = __shfl_down_sync(kFull, idx, o);
    if (better(oc, oi, cost, idx)) {
      cost = oc;
      idx = oi;
    }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    s_c[wid] = cost;
    s_i[wid] = idx;
  }
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    cost = lane < nw ? s_c[lane] : __longlong_as_double(0x7ff0000000000000ll);
    idx = lane < nw ? s_i[lane] : ~0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double oc = __shfl_down_sync(kFull, cost, o);
      const unsigned long long oi = __shfl_down_sync(kFull, idx, o);
      if (better(oc, oi, cost, idx)) {
        cost = oc;
        idx = oi;
      }
    }
    if (lane == 0) {
      out->cost = cost;
      out->index = idx;
    }
  }
}

__global__ void k_argmin_pairs(const BestPair* in, int count, BestPair* out) {
  double c = __longlong_as_double(0x7ff0000000000000ll);
  unsigned long long i = ~0ull;
  for (int k = threadIdx.x; k < count; k += blockDim.x)
    if (better(in[k].cost, in[k].index, c, i)) {
      c = in[k].cost;
      i = in[k].index;
    }
  block_argmin(c, i, out);
}

// ------------------------------------------------------- ring, integer ----
constexpr int kBruteThreads = 128;

template <int K>
struct DfsState {
  const uint32_t* sub;  // [(r*(K+1)+c)*T + tid]
  const uint32_t* wrap; // [r*T + tid]
  int T, tid;
  uint32_t best;
  uint32_t best_leaf;
  uint32_t leaf;
  uint32_t lo, hi;  // admissible leaf range of this thread's prefix
};

template <int D, int K>
__device__ __forceinline__ void dfs(DfsState<K>& s, uint32_t used, int prev, uint32_t cost) {
#pragma unroll 1
  for (int r = 0; r < K; ++r) {
    if (used & (1u << r)) continue;
    const uint32_t c = cost + s.sub[(r * (K + 1) + prev) * s.T + s.tid];
    if constexpr (D == K - 1) {
      const uint32_t total = c + s.wrap[r * s.T + s.tid];
      if (total < s.best && s.leaf >= s.lo && s.leaf < s.hi) {
        s.best = total;
        s.best_leaf = s.leaf;
      }
      ++s.leaf;
    } else {
      dfs<D + 1, K>(s, used | (1u << r), r, c);
    }
  }
}

template <int K>
__global__ void __launch_bounds__(kBruteThreads) k_brute_ring_int(const uint16_t* __restrict__ gmat, int n,
                                                                  unsigned long long prefix0,
                                                                  unsigned long long nprefix, unsigned long long first,
                                                                  unsigned long long end, double mul, BestPair* out) {
  __shared__ uint16_t s_mat[32 * 32];
  __shared__ uint32_t s_sub[K * (K + 1) * kBruteThreads];
  __shared__ uint32_t s_wrap[K * kBruteThreads];
  for (int k = threadIdx.x; k < n * n; k += blockDim.x) s_mat[k] = gmat[k];
  __syncthreads();
  const int tid = threadIdx.x;
  const unsigned long long p = prefix0 + (unsigned long long)blockIdx.x * blockDim.x + tid;
  DfsState<K> s;
  s.sub = s_sub;
  s.wrap = s_wrap;
  s.T = kBruteThreads;
  s.tid = tid;
  s.best = 0xffffffffu;
  s.best_leaf = 0;
  s.leaf = 0;
  s.lo = 0;
  s.hi = 0;
  const int free_n = n - 1;
  const unsigned long long kf = c_fact[K];
  if (p < prefix0 + nprefix) {
    // unrank the prefix: positions 1 .. n-1-K
    int remaining[20];
    int nrem = free_n;
    for (int k = 0; k < free_n; ++k) remaining[k] = k + 1;
    int last = 0;  // perm[0] = 0
    uint32_t pre = 0;
    unsigned long long q = p;
    for (int i = 0; i < free_n - K; ++i) {
      const unsigned long long w = c_fact[free_n - 1 - i] / kf;
      const int d = (int)(q / w);
      q -= (unsigned long long)d * w;
      const int h = remaining[d];
      for (int k = d; k < nrem - 1; ++k) remaining[k] = remaining[k + 1];
      --nrem;
      pre += s_mat[h * n + last];  // hop (perm[pos], perm[pos-1])
      last = h;
    }
    // suffix-local lookup tables
    for (int r = 0; r < K; ++r) {
      const int hr = remaining[r];
      for (int c = 0; c < K; ++c) s_sub[(r * (K + 1) + c) * kBruteThreads + tid] = s_mat[hr * n + remaining[c]];
      s_sub[(r * (K + 1) + K) * kBruteThreads + tid] = s_mat[hr * n + last];
      s_wrap[r * kBruteThreads + tid] = s_mat[0 * n + hr];  // hop 0: (perm[0], perm[n-1])
    }
    const unsigned long long base = p * kf;
    s.lo = base >= first ? 0u : (uint32_t)(first - base);
    s.hi = (uint32_t)(end - base < kf ? end - base : kf);
    dfs<0, K>(s, 0u, K, pre);
  }
  __syncthreads();  // (shared tables are per-thread; nothing to order)
  const bool found = s.best != 0xffffffffu;
  const double cost = found ? __dmul_rn((double)s.best, mul) : __longlong_as_double(0x7ff0000000000000ll);
  const unsigned long long idx = found ? p * kf + s.best_leaf : ~0ull;
  block_argmin(cost, idx, out + blockIdx.x);
}

// -------------------------------------------------------------- generic ----
constexpr int kNMax = 16;

struct GenericArgs {
  int n;
  int pinned;
  int model;
  int mode;
  int kind;  // rounds kind: 0 paper, 1 xor, 2 bcube
  int rounds;
  int b;
  double size_bytes;
  double half;
  double rbytes[kMaxRounds];
  int dbt_edges;
  int dbt_depths;
  int32_t dbt_src[2 * kNMax + 8];
  int32_t dbt_dst[2 * kNMax + 8];
  int32_t dbt_c0[2 * kNMax + 8];
  int32_t dbt_c1[2 * kNMax + 8];
  int32_t dbt_off[kNMax + 2];
};

__device__ double eval_exact(const GenericArgs& a, const double* m, const int* perm) {
  const int n = a.n;
  if (n == 1) return 0.0;
  if (a.model == kRing) {
    double h[kNMax];
    for (int i = 0; i < n; ++i) {
      double v = m[perm[i] * n + perm[i == 0 ? n - 1 : i - 1]];
      if (a.mode == RW_LATENCY_TIMES_SIZE) v = __dmul_rn(v, a.size_bytes);
      // insertion into the sorted prefix h[0..i)
      int j = i;
      while (j > 0 && h[j - 1] > v) {
        h[j] = h[j - 1];
        --j;
      }
      h[j] = v;
    }
    double total = 0.0;
    for (int i = 0; i < n; ++i) total = __dadd_rn(total, h[i]);
    return total;
  }
  if (a.model == kDoubleBinaryTree) {
    double val[2 * kNMax + 8];
    for (int d = a.dbt_depths - 1; d >= 0; --d)
      for (int e = a.dbt_off[d]; e < a.dbt_off[d + 1]; ++e) {
        double c = m[perm[a.dbt_src[e]] * n + perm[a.dbt_dst[e]]];
        if (a.mode == RW_LATENCY_TIMES_SIZE) c = __dmul_rn(c, a.half);
        const double sub = a.dbt_c0[e] >= 0 ? ref_max(val[a.dbt_c0[e]], val[a.dbt_c1[e]]) : 0.0;
        val[e] = __dadd_rn(c, sub);
      }
    return dbt_top_max<double>(a.dbt_off[1], [&](int e) { return val[e]; });
  }
  double total = 0.0;
  long long stride = 1;
  for (int r = 0; r < a.rounds; ++r) {
    double mx = 0.0;
    if (a.kind == 0) {
      for (int j = 0; j < n / 2; ++j) mx = ref_max(mx, m[perm[j] * n + perm[j + (1 << r)]]);
    } else if (a.kind == 1) {
      for (int j = 0; j < n; ++j) mx = ref_max(mx, m[perm[j] * n + perm[j ^ (1 << r)]]);
    } else {
      for (int j = 0; j < n / a.b; ++j)
        for (int k = 1; k < a.b; ++k) mx = ref_max(mx, m[perm[j] * n + perm[(int)((j + k * stride) % n)]]);
      stride *= a.b;
    }
    if (a.mode == RW_LATENCY_TIMES_SIZE) mx = __dmul_rn(mx, a.rbytes[r]);
    total = __dadd_rn(total, mx);
  }
  return total;
}

template <typename T>
__global__ void __launch_bounds__(256) k_brute_generic(GenericArgs a, const T* __restrict__ gmat, double scale,
                                                       unsigned long long first, unsigned long long end,
                                                       unsigned long long chunk, BestPair* out) {
  __shared__ double s_m[kNMax * kNMax];
  const int n = a.n;
  for (int k = threadIdx.x; k < n * n; k += blockDim.x) s_m[k] = to_double(gmat[k], scale);
  __syncthreads();
  double best = __longlong_as_double(0x7ff0000000000000ll);
  unsigned long long best_i = ~0ull;
  const unsigned long long t = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned long long start = first + t * chunk;
  if (start < end) {
    const unsigned long long stop = min(end, start + chunk);
    int perm[kNMax];
    // unrank start into perm (free positions pinned..n-1)
    int rem[kNMax];
    const int f = n - a.pinned;
    for (int k = 0; k < f; ++k) rem[k] = k + a.pinned;
    for (int k = 0; k < a.pinned; ++k) perm[k] = k;
    unsigned long long q = start;
    int nrem = f;
    for (int i = 0; i < f; ++i) {
      const unsigned long long w = c_fact[f - 1 - i];
      const int d = (int)(q / w);
      q -= (unsigned long long)d * w;
      perm[a.pinned + i] = rem[d];
      for (int k = d; k < nrem - 1; ++k) rem[k] = rem[k + 1];
      --nrem;
    }
    for (unsigned long long idx = start; idx < stop; ++idx) {
      const double c = eval_exact(a, s_m, perm);
      if (c < best) {
        best = c;
        best_i = idx;
      }
      // std::next_permutation on perm[pinned..n)
      int* v = perm + a.pinned;
      int i = f - 2;
      while (i >= 0 && v[i] >= v[i + 1]) --i;
      if (i < 0) break;
      int j = f - 1;
      while (v[j] <= v[i]) --j;
      int tmp = v[i];
      v[i] = v[j];
      v[j] = tmp;
      for (int l = i + 1, r = f - 1; l < r; ++l, --r) {
        tmp = v[l];
        v[l] = v[r];
        v[r] = tmp;
      }
    }
  }
  block_argmin(best, best_i, out + blockIdx.x);
}

unsigned long long factorial(int k) {
  unsigned long long f = 1;
  for (int i = 2; i <= k; ++i) f *= (unsigned long long)i;
  return f;
}

void upload_factorials() {
  static bool done[64] = {};
  int dev = 0;
  RW_CUDA(cudaGetDevice(&dev));
  if (dev < 64 && done[dev]) return;
  unsigned long long f[21];
  for (int k = 0; k <= 20; ++k) f[k] = factorial(k);
  RW_CUDA(cudaMemcpyToSymbol(c_fact, f, sizeof(f)));
  if (dev < 64) done[dev] = true;
}

template <int K>
void launch_ring_int(const Problem& p, const EvalPlan& plan, uint64_t first, uint64_t end, BestPair* d_part,
                     int& blocks, cudaStream_t st) {
  const unsigned long long kf = factorial(K);
  const unsigned long long p0 = first / kf;
  const unsigned long long p1 = (end + kf - 1) / kf;
  const unsigned long long np = p1 - p0;
  blocks = (int)((np + kBruteThreads - 1) / kBruteThreads);
  k_brute_ring_int<K><<<blocks, kBruteThreads, 0, st>>>(static_cast<const uint16_t*>(p.d_mat), plan.n, p0, np, first,
                                                       end, plan.ring_mul, d_part);
  RW_CUDA(cudaGetLastError());
}

}  // namespace

uint64_t brute_force_space(const rw_spec& s) {
  const int pinned = (s.algorithm == kRing && s.n >= 2) ? 1 : 0;
  const int f = s.n - pinned;
  if (f > 20) fail_domain("exhaustive search space exceeds 20! orders");
  return factorial(f);
}

void unrank(const rw_spec& s, uint64_t index, int32_t* perm) {
  const int n = s.n;
  const int pinned = (s.algorithm == kRing && n >= 2) ? 1 : 0;
  const int f = n - pinned;
  std::vector<int> rem;
  for (int k = pinned; k < n; ++k) rem.push_back(k);
  for (int k = 0; k < pinned; ++k) perm[k] = k;
  for (int i = 0; i < f; ++i) {
    const uint64_t w = factorial(f - 1 - i);
    const int d = static_cast<int>(index / w);
    index -= static_cast<uint64_t>(d) * w;
    perm[pinned + i] = rem[static_cast<size_t>(d)];
    rem.erase(rem.begin() + d);
  }
}

uint64_t brute_force_resolve(Problem& p, const EvalPlan& plan, const rw_spec& s, uint64_t index) {
  if (index >= brute_force_space(s)) return 0;
  std::vector<int32_t> first(static_cast<size_t>(s.n));
  unrank(s, 0, first.data());
  double c0 = 0.0;
  evaluate_host_orders(p, plan, first.data(), 1, &c0, true, false, nullptr);
  return std::isnan(c0) ? 0 : index;
}

void brute_force_range(const Problem& p, const EvalPlan& plan, uint64_t first, uint64_t count, double* cost_out,
                       uint64_t* index_out) {
  NvtxRange nvtx("K2 exhaustive range");
  DeviceGuard g(p.device);
  ThreadCtx& c = thread_ctx(p.device);
  cudaStream_t st = c.stream[0];
  upload_factorials();
  const uint64_t end = first + count;
  const int n = plan.n;
  if (count == 0) {
    *cost_out = std::numeric_limits<double>::infinity();
    *index_out = ~0ull;
    return;
  }
  int blocks = 0;
  BestPair* d_part = nullptr;
  const bool ring_int = plan.model == kRing && plan.ring_int && plan.bit_exact && n >= 4 && n <= 20;
  if (ring_int) {
    const int free_n = n - 1;
    // suffix length: at least ~2^17 prefixes (threads) when the space allows
    int K = std::min(8, free_n - 1);
    while (K > 3 && factorial(free_n) / factorial(K) < (1ull << 17)) --K;
    const unsigned long long kf = factorial(K);
    const uint64_t np = (end + kf - 1) / kf - first / kf;
    blocks = (int)((np + kBruteThreads - 1) / kBruteThreads);
    d_part = static_cast<BestPair*>(c.scratch(4, (size_t)(blocks + 1) * sizeof(BestPair)));
    switch (K) {
      case 3: launch_ring_int<3>(p, plan, first, end, d_part, blocks, st); break;
      case 4: launch_ring_int<4>(p, plan, first, end, d_part, blocks, st); break;
      case 5: launch_ring_int<5>(p, plan, first, end, d_part, blocks, st); break;
      case 6: launch_ring_int<6>(p, plan, first, end, d_part, blocks, st); break;
      case 7: launch_ring_int<7>(p, plan, first, end, d_part, blocks, st); break;
      default: launch_ring_int<8>(p, plan, first, end, d_part, blocks, st); break;
    }
  } else {
    if (n > kNMax) fail_domain("exhaustive search supports N <= 16 for this model/matrix");
    GenericArgs a{};
    a.n = n;
    a.pinned = (plan.model == kRing && n >= 2) ? 1 : 0;
    a.model = plan.model;
    a.mode = plan.mode;
    a.kind = plan.model == kBCube ? 2 : (plan.pairing == RW_PAIRING_PAPER ? 0 : 1);
    a.rounds = plan.rounds;
    a.b = plan.bcube_b;
    a.size_bytes = plan.size_bytes;
    a.half = plan.half;
    for (int r = 0; r < plan.rounds; ++r) a.rbytes[r] = plan.round_bytes[r];
    if (plan.model == kDoubleBinaryTree && n > 1) {
      const DbtPlan& d = *plan.dbt;
      a.dbt_edges = d.edges;
      a.dbt_depths = d.depths;
      for (int e = 0; e < d.edges; ++e) {
        a.dbt_src[e] = d.h_src[e];
        a.dbt_dst[e] = d.h_dst[e];
        a.dbt_c0[e] = d.h_c0[e];
        a.dbt_c1[e] = d.h_c1[e];
      }
      for (int k = 0; k <= d.depths; ++k) a.dbt_off[k] = d.h_depth_off[k];
    }
    const uint64_t threads_wanted = 148ull * 2048;
    const uint64_t chunk = std::max<uint64_t>(1, (count + threads_wanted - 1) / threads_wanted);
    const uint64_t nthreads = (count + chunk - 1) / chunk;
    blocks = (int)((nthreads + 255) / 256);
    d_part = static_cast<BestPair*>(c.scratch(4, (size_t)(blocks + 1) * sizeof(BestPair)));
    switch (p.storage) {
      case RW_STORAGE_U16:
        k_brute_generic<uint16_t><<<blocks, 256, 0, st>>>(a, static_cast<const uint16_t*>(p.d_mat), p.scale, first,
                                                          end, chunk, d_part);
        break;
      case RW_STORAGE_F32:
        k_brute_generic<float><<<blocks, 256, 0, st>>>(a, static_cast<const float*>(p.d_mat), p.scale, first, end,
                                                       chunk, d_part);
        break;
      default:
        k_brute_generic<double><<<blocks, 256, 0, st>>>(a, static_cast<const double*>(p.d_mat), p.scale, first, end,
                                                        chunk, d_part);
        break;
    }
    RW_CUDA(cudaGetLastError());
  }
  k_argmin_pairs<<<1, 1024, 0, st>>>(d_part, blocks, d_part + blocks);
  RW_CUDA(cudaGetLastError());
  BestPair h{};
  RW_CUDA(cudaMemcpyAsync(&h, d_part + blocks, sizeof(h), cudaMemcpyDeviceToHost, st));
  RW_CUDA(cudaStreamSynchronize(st));
  *cost_out = h.cost;
  *index_out = h.index;
}

namespace {
__global__ void k_select_key(SetReduce* r) {
  r->min_key = r->cost == r->min_cost ? r->key : ~0ull;
}
}  // namespace

void launch_select_key(SetReduce* d, cudaStream_t st) {
  k_select_key<<<1, 1, 0, st>>>(d);
  RW_CUDA(cudaGetLastError());
}

}  // namespace rwb
