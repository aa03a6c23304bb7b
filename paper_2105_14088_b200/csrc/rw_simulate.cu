// rw_simulate.cu -- batched simulate_collective (proj/src/simulate.cpp:52-138)
// on the device: the equal-share flow model used as validation ground truth
// (SPEC.md cmd_validate).
//
// One warp per order.  For every round of the expanded schedule the warp
// counts, per directed link, the transfers crossing it (shared-memory
// counters, dense link index per level), then prices every transfer as
//   rtt[a][b] / 2 + bytes / min over its links (capacity / load)
// with the reference's FP64 operations, and combines rounds by the schedule
// semantics: serial sum in schedule order (sequential hops), sum of round
// maxima (bulk synchronous) or the critical path (double binary tree).
#include <algorithm>
#include <cmath>

#include "rw_device.cuh"
#include "rw_internal.h"

namespace rwb {

using namespace dev;

namespace {

constexpr int kMaxLevels = 8;

struct SimArgs {
  int n;
  int levels;
  long long group[kMaxLevels];    // product of fanouts[0..l]
  int link_base[kMaxLevels + 1];  // dense link index base per level (2 directions per link)
  double cap[kMaxLevels];         // bandwidth / oversub
  int semantics;
  int nrounds;
  const int32_t* off;
  const int32_t* src;
  const int32_t* dst;
  const double* bytes;
  const int32_t* parent;
  int edges;
  int unit_rounds;                // every round has exactly one transfer
  double* scratch;                // per warp: edges doubles (durations) + edges doubles (values)
  int link_words;
  double scale;
};

__device__ __forceinline__ int lca_level(const SimArgs& a, int i, int j) {
  for (int l = 0; l < a.levels; ++l)
    if (i / a.group[l] == j / a.group[l]) return l;
  return a.levels - 1;
}

__device__ __forceinline__ int link_index(const SimArgs& a, int host, int level, int dir) {
  const long long id = level == 0 ? host : host / a.group[level - 1];
  return a.link_base[level] + (int)(id * 2 + dir);
}

template <typename T>
__device__ double transfer_duration(const SimArgs& a, const T* mat, const uint32_t* load, int ha, int hb,
                                    double by) {
  double rate = __longlong_as_double(0x7ff0000000000000ll);  // +inf
  const int top = lca_level(a, ha, hb);
  for (int l = 0; l <= top; ++l) {
    rate = fmin(rate, __ddiv_rn(a.cap[l], (double)load[link_index(a, ha, l, 0)]));
    rate = fmin(rate, __ddiv_rn(a.cap[l], (double)load[link_index(a, hb, l, 1)]));
  }
  const double rtt = to_double(ld_matrix<T>(mat, (size_t)ha * a.n + hb), a.scale);
  return __dadd_rn(__ddiv_rn(rtt, 2.0), __ddiv_rn(by, rate));
}

template <typename T>
__global__ void __launch_bounds__(128) k_simulate(SimArgs a, const int32_t* __restrict__ perms, int64_t batch,
                                                  const T* __restrict__ mat, double* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint32_t* load = reinterpret_cast<uint32_t*>(smem) + (size_t)wib * a.link_words;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double* dur = a.scratch + (size_t)gw * 2 * a.edges;
  double* val = dur + a.edges;
  const int n = a.n;
  for (int64_t b = gw; b < batch; b += nw) {
    const int32_t* perm = perms + b * n;
    double total = 0.0;
    if (a.unit_rounds) {
      // every round is one transfer: each link carries load 1 in its round
      for (int k = lane; k < a.link_words; k += 32) load[k] = 1u;
      __syncwarp();
      for (int t = lane; t < a.edges; t += 32) {
        const int s = a.src[t], d = a.dst[t];
        dur[t] = s == d ? 0.0 : transfer_duration<T>(a, mat, load, perm[s], perm[d], a.bytes[t]);
      }
      __syncwarp();
      if (lane == 0)
        for (int t = 0; t < a.edges; ++t) total = __dadd_rn(total, dur[t]);  // schedule order
    } else {
      for (int r = 0; r < a.nrounds; ++r) {
        const int lo = a.off[r], hi = a.off[r + 1];
        for (int k = lane; k < a.link_words; k += 32) load[k] = 0u;
        __syncwarp();
        for (int t = lo + lane; t < hi; t += 32) {
          const int s = a.src[t], d = a.dst[t];
          if (s == d) continue;
          const int ha = perm[s], hb = perm[d];
          const int top = lca_level(a, ha, hb);
          for (int l = 0; l <= top; ++l) {
            atomicAdd(&load[link_index(a, ha, l, 0)], 1u);
            atomicAdd(&load[link_index(a, hb, l, 1)], 1u);
          }
        }
        __syncwarp();
        double rmax = 0.0;
        for (int t = lo + lane; t < hi; t += 32) {
          const int s = a.src[t], d = a.dst[t];
          const double dd = s == d ? 0.0 : transfer_duration<T>(a, mat, load, perm[s], perm[d], a.bytes[t]);
          dur[t] = dd;
          rmax = ref_max(rmax, dd);
        }
        __syncwarp();
        if (a.semantics == RW_BULK_SYNCHRONOUS_ROUNDS) {
          rmax = warp_max(rmax);
          total = __dadd_rn(total, rmax);
        } else if (a.semantics == RW_SEQUENTIAL_HOPS && lane == 0) {
          for (int t = lo; t < hi; ++t) total = __dadd_rn(total, dur[t]);
        }
      }
      if (a.semantics == RW_CRITICAL_PATH && lane == 0) {
        // leaf-up accumulation (simulate.cpp:114-135), value[t] = dur[t] + max child
        double best = 0.0;
        for (int r = a.nrounds - 1; r >= 0; --r) {
          const int lo = a.off[r], hi = a.off[r + 1];
          for (int t = lo; t < hi; ++t) val[t] = 0.0;  // child max, then value
          if (r + 1 < a.nrounds)
            for (int t = a.off[r + 1]; t < a.off[r + 2]; ++t) {
              const int pa = a.parent[t];
              if (pa >= 0 && lo + pa < hi) val[lo + pa] = ref_max(val[lo + pa], dur[t]);
            }
          for (int t = lo; t < hi; ++t) {
            dur[t] = __dadd_rn(dur[t], val[t]);  // dur now holds value[t]
            if (r == 0) best = ref_max(best, dur[t]);
          }
        }
        total = best;
      }
    }
    if (lane == 0) out[b] = total;
    __syncwarp();
  }
}

}  // namespace

void simulate_batch_device(Problem& p, const TopologyDesc& topo, const Expanded& sch, const int32_t* perms,
                           int64_t batch, double* out) {
  if (batch <= 0) return;
  const int levels = static_cast<int>(topo.fanout.size());
  if (levels < 1 || levels > kMaxLevels) fail_domain("simulate: 1..8 topology levels supported");
  DeviceGuard g(p.device);
  ThreadCtx& c = thread_ctx(p.device);
  cudaStream_t st = c.stream[0];
  const int n = p.n;
  SimArgs a{};
  a.n = n;
  a.levels = levels;
  long long grp = 1;
  int base = 0;
  for (int l = 0; l < levels; ++l) {
    const long long ids = (l == 0) ? n : n / grp;  // links at level l: one per level-(l-1) group
    a.link_base[l] = base;
    base += static_cast<int>(ids * 2);
    grp *= topo.fanout[static_cast<size_t>(l)];
    a.group[l] = grp;
    a.cap[l] = topo.capacity[static_cast<size_t>(l)];
  }
  a.link_base[levels] = base;
  a.link_words = base;
  a.semantics = sch.semantics;
  a.nrounds = sch.nrounds();
  a.edges = static_cast<int>(sch.src.size());
  a.scale = p.scale;
  bool unit = sch.semantics == RW_SEQUENTIAL_HOPS;
  for (int r = 0; r < a.nrounds && unit; ++r) unit = sch.off[r + 1] - sch.off[r] == 1;
  a.unit_rounds = unit ? 1 : 0;

  const int warps = 4;
  const size_t dyn = (size_t)warps * base * 4;
  if (dyn > 200 * 1024) fail_domain("simulate: topology has too many links for shared-memory counters");
  const int64_t want = (batch + warps - 1) / warps;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, 148 * 8));
  const size_t total_warps = (size_t)grid * warps;
  // device buffers: schedule | orders | out | per-warp scratch
  const size_t ints = (size_t)(a.nrounds + 1) + 3 * (size_t)a.edges;
  const size_t perm_bytes = (size_t)batch * n * 4;
  const size_t bytes_total = ((ints * 4 + 15) & ~size_t(15)) + (size_t)a.edges * 8 + ((perm_bytes + 15) & ~size_t(15)) +
                             (size_t)batch * 8 + total_warps * 2 * std::max(1, a.edges) * 8;
  char* buf = static_cast<char*>(c.scratch(7, bytes_total));
  int32_t* d_ints = reinterpret_cast<int32_t*>(buf);
  double* d_bytes = reinterpret_cast<double*>(buf + ((ints * 4 + 15) & ~size_t(15)));
  int32_t* d_perms = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(d_bytes) + (size_t)a.edges * 8);
  double* d_out = reinterpret_cast<double*>(reinterpret_cast<char*>(d_perms) + ((perm_bytes + 15) & ~size_t(15)));
  a.scratch = d_out + batch;
  std::vector<int32_t> hi;
  hi.reserve(ints);
  hi.insert(hi.end(), sch.off.begin(), sch.off.end());
  hi.insert(hi.end(), sch.src.begin(), sch.src.end());
  hi.insert(hi.end(), sch.dst.begin(), sch.dst.end());
  hi.insert(hi.end(), sch.parent.begin(), sch.parent.end());
  RW_CUDA(cudaMemcpyAsync(d_ints, hi.data(), hi.size() * 4, cudaMemcpyHostToDevice, st));
  if (a.edges) RW_CUDA(cudaMemcpyAsync(d_bytes, sch.bytes.data(), (size_t)a.edges * 8, cudaMemcpyHostToDevice, st));
  RW_CUDA(cudaMemcpyAsync(d_perms, perms, perm_bytes, cudaMemcpyHostToDevice, st));
  a.off = d_ints;
  a.src = d_ints + a.nrounds + 1;
  a.dst = a.src + a.edges;
  a.parent = a.dst + a.edges;
  a.bytes = d_bytes;
  switch (p.storage) {
    case RW_STORAGE_U16:
      if (dyn > 48 * 1024)
        RW_CUDA(cudaFuncSetAttribute(k_simulate<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
      k_simulate<uint16_t><<<grid, warps * 32, dyn, st>>>(a, d_perms, batch, static_cast<const uint16_t*>(p.d_mat), d_out);
      break;
    case RW_STORAGE_F32:
      if (dyn > 48 * 1024)
        RW_CUDA(cudaFuncSetAttribute(k_simulate<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
      k_simulate<float><<<grid, warps * 32, dyn, st>>>(a, d_perms, batch, static_cast<const float*>(p.d_mat), d_out);
      break;
    default:
      if (dyn > 48 * 1024)
        RW_CUDA(cudaFuncSetAttribute(k_simulate<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
      k_simulate<double><<<grid, warps * 32, dyn, st>>>(a, d_perms, batch, static_cast<const double*>(p.d_mat), d_out);
      break;
  }
  RW_CUDA(cudaGetLastError());
  RW_CUDA(cudaMemcpyAsync(out, d_out, (size_t)batch * 8, cudaMemcpyDeviceToHost, st));
  RW_CUDA(cudaStreamSynchronize(st));
}

}  // namespace rwb
