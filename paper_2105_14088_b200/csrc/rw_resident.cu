// rw_resident.cu -- resident evaluator for single-order calls (rw_evaluate,
// the reference's evaluate(), cost_model.cpp:140-148).
//
// A launched single-order evaluation pays a kernel launch (3.6 us of host time
// on the B200 boxes, ~7.5 us until a store of the kernel is visible to a
// polling host; scripts/microbench/roundtrip.cu) on top of the work.  With
// rw_problem_set_resident the problem instead keeps ONE CTA resident on its
// device that polls a mailbox in mapped pinned host memory: the host writes
// the request (the EvalPlan facts the kernels take as launch arguments) and
// the order, then bumps a sequence number; the CTA reads both over PCIe,
// evaluates with the same device code and operation sequence as the launched
// kernels (ring: k_ring's integer sum or k_ring_exact's sorted sum; HD /
// BCube: warp_rounds_cost; DBT: warp_dbt_cost), stores the cost and then the
// sequence number back into the mailbox.
//
// Lifetime: the CTA leaves after `idle` without a request (and after at most
// kLifeNs even under load, so a device-wide synchronisation elsewhere in the
// process waits a bounded time).  Before leaving it takes a final look at the
// request slot; only when that is still empty does it publish its epoch in
// `exited`.  A host that finds its request unanswered and the current epoch
// exited relaunches with the last served sequence number, so no request is
// lost or served twice.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>

#include "rw_device.cuh"
#include "rw_internal.h"
#include "rw_models.cuh"

namespace rwb {
namespace {

using namespace dev;

constexpr int kResThreads = 256;
constexpr unsigned long long kStop = ~0ull;
constexpr long long kLifeNs = 5'000'000;  // 5 ms

struct ResRequest {
  int32_t model;
  int32_t ring_fast;  // ring on u16 with EvalPlan::bit_exact: integer code sum (k_ring)
  int32_t mode;
  int32_t pad;
  double ring_mul;
  double size_bytes;
  RoundsArgs r;
  DbtArgs d;
};
static_assert(sizeof(ResRequest) % 16 == 0, "request is copied as 16-byte words");

struct Mailbox {
  unsigned long long req;     // host: sequence number of the posted request (written last)
  unsigned long long done;    // device: sequence number served (written after `cost`)
  unsigned long long exited;  // device: epoch of a server that has left
  unsigned long long pad0;
  double cost;
  double pad1;
  ResRequest rq;
  alignas(16) int32_t order[kResidentMaxN];
};

__host__ __device__ inline size_t al16(size_t x) { return (x + 15) & ~size_t(15); }
// DBT edges and depths the shared-memory layout holds (2N - 2 edges; depths <= 64)
__host__ __device__ inline int resident_edge_cap(int n) { return 2 * n + 64; }
constexpr int kResDepthCap = 64;

__device__ __forceinline__ long long global_ns() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <typename T>
__global__ void __launch_bounds__(kResThreads, 1) k_resident(Mailbox* mb, const T* __restrict__ gmat, double scale,
                                                            int n, unsigned long long last, unsigned long long epoch,
                                                            long long idle_ns) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ __align__(16) ResRequest s_rq;
  __shared__ unsigned long long s_seq;
  __shared__ unsigned long long s_part[kResThreads / 32];
  __shared__ typename MaxAcc<T>::type s_red[kMaxRounds * (kResThreads / 32)];
  __shared__ const uint2* s_plan_src;  // DBT plan currently staged in shared memory
  volatile Mailbox* vmb = mb;
  const int ecap = resident_edge_cap(n);
  uint16_t* s_perm = reinterpret_cast<uint16_t*>(smem);
  double* vals = reinterpret_cast<double*>(smem + al16((size_t)n * 2));
  uint2* s_rec = reinterpret_cast<uint2*>(smem + al16((size_t)n * 2) + (size_t)ecap * 8);
  int32_t* s_doff = reinterpret_cast<int32_t*>(s_rec + ecap);
  if (threadIdx.x == 0) s_plan_src = nullptr;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long t_start = global_ns();
  long long t_last = t_start;
  for (;;) {
    if (threadIdx.x == 0) {
      unsigned long long seq = 0;  // 0: leave
      for (;;) {
        const unsigned long long r = vmb->req;
        if (r != last) {
          seq = r;
          break;
        }
        const long long now = global_ns();
        if (now - t_last > idle_ns || now - t_start > kLifeNs) {
          __threadfence_system();
          const unsigned long long r2 = vmb->req;  // final look before announcing the exit
          if (r2 != last) seq = r2;
          break;
        }
      }
      s_seq = seq;
    }
    __syncthreads();
    const unsigned long long seq = s_seq;
    if (seq == 0 || seq == kStop) {
      if (threadIdx.x == 0) {
        __threadfence_system();
        vmb->exited = epoch;
      }
      return;
    }
    // request and order: uncached loads of host memory, one PCIe round trip
    {
      const int4* src = reinterpret_cast<const int4*>(&mb->rq);
      int4* dst = reinterpret_cast<int4*>(&s_rq);
      constexpr int kWords = (int)(sizeof(ResRequest) / 16);
      for (int k = threadIdx.x; k < kWords; k += blockDim.x) dst[k] = __ldcv(src + k);
      const int4* o4 = reinterpret_cast<const int4*>(mb->order);
      for (int k = threadIdx.x; k < (n + 3) >> 2; k += blockDim.x) {
        const int4 v = __ldcv(o4 + k);
        const int i = k << 2;
        s_perm[i] = (uint16_t)v.x;
        if (i + 1 < n) s_perm[i + 1] = (uint16_t)v.y;
        if (i + 2 < n) s_perm[i + 2] = (uint16_t)v.z;
        if (i + 3 < n) s_perm[i + 3] = (uint16_t)v.w;
      }
    }
    __syncthreads();
    const ResRequest& q = s_rq;
    double cost = 0.0;
    if (n > 1) {
      if (q.model == kRing && q.ring_fast) {
        // k_ring: sum of the raw u16 codes (exact integer), times ring_mul
        unsigned long long acc = 0;
        for (int i = threadIdx.x; i < n; i += blockDim.x)
          acc += (unsigned long long)ld_matrix<T>(gmat, (size_t)s_perm[i] * n + s_perm[i == 0 ? n - 1 : i - 1]);
        acc = warp_sum(acc);
        if (lane == 0) s_part[warp] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
          unsigned long long t = 0;
          for (int w = 0; w < kResThreads / 32; ++w) t += s_part[w];
          cost = __dmul_rn((double)t, q.ring_mul);
        }
      } else if (q.model == kRing) {
        // k_ring_exact: fl(rtt * S) per hop, sorted ascending, summed serially
        const int np2 = 1 << (32 - __clz(n - 1));
        for (int i = threadIdx.x; i < np2; i += blockDim.x) {
          double h = __longlong_as_double(0x7ff0000000000000ll);
          if (i < n) {
            h = to_double(ld_matrix<T>(gmat, (size_t)s_perm[i] * n + s_perm[i == 0 ? n - 1 : i - 1]), scale);
            if (q.mode == RW_LATENCY_TIMES_SIZE) h = __dmul_rn(h, q.size_bytes);
          }
          vals[i] = h;
        }
        __syncthreads();
        bitonic_sort_block(vals, np2);
        if (threadIdx.x == 0) {
          double total = 0.0;
          for (int i = 0; i < n; ++i) total = __dadd_rn(total, vals[i]);
          cost = total;
        }
      } else if (q.model == kDoubleBinaryTree) {
        // the plan (edge records + depth offsets) stays staged across requests
        if (s_plan_src != q.d.rec) {
          for (int e = threadIdx.x; e < q.d.edges; e += blockDim.x) s_rec[e] = q.d.rec[e];
          for (int k = threadIdx.x; k <= q.d.depths; k += blockDim.x) s_doff[k] = q.d.depth_off[k];
          __syncthreads();
          if (threadIdx.x == 0) s_plan_src = q.d.rec;
        }
        DbtArgs d = q.d;
        d.rec = s_rec;
        d.depth_off = s_doff;
        const double best = cta_dbt_cost<kResThreads, T, false>(s_perm, n, gmat, d, scale, vals);
        if (threadIdx.x == 0) cost = best;
      } else {
        const double total = cta_rounds_cost<kResThreads, T, false, true>(s_perm, n, gmat, q.r, scale, s_red);
        if (threadIdx.x == 0) cost = total;
      }
    }
    if (threadIdx.x == 0) {
      vmb->cost = cost;
      __threadfence_system();
      vmb->done = seq;
      last = seq;
      t_last = global_ns();
    }
    __syncthreads();  // s_perm / s_rq / vals are rewritten by the next request
  }
}

// order (u16) | edge values (FP64) | DBT plan (8-byte records, depth offsets)
size_t resident_smem(int n) {
  const size_t e = (size_t)resident_edge_cap(n);
  return al16((size_t)n * 2) + e * 8 + e * 8 + (kResDepthCap + 1) * 4;
}

}  // namespace

struct ResidentServer {
  ~ResidentServer();
  std::mutex mu;
  int device = 0;
  long long idle_ns = 0;
  Mailbox* mb = nullptr;  // mapped pinned host memory
  Mailbox* d_mb = nullptr;
  cudaStream_t st = nullptr;
  unsigned long long epoch = 0;  // epoch of the last launched server
  unsigned long long seq = 0;    // last posted request
  bool launched = false;
};

namespace {

void launch_server(const Problem& p, ResidentServer& s) {
  const size_t smem = resident_smem(p.n);
  ++s.epoch;
  const unsigned long long last = static_cast<volatile Mailbox*>(s.mb)->done;
  switch (p.storage) {
    case RW_STORAGE_U16: {
      RW_CUDA(cudaFuncSetAttribute(k_resident<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_resident<uint16_t><<<1, kResThreads, smem, s.st>>>(s.d_mb, static_cast<const uint16_t*>(p.d_mat), p.scale,
                                                           p.n, last, s.epoch, s.idle_ns);
      break;
    }
    case RW_STORAGE_F32: {
      RW_CUDA(cudaFuncSetAttribute(k_resident<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_resident<float><<<1, kResThreads, smem, s.st>>>(s.d_mb, static_cast<const float*>(p.d_mat), p.scale, p.n,
                                                        last, s.epoch, s.idle_ns);
      break;
    }
    default: {
      RW_CUDA(cudaFuncSetAttribute(k_resident<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_resident<double><<<1, kResThreads, smem, s.st>>>(s.d_mb, static_cast<const double*>(p.d_mat), p.scale, p.n,
                                                         last, s.epoch, s.idle_ns);
      break;
    }
  }
  RW_CUDA(cudaGetLastError());
  s.launched = true;
}

// Stops a running server and waits for it (the CTA answers the stop request
// within one poll, or leaves on its own idle timeout).
void stop_server(ResidentServer& s) {
  if (!s.launched) return;
  volatile Mailbox* v = s.mb;
  if (v->exited != s.epoch) {
    std::atomic_thread_fence(std::memory_order_seq_cst);
    v->req = kStop;
  }
  RW_CUDA(cudaStreamSynchronize(s.st));
  v->req = v->done;  // no pending request for a later server
  s.seq = v->done;
  s.launched = false;
}

}  // namespace

// The last holder (the problem, or a call still in flight) stops the CTA and
// frees the mailbox.
ResidentServer::~ResidentServer() {
  DeviceGuard g(device);
  try {
    stop_server(*this);
  } catch (...) {
  }
  if (st) cudaStreamDestroy(st);
  if (mb) cudaFreeHost(mb);
}

void resident_release(Problem& p) {
  std::shared_ptr<ResidentServer> s = std::atomic_exchange(&p.resident, std::shared_ptr<ResidentServer>());
  s.reset();
}

void resident_configure(Problem& p, int idle_us) {
  if (idle_us <= 0) {
    resident_release(p);
    return;
  }
  if (p.n > kResidentMaxN) fail_domain("resident evaluation supports N <= " + std::to_string(kResidentMaxN));
  if (resident_smem(p.n) > 220 * 1024) fail_domain("resident evaluation: shared memory budget exceeded");
  const long long idle_ns = (long long)std::min(idle_us, 100000) * 1000;
  if (std::shared_ptr<ResidentServer> cur = std::atomic_load(&p.resident)) {
    std::lock_guard<std::mutex> lock(cur->mu);
    cur->idle_ns = idle_ns;  // taken by the next launch
    return;
  }
  DeviceGuard g(p.device);
  auto s = std::make_shared<ResidentServer>();
  s->device = p.device;
  s->idle_ns = idle_ns;
  RW_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&s->mb), sizeof(Mailbox), cudaHostAllocMapped | cudaHostAllocPortable));
  RW_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&s->d_mb), s->mb, 0));
  RW_CUDA(cudaStreamCreateWithFlags(&s->st, cudaStreamNonBlocking));
  std::memset(s->mb, 0, sizeof(Mailbox));
  std::shared_ptr<ResidentServer> expected;
  // a concurrent configure may have installed one first: keep that one
  std::atomic_compare_exchange_strong(&p.resident, &expected, s);
}

bool resident_evaluate(Problem& p, const EvalPlan& plan, const int32_t* perm, double* cost) {
  const std::shared_ptr<ResidentServer> s = std::atomic_load(&p.resident);
  if (!s || plan.n != p.n) return false;
  std::unique_lock<std::mutex> lock(s->mu, std::try_to_lock);
  if (!lock.owns_lock()) return false;  // another thread holds the server: take the launched path
  DeviceGuard g(p.device);
  NvtxRange nvtx("resident evaluate");
  ResRequest rq{};
  rq.model = plan.n <= 1 ? kRing : plan.model;
  rq.ring_fast = (plan.model == kRing && plan.bit_exact && p.storage == RW_STORAGE_U16) ? 1 : 0;
  rq.mode = plan.mode;
  rq.ring_mul = plan.ring_mul;
  rq.size_bytes = plan.size_bytes;
  if (plan.model == kDoubleBinaryTree && plan.n > 1) {
    rq.d.rec = plan.dbt->d_rec();
    rq.d.depth_off = plan.dbt->d_depth_off();
    rq.d.depths = plan.dbt->depths;
    rq.d.edges = plan.dbt->edges;
    rq.d.mode = plan.mode;
    rq.d.half = plan.half;
    rq.d.int_mode = plan.dbt_int ? 1 : 0;
    rq.d.w = plan.dbt_w;
    if (plan.dbt->edges > resident_edge_cap(p.n) || plan.dbt->depths > kResDepthCap) return false;
  } else if (plan.model == kHalvingDoubling || plan.model == kBCube) {
    rq.r.kind = plan.model == kBCube ? 2 : (plan.pairing == RW_PAIRING_PAPER ? 0 : 1);
    rq.r.sym = p.symmetric ? 1 : 0;
    rq.r.rounds = plan.rounds;
    rq.r.b = plan.bcube_b;
    rq.r.mode = plan.mode;
    for (int k = 0; k < plan.rounds; ++k) rq.r.bytes[k] = plan.round_bytes[k];
  }
  volatile Mailbox* v = s->mb;
  if (!s->launched || v->exited == s->epoch) launch_server(p, *s);
  std::memcpy(const_cast<ResRequest*>(&s->mb->rq), &rq, sizeof(rq));
  std::memcpy(const_cast<int32_t*>(s->mb->order), perm, (size_t)p.n * 4);
  std::atomic_thread_fence(std::memory_order_seq_cst);
  const unsigned long long seq = ++s->seq;
  v->req = seq;
  const auto t0 = std::chrono::steady_clock::now();
  for (unsigned spin = 1;; ++spin) {
    if (v->done == seq) break;
    if (v->exited == s->epoch && v->done != seq) {
      // the server left before it saw the request: a new one picks it up
      launch_server(p, *s);
      continue;
    }
    if ((spin & 4095u) == 0) {
      const cudaError_t e = cudaStreamQuery(s->st);
      if (e != cudaSuccess && e != cudaErrorNotReady) RW_CUDA(e);
      // a server that never gets an SM (the device is held by other work) must
      // not spin the caller forever
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(30))
        throw Failure(RW_ERR_CUDA, "resident evaluator: no answer within 30 s");
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  *cost = v->cost;
  return true;
}

}  // namespace rwb
