// rw_models.cuh -- warp-cooperative cost models over an order staged in
// shared memory.  Shared by the batch scorer (rw_eval.cu) and the annealer
// (rw_anneal.cu).  Each function returns the reference-identical FP64 cost
// (for ring: see the summation note in rw_eval.cu) in every lane.
#pragma once

#include "rw_device.cuh"
#include "rw_internal.h"

namespace rwb {
namespace dev {

template <typename T, bool kSmem>
__device__ __forceinline__ T mat_at(const T* m, int n, int a, int b) {
  if constexpr (kSmem) return m[a * n + b];
  else return ld_matrix<T>(m, (size_t)a * (size_t)n + (size_t)b);
}

struct RoundsArgs {
  int kind;  // 0 hd paper, 1 hd xor, 2 bcube
  int sym;   // symmetric matrix: xor pairs are looked up once (c(a,b) == c(b,a))
  int rounds;
  int b;
  int mode;
  double bytes[kMaxRounds];
};

struct DbtArgs {
  const uint2* rec;  // per edge {src | dst << 16, c0}: positions, first child edge (-1: none; c1 = c0 + 1)
  const int32_t* depth_off;
  int depths;
  int edges;
  int mode;
  double half;
  double* gvals;  // global per-warp scratch when shared memory is too small
  int stage_plan;  // kernels copy the plan arrays into shared memory at plan_off
  int plan_off;    // byte offset in the kernel's dynamic shared memory
  int int_mode;    // u16 storage, EvalPlan::dbt_int: uint32 path sums, vals as uint32
  double w;        // int_mode: value = sum * w
  const int32_t* pd;        // delta tables (anneal): per edge (parent << 8) | depth
  const int32_t* posedges;  //   per position 8 incident edges, -1 padded
};

// Unpacked edge record {src, dst, c0, c1} (children -1 when none).
__device__ __forceinline__ int4 dbt_rec(uint2 v) {
  const int c0 = (int)v.y;
  return make_int4((int)(v.x & 0xFFFFu), (int)(v.x >> 16), c0, c0 < 0 ? -1 : c0 + 1);
}

// Plan (edge records | depth_off, int32) in shared memory: 8 B per edge, one
// LDS.64 per edge.  All threads of the CTA call it before any early exit.
__host__ __device__ inline size_t dbt_plan_bytes(int edges, int depths) {
  return ((size_t)2 * edges + depths + 1) * 4 + 16;
}
__device__ __forceinline__ void stage_dbt_plan(DbtArgs& d, unsigned char* smem) {
  if (!d.stage_plan) return;
  uint2* r = reinterpret_cast<uint2*>(smem + d.plan_off);
  const int E = d.edges;
  for (int k = threadIdx.x; k < E; k += blockDim.x) r[k] = d.rec[k];
  int32_t* off = reinterpret_cast<int32_t*>(r + E);
  for (int k = threadIdx.x; k <= d.depths; k += blockDim.x) off[k] = d.depth_off[k];
  __syncthreads();
  d.rec = r;
  d.depth_off = off;
}

// Sum over rounds of the round maximum (cost_model.cpp:71-92, 118-138).
template <typename T, bool kSmem>
__device__ double warp_rounds_cost(const uint16_t* s_perm, int n, const T* mat, const RoundsArgs& r, double scale,
                                   int lane) {
  using Acc = typename MaxAcc<T>::type;
  double total = 0.0;
  long long stride = 1;
  for (int rd = 0; rd < r.rounds; ++rd) {
    Acc mx = Acc(0);
    if (r.kind == 0) {
      const int s = 1 << rd;
      for (int j = lane; j < (n >> 1); j += 32)
        mx = ref_max<Acc>(mx, (Acc)mat_at<T, kSmem>(mat, n, s_perm[j], s_perm[j + s]));
    } else if (r.kind == 1) {
      const int s = 1 << rd;
      if (r.sym) {
        // each unordered pair {j, j^s} once: j with bit s clear.  On a
        // symmetric matrix both directions hold the same value, so the round
        // maximum is unchanged (NaN is never symmetric-equal; -0.0 never wins).
        for (int k = lane; k < (n >> 1); k += 32) {
          const int j = ((k >> rd) << (rd + 1)) | (k & (s - 1));
          mx = ref_max<Acc>(mx, (Acc)mat_at<T, kSmem>(mat, n, s_perm[j], s_perm[j + s]));
        }
      } else {
        for (int j = lane; j < n; j += 32) mx = ref_max<Acc>(mx, (Acc)mat_at<T, kSmem>(mat, n, s_perm[j], s_perm[j ^ s]));
      }
    } else {
      // BCube: sources j < N/B, partners j + k*B^i for k = 1..B-1.  The
      // reference's "% n" never fires (j + (B-1)*B^i <= N-1), so the pairs are
      // walked source by source with no division or modulo; the round maximum
      // is the same under any order.
      const int st = (int)stride;
      for (int j = lane; j < n / r.b; j += 32) {
        const int a = s_perm[j];
        for (int k = 1; k < r.b; ++k) mx = ref_max<Acc>(mx, (Acc)mat_at<T, kSmem>(mat, n, a, s_perm[j + k * st]));
      }
      stride *= r.b;
    }
    mx = warp_max(mx);
    double rm = to_double((T)mx, scale);
    if (r.mode == RW_LATENCY_TIMES_SIZE) rm = __dmul_rn(rm, r.bytes[rd]);
    total = __dadd_rn(total, rm);
  }
  return total;
}

// Double binary tree critical path (cost_model.cpp:94-116) over the
// depth-ordered expansion; vals is per-warp scratch of `edges` doubles.
template <typename T, bool kSmem>
__device__ double warp_dbt_cost(const uint16_t* s_perm, int n, const T* mat, const DbtArgs& d, double scale,
                                double* vals, int lane) {
  if (n <= 1) return 0.0;
  if constexpr (std::is_same<T, uint16_t>::value) {
    if (d.int_mode) {
      // exact integer form (EvalPlan::dbt_int): path sums of raw codes
      uint32_t* iv = reinterpret_cast<uint32_t*>(vals);
      for (int depth = d.depths - 1; depth >= 0; --depth) {
        const int lo = d.depth_off[depth], hi = d.depth_off[depth + 1];
#pragma unroll 4
        for (int e = lo + lane; e < hi; e += 32) {
          const int4 r = dbt_rec(d.rec[e]);
          const uint32_t c = (uint32_t)mat_at<T, kSmem>(mat, n, s_perm[r.x], s_perm[r.y]);
          uint32_t sub = 0;
          if (r.z >= 0) {
            const uint32_t x = iv[r.z], y = iv[r.w];
            sub = x > y ? x : y;
          }
          iv[e] = c + sub;
        }
        __syncwarp();
      }
      const uint32_t best = dbt_top_max<uint32_t>(d.depth_off[1], [&](int e) { return iv[e]; });
      __syncwarp();
      return __dmul_rn((double)best, d.w);
    }
  }
  for (int depth = d.depths - 1; depth >= 0; --depth) {
    const int lo = d.depth_off[depth], hi = d.depth_off[depth + 1];
#pragma unroll 4
    for (int e = lo + lane; e < hi; e += 32) {
      const int4 r = dbt_rec(d.rec[e]);
      double c = to_double(mat_at<T, kSmem>(mat, n, s_perm[r.x], s_perm[r.y]), scale);
      if (d.mode == RW_LATENCY_TIMES_SIZE) c = __dmul_rn(c, d.half);
      // value = cost(edge) + T(sub-interval); T(empty) = 0.0 (cost_model.cpp:105-113)
      const double sub = r.z >= 0 ? ref_max(vals[r.z], vals[r.w]) : 0.0;
      vals[e] = __dadd_rn(c, sub);
    }
    __syncwarp();
  }
  const double best = dbt_top_max<double>(d.depth_off[1], [&](int e) { return vals[e]; });
  __syncwarp();
  return best;
}

// Ring: sum of raw codes (integer for u16) -- used for exact resyncs in SA.
template <typename T, bool kSmem>
__device__ double warp_ring_raw(const uint16_t* s_perm, int n, const T* mat, int lane) {
  if constexpr (std::is_same<T, uint16_t>::value) {
    unsigned long long acc = 0;
    for (int i = lane; i < n; i += 32) acc += mat_at<T, kSmem>(mat, n, s_perm[i], s_perm[i == 0 ? n - 1 : i - 1]);
    return (double)warp_sum(acc);
  } else {
    double acc = 0.0;
    for (int i = lane; i < n; i += 32)
      acc = __dadd_rn(acc, (double)mat_at<T, kSmem>(mat, n, s_perm[i], s_perm[i == 0 ? n - 1 : i - 1]));
    return warp_sum(acc);
  }
}

// Double binary tree critical path by a CTA of kCta threads: each depth's
// edges are spread over the CTA, values in shared memory (vals: `edges`
// doubles, or uint32 in the exact integer form).  Same per-edge operation
// sequence and final max as warp_dbt_cost, so the value is bit-identical.
template <int kCta, typename T, bool kSmem>
__device__ __forceinline__ double cta_dbt_cost(const uint16_t* s_perm, int n, const T* mat, const DbtArgs& d,
                                               double scale, double* vals) {
  if (n <= 1) return 0.0;
  if constexpr (std::is_same<T, uint16_t>::value) {
    if (d.int_mode) {
      uint32_t* iv = reinterpret_cast<uint32_t*>(vals);
      for (int depth = d.depths - 1; depth >= 0; --depth) {
        const int lo = d.depth_off[depth], hi = d.depth_off[depth + 1];
#pragma unroll 2
        for (int e = lo + (int)threadIdx.x; e < hi; e += kCta) {
          const int4 r = dbt_rec(d.rec[e]);
          const uint32_t c = (uint32_t)mat_at<T, kSmem>(mat, n, s_perm[r.x], s_perm[r.y]);
          uint32_t sub = 0;
          if (r.z >= 0) {
            const uint32_t x = iv[r.z], y = iv[r.w];
            sub = x > y ? x : y;
          }
          iv[e] = c + sub;
        }
        __syncthreads();
      }
      const uint32_t best = dbt_top_max<uint32_t>(d.depth_off[1], [&](int e) { return iv[e]; });
      return __dmul_rn((double)best, d.w);
    }
  }
  for (int depth = d.depths - 1; depth >= 0; --depth) {
    const int lo = d.depth_off[depth], hi = d.depth_off[depth + 1];
#pragma unroll 2
    for (int e = lo + (int)threadIdx.x; e < hi; e += kCta) {
      const int4 r = dbt_rec(d.rec[e]);
      double c = to_double(mat_at<T, kSmem>(mat, n, s_perm[r.x], s_perm[r.y]), scale);
      if (d.mode == RW_LATENCY_TIMES_SIZE) c = __dmul_rn(c, d.half);
      const double sub = r.z >= 0 ? ref_max(vals[r.z], vals[r.w]) : 0.0;
      vals[e] = __dadd_rn(c, sub);
    }
    __syncthreads();
  }
  const double best = dbt_top_max<double>(d.depth_off[1], [&](int e) { return vals[e]; });
  return best;
}

// Sum over rounds of the round maximum by a CTA of kCta threads; red holds
// 2 * kCta / 32 entries (kFlat: rounds * kCta / 32, and the rounds' gathers
// run without a barrier between them).  The per-round maximum of raw codes is
// exact under any grouping (no NaN survives the running max from 0), and the
// rounds are summed in order, so the value equals warp_rounds_cost's.
template <int kCta, typename T, bool kSmem, bool kFlat = false>
__device__ __forceinline__ double cta_rounds_cost(const uint16_t* s_perm, int n, const T* mat, const RoundsArgs& r,
                                                  double scale, typename MaxAcc<T>::type* red) {
  using Acc = typename MaxAcc<T>::type;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  double total = 0.0;
  long long stride = 1;
  for (int rd = 0; rd < r.rounds; ++rd) {
    Acc mx = Acc(0);
    if (r.kind == 0) {
      const int s = 1 << rd;
      for (int j = t; j < (n >> 1); j += kCta)
        mx = ref_max<Acc>(mx, (Acc)mat_at<T, kSmem>(mat, n, s_perm[j], s_perm[j + s]));
    } else if (r.kind == 1) {
      const int s = 1 << rd;
      if (r.sym && n >= 2 * kCta) {  // each unordered pair once (warp_rounds_cost); small n: all lanes busy anyway
        for (int k = t; k < (n >> 1); k += kCta) {
          const int j = ((k >> rd) << (rd + 1)) | (k & (s - 1));
          mx = ref_max<Acc>(mx, (Acc)mat_at<T, kSmem>(mat, n, s_perm[j], s_perm[j + s]));
        }
      } else {
        for (int j = t; j < n; j += kCta) mx = ref_max<Acc>(mx, (Acc)mat_at<T, kSmem>(mat, n, s_perm[j], s_perm[j ^ s]));
      }
    } else {
      const int st = (int)stride;  // j + (B-1)*B^i <= N-1: no modulo (warp_rounds_cost)
      for (int j = t; j < n / r.b; j += kCta) {
        const int a = s_perm[j];
        for (int k = 1; k < r.b; ++k) mx = ref_max<Acc>(mx, (Acc)mat_at<T, kSmem>(mat, n, a, s_perm[j + k * st]));
      }
      stride *= r.b;
    }
    mx = warp_max(mx);
    if constexpr (kFlat) {
      // red holds rounds x (kCta / 32) entries: no barrier per round, one at the end
      if (lane == 0) red[rd * (kCta / 32) + w] = mx;
      continue;
    }
    if (lane == 0) red[(rd & 1) * (kCta / 32) + w] = mx;  // double-buffered by round parity
    __syncthreads();
    Acc m = red[(rd & 1) * (kCta / 32)];
#pragma unroll
    for (int k = 1; k < kCta / 32; ++k) m = ref_max<Acc>(m, red[(rd & 1) * (kCta / 32) + k]);
    double rm = to_double((T)m, scale);
    if (r.mode == RW_LATENCY_TIMES_SIZE) rm = __dmul_rn(rm, r.bytes[rd]);
    total = __dadd_rn(total, rm);
  }
  if constexpr (kFlat) {
    __syncthreads();
    for (int rd = 0; rd < r.rounds; ++rd) {
      Acc m = red[rd * (kCta / 32)];
#pragma unroll
      for (int k = 1; k < kCta / 32; ++k) m = ref_max<Acc>(m, red[rd * (kCta / 32) + k]);
      double rm = to_double((T)m, scale);
      if (r.mode == RW_LATENCY_TIMES_SIZE) rm = __dmul_rn(rm, r.bytes[rd]);
      total = __dadd_rn(total, rm);  // rounds summed in order, as above
    }
  }
  return total;
}

}  // namespace dev
}  // namespace rwb
