// rw_device.cuh -- device helpers shared by the scoring and search kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace rwb {
namespace dev {

constexpr unsigned kFull = 0xffffffffu;

// Raw matrix element -> FP64 value exactly as the reference's CostMatrix
// holds it.  u16 codes are q * 2^-f (scale is a power of two: exact).
__device__ __forceinline__ double to_double(uint16_t q, double scale) { return __dmul_rn((double)q, scale); }
__device__ __forceinline__ double to_double(float v, double) { return (double)v; }
__device__ __forceinline__ double to_double(double v, double) { return v; }

// std::max(a, b) == (a < b) ? b : a  (keeps the first argument on ties/NaN)
template <typename T>
__device__ __forceinline__ T ref_max(T a, T b) {
  return (a < b) ? b : a;
}

// The tree model's cost over its top edges.  For n >= 2 there are four, in
// plan order {primary left, primary right, mirrored left, mirrored right}:
// max(max(L0, R0), max(L1, R1)), the reference's std::max nesting
// (cost_model.cpp:112, 115).  A left-to-right fold differs from it when a
// path value is NaN, because std::max keeps its first argument then.
template <typename V, typename Get>
__device__ __forceinline__ V dbt_top_max(int top, Get v) {
  if (top == 4) return ref_max(ref_max(v(0), v(1)), ref_max(v(2), v(3)));
  V b = v(0);
  for (int e = 1; e < top; ++e) b = ref_max(b, v(e));
  return b;
}

template <typename T>
__device__ __forceinline__ T ld_matrix(const T* __restrict__ m, size_t idx) {
  return __ldg(m + idx);
}
template <>
__device__ __forceinline__ uint16_t ld_matrix<uint16_t>(const uint16_t* __restrict__ m, size_t idx) {
  return __ldg(reinterpret_cast<const unsigned short*>(m) + idx);
}

// Deterministic warp reductions (tree order fixed; result broadcast from lane 0).
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_down_sync(kFull, v, o));
  return __shfl_sync(kFull, v, 0);
}
__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(kFull, v, o);
  return __shfl_sync(kFull, v, 0);
}
__device__ __forceinline__ uint32_t warp_max(uint32_t v) { return __reduce_max_sync(kFull, v); }
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = ref_max(v, __shfl_xor_sync(kFull, v, o));
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = ref_max(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

// Accumulator type for max-of-rounds: u16 codes are compared as u32.
template <typename T>
struct MaxAcc {
  using type = T;
};
template <>
struct MaxAcc<uint16_t> {
  using type = uint32_t;
};

// Order element loaders (perm storage is uint16 or int32).
template <typename P>
__device__ __forceinline__ int ld_order(const P* __restrict__ p, int64_t i) {
  return (int)__ldg(p + i);
}
template <>
__device__ __forceinline__ int ld_order<uint16_t>(const uint16_t* __restrict__ p, int64_t i) {
  return (int)__ldg(reinterpret_cast<const unsigned short*>(p) + i);
}

// Error slot: {(n << 32) | 1, min bad batch index}.
__device__ __forceinline__ void report_bad_order(unsigned long long* err, int n, int64_t b) {
  atomicOr(err, ((unsigned long long)(unsigned)n << 32) | 1ull);
  atomicMin(err + 1, (unsigned long long)b);
}

// Bijection check of one order against per-warp marker bytes: every value in
// [0, n) must have been marked with `marker` by exactly the order's entries.
__device__ __forceinline__ bool flags_complete(const uint8_t* flags, int n, uint8_t marker, int lane) {
  bool bad = false;
  const uint32_t want = 0x01010101u * marker;
  const int words = n >> 2;
  const uint32_t* w = reinterpret_cast<const uint32_t*>(flags);
  for (int k = lane; k < words; k += 32) bad |= (w[k] != want);
  for (int k = (words << 2) + lane; k < n; k += 32) bad |= (flags[k] != marker);
  return !__any_sync(kFull, bad);
}

// ------------------------------------------------------------- Philox ----
// Philox4x32-10 (Salmon et al., SC'11): counter-based, keyed by (seed, chain).
struct Philox {
  uint4 ctr;
  uint2 key;
  uint4 buf;
  int used;
  __device__ __forceinline__ void init(uint64_t seed, uint64_t stream) {
    key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
    ctr = make_uint4(0u, 0u, (uint32_t)stream, (uint32_t)(stream >> 32));
    used = 4;
  }
  __device__ __forceinline__ static uint4 round(uint4 c, uint2 k) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    return make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  __device__ __forceinline__ uint4 block() {
    uint4 c = ctr;
    uint2 k = key;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      c = round(c, k);
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
    if (++ctr.x == 0) ++ctr.y;
    return c;
  }
  __device__ __forceinline__ uint32_t next() {
    if (used == 4) {
      buf = block();
      used = 0;
    }
    const uint32_t v = used == 0 ? buf.x : used == 1 ? buf.y : used == 2 ? buf.z : buf.w;
    ++used;
    return v;
  }
  // uniform integer in [0, range) (Lemire multiply-shift; bias < 2^-32 * range)
  __device__ __forceinline__ uint32_t below(uint32_t range) {
    return (uint32_t)(((uint64_t)next() * (uint64_t)range) >> 32);
  }
  // uniform double in [0, 1) with 53 random bits
  __device__ __forceinline__ double uniform() {
    const uint64_t hi = next(), lo = next();
    return (double)((hi << 21) | (lo >> 11)) * 0x1.0p-53;
  }
};

// Ascending bitonic sort of np2 (a power of two) doubles by the whole CTA
// (the sorted_sum order of cost_model.cpp:38-43; +inf pads sort last).
__device__ inline void bitonic_sort_block(double* v, int np2) {
  for (int k = 2; k <= np2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < np2; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const double x = v[i], y = v[ixj];
          const bool up = (i & k) == 0;
          if (up ? (x > y) : (x < y)) {
            v[i] = y;
            v[ixj] = x;
          }
        }
      }
      __syncthreads();
    }
  }
}
}  // namespace dev
}  // namespace rwb
