// rw_rounds_transpose.cu -- halving-doubling scoring (paper and xor pairing)
// for matrices beyond one CTA's shared memory (C5: N=4096, 32 MiB u16),
// without random L2 gathers.  Same plan as the ring transpose path
// (rw_ring_transpose.cu):
//
//   route     one CTA per order: stage the order and its inverse pos = p^-1
//             in shared memory, then gather partner-by-host for every round,
//             part_r[h] = p[partner_r(pos[h])] (paper pairing: sources
//             pos[h] < N/2 only, other hosts get the 0xFFFF sentinel; xor:
//             every host is a source), written in 16-byte chunks grouped by
//             row block: buf[block][round][order][R].  It also resets the
//             order's per-round max keys.
//   score     a CTA keeps R matrix rows in shared memory; a producer warp
//             streams the block's partner slices with TMA bulk copies (one per
//             round and stage) through a full/empty mbarrier ring; each
//             consumer thread takes (round, order) tasks, walks the R rows and
//             folds the block maximum into key[round][order] with atomicMax.
//   finalize  per order, the reference's FP64 sequence fl(max * bytes_r)
//             summed over rounds in order (halving_doubling_cost,
//             proj/src/cost_model.cpp:71-92).
//
// Paper pairing and BCube take a source-compacted variant of route and score
// (k_rounds_route_compact / k_rounds_score_compact, below): per row block and
// order only the block's sources and their partners are written.
//
// Max is exact under any grouping, so the result is bit-identical to the
// L2-gather kernel on every storage kind.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "rw_device.cuh"
#include "rw_internal.h"
#include "rw_tma.cuh"

#include <cub/cub.cuh>

namespace rwb {

using namespace dev;

namespace {

__host__ __device__ inline size_t al16(size_t x) { return (x + 15) & ~size_t(15); }

// Order-preserving keys for the raw matrix codes (max over keys == the
// reference's running std::max from 0, cost_model.cpp:83: NaN never wins).
template <typename T>
struct KeyOf;
template <>
struct KeyOf<uint16_t> {
  using type = unsigned int;
  __device__ static unsigned int enc(uint16_t v) { return v; }
  __device__ static uint16_t dec(unsigned int k) { return (uint16_t)k; }
};
template <>
struct KeyOf<uint32_t> {  // ranks of FP64 values (order-preserving as integers)
  using type = unsigned int;
  __device__ static unsigned int enc(uint32_t v) { return v; }
  __device__ static uint32_t dec(unsigned int k) { return k; }
};
template <>
struct KeyOf<float> {
  using type = unsigned int;
  __device__ static unsigned int enc(float v) {
    if (v != v) return 0u;
    const unsigned int b = __float_as_uint(v);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
  }
  __device__ static float dec(unsigned int k) { return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k); }
};
template <>
struct KeyOf<double> {
  using type = unsigned long long;
  __device__ static unsigned long long enc(double v) {
    if (v != v) return 0ull;
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
  }
  __device__ static double dec(unsigned long long k) {
    return __longlong_as_double((long long)((k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k));
  }
};

// ------------------------------------------------------------------ route --
struct RRouteArgs {
  int64_t count;
  int64_t base;
  int n;
  int rounds;
  int xor_pairing;
  int R;
  unsigned long long* err;
  void* keys;       // [round][order], reset to key(0) here
  int key_bytes;    // 4 or 8
  unsigned long long zero_key;
  int aligned;      // order rows are 16-byte aligned
  int slots;        // partner slots per host: rounds, or ceil(rounds / 2) when paired
  int paired;       // symmetric matrix, xor pairing: one slot per round pair (below)
  int prefetch;     // register prefetch of the next order (uint16, aligned, n <= 4096)
};

// Stages one order into shared memory as uint16 (vectorised when the row is
// 16-byte aligned); out-of-range entries are masked into range and reported.
template <typename P>
__device__ __forceinline__ bool stage_order_vec(const P* __restrict__ pp, int n, uint16_t* p, bool aligned) {
  bool bad = false;
  const uint32_t mask = (uint32_t)n - 1;  // n is a power of two
  if (aligned) {
    uint4* p4 = reinterpret_cast<uint4*>(p);
    for (int c = threadIdx.x; c < (n >> 3); c += blockDim.x) {
      uint32_t v[8];
      if constexpr (sizeof(P) == 2) {
        const uint4 w = __ldg(reinterpret_cast<const uint4*>(pp) + c);
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          v[2 * k] = ws[k] & 0xFFFFu;
          v[2 * k + 1] = ws[k] >> 16;
        }
      } else {
        const int4 w0 = __ldg(reinterpret_cast<const int4*>(pp) + 2 * c);
        const int4 w1 = __ldg(reinterpret_cast<const int4*>(pp) + 2 * c + 1);
        const int ws[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = (uint32_t)ws[k];
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        bad |= v[k] > mask;
        v[k] &= mask;
      }
      p4[c] = make_uint4(v[0] | (v[1] << 16), v[2] | (v[3] << 16), v[4] | (v[5] << 16), v[6] | (v[7] << 16));
    }
  } else {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const uint32_t v = (uint32_t)ld_order<P>(pp, i);
      bad |= v > mask;
      p[i] = (uint16_t)(v & mask);
    }
  }
  return bad;
}

// One CTA per order.  pos = p^-1 (one scatter per order); then every thread
// emits 8 consecutive hosts' partners for one round as a 16-byte store:
// part_r[h] = p[pos[h] ^ s] (xor) or p[pos[h] + s] for pos[h] < N/2 (paper).
// Bijection check: p[pos[h]] == h for every host h.
template <typename P, bool kValidate>
__global__ void __launch_bounds__(256) k_rounds_route(RRouteArgs a, const P* __restrict__ perms,
                                                      uint16_t* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = a.n;
  uint16_t* p = reinterpret_cast<uint16_t*>(smem);
  uint16_t* pos = reinterpret_cast<uint16_t*>(smem + al16((size_t)n * 2));
  uint4* pos4 = reinterpret_cast<uint4*>(pos);
  // pos starts (and is reset to) the 0xFFFF sentinel: a host no position
  // names keeps it, which is how a repeated host (the bijection check) shows.
  const uint4 none = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
  for (int k = threadIdx.x; k < (n >> 3); k += blockDim.x) pos4[k] = none;
  const int half = n >> 1;
  const int chunks8 = n >> 3;
  const int cshift = 31 - __clz(chunks8);
  const int rshift = 31 - __clz(a.R);
  const int items = a.slots << cshift;
  const bool aligned = a.aligned != 0;
  const uint32_t jm = (uint32_t)(n - 1) * 0x10001u;
  // uint16 orders, 16-byte aligned, n <= 4096: the next order is loaded into
  // registers during this order's gathers (RW_HD_ROUTE_PF=0 disables it)
  constexpr int kPF = 2;
  const int nc8 = n >> 3;
  const bool use_pf = sizeof(P) == 2 && aligned && a.prefetch && nc8 <= kPF * (int)blockDim.x;
  uint4 pf[kPF];
  auto prefetch = [&](int64_t oo) {
    const uint4* src = reinterpret_cast<const uint4*>(perms + oo * n);
#pragma unroll
    for (int k = 0; k < kPF; ++k) {
      const int c = threadIdx.x + k * blockDim.x;
      if (c < nc8) pf[k] = __ldg(src + c);
    }
  };
  if (use_pf && blockIdx.x < a.count) prefetch(blockIdx.x);
  for (int64_t o = blockIdx.x; o < a.count; o += gridDim.x) {
    __syncthreads();  // the previous order's readers of p / pos are done
    bool bad = false;
    if (use_pf) {
      uint4* p4 = reinterpret_cast<uint4*>(p);
#pragma unroll
      for (int k = 0; k < kPF; ++k) {
        const int c = threadIdx.x + k * blockDim.x;
        if (c < nc8) {
          const uint4 q = pf[k];
          bad |= ((q.x | q.y | q.z | q.w) & ~jm) != 0;
          p4[c] = make_uint4(q.x & jm, q.y & jm, q.z & jm, q.w & jm);
        }
      }
    } else {
      bad = stage_order_vec<P>(perms + o * n, n, p, aligned);
    }
    if ((int)threadIdx.x < a.rounds) {
      if (a.key_bytes == 8)
        static_cast<unsigned long long*>(a.keys)[(size_t)threadIdx.x * a.count + o] = a.zero_key;
      else
        static_cast<unsigned int*>(a.keys)[(size_t)threadIdx.x * a.count + o] = (unsigned int)a.zero_key;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) pos[p[i]] = (uint16_t)i;
    __syncthreads();
    if (use_pf && o + gridDim.x < a.count) prefetch(o + gridDim.x);
    const uint32_t jmask = (uint32_t)(n - 1) * 0x10001u;  // keeps sentinel positions in range
    for (int w = threadIdx.x; w < items; w += blockDim.x) {
      const int r = w >> cshift;  // round, or round pair when a.paired
      const int c = w & (chunks8 - 1);
      const int s = 1 << r;
      uint4 q4 = pos4[c];
      // valid positions are < n (a power of two): any bit outside n-1 is the
      // sentinel of a host no position names, i.e. a repeated host elsewhere
      if (r == 0 && ((q4.x | q4.y | q4.z | q4.w) & ~jmask) != 0) bad = true;
      q4 = make_uint4(q4.x & jmask, q4.y & jmask, q4.z & jmask, q4.w & jmask);
      const uint32_t js[4] = {q4.x, q4.y, q4.z, q4.w};
      uint32_t outw[4];
      if (a.paired) {
        // Round pair (2r, 2r+1), symmetric matrix: the four hosts at positions
        // with bits (2r+1, 2r) = 00, 01, 10, 11 of an aligned group form two
        // pairs per round; 00 and 11 own the round-2r pairs (00,01), (10,11),
        // 01 and 10 own the round-(2r+1) pairs (01,11), (00,10).  Every pair
        // is looked up exactly once (c(a,b) == c(b,a)) and every host holds
        // exactly one lookup; bit 15 tags round 2r+1.  A lone last round
        // (odd round count) keeps both directions (max is unchanged).
        const int r0 = 2 * r;
        const bool lone = r0 + 1 >= a.rounds;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          uint32_t v[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const uint32_t j = e ? (js[k] >> 16) : (js[k] & 0xFFFFu);
            const uint32_t b0 = (j >> r0) & 1u, b1 = (j >> (r0 + 1)) & 1u;
            const uint32_t second = lone ? 0u : (b0 ^ b1);
            v[e] = (uint32_t)p[j ^ ((1u + second) << r0)] | (second << 15);  // one gather
          }
          outw[k] = v[0] | (v[1] << 16);
        }
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t j0 = js[k] & 0xFFFFu, j1 = js[k] >> 16;
          uint32_t v0, v1;
          if (a.xor_pairing) {
            v0 = p[j0 ^ s];
            v1 = p[j1 ^ s];
          } else {
            v0 = (int)j0 < half ? (uint32_t)p[j0 + s] : 0xFFFFu;
            v1 = (int)j1 < half ? (uint32_t)p[j1 + s] : 0xFFFFu;
          }
          outw[k] = v0 | (v1 << 16);
        }
      }
      const int h0 = c << 3;
      const int b = h0 >> rshift;
      const int s0 = h0 & (a.R - 1);
      *reinterpret_cast<uint4*>(out + (((size_t)b * a.slots + r) * a.count + o) * a.R + s0) =
          make_uint4(outw[0], outw[1], outw[2], outw[3]);
    }
    __syncthreads();  // every reader of pos is done: reset it to the sentinel
    for (int k = threadIdx.x; k < (n >> 3); k += blockDim.x) pos4[k] = none;
    if (kValidate && __syncthreads_or(bad) && threadIdx.x == 0) report_bad_order(a.err, n, a.base + o);
  }
}

// ------------------------------------------------------------------ score --
constexpr int kRMaxStages = 4;
// 16 consumer warps + 1 producer warp: a 256-order stage is 1,536 (xor, round
// pairs) or 3,072 (paper) tasks, 3 or 6 per consumer thread.  Measured on B200
// at C5 (u16 xor / paper, evals/s): 1024 threads 2.38e7 / 1.24e7, 800 2.42e7 /
// 1.26e7, 544 2.49e7 / 1.33e7, 416 2.47e7 / 1.33e7, 288 2.39e7 / 1.28e7.
constexpr int kRThreads = 544;

struct RScoreArgs {
  int64_t count;
  int n;
  int rounds;    // partner slots per host (round pairs when kPaired)
  int nrounds;   // reduction rounds (keys rows)
  int nblocks;
  int stages;   // ring depth
  int stage_orders;  // orders per stage (a multiple of 32)
  void* keys;   // [round][order]
};

// kAll: every host is a source (xor pairing), so the route wrote no
// sentinels and every partner is < n (stage_order_vec masks entries into
// range): the per-lookup range test is dropped.
template <typename T, int R, bool kAll, bool kPaired>
__global__ void __launch_bounds__(kRThreads, 1) k_rounds_score(RScoreArgs a, const uint16_t* __restrict__ buf,
                                                               const T* __restrict__ gmat) {
  extern __shared__ __align__(16) unsigned char smem[];
  using K = typename KeyOf<T>::type;
  const int n = a.n, rounds = a.rounds;
  T* blk = reinterpret_cast<T*>(smem);
  uint16_t* ring = reinterpret_cast<uint16_t*>(smem + al16((size_t)R * n * sizeof(T)));
  __shared__ __align__(8) uint64_t full[kRMaxStages], empty[kRMaxStages], mat_bar;
  unsigned mat_phase = 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kConsumers = kRThreads - 32;
  const bool producer = warp == (kRThreads >> 5) - 1;
  const int kRStageOrders = a.stage_orders;
  const size_t stage_elems = (size_t)kRStageOrders * rounds * R;
  if (threadIdx.x == 0)
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers / 32);
    }
  if (threadIdx.x == 0) mbar_init(&mat_bar, 1);
  __syncthreads();
  K* keys = static_cast<K*>(a.keys);
  // Stream-K split: the (block, stage) units are cut into gridDim.x equal
  // contiguous ranges, so every CTA does the same work and reloads the matrix
  // only where its range crosses a row block.
  const int64_t nstage = (a.count + kRStageOrders - 1) / kRStageOrders;
  const int64_t units = nstage * a.nblocks;
  const int64_t u_end = units * (blockIdx.x + 1) / gridDim.x;
  uint32_t g = 0;  // running stage counter of this CTA (same sequence in every role)
  for (int64_t u = units * blockIdx.x / gridDim.x; u < u_end;) {
    const int b = (int)(u / nstage);
    const int64_t st0 = u - (int64_t)b * nstage;
    const int64_t my_stages = min(nstage - st0, u_end - u);
    u += my_stages;
    __syncthreads();  // previous block's consumers are done with blk
    stage_rows(blk, gmat + (size_t)b * R * n, (size_t)R * n * sizeof(T), &mat_bar, &mat_phase);
    if (producer) {
      if (lane == 0) {
        for (int64_t i = 0; i < my_stages; ++i) {
          const uint32_t gi = g + (uint32_t)i;
          const int slot = (int)(gi % a.stages);
          const uint32_t use = gi / a.stages;
          if (use > 0) mbar_wait(&empty[slot], (use - 1) & 1u);
          const int64_t o0 = (st0 + i) * kRStageOrders;
          const int cnt = (int)min((int64_t)kRStageOrders, a.count - o0);
          const unsigned bytes = (unsigned)cnt * R * 2;
          mbar_expect_tx(&full[slot], bytes * rounds);
          uint16_t* dst = ring + slot * stage_elems;
          for (int r = 0; r < rounds; ++r)
            bulk_g2s(dst + (size_t)r * kRStageOrders * R, buf + (((size_t)b * rounds + r) * a.count + o0) * R, bytes,
                      &full[slot]);
        }
      }
    } else {
      for (int64_t i = 0; i < my_stages; ++i) {
        const uint32_t gi = g + (uint32_t)i;
        const int slot = (int)(gi % a.stages);
        mbar_wait(&full[slot], (gi / a.stages) & 1u);
        const int64_t o0 = (st0 + i) * kRStageOrders;
        const int cnt = (int)min((int64_t)kRStageOrders, a.count - o0);
        const uint16_t* sp = ring + slot * stage_elems;
        const int tasks = cnt * rounds;
        const float inv_cnt = 1.0f / (float)cnt;
        for (int t = threadIdx.x; t < tasks; t += kConsumers) {
          // t = r * cnt + k via a float reciprocal and one correction step
          int r = (int)((float)t * inv_cnt);
          int k = t - r * cnt;
          if (k < 0) {
            --r;
            k += cnt;
          } else if (k >= cnt) {
            ++r;
            k -= cnt;
          }
          const uint4* q4 = reinterpret_cast<const uint4*>(sp + ((size_t)r * kRStageOrders + k) * R);
          const K zero = KeyOf<T>::enc(T(0));
          K key = zero, key1 = zero;
#pragma unroll
          for (int c = 0; c < R / 8; ++c) {
            const uint4 q = q4[c];
            const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int h = 0; h < 8; ++h) {
              const uint32_t col = (h & 1) ? (w[h >> 1] >> 16) : (w[h >> 1] & 0xFFFFu);
              if constexpr (kPaired) {
                // bit 15 tags the second round of the pair (partners < 2^15)
                const K v = KeyOf<T>::enc(blk[(c * 8 + h) * n + (col & 0x7FFFu)]);
                if (col & 0x8000u) key1 = v > key1 ? v : key1;
                else key = v > key ? v : key;
              } else if (kAll || col < (uint32_t)n) {
                const K v = KeyOf<T>::enc(blk[(c * 8 + h) * n + col]);
                key = v > key ? v : key;
              }
            }
          }
          const int r0 = kPaired ? 2 * r : r;
          if (key != zero) atomicMax(keys + (size_t)r0 * a.count + o0 + k, key);
          if (kPaired && key1 != zero) atomicMax(keys + (size_t)(r0 + 1) * a.count + o0 + k, key1);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
      }
    }
    g += (uint32_t)my_stages;
  }
}

// ------------------------------------- source-compacted rounds (paper, BCube) --
// Paper pairing (the reference's default, cost_model.cpp:84-85) and BCube
// (cost_model.cpp:118-138) share one shape: in round r the sources are the
// positions j < N/B (B = 2 for paper pairing) and source j meets the B-1
// partners j + k*B^r, k = 1..B-1 (the reference's % n never fires).  The slot
// layout above would store a sentinel for every non-source host in every
// round.  The compact layout keeps, per (row block, order), the first C
// sources of the block's R hosts:
//   msk[block][order]                  u16, the hosts (bits of the block) stored
//   rec[block][order][r][k-1][C]       their partners, round-major, padded to
//                                      whole groups of GR rounds (16-byte multiples)
// A block holds Binomial(R, 1/B) sources; the few beyond C (R=16, paper C=10:
// 0.16 hosts per block) are looked up by the route itself from the global
// matrix and folded into the order's initial round keys, so nothing is dropped.

struct RCompactArgs {
  int64_t count;
  int64_t count_pad;  // multiple of 8: row stride of msk / rec (16-byte aligned stage copies)
  int64_t base;
  int n;
  int rounds;
  int groups;         // ceil(rounds / GR)
  int rec_u16;        // groups * GR * (B-1) * C
  unsigned long long* err;
  unsigned int* keys;  // [round][order]: set to max(zero key, overflow lookups)
  unsigned int zero_key;
  int aligned;
};

// One CTA per order: stage p, scatter pos; phase 1, one thread per row block:
// the block's source mask, its first C sources' positions (shared memory) and
// a list of the over-capacity sources; phase 2, their lookups in the global
// matrix, one (host, round, partner) per thread, then one thread per (block,
// group of GR rounds): the stored sources' partners, 16-byte stores.
template <typename P, typename T, int R, int C, int B, int GR, bool kValidate>
__global__ void __launch_bounds__(256) k_rounds_route_compact(RCompactArgs a, const P* __restrict__ perms,
                                                              const T* __restrict__ gmat,
                                                              uint16_t* __restrict__ rec, uint16_t* __restrict__ msk) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ unsigned int okey[kMaxRounds];
  const int n = a.n;
  const int nblocks = n / R;
  uint16_t* p = reinterpret_cast<uint16_t*>(smem);
  uint16_t* pos = reinterpret_cast<uint16_t*>(smem + al16((size_t)n * 2));
  uint16_t* cpos = reinterpret_cast<uint16_t*>(smem + 2 * al16((size_t)n * 2));  // [block][C]
  uint32_t* ovf = reinterpret_cast<uint32_t*>(smem + 2 * al16((size_t)n * 2) + al16((size_t)nblocks * C * 2));
  __shared__ unsigned int novf;
  uint4* pos4 = reinterpret_cast<uint4*>(pos);
  const uint4 none = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
  for (int k = threadIdx.x; k < (n >> 3); k += blockDim.x) pos4[k] = none;
  constexpr int LB = B == 2 ? 1 : B == 4 ? 2 : 3;  // log2 B
  constexpr int E = (B - 1) * C;                   // entries per round
  const uint32_t nsrc = (uint32_t)n >> LB;
  const uint32_t pmask = (uint32_t)n - 1;
  const uint32_t jmask = pmask * 0x10001u;
  const bool aligned = a.aligned != 0;
  // uint16 orders, 16-byte aligned, n <= 4096: the next order is loaded into
  // registers during this order's gathers (its HBM latency hidden)
  constexpr int kPF = 2;
  const int nc8 = n >> 3;
  const bool use_pf = sizeof(P) == 2 && aligned && nc8 <= kPF * (int)blockDim.x;
  uint4 pf[kPF];
  auto prefetch = [&](int64_t oo) {
    const uint4* src = reinterpret_cast<const uint4*>(perms + oo * n);
#pragma unroll
    for (int k = 0; k < kPF; ++k) {
      const int c = threadIdx.x + k * blockDim.x;
      if (c < nc8) pf[k] = __ldg(src + c);
    }
  };
  if (use_pf && blockIdx.x < a.count) prefetch(blockIdx.x);
  for (int64_t o = blockIdx.x; o < a.count; o += gridDim.x) {
    __syncthreads();
    bool bad = false;
    if (use_pf) {
      uint4* p4 = reinterpret_cast<uint4*>(p);
#pragma unroll
      for (int k = 0; k < kPF; ++k) {
        const int c = threadIdx.x + k * blockDim.x;
        if (c < nc8) {
          const uint4 q = pf[k];
          bad |= ((q.x | q.y | q.z | q.w) & ~jmask) != 0;
          p4[c] = make_uint4(q.x & jmask, q.y & jmask, q.z & jmask, q.w & jmask);
        }
      }
    } else {
      bad = stage_order_vec<P>(perms + o * n, n, p, aligned);
    }
    if ((int)threadIdx.x < a.rounds) okey[threadIdx.x] = a.zero_key;
    if (threadIdx.x == 0) novf = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) pos[p[i]] = (uint16_t)i;
    __syncthreads();
    for (int b = threadIdx.x; b < nblocks; b += blockDim.x) {
      // the block's sources (positions < N/B) in host order: the first C go
      // to cpos (independent stores, no dependent re-reads of pos), the rest
      // to the over-capacity list; a host no position names keeps the
      // sentinel (the bijection check)
      uint32_t mc = 0;
      int i = 0;
#pragma unroll
      for (int c = 0; c < R / 8; ++c) {
        const uint4 q = pos4[b * (R / 8) + c];
        const uint32_t qs[4] = {q.x, q.y, q.z, q.w};
        if ((q.x | q.y | q.z | q.w) & ~jmask) bad = true;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t j = (qs[k >> 1] >> ((k & 1) * 16)) & pmask;
          const int e = c * 8 + k;
          if (j < nsrc) {
            if (i < C) {
              cpos[b * C + i] = (uint16_t)j;
              mc |= 1u << e;
            } else {
              ovf[atomicAdd(&novf, 1u)] = ((uint32_t)(b * R + e) << 16) | j;
            }
            ++i;
          }
        }
      }
      for (; i < C; ++i) cpos[b * C + i] = 0;
      msk[(size_t)b * a.count_pad + o] = (uint16_t)mc;
    }
    __syncthreads();
    if (use_pf && o + gridDim.x < a.count) prefetch(o + gridDim.x);
    // over-capacity lookups, one (host, round, partner) per thread: the L2
    // latencies overlap instead of serialising on the threads that found them
    const int per_host = a.rounds * (B - 1);
    const int oitems = (int)novf * per_host;
    for (int w = threadIdx.x; w < oitems; w += blockDim.x) {
      const int h = w / per_host;
      const int rk = w - h * per_host;
      const int r = rk / (B - 1);
      const uint32_t k = (uint32_t)(rk - r * (B - 1)) + 1u;
      const uint32_t e = ovf[h];
      const T v = gmat[(size_t)(e >> 16) * n + p[(e & 0xFFFFu) + (k << (r * LB))]];
      atomicMax(&okey[r], KeyOf<T>::enc(v));
    }
    // one thread per (block, group of GR rounds): C positions, GR*E gathers,
    // GR*E/8 16-byte stores.  Entries past the block's count gather from
    // position 0 and padding rounds use offset 0 (always in range; the score
    // never reads them).
    const int gitems = nblocks * a.groups;
    for (int w = threadIdx.x; w < gitems; w += blockDim.x) {
      const int b = w / a.groups;
      const int g = w - b * a.groups;
      const uint32_t* c2 = reinterpret_cast<const uint32_t*>(cpos + b * C);
      uint32_t jc2[C / 2];
#pragma unroll
      for (int k = 0; k < C / 2; ++k) jc2[k] = c2[k];
      uint32_t outw[GR * E / 2];
#pragma unroll
      for (int k = 0; k < GR * E / 2; ++k) outw[k] = 0;
#pragma unroll
      for (int rr = 0; rr < GR; ++rr) {
        const int r = g * GR + rr;
#pragma unroll
        for (int kk = 1; kk < B; ++kk) {
          const uint32_t off = r < a.rounds ? (uint32_t)kk << (r * LB) : 0u;
#pragma unroll
          for (int i = 0; i < C; ++i) {
            const uint32_t j = (jc2[i >> 1] >> ((i & 1) * 16)) & 0xFFFFu;
            const int idx = rr * E + (kk - 1) * C + i;
            outw[idx >> 1] |= (uint32_t)p[j + off] << ((idx & 1) * 16);
          }
        }
      }
      uint4* dst = reinterpret_cast<uint4*>(rec + ((size_t)b * a.count_pad + o) * a.rec_u16) + g * (GR * E / 8);
#pragma unroll
      for (int k = 0; k < GR * E / 8; ++k)
        dst[k] = make_uint4(outw[4 * k], outw[4 * k + 1], outw[4 * k + 2], outw[4 * k + 3]);
    }
    __syncthreads();  // every reader of pos and okey is done
    for (int k = threadIdx.x; k < (n >> 3); k += blockDim.x) pos4[k] = none;
    if ((int)threadIdx.x < a.rounds) a.keys[(size_t)threadIdx.x * a.count + o] = okey[threadIdx.x];
    if (kValidate && __syncthreads_or(bad) && threadIdx.x == 0) report_bad_order(a.err, n, a.base + o);
  }
}

// Consumer warps + 1 producer warp: with 3 round groups (paper pairing at
// C5) a stage of 192 (R=16) or 288 (R=8) orders is one task per consumer thread.
template <int R>
struct CompactThreads {
  static constexpr int value = R == 16 ? 608 : 896;
};

struct RCompactScoreArgs {
  int64_t count;
  int64_t count_pad;
  int n;
  int rounds;
  int groups;
  int rec_u16;
  int nblocks;
  int stages;
  int stage_orders;
  unsigned int* keys;
};

template <typename T, int R, int C, int B, int GR, int kCThreads = CompactThreads<R>::value>
__global__ void __launch_bounds__(kCThreads, 1) k_rounds_score_compact(RCompactScoreArgs a,
                                                                       const uint16_t* __restrict__ rec,
                                                                       const uint16_t* __restrict__ msk,
                                                                       const T* __restrict__ gmat) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int E = (B - 1) * C;  // entries per round
  const int n = a.n;
  T* blk = reinterpret_cast<T*>(smem);
  unsigned char* ring = smem + al16((size_t)R * n * sizeof(T));
  __shared__ __align__(8) uint64_t full[kRMaxStages], empty[kRMaxStages], mat_bar;
  unsigned mat_phase = 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kConsumers = kCThreads - 32;
  const bool producer = warp == (kCThreads >> 5) - 1;
  const int so = a.stage_orders;
  const size_t rec_bytes = (size_t)a.rec_u16 * 2;
  const size_t stage_bytes = (size_t)so * rec_bytes + (size_t)so * 2;
  if (threadIdx.x == 0) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers / 32);
    }
    mbar_init(&mat_bar, 1);
  }
  __syncthreads();
  const int64_t nstage = (a.count + so - 1) / so;
  const int64_t units = nstage * a.nblocks;
  const int64_t u_end = units * (blockIdx.x + 1) / gridDim.x;
  uint32_t g = 0;
  for (int64_t u = units * blockIdx.x / gridDim.x; u < u_end;) {
    const int b = (int)(u / nstage);
    const int64_t st0 = u - (int64_t)b * nstage;
    const int64_t my_stages = min(nstage - st0, u_end - u);
    u += my_stages;
    __syncthreads();
    stage_rows(blk, gmat + (size_t)b * R * n, (size_t)R * n * sizeof(T), &mat_bar, &mat_phase);
    if (producer) {
      if (lane == 0) {
        for (int64_t i = 0; i < my_stages; ++i) {
          const uint32_t gi = g + (uint32_t)i;
          const int slot = (int)(gi % a.stages);
          const uint32_t use = gi / a.stages;
          if (use > 0) mbar_wait(&empty[slot], (use - 1) & 1u);
          const int64_t o0 = (st0 + i) * so;
          const int cnt = (int)min((int64_t)so, a.count - o0);
          const unsigned rb = (unsigned)(cnt * rec_bytes);
          const unsigned mb = (unsigned)(((cnt + 7) & ~7) * 2);  // within count_pad
          mbar_expect_tx(&full[slot], rb + mb);
          unsigned char* dst = ring + slot * stage_bytes;
          bulk_g2s(dst, rec + ((size_t)b * a.count_pad + o0) * a.rec_u16, rb, &full[slot]);
          bulk_g2s(dst + (size_t)so * rec_bytes, msk + (size_t)b * a.count_pad + o0, mb, &full[slot]);
        }
      }
    } else {
      for (int64_t i = 0; i < my_stages; ++i) {
        const uint32_t gi = g + (uint32_t)i;
        const int slot = (int)(gi % a.stages);
        mbar_wait(&full[slot], (gi / a.stages) & 1u);
        const int64_t o0 = (st0 + i) * so;
        const int cnt = (int)min((int64_t)so, a.count - o0);
        const unsigned char* sp = ring + slot * stage_bytes;
        const uint16_t* sm = reinterpret_cast<const uint16_t*>(sp + (size_t)so * rec_bytes);
        const int tasks = cnt * a.groups;
        const float inv_cnt = 1.0f / (float)cnt;
        for (int t = threadIdx.x; t < tasks; t += kConsumers) {
          int gr = (int)((float)t * inv_cnt);
          int k = t - gr * cnt;
          if (k < 0) {
            --gr;
            k += cnt;
          } else if (k >= cnt) {
            ++gr;
            k -= cnt;
          }
          uint32_t m = sm[k];
          const int cntm = __popc(m);
          int hoff[C];
#pragma unroll
          for (int i = 0; i < C; ++i) {
            const int e = m ? __ffs(m) - 1 : 0;
            m &= m - 1;
            hoff[i] = e * n;
          }
          const uint4* q4 = reinterpret_cast<const uint4*>(sp + (size_t)k * rec_bytes) + gr * (GR * E / 8);
          uint32_t w[GR * E / 2];
#pragma unroll
          for (int c = 0; c < GR * E / 8; ++c) {
            const uint4 q = q4[c];
            w[4 * c] = q.x;
            w[4 * c + 1] = q.y;
            w[4 * c + 2] = q.z;
            w[4 * c + 3] = q.w;
          }
          using K = typename KeyOf<T>::type;
          const K zero = KeyOf<T>::enc(T(0));
#pragma unroll
          for (int rr = 0; rr < GR; ++rr) {
            const int r = gr * GR + rr;
            K key = zero;
#pragma unroll
            for (int q = 0; q < E; ++q) {
              const int i = q % C;
              const int idx = rr * E + q;
              const uint32_t col = (w[idx >> 1] >> ((idx & 1) * 16)) & 0xFFFFu;
              if (i < cntm) {
                const K v = KeyOf<T>::enc(blk[hoff[i] + col]);
                key = v > key ? v : key;
              }
            }
            if (r < a.rounds && key != zero) atomicMax(a.keys + (size_t)r * a.count + o0 + k, key);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
      }
    }
    g += (uint32_t)my_stages;
  }
}

// --------------------------------------------------------------- finalize --
struct RFinalArgs {
  int64_t count;
  int rounds;
  int mode;
  double scale;
  double bytes[kMaxRounds];
};

template <typename T>
__global__ void k_rounds_finalize(RFinalArgs a, const void* __restrict__ keys_v, double* __restrict__ costs) {
  using K = typename KeyOf<T>::type;
  const K* keys = static_cast<const K*>(keys_v);
  const int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= a.count) return;
  double total = 0.0;
  for (int r = 0; r < a.rounds; ++r) {
    double v = to_double(KeyOf<T>::dec(keys[(size_t)r * a.count + o]), a.scale);
    if (a.mode == RW_LATENCY_TIMES_SIZE) v = __dmul_rn(v, a.bytes[r]);
    total = __dadd_rn(total, v);
  }
  costs[o] = total;
}

// Rank finalize: the round's maximum rank decodes to its FP64 value through
// the sorted distinct values, then the reference's fl(max * bytes_r) sum.
__global__ void k_rounds_finalize_ranks(RFinalArgs a, const unsigned int* __restrict__ keys,
                                        const double* __restrict__ vals, double* __restrict__ costs) {
  const int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= a.count) return;
  double total = 0.0;
  for (int r = 0; r < a.rounds; ++r) {
    double v = vals[keys[(size_t)r * a.count + o]];
    if (a.mode == RW_LATENCY_TIMES_SIZE) v = __dmul_rn(v, a.bytes[r]);
    total = __dadd_rn(total, v);
  }
  costs[o] = total;
}

// ---------------------------------------------------------- rank transform --
// v -> the value whose rank represents it: NaN never wins the reference's
// running max (std::max from 0, cost_model.cpp:83) and -0.0 == 0.0, so both
// map to +0.0, which is always in the table.
__device__ __forceinline__ double rank_value(double v) { return (v != v || v == 0.0) ? 0.0 : v; }

__global__ void k_rank_prepare(const double* __restrict__ m, int64_t nn, double* __restrict__ out) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k <= nn; k += (int64_t)gridDim.x * blockDim.x)
    out[k] = k < nn ? rank_value(m[k]) : 0.0;
}

__global__ void k_rank_assign(const double* __restrict__ m, int64_t nn, const double* __restrict__ uniq,
                              const int* __restrict__ count, uint32_t* __restrict__ rank) {
  const int cnt = *count;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nn; k += (int64_t)gridDim.x * blockDim.x) {
    const double v = rank_value(m[k]);
    int lo = 0, hi = cnt - 1;  // v is in the table: exact lower_bound
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (uniq[mid] < v) lo = mid + 1;
      else hi = mid;
    }
    rank[k] = (uint32_t)lo;
  }
}

// Builds Problem::d_rank / d_rank_vals (FP64 storage): sort + unique of the
// sanitised entries (cub), then one binary search per entry.  Exact: a
// round's maximum rank is the rank of its maximum value.
void ensure_ranks(Problem& p, cudaStream_t st) {
  std::lock_guard<std::mutex> lock(p.mu);
  if (p.d_rank) return;
  const int64_t nn = (int64_t)p.n * p.n;
  double *d_in = nullptr, *d_sorted = nullptr, *d_uniq = nullptr;
  int* d_cnt = nullptr;
  void* d_tmp = nullptr;
  size_t tmp_sort = 0, tmp_uniq = 0;
  RW_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp_sort, d_in, d_sorted, (int)(nn + 1)));
  RW_CUDA(cub::DeviceSelect::Unique(nullptr, tmp_uniq, d_sorted, d_uniq, d_cnt, (int)(nn + 1)));
  RW_CUDA(cudaMalloc(&d_in, (size_t)(nn + 1) * 8));
  RW_CUDA(cudaMalloc(&d_sorted, (size_t)(nn + 1) * 8));
  RW_CUDA(cudaMalloc(&d_uniq, (size_t)(nn + 1) * 8));
  RW_CUDA(cudaMalloc(&d_cnt, sizeof(int)));
  RW_CUDA(cudaMalloc(&d_tmp, std::max(tmp_sort, tmp_uniq)));
  uint32_t* d_rank = nullptr;
  RW_CUDA(cudaMalloc(&d_rank, (size_t)nn * 4));
  const double* m = static_cast<const double*>(p.d_mat);
  k_rank_prepare<<<148 * 8, 256, 0, st>>>(m, nn, d_in);
  RW_CUDA(cub::DeviceRadixSort::SortKeys(d_tmp, tmp_sort, d_in, d_sorted, (int)(nn + 1), 0, 64, st));
  RW_CUDA(cub::DeviceSelect::Unique(d_tmp, tmp_uniq, d_sorted, d_uniq, d_cnt, (int)(nn + 1), st));
  k_rank_assign<<<148 * 8, 256, 0, st>>>(m, nn, d_uniq, d_cnt, d_rank);
  RW_CUDA(cudaGetLastError());
  int cnt = 0;
  RW_CUDA(cudaMemcpyAsync(&cnt, d_cnt, sizeof(int), cudaMemcpyDeviceToHost, st));
  RW_CUDA(cudaStreamSynchronize(st));
  std::vector<double> uniq((size_t)cnt);
  RW_CUDA(cudaMemcpy(uniq.data(), d_uniq, (size_t)cnt * 8, cudaMemcpyDeviceToHost));
  double* d_vals = nullptr;
  RW_CUDA(cudaMalloc(&d_vals, (size_t)cnt * 8));
  RW_CUDA(cudaMemcpy(d_vals, uniq.data(), (size_t)cnt * 8, cudaMemcpyHostToDevice));
  p.zero_rank = (uint32_t)(std::lower_bound(uniq.begin(), uniq.end(), 0.0) - uniq.begin());
  cudaFree(d_in);
  cudaFree(d_sorted);
  cudaFree(d_uniq);
  cudaFree(d_cnt);
  cudaFree(d_tmp);
  p.d_rank_vals = d_vals;
  p.d_rank = d_rank;
}

template <typename T, int R>
void launch_score(const RScoreArgs& sa, int grid, size_t smem, const uint16_t* buf, const void* mat, cudaStream_t st,
                  bool all, bool paired) {
  auto k = paired ? k_rounds_score<T, R, true, true>
                  : (all ? k_rounds_score<T, R, true, false> : k_rounds_score<T, R, false, false>);
  RW_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k<<<grid, kRThreads, smem, st>>>(sa, buf, static_cast<const T*>(mat));
}

template <typename T>
void launch_score_r(int R, const RScoreArgs& sa, int grid, size_t smem, const uint16_t* buf, const void* mat,
                    cudaStream_t st, bool all, bool paired) {
  if (R == 32) launch_score<T, 32>(sa, grid, smem, buf, mat, st, all, paired);
  else if (R == 16) launch_score<T, 16>(sa, grid, smem, buf, mat, st, all, paired);
  else launch_score<T, 8>(sa, grid, smem, buf, mat, st, all, paired);
}

template <typename T, int R, int C, int B, int GR>
void launch_compact_kernels(const RCompactArgs& ra, const RCompactScoreArgs& sa, bool validate, int perm_bytes,
                            const char* perms, const T* mat, uint16_t* rec, uint16_t* msk, int rgrid, size_t route_smem,
                            int sgrid, size_t score_smem, cudaStream_t st) {
  auto route = validate ? (perm_bytes == 2 ? (void*)k_rounds_route_compact<uint16_t, T, R, C, B, GR, true>
                                           : (void*)k_rounds_route_compact<int32_t, T, R, C, B, GR, true>)
                        : (perm_bytes == 2 ? (void*)k_rounds_route_compact<uint16_t, T, R, C, B, GR, false>
                                           : (void*)k_rounds_route_compact<int32_t, T, R, C, B, GR, false>);
  RW_CUDA(cudaFuncSetAttribute(route, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)route_smem));
  RW_CUDA(cudaFuncSetAttribute(route, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  RCompactArgs rac = ra;
  void* rargs[] = {&rac, (void*)&perms, (void*)&mat, (void*)&rec, (void*)&msk};
  RW_CUDA(cudaLaunchKernel(route, dim3(rgrid), dim3(256), rargs, route_smem, st));
  auto score = k_rounds_score_compact<T, R, C, B, GR>;
  RW_CUDA(cudaFuncSetAttribute(score, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)score_smem));
  score<<<sgrid, CompactThreads<R>::value, score_smem, st>>>(sa, rec, msk, mat);
  RW_CUDA(cudaGetLastError());
}

// Record shape per (R, B): capacity C of a block's Binomial(R, 1/B) sources
// and GR rounds per score task, with GR*(B-1)*C a multiple of 8 (16 bytes).
struct CompactShape {
  int C, GR;
};
inline CompactShape compact_shape(int R, int B) {
  if (R == 16) return B == 2 ? CompactShape{10, 4} : B == 4 ? CompactShape{8, 1} : CompactShape{4, 2};
  return B == 2 ? CompactShape{6, 4} : B == 4 ? CompactShape{4, 2} : CompactShape{2, 4};
}

template <typename T>
void launch_compact_r(int R, int B, const RCompactArgs& ra, const RCompactScoreArgs& sa, bool validate,
                      int perm_bytes, const char* perms, const void* mat, uint16_t* rec, uint16_t* msk, int rgrid,
                      size_t route_smem, int sgrid, size_t score_smem, cudaStream_t st) {
  const T* m = static_cast<const T*>(mat);
#define RW_COMPACT(RR, BB, CC, GG)                                                                                    \
  if (R == RR && B == BB)                                                                                           \
    return launch_compact_kernels<T, RR, CC, BB, GG>(ra, sa, validate, perm_bytes, perms, m, rec, msk, rgrid,        \
                                                     route_smem, sgrid, score_smem, st);
  RW_COMPACT(16, 2, 10, 4)
  RW_COMPACT(16, 4, 8, 1)
  RW_COMPACT(16, 8, 4, 2)
  RW_COMPACT(8, 2, 6, 4)
  RW_COMPACT(8, 4, 4, 2)
  RW_COMPACT(8, 8, 2, 4)
#undef RW_COMPACT
  fail_internal("source-compacted transpose: no record shape for this row block / base");
}

// Paper pairing (B = 2) and BCube (B = 4, 8) through the source-compacted
// layout (k_rounds_route_compact / k_rounds_score_compact); 4-byte keys only
// (u16, FP32, FP64 ranks).
bool launch_paper_compact(const Problem& p, const EvalPlan& plan, const void* d_perms, int perm_bytes, int64_t batch,
                          double* d_costs, bool validate, int* err_slot, cudaStream_t st, int slot, int R, int B,
                          bool ranks, int sms, size_t budget) {
  const int n = plan.n;
  const int rounds = plan.rounds;
  const CompactShape shape = compact_shape(R, B);
  const int C = shape.C;
  const int groups = (rounds + shape.GR - 1) / shape.GR;
  const int rec_u16 = groups * shape.GR * (B - 1) * C;
  const size_t esz = ranks ? 4 : p.elem_bytes();
  const int nblocks = n / R;
  const size_t mat = al16((size_t)R * n * esz);
  const size_t per_order = (size_t)rec_u16 * 2 + 2;
  int so = (int)std::min<size_t>(512, (budget - mat) / (2 * per_order));
  // whole tasks per consumer thread where the group count allows it
  const int quantum = (groups == 3) ? 96 : 32;
  so = so / quantum * quantum;
  if (so < 32) return false;
  const int stages = 2;
  const size_t score_smem = mat + (size_t)stages * so * per_order;
  const size_t route_smem = 2 * al16((size_t)n * 2) + al16((size_t)nblocks * C * 2) + (size_t)nblocks * (R - C) * 4;
  const int64_t per_order_bytes = (int64_t)nblocks * (int64_t)per_order;
  static const int64_t buf_override = [] {
    const char* e = std::getenv("RW_TRANSPOSE_BUF_MB");
    return e ? std::max(8L, std::atol(e)) << 20 : 0L;
  }();
  const int64_t buf_bytes =
      buf_override ? buf_override : std::min<int64_t>(384ll << 20, std::max<int64_t>(48ll << 20, per_order_bytes * 16384));
  const int64_t chunk = std::max<int64_t>(so, buf_bytes / per_order_bytes) & ~int64_t(7);
  const int64_t kmax = std::min(batch, chunk);
  const int64_t kpad = (kmax + 7) & ~int64_t(7);
  ThreadCtx& c = thread_ctx(p.device);
  const size_t rec_bytes_total = (size_t)nblocks * kpad * rec_u16 * 2;
  uint16_t* rec = static_cast<uint16_t*>(c.scratch(slot, rec_bytes_total + (size_t)nblocks * kpad * 2 + 64));
  uint16_t* msk = rec + rec_bytes_total / 2;
  unsigned int* keys = static_cast<unsigned int*>(c.scratch(slot + 1, (size_t)rounds * kmax * 4));
  unsigned int zero_key = 0;
  if (p.storage == RW_STORAGE_F32) zero_key = 0x80000000u;
  if (ranks) zero_key = p.zero_rank;
  RFinalArgs fa{};
  fa.rounds = rounds;
  fa.mode = plan.mode;
  fa.scale = p.scale;
  for (int r = 0; r < rounds; ++r) fa.bytes[r] = plan.round_bytes[r];
  for (int64_t off = 0; off < batch; off += kmax) {
    const int64_t cnt_o = std::min(kmax, batch - off);
    const int64_t cpad = (cnt_o + 7) & ~int64_t(7);
    RCompactArgs ra{cnt_o, cpad, off, n, rounds, groups, rec_u16, reinterpret_cast<unsigned long long*>(err_slot),
                    keys, zero_key, 0};
    const char* perms = static_cast<const char*>(d_perms) + (size_t)off * n * perm_bytes;
    ra.aligned = (reinterpret_cast<uintptr_t>(perms) & 15) == 0 ? 1 : 0;
    const int rgrid = (int)std::min<int64_t>(cnt_o, (int64_t)sms * 8);
    RCompactScoreArgs sa{cnt_o, cpad, n, rounds, groups, rec_u16, nblocks, stages, so, keys};
    const int sgrid = (int)std::min<int64_t>(sms, nblocks * ((cnt_o + so - 1) / so));
    switch (p.storage) {
      case RW_STORAGE_U16:
        launch_compact_r<uint16_t>(R, B, ra, sa, validate, perm_bytes, perms, p.d_mat, rec, msk, rgrid, route_smem, sgrid,
                                   score_smem, st);
        break;
      case RW_STORAGE_F32:
        launch_compact_r<float>(R, B, ra, sa, validate, perm_bytes, perms, p.d_mat, rec, msk, rgrid, route_smem, sgrid,
                                score_smem, st);
        break;
      default:
        launch_compact_r<uint32_t>(R, B, ra, sa, validate, perm_bytes, perms, p.d_rank, rec, msk, rgrid, route_smem,
                                   sgrid, score_smem, st);
        break;
    }
    fa.count = cnt_o;
    const int fgrid = (int)((cnt_o + 127) / 128);
    switch (p.storage) {
      case RW_STORAGE_U16: k_rounds_finalize<uint16_t><<<fgrid, 128, 0, st>>>(fa, keys, d_costs + off); break;
      case RW_STORAGE_F32: k_rounds_finalize<float><<<fgrid, 128, 0, st>>>(fa, keys, d_costs + off); break;
      default:
        k_rounds_finalize_ranks<<<fgrid, 128, 0, st>>>(fa, keys, p.d_rank_vals, d_costs + off);
        break;
    }
    RW_CUDA(cudaGetLastError());
  }
  return true;
}

}  // namespace

bool launch_rounds_transpose(const Problem& p, const EvalPlan& plan, const void* d_perms, int perm_bytes, int64_t batch,
                             double* d_costs, bool validate, int* err_slot, cudaStream_t st, int slot) {
  const int n = plan.n;
  // BCube (B = 2, 4, 8) takes the source-compacted layout only
  const bool bcube = plan.model == kBCube;
  if ((plan.model != kHalvingDoubling && !bcube) || n < 512 || n > 16384 || (n & (n - 1)) != 0 || batch <= 0)
    return false;
  if (bcube && plan.bcube_b != 2 && plan.bcube_b != 4 && plan.bcube_b != 8) return false;
  const int rounds = plan.rounds;
  if (rounds < 1 || rounds > 14) return false;
  // Symmetric matrix + xor pairing: one partner slot per host per round pair
  // (half the lookups and half the exchange buffer, see k_rounds_route).
  const bool paired = !bcube && plan.pairing == RW_PAIRING_XOR && p.symmetric && rounds >= 2;
  const int slots = paired ? (rounds + 1) / 2 : rounds;
  int sms = 148, optin = 227 * 1024;
  RW_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p.device));
  RW_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, p.device));
  const size_t budget = (size_t)std::min(optin, 227 * 1024) - 1024;
  // FP64 rows do not fit a row block of 8 at N=4096 (256 KB): max-based
  // scoring runs on the u32 ranks of the entries instead (exact, see
  // ensure_ranks), which halves the bytes per lookup.
  const bool ranks = p.storage == RW_STORAGE_F64 && n >= 2048;
  if (ranks) ensure_ranks(const_cast<Problem&>(p), st);
  const size_t esz = ranks ? 4 : p.elem_bytes();
  // Largest row block that leaves room for two stages of >= 64 orders; the
  // rest of shared memory becomes two stages of up to 512 orders (larger bulk
  // copies and fewer hand-offs, as measured for the ring score; 256 -> 512
  // measured +4% FP32 / +6% FP64 ranks at C5 xor, where the 8-row blocks leave
  // room for it, and neutral for u16).
  int R = 0, stages = 2, kRStageOrders = 0;
  for (int cand : {32, 16, 8}) {
    const size_t mat = al16((size_t)cand * n * esz);
    const size_t per_order = (size_t)slots * cand * 2;
    if (mat + 2 * 64 * per_order <= budget) {
      R = cand;
      kRStageOrders = (int)std::min<size_t>(512, (budget - mat) / (2 * per_order)) & ~31;
      break;
    }
  }
  if (!R) return false;
  const int nblocks = n / R;
  static const bool compact_env = [] {
    const char* e = std::getenv("RW_HD_COMPACT");
    return !(e && e[0] == '0');
  }();
  // (a 32-row block takes the 16-row compact layout: its route has 64 blocks
  // per order to spread over the CTA instead of 32)
  if ((bcube || (compact_env && plan.pairing == RW_PAIRING_PAPER)) && esz <= 4 && (R == 32 || R == 16 || R == 8))
    return launch_paper_compact(p, plan, d_perms, perm_bytes, batch, d_costs, validate, err_slot, st, slot,
                                R == 32 ? 16 : R, bcube ? plan.bcube_b : 2, ranks, sms, budget);
  if (bcube) return false;  // FP64 matrices below N=2048: the gather kernels
  const size_t score_smem = al16((size_t)R * n * esz) + (size_t)stages * kRStageOrders * slots * R * 2;
  const size_t route_smem = 2 * al16((size_t)n * 2);

  const int64_t per_order_bytes = (int64_t)2 * slots * n;
  // Partner-buffer size: every score CTA restages ~2.5 row blocks per chunk,
  // so chunks of >= 4096 orders keep that below a quarter of the partner
  // traffic (measured on B200: 48 MB -> 7.8e6, 384 MB -> 1.14e7 evals/s at
  // N=4096).  The buffer then streams through HBM; RW_TRANSPOSE_BUF_MB overrides.
  static const int64_t buf_override = [] {
    const char* e = std::getenv("RW_TRANSPOSE_BUF_MB");
    return e ? std::max(8L, std::atol(e)) << 20 : 0L;
  }();
  const int64_t buf_bytes =
      buf_override ? buf_override : std::min<int64_t>(384ll << 20, std::max<int64_t>(48ll << 20, per_order_bytes * 16384));
  const int64_t chunk = std::max<int64_t>(kRStageOrders, buf_bytes / per_order_bytes);
  const int64_t kmax = std::min(batch, chunk);
  ThreadCtx& c = thread_ctx(p.device);
  uint16_t* buf = static_cast<uint16_t*>(c.scratch(slot, (size_t)kmax * per_order_bytes));
  const int key_bytes = esz == 8 ? 8 : 4;
  void* keys = c.scratch(slot + 1, (size_t)rounds * kmax * key_bytes);
  unsigned long long zero_key = 0;
  if (p.storage == RW_STORAGE_F32) zero_key = 0x80000000ull;
  if (p.storage == RW_STORAGE_F64) zero_key = ranks ? p.zero_rank : 0x8000000000000000ull;

  auto route = validate ? (perm_bytes == 2 ? (void*)k_rounds_route<uint16_t, true> : (void*)k_rounds_route<int32_t, true>)
                        : (perm_bytes == 2 ? (void*)k_rounds_route<uint16_t, false> : (void*)k_rounds_route<int32_t, false>);
  RW_CUDA(cudaFuncSetAttribute(route, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)route_smem));
  RFinalArgs fa{};
  fa.rounds = rounds;
  fa.mode = plan.mode;
  fa.scale = p.scale;
  for (int r = 0; r < rounds; ++r) fa.bytes[r] = plan.round_bytes[r];
  for (int64_t off = 0; off < batch; off += kmax) {
    const int64_t cnt_o = std::min(kmax, batch - off);
    static const int route_pf = [] {
      const char* e = std::getenv("RW_HD_ROUTE_PF");
      return (e && e[0] == '0') ? 0 : 1;
    }();
    RRouteArgs ra{cnt_o, off, n, rounds, plan.pairing == RW_PAIRING_XOR ? 1 : 0, R,
                  reinterpret_cast<unsigned long long*>(err_slot), keys, key_bytes, zero_key, 0, slots,
                  paired ? 1 : 0, route_pf};
    const int rgrid = (int)std::min<int64_t>(cnt_o, (int64_t)sms * 8);
    const char* perms = static_cast<const char*>(d_perms) + (size_t)off * n * perm_bytes;
    ra.aligned = (reinterpret_cast<uintptr_t>(perms) & 15) == 0 ? 1 : 0;
    void* args[] = {&ra, (void*)&perms, (void*)&buf};
    RW_CUDA(cudaLaunchKernel(route, dim3(rgrid), dim3(256), args, route_smem, st));
    RScoreArgs sa{cnt_o, n, slots, rounds, nblocks, stages, kRStageOrders, keys};
    const bool xor_all = plan.pairing == RW_PAIRING_XOR;
    const int sgrid = (int)std::min<int64_t>(sms, nblocks * ((cnt_o + kRStageOrders - 1) / kRStageOrders));
    switch (p.storage) {
      case RW_STORAGE_U16: launch_score_r<uint16_t>(R, sa, sgrid, score_smem, buf, p.d_mat, st, xor_all, paired); break;
      case RW_STORAGE_F32: launch_score_r<float>(R, sa, sgrid, score_smem, buf, p.d_mat, st, xor_all, paired); break;
      default:
        if (ranks) launch_score_r<uint32_t>(R, sa, sgrid, score_smem, buf, p.d_rank, st, xor_all, paired);
        else launch_score_r<double>(R, sa, sgrid, score_smem, buf, p.d_mat, st, xor_all, paired);
        break;
    }
    RW_CUDA(cudaGetLastError());
    fa.count = cnt_o;
    const int fgrid = (int)((cnt_o + 127) / 128);
    switch (p.storage) {
      case RW_STORAGE_U16: k_rounds_finalize<uint16_t><<<fgrid, 128, 0, st>>>(fa, keys, d_costs + off); break;
      case RW_STORAGE_F32: k_rounds_finalize<float><<<fgrid, 128, 0, st>>>(fa, keys, d_costs + off); break;
      default:
        if (ranks)
          k_rounds_finalize_ranks<<<fgrid, 128, 0, st>>>(fa, static_cast<const unsigned int*>(keys), p.d_rank_vals,
                                                         d_costs + off);
        else k_rounds_finalize<double><<<fgrid, 128, 0, st>>>(fa, keys, d_costs + off);
        break;
    }
    RW_CUDA(cudaGetLastError());
  }
  return true;
}

}  // namespace rwb
