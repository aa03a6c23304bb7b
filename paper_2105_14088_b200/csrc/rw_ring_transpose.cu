// rw_ring_transpose.cu -- ring scoring for matrices that do not fit one CTA's
// shared memory (N=1024 fixed point is 2 MiB, N=4096 is 32 MiB), without
// random L2 gathers.
//
// The L2-gather kernel (k_ring / k_ring_vec) issues one random 2-byte load per
// hop; each costs a full L1TEX wavefront (32 lanes hit 32 different 128-byte
// lines), and ncu shows it at ~96% of L1TEX throughput -- one sector per cycle
// per SM.  This path changes the access pattern instead of the kernel:
//
//   pass 1 (k_ring_route)  one warp per order scatters hop (cur, prev) into a
//       shared-memory "predecessor by host" array, pred[cur] = prev, then
//       writes it out in 16-byte chunks grouped by row block of the matrix:
//       predbuf[block][order][row-in-block].  Every global access is
//       coalesced.  The same pass validates the order: a host that is never
//       `cur` keeps the 0xFFFF sentinel (duplicates imply a missing host).
//   pass 2 (k_ring_score)  a CTA holds a row block of the matrix in shared
//       memory (one TMA bulk copy); a producer warp streams the block's
//       predecessor slices through a two-stage TMA bulk-copy ring (full /
//       empty mbarriers) and 24 consumer warps do the shared-memory lookups
//       blk[row][pred[row]].  (row block, stage) units are split stream-K
//       over every SM.  u16 codes: per-(order, block) integer partials are
//       added atomically into the cost array (exact, order-independent) and
//       scaled once by k_ring_finalize; FP32/FP64 matrices: partials go to
//       part[block][order] and k_ring_combine sums them in block order.
//   Chunks of up to 512 MB of predecessor buffer: the per-chunk fixed cost
//   (launches, row-block staging, ring fill) outweighs L2 residency.
//
// Reference semantics: ring_cost (proj/src/cost_model.cpp:59-69), hop i =
// rtt[perm[i]][perm[i-1]]; every host is `cur` of exactly one hop, so
// sum over hosts h of rtt[h][pred(h)] is the same multiset of hops.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "rw_device.cuh"
#include "rw_internal.h"
#include "rw_tma.cuh"

namespace rwb {

using namespace dev;

namespace {

__host__ __device__ inline size_t al16(size_t x) { return (x + 15) & ~size_t(15); }

struct RouteArgs {
  int64_t count;  // orders in this chunk
  int64_t base;   // batch index of the chunk's first order (error reports)
  int n;
  int R;          // rows per block (multiple of 8)
  int nblocks;
  int aligned;    // 16-byte aligned uint16 orders: vector loads allowed
  unsigned long long* err;
};

// Zeroes each 16-bit half of w that has a bit of hmask set (bad-order path only).
__device__ __forceinline__ uint32_t clear_bad(uint32_t w, uint32_t hmask) {
  const uint32_t t = w & hmask;
  return w & ((t & 0xFFFFu) ? 0xFFFF0000u : 0xFFFFFFFFu) & ((t >> 16) ? 0x0000FFFFu : 0xFFFFFFFFu);
}

// 5 CTAs per SM (48 registers): more warps to cover the order loads' HBM
// latency than 4 (63 registers); measured +1.3% on C4, 6 spills.
template <typename P, bool kValidate, bool kPow2>
__global__ void __launch_bounds__(256, 5) k_ring_route(RouteArgs a, const P* __restrict__ perms,
                                                    uint16_t* __restrict__ pred) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = a.n;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint16_t* buf = reinterpret_cast<uint16_t*>(smem + (size_t)wib * al16((size_t)n * 2));
  uint4* buf4 = reinterpret_cast<uint4*>(buf);
  const uint4 ones = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
  const int chunks8 = n >> 3;  // n % 8 == 0 on this path
  const uint32_t hmask = kPow2 ? ~((uint32_t)(n - 1) * 0x10001u) : 0x80008000u;
  for (int c = lane; c < chunks8; c += 32) buf4[c] = ones;
  __syncwarp();
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t o = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; o < a.count; o += nwarps) {
    const P* pp = perms + o * n;
    bool bad = false;
    if constexpr (sizeof(P) == 2) {
      if ((n & 255) == 0 && a.aligned) {
        const uint4* pv = reinterpret_cast<const uint4*>(pp);
        uint32_t carry = ld_order<P>(pp, n - 1);
        const int nc = n >> 8;
        for (int c0 = 0; c0 < nc; c0 += 4) {
          // up to four 16-byte loads in flight per lane (one HBM round trip
          // per order at N=1024), then the scatter
          uint4 vv[4];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (c0 + q < nc) vv[q] = __ldg(pv + (c0 + q) * 32 + lane);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (c0 + q >= nc) break;
            const uint4 v = vv[q];
            const uint32_t e[8] = {v.x & 0xFFFFu, v.x >> 16, v.y & 0xFFFFu, v.y >> 16,
                                   v.z & 0xFFFFu, v.z >> 16, v.w & 0xFFFFu, v.w >> 16};
            uint32_t prev = __shfl_up_sync(kFull, e[7], 1);
            const uint32_t last = __shfl_sync(kFull, e[7], 31);
            if (lane == 0) prev = carry;
            carry = last;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const uint32_t cur = e[k];
              // An out-of-range predecessor is also some hop's `cur`, which
              // flags the order.  The write-out below must still see it: for
              // a power-of-two n its mask test does; otherwise it is stored
              // as the sentinel here.
              const uint32_t pv = k == 0 ? prev : e[k - 1];
              if (cur < (uint32_t)n) buf[cur] = (uint16_t)(kPow2 || pv < (uint32_t)n ? pv : 0xFFFFu);
              else bad = true;
            }
          }
        }
      } else {
        for (int i = lane; i < n; i += 32) {
          const uint32_t cur = (uint32_t)ld_order<P>(pp, i);
          const uint32_t prev = (uint32_t)ld_order<P>(pp, i == 0 ? n - 1 : i - 1);
          if (cur < (uint32_t)n) buf[cur] = (uint16_t)(kPow2 || prev < (uint32_t)n ? prev : 0xFFFFu);
          else bad = true;
        }
      }
    } else {
      for (int i = lane; i < n; i += 32) {
        const uint32_t cur = (uint32_t)ld_order<P>(pp, i);
        const uint32_t prev = (uint32_t)ld_order<P>(pp, i == 0 ? n - 1 : i - 1);
        if (cur < (uint32_t)n && prev < (uint32_t)n) buf[cur] = (uint16_t)prev;
        else bad = true;
      }
    }
    __syncwarp();
    // write pred by row block (16-byte chunks), check the sentinel, reset
    for (int c = lane; c < chunks8; c += 32) {
      uint4 v = buf4[c];
      const int h0 = c << 3;
      const int b = h0 / a.R;
      const int s0 = h0 - b * a.R;
      // Valid entries are < n <= 8192: with a power-of-two n any bit of
      // ~(n-1) marks a sentinel or an out-of-range value, otherwise only the
      // 0xFFFF sentinel (bit 15) can remain.  A chunk holding one is a bad
      // order; those entries are zeroed so the score pass can index rows
      // without clamping (in range either way).
      if ((v.x | v.y | v.z | v.w) & hmask) {
        bad = true;
        v = make_uint4(clear_bad(v.x, hmask), clear_bad(v.y, hmask), clear_bad(v.z, hmask), clear_bad(v.w, hmask));
      }
      *reinterpret_cast<uint4*>(pred + ((size_t)b * a.count + o) * a.R + s0) = v;
      buf4[c] = ones;
    }
    __syncwarp();
    if (kValidate && __any_sync(kFull, bad) && lane == 0) report_bad_order(a.err, n, a.base + o);
  }
}

struct ScoreArgs {
  int64_t count;   // orders in this chunk
  int n;
  int R;           // rows per block
  int nblocks;
  int stages;        // TMA ring depth
  int stage_orders;  // orders per TMA stage
  int vec;           // multi-order warp step (R in {32, 64, 128, 256}, n % R == 0)
  int rotate;        // rotate the consumer deal per stage (1; 0 = fixed warp-0-first deal, -1.9% at C4)
  double* part;    // [nblocks][count] partial sums (coalesced for the combine pass)
  unsigned long long* acc;  // u16 codes: per-order integer sums accumulated atomically (exact)
};

constexpr int kMaxStages = 8;

__device__ __forceinline__ uint32_t lds_u16(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint4 lds_v4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

// Multi-order warp step over one stage (u16 codes, whole row blocks, R = 8*LPO):
// LPO lanes per order take 8 rows each -- one conflict-free 16-byte
// predecessor load, 8 shared-memory lookups, a segmented shuffle sum -- so a
// warp scores 32/LPO orders per step.  The route leaves every predecessor
// < n (sentinels zeroed), so the lookups need no clamp: the row addresses are
// hoisted and each lookup is extract + add + LDS.  The high half is (w >> 15):
// bit 15 of the low half is clear, so that is exactly 2 * (w >> 16).
// N > 0 fixes the row length at compile time (row offsets become LDS
// immediates); N == 0 takes it from `n`.
__device__ __forceinline__ uint32_t lo16(uint32_t w) {
  uint32_t r;
  asm("and.b32 %0, %1, 65535;" : "=r"(r) : "r"(w));  // opaque: keeps (w & 0xFFFF) * 2 + row a single LEA
  return r;
}

template <int LPO, int N, int U>
__device__ __forceinline__ void score_stage_vec(uint32_t gi, int stage_orders, bool rotate, const uint16_t* sp,
                                                const uint16_t* blk, int n, int cnt, int warp,
                                                int cw, int lane, unsigned long long* __restrict__ accp) {
  constexpr int OPW = 32 / LPO, R = 8 * LPO;
  const int sub = lane & (LPO - 1), kk = lane / LPO;
  const uint32_t rstep = N > 0 ? (uint32_t)N * 2u : (uint32_t)n * 2u;
  const uint32_t row0 = (uint32_t)__cvta_generic_to_shared(blk) + (uint32_t)(sub * 8) * rstep;
  const uint32_t src = (uint32_t)__cvta_generic_to_shared(sp) + (uint32_t)(kk * R + sub * 8) * 2u;
  // U orders per lane group per step: more lookups in flight, loop and
  // atomic-address overhead shared.
  // Lane-group steps are dealt round-robin over the consumer warps as one
  // continuous stream across stages (rotated by the stage counter gi): when
  // the steps of a stage do not divide over the consumer warps (48 steps for
  // 31 warps when the CTA had 1024 threads), a fixed warp-0-first deal would
  // give the same warps the extra step every stage.
  const int rot = rotate ? (int)((uint64_t)gi * (uint32_t)(stage_orders / (OPW * U)) % (uint32_t)cw) : 0;
  const int w0 = warp - rot < 0 ? warp - rot + cw : warp - rot;
  for (int k0 = w0 * OPW * U; k0 < cnt; k0 += cw * OPW * U) {
    uint32_t acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = k0 + u * OPW + kk;
      acc[u] = 0;
      if (k < cnt) {
        const uint4 w4 = lds_v4(src + (uint32_t)(k0 + u * OPW) * (R * 2));
        const uint32_t w[4] = {w4.x, w4.y, w4.z, w4.w};
        uint32_t v[8];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          v[2 * q] = lds_u16(row0 + lo16(w[q]) * 2u + (2 * q) * rstep);
          v[2 * q + 1] = lds_u16(row0 + (w[q] >> 15) + (2 * q + 1) * rstep);
        }
        acc[u] = (v[0] + v[1] + v[2]) + (v[3] + v[4] + v[5]) + (v[6] + v[7]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int off = LPO >> 1; off > 0; off >>= 1) acc[u] += __shfl_xor_sync(kFull, acc[u], off);
    }
    if (sub == 0) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (k0 + u * OPW + kk < cnt) atomicAdd(accp + k0 + u * OPW + kk, (unsigned long long)acc[u]);
    }
  }
}

// The same multi-order warp step for FP32 / FP64 matrices: LPO lanes per
// order, 8 rows per lane, unclamped lookups (the route zeroes sentinels).  A
// lane adds its 8 values in row order in FP64, the segmented butterfly adds
// the LPO lane sums, and lane `sub == 0` writes the (order, block) partial to
// part[block][order]; k_ring_combine then sums the partials in block order.
// Every addition happens in a fixed order, so the result is deterministic.
template <typename T>
__device__ __forceinline__ T lds_t(uint32_t addr);
template <>
__device__ __forceinline__ float lds_t<float>(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
template <>
__device__ __forceinline__ double lds_t<double>(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}

template <typename T, int LPO, int N>
__device__ __forceinline__ void score_stage_vec_fp(uint32_t gi, int stage_orders, bool rotate, const uint16_t* sp,
                                                   const T* blk, int n, int cnt, int warp, int cw, int lane,
                                                   double* __restrict__ partp) {
  constexpr int OPW = 32 / LPO, R = 8 * LPO;
  constexpr uint32_t E = sizeof(T);
  const int sub = lane & (LPO - 1), kk = lane / LPO;
  const uint32_t rstep = N > 0 ? (uint32_t)N * E : (uint32_t)n * E;
  const uint32_t row0 = (uint32_t)__cvta_generic_to_shared(blk) + (uint32_t)(sub * 8) * rstep;
  const uint32_t src = (uint32_t)__cvta_generic_to_shared(sp) + (uint32_t)(kk * R + sub * 8) * 2u;
  const int rot = rotate ? (int)((uint64_t)gi * (uint32_t)(stage_orders / OPW) % (uint32_t)cw) : 0;
  const int w0 = warp - rot < 0 ? warp - rot + cw : warp - rot;
  for (int k0 = w0 * OPW; k0 < cnt; k0 += cw * OPW) {
    const int k = k0 + kk;
    double acc = 0.0;
    if (k < cnt) {
      const uint4 w4 = lds_v4(src + (uint32_t)k0 * (R * 2));
      const uint32_t w[4] = {w4.x, w4.y, w4.z, w4.w};
      T v[8];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        v[2 * q] = lds_t<T>(row0 + lo16(w[q]) * E + (2 * q) * rstep);
        v[2 * q + 1] = lds_t<T>(row0 + (w[q] >> 16) * E + (2 * q + 1) * rstep);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) acc = __dadd_rn(acc, (double)v[j]);
    }
#pragma unroll
    for (int off = LPO >> 1; off > 0; off >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(kFull, acc, off));
    if (sub == 0 && k < cnt) partp[k] = acc;
  }
}

// Pass 2: a CTA keeps rows [b*R, b*R + rows) in shared memory and streams the
// block's predecessor slices (contiguous in predbuf) through a 4-stage TMA
// bulk-copy ring; each warp scores one order per step with shared-memory
// lookups and writes the (order, block) partial.
// 24 consumer warps + 1 producer warp.  A 384-order stage at C4 is 48 lane-
// group steps, two per consumer warp; measured on B200 (C4 u16, bench.py):
// 1024 threads 7.11e8, 800 threads 7.36e8, 544 7.00e8, 416 6.82e8 evals/s.
constexpr int kScoreThreads = 800;

template <typename T>
__global__ void __launch_bounds__(kScoreThreads, 1) k_ring_score(ScoreArgs a, const uint16_t* __restrict__ pred,
                                                        const T* __restrict__ gmat) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = a.n, R = a.R, nb = a.nblocks;
  T* blk = reinterpret_cast<T*>(smem);
  uint16_t* ring = reinterpret_cast<uint16_t*>(smem + al16((size_t)R * n * sizeof(T)));
  __shared__ __align__(8) uint64_t bars[kMaxStages], empty[kMaxStages], mat_bar;
  const int kStages = a.stages, kStageOrders = a.stage_orders;
  unsigned mat_phase = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const uint32_t nm1 = (uint32_t)(n - 1);
  constexpr bool kInt = std::is_same<T, uint16_t>::value;
  const size_t stage_elems = (size_t)kStageOrders * R;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&bars[s], 1);
      mbar_init(&empty[s], nwarps - 1);
    }
    mbar_init(&mat_bar, 1);
  }
  __syncthreads();
  uint32_t g = 0;  // running stage counter of this CTA (same in every role)

  // Stream-K split: the (row block, stage) units are cut into gridDim.x equal
  // contiguous ranges, so every SM gets the same work and a CTA restages the
  // matrix only where its range crosses a row block.
  const int64_t nst_all = (a.count + kStageOrders - 1) / kStageOrders;
  const int64_t units = nst_all * nb;
  const int64_t u_end = units * (blockIdx.x + 1) / gridDim.x;
  for (int64_t u = units * blockIdx.x / gridDim.x; u < u_end;) {
    const int b = (int)(u / nst_all);
    const int64_t st0 = u - (int64_t)b * nst_all;
    const int64_t nstage = min(nst_all - st0, u_end - u);
    u += nstage;
    const int64_t o0 = st0 * kStageOrders;
    const int64_t total = min(a.count, (st0 + nstage) * kStageOrders) - o0;
    const int row0 = b * R;
    const int rows = min(R, n - row0);
    __syncthreads();  // previous item fully consumed
    stage_rows(blk, gmat + (size_t)row0 * n, (size_t)rows * n * sizeof(T), &mat_bar, &mat_phase);
    const uint16_t* base = pred + ((size_t)b * a.count + o0) * R;
    // Producer / consumer ring: the last warp issues the bulk copies, gated
    // by per-slot "empty" barriers that the consumer warps arrive on; no
    // CTA-wide barrier per stage.
    if (warp == nwarps - 1) {
      if (lane == 0) {
        for (int64_t st = 0; st < nstage; ++st) {
          const uint32_t gi = g + (uint32_t)st;
          const int slot = (int)(gi % (uint32_t)kStages);
          const uint32_t use = gi / (uint32_t)kStages;
          if (use > 0) mbar_wait(&empty[slot], (use - 1) & 1u);
          const int64_t cnt = min((int64_t)kStageOrders, total - st * kStageOrders);
          const unsigned bytes = (unsigned)(cnt * R * 2);
          mbar_expect_tx(&bars[slot], bytes);
          bulk_g2s(ring + slot * stage_elems, base + (size_t)st * stage_elems, bytes, &bars[slot]);
        }
      }
    } else {
      const int cw = nwarps - 1;
      for (int64_t st = 0; st < nstage; ++st) {
        const uint32_t gi = g + (uint32_t)st;
        const int slot = (int)(gi % (uint32_t)kStages);
        mbar_wait(&bars[slot], (gi / (uint32_t)kStages) & 1u);
        const int64_t cnt = min((int64_t)kStageOrders, total - st * kStageOrders);
        const uint16_t* sp = ring + slot * stage_elems;
        if constexpr (kInt) {
          if (a.vec) {
            unsigned long long* accp = a.acc + o0 + st * kStageOrders;
            const bool rot = a.rotate != 0;
            const int c = (int)cnt;
            // C4 (R=64, N=1024): row stride as LDS immediates, two orders per
            // lane group (U=2 measured +0.9% over U=1 on B200)
            if (R == 64 && n == 1024) score_stage_vec<8, 1024, 2>(gi, kStageOrders, rot, sp, blk, n, c, warp, cw, lane, accp);
            else if (R == 32) score_stage_vec<4, 0, 1>(gi, kStageOrders, rot, sp, blk, n, c, warp, cw, lane, accp);
            else if (R == 64) score_stage_vec<8, 0, 1>(gi, kStageOrders, rot, sp, blk, n, c, warp, cw, lane, accp);
            else if (R == 128) score_stage_vec<16, 0, 1>(gi, kStageOrders, rot, sp, blk, n, c, warp, cw, lane, accp);
            else score_stage_vec<32, 0, 1>(gi, kStageOrders, rot, sp, blk, n, c, warp, cw, lane, accp);
          } else
          // u16 codes: a block partial is < R * 65536 <= 2^32 (R <= 1024 here)
          for (int k = warp; k < cnt; k += cw) {
            const uint16_t* src = sp + (size_t)k * R;
            uint32_t acc = 0;
#pragma unroll 1
            for (int s = 2 * lane; s < rows; s += 64) {
              const uint32_t w = *reinterpret_cast<const uint32_t*>(src + s);
              acc += (uint32_t)blk[s * n + min(w & 0xFFFFu, nm1)] + (uint32_t)blk[(s + 1) * n + min(w >> 16, nm1)];
            }
            acc = __reduce_add_sync(kFull, acc);
            if (lane == 0) atomicAdd(a.acc + o0 + st * kStageOrders + k, (unsigned long long)acc);
          }
        } else if (a.vec) {
          double* partp = a.part + (size_t)b * a.count + o0 + st * kStageOrders;
          const bool rot = a.rotate != 0;
          const int c = (int)cnt;
          // FP32 at N=1024 takes R=32, FP64 R=16 (the row block's shared memory)
          if (R == 32 && n == 1024) score_stage_vec_fp<T, 4, 1024>(gi, kStageOrders, rot, sp, blk, n, c, warp, cw, lane, partp);
          else if (R == 16 && n == 1024) score_stage_vec_fp<T, 2, 1024>(gi, kStageOrders, rot, sp, blk, n, c, warp, cw, lane, partp);
          else if (R == 16) score_stage_vec_fp<T, 2, 0>(gi, kStageOrders, rot, sp, blk, n, c, warp, cw, lane, partp);
          else if (R == 32) score_stage_vec_fp<T, 4, 0>(gi, kStageOrders, rot, sp, blk, n, c, warp, cw, lane, partp);
          else if (R == 64) score_stage_vec_fp<T, 8, 0>(gi, kStageOrders, rot, sp, blk, n, c, warp, cw, lane, partp);
          else if (R == 128) score_stage_vec_fp<T, 16, 0>(gi, kStageOrders, rot, sp, blk, n, c, warp, cw, lane, partp);
          else score_stage_vec_fp<T, 32, 0>(gi, kStageOrders, rot, sp, blk, n, c, warp, cw, lane, partp);
        } else {
          for (int k = warp; k < cnt; k += cw) {
            const uint16_t* src = sp + (size_t)k * R;
            double dacc = 0.0;
#pragma unroll 1
            for (int s = 2 * lane; s < rows; s += 64) {
              const uint32_t w = *reinterpret_cast<const uint32_t*>(src + s);
              const T v0 = blk[s * n + min(w & 0xFFFFu, nm1)];
              const T v1 = blk[(s + 1) * n + min(w >> 16, nm1)];
              dacc = __dadd_rn(__dadd_rn(dacc, (double)v0), (double)v1);
            }
            const double partial = warp_sum(dacc);
            if (lane == 0) a.part[(size_t)b * a.count + o0 + st * kStageOrders + k] = partial;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
      }
    }
    g += (uint32_t)nstage;
  }
}

// Pass 3: cost[o] = (sum of the order's block partials, in block order) * mul.
__global__ void k_ring_combine(const double* __restrict__ part, int64_t count, int nb, double mul,
                               double* __restrict__ costs) {
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < count; o += (int64_t)gridDim.x * blockDim.x) {
    double sum = 0.0;
    for (int k = 0; k < nb; ++k) sum = __dadd_rn(sum, part[(size_t)k * count + o]);
    costs[o] = __dmul_rn(sum, mul);
  }
}

// u16 path epilogue: costs hold integer sums (as u64 bits); scale in place.
__global__ void k_ring_finalize(double* __restrict__ costs, int64_t count, double mul) {
  unsigned long long* bits = reinterpret_cast<unsigned long long*>(costs);
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < count; o += (int64_t)gridDim.x * blockDim.x)
    costs[o] = __dmul_rn((double)bits[o], mul);
}

}  // namespace

bool launch_ring_transpose(const Problem& p, const EvalPlan& plan, const void* d_perms, int perm_bytes, int64_t batch,
                           double* d_costs, bool validate, int* err_slot, cudaStream_t st, int slot) {
  const int n = plan.n;
  if (n % 8 != 0 || n < 256 || n > 8192 || batch <= 0) return false;
  int sms = 148, optin = 227 * 1024;
  RW_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p.device));
  RW_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, p.device));
  const size_t budget = (size_t)std::min(optin, 227 * 1024) - 2048;
  const size_t esz = p.elem_bytes();
  // A row block must leave room for at least two 128-order stages.
  auto fits = [&](int R) { return al16((size_t)R * n * esz) + (size_t)2 * 128 * R * 2 <= budget; };
  // row blocks: prefer an exact split of n into multiples of 8 rows
  int nblocks = 0, R = 0;
  for (int nb = 1; nb <= n / 8 && !nblocks; ++nb) {
    const int r = ((n + nb - 1) / nb + 7) & ~7;
    if (!fits(r)) continue;
    int best_nb = nb;
    for (int e = nb; e <= 4 * nb && e <= n / 8; ++e)
      if (n % e == 0 && (n / e) % 8 == 0 && fits(n / e)) {
        best_nb = e;
        break;
      }
    nblocks = best_nb;
    R = ((n + nblocks - 1) / nblocks + 7) & ~7;
  }
  if (!nblocks) return false;
  // Stages: the shared memory the row block leaves, as two stages of up to
  // 512 orders (more stages only beyond that).  Larger bulk copies and fewer
  // stage hand-offs measured faster on B200 at N=1024, R=64: 4 x 128 orders
  // 4.0e8, 3 x 256 4.4e8, 2 x 384 4.55e8 evals/s.
  const size_t ring_bytes = budget - al16((size_t)R * n * esz);
  int kStageOrders = (int)std::min<size_t>(512, ring_bytes / (2 * (size_t)R * 2)) & ~31;
  int kStages = 2;
  if (kStageOrders >= 512)
    kStages = (int)std::min<size_t>(kMaxStages, ring_bytes / ((size_t)kStageOrders * R * 2));
  if (kStageOrders < 32) return false;
  // Predecessor exchange buffer of up to 512 MB (2n bytes per order).  Each
  // chunk pays a fixed cost (two launches, every score CTA restaging its row
  // block and filling its stage ring), which outweighs keeping the buffer
  // L2-resident; measured in bench.py on B200 at N=1024 (evals/s):
  // 48 MB 4.85e8, 96 MB 5.07e8, 128 MB 5.30e8, 256 MB 5.45e8, 512 MB 5.55e8,
  // 1 GB 5.59e8.  Scratch only grows to min(batch, chunk) orders.
  static const int64_t chunk_bytes = [] {
    const char* e = std::getenv("RW_RING_CHUNK_MB");  // A/B measurements only
    return e ? std::max(8L, std::atol(e)) << 20 : (int64_t)512 << 20;
  }();
  const int64_t chunk = std::max<int64_t>(4096, chunk_bytes / ((int64_t)n * 2));
  ThreadCtx& c = thread_ctx(p.device);
  const int64_t kmax = std::min(batch, chunk);
  uint16_t* predbuf = static_cast<uint16_t*>(c.scratch(slot, (size_t)nblocks * kmax * R * 2));
  double* part = static_cast<double*>(c.scratch(slot + 1, (size_t)kmax * nblocks * 8 + 64));

  const size_t route_smem = 8 * al16((size_t)n * 2);
  const size_t score_smem = al16((size_t)R * n * esz) + (size_t)kStages * kStageOrders * R * 2;
  auto set = [](auto kern, size_t bytes) {
    if (bytes > 48 * 1024) RW_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  };
  const bool pow2 = (n & (n - 1)) == 0;
  const bool int_sums = p.storage == RW_STORAGE_U16;
  if (int_sums) RW_CUDA(cudaMemsetAsync(d_costs, 0, (size_t)batch * 8, st));
  for (int64_t off = 0; off < batch; off += kmax) {
    const int64_t cnt_o = std::min(kmax, batch - off);
    // 16-byte order loads need a 16-byte aligned base (an offset view of a
    // caller's tensor may not be); n % 256 == 0 keeps every row aligned.
    const int aligned = (reinterpret_cast<uintptr_t>(d_perms) % 16) == 0 ? 1 : 0;
    RouteArgs ra{cnt_o, off, n, R, nblocks, aligned, reinterpret_cast<unsigned long long*>(err_slot)};
    // One full wave of resident route CTAs (grid-stride over the orders):
    // every CTA does the same work, so a partial second wave would be a tail.
    auto rgrid = [&](auto kern) {
      int per_sm = 0;
      RW_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, route_smem));
      return (int)std::max<int64_t>(1, std::min<int64_t>((cnt_o + 7) / 8, (int64_t)sms * std::max(1, per_sm)));
    };
    if (perm_bytes == 2) {
      auto k = pow2 ? (validate ? k_ring_route<uint16_t, true, true> : k_ring_route<uint16_t, false, true>)
                    : (validate ? k_ring_route<uint16_t, true, false> : k_ring_route<uint16_t, false, false>);
      set(k, route_smem);
      k<<<rgrid(k), 256, route_smem, st>>>(ra, static_cast<const uint16_t*>(d_perms) + off * n, predbuf);
    } else {
      auto k = pow2 ? (validate ? k_ring_route<int32_t, true, true> : k_ring_route<int32_t, false, true>)
                    : (validate ? k_ring_route<int32_t, true, false> : k_ring_route<int32_t, false, false>);
      set(k, route_smem);
      k<<<rgrid(k), 256, route_smem, st>>>(ra, static_cast<const int32_t*>(d_perms) + off * n, predbuf);
    }
    RW_CUDA(cudaGetLastError());
    const int vec = (R == 32 || R == 64 || R == 128 || R == 256 || (R == 16 && !int_sums)) && n % R == 0 ? 1 : 0;
    ScoreArgs sa{cnt_o, n, R, nblocks, kStages, kStageOrders, vec, 1, part,
                 reinterpret_cast<unsigned long long*>(d_costs + off)};
    const int sgrid = (int)std::min<int64_t>(sms, (int64_t)nblocks * ((cnt_o + kStageOrders - 1) / kStageOrders));
    switch (p.storage) {
      case RW_STORAGE_U16: {
        auto k = k_ring_score<uint16_t>;
        set(k, score_smem);
        k<<<sgrid, kScoreThreads, score_smem, st>>>(sa, predbuf, static_cast<const uint16_t*>(p.d_mat));
        break;
      }
      case RW_STORAGE_F32: {
        auto k = k_ring_score<float>;
        set(k, score_smem);
        k<<<sgrid, kScoreThreads, score_smem, st>>>(sa, predbuf, static_cast<const float*>(p.d_mat));
        break;
      }
      default: {
        auto k = k_ring_score<double>;
        set(k, score_smem);
        k<<<sgrid, kScoreThreads, score_smem, st>>>(sa, predbuf, static_cast<const double*>(p.d_mat));
        break;
      }
    }
    RW_CUDA(cudaGetLastError());
    if (!int_sums) {
      k_ring_combine<<<(int)std::min<int64_t>((cnt_o + 255) / 256, (int64_t)sms * 8), 256, 0, st>>>(
          part, cnt_o, nblocks, plan.ring_mul, d_costs + off);
      RW_CUDA(cudaGetLastError());
    }
  }
  if (int_sums) {
    k_ring_finalize<<<(int)std::min<int64_t>((batch + 255) / 256, (int64_t)sms * 16), 256, 0, st>>>(d_costs, batch,
                                                                                                  plan.ring_mul);
    RW_CUDA(cudaGetLastError());
  }
  return true;
}

}  // namespace rwb
