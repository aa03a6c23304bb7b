// rw_tma.cuh -- mbarrier + TMA bulk-copy helpers (sm_90+ PTX, used on
// sm_100a) shared by the transpose scoring kernels.
#pragma once

#include <cstdint>

namespace rwb {
namespace dev {

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}
// TMA bulk copy global -> shared (1D, 16-byte multiple), completion on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar))
               : "memory");
}

// Stages `bytes` of contiguous matrix rows into shared memory.  Must be called
// by the whole CTA (after a barrier that retires the previous contents); on
// return the rows are visible to every thread.  With 16-byte aligned sizes
// the copy is one TMA bulk stream completing on `bar` (phase parity tracked
// by the caller in *phase); otherwise a vectorised-by-16 fallback loop.
__device__ __forceinline__ void stage_rows(void* dst, const void* src, size_t bytes, uint64_t* bar,
                                           unsigned* phase) {
  const bool tma = ((bytes & 15) == 0) && ((reinterpret_cast<uintptr_t>(src) & 15) == 0);
  if (tma) {
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads of dst
      mbar_expect_tx(bar, (unsigned)bytes);
      constexpr size_t kPiece = 32768;
      for (size_t off = 0; off < bytes; off += kPiece) {
        const size_t len = bytes - off < kPiece ? bytes - off : kPiece;
        bulk_g2s(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off, (unsigned)len, bar);
      }
    }
    mbar_wait(bar, *phase);
    *phase ^= 1u;
  } else {
    const size_t words = bytes >> 1;  // every matrix element is >= 2 bytes
    const uint16_t* s = static_cast<const uint16_t*>(src);
    uint16_t* d = static_cast<uint16_t*>(dst);
    for (size_t k = threadIdx.x; k < words; k += blockDim.x) d[k] = __ldg(s + k);
    __syncthreads();
  }
}

}  // namespace dev
}  // namespace rwb
