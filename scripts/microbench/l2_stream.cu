// l2_stream.cu -- how fast can the SMs read back a buffer another kernel just
// wrote (the transpose paths' exchange buffer)?  Plain 16-byte loads vs TMA
// bulk stages vs the same read from a cold (HBM) buffer.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2s l2_stream.cu && /tmp/l2s
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_write(uint4* b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = make_uint4((uint32_t)i, 1, 2, 3);
}
__global__ void k_read_ldg(const uint4* b, size_t n, unsigned* out) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const uint4 v = __ldg(b + i);
    acc += v.x ^ v.w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(c));
}
__device__ __forceinline__ void mbar_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned par) {
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(par) : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"((uint32_t)__cvta_generic_to_shared(d)), "l"(s), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}
// each CTA streams its contiguous share in `stage` byte pieces through `depth` slots
__global__ void k_read_tma(const char* b, size_t bytes, int stage, int depth, unsigned* out) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ __align__(8) uint64_t bars[16];
  if (threadIdx.x == 0) for (int s = 0; s < depth; ++s) mbar_init(&bars[s], 1);
  __syncthreads();
  const size_t per = (bytes / gridDim.x / stage) * stage;
  const char* base = b + per * blockIdx.x;
  const int nst = (int)(per / stage);
  unsigned par = 0;
  if (threadIdx.x == 0) for (int s = 0; s < depth && s < nst; ++s) { mbar_tx(&bars[s], stage); bulk(sm + (size_t)s * stage, base + (size_t)s * stage, stage, &bars[s]); }
  uint32_t acc = 0;
  for (int st = 0; st < nst; ++st) {
    const int slot = st % depth;
    mbar_wait(&bars[slot], (par >> slot) & 1u);
    acc += reinterpret_cast<const uint32_t*>(sm + (size_t)slot * stage)[threadIdx.x];
    par ^= 1u << slot;
    __syncthreads();
    if (threadIdx.x == 0 && st + depth < nst) { mbar_tx(&bars[slot], stage); bulk(sm + (size_t)slot * stage, base + (size_t)(st + depth) * stage, stage, &bars[slot]); }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

int main() {
  const size_t bytes = 50ull << 20;
  const size_t cold_bytes = 2048ull << 20;
  char *buf, *cold;
  unsigned* out;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&cold, cold_bytes);
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  auto rep = [&](const char* name, size_t nb, auto fn) {
    for (int w = 0; w < 2; ++w) { k_write<<<148 * 8, 256>>>((uint4*)buf, bytes / 16); fn(); }
    float tot = 0;
    for (int r = 0; r < 10; ++r) {
      k_write<<<148 * 8, 256>>>((uint4*)buf, bytes / 16);
      cudaEventRecord(e0);
      fn();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      tot += ms;
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaGetLastError();
    printf("%-40s %8.1f GB/s  (%.1f us) %s\n", name, nb / (tot / 10 * 1e-3) / 1e9, tot / 10 * 1e3, cudaGetErrorString(e));
  };
  rep("ldg.128 148x8x256 (fresh L2)", bytes, [&] { k_read_ldg<<<148 * 8, 256>>>((const uint4*)buf, bytes / 16, out); });
  rep("ldg.128 148x4x1024 (fresh L2)", bytes, [&] { k_read_ldg<<<148 * 2, 1024>>>((const uint4*)buf, bytes / 16, out); });
  for (int stage : {16384, 32768, 65536})
    for (int depth : {2, 4, 8}) {
      if ((size_t)stage * depth > 200 * 1024) continue;
      cudaFuncSetAttribute(k_read_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, stage * depth);
      char name[64];
      snprintf(name, sizeof name, "tma stage %dK depth %d (fresh L2)", stage / 1024, depth);
      rep(name, bytes, [&] { k_read_tma<<<144, 1024, stage * depth>>>(buf, bytes, stage, depth, out); });
    }
  // cold HBM stream for reference
  k_write<<<148 * 8, 256>>>((uint4*)cold, cold_bytes / 16);
  cudaEventRecord(e0);
  k_read_ldg<<<148 * 8, 256>>>((const uint4*)cold, cold_bytes / 16, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("%-40s %8.1f GB/s %s\n", "ldg.128 2 GiB (HBM)", cold_bytes / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
