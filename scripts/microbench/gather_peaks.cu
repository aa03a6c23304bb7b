// gather_peaks.cu -- random-gather peaks on this GPU ("L2 and
// DSMEM random-gather peaks are not in MEASURED_PEAKS.json; microbenchmark
// them before quoting fractions").  Random 2-byte lookups, the access the
// scoring kernels make into the cost matrix:
//   * shared memory: a 32 KB u16 table per CTA, 32 warps per SM;
//   * L2: a 32 MB u16 table (the C5 matrix size), 64 warps per SM.
// Indices come from a per-thread xorshift in registers, so the only memory
// traffic is the gathers themselves.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_peaks_bin gather_peaks.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t xs(uint32_t& s) {
  s ^= s << 13;
  s ^= s >> 17;
  s ^= s << 5;
  return s;
}

__global__ void __launch_bounds__(1024, 1) k_smem(int iters, unsigned* out) {
  __shared__ uint16_t tab[16384];  // 32 KB (static limit 48 KB)
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) tab[i] = (uint16_t)(i * 7);
  __syncthreads();
  uint32_t s = 0x9E3779B9u * (blockIdx.x * blockDim.x + threadIdx.x + 1);
  uint32_t acc = 0;
  for (int k = 0; k < iters; ++k) {
    const uint32_t r = xs(s);
#pragma unroll
    for (int q = 0; q < 4; ++q) acc += tab[(r >> (q * 4)) & 16383];
  }
  if (acc == 0x12345678u) out[0] = acc;
}

__global__ void __launch_bounds__(256) k_l2(const uint16_t* __restrict__ tab, uint32_t mask, int iters, unsigned* out) {
  uint32_t s = 0x9E3779B9u * (blockIdx.x * blockDim.x + threadIdx.x + 1);
  uint32_t acc = 0;
  for (int k = 0; k < iters; ++k) {
    const uint32_t r0 = xs(s), r1 = xs(s);
    acc += __ldg(tab + (r0 & mask)) + __ldg(tab + (r1 & mask)) + __ldg(tab + ((r0 >> 7 ^ r1) & mask)) +
           __ldg(tab + ((r1 >> 5 ^ r0) & mask));
  }
  if (acc == 0x12345678u) out[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* out;
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  {
    const int iters = 20000;
    k_smem<<<sms, 1024>>>(100, out);
    cudaEventRecord(e0);
    k_smem<<<sms, 1024>>>(iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double lookups = (double)sms * 1024 * iters * 4;
    printf("smem random u16 gather : %.3e lookups/s (%.2f per SM-cycle at 1.965 GHz) %s\n", lookups / (ms * 1e-3),
           lookups / (ms * 1e-3) / sms / 1.965e9, cudaGetErrorString(cudaGetLastError()));
  }
  {
    const size_t n = (size_t)16 << 20;  // 16M u16 = 32 MB
    uint16_t* tab;
    cudaMalloc(&tab, n * 2);
    cudaMemset(tab, 1, n * 2);
    const int iters = 2000;
    k_l2<<<sms * 8, 256>>>(tab, (uint32_t)(n - 1), 50, out);
    cudaEventRecord(e0);
    k_l2<<<sms * 8, 256>>>(tab, (uint32_t)(n - 1), iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double lookups = (double)sms * 8 * 256 * iters * 4;
    printf("L2 random u16 gather   : %.3e lookups/s (%.2f per SM-cycle at 1.965 GHz) %s\n", lookups / (ms * 1e-3),
           lookups / (ms * 1e-3) / sms / 1.965e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
