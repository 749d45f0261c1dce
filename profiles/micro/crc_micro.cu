// Micro-benchmark: CRC pass throughput from shared memory (the decode CRC
// warp's inner loop) — cycles per 4608-byte pass per warp, and SM-level B/clk.
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../../paper_2004_03054_b200/csrc/luda_common.cuh"
#include "../../paper_2004_03054_b200/csrc/luda_tables.cuh"
using namespace luda;

__global__ void __launch_bounds__(1024, 1) crc_bench(int warps, int iters, uint32_t* out, unsigned long long* cyc) {
  extern __shared__ __align__(128) uint8_t sm[];
  CrcSmem& cs = *reinterpret_cast<CrcSmem*>(sm);
  uint8_t* buf = sm + sizeof(CrcSmem);
  crc_smem_init(cs);
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) buf[i] = (uint8_t)(i * 131 + 7);
  __syncthreads();
  const int w = threadIdx.x >> 5;
  if (w >= warps) return;
  uint8_t* data = buf + 64 + (w % 4) * 16;  // shared read-only data
  uint32_t acc = 0;
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    acc ^= warp_xor(pass_lane_value_al(data + 4608, 4608, 0, cs));
    data = buf + 64 + (w % 4) * 16 + ((acc >> 31) & 1) * 16;  // loop-carried: no hoisting
  }
  unsigned long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) { out[blockIdx.x * 32 + w] = acc; cyc[blockIdx.x * 32 + w] = t1 - t0; }
}

int main() {
  if (upload_crc_tables()) { printf("tables failed\n"); return 1; }
  uint32_t* out; unsigned long long* cyc;
  cudaMalloc(&out, 148 * 32 * 4); cudaMalloc(&cyc, 148 * 32 * 8);
  size_t smem = sizeof(CrcSmem) + 8192 + 256;
  cudaFuncSetAttribute(crc_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int warps : {1, 2, 4, 8, 12, 16, 24, 32}) {
    int iters = 200;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    crc_bench<<<148, 1024, smem>>>(warps, 10, out, cyc);
    cudaEventRecord(a);
    crc_bench<<<148, 1024, smem>>>(warps, iters, out, cyc);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    std::vector<unsigned long long> h(148 * 32);
    cudaMemcpy(h.data(), cyc, h.size() * 8, cudaMemcpyDeviceToHost);
    double cpp = (double)h[0] / iters;
    double bytes = 148.0 * warps * iters * 4608;
    printf("warps/SM %2d: %.0f cycles/pass/warp, %.1f B/clk/SM (clock), %.2f TB/s (events, incl. init)\n", warps, cpp,
           4608.0 * warps / cpp, bytes / (ms * 1e-3) / 1e12);
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
