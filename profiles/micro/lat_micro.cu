// Latency micro-benchmark: dependent LDS.U8 / LDS.32 pointer chase and SHFL chain on one warp.
#include <cstdio>
#include <cstdint>
__global__ void lat(int iters, unsigned long long* out, uint32_t* sink) {
  __shared__ uint8_t b8[4096];
  __shared__ uint32_t b32[1024];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) b8[i] = (uint8_t)((i * 37 + 11) & 0xFF);
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) b32[i] = (i * 97 + 5) & 1023;
  __syncthreads();
  uint32_t p = threadIdx.x;
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) p = (p + b8[p & 4095]) & 4095;
  unsigned long long t1 = clock64();
  for (int i = 0; i < iters; ++i) p = b32[p & 1023];
  unsigned long long t2 = clock64();
  uint32_t v = p;
  for (int i = 0; i < iters; ++i) v = __shfl_sync(0xFFFFFFFFu, v, (v + 1) & 31) + 1;
  unsigned long long t3 = clock64();
  for (int i = 0; i < iters; ++i) v = v * 3 + 1;
  unsigned long long t4 = clock64();
  for (int i = 0; i < iters; ++i) v = (v ^ (v >> 3)) + p;
  unsigned long long t5 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3; out[4] = t5 - t4; }
  sink[threadIdx.x] = p + v;
}
int main() {
  unsigned long long* d; uint32_t* s; cudaMalloc(&d, 64); cudaMalloc(&s, 4096);
  int it = 10000;
  lat<<<1, 32>>>(it, d, s); cudaDeviceSynchronize();
  lat<<<1, 32>>>(it, d, s);
  unsigned long long h[5]; cudaMemcpy(h, d, 40, cudaMemcpyDeviceToHost);
  printf("LDS.U8 chase %.1f  LDS.32 chase %.1f  SHFL chain %.1f  IMAD chain %.1f  ALU chain %.1f cycles/step\n",
         h[0] / (double)it, h[1] / (double)it, h[2] / (double)it, h[3] / (double)it, h[4] / (double)it);
  return 0;
}
