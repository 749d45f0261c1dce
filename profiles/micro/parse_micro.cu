// Micro-benchmark: the decode PARSE path (dec_phase1 + dec_phase2: walk,
// validation, key rebuild, record writes) on real c3 blocks staged in smem —
// cycles per block per warp at 1..N warps per SM (no TMA, no CRC).
#define DEC_TIMING 1
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../../paper_2004_03054_b200/csrc/luda_common.cuh"
#include "../../paper_2004_03054_b200/csrc/luda_decode.cuh"
#include "../../paper_2004_03054_b200/csrc/luda_tables.cuh"
using namespace luda;

constexpr int kSlotB = 4416;
__global__ void __launch_bounds__(1024, 1) parse_bench(const uint8_t* blocks, const uint32_t* boff, const uint32_t* blen,
                                                       int nblk, int warps, int iters, int mode, Rec<2>* out,
                                                       unsigned long long* cyc, unsigned long long* err) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int w = threadIdx.x >> 5;
  if (w >= warps) return;
  uint8_t* slot = sm + w * (kSlotB + kDecSlots * 8);
  DecSlot* slots = reinterpret_cast<DecSlot*>(slot + kSlotB);
  DecodeArgs<2> a{};
  a.K = 24;
  a.out = out + (size_t)(blockIdx.x * 32 + w) * 4096;
  a.err_ref = err;
  a.err_unsup = err + 1;
  unsigned long long tot = 0, tot1 = 0;
  int b = (blockIdx.x * 7 + w * 13) % nblk;
  for (int it = 0; it < iters; ++it, b = (b + 1) % nblk) {
    const uint8_t* g = blocks + boff[b];
    const uint32_t len = blen[b];
    uint8_t* d = slot + 48 + ((uintptr_t)g & 15);
    for (uint32_t i = threadIdx.x & 31; i < len; i += 32) d[i] = g[i];
    __syncwarp();
    const unsigned long long t0 = clock64();
    DecState st = dec_phase1(a, b, 0, len, d, slots);
    __syncwarp();
    const unsigned long long t1 = clock64();
    if (mode == 0) dec_phase2<2, true>(a, b, st, 0, 1 << 20, d, slots);
    __syncwarp();
    tot += clock64() - t0;
    tot1 += t1 - t0;
  }
  if ((threadIdx.x & 31) == 0) { cyc[blockIdx.x * 32 + w] = tot; cyc[148 * 32 + blockIdx.x * 32 + w] = tot1; }
}

int main() {
  FILE* f = fopen("profiles/micro/c3_blocks.bin", "rb");
  if (!f) { printf("no blocks\n"); return 1; }
  uint32_t n; fread(&n, 4, 1, f);
  std::vector<uint8_t> all; std::vector<uint32_t> off, len;
  for (uint32_t i = 0; i < n; ++i) {
    uint32_t l; fread(&l, 4, 1, f);
    // keep each block's address phase varied: place at offset with (i*5) % 16 misalignment
    while ((all.size() & 15) != (i * 5) % 16) all.push_back(0);
    off.push_back(all.size()); len.push_back(l);
    size_t p = all.size(); all.resize(p + l); fread(all.data() + p, 1, l, f);
  }
  fclose(f);
  uint8_t* d_all; uint32_t *d_off, *d_len; Rec<2>* d_out; unsigned long long *d_cyc, *d_err;
  cudaMalloc(&d_all, all.size() + 64); cudaMemcpy(d_all, all.data(), all.size(), cudaMemcpyHostToDevice);
  cudaMalloc(&d_off, 4 * n); cudaMemcpy(d_off, off.data(), 4 * n, cudaMemcpyHostToDevice);
  cudaMalloc(&d_len, 4 * n); cudaMemcpy(d_len, len.data(), 4 * n, cudaMemcpyHostToDevice);
  cudaMalloc(&d_out, sizeof(Rec<2>) * 148 * 32 * 4096);
  cudaMalloc(&d_cyc, 2 * 8 * 148 * 32); cudaMalloc(&d_err, 16);
  size_t smem = 32 * (kSlotB + kDecSlots * 8);
  if (smem > 232448) smem = 232448;
  cudaFuncSetAttribute(parse_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int warps : {1, 4, 8, 10, 16, 24, 32}) {
    if ((size_t)warps * (kSlotB + kDecSlots * 8) > smem) break;
    cudaMemset(d_err, 0xFF, 16);
    int iters = 200;
    parse_bench<<<148, warps * 32, smem>>>(d_all, d_off, d_len, n, warps, iters, 0, d_out, d_cyc, d_err);
    cudaDeviceSynchronize();
    std::vector<unsigned long long> h(2 * 148 * 32);
    cudaMemcpy(h.data(), d_cyc, 8 * h.size(), cudaMemcpyDeviceToHost);
    printf("   phase1 %.0f cycles, phase2 %.0f cycles\n", (double)h[148 * 32] / iters, (double)(h[0] - h[148 * 32]) / iters);
    unsigned long long tt[16];
    cudaMemcpyFromSymbol(tt, g_dec_t, sizeof(tt));
    double nb = 148.0 * warps * iters;
    printf("   p1 sections: restarts %.0f walk %.0f validate %.0f scan %.0f | p2: slot+hdr %.0f validate %.0f keyload %.0f resolve %.0f write %.0f\n", tt[0] / nb, tt[1] / nb, tt[2] / nb, tt[3] / nb, tt[4] / nb, tt[5] / nb, tt[6] / nb, tt[7] / nb, tt[8] / nb);
    { unsigned long long z[16] = {0}; cudaMemcpyToSymbol(g_dec_t, z, sizeof(z)); }
    unsigned long long e[2]; cudaMemcpy(e, d_err, 16, cudaMemcpyDeviceToHost);
    double cpb = (double)h[0] / iters;
    printf("warps/SM %2d: %.0f cycles/block/warp -> %.1f blocks/kcycle/SM (%.2f TB/s equiv @1.9GHz) err %llx\n", warps, cpb,
           1000.0 * warps / cpb, warps / cpb * 4009 * 148 * 1.9e9 / 1e12, e[0]);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
