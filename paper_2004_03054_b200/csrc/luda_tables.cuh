// luda_tables.cuh — CRC-32/IEEE tables and GF(2) shift operators.
//
// Host code computes, once per process (luda_init):
//   g_crc_tab   byte table of the reflected polynomial 0xEDB88320
//   g_crc_tab1  slicing-by-2 partner table (byte, then a zero byte)
//   g_seg_nib   nibble tables of Z_{kSeg*d}, d = 0..31 (segment combine)
//   g_half_tab  byte tables of Z_kHalf (between a lane's segments)
//   c_zpow      columns of Z_{2^i}, i = 0..47 (arbitrary shifts)
//   c_zgroup    columns of Z_4352 (one warp pass)
// where Z_n advances a raw CRC register over n zero bytes (the operator
// behind zlib's crc32_combine).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <utility>

#include "luda_common.cuh"

namespace luda {

namespace tables_detail {

void host_table(uint32_t* t) {
  for (uint32_t b = 0; b < 256; ++b) {
    uint32_t c = b;
    for (int k = 0; k < 8; ++k) c = (c & 1) ? (c >> 1) ^ kCrcPoly : (c >> 1);
    t[b] = c;
  }
}

uint32_t zero_bytes(const uint32_t* t, uint32_t c, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) c = t[c & 0xFF] ^ (c >> 8);
  return c;
}

uint32_t apply_cols(const uint32_t* cols, uint32_t c) {
  uint32_t r = 0;
  for (int j = 0; j < 32; ++j)
    if ((c >> j) & 1) r ^= cols[j];
  return r;
}

}  // namespace tables_detail

// Returns 0 on success.
using namespace tables_detail;
int upload_crc_tables() {
  uint32_t t[256];
  host_table(t);
  // Z_kSeg columns, then Z_{kSeg d} by repeated application.
  uint32_t z132[32];
  for (int j = 0; j < 32; ++j) z132[j] = zero_bytes(t, 1u << j, kSeg);
  static uint32_t nib[8 * 16 * 32];
  uint32_t cols[32];
  for (int j = 0; j < 32; ++j) cols[j] = 1u << j;  // Z_0 = identity
  for (int d = 0; d < 32; ++d) {
    for (int n = 0; n < 8; ++n)
      for (int v = 0; v < 16; ++v) nib[((n * 16) + v) * 32 + d] = apply_cols(cols, (uint32_t)v << (4 * n));
    uint32_t next[32];
    for (int j = 0; j < 32; ++j) next[j] = apply_cols(z132, cols[j]);
    memcpy(cols, next, sizeof(cols));
  }
  // Z_{2^i}: Z_1 columns then squaring.
  static uint32_t zpow[48][32];
  for (int j = 0; j < 32; ++j) zpow[0][j] = zero_bytes(t, 1u << j, 1);
  for (int i = 1; i < 48; ++i)
    for (int j = 0; j < 32; ++j) zpow[i][j] = apply_cols(zpow[i - 1], zpow[i - 1][j]);
  uint32_t zg[32];
  for (int j = 0; j < 32; ++j) zg[j] = zero_bytes(t, 1u << j, kGroup);
  uint32_t zh[32];
  for (int j = 0; j < 32; ++j) zh[j] = zero_bytes(t, 1u << j, kHalf);
  static uint32_t half[4 * 256];
  for (int k = 0; k < 4; ++k)
    for (int b = 0; b < 256; ++b) half[k * 256 + b] = apply_cols(zh, (uint32_t)b << (8 * k));
  if (cudaMemcpyToSymbol(g_half_tab, half, sizeof(half)) != cudaSuccess) return 1;
  if (cudaMemcpyToSymbol(g_crc_tab, t, sizeof(t)) != cudaSuccess) return 1;
  uint32_t t1[256];
  for (int b = 0; b < 256; ++b) t1[b] = t[t[b] & 0xFF] ^ (t[b] >> 8);  // byte b, then a zero byte
  if (cudaMemcpyToSymbol(g_crc_tab1, t1, sizeof(t1)) != cudaSuccess) return 1;
  if (cudaMemcpyToSymbol(g_seg_nib, nib, sizeof(nib)) != cudaSuccess) return 1;
  if (cudaMemcpyToSymbol(c_zpow, zpow, sizeof(zpow)) != cudaSuccess) return 1;
  if (cudaMemcpyToSymbol(c_zgroup, zg, sizeof(zg)) != cudaSuccess) return 1;
  // Z_{-p}: Z_1 is invertible (x is a unit mod the CRC polynomial); find the
  // inverse columns by solving Z_1 * v = e_j over GF(2) (Gaussian elimination).
  uint32_t inv1[32];
  {
    uint32_t m[32], rhs[32];
    for (int i = 0; i < 32; ++i) { m[i] = 0; rhs[i] = 0; }
    // row i of Z_1: bit i of each column
    for (int i = 0; i < 32; ++i)
      for (int j = 0; j < 32; ++j)
        if ((zpow[0][j] >> i) & 1) m[i] |= 1u << j;
    for (int i = 0; i < 32; ++i) rhs[i] = 1u << i;  // rhs columns packed per row: solve Z_1 X = I
    for (int col = 0; col < 32; ++col) {
      int piv = -1;
      for (int r = col; r < 32; ++r)
        if ((m[r] >> col) & 1) { piv = r; break; }
      if (piv < 0) return 1;
      std::swap(m[piv], m[col]);
      std::swap(rhs[piv], rhs[col]);
      for (int r = 0; r < 32; ++r)
        if (r != col && ((m[r] >> col) & 1)) { m[r] ^= m[col]; rhs[r] ^= rhs[col]; }
    }
    // now X = rhs as rows: X[i] row i, bit j = X(i, j); column j of X
    for (int j = 0; j < 32; ++j) {
      uint32_t c = 0;
      for (int i = 0; i < 32; ++i)
        if ((rhs[i] >> j) & 1) c |= 1u << i;
      inv1[j] = c;
    }
    for (int j = 0; j < 32; ++j)
      if (apply_cols(zpow[0], inv1[j]) != (1u << j)) return 1;
  }
  static uint32_t zinv[3][8][16];
  uint32_t cur[32];
  memcpy(cur, inv1, sizeof(cur));
  for (int p = 0; p < 3; ++p) {
    for (int nb = 0; nb < 8; ++nb)
      for (int v = 0; v < 16; ++v) zinv[p][nb][v] = apply_cols(cur, (uint32_t)v << (4 * nb));
    uint32_t next[32];
    for (int j = 0; j < 32; ++j) next[j] = apply_cols(inv1, cur[j]);
    memcpy(cur, next, sizeof(cur));
  }
  if (cudaMemcpyToSymbol(c_zinv, zinv, sizeof(zinv)) != cudaSuccess) return 1;
  static uint32_t zone[kZoneMax];
  {
    uint32_t c = 0xFFFFFFFFu;
    for (int n = 0; n < kZoneMax; ++n) {
      zone[n] = c;
      c = t[c & 0xFF] ^ (c >> 8);
    }
  }
  if (cudaMemcpyToSymbol(g_zone, zone, sizeof(zone)) != cudaSuccess) return 1;
  return 0;
}

}  // namespace luda
