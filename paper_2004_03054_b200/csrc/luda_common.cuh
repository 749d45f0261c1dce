// luda_common.cuh — shared device utilities of the B200 LUDA compaction path.
//
// CRC-32/IEEE (reflected 0xEDB88320, init/xorout 0xFFFFFFFF; the zlib flavour
// of checksum.py:12-13) is computed warp-parallel: a byte range is cut into
// END-ALIGNED 132-byte segments (33 words), lane d owning the segment that ends
// 132*d bytes before the range end. Each lane computes the raw CRC register of
// its segment with a bank-replicated byte table in shared memory, and the
// segments are combined with the GF(2) "advance over n zero bytes" operator
// Z_n (the crc32_combine algebra): raw(A∥B) = Z_|B|(raw(A)) ^ raw(B).
// 132 (not 128) makes the 32 lanes' LDS.32 streams hit 32 distinct banks.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace luda {

constexpr uint32_t kCrcPoly = 0xEDB88320u;
constexpr int kSeg = 132;           // bytes per CRC segment
constexpr int kSegWords = kSeg / 4; // 33
constexpr int kGroup = kSeg * 32;   // bytes one warp covers per pass (4224)

// ---- tables (device globals; initialised by luda_init) ---------------------
// g_crc_tab[b]          : byte table T[b]
// g_seg_nib[n][v][d]    : Z_{132*d}(v << 4n)   (8 x 16 x 32 words)
// g_zpow[i][j]          : Z_{2^i}(1 << j)      (48 x 32 words) for arbitrary shifts
// (single translation unit: luda_b200.cu includes every stage header)
__device__ uint32_t g_crc_tab[256];
__device__ uint32_t g_seg_nib[8 * 16 * 32];
__constant__ uint32_t c_zpow[48][32];
__constant__ uint32_t c_zgroup[32]; // Z_{4224}(1<<j)

// Shared-memory CRC state: 32 bank-replicated copies of T (32 KB) + the
// per-lane nibble tables (16 KB). Lane l reads tab[(idx<<5)|l] → bank l.
struct CrcSmem {
  uint32_t tab[256 * 32];
  uint32_t nib[8 * 16 * 32];
};

__device__ __forceinline__ void crc_smem_init(CrcSmem& s) {
  for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) s.tab[i] = g_crc_tab[i >> 5];
  for (int i = threadIdx.x; i < 8 * 16 * 32; i += blockDim.x) s.nib[i] = g_seg_nib[i];
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

// One word through the byte-table register update (4 dependent lookups).
// `tl` = s.tab + lane.
__device__ __forceinline__ uint32_t crc_word(uint32_t c, uint32_t w, const uint32_t* __restrict__ tl) {
  c ^= w;
  c = tl[(c & 0xFFu) << 5] ^ (c >> 8);
  c = tl[(c & 0xFFu) << 5] ^ (c >> 8);
  c = tl[(c & 0xFFu) << 5] ^ (c >> 8);
  c = tl[(c & 0xFFu) << 5] ^ (c >> 8);
  return c;
}

__device__ __forceinline__ uint32_t crc_byte(uint32_t c, uint32_t b, const uint32_t* __restrict__ tl) {
  return tl[((c ^ b) & 0xFFu) << 5] ^ (c >> 8);
}

// Z_{132*lane}(c) via the lane's nibble tables. `nl` = s.nib + lane.
__device__ __forceinline__ uint32_t seg_shift(uint32_t c, const uint32_t* __restrict__ nl) {
  uint32_t r = 0;
#pragma unroll
  for (int n = 0; n < 8; ++n) r ^= nl[((n << 4) | ((c >> (4 * n)) & 0xFu)) << 5];
  return r;
}

// Apply a 32x32 GF(2) operator given by its columns (constant memory; the
// whole warp must use the same operator so reads broadcast).
__device__ __forceinline__ uint32_t gf2_apply(const uint32_t* op, uint32_t c) {
  uint32_t r = 0;
#pragma unroll
  for (int j = 0; j < 32; ++j) r ^= (0u - ((c >> j) & 1u)) & op[j];
  return r;
}

// Z_n(c) for arbitrary n (bytes) by binary decomposition (warp-uniform n).
__device__ __forceinline__ uint32_t crc_shift(uint32_t c, uint64_t n) {
  for (int i = 0; n != 0 && i < 48; ++i, n >>= 1)
    if (n & 1) c = gf2_apply(c_zpow[i], c);
  return c;
}

// Raw CRC register over 33 words of shared memory starting at byte address p
// (may be unaligned; reads the aligned words covering it). Bytes whose
// data-index (idx0 + k) is < 0 are replaced by zero and bytes with index in
// [0,4) are complemented: F(~0, D) = F(0, D with its first 4 bytes inverted)
// and leading zero bytes leave a zero register unchanged, so the preset folds
// into the data (requires n >= 4). The smem window [p, p+136) must be readable.
__device__ __forceinline__ uint32_t seg_crc_smem(const uint8_t* p, int64_t idx0,
                                                 const uint32_t* __restrict__ tl) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const uint32_t* wp = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
  const uint32_t sh = (uint32_t)(a & 3u) * 8u;
  uint32_t c = 0;
  uint32_t lo = wp[0];
#pragma unroll 11
  for (int j = 0; j < kSegWords; ++j) {
    uint32_t hi = wp[j + 1];
    uint32_t w = __funnelshift_r(lo, hi, sh);
    lo = hi;
    int64_t bi = idx0 + 4 * j;  // data index of byte 0 of this word
    if (bi < 4) {               // only the leading words of the first segment
      uint32_t keep = 0, inv = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        int64_t d = bi + k;
        if (d >= 0) keep |= 0xFFu << (8 * k);
        if (d >= 0 && d < 4) inv |= 0xFFu << (8 * k);
      }
      w = (w & keep) ^ inv;
    }
    c = crc_word(c, w, tl);
  }
  return c;
}

// Warp-cooperative CRC-32 of `n` bytes at shared address `data` (n >= 4).
// All 32 lanes must call; every lane returns the final CRC. Requires the smem
// window [data - kSeg - 4, data + n + 8) to be readable (callers pad).
__device__ __forceinline__ uint32_t warp_crc32_smem(const uint8_t* data, uint32_t n, const CrcSmem& s) {
  const uint32_t lane = lane_id();
  const uint32_t* tl = s.tab + lane;
  const uint32_t* nl = s.nib + lane;
  const int64_t nseg = (int64_t)((n + kSeg - 1) / kSeg);
  const int64_t npass = (nseg + 31) / 32;
  uint32_t acc = 0;
  for (int64_t q = npass - 1; q >= 0; --q) {
    const int64_t d = (int64_t)lane + 32 * q;  // segment distance from the end
    uint32_t r = 0;
    if (d < nseg) {
      int64_t start = (int64_t)n - (int64_t)kSeg * (d + 1);  // may be negative (first segment)
      r = seg_crc_smem(data + start, start, tl);
    }
    if (q != npass - 1) acc = gf2_apply(c_zgroup, acc);
    acc ^= r;
  }
  acc = seg_shift(acc, nl);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc ^= __shfl_xor_sync(0xFFFFFFFFu, acc, o);
  return ~acc;
}

// Scalar CRC (any n) for tiny ranges; `tl` = table row of the calling lane.
__device__ __forceinline__ uint32_t crc32_bytes(const uint8_t* p, uint32_t n, const uint32_t* tl) {
  uint32_t c = 0xFFFFFFFFu;
  for (uint32_t i = 0; i < n; ++i) c = crc_byte(c, p[i], tl);
  return ~c;
}

// ---- small helpers ------------------------------------------------------------
__device__ __forceinline__ uint32_t varint_size(uint64_t v) {
  uint32_t n = 1;
  while (v >= 0x80) { v >>= 7; ++n; }
  return n;
}

__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T u = __shfl_up_sync(0xFFFFFFFFu, v, o);
    if (lane >= (uint32_t)o) v += u;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T u = __shfl_xor_sync(0xFFFFFFFFu, v, o);
    v = u > v ? u : v;
  }
  return v;
}

// ---- decoupled look-back (single-pass prefix over tiles) ----------------------
// status word: bits 62-63 flag (1 = aggregate, 2 = inclusive), low 62 bits value.
constexpr uint64_t kLbAgg = 1ull << 62;
constexpr uint64_t kLbInc = 2ull << 62;
constexpr uint64_t kLbMask = (1ull << 62) - 1;

__device__ __forceinline__ void lb_publish(uint64_t* st, uint64_t tile, uint64_t flag, uint64_t v) {
  __threadfence();
  atomicExch(reinterpret_cast<unsigned long long*>(st + tile), (unsigned long long)(flag | v));
}

__device__ __forceinline__ uint64_t lb_load(const uint64_t* st, int64_t i) {
  return *reinterpret_cast<const volatile uint64_t*>(st + i);
}

// Whole warp: returns the exclusive prefix of tile `tile` (tile 0 → 0).
// The caller must have published its aggregate already.
__device__ __forceinline__ uint64_t lb_exclusive(const uint64_t* st, uint64_t tile) {
  const uint32_t lane = lane_id();
  uint64_t excl = 0;
  int64_t pos = (int64_t)tile - 1;
  while (pos >= 0) {
    int64_t i = pos - (int64_t)lane;
    uint64_t s = 0;
    uint32_t ready;
    do {
      s = (i >= 0) ? lb_load(st, i) : kLbInc;
      ready = __all_sync(0xFFFFFFFFu, (s >> 62) != 0);
    } while (!ready);
    uint32_t inc_mask = __ballot_sync(0xFFFFFFFFu, (s >> 62) == 2);
    // lanes up to and including the first inclusive one contribute
    uint32_t first_inc = inc_mask ? (uint32_t)(__ffs(inc_mask) - 1) : 32u;
    uint64_t contrib = (lane <= first_inc && i >= 0) ? (s & kLbMask) : 0;
    excl += warp_sum(contrib);
    if (inc_mask) break;
    pos -= 32;
  }
  __threadfence();
  return excl;
}

}  // namespace luda
