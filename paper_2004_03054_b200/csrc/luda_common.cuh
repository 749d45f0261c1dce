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
// data-index (idx0 + k) is < 0 are treated as zero and bytes with index in
// [0,4) are complemented: F(~0, D) = F(0, D with its first 4 bytes inverted)
// and leading zero bytes leave a zero register unchanged, so the preset folds
// into the data (requires n >= 4). Only the first segment (idx0 < 4) has such
// bytes: it skips its all-zero leading words and masks the next two, so the
// main loop carries no per-word checks. Reads the smem window [p, p+136).
__device__ __forceinline__ uint32_t seg_crc_smem(const uint8_t* p, int64_t idx0,
                                                 const uint32_t* __restrict__ tl) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const uint32_t* wp = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
  const uint32_t sh = (uint32_t)(a & 3u) * 8u;
  // first word holding a data byte, and the masks of words j0, j0+1
  int32_t j0 = 0;
  uint32_t keep0 = 0xFFFFFFFFu, inv0 = 0, keep1 = 0xFFFFFFFFu, inv1 = 0;
  if (idx0 < 4) {
    const int32_t i0 = (int32_t)idx0;  // in (-132, 4)
    j0 = i0 < 0 ? (-i0) >> 2 : 0;      // words entirely before data index 0 are zero
    const int32_t b0 = i0 + 4 * j0;    // data index of byte 0 of word j0 (in (-4, 4))
    keep0 = inv0 = keep1 = inv1 = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int32_t d0 = b0 + k, d1 = b0 + 4 + k;
      if (d0 >= 0) keep0 |= 0xFFu << (8 * k);
      if (d0 >= 0 && d0 < 4) inv0 |= 0xFFu << (8 * k);
      if (d1 >= 0) keep1 |= 0xFFu << (8 * k);
      if (d1 >= 0 && d1 < 4) inv1 |= 0xFFu << (8 * k);
    }
  }
  uint32_t c = 0;
  uint32_t lo = wp[j0];
  {
    const uint32_t hi = wp[j0 + 1];
    c = crc_word(c, (__funnelshift_r(lo, hi, sh) & keep0) ^ inv0, tl);
    lo = hi;
  }
  if (j0 + 1 < kSegWords) {
    const uint32_t hi = wp[j0 + 2];
    c = crc_word(c, (__funnelshift_r(lo, hi, sh) & keep1) ^ inv1, tl);
    lo = hi;
  }
#pragma unroll 4
  for (int32_t j = j0 + 2; j < kSegWords; ++j) {
    const uint32_t hi = wp[j + 1];
    c = crc_word(c, __funnelshift_r(lo, hi, sh), tl);
    lo = hi;
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

// ---- TMA bulk copies (cp.async.bulk) + mbarrier -----------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// 1-D bulk copy global → shared (16-byte aligned addresses, size % 16 == 0).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred P1;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Order this thread's earlier generic-proxy smem accesses before later
// async-proxy (TMA) writes to the same smem.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Warp copy of n bytes between two shared-memory buffers of any alignment:
// lanes own destination-aligned words (funnel-shifted from the source);
// the two partial edge words are read-modify-written (callers guarantee no
// other thread writes those words concurrently). Reads [src-3, src+n+4).
__device__ __forceinline__ void warp_smem_copy(uint8_t* dst, const uint8_t* src, uint32_t n, uint32_t lane) {
  if (n == 0) return;
  const uintptr_t da = reinterpret_cast<uintptr_t>(dst);
  const uintptr_t w0 = da & ~uintptr_t(3);
  const uint32_t nw = (uint32_t)((((da + n + 3) & ~uintptr_t(3)) - w0) >> 2);
  const intptr_t delta = reinterpret_cast<intptr_t>(src) - (intptr_t)da;
  for (uint32_t w = lane; w < nw; w += 32) {
    const uintptr_t A = w0 + 4ull * w;
    const uintptr_t sA = (uintptr_t)((intptr_t)A + delta);
    const uint32_t* sp = reinterpret_cast<const uint32_t*>(sA & ~uintptr_t(3));
    const uint32_t v = __funnelshift_r(sp[0], sp[1], (uint32_t)(sA & 3u) * 8u);
    const uint32_t lo = A < da ? (uint32_t)(da - A) : 0u;
    const uint32_t hi = (A + 4 > da + n) ? (uint32_t)(da + n - A) : 4u;
    uint32_t* p = reinterpret_cast<uint32_t*>(A);
    if (lo == 0 && hi == 4) {
      *p = v;
    } else {
      const uint32_t m = (hi == 4 ? 0xFFFFFFFFu : ((1u << (8 * hi)) - 1u)) & ~((1u << (8 * lo)) - 1u);
      *p = (*p & ~m) | (v & m);
    }
  }
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

// The status word is self-contained (flag + count), so no memory fence is
// needed: nothing else is communicated through the look-back.
__device__ __forceinline__ void lb_publish(uint64_t* st, uint64_t tile, uint64_t flag, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(st + tile), "l"(flag | v) : "memory");
}

__device__ __forceinline__ uint64_t lb_load(const uint64_t* st, int64_t i) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(st + i) : "memory");
  return v;
}

// Whole warp: returns the exclusive prefix of tile `tile` (tile 0 → 0).
// The caller must have published its aggregate already.
__device__ __forceinline__ uint64_t lb_exclusive(const uint64_t* st, uint64_t tile) {
  const uint32_t lane = lane_id();
  uint64_t excl = 0;
  int64_t pos = (int64_t)tile - 1;
  while (pos >= 0) {
    const int64_t i = pos - (int64_t)lane;
    uint64_t s = 0;
    uint32_t spins = 0;
    while (true) {
      s = (i >= 0) ? lb_load(st, i) : kLbInc;
      if (__all_sync(0xFFFFFFFFu, (s >> 62) != 0)) break;
      if (++spins > 2) __nanosleep(64);
    }
    const uint32_t inc_mask = __ballot_sync(0xFFFFFFFFu, (s >> 62) == 2);
    // lanes up to and including the first inclusive one contribute
    const uint32_t first_inc = inc_mask ? (uint32_t)(__ffs(inc_mask) - 1) : 32u;
    const uint64_t contrib = (lane <= first_inc && i >= 0) ? (s & kLbMask) : 0;
    excl += warp_sum(contrib);
    if (inc_mask) break;
    pos -= 32;
  }
  return excl;
}

}  // namespace luda
