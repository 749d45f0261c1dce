// luda_common.cuh — shared device utilities of the B200 LUDA compaction path.
//
// CRC-32/IEEE (reflected 0xEDB88320, init/xorout 0xFFFFFFFF; the zlib flavour
// of checksum.py:12-13) is computed warp-parallel: a byte range is cut into
// END-ALIGNED 44-byte segments (11 words). In one pass a warp covers 96
// segments (4224 B — a whole 4 KiB block plus the alignment pad, so a typical
// block is one pass with ~4% idle segments): lane d owns the segments at
// distance d, d+32, d+64 from the pass end and runs their three table chains
// interleaved (3-way ILP: the chains are latency-bound, two dependent LDS per
// word). Segment
// registers are combined with the GF(2) "advance over n zero bytes" operator
// Z_n (the crc32_combine algebra: raw(A∥B) = Z_|B|(raw(A)) ^ raw(B)), by
// Horner over the lane's chains with H = Z_1408:
//   lane value = Z_{44d}( r_d ^ H(r_{d+32} ^ H(r_{d+64})) ), XOR over lanes.
// Words go through SLICING-BY-2 tables (two 16-bit steps per word). The two
// byte tables T1 (byte then a zero byte) and T0 are replicated once per lane
// and interleaved so that one PRMT forms the whole shared-memory offset:
//   offset = idx << 8 | table << 7 | lane << 2      (64 KB, bank = lane)
// i.e. per 2 bytes: 2 PRMT + 2 LDS + SHF + LOP3, no bank conflicts.
// 11 words (odd) per segment makes the 32 lanes' LDS.32 data streams hit 32
// distinct banks. The ~0 preset is folded into the data: callers run
// crc_prep() on the smem copy (zero the 72 bytes before it, complement the
// first 4 bytes: F(~0, D) = F(0, D') and leading zeros leave a zero register
// unchanged) and crc_unprep() afterwards; the inner loop has no masking.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

// Ablation experiments (profiles/*_ablation.py) switch pipeline stages off in
// a separate -DLUDA_ABLATION build; production builds compile them out.
#ifdef LUDA_ABLATION
#define LUDA_ABLATE(args, bit) (((args).dbg & (bit)) != 0)
#else
#define LUDA_ABLATE(args, bit) false
#endif

namespace luda {

constexpr uint32_t kCrcPoly = 0xEDB88320u;
constexpr int kSeg = 44;             // bytes per CRC segment
constexpr int kSegWords = kSeg / 4;  // 11 (odd: the lanes' word streams hit distinct banks)
constexpr int kChains = 3;           // segments (independent table chains) per lane per pass
constexpr int kHalf = 32 * kSeg;     // 1408: distance between a lane's consecutive segments
constexpr int kGroup = 32 * kChains * kSeg;  // 4224: bytes one warp covers per pass (>= a 4 KiB block + pad)
constexpr int kCrcLead = 72;         // zeroed bytes required before the data

// ---- tables (device globals; initialised by luda_init) ---------------------
// g_crc_tab[b]          : byte table T0[b]
// g_crc_tab1[b]         : T1[b] = T0 advanced over one more (zero) byte
// g_seg_nib[n][v][d]    : Z_{44*d}(v << 4n)    (8 x 16 x 32 words)
// g_half_tab[k][b]      : Z_1408(b << 8k)     (4 x 256 words)
// c_zpow[i][j]          : Z_{2^i}(1 << j)      (48 x 32 words) for arbitrary shifts
// c_zgroup[j]           : Z_4224(1 << j)       (one warp pass)
// (single translation unit: luda_b200.cu includes every stage header)
__device__ uint32_t g_crc_tab[256];
__device__ uint32_t g_crc_tab1[256];
__device__ uint32_t g_seg_nib[8 * 16 * 32];
__device__ uint32_t g_half_tab[4 * 256];
__constant__ uint32_t c_zpow[48][32];
__constant__ uint32_t c_zgroup[32];
__constant__ uint32_t c_zinv[3][8][16];  // nibble tables of Z_{-p}, p = 1..3 (inverse shifts)
constexpr int kZoneMax = 8192;
__device__ uint32_t g_zone[kZoneMax];    // Z_n(0xFFFFFFFF): the ~0 preset advanced over n bytes

// Shared-memory CRC state: the lane-replicated slicing-by-2 tables (64 KB),
// the per-lane nibble tables of Z_{44d} (16 KB) and the Z_1408 byte tables
// (4 KB). (LUDA_CRC_SMEM_COMBINE=0 reads the two combine tables through the
// read-only path from global memory instead, freeing 20 KB of shared memory:
// measured slower — decode 4.27 → 4.55 ms on c3 — the L1 left over misses.)
#ifndef LUDA_CRC_SMEM_COMBINE
#define LUDA_CRC_SMEM_COMBINE 1
#endif
struct CrcSmem {
  uint32_t s2[256 * 64];  // row idx: [T1 lane 0..31][T0 lane 0..31]
#if LUDA_CRC_SMEM_COMBINE
  uint32_t nib[8 * 16 * 32];
  uint32_t half[4 * 256];
#endif
};

__device__ __forceinline__ void crc_smem_init(CrcSmem& s) {
  for (int i = threadIdx.x; i < 256 * 64; i += blockDim.x)
    s.s2[i] = (i & 32) ? g_crc_tab[i >> 6] : g_crc_tab1[i >> 6];
#if LUDA_CRC_SMEM_COMBINE
  for (int i = threadIdx.x; i < 8 * 16 * 32; i += blockDim.x) s.nib[i] = g_seg_nib[i];
  for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x) s.half[i] = g_half_tab[i];
#endif
}
__device__ __forceinline__ const uint32_t* crc_nib_tab(const CrcSmem& s) {
#if LUDA_CRC_SMEM_COMBINE
  return s.nib;
#else
  return g_seg_nib;
#endif
}
__device__ __forceinline__ const uint32_t* crc_half_tab(const CrcSmem& s) {
#if LUDA_CRC_SMEM_COMBINE
  return s.half;
#else
  return g_half_tab;
#endif
}
__device__ __forceinline__ uint32_t crc_tab_ld(const uint32_t* p) {
#if LUDA_CRC_SMEM_COMBINE
  return *p;
#else
  return __ldg(p);
#endif
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

// A lane's view of the slicing tables: base + the two PRMT partner words
// (byte 0 = lane << 2 | table << 7, bytes 1-3 zero).
struct CrcLane {
  const uint8_t* base;
  uint32_t a1, a0;
};
__device__ __forceinline__ CrcLane crc_lane(const CrcSmem& s, uint32_t lane) {
  return CrcLane{reinterpret_cast<const uint8_t*>(s.s2), lane << 2, (lane << 2) | 0x80u};
}
__device__ __forceinline__ uint32_t crc_lut(const CrcLane& t, uint32_t off) {
  return *reinterpret_cast<const uint32_t*>(t.base + off);
}

// One 16-bit step: x already holds crc ^ data in its low half. (x >> 16 as
// a multiply-high keeps it on the FMA pipe; PRMT/LOP3 load the ALU pipe.)
__device__ __forceinline__ uint32_t crc_half(uint32_t x, const CrcLane& t) {
  const uint32_t a = crc_lut(t, prmt(x, t.a1, 0x7604u));  // T1[x & 0xFF]
  const uint32_t b = crc_lut(t, prmt(x, t.a0, 0x7614u));  // T0[(x >> 8) & 0xFF]
  return __umulhi(x, 0x10000u) ^ a ^ b;
}

// One word through the register update (two slicing-by-2 steps).
__device__ __forceinline__ uint32_t crc_word(uint32_t c, uint32_t w, const CrcLane& t) {
  return crc_half(crc_half(c ^ w, t), t);
}

__device__ __forceinline__ uint32_t crc_byte(uint32_t c, uint32_t b, const CrcLane& t) {
  return crc_lut(t, prmt(c ^ b, t.a0, 0x7604u)) ^ (c >> 8);  // T0[(c ^ b) & 0xFF] ^ (c >> 8)
}

// Z_{44*lane}(c) via the lane's nibble tables. `nl` = s.nib + lane.
__device__ __forceinline__ uint32_t seg_shift(uint32_t c, const uint32_t* __restrict__ nl) {
  uint32_t r = 0;
#pragma unroll
  for (int n = 0; n < 8; ++n) r ^= crc_tab_ld(nl + (((n << 4) | ((c >> (4 * n)) & 0xFu)) << 5));
  return r;
}

// Z_1408(c) (byte tables).
__device__ __forceinline__ uint32_t half_shift(uint32_t c, const uint32_t* __restrict__ ht) {
  return crc_tab_ld(ht + (c & 0xFFu)) ^ crc_tab_ld(ht + 256 + ((c >> 8) & 0xFFu)) ^
         crc_tab_ld(ht + 512 + ((c >> 16) & 0xFFu)) ^ crc_tab_ld(ht + 768 + (c >> 24));
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

// Prepare / restore an smem copy of the data for crc: zero [data-72, data)
// and complement data[0..4). Whole warp; n >= 4.
__device__ __forceinline__ void crc_prep(uint8_t* data) {
  const uint32_t lane = lane_id();
  for (uint32_t i = lane; i < (uint32_t)kCrcLead; i += 32) data[(int)i - kCrcLead] = 0;
  if (lane < 4) data[lane] ^= 0xFFu;
  __syncwarp();
}
__device__ __forceinline__ void crc_unprep(uint8_t* data) {
  __syncwarp();
  if (lane_id() < 4) data[lane_id()] ^= 0xFFu;
  __syncwarp();
}

// Segment pointer at smem byte address p (any alignment): the aligned words
// covering [p, p + kSeg + 4) and the funnel shift.
struct SegPtr {
  const uint32_t* wp;
  uint32_t sh;
};
__device__ __forceinline__ SegPtr seg_ptr(const uint8_t* p) {
  // pointer arithmetic (not an integer round trip) keeps the smem address space
  const uint32_t mis = (uint32_t)(reinterpret_cast<uintptr_t>(p) & 3u);
  return SegPtr{reinterpret_cast<const uint32_t*>(p - mis), mis * 8u};
}

// Horner combine of a lane's chain registers r[0..kChains) (r[c] = segment at
// distance d + 32c), then the lane's Z_{36d}.
__device__ __forceinline__ uint32_t lane_combine(const uint32_t (&r)[kChains], const CrcSmem& cs, uint32_t lane) {
  uint32_t v = r[kChains - 1];
#pragma unroll
  for (int c = kChains - 2; c >= 0; --c) v = half_shift(v, crc_half_tab(cs)) ^ r[c];
  return seg_shift(v, crc_nib_tab(cs) + lane);
}

// Warp: un-combined pass value of pass q over prepared smem data of length n:
// this lane's combined chains before the cross-lane XOR, with segment
// distances d = lane + 32c + 96q (pass q covers distances [96q, 96q+96)).
__device__ __forceinline__ uint32_t pass_lane_value(const uint8_t* data, uint64_t n, uint32_t q, const CrcSmem& cs,
                                                    const uint8_t* safe) {
  const uint32_t lane = lane_id();
  const CrcLane tl = crc_lane(cs, lane);
  const int64_t nseg = ((int64_t)n + kSeg - 1) / kSeg;
  SegPtr sp[kChains];
  bool val[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    const int64_t dd = (int64_t)lane + 32 * c + 32 * kChains * (int64_t)q;
    val[c] = dd < nseg;
    sp[c] = seg_ptr(val[c] ? data + ((int64_t)n - (int64_t)kSeg * (dd + 1)) : safe);  // `safe`: any readable smem
  }
  uint32_t r[kChains], lo[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    r[c] = 0;
    lo[c] = sp[c].wp[0];
  }
#pragma unroll
  for (int j = 0; j < kSegWords; ++j) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      const uint32_t hi = sp[c].wp[j + 1];
      r[c] = crc_word(r[c], __funnelshift_r(lo[c], hi, sp[c].sh), tl);
      lo[c] = hi;
    }
  }
#pragma unroll
  for (int c = 0; c < kChains; ++c) r[c] = val[c] ? r[c] : 0u;
  return lane_combine(r, cs, lane);
}

__device__ __forceinline__ uint32_t warp_xor(uint32_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v ^= __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}

// Z_{-p}(c), p in 1..3, warp-uniform p and c (constant-memory broadcast).
__device__ __forceinline__ uint32_t crc_unshift(uint32_t c, uint32_t p) {
  uint32_t r = 0;
#pragma unroll
  for (int n = 0; n < 8; ++n) r ^= c_zinv[p - 1][n][(c >> (4 * n)) & 0xFu];
  return r;
}

// Z_n(~0) (the preset's contribution to the raw register after n bytes).
__device__ __forceinline__ uint32_t crc_zone(uint32_t n) {
  return n < (uint32_t)kZoneMax ? g_zone[n] : crc_shift(0xFFFFFFFFu, n);
}

// WORD-ALIGNED variant of pass_lane_value: `end` is 4-byte aligned, so every
// segment is whole words (no funnel shifts). n = bytes covered before `end`.
__device__ __forceinline__ uint32_t pass_lane_value_al(const uint8_t* end, uint32_t n, uint32_t q, const CrcSmem& cs) {
  const uint32_t lane = lane_id();
  const CrcLane tl = crc_lane(cs, lane);
  const int32_t nseg = ((int32_t)n + kSeg - 1) / kSeg;
  const uint32_t* p[kChains];
  bool val[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    const int32_t dd = (int32_t)lane + 32 * c + 32 * kChains * (int32_t)q;
    val[c] = dd < nseg;
    p[c] = reinterpret_cast<const uint32_t*>(end - kSeg * (val[c] ? dd + 1 : 1));
  }
  uint32_t r[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) r[c] = 0;
#pragma unroll
  for (int j = 0; j < kSegWords; ++j) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) r[c] = crc_word(r[c], p[c][j], tl);
  }
#pragma unroll
  for (int c = 0; c < kChains; ++c) r[c] = val[c] ? r[c] : 0u;
  return lane_combine(r, cs, lane);
}

// Warp-cooperative CRC-32 of n >= 4 bytes of PREPARED smem data (crc_prep).
// All 32 lanes call; every lane returns the final CRC.
__device__ __forceinline__ uint32_t warp_crc32_prepped(const uint8_t* data, uint32_t n, const CrcSmem& cs) {
  const uint32_t npass = (n + kGroup - 1) / kGroup;
  uint32_t acc = 0;
  for (int q = (int)npass - 1; q >= 0; --q) {
    const uint32_t v = warp_xor(pass_lane_value(data, n, (uint32_t)q, cs, data));
    acc = (q == (int)npass - 1) ? v : (gf2_apply(c_zgroup, acc) ^ v);
  }
  return ~acc;
}

// Warp CRC-32 of n >= 4 bytes of smem data (72 writable bytes before it, 3
// after it). The range is extended with zero bytes to a word-aligned end so
// every segment is whole words; raw(D ∥ 0^p) = Z_p(raw(D)) is undone with
// Z_{-p}. All modified bytes are restored.
__device__ __forceinline__ uint32_t warp_crc32_smem(uint8_t* data, uint32_t n, const CrcSmem& cs) {
  const uint32_t lane = lane_id();
  const uint32_t pad = (uint32_t)(0u - (uint32_t)reinterpret_cast<uintptr_t>(data + n)) & 3u;
  uint8_t saved = 0;
  if (lane < pad) saved = data[n + lane];
  __syncwarp();
  crc_prep(data);  // (syncs)
  if (lane < pad) data[n + lane] = 0;
  __syncwarp();
  const uint32_t m = n + pad;
  const uint8_t* end = data + m;
  const uint32_t npass = (m + kGroup - 1) / kGroup;
  uint32_t acc = 0;
  for (int q = (int)npass - 1; q >= 0; --q) {
    const uint32_t v = warp_xor(pass_lane_value_al(end, m, (uint32_t)q, cs));
    acc = (q == (int)npass - 1) ? v : (gf2_apply(c_zgroup, acc) ^ v);
  }
  __syncwarp();
  if (lane < pad) data[n + lane] = saved;
  crc_unprep(data);
  return ~(pad ? crc_unshift(acc, pad) : acc);
}

// Scalar CRC (any n) for tiny ranges; `tl` = table view of the calling lane.
__device__ __forceinline__ uint32_t crc32_bytes(const uint8_t* p, uint32_t n, const CrcLane& tl) {
  uint32_t c = 0xFFFFFFFFu;
  for (uint32_t i = 0; i < n; ++i) c = crc_byte(c, p[i], tl);
  return ~c;
}

// ---- per-thread async copies (cp.async, LDGSTS): global → smem without registers ----
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem_dst)),
               "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(smem_dst)),
               "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

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
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// try_wait with a suspend-time hint: a waiting warp is parked (no issue slots
// spent spinning) until the phase completes or the hint elapses.
constexpr uint32_t kMbarSuspendNs = 20000;
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred P1;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      " @!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(kMbarSuspendNs)
      : "memory");
}
// smem → global bulk copy (TMA store; 16-byte aligned addresses and size),
// tracked by the issuing thread's bulk async-group.
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"((uint32_t)__cvta_generic_to_shared(ssrc)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// the smem source of every committed bulk store has been read (buffer reusable)
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// every committed bulk store is complete (its global writes performed)
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Order this thread's earlier generic-proxy smem accesses before later
// async-proxy (TMA) accesses to the same smem.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Warp copy of n bytes between two shared-memory buffers of any alignment:
// lanes own destination-aligned words (funnel-shifted from the source);
// the two partial edge words are read-modify-written (callers guarantee no
// other thread writes those words concurrently). Reads [src-3, src+n+4).
__device__ __forceinline__ void warp_smem_copy(uint8_t* dst, const uint8_t* src, uint32_t n, uint32_t lane) {
  if (n == 0) return;
  // pointer arithmetic only (no integer round trips) so smem stays LDS/STS
  const uint32_t dmis = (uint32_t)(reinterpret_cast<uintptr_t>(dst) & 3u);
  uint32_t* dw = reinterpret_cast<uint32_t*>(dst - dmis);
  const uint32_t nw = (dmis + n + 3) >> 2;
  const uint8_t* s0 = src - dmis;  // source byte for dst word 0, byte 0
  const uint32_t smis = (uint32_t)(reinterpret_cast<uintptr_t>(s0) & 3u);
  const uint32_t* sw = reinterpret_cast<const uint32_t*>(s0 - smis);
  const uint32_t sh = smis * 8u;
  for (uint32_t w = lane; w < nw; w += 32) {
    const uint32_t v = __funnelshift_r(sw[w], sw[w + 1], sh);
    const uint32_t lo = w == 0 ? dmis : 0u;
    const uint32_t hi = (4 * w + 4 > dmis + n) ? (dmis + n - 4 * w) : 4u;
    if (lo == 0 && hi == 4) {
      dw[w] = v;
    } else {
      const uint32_t m = (hi == 4 ? 0xFFFFFFFFu : ((1u << (8 * hi)) - 1u)) & ~((1u << (8 * lo)) - 1u);
      dw[w] = (dw[w] & ~m) | (v & m);
    }
  }
}

// ---- small helpers ------------------------------------------------------------
// 4 bytes at any address (smem or global): two aligned words + byte funnel.
__device__ __forceinline__ uint32_t ld_u32_any(const uint8_t* p) {
  const uint32_t mis = (uint32_t)(reinterpret_cast<uintptr_t>(p) & 3u);
  const uint32_t* wp = reinterpret_cast<const uint32_t*>(p - mis);
  uint32_t r;
  asm("prmt.b32.f4e %0, %1, %2, %3;" : "=r"(r) : "r"(wp[0]), "r"(wp[1]), "r"(mis));
  return r;
}

// Little-endian word i of a byte string: mask of its bytes at index >= v.
__device__ __forceinline__ uint32_t byte_keep_mask(uint32_t v, int i) {
  const int32_t sh = (int32_t)(8 * v) - 32 * i;
  return __funnelshift_lc(0u, 0xFFFFFFFFu, (uint32_t)(sh > 0 ? sh : 0));
}

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

// Warp copy of up to 32 (src, dst, n) ranges (one per lane; n = 0 for idle
// lanes; base_dst and base_src 16-byte aligned, src in smem, dst smem or
// global), any alignments. Pass 1 (branch-free): the INTERIOR 16-byte
// destination chunks of all ranges, flattened over lanes through a
// chunk→range map; each is realigned from two LDS.128 with funnel shifts and
// written with one STS.128. Pass 2: the <= 2 partial edge chunks per range,
// one per lane, written per word (partial words read-modify-written —
// distinct ranges are >= 12 bytes apart so they never share a word).
// `scratch` = smem of 512 + kCopyMap bytes; the interior chunk count of one
// call must be <= kCopyMap (callers bound it by their staging size). Source
// windows must be readable 16 bytes beyond each range.
constexpr int kCopyMap = 512;
__device__ __forceinline__ void copy_chunk16(uint8_t* base_dst, const uint8_t* base_src, uint32_t dchunk,
                                             int32_t sstart, uint32_t& v0, uint32_t& v1, uint32_t& v2,
                                             uint32_t& v3) {
  const uint32_t o = (uint32_t)sstart & 15u;
  const uint4* sp = reinterpret_cast<const uint4*>(base_src + (sstart - (int32_t)o));
  const uint4 A = sp[0], B = sp[1];
  const uint32_t w[8] = {A.x, A.y, A.z, A.w, B.x, B.y, B.z, B.w};
  const uint32_t q = o >> 2, sh = (o & 3u) * 8u;
  uint32_t x[6], y[5];
#pragma unroll
  for (int k = 0; k < 6; ++k) x[k] = (q & 2u) ? w[k + 2] : w[k];
#pragma unroll
  for (int k = 0; k < 5; ++k) y[k] = (q & 1u) ? x[k + 1] : x[k];
  v0 = __funnelshift_r(y[0], y[1], sh);
  v1 = __funnelshift_r(y[1], y[2], sh);
  v2 = __funnelshift_r(y[2], y[3], sh);
  v3 = __funnelshift_r(y[3], y[4], sh);
}

// Per-lane copy of one range src → dst (both in smem; 16-aligned bases, any
// offsets): every destination 16-byte chunk the range touches is realigned
// from two aligned LDS.128; interior chunks are one STS.128, the <= 2 partial
// edge chunks are written per word (partial words read-modify-written — the
// caller guarantees no other lane writes those words concurrently). Source
// windows must be readable 16 bytes beyond the range.
__device__ __forceinline__ void lane_copy16(uint8_t* base_dst, const uint8_t* base_src, uint32_t dst_off,
                                            uint32_t src_off, uint32_t n) {
  if (n == 0) return;
  const uint32_t c_lo = dst_off & ~15u, c_hi = (dst_off + n + 15) & ~15u;
  for (uint32_t dchunk = c_lo; dchunk < c_hi; dchunk += 16) {
    const int32_t sstart = (int32_t)(src_off + dchunk) - (int32_t)dst_off;
    uint32_t v[4];
    copy_chunk16(base_dst, base_src, dchunk, sstart, v[0], v[1], v[2], v[3]);
    const uint32_t lo = dchunk < dst_off ? dst_off - dchunk : 0u;
    const uint32_t hi = (dchunk + 16 > dst_off + n) ? dst_off + n - dchunk : 16u;
    if (lo == 0 && hi == 16) {
      *reinterpret_cast<uint4*>(base_dst + dchunk) = make_uint4(v[0], v[1], v[2], v[3]);
    } else {
      uint32_t* dw = reinterpret_cast<uint32_t*>(base_dst + dchunk);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int32_t a = (int32_t)lo - 4 * k, b = (int32_t)hi - 4 * k;  // valid bytes [a, b) of word k
        if (b <= 0 || a >= 4) continue;
        const uint32_t m =
            (b >= 4 ? 0xFFFFFFFFu : ((1u << (8 * b)) - 1u)) & (a <= 0 ? 0xFFFFFFFFu : ~((1u << (8 * a)) - 1u));
        dw[k] = m == 0xFFFFFFFFu ? v[k] : ((dw[k] & ~m) | (v[k] & m));
      }
    }
  }
}

// lane_copy16 for an entry's value inside an assembled block: the source
// chunk is carried between iterations (one LDS.128 per destination chunk),
// and the two edge words are completed from registers instead of being
// read-modified-written: bytes below the value in its first word are the
// entry's own prefix (`head`, when use_head), bytes above the value in its last
// word are the next entry's first prefix word (`tail`, when use_tail). The
// edge words are composed once, outside the chunk loop; other partial words
// are read-modified-written.
__device__ __forceinline__ void value_copy16(uint8_t* base_dst, const uint8_t* base_src, uint32_t dst_off,
                                             uint32_t src_off, uint32_t n, uint32_t head, bool use_head,
                                             uint32_t tail, bool use_tail) {
  if (n == 0) return;
  const uint32_t end = dst_off + n;
  const uint32_t hw = dst_off & ~3u, tw = (end - 1) & ~3u;
  const uint32_t ha = dst_off & 3u, ta = end & 3u;
  const bool do_head = use_head && ha != 0;
  const bool do_tail = use_tail && ta != 0;
  const bool one = hw == tw;  // the value sits inside one word
  // chunk loop over [lo_all, hi_all)
  const uint32_t lo_all = do_head ? hw + 4 : dst_off;
  const uint32_t hi_all = do_tail ? tw : end;
  if (lo_all < hi_all) {
    const uint32_t c_lo = lo_all & ~15u, c_hi = (hi_all + 15) & ~15u;
    const int32_t s0 = (int32_t)src_off + (int32_t)c_lo - (int32_t)dst_off;  // source of byte c_lo
    const uint32_t o = (uint32_t)s0 & 15u;
    const uint4* sp = reinterpret_cast<const uint4*>(base_src + (s0 - (int32_t)o));
    const uint32_t q = o >> 2, sh = (o & 3u) * 8u;
    uint4 A = sp[0];
    uint32_t i = 1;
    for (uint32_t dchunk = c_lo; dchunk < c_hi; dchunk += 16, ++i) {
      const uint4 B = sp[i];
      const uint32_t w[8] = {A.x, A.y, A.z, A.w, B.x, B.y, B.z, B.w};
      A = B;
      uint32_t x[6], y[5], v[4];
#pragma unroll
      for (int k = 0; k < 6; ++k) x[k] = (q & 2u) ? w[k + 2] : w[k];
#pragma unroll
      for (int k = 0; k < 5; ++k) y[k] = (q & 1u) ? x[k + 1] : x[k];
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] = __funnelshift_r(y[k], y[k + 1], sh);
      const uint32_t lo = dchunk < lo_all ? lo_all - dchunk : 0u;
      const uint32_t hi = (dchunk + 16 > hi_all) ? hi_all - dchunk : 16u;
      if (lo == 0 && hi == 16) {
        *reinterpret_cast<uint4*>(base_dst + dchunk) = make_uint4(v[0], v[1], v[2], v[3]);
      } else {
        uint32_t* dw = reinterpret_cast<uint32_t*>(base_dst + dchunk);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int32_t a = (int32_t)lo - 4 * k, b = (int32_t)hi - 4 * k;  // bytes [a, b) of word k
          if (b <= 0 || a >= 4) continue;
          const uint32_t m =
              (b >= 4 ? 0xFFFFFFFFu : ((1u << (8 * b)) - 1u)) & (a <= 0 ? 0xFFFFFFFFu : ~((1u << (8 * a)) - 1u));
          dw[k] = m == 0xFFFFFFFFu ? v[k] : ((dw[k] & ~m) | (v[k] & m));
        }
      }
    }
  }
  // edge words
  const uint32_t tmask = ta ? (1u << (8 * ta)) - 1u : 0xFFFFFFFFu;  // bytes below the value end (tail word)
  if (do_head) {
    const uint32_t hmask = 0xFFFFFFFFu << (8 * ha);  // value bytes and above
    uint32_t v = (head & ~hmask) | ((ld_u32_any(base_src + src_off) << (8 * ha)) & hmask);
    uint32_t* p = reinterpret_cast<uint32_t*>(base_dst + hw);
    if (one && ta) {
      if (do_tail) *p = (v & tmask) | (tail & ~tmask);
      else *p = (v & tmask) | (*p & ~tmask);
    } else {
      *p = v;
    }
  }
  if (do_tail && !(do_head && one)) {
    uint32_t v = ld_u32_any(base_src + src_off + (tw - dst_off));
    uint32_t* p = reinterpret_cast<uint32_t*>(base_dst + tw);
    if (one && ha) {  // value starts inside this word too, below it is not ours
      v = ld_u32_any(base_src + src_off) << (8 * ha);
      const uint32_t m = 0xFFFFFFFFu << (8 * ha);
      *p = (*p & ~m) | (((v & tmask) | (tail & ~tmask)) & m);
    } else {
      *p = (v & tmask) | (tail & ~tmask);
    }
  }
}

// value_copy16 for a value shared by G lanes (few, large values per block —
// BASELINE c4 256-byte values, c2 1 KiB values): this lane writes destination
// chunks sub, sub+G, sub+2G, ... of [dst_off, dst_off+n), each realigned
// from two aligned LDS.128; partial words are read-modified-written (a value's
// edge words never share a word with another value's).
__device__ __forceinline__ void value_copy16_strided(uint8_t* base_dst, const uint8_t* base_src, uint32_t dst_off,
                                                     uint32_t src_off, uint32_t n, uint32_t sub, uint32_t G) {
  if (n == 0) return;
  const uint32_t end = dst_off + n;
  const uint32_t c_lo = dst_off & ~15u, c_hi = (end + 15) & ~15u;
  const int32_t s0 = (int32_t)src_off - (int32_t)(dst_off - c_lo);  // source of byte c_lo
  const uint32_t o = (uint32_t)s0 & 15u;
  const uint8_t* sbase = base_src + (s0 - (int32_t)o);
  const uint32_t q = o >> 2, sh = (o & 3u) * 8u;
  for (uint32_t dchunk = c_lo + 16 * sub; dchunk < c_hi; dchunk += 16 * G) {
    const uint4* sp = reinterpret_cast<const uint4*>(sbase + (dchunk - c_lo));
    const uint4 A = sp[0], B = sp[1];
    const uint32_t w[8] = {A.x, A.y, A.z, A.w, B.x, B.y, B.z, B.w};
    uint32_t x[6], y[5], v[4];
#pragma unroll
    for (int k = 0; k < 6; ++k) x[k] = (q & 2u) ? w[k + 2] : w[k];
#pragma unroll
    for (int k = 0; k < 5; ++k) y[k] = (q & 1u) ? x[k + 1] : x[k];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = __funnelshift_r(y[k], y[k + 1], sh);
    const uint32_t lo = dchunk < dst_off ? dst_off - dchunk : 0u;
    const uint32_t hi = (dchunk + 16 > end) ? end - dchunk : 16u;
    if (lo == 0 && hi == 16) {
      *reinterpret_cast<uint4*>(base_dst + dchunk) = make_uint4(v[0], v[1], v[2], v[3]);
    } else {
      uint32_t* dw = reinterpret_cast<uint32_t*>(base_dst + dchunk);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int32_t a = (int32_t)lo - 4 * k, b = (int32_t)hi - 4 * k;  // bytes [a, b) of word k
        if (b <= 0 || a >= 4) continue;
        const uint32_t m =
            (b >= 4 ? 0xFFFFFFFFu : ((1u << (8 * b)) - 1u)) & (a <= 0 ? 0xFFFFFFFFu : ~((1u << (8 * a)) - 1u));
        dw[k] = m == 0xFFFFFFFFu ? v[k] : ((dw[k] & ~m) | (v[k] & m));
      }
    }
  }
}

__device__ __forceinline__ void warp_copy_ranges16(uint8_t* base_dst, const uint8_t* base_src, uint32_t dst_off,
                                                   uint32_t src_off, uint32_t n, uint32_t* scratch) {
  const uint32_t lane = lane_id();
  uint32_t* rd = scratch;          // [32] dst offsets
  uint32_t* rs = scratch + 32;     // [32] src offsets
  uint32_t* rn = scratch + 64;     // [32] lengths
  uint32_t* rf = scratch + 96;     // [32] first flattened interior chunk of each range
  uint8_t* map = reinterpret_cast<uint8_t*>(scratch + 128);  // [kCopyMap] interior chunk → range
  const uint32_t c0 = (dst_off + 15) & ~15u;             // first interior chunk (offset)
  const uint32_t c1 = (dst_off + n) & ~15u;              // end of interior chunks
  const uint32_t nint = (n && c1 > c0) ? (c1 - c0) >> 4 : 0u;
  const uint32_t incl = warp_incl_scan<uint32_t>(nint);
  const uint32_t total = __shfl_sync(0xFFFFFFFFu, incl, 31);
  rd[lane] = dst_off;
  rs[lane] = src_off;
  rn[lane] = n;
  rf[lane] = incl - nint;
  for (uint32_t i = incl - nint; i < incl; ++i) map[i] = (uint8_t)lane;  // total <= kCopyMap (staging bound)
  __syncwarp();
  // pass 1: interior chunks, branch-free
  for (uint32_t t = lane; t < total; t += 32) {
    const uint32_t j = map[t];
    const uint32_t dj = rd[j], sj = rs[j];
    const uint32_t dchunk = ((dj + 15) & ~15u) + 16u * (t - rf[j]);
    const int32_t sstart = (int32_t)(sj + dchunk) - (int32_t)dj;
    uint32_t v0, v1, v2, v3;
    copy_chunk16(base_dst, base_src, dchunk, sstart, v0, v1, v2, v3);
    *reinterpret_cast<uint4*>(base_dst + dchunk) = make_uint4(v0, v1, v2, v3);
  }
  // pass 2: edge chunks: lane e → range e>>1, side e&1 (head / tail)
  for (uint32_t e = lane; e < 64; e += 32) {
    const uint32_t j = e >> 1;
    const uint32_t dj = rd[j], sj = rs[j], nj = rn[j];
    if (nj == 0) continue;
    const uint32_t head = (dj & ~15u);
    const uint32_t tail = (dj + nj - 1) & ~15u;
    uint32_t dchunk;
    if ((e & 1) == 0) {
      if ((dj & 15u) == 0 && (dj + nj >= head + 16)) continue;  // head chunk fully interior
      dchunk = head;
    } else {
      if (tail == head) continue;                                 // single chunk: done by the head lane
      if (((dj + nj) & 15u) == 0) continue;                       // tail chunk fully interior
      dchunk = tail;
    }
    const int32_t sstart = (int32_t)(sj + dchunk) - (int32_t)dj;
    uint32_t v[4];
    copy_chunk16(base_dst, base_src, dchunk, sstart, v[0], v[1], v[2], v[3]);
    const uint32_t lo = dchunk < dj ? dj - dchunk : 0u;
    const uint32_t hi = (dchunk + 16 > dj + nj) ? dj + nj - dchunk : 16u;
    uint32_t* dw = reinterpret_cast<uint32_t*>(base_dst + dchunk);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int32_t a = (int32_t)lo - 4 * k, b = (int32_t)hi - 4 * k;  // valid bytes [a, b) of word k
      if (b <= 0 || a >= 4) continue;
      const uint32_t m =
          (b >= 4 ? 0xFFFFFFFFu : ((1u << (8 * b)) - 1u)) & (a <= 0 ? 0xFFFFFFFFu : ~((1u << (8 * a)) - 1u));
      dw[k] = m == 0xFFFFFFFFu ? v[k] : ((dw[k] & ~m) | (v[k] & m));
    }
  }
  __syncwarp();
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
