// luda_encode.cuh — output SST emission.
//
// encode_kernel (warp per data block) restates assemble_block
// (blocks.py:77-103) + compute_layouts (blocks.py:41-58) — the reference's
// `shared_key` and `encode` kernel items (kernels.py:107-155) fused:
//   entry = varint shared ∥ varint unshared ∥ varint value_len ∥ key[shared:] ∥ value
//   shared = LCP with the previous key, 0 at i % restart_interval == 0
//   block = entries ∥ u32le restart offsets ∥ u32le n_restarts ∥ u32le crc
// Lanes take 32 consecutive entries: sizes → warp scan → offsets; headers and
// key suffixes are written by their lane, values are gathered straight from
// the staged input SSTs by the whole warp (one copy; the reference copies
// twice). The block is assembled in shared memory at the
// same 16-byte phase as its destination, CRC'd there and streamed out with
// 16-byte stores. Blocks larger than kEncStage are written in place.
//
// sst_meta_kernel (CTA per output SST) builds the filter block
// (bloom.py:71-88 + FilterBlock.encode :53-55: h = crc32(user_key),
// delta = rotr(h, 17), bit (h + j*delta) mod n_bits for j < k, atomicOr into
// a shared bit array), the index block (sst.py:67-76) and the footer
// (sst.py:206-208).
#pragma once
#include "luda_parse.cuh"
#include "luda_plan.cuh"
#include "luda_rec.cuh"

namespace luda {

// Default (LUDA_ENC_FUSED=1): 15 warps per SM, each builds AND finishes its
// own blocks (records, layout, value TMA, assembly, then CRC + bulk store)
// with one assembly buffer — the next block's value gather is in flight while
// the current one is CRC'd. LUDA_ENC_FUSED=0: pairs of a BUILDER warp and a
// CRC warp (CRC + copy-out) hand blocks over through two buffers. Measured on
// c3: pairs x10 3.17 ms, fused x12 3.17, x14 3.05, x15 2.89 ms (shared
// memory bounds the warp count: 84 KB CRC tables + 9.5 KB per warp).
#ifndef LUDA_ENC_FUSED
#define LUDA_ENC_FUSED 1
#endif
#ifndef LUDA_ENC_PAIRS
#define LUDA_ENC_PAIRS (LUDA_ENC_FUSED ? 15 : 10)
#endif
// LUDA_ENC_FUSED: every warp builds AND finishes (CRC + bulk store) its own
// blocks — one assembly buffer per warp instead of a builder/CRC pair with two.
constexpr bool kEncFused = LUDA_ENC_FUSED != 0;
constexpr int kEncPairs = LUDA_ENC_PAIRS;  // fused: warps
constexpr int kEncWarps = kEncFused ? kEncPairs : 2 * kEncPairs;
constexpr int kEncBufs = kEncFused ? 1 : 2;
constexpr int kEncStage = 4608;                        // blocks up to this size are assembled in smem
constexpr int kEncPre = 160;
constexpr int kEncBuf = kEncPre + 16 + kEncStage + 64;
constexpr int kEncStg = 4608;                          // per-pair TMA staging for value windows
constexpr int kEncGap = 128;                            // arena gap bridged by one value window
struct EncMeta {
  uint64_t out_off;
  uint32_t size;
  uint32_t skip;  // the builder finished the block itself (generic path)
};
struct alignas(16) EncPairSmem {
  uint8_t buf[kEncBufs][kEncBuf];
  uint8_t stg[kEncStg];
  uint64_t bar;                 // value TMA
  uint64_t full[2], empty[2];
  EncMeta meta[2];
};
// Per-CTA copy scratch of the generic (rare) block path, taken under a lock
// so the pairs need not each carry 1 KB.
struct alignas(16) EncCtaSmem {
  uint32_t pre[128 + kCopyMap / 4];  // 512 B + chunk map
  int lock;
};
static_assert(kEncStg / 16 <= kCopyMap, "copy map smaller than the staging chunk count");
static_assert(sizeof(CrcSmem) + kEncPairs * sizeof(EncPairSmem) + sizeof(EncCtaSmem) <= 232448,
              "encode smem over the 227 KB limit");
static_assert(sizeof(EncPairSmem) % 16 == 0 && kEncBuf % 16 == 0, "TMA / vector alignment");

// Copy n bytes src → dst (any alignment; dst generic: smem or global) with
// `nl` cooperating threads (rank `r`). Destination-aligned 32-bit words are
// assembled from two aligned source words; partial edge words are written
// bytewise so neighbouring data is never touched. src window [src-3, src+n+4)
// must be readable.
__device__ __forceinline__ void coop_copy(uint8_t* dst, const uint8_t* src, uint64_t n, uint32_t r, uint32_t nl) {
  if (n == 0) return;
  const uintptr_t da = reinterpret_cast<uintptr_t>(dst);
  const uintptr_t w0 = da & ~uintptr_t(3);
  const uintptr_t w1 = (da + n + 3) & ~uintptr_t(3);
  const uint64_t nw = (w1 - w0) >> 2;
  const intptr_t delta = reinterpret_cast<intptr_t>(src) - (intptr_t)da;
  for (uint64_t w = r; w < nw; w += nl) {
    const uintptr_t A = w0 + 4 * w;
    const uintptr_t sA = (uintptr_t)((intptr_t)A + delta);
    const uint32_t* sp = reinterpret_cast<const uint32_t*>(sA & ~uintptr_t(3));
    const uint32_t v = __funnelshift_r(sp[0], sp[1], (uint32_t)(sA & 3u) * 8u);
    if (A >= da && A + 4 <= da + n) {
      *reinterpret_cast<uint32_t*>(A) = v;
    } else {
#pragma unroll
      for (int b = 0; b < 4; ++b)
        if (A + b >= da && A + b < da + n) reinterpret_cast<uint8_t*>(A)[b] = (uint8_t)(v >> (8 * b));
    }
  }
}

__device__ __forceinline__ uint32_t put_varint(uint8_t* p, uint64_t v) {
  uint32_t n = 0;
  while (v >= 0x80) { p[n++] = (uint8_t)(v | 0x80); v >>= 7; }
  p[n++] = (uint8_t)v;
  return n;
}

__device__ __forceinline__ void put_u32(uint8_t* p, uint32_t v) {
  p[0] = (uint8_t)v; p[1] = (uint8_t)(v >> 8); p[2] = (uint8_t)(v >> 16); p[3] = (uint8_t)(v >> 24);
}

// Write bytes [from, K) of the internal key of r to p[0..).
template <int W>
__device__ __forceinline__ void put_key_tail(uint8_t* p, const Rec<W>& r, uint32_t L, uint32_t from) {
  constexpr int KMAX = 8 * W + 8;
  const uint64_t tr = ~r.t;
#pragma unroll
  for (int j = 0; j < KMAX; ++j) {
    if ((uint32_t)j >= from && (uint32_t)j < L + 8) {
      uint32_t byte;
      if ((uint32_t)j < L) byte = (uint32_t)(r.k[j >> 3] >> (56 - 8 * (j & 7))) & 0xFFu;
      else byte = (uint32_t)(tr >> (8 * (j - L))) & 0xFFu;
      p[j - from] = (uint8_t)byte;
    }
  }
}

// Entry prefix (varint shared ∥ varint unshared ∥ varint value_len ∥
// key[shared:]) written to smem as aligned 32-bit words instead of byte
// stores. Phase 1 (this function) writes every word except the first when the
// entry does not start on a word boundary; those bytes may belong to the
// previous entry, whose lane is writing in the same phase. The bytes past the
// prefix in its last word are placeholders: the entry's own value (written
// later with masked edges) or, for an empty value, the next entry's first
// word (written in phase 2). Returns the first word for phase 2. Requires the
// header to fit 8 bytes (shared, unshared < 128 — every key length <= 120).
template <int W>
__device__ __forceinline__ uint32_t put_prefix_words(uint8_t* D, const Rec<W>& r, uint32_t L, uint32_t s,
                                                     uint32_t vl, uint32_t hv) {
  constexpr int NK = 2 * W + 2;             // internal-key words (K <= 8W + 8)
  constexpr int NO = (8 * W + 8 + 7 + 3 + 3) / 4;  // output words: a + hv + u <= 3 + 7 + K
  constexpr int QM = (8 * W + 8 + 12) / 4;  // max word shift
  constexpr int NB = NO + 1 + QM;
  const uint32_t K = L + 8, u = K - s;
  const uint32_t a = (uint32_t)reinterpret_cast<uintptr_t>(D) & 3u;
  uint32_t kw[NK];
  rec_to_words<W, NK>(r, L, kw);
  // Z = 3 zero words ∥ key words; output word w = Z bytes [4w + c, 4w + c + 4), c = s - a - hv + 12
  const uint32_t c = s + 12u - a - hv;
  const uint32_t q = c >> 2, sh = 8u * (c & 3u);
  uint32_t B[NB];
#pragma unroll
  for (int i = 0; i < NB; ++i) B[i] = (i >= 3 && i - 3 < NK) ? kw[i - 3] : 0u;
#pragma unroll
  for (int k = 0; (1 << k) <= QM; ++k) {
    const bool take = (q >> k) & 1u;
#pragma unroll
    for (int i = 0; i < NB; ++i) B[i] = take ? (i + (1 << k) < NB ? B[i + (1 << k)] : 0u) : B[i];
  }
  // header bytes at output positions [a, a + hv)
  uint64_t H = 0;
  {
    uint32_t n = 0;
    H = (uint64_t)s | ((uint64_t)u << 8);
    n = 2;
    uint32_t v = vl;
    while (v >= 0x80u) { H |= (uint64_t)((v & 0x7Fu) | 0x80u) << (8 * n); ++n; v >>= 7; }
    H |= (uint64_t)v << (8 * n);
  }
  const uint64_t Mv = (hv >= 8) ? ~0ull : ((1ull << (8 * hv)) - 1ull);
  const uint32_t ab = 8u * a;
  const uint32_t h0 = (uint32_t)H << ab, m0 = (uint32_t)Mv << ab;
  const uint32_t h1 = ab ? (uint32_t)(H >> (32 - ab)) : (uint32_t)(H >> 32);
  const uint32_t m1 = ab ? (uint32_t)(Mv >> (32 - ab)) : (uint32_t)(Mv >> 32);
  const uint32_t h2 = ab ? (uint32_t)(H >> (64 - ab)) : 0u;
  const uint32_t m2 = ab ? (uint32_t)(Mv >> (64 - ab)) : 0u;
  const uint32_t nout = (a + hv + u + 3) >> 2;
  uint32_t* A0 = reinterpret_cast<uint32_t*>(D - a);
  uint32_t first = 0;
#pragma unroll
  for (int w = 0; w < NO; ++w) {
    uint32_t v = __funnelshift_r(B[w], B[w + 1], sh);
    if (w == 0) v = (v & ~m0) | (h0 & m0);
    if (w == 1) v = (v & ~m1) | (h1 & m1);
    if (w == 2) v = (v & ~m2) | (h2 & m2);
    if (w == 0) first = v;
    if ((uint32_t)w < nout && (w > 0 || a == 0)) A0[w] = v;
  }
  return first;
}

// Phase 2 of put_prefix_words: the shared first word, bytes [a, 4) ours.
__device__ __forceinline__ void put_prefix_first(uint8_t* D, uint32_t first) {
  const uint32_t a = (uint32_t)reinterpret_cast<uintptr_t>(D) & 3u;
  if (a == 0) return;
  uint32_t* A0 = reinterpret_cast<uint32_t*>(D - a);
  const uint32_t m = 0xFFFFFFFFu << (8 * a);
  *A0 = (*A0 & ~m) | (first & m);
}

// CTA-wide CRC-32 of smem data (passes spread over warps). All threads call;
// returns the CRC in every thread. The data needs kCrcLead writable bytes
// before it (prepared and restored here). `red` = smem scratch of >= 32 words.
__device__ __forceinline__ uint32_t cta_crc32_smem(uint8_t* data, uint32_t n, const CrcSmem& cs, uint32_t* red) {
  const uint32_t nwarps = blockDim.x >> 5, wid = threadIdx.x >> 5;
  if (n < 4) {
    if (threadIdx.x == 0) red[0] = crc32_bytes(data, n, crc_lane(cs, lane_id()));
    __syncthreads();
    const uint32_t v = red[0];
    __syncthreads();
    return v;
  }
  if (wid == 0) crc_prep(data);
  __syncthreads();
  uint32_t acc = 0;
  const uint32_t npass = (n + kGroup - 1) / kGroup;
  for (uint32_t q = wid; q < npass; q += nwarps)
    acc ^= crc_shift(warp_xor(pass_lane_value(data, n, q, cs, data)), (uint64_t)kGroup * q);
  if (lane_id() == 0) red[wid] = acc;
  __syncthreads();
  uint32_t v = 0;
  for (uint32_t w = 0; w < nwarps; ++w) v ^= red[w];
  if (wid == 0) crc_unprep(data);
  __syncthreads();
  return ~v;
}

constexpr int kMetaBufBytes = 48 * 1024;  // staging available to cta_crc32_global (sst_meta's buffer)

// CTA-wide CRC-32 of a global range, staging passes through per-warp smem.
__device__ __forceinline__ uint32_t cta_crc32_global(const uint8_t* g, uint64_t n, const CrcSmem& cs, uint8_t* stage,
                                                     uint32_t* red) {
  const uint32_t nwarps = blockDim.x >> 5, wid = threadIdx.x >> 5;
  if (n < 4) {
    if (threadIdx.x == 0) red[0] = crc32_bytes(g, (uint32_t)n, crc_lane(cs, lane_id()));
    __syncthreads();
    const uint32_t v = red[0];
    __syncthreads();
    return v;
  }
  uint32_t acc = 0;
  const uint64_t npass = (n + kGroup - 1) / kGroup;
  constexpr uint32_t kStageWarps = kMetaBufBytes / (kGroup + 192);  // warps whose staging fits `stage`
  static_assert(kStageWarps >= 1, "meta staging buffer too small");
  const uint32_t sw = nwarps < kStageWarps ? nwarps : kStageWarps;
  uint8_t* my = stage + wid * (kGroup + 192);
  if (wid < sw)
    for (uint64_t q = wid; q < npass; q += sw) acc ^= warp_crc_pass_global(g, n, q, my, cs);
  if (lane_id() == 0) red[wid] = acc;
  __syncthreads();
  uint32_t v = 0;
  for (uint32_t w = 0; w < nwarps; ++w) v ^= red[w];
  __syncthreads();
  return ~v;
}

template <int W>
struct EncodeArgs {
  const uint8_t* arena;
  const Rec<W>* rec;
  uint32_t K;
  uint32_t ri;
  uint32_t nblk;
  const uint32_t* blk_first;
  const uint32_t* blk_n;
  const uint32_t* blk_size;
  const uint64_t* blk_pos;
  const uint32_t* sst_first_blk;
  uint32_t nsst;
  const uint64_t* sst_off;
  const uint64_t* blk_out;   // output offset of every block
  uint8_t* out;
  uint32_t dbg;              // ablation switches (LUDA_ABLATION builds only)
  bool var;                  // generic-length keys: K per record, generic block path
};

// Output offset of every block: its SST's offset + its data offset in the SST.
__global__ void block_out_kernel(const uint64_t* blk_pos, uint32_t nblk, const uint32_t* sst_first_blk,
                                 uint32_t nsst, const uint64_t* sst_off, uint64_t* blk_out) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nblk) return;
  uint32_t lo = 0, hi = nsst;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (sst_first_blk[mid] <= k) lo = mid;
    else hi = mid;
  }
  blk_out[k] = sst_off[lo] + (blk_pos[k] - blk_pos[sst_first_blk[lo]]);
}

template <int W, bool kStaged>
__device__ __forceinline__ void encode_one_block(const EncodeArgs<W>& a, uint32_t k, uint64_t first, uint32_t cnt,
                                                 uint32_t size, uint64_t out_off, uint8_t* wbuf, uint8_t* stg,
                                                 uint64_t* bar, uint32_t& phase, uint32_t* pre,
                                                 const CrcSmem& cs) {
  const uint32_t lane = lane_id();
  const uint32_t K = a.K, L = K - 8, ri = a.ri;
  const uint32_t nres = (cnt + ri - 1) / ri;
  const uint32_t entries_end = size - 8 - 4 * nres;
  constexpr bool staged = kStaged;
  uint8_t* sbase = wbuf + kEncPre;
  uint8_t* dst = kStaged ? sbase + (out_off & 15) : a.out + out_off;
  uint32_t carry = 0;
  Rec<W> prev_rec;  // entry c0-1 (only used when the block has > 32 entries)
#pragma unroll
  for (int q = 0; q < W; ++q) prev_rec.k[q] = 0;
  prev_rec.t = 0;
  prev_rec.h = 0;
  for (uint32_t c0 = 0; c0 < cnt; c0 += 32) {
    const uint32_t i = c0 + lane;
    const bool act = i < cnt;
    Rec<W> r;
    if (act) r = a.rec[first + i];
    // previous record: from lane-1 (lane 0: the last record of the previous chunk)
    Rec<W> pr;
#pragma unroll
    for (int q = 0; q < W; ++q) pr.k[q] = __shfl_up_sync(0xFFFFFFFFu, r.k[q], 1);
    pr.t = __shfl_up_sync(0xFFFFFFFFu, r.t, 1);
    if (lane == 0) pr = prev_rec;
#pragma unroll
    for (int q = 0; q < W; ++q) prev_rec.k[q] = __shfl_sync(0xFFFFFFFFu, r.k[q], 31);
    prev_rec.t = __shfl_sync(0xFFFFFFFFu, r.t, 31);
    uint32_t s = 0, u = 0, vl = 0, hv = 0, esz = 0;
    uint64_t voff = 0;
    uint32_t Lr = L;
    if (act) {
      Lr = rec_ulen(r, is_var<W>(), L);
      if (i % ri != 0) s = ikey_lcp_any(pr, r, is_var<W>(), L);
      u = Lr + 8 - s;
      vl = handle_len(r.h);
      voff = handle_off(r.h);
      hv = varint_size(s) + varint_size(u) + varint_size(vl);
      esz = hv + u + vl;
    }
    const uint32_t incl = warp_incl_scan<uint32_t>(esz);
    const uint32_t off = carry + incl - esz;
    carry += __shfl_sync(0xFFFFFFFFu, incl, 31);
    if (act) {
      uint8_t* p = dst + off;
      uint32_t h = put_varint(p, s);
      h += put_varint(p + h, u);
      h += put_varint(p + h, vl);
      put_key_tail<W>(p + h, r, Lr, s);
      if (i % ri == 0) put_u32(dst + entries_end + 4 * (i / ri), off);
    }
    __syncwarp();  // headers/keys written before values (edge words are read-modified-written)
    // ---- values: TMA bulk copies of each entry's 16-byte-aligned source window
    // into the warp's staging area (all in flight at once), then realigned
    // smem→block. Windows larger than the staging area are copied directly.
    const uintptr_t vs = reinterpret_cast<uintptr_t>(a.arena) + voff;
    const uint32_t win = (act && vl) ? (uint32_t)(((vs + vl + 15) & ~uintptr_t(15)) - (vs & ~uintptr_t(15))) : 0u;
    const uint32_t dpos = off + hv + u;
    uint32_t pending = __ballot_sync(0xFFFFFFFFu, win != 0 && win <= (uint32_t)kEncStg);
    while (pending) {
      const uint32_t my = ((pending >> lane) & 1u) ? win : 0u;
      const uint32_t inc = warp_incl_scan<uint32_t>(my);
      const bool take = my != 0 && inc <= (uint32_t)kEncStg;
      const uint32_t tmask = __ballot_sync(0xFFFFFFFFu, take);
      const uint32_t total = __shfl_sync(0xFFFFFFFFu, inc, 31 - __clz(tmask));
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive_expect_tx(bar, total);
      __syncwarp();
      if (take) bulk_g2s(stg + inc - my, reinterpret_cast<const void*>(vs & ~uintptr_t(15)), my, bar);
      mbar_wait(bar, phase);
      phase ^= 1u;
      const uint32_t soff = inc - my + (uint32_t)(vs & 15u);
      warp_copy_ranges16(kStaged ? sbase : a.out + (out_off & ~15ull), stg, (uint32_t)(out_off & 15u) + dpos, soff,
                         take ? vl : 0u, pre);
      __syncwarp();
      pending &= ~tmask;
    }
    for (uint32_t m = __ballot_sync(0xFFFFFFFFu, win > (uint32_t)kEncStg); m; m &= m - 1) {
      const uint32_t j = __ffs(m) - 1;
      const uint64_t so = __shfl_sync(0xFFFFFFFFu, voff, j);
      const uint32_t sl = __shfl_sync(0xFFFFFFFFu, vl, j);
      const uint32_t dp = __shfl_sync(0xFFFFFFFFu, dpos, j);
      coop_copy(dst + dp, a.arena + so, sl, lane, 32);
    }
  }
  if (lane == 0) put_u32(dst + entries_end + 4 * nres, nres);
  __syncwarp();
  uint32_t crc;
  if (staged) {
    crc = warp_crc32_smem(dst, size - 4, cs);
  } else {
    __threadfence();
    __syncwarp();
    const uint64_t np = ((uint64_t)size - 4 + kGroup - 1) / kGroup;
    uint32_t raw = 0;
    for (uint64_t q = 0; q < np; ++q) raw ^= warp_crc_pass_global(dst, size - 4, q, wbuf, cs);
    crc = ~raw;
  }
  if (lane == 0) put_u32(dst + size - 4, crc);
  __syncwarp();
  if (staged) {
    const uintptr_t g = reinterpret_cast<uintptr_t>(a.out + out_off);
    const uintptr_t g0 = g & ~uintptr_t(15), g1 = (g + size + 15) & ~uintptr_t(15);
    const uint32_t nch = (uint32_t)((g1 - g0) >> 4);
    // interior 16-byte chunks (fully inside the block)
    const uint32_t c_first = (g0 == g) ? 0u : 1u;
    const uint32_t c_last = ((g + size) & 15u) ? nch - 1 : nch;  // exclusive
    for (uint32_t c = c_first + lane; c < c_last; c += 32)
      *reinterpret_cast<uint4*>(g0 + 16ull * c) = *reinterpret_cast<const uint4*>(sbase + 16 * c);
    // partial head / tail chunks: bytewise, lanes 0-15 head, 16-31 tail (neighbouring blocks own the rest)
    {
      const uint32_t c = lane < 16 ? 0u : nch - 1;
      const bool partial = lane < 16 ? (c_first == 1) : (c_last == nch - 1 && !(c == 0 && c_first == 1));
      const uint32_t bb = lane & 15u;
      const uintptr_t A = g0 + 16ull * c + bb;
      if (partial && A >= g && A < g + size) *reinterpret_cast<uint8_t*>(A) = sbase[16 * c + bb];
    }
  }
  __syncwarp();
}

// Section timing (instrumentation builds only: -DENC_TIMING, read with
// luda_dbg_enc_timing / profiles/encode_timing.py): per-warp clock64 deltas
// accumulated in shared memory, flushed once per warp.
#ifdef ENC_TIMING
__device__ unsigned long long g_enc_t[16];
__shared__ unsigned long long s_enc_t[kEncWarps][16];
#define ENC_T(i)                                                              \
  do {                                                                        \
    __syncwarp();                                                             \
    const unsigned long long t_ = clock64();                                  \
    if (lane_id() == 0) s_enc_t[threadIdx.x >> 5][i] += t_ - t_last;         \
    t_last = t_;                                                              \
  } while (0)
#define ENC_T0() unsigned long long t_last = clock64()
#else
#define ENC_T(i) do {} while (0)
#define ENC_T0() do {} while (0)
#endif

// ---- software-pipelined fast path ------------------------------------------------
// Blocks of <= 32 entries whose value windows fit the staging area (every
// BASELINE shape): lane i owns entry i. While block k is finished (CRC +
// copy-out), the records of block k+1 are already in registers and its value
// windows are in flight (TMA into the staging area, free once block k's
// values are realigned), so neither the record loads nor the value gather sit
// on the per-block critical path.
template <int W>
struct EncLane {
  uint64_t first, out_off;
  uint32_t cnt, size, k;
  bool valid;
  Rec<W> r;            // this lane's record (lane < cnt)
  // layout (lane's entry)
  uint32_t s, hv, esz, off, win, wpre, soff;
  uint64_t voff;
  uint32_t vl;
  uint32_t kl;         // internal key length of the entry (the job's K, or per record for var jobs)
  bool fast;
};

template <int W>
__device__ __forceinline__ void enc_load(const EncodeArgs<W>& a, uint32_t k, EncLane<W>& e) {
  e.k = k;
  e.valid = k < a.nblk;
  if (!e.valid) return;
  e.first = a.blk_first[k];
  e.cnt = a.blk_n[k];
  e.size = a.blk_size[k];
  e.out_off = a.blk_out[k];
  if (lane_id() < e.cnt && e.cnt <= 32) e.r = a.rec[e.first + lane_id()];
}

// sizes, offsets and value windows of a block of <= 32 entries
template <int W>
__device__ __forceinline__ void enc_layout(const EncodeArgs<W>& a, EncLane<W>& e) {
  const uint32_t lane = lane_id();
  // var records of <= 71-byte keys (W = kVarW) take the fast path with a key
  // length per lane (internal keys <= 79 bytes: one-byte shared / unshared
  // varints, as put_prefix_words needs); the long records stay generic
  e.fast = e.valid && e.cnt <= 32 && e.size <= (uint32_t)kEncStage && a.K < 128 && W != kVarWLong;
  if (!e.fast) return;
  const uint32_t K = a.K, L = K - 8;
  const bool act = lane < e.cnt;
  Rec<W> pr;
#pragma unroll
  for (int q = 0; q < W; ++q) pr.k[q] = __shfl_up_sync(0xFFFFFFFFu, e.r.k[q], 1);
  pr.t = __shfl_up_sync(0xFFFFFFFFu, e.r.t, 1);
  e.s = 0;
  e.hv = e.esz = e.vl = 0;
  e.voff = 0;
  e.kl = K;
  if (act) {
    if (is_var<W>()) e.kl = rec_ulen(e.r, true, 0) + 8;
    if (lane % a.ri != 0) e.s = ikey_lcp_any(pr, e.r, is_var<W>(), L);
    e.vl = handle_len(e.r.h);
    e.voff = handle_off(e.r.h);
    e.hv = varint_size(e.s) + varint_size(e.kl - e.s) + varint_size(e.vl);
    e.esz = e.hv + (e.kl - e.s) + e.vl;
  }
  const uint32_t incl = warp_incl_scan<uint32_t>(e.esz);
  e.off = incl - e.esz;
  // value windows: 16-byte-aligned source spans. Consecutive entries whose
  // values sit close together in the arena (same input block) share one
  // window — one bulk copy instead of one per entry; the gap bytes are staged
  // too. If merged windows overflow the staging area, entries get their own.
  const uintptr_t vs = reinterpret_cast<uintptr_t>(a.arena) + e.voff;
  const bool has = act && e.vl;
  const uintptr_t ws = vs & ~uintptr_t(15), we = (vs + e.vl + 15) & ~uintptr_t(15);
  const uintptr_t pve = __shfl_up_sync(0xFFFFFFFFu, vs + e.vl, 1);  // previous value's end
  const bool phas = __shfl_up_sync(0xFFFFFFFFu, (uint32_t)has, 1) && lane > 0;
  const bool cont = has && phas && vs >= pve && vs <= pve + (uintptr_t)kEncGap;  // windows stay monotone
  for (int attempt = 0; attempt < 2; ++attempt) {
    const bool join = attempt == 0 && cont;
    const uint32_t heads = __ballot_sync(0xFFFFFFFFu, has && !join);
    const uint32_t joins = __ballot_sync(0xFFFFFFFFu, join);
    // last lane of my group: first lane after me that does not join, minus one
    const uint32_t after = ~joins & ~((2u << lane) - 1u);
    const uint32_t last = after ? (uint32_t)(__ffs(after) - 2) : 31u;
    const uint32_t head = has ? 31u - __clz(heads & ((2u << lane) - 1u)) : lane;
    const uintptr_t gws = __shfl_sync(0xFFFFFFFFu, ws, head);
    const uintptr_t gwe = __shfl_sync(0xFFFFFFFFu, we, last);
    e.win = (has && !join) ? (uint32_t)(gwe - ws) : 0u;  // group window, at the head lane
    const uint32_t winc = warp_incl_scan<uint32_t>(e.win);
    e.wpre = winc - e.win;
    const uint32_t gpre = __shfl_sync(0xFFFFFFFFu, e.wpre, head);
    e.soff = gpre + (uint32_t)(vs - gws);
    e.fast = __shfl_sync(0xFFFFFFFFu, winc, 31) <= (uint32_t)kEncStg;
    if (e.fast || !__any_sync(0xFFFFFFFFu, cont)) break;
  }
}

template <int W>
__device__ __forceinline__ void enc_issue(const EncodeArgs<W>& a, const EncLane<W>& e, uint8_t* stg, uint64_t* bar) {
  const uint32_t total = __shfl_sync(0xFFFFFFFFu, e.wpre + e.win, 31);
  fence_proxy_async_smem();
  __syncwarp();
  if (lane_id() == 0) mbar_arrive_expect_tx(bar, total);
  __syncwarp();
  if (e.win) {
    const uintptr_t vs = reinterpret_cast<uintptr_t>(a.arena) + e.voff;
    bulk_g2s(stg + e.wpre, reinterpret_cast<const void*>(vs & ~uintptr_t(15)), e.win, bar);  // group head
  }
}

// headers + keys, then (after the values landed) the value realignment
template <int W>
__device__ __forceinline__ void enc_assemble(const EncodeArgs<W>& a, const EncLane<W>& e, uint8_t* wbuf, uint8_t* stg,
                                             uint64_t* bar, uint32_t& phase, uint32_t* pre) {
  const uint32_t lane = lane_id();
  const uint32_t K = a.K, L = K - 8, ri = a.ri;
  const uint32_t nres = (e.cnt + ri - 1) / ri;
  const uint32_t entries_end = e.size - 8 - 4 * nres;
  uint8_t* sbase = wbuf + kEncPre;
  uint8_t* dst = sbase + (e.out_off & 15);
  uint32_t first = 0;
  if (lane < e.cnt) first = put_prefix_words<W>(dst + e.off, e.r, e.kl - 8, e.s, e.vl, e.hv);
  __syncwarp();
  if (lane < e.cnt) {
    put_prefix_first(dst + e.off, first);
    if (lane % ri == 0) put_u32(dst + entries_end + 4 * (lane / ri), e.off);
  }
  if (lane == 0) put_u32(dst + entries_end + 4 * nres, nres);
  __syncwarp();  // headers/keys written before values (edge words are read-modified-written)
  ENC_T0();
  mbar_wait(bar, phase);
  phase ^= 1u;
  ENC_T(4);
  const uint32_t soff = e.soff;
  // each lane realigns its own value (no chunk map; edge words of neighbouring
  // entries are >= 12 bytes apart, so the per-word read-modify-writes never race)
  // Blocks of few, large values (cnt <= 16) share each value among G = 32/2^ceil(log2 cnt) lanes.
  const uint32_t lgc = e.cnt <= 1 ? 0u : 32u - __clz(e.cnt - 1u);
  const uint32_t G = 32u >> lgc;
  const uint32_t vdst = (uint32_t)(e.out_off & 15u) + e.off + e.hv + (e.kl - e.s);
  if (G == 1) {
    if (!LUDA_ABLATE(a, 4) && lane < e.cnt) value_copy16(sbase, stg, vdst, soff, e.vl, 0u, false, 0u, false);
  } else {
    const uint32_t v = lane / G;
    const uint32_t gd = __shfl_sync(0xFFFFFFFFu, vdst, v), gs = __shfl_sync(0xFFFFFFFFu, soff, v);
    const uint32_t gn = __shfl_sync(0xFFFFFFFFu, e.vl, v);
    if (!LUDA_ABLATE(a, 4) && v < e.cnt) value_copy16_strided(sbase, stg, gd, gs, gn, lane % G, G);
  }
  __syncwarp();
  ENC_T(5);
}

// CRC + 16-byte copy-out of an assembled (staged) block
template <int W>
__device__ __forceinline__ void enc_finish(const EncodeArgs<W>& a, const EncLane<W>& e, uint8_t* wbuf,
                                           const CrcSmem& cs) {
  const uint32_t lane = lane_id();
  uint8_t* sbase = wbuf + kEncPre;
  uint8_t* dst = sbase + (e.out_off & 15);
  const uint32_t size = e.size;
  const uint32_t crc = LUDA_ABLATE(a, 1) ? 0u : warp_crc32_smem(dst, size - 4, cs);
  if (lane == 0) put_u32(dst + size - 4, crc);
  __syncwarp();
  const uintptr_t g = reinterpret_cast<uintptr_t>(a.out + e.out_off);
  const uintptr_t g0 = g & ~uintptr_t(15), g1 = (g + size + 15) & ~uintptr_t(15);
  const uint32_t nch = (uint32_t)((g1 - g0) >> 4);
  const uint32_t c_first = (g0 == g) ? 0u : 1u;
  const uint32_t c_last = ((g + size) & 15u) ? nch - 1 : nch;  // exclusive
  // interior 16-byte chunks: one TMA bulk store (the smem reads leave the LSU
  // pipe); the caller waits for its smem reads before releasing the buffer
  fence_proxy_async_smem();  // every lane's smem writes (CRC prep/unprep, CRC word) → async proxy
  __syncwarp();
  if (!LUDA_ABLATE(a, 2) && lane == 0 && c_last > c_first) {
    bulk_s2g(reinterpret_cast<void*>(g0 + 16ull * c_first), sbase + 16 * c_first, 16u * (c_last - c_first));
    bulk_commit();
  }
  {
    const uint32_t c = lane < 16 ? 0u : nch - 1;
    const bool partial = lane < 16 ? (c_first == 1) : (c_last == nch - 1 && !(c == 0 && c_first == 1));
    const uint32_t bb = lane & 15u;
    const uintptr_t A = g0 + 16ull * c + bb;
    if (partial && A >= g && A < g + size) *reinterpret_cast<uint8_t*>(A) = sbase[16 * c + bb];
  }
  __syncwarp();
}

template <int W>
__global__ void __launch_bounds__(kEncWarps * 32, 1) encode_kernel(EncodeArgs<W> a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  CrcSmem& cs = *reinterpret_cast<CrcSmem*>(smem_raw);
  EncPairSmem* pairs = reinterpret_cast<EncPairSmem*>(smem_raw + sizeof(CrcSmem));
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  const bool builder = kEncFused || warp < kEncPairs;
  const uint32_t p = warp % kEncPairs;
  EncPairSmem& ps = pairs[p];
  EncCtaSmem& cta = *reinterpret_cast<EncCtaSmem*>(smem_raw + sizeof(CrcSmem) + kEncPairs * sizeof(EncPairSmem));
  if (threadIdx.x == 0) cta.lock = 0;
  crc_smem_init(cs);
#ifdef ENC_TIMING
  if (lane < 16) s_enc_t[warp][lane] = 0;
#endif
  if (builder && lane == 0) {
    mbar_init(&ps.bar, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&ps.full[b], 1);
      mbar_init(&ps.empty[b], 1);
    }
  }
  __syncthreads();
  const uint32_t gw = blockIdx.x * kEncPairs + p;
  const uint32_t nw = gridDim.x * kEncPairs;
  if (builder) {
    uint32_t phase = 0;
    EncLane<W> cur, nxt;
    enc_load(a, gw, cur);
    enc_layout(a, cur);
    if (cur.fast) enc_issue(a, cur, ps.stg, &ps.bar);
    for (uint32_t i = 0; cur.valid; ++i) {
      const uint32_t b = kEncFused ? 0u : (i & 1u);
      uint8_t* wbuf = ps.buf[b];
      ENC_T0();
      if (kEncFused) {
        if (lane == 0) bulk_wait_read0();  // the previous block's bulk store has read the buffer
        __syncwarp();
      } else if (i >= 2) {
        mbar_wait(&ps.empty[b], ((i - 2) >> 1) & 1u);  // the CRC warp is done with block i-2
      }
      ENC_T(0);
      enc_load(a, cur.k + nw, nxt);  // records of the next block: loads in flight
      ENC_T(1);
      EncMeta mt{cur.out_off, cur.size, 0u};
      if (cur.fast) {
        enc_assemble(a, cur, wbuf, ps.stg, &ps.bar, phase, nullptr);
        ENC_T(2);
        enc_layout(a, nxt);  // staging is free again: start the next block's value gather
        ENC_T(3);
        if (nxt.fast) enc_issue(a, nxt, ps.stg, &ps.bar);
        ENC_T(6);
      } else {
        const uint32_t k = cur.k;
        if (lane == 0)
          while (atomicCAS(&cta.lock, 0, 1) != 0) __nanosleep(64);
        __syncwarp();
        if (cur.size <= (uint32_t)kEncStage)
          encode_one_block<W, true>(a, k, cur.first, cur.cnt, cur.size, cur.out_off, wbuf, ps.stg, &ps.bar, phase,
                                    cta.pre, cs);
        else
          encode_one_block<W, false>(a, k, cur.first, cur.cnt, cur.size, cur.out_off, wbuf, ps.stg, &ps.bar, phase,
                                     cta.pre, cs);
        __syncwarp();
        if (lane == 0) atomicExch(&cta.lock, 0);
        mt.skip = 1;
        enc_layout(a, nxt);
        if (nxt.fast) enc_issue(a, nxt, ps.stg, &ps.bar);
      }
      if (kEncFused) {
        if (!mt.skip) enc_finish(a, cur, wbuf, cs);  // CRC + bulk store; the buffer is waited for above
      } else {
        if (lane == 0) ps.meta[b] = mt;
        fence_proxy_async_smem();  // the assembled bytes are read by the CRC warp's bulk store
        __syncwarp();
        if (lane == 0) mbar_arrive(&ps.full[b]);  // release: the assembled block and its meta
      }
      cur = nxt;
      ENC_T(7);
    }
    if (kEncFused && lane == 0) bulk_wait0();
  } else {
    // CRC warp: CRC + copy-out of the blocks the builder assembled, in order
    for (uint32_t i = 0, k = gw; k < a.nblk; ++i, k += nw) {
      const uint32_t b = i & 1u;
      ENC_T0();
      mbar_wait(&ps.full[b], (i >> 1) & 1u);
      ENC_T(8);
      const EncMeta mt = ps.meta[b];
      if (!mt.skip) {
        EncLane<W> e;
        e.out_off = mt.out_off;
        e.size = mt.size;
        enc_finish(a, e, ps.buf[b], cs);
        if (lane == 0) bulk_wait_read0();  // the bulk store has read the buffer
      }
      ENC_T(9);
      __syncwarp();
      if (lane == 0) mbar_arrive(&ps.empty[b]);
    }
    if (lane == 0) bulk_wait0();
  }
#ifdef ENC_TIMING
  __syncwarp();
  if (lane < 16) atomicAdd(&g_enc_t[lane], s_enc_t[warp][lane]);
#endif
}

// ---- per-SST filter + index + footer -----------------------------------------------------
#ifndef LUDA_META_THREADS
#define LUDA_META_THREADS 896
#endif
constexpr int kMetaThreads = LUDA_META_THREADS;
// keys in flight per thread in the bloom loop (var records: 4, else they spill)
template <int W>
__host__ __device__ constexpr int meta_unroll() { return W <= 4 ? 8 : 4; }

// a mod d for 32-bit a, d >= 1 with rcp = floor((2^64 - 1) / d) + 1
// (Lemire, Kaser, Kurz: "Faster remainder by direct computation").
__device__ __forceinline__ uint32_t fastmod_u32(uint32_t a, uint64_t rcp, uint32_t d) {
  const uint64_t low = rcp * a;
  return (uint32_t)__umul64hi(low, d);
}
constexpr int kMetaBuf = kMetaBufBytes;
constexpr int kMetaSmem = (int)sizeof(CrcSmem) + kEncPre + kMetaBuf + 64;

template <int W>
struct MetaArgs {
  const Rec<W>* rec;
  uint32_t K;
  uint32_t bits_per_key;
  uint32_t kprobes;
  uint32_t nsst;
  const uint32_t* sst_first_blk;
  const uint32_t* sst_last_blk;
  const uint64_t* sst_off;
  const uint64_t* sst_data;
  const uint64_t* sst_nent;
  const uint64_t* sst_size;
  const uint32_t* blk_first;
  const uint32_t* blk_n;
  const uint32_t* blk_size;
  const uint64_t* blk_pos;
  uint8_t* out;
  uint32_t* scratch;           // zeroed, for filters larger than kMetaBuf
  const uint64_t* scratch_off; // per SST word offset into scratch (or ~0)
  uint8_t* sst_keys;           // [nsst][2][key_slot]
  uint32_t* sst_key_len;       // [nsst][2] internal key lengths
  uint32_t key_slot;           // bytes per key slot (K, or 8 W + 8 for var jobs)
  bool var;
  const uint64_t* blk_ipos;    // var jobs: index-entry offsets (luda_plan.cuh), else nullptr
};

// Bloom hash h = crc32(user key) (bloom.py:28-29): the L/4 whole 4-byte words
// of the key through the slicing-by-2 update, then the L%4 tail bytes of the
// next word. wmax: a warp-uniform bound on L/4 (var records: the warp's
// longest key, so short keys do not walk all 2W predicated words).
template <int W>
__device__ __forceinline__ uint32_t key_word_be(const Rec<W>& r, int w) {
  return (uint32_t)(r.k[w >> 1] >> ((w & 1) ? 0 : 32));
}
template <int W>
__device__ __forceinline__ uint32_t user_key_crc(const Rec<W>& r, uint32_t L, const CrcLane& tl,
                                                 uint32_t wmax = 2 * W) {
  uint32_t c = 0xFFFFFFFFu;
  const uint32_t nw = L >> 2;
#pragma unroll
  for (int w = 0; w < 2 * W; ++w) {
    if (is_var<W>() && (uint32_t)w >= wmax) break;
    if ((uint32_t)w < nw) c = crc_word(c, bswap32(key_word_be<W>(r, w)), tl);
  }
  uint32_t tw = 0;  // the word holding the tail bytes (static indices: the record stays in registers)
#pragma unroll
  for (int w = 0; w < 2 * W; ++w) tw = ((uint32_t)w == nw) ? key_word_be<W>(r, w) : tw;
  for (uint32_t t = 0; t < (L & 3u); ++t) c = crc_byte(c, (tw >> (24 - 8 * t)) & 0xFFu, tl);
  return ~c;
}

// Persistent: one CTA per SM loops over the output SSTs (the CRC tables are
// loaded into shared memory once per CTA).
template <int W>
__global__ void __launch_bounds__(kMetaThreads, 1) sst_meta_kernel(MetaArgs<W> a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  CrcSmem& cs = *reinterpret_cast<CrcSmem*>(smem_raw);
  uint8_t* buf = smem_raw + sizeof(CrcSmem) + kEncPre;  // 16-aligned, 160 B lead-in
  __shared__ uint32_t red[32];
  crc_smem_init(cs);
  __syncthreads();
  const uint32_t tid = threadIdx.x, lane = lane_id();
  const uint32_t K = a.K, L = K - 8;
  const CrcLane tl = crc_lane(cs, lane);
  for (uint32_t s = blockIdx.x; s < a.nsst; s += gridDim.x) {
    const uint32_t fb = a.sst_first_blk[s], eb = a.sst_last_blk[s];
    const uint64_t fe = a.blk_first[fb];
    const uint64_t ne = a.sst_nent[s];
    const uint64_t data = a.sst_data[s];
    uint8_t* fout = a.out + a.sst_off[s];
    uint64_t nbits = ne * a.bits_per_key;
    if (nbits < 64) nbits = 64;
    nbits = (nbits + 7) & ~7ull;
    const uint64_t nbytes = nbits / 8;
    const bool small = nbytes + 1 <= (uint64_t)kMetaBuf;
    uint32_t* bits = small ? reinterpret_cast<uint32_t*>(buf) : a.scratch + a.scratch_off[s];
    if (small)
      for (uint32_t i = tid; i < (nbytes + 1 + 3) / 4; i += kMetaThreads) bits[i] = 0;
    __syncthreads();
    // ---- bloom bits: positions (h + j*delta) mod n_bits, 64-bit (bloom.py:81-87) ----
    if (nbits < (1ull << 31)) {
      // 32-bit positions; h mod n and delta mod n by Lemire's fastmod (one
      // 64-bit reciprocal per SST). Records are loaded meta_unroll<W>() at a time
      // so the loop is not one DRAM latency per key.
      const uint32_t nb32 = (uint32_t)nbits;
      const uint64_t rcp = ~0ull / nb32 + 1;
      const uint64_t e_end = fe + ne;
      for (uint64_t e0 = fe + tid; e0 < e_end; e0 += meta_unroll<W>() * kMetaThreads) {
        Rec<W> r[meta_unroll<W>()];  // key words only: the hash never reads the trailer / handle
#pragma unroll
        for (int u = 0; u < meta_unroll<W>(); ++u) {
          const uint64_t e = e0 + (uint64_t)u * kMetaThreads;
          const Rec<W>& src = a.rec[e < e_end ? e : fe];
#pragma unroll
          for (int w = 0; w < W; ++w) r[u].k[w] = src.k[w];
        }
        // the meta_unroll<W>() key hashes are independent table chains: computed
        // together (ILP) before any probe
        uint32_t h[meta_unroll<W>()];
#pragma unroll
        for (int u = 0; u < meta_unroll<W>(); ++u) {
          const uint32_t Lu = rec_ulen(r[u], is_var<W>(), L);
          const uint32_t wmax = is_var<W>() ? __reduce_max_sync(__activemask(), Lu >> 2) : 2 * W;
          h[u] = user_key_crc<W>(r[u], Lu, tl, wmax);
        }
#pragma unroll
        for (int u = 0; u < meta_unroll<W>(); ++u) {
          if (e0 + (uint64_t)u * kMetaThreads < e_end) {
            const uint32_t delta = (h[u] >> 17) | (h[u] << 15);
            uint32_t p = fastmod_u32(h[u], rcp, nb32);
            const uint32_t step = fastmod_u32(delta, rcp, nb32);
            for (uint32_t j = 0; j < a.kprobes; ++j) {
              atomicOr(bits + (p >> 5), 1u << (p & 31));
              p += step;
              if (p >= nb32) p -= nb32;
            }
          }
        }
      }
    } else {
      for (uint64_t e = fe + tid; e < fe + ne; e += kMetaThreads) {
        const Rec<W> re = a.rec[e];
        const uint32_t h = user_key_crc<W>(re, rec_ulen(re, is_var<W>(), L), tl);
        const uint32_t delta = (h >> 17) | (h << 15);
        uint64_t p = (uint64_t)h % nbits;
        const uint64_t step = (uint64_t)delta % nbits;
        for (uint32_t j = 0; j < a.kprobes; ++j) {
          atomicOr(bits + (p >> 5), 1u << (p & 31));
          p += step;
          if (p >= nbits) p -= nbits;
        }
      }
    }
    __syncthreads();
    // ---- filter block: bits ∥ k ∥ crc ----
    uint8_t* fb8 = reinterpret_cast<uint8_t*>(bits);
    if (tid == 0) fb8[nbytes] = (uint8_t)a.kprobes;
    __syncthreads();
    const uint32_t fcrc = small ? cta_crc32_smem(fb8, (uint32_t)(nbytes + 1), cs, red)
                                : cta_crc32_global(fb8, nbytes + 1, cs, buf, red);
    coop_copy(fout + data, fb8, nbytes + 1, tid, kMetaThreads);
    if (tid == 0) put_u32(fout + data + nbytes + 1, fcrc);
    __syncthreads();
    // ---- index block ----
    const uint64_t flen = nbytes + 5;
    const uint32_t vK = varint_size(K);
    const uint64_t E = vK + K + 8;
    const uint32_t nb = eb - fb;
    const uint64_t ibody = (a.blk_ipos ? a.blk_ipos[eb] - a.blk_ipos[fb] : (uint64_t)nb * E) + 4;  // entries ∥ count
    const bool ismall = ibody <= (uint64_t)kMetaBuf;
    uint8_t* ib = ismall ? buf : fout + data + flen;
    for (uint32_t i = tid; i < nb; i += kMetaThreads) {
      const uint32_t b = fb + i;
      const Rec<W> last = a.rec[(uint64_t)a.blk_first[b] + a.blk_n[b] - 1];
      const uint32_t Lb = rec_ulen(last, is_var<W>(), L), Kb = Lb + 8;
      uint8_t* p = ib + (a.blk_ipos ? a.blk_ipos[b] - a.blk_ipos[fb] : (uint64_t)i * E);
      const uint32_t vKb = put_varint(p, Kb);
      put_key_tail<W>(p + vKb, last, Lb, 0);
      put_u32(p + vKb + Kb, (uint32_t)(a.blk_pos[b] - a.blk_pos[fb]));
      put_u32(p + vKb + Kb + 4, a.blk_size[b]);
    }
    if (tid == 0) put_u32(ib + ibody - 4, nb);
    __syncthreads();
    if (!ismall) __threadfence();
    __syncthreads();
    const uint32_t icrc = ismall ? cta_crc32_smem(ib, (uint32_t)ibody, cs, red)
                                 : cta_crc32_global(ib, ibody, cs, buf, red);
    if (ismall) coop_copy(fout + data + flen, ib, ibody, tid, kMetaThreads);
    if (tid == 0) {
      put_u32(fout + data + flen + ibody, icrc);
      // footer <IIIIQ>: filter_off, filter_len, index_off, index_len, magic
      uint8_t* ft = fout + a.sst_size[s] - 24;
      put_u32(ft, (uint32_t)data);
      put_u32(ft + 4, (uint32_t)flen);
      put_u32(ft + 8, (uint32_t)(data + flen));
      put_u32(ft + 12, (uint32_t)(ibody + 4));
      put_u32(ft + 16, (uint32_t)kMagic);
      put_u32(ft + 20, (uint32_t)(kMagic >> 32));
    }
    // smallest / largest internal keys
    if (tid < 2 && ne > 0) {
      const Rec<W> r = a.rec[tid == 0 ? fe : fe + ne - 1];
      const uint32_t Lr = rec_ulen(r, is_var<W>(), L);
      put_key_tail<W>(a.sst_keys + ((uint64_t)s * 2 + tid) * a.key_slot, r, Lr, 0);
      a.sst_key_len[(uint64_t)s * 2 + tid] = Lr + 8;
    }
    __syncthreads();  // buf is reused by the next SST
  }
}

}  // namespace luda
