// luda_decode.cuh — data-block decode: CRC verify + entry parse → records.
//
// Restates decode_data_block (blocks.py:130-165) for every data block listed
// by the index blocks (Table.scan, sst.py:370-375), and the `unpack` kernel
// work item (kernels.py:72-104), except that it emits fixed-width sort
// records (luda_rec.cuh) with a value HANDLE instead of copying values.
//
// One warp per block, blocks taken in order from a global counter. Per warp:
//  * two smem staging buffers; while block b is processed, the 16-byte-aligned
//    window of the next block is already in flight (cp.async.bulk + mbarrier);
//    blocks longer than kDecStage are read in place from global memory;
//  * phase 1 — entry walk. Fast path: lane k walks restart interval k
//    (offsets from the block tail) with a 1–2-byte varint header decoder and
//    records every entry (key-suffix position, shared, value length) in smem.
//    It is accepted only if every interval starts with shared == 0 and ends
//    exactly on the next restart offset — then the sequential reference parse
//    passes through the same entry boundaries and yields identical keys.
//    Otherwise lane 0 runs the exact sequential reference parse (errors
//    included);
//  * every warp owns a CONTIGUOUS range of blocks and writes their records
//    back to back into its own segment of the record array (segment w at
//    w * seg_cap); a block's record base is the warp's running count, so
//    there is no inter-warp dependency at all (no count pre-pass, no
//    look-back). The merge reads the segmented array through a logical →
//    physical index view (luda_merge.cuh, SegRun);
//  * warp CRC-32 of the payload (end-aligned segments, luda_common.cuh);
//  * phase 2 — lanes take consecutive entries; each loads its key suffix and
//    the prefix bytes it shares are filled from earlier lanes by a
//    Hillis-Steele scan over "valid-from" byte positions (shuffles only);
//    records are written coalesced (lane i → record base+i).
// Errors: reference errors → min((block << 8) | code) in err_ref; inputs that
// are valid for the reference but outside the fixed-key-length envelope →
// err_unsup (the host raises those only if no reference error exists).
#pragma once
#include "luda_parse.cuh"
#include "luda_rec.cuh"

namespace luda {

enum BlockCode : uint32_t {
  B_OK = 0,
  B_SHORT = 1,          // block too short
  B_CRC = 2,            // data block checksum mismatch
  B_RESTART = 3,        // bad restart array
  B_VARINT_TRUNC = 4,   // truncated varint
  B_VARINT_LONG = 5,    // varint too long
  B_TRUNC_ENTRY = 6,    // truncated block entry
  B_TRAILING = 7,       // trailing garbage in block entries
  B_KEYLEN = 8,         // (unsupported) key length differs from the job's K
  B_VALUE_BIG = 9,      // (unsupported) value length >= 2^24 or arena offset >= 2^40
  B_KEYLONG = 10,       // (unsupported) user key longer than the var record holds (71 / 255 bytes)
};

// Paired warps: a PARSE warp (producer + walk + records) and a CRC warp share
// a pair of staging slots; both consume every block of the pair's contiguous
// block range concurrently (the CRC never modifies bytes the parse warp reads).
#ifndef LUDA_DEC_PAIRS
#define LUDA_DEC_PAIRS 12
#endif
constexpr int kDecPairs = LUDA_DEC_PAIRS;
constexpr int kDecWarps = 2 * kDecPairs;
#ifndef LUDA_DEC_CHUNKS
#define LUDA_DEC_CHUNKS 4
#endif
constexpr uint32_t kDecChunksPerPair = LUDA_DEC_CHUNKS;  // block chunks (record segments) per pair, on average
#ifndef LUDA_DEC_NSLOT
#define LUDA_DEC_NSLOT 2
#endif
constexpr int kDecNSlot = LUDA_DEC_NSLOT;        // staging slots per pair (NSLOT - 1 blocks in flight)
constexpr int kDecLead = 48;                     // zero lead before the TMA window (never written by TMA)
constexpr int kDecStage = 4352;                  // TMA window capacity
constexpr int kDecSlot = kDecLead + kDecStage;   // bytes per staging slot
constexpr int kDecSlots = 104;
constexpr int kDecStride = 16;                   // slots per restart interval (single-walk path)
constexpr int kDecBig = kGroup + 192;            // CTA staging for CRC passes of unstaged (large) blocks
struct DecSlotMeta {
  uint64_t addr;  // arena offset of the block
  uint32_t len;   // block length
  uint32_t tag;   // block index | staged << 31 (kDecEnd: end of the pair's sequence)
  __device__ __forceinline__ uint32_t blk() const { return tag & 0x7FFFFFFFu; }
  __device__ __forceinline__ bool staged() const { return tag >> 31; }
};
constexpr uint32_t kDecEnd = 0x7FFFFFFFu;  // (jobs have fewer blocks: luda_compact checks)
struct DecPairSmem {
  uint8_t slot[kDecNSlot][kDecSlot];
  uint64_t full[kDecNSlot], empty[kDecNSlot];
  DecSlotMeta meta[kDecNSlot];  // written by the producer before it arrives on full
  uint8_t entries[kDecSlots * 8];  // DecSlot array of the parse warp
};
struct DecCtaSmem {
  uint8_t big[kDecBig];
  int lock;
};
static_assert(sizeof(CrcSmem) + kDecPairs * sizeof(DecPairSmem) + sizeof(DecCtaSmem) <= 232448,
              "decode smem over the 227 KB limit");
static_assert(kDecLead >= kSeg && kDecLead % 16 == 0, "CRC segments may start kSeg-1 bytes before the data");
static_assert(kDecSlot % 16 == 0 && sizeof(DecPairSmem) % 16 == 0, "TMA destinations must be 16-byte aligned");

struct DecSlot {
  uint32_t pos;  // block-relative offset of the key suffix
  uint32_t sv;   // value_len << 8 | shared
};

template <int W>
struct DecodeArgs {
  const uint8_t* arena;
  BlockTable bt;
  uint32_t nblk;
  uint32_t K;               // internal key length of the job
  Rec<W>* out;              // segmented: chunk c's records at out[c * seg_cap ...]
  uint64_t seg_cap;         // records per warp segment
  uint32_t* blk_local;      // out [nblk]: block's first record index within its warp segment
  uint64_t* seg_count;      // out [nseg]: records of each segment (may exceed seg_cap → rerun)
  uint32_t nseg;            // record segments = block chunks
  unsigned int* chunk_ctr;  // chunk counter (zeroed before the launch)
  unsigned long long* err_ref;
  unsigned long long* err_unsup;
  uint32_t dbg;             // ablation switches (LUDA_ABLATION builds only)
  bool var;                 // generic-length keys (W = kVarW records, dec_var_block)
};

// Block range of warp segment w of nw: [w*nblk/nw, (w+1)*nblk/nw).
__host__ __device__ __forceinline__ uint32_t seg_first_block(uint32_t w, uint32_t nblk, uint32_t nw) {
  return (uint32_t)(((uint64_t)w * nblk) / nw);
}
__device__ __forceinline__ uint32_t seg_of_block(uint32_t b, uint32_t nblk, uint32_t nw) {
  uint32_t w = (uint32_t)(((uint64_t)b * nw) / nblk);
  while (w + 1 < nw && seg_first_block(w + 1, nblk, nw) <= b) ++w;
  while (w > 0 && seg_first_block(w, nblk, nw) > b) --w;
  return w;
}

// Walk one restart interval [start, end) under fast-path rules and call
// emit(j, pos_suffix, shared, vlen) per entry; returns the entry count or -1
// when the interval is not in canonical form (the exact path then decides).
// Fast form: 1-byte shared/unshared varints, 1–2-byte value length,
// shared + unshared == K (so shared <= len(prev key) == K), shared == 0 on the
// interval's first entry, entries tiling [start, end) exactly.
// Branch-free per entry: errors are OR-ed into `bad` and decided once at the
// end (every step advances >= 3 bytes, so garbage still terminates).
template <typename Emit>
__device__ __forceinline__ int32_t interval_walk(const uint8_t* d, uint32_t start, uint32_t end, uint32_t K,
                                                 Emit emit) {
  uint32_t pos = start;
  int32_t j = 0;
  uint32_t bad = 0;
  while (pos < end) {
    const uint32_t w = ld_u32_any(d + pos);  // shared | unshared | vlen byte 0 | vlen byte 1
    const uint32_t s = w & 0xFFu;
    const uint32_t u = prmt(w, 0u, 0x4441u);
    const uint32_t v1 = prmt(w, 0u, 0x4442u);
    const uint32_t two = (w >> 23) & 1u;  // 2-byte value length
    const uint32_t vl = two ? ((v1 & 0x7Fu) | ((w >> 17) & 0x7F80u)) : v1;
    bad |= (w & 0x8080u) | (two & (w >> 31)) | ((s + u) ^ K) | (j == 0 ? s : 0u);
    emit(j, pos + 3u + two, s, vl);
    pos += 3u + two + u + vl;
    ++j;
  }
  return (bad || pos != end) ? -1 : j;
}

// Entry-header positions of one restart interval (no validation: every
// header is checked afterwards, lane per entry). Value-length varints of 1 or
// 2 bytes are assumed; any other header makes the chain miss `end` or fail the
// later check. Returns the entry count, or -1 if the chain does not end
// exactly at `end`.
template <typename Emit>
__device__ __forceinline__ int32_t interval_positions(const uint8_t* d, uint32_t start, uint32_t end, Emit emit) {
  // The chain is one byte-load latency + 3 integer ops per entry: the three
  // header bytes that decide the next position are loaded independently
  // straight from the running pointer (no alignment arithmetic before the
  // loads): next = p + 3 + u + b2 + (b2 >> 7) * (128 b3 - 127).
  const uint8_t* p = d + start;
  const uint8_t* e = d + end;
  int32_t j = 0;
  while (p < e) {
    const uint32_t u = p[1], b2 = p[2], b3 = p[3];
    emit(j, (uint32_t)(p - d));
    const uint32_t two = b2 >> 7;
    p += (3u + u + b2) + two * (b3 * 128u - 127u);
    ++j;
  }
  return p == e ? j : -1;
}

// interval_positions into a lane's 16 slots: slot j & 15 (an interval with
// more than 16 entries overwrites its own slots, but then the block leaves
// the slot fast path), no predicate or running position in the loop.
__device__ __forceinline__ int32_t interval_positions_slots(const uint8_t* d, uint32_t start, uint32_t end,
                                                            uint32_t* mine) {
  uint32_t pos = start;
  uint32_t j = 0;
  while (pos < end) {
    const uint8_t* h = d + pos;
    const uint32_t u = h[1], b2 = h[2], b3 = h[3];
    mine[j & (kDecStride - 1)] = pos;
    pos += (3u + u + b2) + (b2 >> 7) * (b3 * 128u - 127u);
    ++j;
  }
  return pos == end ? (int32_t)j : -1;
}

__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// Staged-block variant of interval_positions_slots on 32-bit shared
// addresses: the running position IS the header's shared address (no
// base + offset per step), the slot pointer runs alongside, and the ABSOLUTE
// address is stored (the records phase subtracts the block base once per
// lane): 11 instructions per step instead of 16. Intervals of more than 16
// entries return -1, as the slot fast path needs <= 16 anyway. Not unrolled:
// this kernel is instruction-cache sensitive (c3 decode: rolled 4.15 ms,
// unrolled x2 4.20, fully unrolled 4.47, previous loop 4.26).
__device__ __forceinline__ int32_t interval_positions_smem(uint32_t a, uint32_t e, uint32_t m) {
  const uint32_t m_end = m + 4 * kDecStride;
#pragma unroll 1
  for (; a < e && m < m_end; m += 4) {
    const uint32_t u = lds_u8(a + 1), b2 = lds_u8(a + 2), b3 = lds_u8(a + 3);
    sts_u32(m, a);
    a += (3u + u + b2) + (b2 >> 7) * (b3 * 128u - 127u);
  }
  return a == e ? (int32_t)((m - (m_end - 4 * kDecStride)) >> 2) : -1;
}

// Exact sequential decode_data_block walk (blocks.py:151-164). Returns the
// reference error code (0 ok) and sets `unsup` for envelope violations.
template <typename Emit>
__device__ uint32_t block_walk_exact(const uint8_t* d, uint64_t payload, uint64_t entries_end, uint32_t K,
                                     uint64_t& n_out, uint32_t& unsup, Emit emit) {
  uint64_t pos = 0, prev_len = 0, n = 0;
  unsup = 0;
  while (pos < entries_end) {
    uint64_t s, u, vl;
    int r;
    if ((r = varint_read(d, payload, pos, s)) || (r = varint_read(d, payload, pos, u)) ||
        (r = varint_read(d, payload, pos, vl))) {
      n_out = n;
      return r == 1 ? B_VARINT_TRUNC : B_VARINT_LONG;
    }
    if (s > prev_len || u > entries_end || vl > entries_end || pos + u + vl > entries_end) {
      n_out = n;
      return B_TRUNC_ENTRY;
    }
    if (s + u != K) unsup = unsup ? unsup : B_KEYLEN;
    if (vl > kMaxValueLen) unsup = unsup ? unsup : B_VALUE_BIG;
    emit(n, (uint32_t)pos, (uint32_t)s, (uint32_t)vl);
    prev_len = s + u;
    pos += u + vl;
    ++n;
  }
  n_out = n;
  return pos != entries_end ? B_TRAILING : B_OK;
}

__device__ __forceinline__ uint32_t dec_window(const uint8_t* g, uint32_t len) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(g);
  return (uint32_t)(((a + len + 15) & ~uintptr_t(15)) - (a & ~uintptr_t(15)));
}

// Per-block state carried from phase 1 to phase 2.
struct DecState {
  uint64_t addr;          // arena offset of the block
  uint32_t len;
  uint32_t nres;
  int64_t entries_end;
  uint32_t code;          // reference error so far (before CRC)
  uint32_t restart_bad;
  uint32_t pcode, unsup;
  int mode;               // 1 single walk, 2 fast windows, 3 exact walk
  uint64_t n;
  int32_t my_cnt, my_pre;
  uint32_t my_st, my_en;
};
constexpr int kDecSlotIntervals = (kDecSlots * 2) / kDecStride;  // intervals the mode-1 slot layout holds

// Phase 1: structural checks + entry walk (counts; single-walk fills slots).
#ifdef DEC_TIMING
__device__ unsigned long long g_dec_t[16];
#define DEC_T(i)                                                              \
  do {                                                                        \
    __syncwarp();                                                             \
    const unsigned long long t_ = clock64();                                  \
    if (lane_id() == 0) atomicAdd(&g_dec_t[i], t_ - t_last);                  \
    t_last = t_;                                                              \
  } while (0)
#define DEC_T0() unsigned long long t_last = clock64()
#else
#define DEC_T(i) do {} while (0)
#define DEC_T0() do {} while (0)
#endif

// u32le at p: staged blocks (smem with slack after the window) use two
// aligned word loads + PRMT; blocks read from global keep byte loads (never
// past the block's end).
template <bool kStaged>
__device__ __forceinline__ uint32_t dec_ld32(const uint8_t* p) {
  if (kStaged) return ld_u32_any(p);
  return ld_u32_le(p);
}

template <int W, bool kStaged>
__device__ __forceinline__ DecState dec_phase1(const DecodeArgs<W>& a, uint32_t b, uint64_t addr, uint32_t blen,
                                               const uint8_t* d, DecSlot* slots) {
  const uint32_t lane = lane_id();
  DEC_T0();
  DecState st{};
  st.len = blen;
  st.addr = addr;
  const uint32_t K = a.K;
  const uint32_t len = st.len;
  st.code = len < 12 ? (uint32_t)B_SHORT : 0u;
  if (!st.code) {
    st.nres = dec_ld32<kStaged>(d + len - 8);
    st.entries_end = (int64_t)len - 8 - 4 * (int64_t)st.nres;
    st.restart_bad = st.nres < 1 || st.entries_end < 0;
  }
  st.mode = 3;
  if (!st.code && !st.restart_bad) {
    const uint32_t nres = st.nres;
    const int64_t entries_end = st.entries_end;
    if (nres <= 32) {
      bool ok = true;
      const bool single = nres <= (uint32_t)kDecSlotIntervals;
      if (lane < nres) {
        st.my_st = dec_ld32<kStaged>(d + entries_end + 4 * lane);
        st.my_en = (lane + 1 < nres) ? dec_ld32<kStaged>(d + entries_end + 4 * (lane + 1)) : (uint32_t)entries_end;
        ok = (lane != 0 || st.my_st == 0) && st.my_st < st.my_en && (int64_t)st.my_en <= entries_end;
      }
      DEC_T(0);
      bool fast = false;
      if (single) {
        // Positions-only walk (lane per interval) into the slot layout
        // [interval][<= 16 entries]; the headers are validated and decoded by
        // lane per entry in phase 2 (mode 1), before anything is written.
        uint32_t* pos32 = reinterpret_cast<uint32_t*>(slots);
        if (lane < nres && ok) {
          uint32_t* mine = pos32 + kDecStride * lane;
          if (kStaged) {
            const uint32_t db = smem_u32(d);
            st.my_cnt = interval_positions_smem(db + st.my_st, db + st.my_en, smem_u32(mine));
          } else {
            st.my_cnt = interval_positions_slots(d, st.my_st, st.my_en, mine);
          }
          ok = st.my_cnt >= 0 && st.my_cnt <= kDecStride;
        }
        DEC_T(1);
        if (__all_sync(0xFFFFFFFFu, ok)) {
          fast = true;
          st.mode = 1;
        }
      }
      if (!fast) {
        // general canonical walk (validating); mode 2 re-walks it window by window
        ok = true;
        if (lane < nres) {
          ok = (lane != 0 || st.my_st == 0) && st.my_st < st.my_en && (int64_t)st.my_en <= entries_end;
          if (ok) {
            st.my_cnt = interval_walk(d, st.my_st, st.my_en, K, [](int32_t, uint32_t, uint32_t, uint32_t) {});
            ok = st.my_cnt >= 0;
          }
        }
        if (__all_sync(0xFFFFFFFFu, ok)) st.mode = 2;
      }
      if (st.mode == 2) {
        const int32_t c = lane < nres ? st.my_cnt : 0;
        const int32_t incl = warp_incl_scan<int32_t>(c);
        st.my_pre = incl - c;
        st.n = (uint64_t)(uint32_t)__shfl_sync(0xFFFFFFFFu, incl, 31);
      } else if (st.mode == 1) {
        st.n = __reduce_add_sync(0xFFFFFFFFu, lane < nres ? (uint32_t)st.my_cnt : 0u);
      }
      DEC_T(3);
    }
    if (st.mode == 3) {
      uint64_t nn = 0;
      uint32_t pc = 0, us = 0;
      if (lane == 0)
        pc = block_walk_exact(d, len - 4, (uint64_t)entries_end, K, nn, us,
                              [](uint64_t, uint32_t, uint32_t, uint32_t) {});
      st.n = __shfl_sync(0xFFFFFFFFu, nn, 0);
      st.pcode = __shfl_sync(0xFFFFFFFFu, pc, 0);
      st.unsup = __shfl_sync(0xFFFFFFFFu, us, 0);
    }
  }
  return st;
}

// Mode-1 records. Lane i of chunk q owns slot (interval 2q + i/16, entry
// i%16): restart entries have shared == 0, so a lane's shared prefix always
// comes from lanes of its own interval at or below it, and byte j of an entry
// is written by the LAST lane <= it whose shared <= j — one ballot per
// prefix byte, no scan, no carry between chunks (each starts at a restart).
// Headers are validated (canonical form, shared + unshared == K) before any
// record is written; returns false (nothing written) if one is not.
template <int W>
__device__ __forceinline__ bool dec_fast_records(const DecodeArgs<W>& a, const DecState& st, uint64_t base,
                                                 const uint8_t* d, const uint32_t* pos32, uint32_t pos_base) {
  constexpr int NW = 2 * W + 2;
  const uint32_t lane = lane_id();
  const uint32_t K = a.K, L = K - 8;
  const uint32_t nres = st.nres;
  const uint32_t nchunks = (nres + 1) / 2;
  const uint32_t lt = (1u << lane) - 1u;
  DEC_T0();
  auto slot = [&](uint32_t q, uint32_t& pos, uint32_t& w, uint32_t& j) -> bool {
    const uint32_t k = 2 * q + (lane >> 4);
    j = lane & 15u;
    const int32_t ck = __shfl_sync(0xFFFFFFFFu, st.my_cnt, k < 32 ? k : 31);
    const bool act = k < nres && (int32_t)j < ck;
    pos = act ? pos32[kDecStride * k + j] - pos_base : 0u;  // staged slots hold shared addresses
    w = act ? ld_u32_any(d + pos) : 0u;
    return act;
  };
  // Canonical header (1-byte shared / unshared, 1-2 byte value length), restart
  // entries unshared, and the key length: the job's K, or for var records
  // (generic-length keys) 8..8W+7 bytes with shared <= the previous key's
  // length (decode_data_block's "truncated block entry" check). pk: the
  // previous entry's key length (lane - 1, same interval when j > 0).
  auto bad_of = [&](uint32_t w, uint32_t j, uint32_t pk) -> uint32_t {
    const uint32_t s = w & 0xFFu, u = prmt(w, 0u, 0x4441u), two = (w >> 23) & 1u;
    uint32_t klen_bad;
    if (is_var<W>()) klen_bad = (s + u < 8u) | (s + u - 8u > var_maxlen<W>()) | (j > 0 && s > pk);
    else klen_bad = (s + u) ^ K;
    return (w & 0x8080u) | (two & (w >> 31)) | klen_bad | (j == 0 ? s : 0u);
  };
  auto prev_klen = [&](uint32_t w, bool act) -> uint32_t {  // all lanes call
    const uint32_t ku = act ? (w & 0xFFu) + prmt(w, 0u, 0x4441u) : 0u;
    return is_var<W>() ? __shfl_up_sync(0xFFFFFFFFu, ku, 1) : 0u;
  };
  if (nchunks > 1) {  // validate every chunk before the first record is written
    uint32_t bad = 0;
    for (uint32_t q = 0; q < nchunks; ++q) {
      uint32_t pos, w, j;
      const bool act = slot(q, pos, w, j);
      const uint32_t pk = prev_klen(w, act);
      if (act) bad |= bad_of(w, j, pk);
    }
    if (__any_sync(0xFFFFFFFFu, bad != 0)) return false;
  }
  uint64_t e0 = base;
  for (uint32_t q = 0; q < nchunks; ++q) {
    uint32_t pos, w, j;
    const bool act = slot(q, pos, w, j);
    DEC_T(4);
    if (nchunks == 1) {
      const uint32_t pk = prev_klen(w, act);
      if (__any_sync(0xFFFFFFFFu, act && bad_of(w, j, pk) != 0)) return false;
    }
    DEC_T(5);
    const uint32_t s = act ? (w & 0xFFu) : 0u;
    const uint32_t two = (w >> 23) & 1u;
    const uint32_t v1 = prmt(w, 0u, 0x4442u);
    const uint32_t vl = two ? ((v1 & 0x7Fu) | ((w >> 17) & 0x7F80u)) : v1;
    const uint32_t kpos = pos + 3u + two;  // key suffix
    // key bytes [0, K) as LE words from V = key suffix - shared (prefix bytes are garbage until resolved)
    uint32_t kw[NW];
    {
      const uint8_t* V = d + kpos - s;
      const uint32_t mis = (uint32_t)(reinterpret_cast<uintptr_t>(V) & 3u);
      const uint32_t* wp = reinterpret_cast<const uint32_t*>(V - mis);
      const uint32_t sh = mis * 8u;
      uint32_t lo = act ? wp[0] : 0u;
#pragma unroll
      for (int i = 0; i < NW; ++i) {
        const uint32_t hi = act ? wp[i + 1] : 0u;
        kw[i] = __funnelshift_r(lo, hi, sh);
        lo = hi;
      }
    }
    DEC_T(6);
    const uint32_t smax = __reduce_max_sync(0xFFFFFFFFu, s);
    uint32_t fixed[NW];
#pragma unroll
    for (int i = 0; i < NW; ++i) fixed[i] = kw[i];
#pragma unroll
    for (int wi = 0; wi < NW; ++wi) {
      if ((uint32_t)(4 * wi) < smax) {  // warp-uniform; the 4 bytes of a word are independent (straight-line)
        uint32_t src[4], sw[4];
#pragma unroll
        for (int bb = 0; bb < 4; ++bb) {
          const uint32_t wm = __ballot_sync(0xFFFFFFFFu, act && s <= (uint32_t)(4 * wi + bb));
          const uint32_t mine = wm & (lt | (1u << lane));
          src[bb] = mine ? 31u - __clz(mine) : lane;
        }
#pragma unroll
        for (int bb = 0; bb < 4; ++bb) sw[bb] = __shfl_sync(0xFFFFFFFFu, kw[wi], src[bb]);
        uint32_t f = fixed[wi];
        f = s > (uint32_t)(4 * wi + 0) ? prmt(f, sw[0], 0x3214u) : f;
        f = s > (uint32_t)(4 * wi + 1) ? prmt(f, sw[1], 0x3250u) : f;
        f = s > (uint32_t)(4 * wi + 2) ? prmt(f, sw[2], 0x3610u) : f;
        f = s > (uint32_t)(4 * wi + 3) ? prmt(f, sw[3], 0x7210u) : f;
        fixed[wi] = f;
      }
    }
    DEC_T(7);
    const uint32_t m = __ballot_sync(0xFFFFFFFFu, act);
    if (act) {
      Rec<W> r;
      const uint32_t u = prmt(w, 0u, 0x4441u);  // unshared (== K - s on the fixed path)
      if (is_var<W>()) {
        const uint32_t Lr = s + u - 8u;
        words_to_rec<W, NW>(fixed, Lr, r);
        r.k[W - 1] |= Lr;  // the length byte (byte 8W-1 is padding: Lr <= 8W-1)
      } else {
        words_to_rec<W, NW>(fixed, L, r);
      }
      r.h = handle_pack(st.addr + kpos + u, vl);
      a.out[e0 + __popc(m & lt)] = r;
    }
    e0 += __popc(m);
    DEC_T(8);
  }
  return true;
}

// Phase 2 (parse warp): reference errors of the walk, then records at
// out[base ...]. The CRC is verified concurrently by the pair's CRC warp
// (B_CRC ranks before every parse error of the same block, so the min-reduced
// error code keeps the reference order: length, CRC, restarts, entries).
template <int W, bool kStaged>
__device__ __forceinline__ void dec_phase2(const DecodeArgs<W>& a, uint32_t b, DecState& st, uint64_t base,
                                           uint64_t cap, const uint8_t* d, DecSlot* slots) {
  constexpr int NW = 2 * W + 2;
  const uint32_t lane = lane_id();
  const uint32_t K = a.K;
  const uint32_t len = st.len;
  uint32_t code = st.code;
  if (!code) code = st.restart_bad ? (uint32_t)B_RESTART : st.pcode;
  const uint64_t n = st.n;
  if (code || st.unsup || base + n > cap) {
    if (lane == 0 && code) atomicMin(a.err_ref, ((unsigned long long)b << 8) | code);
    if (lane == 0 && !code && st.unsup) atomicMin(a.err_unsup, ((unsigned long long)b << 8) | st.unsup);
    return;
  }
  if (LUDA_ABLATE(a, 2)) return;
  const uint32_t L = K - 8;
  if (st.mode == 1) {
    if (dec_fast_records<W>(a, st, base, d, reinterpret_cast<const uint32_t*>(slots), kStaged ? smem_u32(d) : 0u))
      return;
    // a header outside the canonical form: the exact sequential path decides
    uint64_t nn = 0;
    uint32_t pc = 0, us = 0;
    if (lane == 0)
      pc = block_walk_exact(d, len - 4, (uint64_t)st.entries_end, K, nn, us,
                            [](uint64_t, uint32_t, uint32_t, uint32_t) {});
    st.n = __shfl_sync(0xFFFFFFFFu, nn, 0);
    st.pcode = __shfl_sync(0xFFFFFFFFu, pc, 0);
    st.unsup = __shfl_sync(0xFFFFFFFFu, us, 0);
    st.mode = 3;
    if (st.pcode || st.unsup || base + st.n > cap) {
      if (lane == 0 && st.pcode) atomicMin(a.err_ref, ((unsigned long long)b << 8) | st.pcode);
      if (lane == 0 && !st.pcode && st.unsup) atomicMin(a.err_unsup, ((unsigned long long)b << 8) | st.unsup);
      return;
    }
  }
  const int mode = st.mode;
  const uint32_t nres = st.nres;
  uint32_t carry[NW];
#pragma unroll
  for (int i = 0; i < NW; ++i) carry[i] = 0;
  const uint64_t wstep = (uint64_t)kDecSlots;
  const uint64_t nall = st.n;
  for (uint64_t w0 = 0; w0 < nall; w0 += wstep) {
    const uint64_t w1 = w0 + kDecSlots;
    {
      auto put = [&](uint64_t j, uint32_t pos, uint32_t s, uint32_t vl) {
        if (j >= w0 && j < w1) slots[j - w0] = DecSlot{pos, (vl << 8) | s};
      };
      __syncwarp();
      if (mode == 2) {
        if (lane < nres && (uint64_t)(st.my_pre + st.my_cnt) > w0 && (uint64_t)st.my_pre < w1) {
          const int32_t pre = st.my_pre;
          interval_walk(d, st.my_st, st.my_en, K, [&](int32_t j, uint32_t pos, uint32_t s, uint32_t vl) {
            put((uint64_t)(pre + j), pos, s, vl);
          });
        }
      } else if (lane == 0) {
        uint64_t nn;
        uint32_t us;
        block_walk_exact(d, len - 4, (uint64_t)st.entries_end, K, nn, us, put);
      }
    }
    __syncwarp();
    const uint32_t wn = (uint32_t)((nall - w0) < wstep ? (nall - w0) : wstep);
    for (uint32_t c0 = 0; c0 < wn; c0 += 32) {
      const uint32_t e = c0 + lane;
      const bool act = e < wn;
      const uint32_t sidx = e;
      const DecSlot sl = act ? slots[sidx] : DecSlot{0, 0};
      const uint32_t s = sl.sv & 0xFFu;
      const uint32_t vl = sl.sv >> 8;
      uint32_t kw[NW];
      {
        const uint8_t* V = d + sl.pos - s;  // key byte i at V + i
        const uint32_t mis = (uint32_t)(reinterpret_cast<uintptr_t>(V) & 3u);
        const uint32_t* wp = reinterpret_cast<const uint32_t*>(V - mis);
        const uint32_t sh = mis * 8u;
        uint32_t lo = act ? wp[0] : 0u;
#pragma unroll
        for (int i = 0; i < NW; ++i) {
          const uint32_t hi = act ? wp[i + 1] : 0u;
          kw[i] = __funnelshift_r(lo, hi, sh);
          lo = hi;
        }
      }
      uint32_t v = act ? s : 0u;  // bytes [v, K) valid
      // only words below the largest shared prefix of the chunk need filling
      const uint32_t nwf = (__reduce_max_sync(0xFFFFFFFFu, v) + 3u) >> 2;
      if (lane == 0 && v) {
#pragma unroll
        for (int i = 0; i < NW; ++i) {
          const uint32_t keep = byte_keep_mask(v, i);
          kw[i] = (kw[i] & keep) | (carry[i] & ~keep);
        }
        v = 0;
      }
#pragma unroll
      for (int dd = 1; dd < 32; dd <<= 1) {
        if (!__any_sync(0xFFFFFFFFu, v != 0)) break;
        const uint32_t ov = __shfl_up_sync(0xFFFFFFFFu, v, dd);
        const bool take = lane >= (uint32_t)dd && v;
#pragma unroll
        for (int i = 0; i < NW; ++i) {
          if ((uint32_t)i < nwf) {  // warp-uniform
            const uint32_t ow = __shfl_up_sync(0xFFFFFFFFu, kw[i], dd);
            const uint32_t keep = byte_keep_mask(v, i);
            if (take) kw[i] = (kw[i] & keep) | (ow & ~keep);
          }
        }
        if (take) v = ov < v ? ov : v;
      }
#pragma unroll
      for (int i = 0; i < NW; ++i) carry[i] = __shfl_sync(0xFFFFFFFFu, kw[i], wn - c0 >= 32 ? 31 : wn - c0 - 1);
      if (act) {
        Rec<W> r;
        words_to_rec<W, NW>(kw, L, r);
        const uint64_t voff = st.addr + sl.pos + (K - s);
        r.h = handle_pack(voff, vl);
        a.out[base + w0 + e] = r;
      }
    }
  }
}

// Var jobs (keys of any length <= 71 bytes): lane 0 walks the block exactly
// like decode_data_block (blocks.py:151-164: sequential, restart offsets
// ignored, the same error order), rebuilds every internal key in `kbuf`
// (prev[:shared] ∥ key bytes) and writes kVarW records (luda_rec.cuh).
// Returns the block's entry count (records beyond `cap` are not written; the
// host re-runs with a larger segment capacity).
template <int W>
__device__ uint64_t dec_var_block(const DecodeArgs<W>& a, uint32_t b, uint64_t addr, uint32_t len, const uint8_t* d,
                                  uint64_t base, uint64_t cap, uint8_t* kbuf) {
  uint64_t n = 0;
  uint32_t code = 0, unsup = 0;
  if (lane_id() == 0) {
    if (len < 12) {
      code = B_SHORT;
    } else {
      const uint32_t nres = ld_u32_le(d + len - 8);
      const int64_t entries_end = (int64_t)len - 8 - 4 * (int64_t)nres;
      if (nres < 1 || entries_end < 0) {
        code = B_RESTART;
      } else {
        const uint64_t payload = len - 4, ee = (uint64_t)entries_end;
        uint64_t pos = 0, prev_len = 0;
        while (pos < ee) {
          uint64_t sh, u, vl;
          int r;
          if ((r = varint_read(d, payload, pos, sh)) || (r = varint_read(d, payload, pos, u)) ||
              (r = varint_read(d, payload, pos, vl))) {
            code = r == 1 ? B_VARINT_TRUNC : B_VARINT_LONG;
            break;
          }
          if (sh > prev_len || u > ee || vl > ee || pos + u + vl > ee) {
            code = B_TRUNC_ENTRY;
            break;
          }
          const uint64_t ke = sh + u;
          if (ke < 8 || ke - 8 > var_maxlen<W>()) unsup = unsup ? unsup : (uint32_t)B_KEYLONG;
          if (vl > kMaxValueLen) unsup = unsup ? unsup : (uint32_t)B_VALUE_BIG;
          if (!unsup) {
            for (uint32_t j = 0; j < (uint32_t)u; ++j) kbuf[sh + j] = d[pos + j];
            if (base + n < cap) {
              const uint32_t lr = (uint32_t)ke - 8;
              Rec<W> rec;
#pragma unroll
              for (int w = 0; w < W; ++w) {
                // big-endian word of kbuf[8w, 8w+8), bytes at or past the key length masked off
                // (explicit word masks: with a per-byte `idx < lr ? kbuf[idx] : 0` select the
                // nvcc 12.9 -O3 build left byte 8w+2 of the last word unmasked — observed on
                // B200, tests/test_gpu_parity.py::test_var_key_prefix_extension)
                uint64_t v = 0;
#pragma unroll
                for (int q = 0; q < 8; ++q) v = (v << 8) | kbuf[8 * w + q];
                const int32_t valid = (int32_t)lr - 8 * w;
                v = valid <= 0 ? 0ull : (valid >= 8 ? v : v & (~0ull << (8 * (8 - valid))));
                rec.k[w] = v;
              }
              rec.k[W - 1] |= lr;  // byte 71: the length (always padding: lr <= 71)
              uint64_t tr = 0;
              for (int q = 7; q >= 0; --q) tr = (tr << 8) | kbuf[lr + q];
              rec.t = ~tr;
              rec.h = handle_pack(addr + pos + u, vl);
              a.out[base + n] = rec;
            }
          }
          prev_len = ke;
          pos += u + vl;
          ++n;
        }
        if (!code && pos != ee) code = B_TRAILING;
      }
    }
  }
  n = __shfl_sync(0xFFFFFFFFu, n, 0);
  code = __shfl_sync(0xFFFFFFFFu, code, 0);
  unsup = __shfl_sync(0xFFFFFFFFu, unsup, 0);
  if (lane_id() == 0 && code) atomicMin(a.err_ref, ((unsigned long long)b << 8) | code);
  if (lane_id() == 0 && !code && unsup) atomicMin(a.err_unsup, ((unsigned long long)b << 8) | unsup);
  return code || unsup ? 0 : n;
}

// CRC-32 of a staged block's payload [data, data + n), n >= 4, WITHOUT
// touching any byte the parse warp reads: the <= 15 garbage bytes between
// the TMA window start and `data` and the <= 3 stored-CRC bytes after the
// payload are zeroed (the slot lead before the window is always zero), the
// range is extended to a word-aligned end, raw(0, D) is recovered with
// Z_{-pad}, and the ~0 preset is added back as Z_n(~0) (g_zone table).
__device__ __forceinline__ uint32_t dec_crc_staged(uint8_t* win, uint8_t* data, uint32_t n, const CrcSmem& cs) {
  const uint32_t lane = lane_id();
  const uint32_t zone = crc_zone(n);  // global load issued first: its latency hides under the passes
  const uint32_t pre = (uint32_t)(data - win);
  if (lane < pre) win[lane] = 0;
  const uint32_t pad = (uint32_t)(0u - (uint32_t)reinterpret_cast<uintptr_t>(data + n)) & 3u;
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
  if (pad) acc = crc_unshift(acc, pad);
  return ~(acc ^ zone);
}

template <int W>
__global__ void __launch_bounds__(kDecWarps * 32, 1) decode_kernel(DecodeArgs<W> a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  CrcSmem& cs = *reinterpret_cast<CrcSmem*>(smem_raw);
  DecPairSmem* pairs = reinterpret_cast<DecPairSmem*>(smem_raw + sizeof(CrcSmem));
  DecCtaSmem& cta = *reinterpret_cast<DecCtaSmem*>(smem_raw + sizeof(CrcSmem) + kDecPairs * sizeof(DecPairSmem));
  const uint32_t lane = lane_id();
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t p = warp % kDecPairs;
  const bool parse = warp < kDecPairs;
  DecPairSmem& ps = pairs[p];
#ifdef LUDA_DEC_CTA_TIMES  // per-CTA start/end timestamps (experiment builds: profiles/cta_times.py)
  uint64_t t_start = 0;
  if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
#endif
  crc_smem_init(cs);
  constexpr int kLeadChunks = kDecLead / 16;
  for (uint32_t i = threadIdx.x; i < kDecPairs * kDecNSlot * kLeadChunks; i += blockDim.x) {
    const uint32_t q = i / (kDecNSlot * kLeadChunks), r = i % (kDecNSlot * kLeadChunks);
    reinterpret_cast<uint4*>(pairs[q].slot[r / kLeadChunks])[r % kLeadChunks] = make_uint4(0, 0, 0, 0);
  }
  if (threadIdx.x == 0) cta.lock = 0;
  if (parse && lane == 0) {
    for (int s = 0; s < kDecNSlot; ++s) {
      mbar_init(&ps.full[s], 1);
      mbar_init(&ps.empty[s], 2);
    }
  }
  __syncthreads();
  // Work distribution: the blocks are cut into a.nseg contiguous chunks (the
  // record segments); each pair takes chunks from a global counter, in
  // order, and its blocks run through the pair's slot pipeline as one
  // sequence (a chunk never straddles a pipeline restart). Dynamic chunks
  // keep every SM busy to the end even when a CTA starts late or a chunk
  // decodes slower than another (static per-pair ranges measured a 2x
  // step when one CTA could not be placed until another had finished).
  if (parse) {
    // Producer cursor: chunk pc, its blocks [pb, pe). Block-table entries are
    // fetched 32 blocks at a time (lane j holds block kb + j) so no global
    // load sits on the per-block path.
    uint32_t pc = 0, pb = 0, pe = 0;
    uint32_t kb = 0xFFFFFFFFu;
    uint64_t t_addr = 0;
    uint32_t t_len = 0;
    uint32_t total = 0xFFFFFFFFu;  // pipeline length, known once the chunks ran out
    auto next_block = [&](uint32_t& b, uint32_t& c) -> bool {  // warp-uniform
      while (pb >= pe) {
#ifdef LUDA_DEC_STATIC_CHUNKS  // experiment: chunk g, g + np, ... (no counter)
        const uint32_t nc = pe == 0 ? blockIdx.x * kDecPairs + p : pc + gridDim.x * kDecPairs;
        pe = 1;
#else
        uint32_t nc = 0;
        if (lane == 0) nc = atomicAdd(a.chunk_ctr, 1u);
        nc = __shfl_sync(0xFFFFFFFFu, nc, 0);
#endif
        if (nc >= a.nseg) return false;
        pc = nc;
        pb = seg_first_block(nc, a.nblk, a.nseg);
        pe = seg_first_block(nc + 1, a.nblk, a.nseg);
        if (pb >= pe && lane == 0) a.seg_count[nc] = 0;  // empty chunk (nblk < nseg)
      }
      b = pb++;
      c = pc;
      return true;
    };
    auto issue = [&](uint32_t k) {
      const uint32_t s = k % kDecNSlot;
      uint32_t bj = 0, c = 0;
      const bool have = next_block(bj, c);
      if (have && (kb == 0xFFFFFFFFu || bj < kb || bj >= kb + 32)) {
        kb = bj;
        const uint32_t bl = bj + lane;
        t_addr = bl < a.nblk ? a.bt.addr[bl] : 0;
        t_len = bl < a.nblk ? a.bt.len[bl] : 0;
      }
      const uint64_t addr = __shfl_sync(0xFFFFFFFFu, t_addr, (bj - kb) & 31u);
      const uint32_t len = __shfl_sync(0xFFFFFFFFu, t_len, (bj - kb) & 31u);
      if (!have) total = k;
      if (lane == 0) {
        if (k >= kDecNSlot) mbar_wait(&ps.empty[s], ((k - kDecNSlot) / kDecNSlot) & 1u);
        if (!have) {  // end marker for the CRC warp
          ps.meta[s] = DecSlotMeta{0, 0, kDecEnd};
          mbar_arrive(&ps.full[s]);
          return;
        }
        const uint8_t* gp = a.arena + addr;
        const uint32_t win = dec_window(gp, len);
        const bool st = len >= 12 && win <= (uint32_t)kDecStage;
        ps.meta[s] = DecSlotMeta{addr, len, bj | (st ? 0x80000000u : 0u)};
        if (st) {
          fence_proxy_async_smem();
          mbar_arrive_expect_tx(&ps.full[s], win);
          bulk_g2s(ps.slot[s] + kDecLead, reinterpret_cast<const void*>(reinterpret_cast<uintptr_t>(gp) & ~uintptr_t(15)),
                   win, &ps.full[s]);
        } else {
          mbar_arrive(&ps.full[s]);
        }
      }
    };
    DecSlot* slots = reinterpret_cast<DecSlot*>(ps.entries);
    uint32_t cur = 0xFFFFFFFFu, cur_end = 0, issued = 0;
    uint64_t seg0 = 0, seg1 = 0, cnt = 0;
    for (uint32_t k = 0;; ++k) {
      // keep kDecNSlot blocks in flight (one issue site: the kernel is
      // instruction-cache sensitive)
      while (issued < k + kDecNSlot && total == 0xFFFFFFFFu) issue(issued++);
      if (k >= total) break;
      const uint32_t s = k % kDecNSlot;
      mbar_wait(&ps.full[s], (k / kDecNSlot) & 1u);
      const DecSlotMeta mt = ps.meta[s];
      const uint32_t b = mt.blk();
      if (b >= cur_end) {  // the pair's next chunk (its blocks follow each other within a chunk)
        if (cur != 0xFFFFFFFFu && lane == 0) a.seg_count[cur] = cnt;
        cur = seg_of_block(b, a.nblk, a.nseg);
        cur_end = seg_first_block(cur + 1, a.nblk, a.nseg);
        seg0 = (uint64_t)cur * a.seg_cap;
        seg1 = seg0 + a.seg_cap;
        cnt = 0;
      }
      const uint8_t* gp = a.arena + mt.addr;
      if (lane == 0) a.blk_local[b] = (uint32_t)cnt;
      uint64_t n = 0;
      if (is_var<W>()) {
        const uint8_t* d = mt.staged() ? ps.slot[s] + kDecLead + (reinterpret_cast<uintptr_t>(gp) & 15) : gp;
        bool fast = false;
        if (W == kVarW && mt.staged()) {
          // the fixed path's positions walk + lane-per-entry records, with a
          // key length per entry; anything outside its envelope (or an error)
          // goes through the exact sequential walk below
          DecState stt = dec_phase1<W, true>(a, b, mt.addr, mt.len, d, slots);
          if (stt.mode == 1 && !stt.code && !stt.restart_bad && seg0 + cnt + stt.n <= seg1 &&
              dec_fast_records<W>(a, stt, seg0 + cnt, d, reinterpret_cast<const uint32_t*>(slots), smem_u32(d))) {
            n = stt.n;
            fast = true;
          }
        }
        if (!fast) n = dec_var_block<W>(a, b, mt.addr, mt.len, d, seg0 + cnt, seg1, ps.entries);
      } else if (!LUDA_ABLATE(a, 4)) {
        if (mt.staged()) {
          const uint8_t* d = ps.slot[s] + kDecLead + (reinterpret_cast<uintptr_t>(gp) & 15);
          DecState stt = dec_phase1<W, true>(a, b, mt.addr, mt.len, d, slots);
          dec_phase2<W, true>(a, b, stt, seg0 + cnt, seg1, d, slots);
          n = stt.n;
        } else {
          DecState stt = dec_phase1<W, false>(a, b, mt.addr, mt.len, gp, slots);
          dec_phase2<W, false>(a, b, stt, seg0 + cnt, seg1, gp, slots);
          n = stt.n;
        }
      }
      cnt += n;
      fence_proxy_async_smem();  // this lane's generic slot accesses before the next TMA into it
      __syncwarp();
      if (lane == 0) mbar_arrive(&ps.empty[s]);
    }
    if (cur != 0xFFFFFFFFu && lane == 0) a.seg_count[cur] = cnt;
  } else {
    // CRC warp: verify every block of the pair's sequence (reference: before
    // parsing), up to the producer's end marker
    for (uint32_t k = 0;; ++k) {
      const uint32_t s = k % kDecNSlot;
      mbar_wait(&ps.full[s], (k / kDecNSlot) & 1u);
      const DecSlotMeta mt = ps.meta[s];
      if (mt.tag == kDecEnd) break;
      const uint32_t b = mt.blk();
      const bool st_ok = mt.staged();
      const uint32_t len = mt.len;
      if (len >= 12 && !LUDA_ABLATE(a, 1)) {
        const uint8_t* gp = a.arena + mt.addr;
        uint32_t crc, stored;
        if (st_ok) {
          uint8_t* wstart = ps.slot[s] + kDecLead;
          uint8_t* d = wstart + (reinterpret_cast<uintptr_t>(gp) & 15);
          stored = ld_u32_any(d + len - 4);
          __syncwarp();
          crc = dec_crc_staged(wstart, d, len - 4, cs);
        } else {
          // rare large block: CRC passes staged through the CTA's shared buffer
          stored = ld_u32_le(gp + len - 4);
          if (lane == 0)
            while (atomicCAS(&cta.lock, 0, 1) != 0) __nanosleep(64);
          __syncwarp();
          const uint64_t npass = ((uint64_t)len - 4 + kGroup - 1) / kGroup;
          uint32_t raw = 0;
          for (uint64_t q = 0; q < npass; ++q) raw ^= warp_crc_pass_global(gp, len - 4, q, cta.big, cs);
          crc = ~raw;
          __syncwarp();
          if (lane == 0) atomicExch(&cta.lock, 0);
        }
        if (lane == 0 && crc != stored) atomicMin(a.err_ref, ((unsigned long long)b << 8) | B_CRC);
      }
      fence_proxy_async_smem();  // this lane's generic slot accesses before the next TMA into it
      __syncwarp();
      if (lane == 0) mbar_arrive(&ps.empty[s]);
    }
  }
#ifdef LUDA_DEC_CTA_TIMES
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t t_end;
    uint32_t smid;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    printf("CTAT %u %u %llu %llu\n", blockIdx.x, smid, (unsigned long long)t_start, (unsigned long long)t_end);
  }
#endif
}

// Segment starts (logical record index): exclusive scan of the segment
// counts (one CTA; nw <= a few thousand).
__global__ void seg_scan_kernel(const uint64_t* count, uint32_t nw, uint64_t* lo, uint64_t* max_count) {
  __shared__ uint64_t s_carry;
  __shared__ uint64_t s_warp[32];
  if (threadIdx.x == 0) s_carry = 0;
  uint64_t mx = 0;
  __syncthreads();
  for (uint32_t c0 = 0; c0 < nw; c0 += blockDim.x) {
    const uint32_t i = c0 + threadIdx.x;
    const uint64_t v = i < nw ? count[i] : 0;
    mx = v > mx ? v : mx;
    const uint64_t incl = warp_incl_scan<uint64_t>(v);
    const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
    if (lane == 31) s_warp[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      const uint64_t x = lane < blockDim.x / 32 ? s_warp[lane] : 0;
      const uint64_t xi = warp_incl_scan<uint64_t>(x);
      if (lane < blockDim.x / 32) s_warp[lane] = xi - x;
    }
    __syncthreads();
    if (i < nw) lo[i] = s_carry + s_warp[wid] + incl - v;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) s_carry += s_warp[wid] + incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) lo[nw] = s_carry;
  mx = warp_max<uint64_t>(mx);
  if (lane_id() == 0) atomicMax(reinterpret_cast<unsigned long long*>(max_count), (unsigned long long)mx);
}

// First record index (logical) of every file: its first block's segment
// start + the block's local base; file nfiles = total.
__global__ void file_entry_base_kernel(const uint32_t* blk_local, const uint64_t* seg_lo, uint32_t nblk, uint32_t nw,
                                       const uint32_t* file_blk_base, uint32_t nfiles, uint64_t* out) {
  const uint32_t f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f > nfiles) return;
  const uint32_t b = file_blk_base[f];
  out[f] = b >= nblk ? seg_lo[nw] : seg_lo[seg_of_block(b, nblk, nw)] + blk_local[b];
}

}  // namespace luda
