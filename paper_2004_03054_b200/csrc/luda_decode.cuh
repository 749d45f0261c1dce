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
};

constexpr int kDecWarps = 14;
constexpr int kDecStage = 4352;                  // staged window bytes (block + alignment)
constexpr int kDecPre = 160;                     // CRC lead-in before the data
constexpr int kDecBuf = kDecPre + kDecStage + 64;
constexpr int kDecSlots = 128;
constexpr int kDecStride = 16;                   // slots per restart interval (single-walk path)
constexpr int kDecWarpBytes = 2 * kDecBuf + kDecSlots * 8 + 16;  // 2 staging buffers, 1 slot array
static_assert(sizeof(CrcSmem) + kDecWarps * kDecWarpBytes <= 232448, "decode smem over the 227 KB limit");

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
  Rec<W>* out;              // segmented: warp w writes out[w * seg_cap ...]
  uint64_t seg_cap;         // records per warp segment
  uint32_t* blk_local;      // out [nblk]: block's first record index within its warp segment
  uint64_t* seg_count;      // out [nwarps]: records of each warp segment (may exceed seg_cap → rerun)
  unsigned long long* err_ref;
  unsigned long long* err_unsup;
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
template <typename Emit>
__device__ __forceinline__ int32_t interval_walk(const uint8_t* d, uint32_t start, uint32_t end, uint32_t K,
                                                 Emit emit) {
  uint32_t pos = start;
  int32_t j = 0;
  while (pos < end) {
    const uint32_t b0 = d[pos], b1 = d[pos + 1], b2 = d[pos + 2], b3 = d[pos + 3];
    uint32_t vl, hl;
    if (((b0 | b1 | b2) & 0x80u) == 0) {
      vl = b2;
      hl = 3;
    } else if (((b0 | b1 | b3) & 0x80u) == 0) {
      vl = (b2 & 0x7Fu) | (b3 << 7);
      hl = 4;
    } else {
      return -1;
    }
    if ((j == 0 && b0 != 0) || b0 + b1 != K) return -1;
    const uint32_t np = pos + hl + b1 + vl;
    if (np > end) return -1;
    emit(j, pos + hl, b0, vl);
    pos = np;
    ++j;
  }
  return j;
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

constexpr int kDecTile = 2;  // staging buffers per warp (double buffer)

// Per-warp smem layout (offsets from the warp's base `wb`, all smem-derived
// pointers so the compiler emits LDS/STS):
//   [0, kDecBuf)            staging buffer 0
//   [kDecBuf, 2 kDecBuf)    staging buffer 1
//   [2 kDecBuf, +1 KB)      entry slots
//   then 2 mbarriers
__device__ __forceinline__ uint8_t* dec_buf(uint8_t* wb, int which) { return wb + which * kDecBuf; }
__device__ __forceinline__ DecSlot* dec_slots(uint8_t* wb) { return reinterpret_cast<DecSlot*>(wb + kDecTile * kDecBuf); }
__device__ __forceinline__ uint64_t* dec_bar(uint8_t* wb, int which) {
  return reinterpret_cast<uint64_t*>(wb + kDecTile * kDecBuf + kDecSlots * 8) + which;
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

// Issue the TMA staging of block b into buffer `which` (lane 0). Returns
// whether the block is staged (else it is read in place).
template <int W>
__device__ __forceinline__ bool dec_prefetch(const DecodeArgs<W>& a, uint32_t b, uint8_t* wb, int which) {
  if (b >= a.nblk) return false;
  const uint32_t len = a.bt.len[b];
  const uint8_t* g = a.arena + a.bt.addr[b];
  const uint32_t win = dec_window(g, len);
  if (len < 12 || win > (uint32_t)kDecStage) return false;
  if (lane_id() == 0) {
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(dec_bar(wb, which), win);
    bulk_g2s(dec_buf(wb, which) + kDecPre,
             reinterpret_cast<const void*>(reinterpret_cast<uintptr_t>(g) & ~uintptr_t(15)), win,
             dec_bar(wb, which));
  }
  return true;
}

// Phase 1: structural checks + entry walk (counts; single-walk fills slots).
template <int W>
__device__ __forceinline__ DecState dec_phase1(const DecodeArgs<W>& a, uint32_t b, const uint8_t* d,
                                               DecSlot* slots) {
  const uint32_t lane = lane_id();
  DecState st{};
  st.len = a.bt.len[b];
  st.addr = a.bt.addr[b];
  const uint32_t K = a.K;
  const uint32_t len = st.len;
  st.code = len < 12 ? (uint32_t)B_SHORT : 0u;
  if (!st.code) {
    st.nres = ld_u32_le(d + len - 8);
    st.entries_end = (int64_t)len - 8 - 4 * (int64_t)st.nres;
    st.restart_bad = st.nres < 1 || st.entries_end < 0;
  }
  st.mode = 3;
  if (!st.code && !st.restart_bad) {
    const uint32_t nres = st.nres;
    const int64_t entries_end = st.entries_end;
    if (nres <= 32) {
      bool ok = true;
      const bool single = nres <= (uint32_t)(kDecSlots / kDecStride);
      if (lane < nres) {
        st.my_st = ld_u32_le(d + entries_end + 4 * lane);
        st.my_en = (lane + 1 < nres) ? ld_u32_le(d + entries_end + 4 * (lane + 1)) : (uint32_t)entries_end;
        ok = (lane != 0 || st.my_st == 0) && st.my_st < st.my_en && (int64_t)st.my_en <= entries_end;
        if (ok) {
          DecSlot* mine = slots + kDecStride * lane;
          st.my_cnt = interval_walk(d, st.my_st, st.my_en, K, [&](int32_t j, uint32_t pos, uint32_t s, uint32_t vl) {
            if (single && j < kDecStride) mine[j] = DecSlot{pos, (vl << 8) | s};
          });
          ok = st.my_cnt >= 0;
        }
      }
      if (__all_sync(0xFFFFFFFFu, ok)) {
        const int32_t c = lane < nres ? st.my_cnt : 0;
        const int32_t incl = warp_incl_scan<int32_t>(c);
        st.my_pre = incl - c;
        st.n = (uint64_t)(uint32_t)__shfl_sync(0xFFFFFFFFu, incl, 31);
        st.mode = (single && __all_sync(0xFFFFFFFFu, c <= kDecStride)) ? 1 : 2;
      }
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

// Phase 2: CRC verify, then records at out[base ...]. kStaged: `d` is the
// smem copy (CRC in place); else the block is read from global memory and its
// CRC staged pass by pass through `stage`.
template <int W, bool kStaged>
__device__ __forceinline__ void dec_phase2(const DecodeArgs<W>& a, uint32_t b, DecState& st, uint64_t base,
                                           uint64_t cap, const uint8_t* d, DecSlot* slots, uint8_t* stage,
                                           const CrcSmem& cs) {
  constexpr int NW = 2 * W + 2;
  const uint32_t lane = lane_id();
  const uint32_t K = a.K;
  const uint32_t len = st.len;
  uint32_t code = st.code;
  if (!code) {
    uint32_t crc;
    if (kStaged) {
      crc = warp_crc32_smem(const_cast<uint8_t*>(d), len - 4, cs);
    } else {
      const uint64_t np = ((uint64_t)len - 4 + kGroup - 1) / kGroup;
      uint32_t raw = 0;
      for (uint64_t q = 0; q < np; ++q) raw ^= warp_crc_pass_global(d, len - 4, q, stage, cs);
      crc = ~raw;
    }
    if (crc != ld_u32_le(d + len - 4)) code = B_CRC;
    else if (st.restart_bad) code = B_RESTART;
    else code = st.pcode;
  }
  const uint64_t n = st.n;
  if (code || st.unsup || base + n > cap) {
    if (lane == 0 && code) atomicMin(a.err_ref, ((unsigned long long)b << 8) | code);
    if (lane == 0 && !code && st.unsup) atomicMin(a.err_unsup, ((unsigned long long)b << 8) | st.unsup);
    return;
  }
  const uint32_t L = K - 8;
  const int mode = st.mode;
  const uint32_t nres = st.nres;
  uint32_t carry[NW];
#pragma unroll
  for (int i = 0; i < NW; ++i) carry[i] = 0;
  const uint64_t wstep = mode == 1 ? n : (uint64_t)kDecSlots;
  for (uint64_t w0 = 0; w0 < n; w0 += wstep) {
    const uint64_t w1 = w0 + kDecSlots;
    if (mode != 1) {
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
    const uint32_t wn = (uint32_t)((n - w0) < wstep ? (n - w0) : wstep);
    for (uint32_t c0 = 0; c0 < wn; c0 += 32) {
      const uint32_t e = c0 + lane;
      const bool act = e < wn;
      uint32_t sidx = e;
      if (mode == 1) {  // entry e lives in interval k with pre_k <= e < pre_{k+1}
        uint32_t k = 0, pk = 0;
        for (uint32_t kk = 1; kk < nres; ++kk) {
          const uint32_t p = (uint32_t)__shfl_sync(0xFFFFFFFFu, (uint32_t)st.my_pre, kk);
          if (p <= e) { k = kk; pk = p; }
        }
        sidx = kDecStride * k + (e - pk);
      }
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
      if (lane == 0 && v) {
#pragma unroll
        for (int i = 0; i < NW; ++i) {
          const int32_t bi = (int32_t)v - 4 * i;
          const uint32_t keep = bi <= 0 ? 0xFFFFFFFFu : (bi >= 4 ? 0u : (0xFFFFFFFFu << (8 * bi)));
          kw[i] = (kw[i] & keep) | (carry[i] & ~keep);
        }
        v = 0;
      }
#pragma unroll
      for (int dd = 1; dd < 32; dd <<= 1) {
        if (!__any_sync(0xFFFFFFFFu, v != 0)) break;
        const uint32_t ov = __shfl_up_sync(0xFFFFFFFFu, v, dd);
        uint32_t ow[NW];
#pragma unroll
        for (int i = 0; i < NW; ++i) ow[i] = __shfl_up_sync(0xFFFFFFFFu, kw[i], dd);
        if (lane >= (uint32_t)dd && v) {
#pragma unroll
          for (int i = 0; i < NW; ++i) {
            const int32_t bi = (int32_t)v - 4 * i;
            const uint32_t keep = bi <= 0 ? 0xFFFFFFFFu : (bi >= 4 ? 0u : (0xFFFFFFFFu << (8 * bi)));
            kw[i] = (kw[i] & keep) | (ow[i] & ~keep);
          }
          v = ov < v ? ov : v;
        }
      }
#pragma unroll
      for (int i = 0; i < NW; ++i) carry[i] = __shfl_sync(0xFFFFFFFFu, kw[i], 31);
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

// `base` = physical record index of the block's first record, `cap` = end of
// the warp's segment; returns the block's entry count.
template <int W, bool kStaged>
__device__ __forceinline__ uint64_t dec_block(const DecodeArgs<W>& a, uint32_t b, uint8_t* wb, int which,
                                              uint32_t& phase, const CrcSmem& cs, uint64_t base, uint64_t cap) {
  uint8_t* buf = dec_buf(wb, which);
  const uint8_t* g = a.arena + a.bt.addr[b];
  const uint8_t* d;
  if (kStaged) {
    mbar_wait(dec_bar(wb, which), (phase >> which) & 1u);
    phase ^= 1u << which;
    d = buf + kDecPre + (reinterpret_cast<uintptr_t>(g) & 15);
  } else {
    d = g;
  }
  DecSlot* slots = dec_slots(wb);
  DecState st = dec_phase1(a, b, d, slots);
  dec_phase2<W, kStaged>(a, b, st, base, cap, d, slots, buf, cs);
  return st.n;
}

template <int W>
__global__ void __launch_bounds__(kDecWarps * 32, 1) decode_kernel(DecodeArgs<W> a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  CrcSmem& cs = *reinterpret_cast<CrcSmem*>(smem_raw);
  uint8_t* wb = smem_raw + sizeof(CrcSmem) + (threadIdx.x >> 5) * kDecWarpBytes;
  const uint32_t lane = lane_id();
  crc_smem_init(cs);
  if (lane == 0) {
    mbar_init(dec_bar(wb, 0), 1);
    mbar_init(dec_bar(wb, 1), 1);
  }
  __syncthreads();
  // Warp segment: a contiguous block range, the next block's TMA staging in
  // flight while the current one is processed.
  const uint32_t nw = gridDim.x * kDecWarps;
  const uint32_t w = blockIdx.x * kDecWarps + (threadIdx.x >> 5);
  const uint32_t b0 = seg_first_block(w, a.nblk, nw), b1 = seg_first_block(w + 1, a.nblk, nw);
  const uint64_t seg0 = (uint64_t)w * a.seg_cap, seg1 = seg0 + a.seg_cap;
  uint64_t cnt = 0;
  uint32_t phase = 0;
  int which = 0;
  bool cur_staged = b0 < b1 && dec_prefetch(a, b0, wb, which);
  for (uint32_t cur = b0; cur < b1; ++cur) {
    const bool nxt_staged = cur + 1 < b1 && dec_prefetch(a, cur + 1, wb, which ^ 1);
    if (lane == 0) a.blk_local[cur] = (uint32_t)cnt;
    cnt += cur_staged ? dec_block<W, true>(a, cur, wb, which, phase, cs, seg0 + cnt, seg1)
                      : dec_block<W, false>(a, cur, wb, which, phase, cs, seg0 + cnt, seg1);
    fence_proxy_async_smem();  // generic smem accesses before the next TMA into this buffer
    __syncwarp();
    cur_staged = nxt_staged;
    which ^= 1;
  }
  if (lane == 0) a.seg_count[w] = cnt;
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
