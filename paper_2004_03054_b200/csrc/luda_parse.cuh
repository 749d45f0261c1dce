// luda_parse.cuh — SST footer / filter / index parsing and range CRCs.
//
// Restates Table.__init__ (sst.py:284-310): footer (last 24 B, <IIIIQ>),
// magic, FilterBlock.decode (bloom.py:57-68: len >= 6, crc, 1 <= k <= 30) and
// decode_index_block (sst.py:79-102: len >= 8, crc, n entries of
// varint klen ∥ key ∥ u32 off ∥ u32 len, no trailing bytes). os.pread short
// reads past EOF are reproduced by clamping every (off, len) to the file.
//
// Stage A (parse_files_a): one warp per file records every reference check
// outcome and the filter/index byte ranges whose CRCs stage B verifies; the
// host then raises the first failure in reference order. Stage C
// (parse_files_c) writes the data-block table (arena address, clamped length,
// file offset, file index) for the decode stage.
#pragma once
#include "luda_common.cuh"

namespace luda {

constexpr uint64_t kMagic = 0x4C55444153535431ull;  // sst.py:42

enum FileCode : uint32_t {
  F_OK = 0,
  F_SHORT = 1,          // file too short for footer
  F_MAGIC = 2,          // bad magic
  F_FILTER_SHORT = 3,   // filter block too short
  F_FILTER_CRC = 4,     // filter block checksum mismatch (Corruption @ filter_off)
  F_FILTER_K = 5,       // bad probe count
  F_INDEX_SHORT = 6,    // index block too short
  F_INDEX_CRC = 7,      // index block checksum mismatch (Corruption @ index_off)
  F_IDX_VARINT_TRUNC = 8,
  F_IDX_VARINT_LONG = 9,
  F_IDX_TRUNC = 10,     // truncated index entry
  F_IDX_TRAILING = 11,  // trailing garbage in index block
};

// Reference check order: code (short/magic/filter short) → filter crc → kbad →
// icode == F_INDEX_SHORT → index crc → icode (parse). CRCs come from stage B.
struct FileInfo {
  uint32_t code;          // F_SHORT / F_MAGIC / F_FILTER_SHORT (stop everything)
  uint32_t kbad;          // probe count byte outside [1, 30]
  uint32_t icode;         // F_INDEX_SHORT or an index parse code
  uint32_t nblocks;       // index entries (valid when parse ok)
  uint32_t klen;          // common index key length; 0xFFFFFFFF if mixed
  uint32_t kbyte;         // filter probe count byte
  uint32_t stride;        // 1: index entries at a fixed stride (every klen byte == klen, < 0x80)
  uint32_t pad_;
  uint64_t filter_off, filter_len;  // clamped, file relative
  uint64_t index_off, index_len;
  uint64_t magic;
};

__device__ __forceinline__ uint32_t ld_u32_le(const uint8_t* p) {
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}
__device__ __forceinline__ uint64_t ld_u64_le(const uint8_t* p) {
  return (uint64_t)ld_u32_le(p) | ((uint64_t)ld_u32_le(p + 4) << 32);
}

// varint.decode (varint.py:28-43) over buf[0,n). Returns 0 ok, 1 truncated,
// 2 too long; values >= 2^64 saturate to ~0 (the reference then fails a
// bounds check downstream, as a Python bigint would).
__device__ __forceinline__ int varint_read(const uint8_t* buf, uint64_t n, uint64_t& pos, uint64_t& out) {
  uint64_t v = 0;
  int shift = 0;
  bool big = false;
  while (true) {
    if (pos >= n) return 1;
    uint32_t b = buf[pos++];
    uint64_t part = (uint64_t)(b & 0x7F);
    if (shift == 63 && part > 1) big = true;
    if (shift < 64) v |= part << shift;
    if (!(b & 0x80)) { out = big ? ~0ull : v; return 0; }
    shift += 7;
    if (shift > 63) return 2;
  }
}

// decode_index_block's sequential walk (sst.py:79-102), by a whole warp
// through a shared-memory window: the lanes load kIdxWin bytes at the current
// entry (coalesced 16-byte granules; a granule holding any payload byte lies
// inside the file's allocation). Lane 0 then chains through the window — for the
// common entry (1-byte varint, entry inside the window and the body) one
// dependent shared-memory byte load per entry — and lists where each entry's
// (off, len) sits; the lanes read and emit those in parallel. Any other entry
// goes through the exact general step (multi-byte varints, errors; off/len
// past the window read from global memory). Checks in the reference's order:
// varint (truncated / too long), entry bounds, then trailing bytes. All lanes
// get the return value / klen (0xFFFFFFFF when the key lengths differ).
constexpr uint32_t kIdxWin = 4096;
constexpr uint32_t kIdxList = kIdxWin / 9 + 1;
struct IdxWalkSmem {
  uint8_t win[kIdxWin + 16];
  uint32_t list[kIdxList];  // (entry - first entry of the window) << 16 | window offset of off/len
};
template <typename Emit>
__device__ int index_walk_warp(const uint8_t* body, uint64_t end, uint32_t n, uint32_t& klen_out, IdxWalkSmem& sm,
                               Emit emit) {
  const uint32_t lane = lane_id();
  const uint64_t pay = end + 4;  // varints may read into the count (payload = body ∥ count)
  uint64_t pos = 0;
  uint32_t i = 0, klen0 = 0xFFFFFFFEu;
  int code = F_OK;
  uint8_t* const win = sm.win;
  while (true) {
    const uint32_t go = __shfl_sync(0xFFFFFFFFu, (uint32_t)(i < n && code == F_OK), 0);
    if (!go) break;
    // window [A0, A0 + kIdxWin) in absolute addresses, A0 16-aligned at/below
    // the entry; all of a lane's loads are issued before the first store
    const uintptr_t A0 = reinterpret_cast<uintptr_t>(body + pos) & ~uintptr_t(15);
    const uintptr_t Aend = reinterpret_cast<uintptr_t>(body + pay);
    {
      constexpr int kPer = kIdxWin / 16 / 32;
      uint4 v[kPer];
#pragma unroll
      for (int t = 0; t < kPer; ++t) {
        const uintptr_t ad = A0 + 16ull * (lane + 32u * t);
        v[t] = ad < Aend ? *reinterpret_cast<const uint4*>(ad) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int t = 0; t < kPer; ++t) reinterpret_cast<uint4*>(win)[lane + 32u * t] = v[t];
    }
    __syncwarp();
    const uint32_t i0 = i;
    uint32_t nl = 0;
    if (lane == 0) {
      const uint32_t mis = (uint32_t)(reinterpret_cast<uintptr_t>(body + pos) & 15u);
      const uint64_t wb = pos - mis;  // body offset of window byte 0 (wraps below 0 at the first entry)
      const uint64_t wlim = pos + (kIdxWin - mis);
      const bool whole = wlim >= pay;
      // fast entries end inside the window and the body (the reference bound)
      const uint64_t capb = wlim < end ? wlim : end;
      const uint32_t qcap = capb >= pos ? (uint32_t)(capb - pos) + mis : mis;
      uint32_t q = mis;
      auto at = [&](uint64_t p) -> uint32_t { return win[p - wb]; };
      while (i < n) {
        const uint32_t b = win[q];
        if (b < 0x80u && q + 9u + b <= qcap) {
          if (klen0 == 0xFFFFFFFEu) klen0 = b;
          else if (klen0 != b) klen0 = 0xFFFFFFFFu;
          sm.list[nl++] = ((i - i0) << 16) | (q + 1u + b);
          q += 9u + b;
          ++i;
          continue;
        }
        pos = wb + q;
        if (!(whole || pos + 10 <= wlim)) break;  // next window
        uint64_t kl = 0;
        int shift = 0;
        bool big = false;
        int r = -1;
        while (r < 0) {
          if (pos >= pay) { r = 1; break; }
          const uint32_t c = at(pos++);
          const uint64_t part = (uint64_t)(c & 0x7F);
          if (shift == 63 && part > 1) big = true;
          if (shift < 64) kl |= part << shift;
          if (!(c & 0x80)) { r = 0; break; }
          shift += 7;
          if (shift > 63) r = 2;
        }
        if (big) kl = ~0ull;
        if (r == 1) { code = F_IDX_VARINT_TRUNC; break; }
        if (r == 2) { code = F_IDX_VARINT_LONG; break; }
        if (kl > end || pos + kl + 8 > end) { code = F_IDX_TRUNC; break; }
        if (klen0 == 0xFFFFFFFEu) klen0 = (uint32_t)kl;
        else if (klen0 != (uint32_t)kl) klen0 = 0xFFFFFFFFu;
        pos += kl;
        uint32_t off, len;
        if (pos + 8 <= wlim) {
          off = at(pos) | (at(pos + 1) << 8) | (at(pos + 2) << 16) | (at(pos + 3) << 24);
          len = at(pos + 4) | (at(pos + 5) << 8) | (at(pos + 6) << 16) | (at(pos + 7) << 24);
        } else {
          off = ld_u32_le(body + pos);
          len = ld_u32_le(body + pos + 4);
        }
        emit(i, off, len);
        pos += 8;
        ++i;
        if (pos >= wlim) break;
        q = (uint32_t)(pos - wb);
      }
      if (code == F_OK && pos < wb + q) pos = wb + q;  // left the loop on the fast path
    }
    nl = __shfl_sync(0xFFFFFFFFu, nl, 0);
    __syncwarp();
    const uint32_t* w32 = reinterpret_cast<const uint32_t*>(win);
    for (uint32_t k = lane; k < nl; k += 32) {
      const uint32_t e = sm.list[k], o = e & 0xFFFFu, sh = (o & 3u) * 8u;
      const uint32_t x = w32[o >> 2], y = w32[(o >> 2) + 1], z = w32[(o >> 2) + 2];
      emit(i0 + (e >> 16), __funnelshift_r(x, y, sh), __funnelshift_r(y, z, sh));
    }
    __syncwarp();
    pos = __shfl_sync(0xFFFFFFFFu, pos, 0);
    i = __shfl_sync(0xFFFFFFFFu, i, 0);
    code = __shfl_sync(0xFFFFFFFFu, code, 0);
  }
  if (code == F_OK && pos != end) code = F_IDX_TRAILING;
  klen_out = __shfl_sync(0xFFFFFFFFu, klen0, 0);
  return code;
}

// Fixed-stride fast path: every entry is a 1-byte varint klen == K0.
// Returns true when the whole index verifies as such (then entries are at
// i*E with E = 1 + K0 + 8).
__device__ __forceinline__ bool index_fixed_stride(const uint8_t* body, uint64_t end, uint32_t n, uint32_t& K0) {
  if (n == 0 || end == 0) return false;
  const uint32_t k0 = body[0];
  if (k0 >= 0x80) return false;
  const uint64_t E = 1ull + k0 + 8ull;
  if ((uint64_t)n * E != end) return false;
  bool ok = true;
  for (uint32_t i = lane_id(); i < n; i += 32) ok &= (body[(uint64_t)i * E] == k0);
  ok = __all_sync(0xFFFFFFFFu, ok);
  K0 = k0;
  return ok;
}

struct ParseArgs {
  const uint8_t* arena;
  const uint64_t* file_addr;  // device: arena offset of file i
  const uint64_t* file_size;
  uint32_t nfiles;
  FileInfo* info;
  uint64_t* crc_addr;  // 2 ranges per file: filter payload, index payload
  uint32_t* crc_len;
  uint32_t* crc_stored;
};

// Stage A: warp per file.
constexpr uint32_t kParseAThreads = 128;
__global__ void __launch_bounds__(kParseAThreads) parse_files_a(ParseArgs a) {
  __shared__ __align__(16) IdxWalkSmem s_win[kParseAThreads / 32];
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = lane_id();
  if (warp >= a.nfiles) return;
  const uint8_t* f = a.arena + a.file_addr[warp];
  const uint64_t size = a.file_size[warp];
  FileInfo fi{};
  fi.klen = 0;
  uint64_t crc_fa = 0, crc_ia = 0;
  uint32_t crc_fl = 0, crc_il = 0, st_f = 0, st_i = 0;
  do {
    if (size < 24) { fi.code = F_SHORT; break; }
    const uint8_t* ft = f + size - 24;
    const uint64_t foff = ld_u32_le(ft), flen = ld_u32_le(ft + 4);
    const uint64_t ioff = ld_u32_le(ft + 8), ilen = ld_u32_le(ft + 12);
    fi.magic = ld_u64_le(ft + 16);
    if (fi.magic != kMagic) { fi.code = F_MAGIC; break; }
    const uint64_t fl = foff >= size ? 0 : (flen < size - foff ? flen : size - foff);
    const uint64_t il = ioff >= size ? 0 : (ilen < size - ioff ? ilen : size - ioff);
    fi.filter_off = foff; fi.filter_len = fl; fi.index_off = ioff; fi.index_len = il;
    if (fl < 6) { fi.code = F_FILTER_SHORT; break; }
    crc_fa = a.file_addr[warp] + foff; crc_fl = (uint32_t)(fl - 4); st_f = ld_u32_le(f + foff + fl - 4);
    fi.kbyte = f[foff + fl - 5];
    fi.kbad = (fi.kbyte < 1 || fi.kbyte > 30);
    if (il < 8) { fi.icode = F_INDEX_SHORT; break; }
    crc_ia = a.file_addr[warp] + ioff; crc_il = (uint32_t)(il - 4); st_i = ld_u32_le(f + ioff + il - 4);
    const uint8_t* body = f + ioff;
    const uint64_t end = il - 8;
    const uint32_t n = ld_u32_le(body + end);
    uint32_t K0 = 0;
    if (index_fixed_stride(body, end, n, K0)) {
      fi.nblocks = n;
      fi.klen = K0;
      fi.stride = 1;
    } else {
      uint32_t kl = 0;
      const uint32_t code = (uint32_t)index_walk_warp(body, end, n, kl, s_win[threadIdx.x >> 5],
                                                      [](uint32_t, uint32_t, uint32_t) {});
      fi.icode = code;
      fi.nblocks = code ? 0 : n;
      fi.klen = (n == 0) ? 0xFFFFFFFEu : kl;
    }
  } while (0);
  if (lane == 0) {
    a.info[warp] = fi;
    a.crc_addr[2 * warp] = crc_fa; a.crc_len[2 * warp] = crc_fl; a.crc_stored[2 * warp] = st_f;
    a.crc_addr[2 * warp + 1] = crc_ia; a.crc_len[2 * warp + 1] = crc_il; a.crc_stored[2 * warp + 1] = st_i;
  }
}

// Warp CRC contribution of pass q (segments at distances [64q, 64q+64) from
// the end) of the n-byte range at global address g, staged through the
// warp's smem buffer `stage` (>= kGroup + 160 bytes, 16-aligned). Returns
// the pass's raw register (not yet advanced over the kGroup·q bytes after
// the pass); Z_{kGroup q} of it XORed over all passes is the range's raw
// register with the ~0 preset folded in (the staged copy is prepared:
// bytes before the range are zeroed, its first 4 bytes complemented).
template <bool kCg = false>
__device__ __forceinline__ uint32_t warp_crc_pass_global_raw(const uint8_t* g, uint64_t n, uint64_t q,
                                                         uint8_t* stage, const CrcSmem& cs) {
  const uint32_t lane = lane_id();
  const int64_t hi = (int64_t)n - (int64_t)kGroup * (int64_t)q;          // pass end (data index)
  const int64_t lo0 = hi - kGroup;
  const int64_t lo = lo0 > -(int64_t)kCrcLead ? lo0 : -(int64_t)kCrcLead;  // first segment starts > -68
  // Stage data indices [lo - 8, hi + 8) into smem, keeping 16-byte phase.
  // Only 16-byte granules that hold bytes of [0, n) are loaded (always mapped).
  const uintptr_t gA = reinterpret_cast<uintptr_t>(g);
  const uintptr_t w0 = (uintptr_t)((int64_t)gA + lo - 8) & ~uintptr_t(15);
  const uintptr_t w1 = (uintptr_t)((int64_t)gA + hi + 8 + 15) & ~uintptr_t(15);
  const uintptr_t l0 = gA & ~uintptr_t(15);
  const uintptr_t l1 = (gA + n + 15) & ~uintptr_t(15);
  const uint32_t nchunks = (uint32_t)((w1 - w0) >> 4);
  for (uint32_t c = lane; c < nchunks; c += 32) {
    const uintptr_t ad = w0 + 16ull * c;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (ad >= l0 && ad < l1) v = kCg ? __ldcg(reinterpret_cast<const uint4*>(ad)) : *reinterpret_cast<const uint4*>(ad);
    reinterpret_cast<uint4*>(stage)[c] = v;
  }
  __syncwarp();
  uint8_t* base = stage + ((uintptr_t)((int64_t)gA + lo) - w0);  // smem addr of data index lo
  if (lo0 < 4) {
    // prepare: zero data indices [lo-8, 0); complement the bytes of [0, 4)
    // (the preset) that THIS pass reads, [max(0, hi - kGroup), hi) — a pass
    // boundary may fall inside the first word
    for (int64_t i = lo - 8 + lane; i < 0; i += 32) base[i - lo] = 0;
    if (lane < 4 && (uint64_t)lane < n && (int64_t)lane >= lo0 && (int64_t)lane < hi) base[lane - lo] ^= 0xFFu;
    __syncwarp();
  }
  const uint32_t v = warp_xor(pass_lane_value(base - lo, n, (uint32_t)q, cs, base));
  __syncwarp();
  return v;
}

// Pass q's contribution, already advanced over the kGroup·q bytes after it.
template <bool kCg = false>
__device__ __forceinline__ uint32_t warp_crc_pass_global(const uint8_t* g, uint64_t n, uint64_t q,
                                                         uint8_t* stage, const CrcSmem& cs) {
  return crc_shift(warp_crc_pass_global_raw<kCg>(g, n, q, stage, cs), (uint64_t)kGroup * q);
}

// CTA width of crc_big_kernel.
constexpr int kCrcWarps = 8;

// Many ranges, flattened: work item = (range, pass). pstart[r] = first item of
// range r (exclusive prefix of max(1, ceil(len/kGroup))), pstart[n] = total.
// Each warp takes a contiguous run of items (one binary search, then a forward
// walk) and XORs its pass values into out[r] (pre-set to 0xFFFFFFFF by
// crc_plan_kernel), so every pass's loads are in flight on their own warp
// instead of queueing behind the range's earlier passes.
constexpr int kCrcFlatWarps = 16;
__global__ void __launch_bounds__(1024) crc_plan_kernel(const uint32_t* len, uint32_t n, uint32_t* pstart,
                                                        uint32_t* out) {
  __shared__ uint32_t s_sum[1024];
  const uint32_t t = threadIdx.x;
  const uint32_t per = (n + 1023) / 1024;
  const uint32_t r0 = t * per, r1 = min(n, r0 + per);
  uint32_t sum = 0;
  for (uint32_t r = r0; r < r1; ++r) {
    const uint32_t L = len[r];
    sum += L < 4 ? 1u : (L + kGroup - 1) / kGroup;
    out[r] = 0xFFFFFFFFu;
  }
  s_sum[t] = sum;
  __syncthreads();
  for (uint32_t o = 1; o < 1024; o <<= 1) {
    const uint32_t v = t >= o ? s_sum[t - o] : 0u;
    __syncthreads();
    s_sum[t] += v;
    __syncthreads();
  }
  uint32_t acc = s_sum[t] - sum;
  for (uint32_t r = r0; r < r1; ++r) {
    pstart[r] = acc;
    const uint32_t L = len[r];
    acc += L < 4 ? 1u : (L + kGroup - 1) / kGroup;
  }
  if (t == 1023) pstart[n] = s_sum[1023];
}

__global__ void __launch_bounds__(kCrcFlatWarps * 32) crc_flat_kernel(const uint8_t* arena, const uint64_t* addr,
                                                                      const uint32_t* len, uint32_t nranges,
                                                                      const uint32_t* pstart, uint32_t* out) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  CrcSmem& cs = *reinterpret_cast<CrcSmem*>(smem_raw);
  uint8_t* stage = smem_raw + sizeof(CrcSmem) + (threadIdx.x >> 5) * (kGroup + 192);
  crc_smem_init(cs);
  __syncthreads();
  const uint32_t lane = lane_id();
  const uint32_t total = pstart[nranges];
  const uint32_t nw = gridDim.x * kCrcFlatWarps, gw = blockIdx.x * kCrcFlatWarps + (threadIdx.x >> 5);
  const uint32_t chunk = (total + nw - 1) / nw;
  const uint32_t i0 = gw * chunk, i1 = min(total, i0 + chunk);
  if (i0 >= i1) return;
  uint32_t l = 0, h = nranges;  // largest r with pstart[r] <= i0
  while (h - l > 1) {
    const uint32_t mid = (l + h) >> 1;
    if (pstart[mid] <= i0) l = mid;
    else h = mid;
  }
  // per range: this warp's passes q_hi..q_lo by Horner (Z_kGroup between
  // passes), one arbitrary shift by kGroup·q_lo at the end
  uint32_t r = l;
  for (uint32_t i = i0; i < i1;) {
    while (i >= pstart[r + 1]) ++r;
    const uint32_t ge = min(i1, pstart[r + 1]);
    const uint8_t* g = arena + addr[r];
    const uint32_t n = len[r];
    uint32_t v = 0;
    if (n < 4) {
      if (lane == 0) v = crc32_bytes(g, n, crc_lane(cs, 0)) ^ 0xFFFFFFFFu;
    } else {
      const uint32_t q_lo = i - pstart[r], q_hi = ge - 1 - pstart[r];
      for (int q = (int)q_hi; q >= (int)q_lo; --q) {
        const uint32_t x = warp_crc_pass_global_raw<false>(g, n, (uint64_t)q, stage, cs);
        v = (q == (int)q_hi) ? x : (gf2_apply(c_zgroup, v) ^ x);
      }
      v = crc_shift(v, (uint64_t)kGroup * q_lo);
    }
    if (lane == 0 && v) atomicXor(out + r, v);
    i = ge;
  }
}

// Single large range: passes spread over all warps, XOR-combined atomically.
// `out` must be pre-set to 0xFFFFFFFF.
__global__ void __launch_bounds__(kCrcWarps * 32) crc_big_kernel(const uint8_t* g, uint64_t n, uint32_t* out) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  CrcSmem& cs = *reinterpret_cast<CrcSmem*>(smem_raw);
  uint8_t* stage = smem_raw + sizeof(CrcSmem) + (threadIdx.x >> 5) * (kGroup + 192);
  crc_smem_init(cs);
  __syncthreads();
  const uint64_t npass = (n + kGroup - 1) / kGroup;
  const uint64_t nw = (uint64_t)gridDim.x * kCrcWarps;
  uint32_t acc = 0;
  for (uint64_t q = blockIdx.x * kCrcWarps + (threadIdx.x >> 5); q < npass; q += nw)
    acc ^= warp_crc_pass_global(g, n, q, stage, cs);
  if (lane_id() == 0 && acc) atomicXor(out, acc);
}

struct BlockTable {
  uint64_t* addr;   // arena byte offset of the (clamped) block
  uint32_t* len;    // clamped length (pread semantics)
  uint32_t* foff;   // file-relative offset (error reporting)
  uint32_t* file;   // file index
};

// Stage C: warp per (valid) file: write the data-block table.
// Stage C: block table. Grid (files, chunks): CTA (f, c) fills the entries
// [c·kParseChunk, (c+1)·kParseChunk) of file f, so a job of a few huge SSTs
// (BASELINE c4 scaled: 1.2 GB files, ~300 K blocks each) spreads over the GPU.
constexpr uint32_t kParseThreads = 256;
constexpr uint32_t kParseChunk = 16 * kParseThreads;
__global__ void __launch_bounds__(kParseThreads) parse_files_c(ParseArgs a, const uint32_t* file_blk_base,
                                                               BlockTable bt) {
  const uint32_t file = blockIdx.x;
  const FileInfo fi = a.info[file];
  const uint32_t n = fi.nblocks;
  const uint32_t i0 = blockIdx.y * kParseChunk;
  if (i0 >= n) return;
  const uint32_t i1 = min(n, i0 + kParseChunk);
  const uint64_t faddr = a.file_addr[file];
  const uint64_t size = a.file_size[file];
  const uint8_t* f = a.arena + faddr;
  const uint8_t* body = f + fi.index_off;
  const uint64_t end = fi.index_len - 8;
  const uint32_t base = file_blk_base[file];
  auto put = [&](uint32_t i, uint32_t off, uint32_t len) {
    const uint64_t o = off;
    const uint64_t l = o >= size ? 0 : ((uint64_t)len < size - o ? len : size - o);
    bt.addr[base + i] = faddr + (o >= size ? size : o);
    bt.len[base + i] = (uint32_t)l;
    bt.foff[base + i] = off;
    bt.file[base + i] = file;
  };
  // parse_files_a verified the fixed stride (fi.klen < 0x80, every entry's klen byte equal)
  const uint32_t K0 = fi.klen;
  if (fi.stride) {
    const uint64_t E = 1ull + K0 + 8ull;
    for (uint32_t i = i0 + threadIdx.x; i < i1; i += kParseThreads) {
      const uint8_t* e = body + (uint64_t)i * E + 1 + K0;
      put(i, ld_u32_le(e), ld_u32_le(e + 4));
    }
  } else if (blockIdx.y == 0 && threadIdx.x < 32) {
    __shared__ __align__(16) IdxWalkSmem s_win;
    uint32_t kl;
    index_walk_warp(body, end, n, kl, s_win, put);
  }
}

}  // namespace luda
