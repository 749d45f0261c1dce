// luda_read.cuh — batched point lookups over SSTs resident in HBM (SURVEY §8f
// row 4: the read path as a consumer of the same formats).
//
// Restates, per (key, table) probe, Table.get (sst.py:342-368):
//   may_contain (bloom.py:91-102)       h = crc32(key), k probes (h + j·δ) mod n_bits
//   index binary search (sst.py:349-355) first index key with sort_key >= seek_key(key)
//   Table._raw_block (sst.py:322-340)   short read → FormatError, CRC → CorruptionError(offset)
//   DataBlockReader.seek (blocks.py:168-218)
//                                       restart-array binary search over the restart
//                                       entries' keys, then a linear scan of one interval
//   user_key_of(found) != key → None    (sst.py:364-366)
// and the SPEC store order on top: L0 tables newest first, then each
// level ≥ 1 by binary search on the file ranges; the first table that answers wins.
//
// Layout (all device, owned by the table set):
//   per table  : file address, filter bits address / n_bits / k, first block id
//   per block  : arena address and clamped length (pread semantics), file offset,
//                verification state (every block's CRC is checked ONCE at open —
//                the reference verifies a block the first time a get reads it and
//                trusts it afterwards; the outcome is kept and raised only by a
//                lookup that touches the block), index key address / length and the
//                key's first 8 user-key bytes big-endian (binary search compares
//                these first and only falls back to the arena bytes on a tie).
// One thread per lookup: the walk is a chain of dependent loads (bloom bytes,
// ~log2(blocks) index prefixes, restart array, ≤ one restart interval), so
// throughput comes from keeping many independent lookups in flight.
#pragma once
#include "luda_parse.cuh"

namespace luda {

// seek_key(user_key) trailer: (MAX_SEQ << 8) | KIND_PUT (keys.py:17-19, 66-68)
constexpr uint64_t kSeekTrailer = ((((uint64_t)1 << 56) - 1) << 8) | 1;

enum BlockState : uint8_t {
  RB_OK = 0,
  RB_SHORT = 1,  // pread returned fewer bytes than the index length: FormatError("short block read")
  RB_TINY = 2,   // block < 4 bytes: the CRC trailer cannot be unpacked (struct.error)
  RB_CRC = 3,    // CorruptionError("data block checksum mismatch", offset)
};

enum GetStatus : uint32_t {
  G_ABSENT = 0,
  G_FOUND = 1,
  G_E_SHORT = 2,        // FormatError("short block read")
  G_E_CRC = 3,          // CorruptionError(offset)
  G_E_RESTART = 4,      // FormatError("bad restart array")
  G_E_VARINT_TRUNC = 5, // FormatError("truncated varint")
  G_E_VARINT_LONG = 6,  // FormatError("varint too long")
  G_E_STRUCT = 7,       // a fixed-width field runs off its buffer (struct.error in the reference)
  G_E_KEYCAP = 8,       // reconstructed key longer than the result slot (UnsupportedInputError)
};

struct TabView {
  const uint8_t* arena;
  const uint64_t* fbits;   // [ntab] arena address of the filter bits
  const uint64_t* fnbits;  // [ntab] n_bits = 8·len(bits)
  const uint32_t* fk;      // [ntab] probe count
  const uint32_t* bbase;   // [ntab+1] first block of each table
  const uint64_t* baddr;   // [nblk] arena address (clamped to the file)
  const uint32_t* blen;    // [nblk] clamped length
  const uint32_t* bfoff;   // [nblk] file-relative offset (error offsets)
  const uint8_t* bstate;   // [nblk] BlockState
  const uint64_t* kaddr;   // [nblk] index key (internal key) arena address
  const uint32_t* klen;    // [nblk] index key length
  const uint64_t* kpfx;    // [nblk] user-key bytes 0..7 big-endian, zero padded
  unsigned long long* n_reject;  // [ntab] Table.filter_rejects
  unsigned long long* n_reads;   // [ntab] Table.data_block_reads
};

__device__ __forceinline__ uint64_t be_prefix8(const uint8_t* p, uint32_t n) {
  uint64_t v = 0;
  const uint32_t m = n < 8 ? n : 8;
  for (uint32_t i = 0; i < m; ++i) v |= (uint64_t)p[i] << (56 - 8 * i);
  return v;
}

// Lexicographic user-key order, a shorter prefix first (bytes comparison).
// pa / pb are be_prefix8 of a / b.
__device__ __forceinline__ int cmp_user(const uint8_t* a, uint32_t la, uint64_t pa, const uint8_t* b, uint32_t lb,
                                        uint64_t pb) {
  if (pa != pb) return pa < pb ? -1 : 1;
  const uint32_t m = la < lb ? la : lb;
  for (uint32_t i = 8; i < m; ++i) {
    const uint32_t x = a[i], y = b[i];
    if (x != y) return x < y ? -1 : 1;
  }
  return (la > lb) - (la < lb);
}

__device__ __forceinline__ int cmp_user_plain(const uint8_t* a, uint32_t la, const uint8_t* b, uint32_t lb) {
  const uint32_t m = la < lb ? la : lb;
  for (uint32_t i = 0; i < m; ++i) {
    const uint32_t x = a[i], y = b[i];
    if (x != y) return x < y ? -1 : 1;
  }
  return (la > lb) - (la < lb);
}

struct Query {
  const uint8_t* key;
  uint32_t len;
  uint64_t pfx;
  uint32_t h;  // crc32(key) (bloom.py:28-29)
};

// sort_key(ikey) < sort_key(seek_key(q)) for an internal key of length L >= 8
// (keys.py:60-63: user key ascending, trailer descending).
__device__ __forceinline__ bool ikey_below_seek(int c_user, uint64_t trailer) {
  return c_user < 0 || (c_user == 0 && trailer > kSeekTrailer);
}

__device__ __forceinline__ uint64_t sat_add(uint64_t a, uint64_t b) { return a + b < a ? ~0ull : a + b; }

// crc32 of a short key, byte-wise from the global byte table (L1-resident).
__device__ __forceinline__ uint32_t key_crc(const uint8_t* p, uint32_t n) {
  uint32_t c = 0xFFFFFFFFu;
  for (uint32_t i = 0; i < n; ++i) c = g_crc_tab[(c ^ p[i]) & 0xFF] ^ (c >> 8);
  return ~c;
}

struct Found {
  uint32_t klen, vlen;
  uint64_t vaddr;  // arena address of the value bytes
  int64_t off;     // error offset (G_E_CRC)
};

// DataBlockReader(data).seek(seek_key(q)) (blocks.py:175-218) followed by the
// user-key equality test of Table.get (sst.py:364-366). The found key is
// reconstructed in `slot` (cap bytes). Returns G_ABSENT / G_FOUND / an error.
__device__ int block_seek(const uint8_t* d, uint64_t n, uint64_t base_addr, const Query& q, uint8_t* slot,
                          uint32_t cap, Found& f) {
  // n_restarts at payload_len - 4 = n - 8 (struct.unpack_from; negative offsets count from the end)
  uint32_t nr;
  if (n >= 8) {
    nr = ld_u32_le(d + n - 8);
  } else if (n == 4) {
    nr = ld_u32_le(d);
  } else {
    return G_E_STRUCT;
  }
  const int64_t entries_end = (int64_t)n - 8 - 4 * (int64_t)nr;
  if (nr < 1 || entries_end < 0) return G_E_RESTART;
  const uint8_t* rs = d + entries_end;
  // rightmost restart whose key <= target (restart keys decoded with prev = b"")
  uint32_t lo = 0, hi = nr - 1;
  while (lo < hi) {
    const uint32_t mid = (lo + hi + 1) >> 1;
    uint64_t pos = ld_u32_le(rs + 4ull * mid), sh, un, vl;
    int r = varint_read(d, n, pos, sh);
    if (!r) r = varint_read(d, n, pos, un);
    if (!r) r = varint_read(d, n, pos, vl);
    if (r) return r == 1 ? G_E_VARINT_TRUNC : G_E_VARINT_LONG;
    const uint64_t kl = pos >= n ? 0 : (un < n - pos ? un : n - pos);
    if (kl < 8) return G_E_STRUCT;
    const uint8_t* k = d + pos;
    const int c = cmp_user_plain(k, (uint32_t)(kl - 8), q.key, q.len);
    const uint64_t tr = ld_u64_le(k + kl - 8);
    if (!ikey_below_seek(c, tr) && !(c == 0 && tr == kSeekTrailer)) {
      hi = mid - 1;  // restart key > target
    } else {
      lo = mid;
    }
  }
  uint64_t pos = ld_u32_le(rs + 4ull * lo);
  uint32_t plen = 0;  // previous key length (the key itself lives in slot)
  while (pos < (uint64_t)entries_end) {
    uint64_t sh, un, vl;
    int r = varint_read(d, n, pos, sh);
    if (!r) r = varint_read(d, n, pos, un);
    if (!r) r = varint_read(d, n, pos, vl);
    if (r) return r == 1 ? G_E_VARINT_TRUNC : G_E_VARINT_LONG;
    const uint64_t keep = sh < plen ? sh : plen;
    const uint64_t avail = pos >= n ? 0 : (un < n - pos ? un : n - pos);
    if (keep + avail > cap) return G_E_KEYCAP;
    for (uint64_t i = 0; i < avail; ++i) slot[keep + i] = d[pos + i];
    const uint32_t kl = (uint32_t)(keep + avail);
    pos = sat_add(pos, un);
    const uint64_t vstart = pos;
    const uint64_t vavail = pos >= n ? 0 : (vl < n - pos ? vl : n - pos);
    pos = sat_add(pos, vl);
    if (kl < 8) return G_E_STRUCT;
    const int c = cmp_user_plain(slot, kl - 8, q.key, q.len);
    const uint64_t tr = ld_u64_le(slot + kl - 8);
    if (!ikey_below_seek(c, tr)) {
      if (c != 0) return G_ABSENT;
      f.klen = kl;
      f.vlen = (uint32_t)vavail;
      f.vaddr = base_addr + (vavail ? vstart : 0);
      return G_FOUND;
    }
    plen = kl;
  }
  return G_ABSENT;
}

// Table.get(q) on table t (sst.py:342-368).
__device__ int table_get(const TabView& tv, uint32_t t, const Query& q, uint8_t* slot, uint32_t cap, Found& f) {
  // may_contain (bloom.py:91-102)
  {
    const uint8_t* bits = tv.arena + tv.fbits[t];
    const uint64_t nb = tv.fnbits[t];
    const uint32_t k = tv.fk[t];
    uint64_t h = q.h;
    const uint64_t delta = ((q.h >> 17) | (q.h << 15)) & 0xFFFFFFFFull;
    for (uint32_t j = 0; j < k; ++j) {
      const uint64_t pos = h % nb;
      if (!((bits[pos >> 3] >> (pos & 7)) & 1)) {
        atomicAdd(tv.n_reject + t, 1ull);
        return G_ABSENT;
      }
      h += delta;
    }
  }
  // index binary search: first index key with sort_key >= target
  const uint32_t b0 = tv.bbase[t], nb = tv.bbase[t + 1] - b0;
  uint32_t lo = 0, hi = nb;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    const uint32_t b = b0 + mid;
    const uint32_t L = tv.klen[b];  // >= 8: checked at open (sort_key of every index key)
    const uint8_t* k = tv.arena + tv.kaddr[b];
    const int c = cmp_user(k, L - 8, tv.kpfx[b], q.key, q.len, q.pfx);
    if (ikey_below_seek(c, ld_u64_le(k + L - 8))) lo = mid + 1;
    else hi = mid;
  }
  if (lo == nb) return G_ABSENT;
  const uint32_t b = b0 + lo;
  const uint8_t st = tv.bstate[b];
  if (st == RB_SHORT) return G_E_SHORT;
  atomicAdd(tv.n_reads + t, 1ull);
  if (st == RB_TINY) return G_E_STRUCT;
  if (st == RB_CRC) {
    f.off = tv.bfoff[b];
    return G_E_CRC;
  }
  return block_seek(tv.arena + tv.baddr[b], tv.blen[b], tv.baddr[b], q, slot, cap, f);
}

// Per-lookup results, structure of arrays (each array D2H'd as is).
struct GetOut {
  uint32_t* status;  // GetStatus
  uint32_t* table;   // table that answered (found) or failed
  uint32_t* klen;    // found key length (0 otherwise)
  uint32_t* vlen;    // found value length
  uint64_t* vaddr;   // arena address of the value
  int64_t* err_off;  // CorruptionError offset (G_E_CRC) or -1
  unsigned int* first_fail;  // min index of a failing lookup (0xFFFFFFFF: none)
};

struct GetArgs {
  TabView tv;
  const uint8_t* keys;
  const uint64_t* koff;  // nullptr: fixed-length keys, key i at keys + i * klen[0]
  const uint32_t* klen;
  uint32_t n;
  const uint32_t* qtable;  // per-query table (Table.get mode) or nullptr (store order)
  // store order: L0 newest first, then levels ≥ 1 by file range
  uint32_t n_l0;
  const uint32_t* l0;
  uint32_t n_levels;
  const uint32_t* lvl_first;  // [n_levels+1] into lvl_tab
  const uint32_t* lvl_tab;    // table ids, ascending ranges per level
  const uint8_t* rk;          // range keys: entry 2i = smallest, 2i+1 = largest user key of lvl_tab[i]
  const uint64_t* rk_off;
  const uint32_t* rk_len;
  const uint64_t* rk_pfx;
  GetOut out;
  uint8_t* slots;  // n × cap bytes: found keys
  uint32_t cap;
  uint32_t* sizes;  // [n] klen + vlen of found entries (packing), else 0
};

#ifndef LUDA_GET_MINB
#define LUDA_GET_MINB 1
#endif
__global__ void __launch_bounds__(256, LUDA_GET_MINB) get_kernel(GetArgs a) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  Query q;
  if (a.koff) {
    q.key = a.keys + a.koff[i];
    q.len = a.klen[i];
  } else {
    q.len = a.klen[0];
    q.key = a.keys + (uint64_t)i * q.len;
  }
  q.pfx = be_prefix8(q.key, q.len);
  q.h = key_crc(q.key, q.len);
  uint8_t* slot = a.slots + (uint64_t)i * a.cap;
  Found f{0, 0, 0, -1};
  int r = G_ABSENT;
  uint32_t t = 0;
  if (a.qtable) {
    t = a.qtable[i];
    r = table_get(a.tv, t, q, slot, a.cap, f);
  } else {
    for (uint32_t j = 0; j < a.n_l0 && r == G_ABSENT; ++j) {
      t = a.l0[j];
      r = table_get(a.tv, t, q, slot, a.cap, f);
    }
    for (uint32_t L = 0; L < a.n_levels && r == G_ABSENT; ++L) {
      // first file whose largest user key >= key; probe it if its smallest <= key
      uint32_t lo = a.lvl_first[L], hi = a.lvl_first[L + 1];
      const uint32_t end = hi;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        const uint32_t e = 2 * mid + 1;
        if (cmp_user(a.rk + a.rk_off[e], a.rk_len[e], a.rk_pfx[e], q.key, q.len, q.pfx) < 0) lo = mid + 1;
        else hi = mid;
      }
      if (lo == end) continue;
      const uint32_t e = 2 * lo;
      if (cmp_user(a.rk + a.rk_off[e], a.rk_len[e], a.rk_pfx[e], q.key, q.len, q.pfx) > 0) continue;
      t = a.lvl_tab[lo];
      r = table_get(a.tv, t, q, slot, a.cap, f);
    }
  }
  const uint32_t kl = r == G_FOUND ? f.klen : 0, vl = r == G_FOUND ? f.vlen : 0;
  a.out.status[i] = (uint32_t)r;
  a.out.table[i] = t;
  a.out.klen[i] = kl;
  a.out.vlen[i] = vl;
  a.out.vaddr[i] = f.vaddr;
  a.out.err_off[i] = r == G_E_CRC ? f.off : -1;
  if (r > G_FOUND) atomicMin(a.out.first_fail, i);
  a.sizes[i] = kl + vl;
}

// Found key ∥ value of query i at packed + pos[i] (pos: exclusive scan of sizes).
__global__ void __launch_bounds__(256) get_pack_kernel(GetOut out, const uint8_t* slots, uint32_t cap,
                                                       const uint8_t* arena, const uint64_t* pos, uint32_t n,
                                                       uint8_t* packed) {
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = lane_id();
  if (warp >= n) return;
  if (out.status[warp] != G_FOUND) return;
  const uint32_t kl = out.klen[warp], vl = out.vlen[warp];
  uint8_t* dst = packed + pos[warp];
  const uint8_t* ks = slots + (uint64_t)warp * cap;
  for (uint32_t j = lane; j < kl; j += 32) dst[j] = ks[j];
  const uint8_t* v = arena + out.vaddr[warp];
  for (uint32_t j = lane; j < vl; j += 32) dst[kl + j] = v[j];
}

// ---- table-set open ----------------------------------------------------------------
// Per block: index key address/length/prefix (thread per index entry on
// fixed-stride indexes, the sequential decode_index_block walk otherwise).
struct IndexKeyArgs {
  const uint8_t* arena;
  const uint64_t* faddr;
  const FileInfo* info;
  const uint32_t* bbase;
  uint64_t* kaddr;
  uint32_t* klen;
  uint64_t* kpfx;
  uint32_t* ilen;       // the index entry's block length (before the pread clamp)
  uint32_t* short_key;  // min(1 + block id) over index keys shorter than a trailer
};

__device__ __forceinline__ void put_ikey(const IndexKeyArgs& a, uint32_t b, uint64_t addr, uint32_t L) {
  a.ilen[b] = ld_u32_le(a.arena + addr + L + 4);
  a.kaddr[b] = addr;
  a.klen[b] = L;
  a.kpfx[b] = be_prefix8(a.arena + addr, L >= 8 ? L - 8 : 0);
  if (L < 8) atomicMin(a.short_key, b + 1);
}

__global__ void __launch_bounds__(kParseThreads) index_keys_kernel(IndexKeyArgs a) {
  const uint32_t file = blockIdx.x;
  const FileInfo fi = a.info[file];
  const uint32_t n = fi.nblocks;
  const uint32_t i0 = blockIdx.y * kParseChunk;
  if (i0 >= n) return;
  const uint32_t i1 = min(n, i0 + kParseChunk);
  const uint64_t body = a.faddr[file] + fi.index_off;
  const uint32_t base = a.bbase[file];
  if (fi.stride) {
    const uint32_t K0 = fi.klen;
    const uint64_t E = 1ull + K0 + 8ull;
    for (uint32_t i = i0 + threadIdx.x; i < i1; i += kParseThreads) put_ikey(a, base + i, body + i * E + 1, K0);
  } else if (blockIdx.y == 0 && threadIdx.x == 0) {
    // parse_files_a validated the walk (no errors on this path)
    const uint8_t* p = a.arena + body;
    const uint64_t end = fi.index_len - 8;
    uint64_t pos = 0;
    for (uint32_t i = 0; i < n; ++i) {
      uint64_t kl;
      varint_read(p, end + 4, pos, kl);
      put_ikey(a, base + i, body + pos, (uint32_t)kl);
      pos += kl + 8;
    }
  }
}

// CRC ranges of every data block: (addr, len - 4) for blocks of >= 4 bytes.
__global__ void block_crc_ranges_kernel(const uint64_t* baddr, const uint32_t* blen, uint32_t n, uint64_t* caddr,
                                        uint32_t* clen) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  caddr[i] = baddr[i];
  clen[i] = blen[i] >= 4 ? blen[i] - 4 : 0;
}

// Block verification state (Table._raw_block, sst.py:322-340), and the filter
// description of every table.
__global__ void block_state_kernel(const uint8_t* arena, const uint64_t* baddr, const uint32_t* blen,
                                   const uint32_t* ilen, const uint32_t* crc, uint32_t n, uint8_t* state) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t L = blen[i];
  uint8_t s = RB_OK;
  if (L != ilen[i]) s = RB_SHORT;
  else if (L < 4) s = RB_TINY;
  else if (ld_u32_le(arena + baddr[i] + L - 4) != crc[i]) s = RB_CRC;
  state[i] = s;
}

}  // namespace luda
