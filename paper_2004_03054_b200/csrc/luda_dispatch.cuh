// luda_dispatch.cuh — the reference's per-kind kernel work items on the GPU.
//
// Restates kernels.py:72-168 (`unpack`, `shared_key`, `encode`, `filter`) for
// the offload-device dispatch protocol (device.py:435-456, 566-607): every
// item is self-contained (region ids + region-relative offsets), items are
// independent, and the first failing item in dispatch order decides the
// error. One warp per item; lane 0 walks the variable-length records
// (entries, tuples) and the warp copies bytes, verifies CRCs (staged warp
// passes, luda_parse.cuh) and hashes keys (lane per key).
//
// Region access mirrors the reference's memoryview slicing: reads past a
// region's capacity are truncated (bytes(src[a:b])), writes that do not fit
// the region are item errors (memoryview slice assignment raises).
#pragma once
#include "luda_encode.cuh"
#include "luda_parse.cuh"

namespace luda {

enum DispatchStatus : uint32_t { D_OK = 0, D_CORRUPT = 1, D_ERR = 2 };
enum DispatchMsg : uint32_t {
  M_NONE = 0,
  M_SHORT,          // block too short
  M_CRC,            // data block checksum mismatch
  M_RESTART,        // bad restart array
  M_VARINT_TRUNC,   // truncated varint
  M_VARINT_LONG,    // varint too long
  M_TRUNC_ENTRY,    // truncated block entry
  M_TRAILING,       // trailing garbage in block entries
  M_PAIR_OVF,       // pair slot overflow
  M_TUP_OVF,        // tuple slot overflow
  M_KEY_U16,        // key longer than 65535 (struct.error packing u16)
  M_REGION,         // region id / range outside the dispatch's regions
  M_RI,             // restart_interval must be >= 1
  M_ENC_OVF,        // encode slot overflow
  M_FILT_OVF,       // filter slot overflow
  M_BPK,            // bits_per_key must be >= 1
  M_TUPLE,          // tuple runs past its region
};

struct DispatchArgs {
  int kind;
  const int64_t* items;   // [n][cols]
  uint32_t n, cols;
  uint8_t* const* rptr;   // region id -> device pointer (nullptr: not a region)
  const uint64_t* rcap;   // region id -> capacity
  uint32_t nreg;
  int64_t* results;       // [n][rcols]
  uint32_t rcols;
  uint32_t* status;       // [n] DispatchStatus
  uint32_t* msg;          // [n] DispatchMsg
  int64_t* err_off;       // [n] corruption offset
};

constexpr int kDispWarps = 8;
constexpr int kDispStage = kGroup + 192;

struct DispRegion {
  uint8_t* p;
  uint64_t cap;
  bool ok;
};
__device__ __forceinline__ DispRegion disp_region(const DispatchArgs& a, int64_t rid) {
  if (rid < 0 || (uint64_t)rid >= a.nreg || a.rptr[rid] == nullptr) return DispRegion{nullptr, 0, false};
  return DispRegion{a.rptr[rid], a.rcap[rid], true};
}

// Warp byte copy (any alignment; global memory).
__device__ __forceinline__ void warp_copy_bytes(uint8_t* dst, const uint8_t* src, uint64_t n) {
  for (uint64_t i = lane_id(); i < n; i += 32) dst[i] = src[i];
}

// Warp CRC-32 of a global range (staged passes through `stage`; kCg: loads
// bypass L1).
template <bool kCg = false>
__device__ __forceinline__ uint32_t warp_crc_global(const uint8_t* g, uint64_t n, uint8_t* stage, const CrcSmem& cs) {
  if (n < 4) {
    uint32_t c = 0;
    if (lane_id() == 0) {
      c = 0xFFFFFFFFu;
      for (uint64_t i = 0; i < n; ++i) c = crc_byte(c, kCg ? (uint32_t)__ldcg(g + i) : (uint32_t)g[i], crc_lane(cs, 0));
      c = ~c;
    }
    return __shfl_sync(0xFFFFFFFFu, c, 0);
  }
  const uint64_t npass = (n + kGroup - 1) / kGroup;
  uint32_t raw = 0;
  for (uint64_t q = 0; q < npass; ++q) raw ^= warp_crc_pass_global<kCg>(g, n, q, stage, cs);
  return ~raw;
}

// Tuple wire (kernels.py:25-51): u16le klen ∥ key ∥ u64le v_off ∥ u32le v_len.
struct Tup {
  uint64_t key;   // region offset of the key
  uint32_t klen;
  uint64_t voff;
  uint32_t vlen;
  uint64_t next;
};
__device__ __forceinline__ bool tup_read(const DispRegion& r, uint64_t pos, Tup& t) {
  if (pos + 2 > r.cap) return false;
  t.klen = (uint32_t)r.p[pos] | ((uint32_t)r.p[pos + 1] << 8);
  t.key = pos + 2;
  if (t.key + t.klen + 12 > r.cap) return false;
  t.voff = ld_u64_le(r.p + t.key + t.klen);
  t.vlen = ld_u32_le(r.p + t.key + t.klen + 8);
  t.next = t.key + t.klen + 12;
  return true;
}

// ---- unpack (kernels.py:72-104 + decode_data_block blocks.py:130-165) --------------
__device__ void disp_unpack(const DispatchArgs& a, uint32_t it, uint8_t* stage, const CrcSmem& cs) {
  const int64_t* x = a.items + (uint64_t)it * a.cols;
  const uint32_t lane = lane_id();
  auto fail = [&](uint32_t st, uint32_t m, int64_t off) {
    if (lane == 0) { a.status[it] = st; a.msg[it] = m; a.err_off[it] = off; }
  };
  const DispRegion src = disp_region(a, x[0]), pr = disp_region(a, x[3]), tr = disp_region(a, x[6]);
  if (!src.ok || !pr.ok || !tr.ok) return fail(D_ERR, M_REGION, -1);
  const uint64_t boff = (uint64_t)x[1];
  uint64_t blen = (uint64_t)x[2];
  blen = boff >= src.cap ? 0 : (blen < src.cap - boff ? blen : src.cap - boff);  // bytes(src[a:b])
  const uint8_t* blk = src.p + boff;
  if (blen < 12) return fail(D_ERR, M_SHORT, -1);
  const uint64_t n = blen - 4;
  const uint32_t crc = warp_crc_global(blk, n, stage, cs);
  if (crc != ld_u32_le(blk + n)) return fail(D_CORRUPT, M_CRC, x[1]);
  const uint32_t nres = ld_u32_le(blk + n - 4);
  const int64_t ee = (int64_t)n - 4 - 4 * (int64_t)nres;
  if (nres < 1 || ee < 0) return fail(D_ERR, M_RESTART, -1);
  const uint64_t entries_end = (uint64_t)ee;
  const uint64_t pair_off = (uint64_t)x[4], pair_cap = (uint64_t)x[5];
  const uint64_t tup_off = (uint64_t)x[7], tup_cap = (uint64_t)x[8];
  // pass 1 (lane 0): parse entries exactly like the reference, record nothing
  uint32_t code = 0;
  uint64_t npairs = 0;
  if (lane == 0) {
    uint64_t pos = 0, prev_len = 0;
    while (pos < entries_end) {
      uint64_t s, u, vl;
      int r;
      if ((r = varint_read(blk, n, pos, s)) || (r = varint_read(blk, n, pos, u)) || (r = varint_read(blk, n, pos, vl))) {
        code = r == 1 ? M_VARINT_TRUNC : M_VARINT_LONG;
        break;
      }
      if (s > prev_len || u > entries_end || vl > entries_end || pos + u + vl > entries_end) {
        code = M_TRUNC_ENTRY;
        break;
      }
      prev_len = s + u;
      pos += u + vl;
      ++npairs;
    }
    if (!code && pos != entries_end) code = M_TRAILING;
  }
  code = __shfl_sync(0xFFFFFFFFu, code, 0);
  if (code) return fail(D_ERR, code, -1);
  npairs = __shfl_sync(0xFFFFFFFFu, npairs, 0);
  // pass 2: write pair records (varint klen ∥ key ∥ value) and tuples
  uint64_t pos = 0, ppos = pair_off, tpos = tup_off, vbytes = 0;
  uint64_t prev_key = 0;  // pair-region offset of the previous key
  for (uint64_t e = 0; e < npairs; ++e) {
    uint64_t s = 0, u = 0, vl = 0, p2 = 0;
    if (lane == 0) {
      p2 = pos;
      varint_read(blk, n, p2, s);
      varint_read(blk, n, p2, u);
      varint_read(blk, n, p2, vl);
    }
    s = __shfl_sync(0xFFFFFFFFu, s, 0);
    u = __shfl_sync(0xFFFFFFFFu, u, 0);
    vl = __shfl_sync(0xFFFFFFFFu, vl, 0);
    p2 = __shfl_sync(0xFFFFFFFFu, p2, 0);
    const uint64_t klen = s + u;
    uint32_t vk = 1;
    for (uint64_t t = klen; t >= 0x80; t >>= 7) ++vk;
    const uint64_t rec = vk + klen + vl;
    if (ppos + rec > pair_off + pair_cap) return fail(D_ERR, M_PAIR_OVF, -1);
    if (klen > 0xFFFF) return fail(D_ERR, M_KEY_U16, -1);
    const uint64_t tl = 2 + klen + 12;
    if (tpos + tl > tup_off + tup_cap) return fail(D_ERR, M_TUP_OVF, -1);
    if (ppos + rec > pr.cap || tpos + tl > tr.cap) return fail(D_ERR, M_REGION, -1);
    uint8_t* pd = pr.p + ppos;
    if (lane == 0) put_varint(pd, klen);
    const uint64_t kpos = ppos + vk;
    // key = prev_key[:s] ∥ payload[p2 : p2+u]; the shared part is copied first
    // (sequentially ordered: source and destination never overlap — the new
    // key is written after the previous pair record)
    warp_copy_bytes(pr.p + kpos, pr.p + prev_key, s);
    warp_copy_bytes(pr.p + kpos + s, blk + p2, u);
    warp_copy_bytes(pr.p + kpos + klen, blk + p2 + u, vl);
    __syncwarp();
    uint8_t* td = tr.p + tpos;
    if (lane == 0) {
      td[0] = (uint8_t)klen;
      td[1] = (uint8_t)(klen >> 8);
      const uint64_t vo = ppos;  // v_offset = offset of the pair record (read_pair_value)
      for (int b = 0; b < 8; ++b) td[2 + klen + b] = (uint8_t)(vo >> (8 * b));
      put_u32(td + 2 + klen + 8, (uint32_t)vl);
    }
    warp_copy_bytes(td + 2, pr.p + kpos, klen);
    __syncwarp();
    prev_key = kpos;
    pos = p2 + u + vl;
    ppos += rec;
    tpos += tl;
    vbytes += vl;
  }
  if (lane == 0) {
    int64_t* r = a.results + (uint64_t)it * a.rcols;
    r[0] = (int64_t)(ppos - pair_off);
    r[1] = (int64_t)(tpos - tup_off);
    r[2] = (int64_t)npairs;
    r[3] = (int64_t)vbytes;
  }
}

// ---- shared_key (kernels.py:107-117 + compute_layouts blocks.py:41-58) -------------
__device__ void disp_shared_key(const DispatchArgs& a, uint32_t it) {
  const int64_t* x = a.items + (uint64_t)it * a.cols;
  const uint32_t lane = lane_id();
  if (lane != 0) return;
  const DispRegion tr = disp_region(a, x[0]), lr = disp_region(a, x[4]);
  auto fail = [&](uint32_t m) { a.status[it] = D_ERR; a.msg[it] = m; a.err_off[it] = -1; };
  if (!tr.ok || !lr.ok) return fail(M_REGION);
  const int64_t ri = x[3];
  const uint64_t end = (uint64_t)x[2];
  uint64_t pos = (uint64_t)x[1], lo = (uint64_t)x[5];
  // parse first (a malformed tuple list fails before compute_layouts)
  uint64_t cnt = 0;
  for (uint64_t p = pos; p < end;) {
    Tup t;
    if (!tup_read(tr, p, t)) return fail(M_TUPLE);
    p = t.next;
    ++cnt;
  }
  if (cnt && ri < 1) return fail(M_RI);
  if (lo + 8 * cnt > lr.cap) return fail(M_REGION);
  uint64_t prev = 0;
  uint32_t prev_len = 0;
  for (uint64_t i = 0; i < cnt; ++i) {
    Tup t;
    tup_read(tr, pos, t);
    uint32_t sh = 0;
    if (i % (uint64_t)ri != 0) {
      const uint32_t m = t.klen < prev_len ? t.klen : prev_len;
      while (sh < m && tr.p[prev + sh] == tr.p[t.key + sh]) ++sh;
    }
    put_u32(lr.p + lo + 8 * i, sh);
    put_u32(lr.p + lo + 8 * i + 4, t.klen - sh);
    prev = t.key;
    prev_len = t.klen;
    pos = t.next;
  }
  a.results[(uint64_t)it * a.rcols] = (int64_t)cnt;
}

// ---- encode (kernels.py:120-155 + assemble_block blocks.py:77-103) -----------------
__device__ void disp_encode(const DispatchArgs& a, uint32_t it, uint8_t* stage, const CrcSmem& cs) {
  const int64_t* x = a.items + (uint64_t)it * a.cols;
  const uint32_t lane = lane_id();
  auto fail = [&](uint32_t m) {
    if (lane == 0) { a.status[it] = D_ERR; a.msg[it] = m; a.err_off[it] = -1; }
  };
  const DispRegion tr = disp_region(a, x[0]), lr = disp_region(a, x[3]), pr = disp_region(a, x[5]),
                   orr = disp_region(a, x[6]);
  if (!tr.ok || !lr.ok || !pr.ok || !orr.ok) return fail(M_REGION);
  const uint64_t end = (uint64_t)x[2], lpos0 = (uint64_t)x[4], out_off = (uint64_t)x[7], out_cap = (uint64_t)x[8];
  const int64_t ri = x[9];
  // pass 1 (lane 0): tuples, layouts and values → block size
  uint32_t code = 0;
  uint64_t cnt = 0, size = 0, vbytes = 0;
  if (lane == 0) {
    uint64_t lp = lpos0;
    for (uint64_t p = (uint64_t)x[1]; p < end; ++cnt) {
      Tup t;
      if (!tup_read(tr, p, t)) { code = M_TUPLE; break; }
      if (lp + 8 > lr.cap) { code = M_REGION; break; }
      const uint32_t sh = ld_u32_le(lr.p + lp), un = ld_u32_le(lr.p + lp + 4);
      lp += 8;
      // read_pair_value: varint klen at v_offset, the value after the key
      uint64_t vp = t.voff, kl;
      if (varint_read(pr.p, pr.cap, vp, kl)) { code = M_REGION; break; }
      const uint64_t vs = vp + kl;  // bytes(buf[vs : vs + v_len]) may be short at the region end
      const uint64_t veff = vs >= pr.cap ? 0 : (t.vlen < pr.cap - vs ? t.vlen : pr.cap - vs);
      const uint64_t keyrest = sh < t.klen ? t.klen - sh : 0;  // key[shared:]
      size += varint_size(sh) + varint_size(un) + varint_size(veff) + keyrest + veff;
      vbytes += t.vlen;
      p = t.next;
    }
    if (!code && cnt && ri < 1) code = M_RI;
    if (!code) {
      const uint64_t nr = cnt ? (cnt + (uint64_t)ri - 1) / (uint64_t)ri : 0;
      size += 4 * nr + 4 + 4;
      if (size > out_cap) code = M_ENC_OVF;
      else if (out_off + size > orr.cap) code = M_REGION;
    }
  }
  code = __shfl_sync(0xFFFFFFFFu, code, 0);
  if (code) return fail(code);
  cnt = __shfl_sync(0xFFFFFFFFu, cnt, 0);
  size = __shfl_sync(0xFFFFFFFFu, size, 0);
  vbytes = __shfl_sync(0xFFFFFFFFu, vbytes, 0);
  // pass 2: entries (lane 0 headers, warp copies), restart array, count, crc
  uint8_t* ob = orr.p + out_off;
  uint64_t p = (uint64_t)x[1], lp = lpos0, o = 0;
  for (uint64_t i = 0; i < cnt; ++i) {
    Tup t;
    tup_read(tr, p, t);
    const uint32_t sh = ld_u32_le(lr.p + lp), un = ld_u32_le(lr.p + lp + 4);
    lp += 8;
    uint64_t vp = t.voff, kl;
    varint_read(pr.p, pr.cap, vp, kl);
    const uint64_t vstart = vp + kl;
    const uint64_t veff = vstart >= pr.cap ? 0 : (t.vlen < pr.cap - vstart ? t.vlen : pr.cap - vstart);
    uint32_t hl = 0;
    if (lane == 0) {
      hl = put_varint(ob + o, sh);
      hl += put_varint(ob + o + hl, un);
      hl += put_varint(ob + o + hl, veff);
      if (i % (uint64_t)ri == 0) put_u32(ob + size - 8 - 4 * ((cnt + ri - 1) / ri) + 4 * (i / ri), (uint32_t)o);
    }
    hl = __shfl_sync(0xFFFFFFFFu, hl, 0);
    const uint64_t keyrest = sh < t.klen ? t.klen - sh : 0;
    warp_copy_bytes(ob + o + hl, tr.p + t.key + (sh < t.klen ? sh : t.klen), keyrest);
    warp_copy_bytes(ob + o + hl + keyrest, pr.p + vstart, veff);
    o += hl + keyrest + veff;
    p = t.next;
  }
  const uint64_t nr = cnt ? (cnt + (uint64_t)ri - 1) / (uint64_t)ri : 0;
  if (lane == 0) put_u32(ob + size - 8, (uint32_t)nr);
  __syncwarp();
  __threadfence_block();
  const uint32_t crc = warp_crc_global(ob, size - 4, stage, cs);
  if (lane == 0) {
    put_u32(ob + size - 4, crc);
    int64_t* r = a.results + (uint64_t)it * a.rcols;
    r[0] = (int64_t)size;
    r[1] = (int64_t)vbytes;
  }
}

// ---- filter (kernels.py:158-168 + build_filter bloom.py:71-88) ---------------------
__device__ void disp_filter(const DispatchArgs& a, uint32_t it, uint8_t* stage, const CrcSmem& cs,
                            uint64_t* keypos) {
  const int64_t* x = a.items + (uint64_t)it * a.cols;
  const uint32_t lane = lane_id();
  auto fail = [&](uint32_t m) {
    if (lane == 0) { a.status[it] = D_ERR; a.msg[it] = m; a.err_off[it] = -1; }
  };
  const DispRegion tr = disp_region(a, x[0]), orr = disp_region(a, x[4]);
  if (!tr.ok || !orr.ok) return fail(M_REGION);
  const uint64_t end = (uint64_t)x[2], out_off = (uint64_t)x[5], out_cap = (uint64_t)x[6];
  const int64_t bpk = x[3];
  uint32_t code = 0;
  uint64_t cnt = 0;
  if (lane == 0) {
    for (uint64_t p = (uint64_t)x[1]; p < end; ++cnt) {
      Tup t;
      if (!tup_read(tr, p, t)) { code = M_TUPLE; break; }
      p = t.next;
    }
    if (!code && bpk < 1) code = M_BPK;
  }
  code = __shfl_sync(0xFFFFFFFFu, code, 0);
  if (code) return fail(code);
  cnt = __shfl_sync(0xFFFFFFFFu, cnt, 0);
  uint64_t nbits = 8, k = 1;
  if (cnt) {
    k = (uint64_t)llround((double)bpk * 0.69314718055994530942);
    k = k < 1 ? 1 : (k > 30 ? 30 : k);
    nbits = cnt * (uint64_t)bpk;
    if (nbits < 64) nbits = 64;
    nbits = (nbits + 7) & ~7ull;
  }
  const uint64_t nbytes = nbits / 8, enc = nbytes + 5;
  if (enc > out_cap) return fail(M_FILT_OVF);
  if (out_off + enc > orr.cap) return fail(M_REGION);
  uint8_t* ob = orr.p + out_off;
  for (uint64_t i = lane; i < nbytes; i += 32) ob[i] = 0;
  __syncwarp();
  __threadfence_block();
  if (cnt) {
    const CrcLane tl = crc_lane(cs, lane);
    uint64_t p = (uint64_t)x[1];
    for (uint64_t c0 = 0; c0 < cnt; c0 += 32) {
      if (lane == 0)
        for (uint32_t j = 0; j < 32 && c0 + j < cnt; ++j) {
          Tup t;
          tup_read(tr, p, t);
          keypos[j] = (t.key << 16) | (t.klen > 8 ? t.klen - 8 : 0);  // user key = key[:-8]
          p = t.next;
        }
      __syncwarp();
      if (c0 + lane < cnt) {
        const uint64_t kp = keypos[lane];
        const uint32_t h = crc32_bytes(tr.p + (kp >> 16), (uint32_t)(kp & 0xFFFF), tl);
        const uint64_t delta = ((h >> 17) | (h << 15)) & 0xFFFFFFFFu;
        for (uint64_t j = 0; j < k; ++j) {
          const uint64_t pos = ((uint64_t)h + j * delta) % nbits;
          const uintptr_t ad = reinterpret_cast<uintptr_t>(ob + (pos >> 3));
          atomicOr(reinterpret_cast<unsigned int*>(ad & ~uintptr_t(3)), 1u << (8 * (ad & 3) + (pos & 7)));
        }
      }
      __syncwarp();
    }
  }
  __threadfence();
  __syncwarp();
  if (lane == 0) ob[nbytes] = (uint8_t)k;
  __syncwarp();
  __threadfence_block();
  const uint32_t crc = warp_crc_global<true>(ob, nbytes + 1, stage, cs);  // L2 reads: bits were set by atomics
  if (lane == 0) {
    put_u32(ob + nbytes + 1, crc);
    a.results[(uint64_t)it * a.rcols] = (int64_t)enc;
  }
}

__global__ void __launch_bounds__(kDispWarps * 32) dispatch_kernel(DispatchArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  CrcSmem& cs = *reinterpret_cast<CrcSmem*>(smem_raw);
  const uint32_t w = threadIdx.x >> 5;
  uint8_t* stage = smem_raw + sizeof(CrcSmem) + w * (kDispStage + 256);
  uint64_t* keypos = reinterpret_cast<uint64_t*>(stage + kDispStage);
  crc_smem_init(cs);
  __syncthreads();
  for (uint32_t it = blockIdx.x * kDispWarps + w; it < a.n; it += gridDim.x * kDispWarps) {
    if (lane_id() == 0) { a.status[it] = D_OK; a.msg[it] = M_NONE; a.err_off[it] = -1; }
    switch (a.kind) {
      case 0: disp_unpack(a, it, stage, cs); break;
      case 1: disp_shared_key(a, it); break;
      case 2: disp_encode(a, it, stage, cs); break;
      default: disp_filter(a, it, stage, cs, keypos); break;
    }
    __syncwarp();
  }
}

}  // namespace luda
