// luda_rec.cuh — fixed-width sort records and key-byte helpers.
//
// An internal key (keys.py:25-34) is user_key ∥ u64le((seq<<8)|kind). Its
// order (keys.py:60-63) is user key bytes ascending (a prefix sorts first),
// then trailer DEScending. For a job whose user keys all have length L
// (8(W-1) < L <= 8W) a record stores
//     k[0..W)  user key as big-endian u64 words, zero padded   (ascending)
//     t        ~trailer                                          (ascending)
//     h        value handle: arena byte offset << 24 | value length
// so the internal-key order is plain lexicographic u64 order over (k, t).
#pragma once
#include <stdint.h>

#include "luda_common.cuh"

namespace luda {

// 16-byte aligned when the record size allows (W = 2, 4: 32 / 48 bytes), so
// record copies are LDG/STG.128.
template <int W>
struct alignas((8 * (W + 2)) % 16 == 0 ? 16 : 8) Rec {
  uint64_t k[W];
  uint64_t t;
  uint64_t h;
};

constexpr int kHandleLenBits = 24;
constexpr uint64_t kMaxValueLen = (1ull << kHandleLenBits) - 1;
constexpr uint64_t kMaxValueOff = (1ull << 40) - 1;

__host__ __device__ __forceinline__ uint64_t handle_pack(uint64_t off, uint64_t len) {
  return (off << kHandleLenBits) | len;
}
__host__ __device__ __forceinline__ uint64_t handle_off(uint64_t h) { return h >> kHandleLenBits; }
__host__ __device__ __forceinline__ uint32_t handle_len(uint64_t h) {
  return (uint32_t)(h & kMaxValueLen);
}

// -1 / 0 / +1 comparison in internal-key order.
template <int W>
__device__ __forceinline__ int rec_cmp(const Rec<W>& a, const Rec<W>& b) {
#pragma unroll
  for (int i = 0; i < W; ++i)
    if (a.k[i] != b.k[i]) return a.k[i] < b.k[i] ? -1 : 1;
  if (a.t != b.t) return a.t < b.t ? -1 : 1;
  return 0;
}

template <int W>
__device__ __forceinline__ bool rec_le(const Rec<W>& a, const Rec<W>& b) { return rec_cmp(a, b) <= 0; }

template <int W>
__device__ __forceinline__ bool same_user(const Rec<W>& a, const Rec<W>& b) {
  bool eq = true;
#pragma unroll
  for (int i = 0; i < W; ++i) eq &= (a.k[i] == b.k[i]);
  return eq;
}

template <int W>
__device__ __forceinline__ bool is_tombstone(const Rec<W>& r) { return ((~r.t) & 0xFFu) == 0; }

// Longest common prefix (bytes) of two DISTINCT user keys of equal length.
template <int W>
__device__ __forceinline__ uint32_t user_lcp(const Rec<W>& a, const Rec<W>& b) {
#pragma unroll
  for (int i = 0; i < W; ++i) {
    uint64_t x = a.k[i] ^ b.k[i];
    if (x) return 8u * i + (uint32_t)(__clzll((long long)x) >> 3);
  }
  return 8u * W;  // identical user keys (callers never pass these)
}

// Longest common prefix (bytes) of the two INTERNAL keys (user key of length
// L ∥ little-endian trailer). Equal user keys continue into the trailer.
template <int W>
__device__ __forceinline__ uint32_t ikey_lcp(const Rec<W>& a, const Rec<W>& b, uint32_t L) {
#pragma unroll
  for (int i = 0; i < W; ++i) {
    uint64_t x = a.k[i] ^ b.k[i];
    if (x) return 8u * i + (uint32_t)(__clzll((long long)x) >> 3);
  }
  const uint64_t x = a.t ^ b.t;  // = trailer_a ^ trailer_b
  if (!x) return L + 8;
  return L + (uint32_t)(__ffsll((long long)x) - 1) / 8;
}

// ---- generic-length keys ("var" jobs) ---------------------------------------
// A job whose user keys differ in length, or are longer than 32 bytes, uses
// W = kVarW records: the key area holds the user key zero-padded to 71 bytes
// and its LENGTH in the last byte (byte 71 = low byte of k[8]). For keys of
// length <= 71, padded bytes then length is exactly Python's bytes order
// (keys.py:60-63): when the padded bytes agree, the shorter key is a prefix of
// the longer one and sorts first. A var job with a user key of 72..255 bytes
// runs again with W = kVarWLong records (255 key bytes + the length byte).
constexpr int kVarW = 9;
constexpr int kVarWLong = 32;
constexpr uint32_t kVarMaxLen = 8 * kVarW - 1;          // 71
constexpr uint32_t kVarMaxLenLong = 8 * kVarWLong - 1;  // 255

// Var records are exactly the W = kVarW / kVarWLong instantiations (fixed-length
// jobs use W <= 4), so the var paths compile out of the fixed kernels.
template <int W>
__host__ __device__ constexpr bool is_var() { return W == kVarW || W == kVarWLong; }
template <int W>
__host__ __device__ constexpr uint32_t var_maxlen() { return 8 * W - 1; }

template <int W>
__device__ __forceinline__ uint32_t rec_ulen(const Rec<W>& r, bool var, uint32_t L) {
  return var ? (uint32_t)(r.k[W - 1] & 0xFFu) : L;
}

// Byte j (0-based) of the internal key encoded by `r` (user key length L).
template <int W>
__device__ __forceinline__ uint32_t ikey_byte(const Rec<W>& r, uint32_t L, uint32_t j) {
  if (j < L) return (uint32_t)(r.k[j >> 3] >> (56 - 8 * (j & 7))) & 0xFFu;
  uint64_t tr = ~r.t;
  return (uint32_t)(tr >> (8 * (j - L))) & 0xFFu;
}

// Internal key → little-endian u32 words (byte b at word b>>2), NW words.
template <int W, int NW>
__device__ __forceinline__ void rec_to_words(const Rec<W>& r, uint32_t L, uint32_t (&kw)[NW]) {
  // user part: big-endian u64 word j covers bytes 8j..8j+7
#pragma unroll
  for (int j = 0; j < W; ++j) {
    kw[2 * j] = bswap32((uint32_t)(r.k[j] >> 32));
    kw[2 * j + 1] = bswap32((uint32_t)r.k[j]);
  }
#pragma unroll
  for (int i = 2 * W; i < NW; ++i) kw[i] = 0;
  // trailer at bytes [L, L+8): zero the padding then OR in shifted trailer
  const uint64_t tr = ~r.t;
  const uint32_t q = L >> 2, sh = (L & 3u) * 8u;
  const uint32_t t0 = (uint32_t)tr, t1 = (uint32_t)(tr >> 32);
  const uint32_t w0 = t0 << sh;
  const uint32_t w1 = sh ? ((t1 << sh) | (t0 >> (32 - sh))) : t1;
  const uint32_t w2 = sh ? (t1 >> (32 - sh)) : 0u;
#pragma unroll
  for (int i = 0; i < NW; ++i) {
    uint32_t keep = 0xFFFFFFFFu;  // bytes < L inside word i
    if ((uint32_t)(4 * i) >= L) keep = 0;
    else if ((uint32_t)(4 * i + 4) > L) keep = 0xFFFFFFFFu >> (8 * (4 * i + 4 - L));
    uint32_t v = kw[i] & keep;
    if ((uint32_t)i == q) v |= w0;
    if ((uint32_t)i == q + 1) v |= w1;
    if ((uint32_t)i == q + 2) v |= w2;
    kw[i] = v;
  }
}

// LE u32 key words (internal key of length K = L + 8) → record key fields.
template <int W, int NW>
__device__ __forceinline__ void words_to_rec(const uint32_t (&kw)[NW], uint32_t L, Rec<W>& r) {
  if (L == 8 * W) {  // user key fills the words exactly (warp-uniform)
#pragma unroll
    for (int j = 0; j < W; ++j) r.k[j] = ((uint64_t)bswap32(kw[2 * j]) << 32) | bswap32(kw[2 * j + 1]);
    r.t = ~(((uint64_t)kw[2 * W + 1] << 32) | kw[2 * W]);
    return;
  }
#pragma unroll
  for (int j = 0; j < W; ++j) {
    uint64_t v = ((uint64_t)bswap32(kw[2 * j]) << 32) | bswap32(kw[2 * j + 1]);
    const int64_t valid = (int64_t)L - 8 * j;  // bytes of this word inside the user key
    if (valid <= 0) v = 0;
    else if (valid < 8) v &= ~0ull << (8 * (8 - valid));
    r.k[j] = v;
  }
  const uint32_t q = L >> 2, sh = (L & 3u) * 8u;
  uint32_t a = 0, b = 0, c = 0;
#pragma unroll
  for (int i = 0; i < NW; ++i) {
    if ((uint32_t)i == q) a = kw[i];
    if ((uint32_t)i == q + 1) b = kw[i];
    if ((uint32_t)i == q + 2) c = kw[i];
  }
  const uint32_t lo = __funnelshift_r(a, b, sh);
  const uint32_t hi = __funnelshift_r(b, c, sh);
  r.t = ~(((uint64_t)hi << 32) | lo);
}

// Longest common prefix (bytes) of two internal keys of a var job (user keys
// of any lengths <= 71, blocks.py:33-38 over user_key ∥ trailer): when one user
// key is a proper prefix of the other, the shorter key's trailer is compared
// with the longer key's next user bytes (the prefix may run into the trailer).
template <int W>
__device__ __forceinline__ uint32_t ikey_lcp_var(const Rec<W>& a, const Rec<W>& b) {
  const uint32_t la = rec_ulen(a, true, 0), lb = rec_ulen(b, true, 0);
  uint32_t p = 8u * W - 1;
#pragma unroll
  for (int i = 0; i < W; ++i) {
    uint64_t x = a.k[i] ^ b.k[i];
    if (i == W - 1) x &= ~0xFFull;  // length byte
    if (x) {
      p = 8u * i + (uint32_t)(__clzll((long long)x) >> 3);
      break;
    }
  }
  const uint32_t m = la < lb ? la : lb;
  if (p < m) return p;
  if (la == lb) {
    const uint64_t x = a.t ^ b.t;
    if (!x) return la + 8;
    return la + (uint32_t)(__ffsll((long long)x) - 1) / 8;
  }
  const Rec<W>& sh = la < lb ? a : b;
  const Rec<W>& lg = la < lb ? b : a;
  const uint32_t ll = la < lb ? lb : la;
  uint32_t n = m;
  for (uint32_t j = 0; j < 8; ++j) {
    if (ikey_byte(sh, m, m + j) != ikey_byte(lg, ll, m + j)) break;
    ++n;
  }
  return n;
}

template <int W>
__device__ __forceinline__ uint32_t ikey_lcp_any(const Rec<W>& a, const Rec<W>& b, bool var, uint32_t L) {
  return var ? ikey_lcp_var(a, b) : ikey_lcp(a, b, L);
}

}  // namespace luda
