// luda_plan.cuh — exact parallel block and SST planning.
//
// SstBuilder (sst.py:138-177) cuts blocks greedily: before adding entry e to a
// non-empty block it flushes if
//     cur_entry_bytes + size(e) + 4*ceil((n+1)/ri) + 4 > block_size
// where size(e) uses shared = 0 when e is at a restart position
// (i % ri == 0 counted from the block start) and the LCP with the previous
// key otherwise (blocks.py:41-74). Then, after a flush, it closes the SST as
// soon as data_bytes >= sst_size_target (sst.py:161-162).
//
// Both are "greedy chains": from a start s the next start is nxt(s), and the
// cut set is the chain 0 → nxt(0) → ... . Here:
//   * block_jump_kernel computes nxt for every survivor (jmp = nxt - s) and
//     the size of the block that would start there; SST jumps come from a
//     binary search over block-size prefix sums.
//   * chain_map_kernel splits the sequence into tiles of T >= D items
//     (D = max jump) and, for every possible entry offset o < D into the
//     tile, follows the chain through the tile → exit offset into the next
//     tile and node count. The maps compose associatively.
//   * chain_group_kernel composes G consecutive tile maps; chain_top_kernel
//     walks the groups from offset 0 (the true chain); chain_emit_kernel
//     re-walks each tile from its true entry and writes the chain nodes.
// The result is exactly the builder's greedy cut, computed in O(n) work.
#pragma once
#include "luda_rec.cuh"

namespace luda {

constexpr uint32_t kChainEnd = 0xFFFFFFFFu;

// ---- block jumps ----------------------------------------------------------------
#ifndef LUDA_JUMP_THREADS
#define LUDA_JUMP_THREADS 512
#endif
#ifndef LUDA_JUMP_TILE
#define LUDA_JUMP_TILE 4096
#endif
constexpr int kJumpThreads = LUDA_JUMP_THREADS;
constexpr int kJumpTile = LUDA_JUMP_TILE;

template <int W>
struct BlockJumpArgs {
  const Rec<W>* rec;
  uint64_t n;
  uint32_t K;
  uint32_t block_size;
  uint32_t ri;
  uint32_t halo;      // >= max entries per block
  uint32_t* jmp;      // out [n]
  uint32_t* bsz;      // out [n]: block size incl. crc if a block starts here
  unsigned int* jmax;
  unsigned int* overflow;
  uint64_t file_entries;  // > 0: a block never crosses a multiple of this (file-cut builds)
  bool var;               // generic-length keys: K per record (luda_rec.cuh)
  uint32_t tile;          // survivors per CTA (<= kJumpTile; smaller for small jobs)
};

// Block size if a block started at local index i held n entries:
//   PB[i+n] - PB[i]                    compressed entry sizes (shared vs prev)
// + sum_{k < m} D[i + k ri]            restart entries use the full size
// + 4 m + 4                            restart array + count (pre-crc)
// with m = ceil(n / ri). Within restart group k (n in (k ri, (k+1) ri]) m is
// fixed, so the greedy cut is found group by group, then by binary search
// inside the group that overflows.
template <int W>
__global__ void __launch_bounds__(kJumpThreads) block_jump_kernel(BlockJumpArgs<W> a) {
  extern __shared__ __align__(16) uint32_t sz[];  // PB[span+1], D[span]
  const uint32_t tile = a.tile;
  const uint32_t span = tile + a.halo;
  uint32_t* PB = sz;
  uint32_t* D = sz + span + 1;
  __shared__ uint32_t s_warp[kJumpThreads / 32];
  const uint64_t t0 = (uint64_t)blockIdx.x * tile;
  const uint32_t K = a.K, L = K - 8, vK = varint_size(K);
  const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
  // sizes → D (full - compressed) and a CTA-wide exclusive scan PB of compressed sizes
  __shared__ uint32_t s_total;
  uint32_t carry = 0;
  for (uint32_t base = 0; base < span; base += kJumpThreads) {
    const uint32_t i = base + threadIdx.x;
    const uint64_t j = t0 + i;
    uint32_t sbv = 0;
    if (i < span && j < a.n) {
      const Rec<W> cur = a.rec[j];
      const uint32_t vl = handle_len(cur.h);
      const uint32_t vv = varint_size(vl);
      const uint32_t Kc = is_var<W>() ? rec_ulen(cur, true, 0) + 8 : K;
      uint32_t sh = 0;
      if (j > 0) sh = ikey_lcp_any(a.rec[j - 1], cur, is_var<W>(), L);
      sbv = varint_size(sh) + varint_size(Kc - sh) + vv + (Kc - sh) + vl;
      D[i] = (1 + (is_var<W>() ? varint_size(Kc) : vK) + vv + Kc + vl) - sbv;
    } else if (i < span) {
      D[i] = 0;
    }
    const uint32_t incl = warp_incl_scan<uint32_t>(sbv);
    if (lane == 31) s_warp[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      const uint32_t v = lane < kJumpThreads / 32 ? s_warp[lane] : 0u;
      const uint32_t vi = warp_incl_scan<uint32_t>(v);
      if (lane < kJumpThreads / 32) s_warp[lane] = vi - v;
      if (lane == 31) s_total = vi;
    }
    __syncthreads();
    if (i < span) PB[i] = carry + s_warp[wid] + incl - sbv;
    carry += s_total;
    __syncthreads();
  }
  if (threadIdx.x == 0) PB[span] = carry;
  __syncthreads();
  const uint32_t ri = a.ri, bs = a.block_size;
  uint32_t mymax = 0;
  for (uint32_t i = threadIdx.x; i < tile; i += kJumpThreads) {
    const uint64_t j = t0 + i;
    if (j >= a.n) break;
    uint64_t rem64 = a.n - j;
    if (a.file_entries) {
      const uint64_t to_file_end = a.file_entries - j % a.file_entries;
      rem64 = rem64 < to_file_end ? rem64 : to_file_end;
    }
    const uint32_t lim = (uint32_t)(rem64 < (uint64_t)(span - i) ? rem64 : (uint64_t)(span - i));  // entries available
    uint32_t fixed = 0;  // sum of D over restart entries of groups < k, plus group k's once added
    uint32_t best = 1, m = 0;
    for (uint32_t k = 0;; ++k) {
      const uint32_t gs = k * ri;                 // group k covers n in (gs, gs + ri]
      if (gs >= lim) break;
      fixed += D[i + gs];
      m = k + 1;
      const uint32_t ge = gs + ri < lim ? gs + ri : lim;
      const uint32_t full = PB[i + ge] - PB[i] + fixed + 4 * m + 4;
      if (full <= bs) {
        best = ge;
        continue;
      }
      // largest n in (gs, ge) with size <= bs; n = 1 always fits (first entry)
      uint32_t lo = gs, hi = ge - 1;  // invariant: n = lo fits (or lo == gs meaning none in group yet)
      while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) >> 1;
        if (PB[i + mid] - PB[i] + fixed + 4 * m + 4 <= bs) lo = mid;
        else hi = mid - 1;
      }
      if (lo > gs) best = lo;
      else if (gs == 0) best = 1;
      break;
    }
    if (best == lim && lim == span - i && rem64 > lim) atomicExch(a.overflow, 1u);
    const uint32_t mb = (best + ri - 1) / ri;
    uint32_t fx = 0;
    for (uint32_t k = 0; k < mb; ++k) fx += D[i + k * ri];
    a.jmp[j] = best;
    a.bsz[j] = PB[i + best] - PB[i] + fx + 4 * mb + 8;
    mymax = best > mymax ? best : mymax;
  }
  mymax = warp_max(mymax);
  if (lane == 0) atomicMax(a.jmax, mymax);
}

// ---- SST jumps -------------------------------------------------------------------
// pos[b] = data bytes before block b (exclusive prefix, pos[nb] = total).
__global__ void sst_jump_kernel(const uint64_t* pos, uint32_t nb, uint64_t target, uint32_t* jmp,
                                unsigned int* jmax) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t j = 0;
  if (b < nb) {
    const uint64_t want = pos[b] + target;
    // first e in (b, nb] with pos[e] >= want, else nb
    uint32_t lo = b + 1, hi = nb;
    while (lo < hi) {
      const uint32_t mid = lo + ((hi - lo) >> 1);
      if (pos[mid] >= want) hi = mid;
      else lo = mid + 1;
    }
    j = lo - b;
    jmp[b] = j;
  }
  j = warp_max(j);
  if (lane_id() == 0) atomicMax(jmax, j);
}

// File-cut builds: every output SST holds exactly `fe` entries (the last
// fewer); its blocks end at the file boundary (block_jump clamps), so the SST
// jump from block b is to the first block starting at the next multiple of fe.
__global__ void sst_jump_files_kernel(const uint32_t* blk_first, uint32_t nb, uint64_t fe, uint32_t* jmp,
                                      unsigned int* jmax) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t j = 0;
  if (b < nb) {
    const uint64_t want = ((uint64_t)blk_first[b] / fe + 1) * fe;
    uint32_t lo = b + 1, hi = nb;  // first e in (b, nb] with blk_first[e] >= want (e = nb: end)
    while (lo < hi) {
      const uint32_t mid = lo + ((hi - lo) >> 1);
      if ((uint64_t)blk_first[mid] >= want) hi = mid;
      else lo = mid + 1;
    }
    j = lo - b;
    jmp[b] = j;
  }
  j = warp_max(j);
  if (lane_id() == 0) atomicMax(jmax, j);
}

// ---- generic chain over jmp[0..n) -------------------------------------------------
struct ChainArgs {
  const uint32_t* jmp;
  uint32_t n;
  uint32_t T;       // tile size (>= D)
  uint32_t D;       // domain: max jump
  uint32_t ntiles;
  uint32_t G;       // tiles per group
  uint32_t ngroups;
  uint32_t* exit_;  // [ntiles*D]
  uint32_t* cnt;    // [ntiles*D]
  uint32_t* gexit;  // [ngroups*D]
  uint32_t* gcnt;   // [ngroups*D]
  uint32_t* gentry; // [ngroups]
  uint32_t* gbase;  // [ngroups]
  uint32_t* nodes;  // out: chain nodes
  uint32_t* nnodes; // out: count
};

constexpr int kChainThreads = 256;

__global__ void __launch_bounds__(kChainThreads) chain_map_kernel(ChainArgs c) {
  extern __shared__ __align__(16) uint32_t sj[];  // tile jumps (when T small enough)
  const uint32_t t = blockIdx.x;
  const uint64_t t0 = (uint64_t)t * c.T;
  const uint64_t tend = t0 + c.T < c.n ? t0 + c.T : c.n;
  const bool use_smem = c.T <= 12288;
  if (use_smem) {
    for (uint64_t x = t0 + threadIdx.x; x < tend; x += kChainThreads) sj[x - t0] = c.jmp[x];
    __syncthreads();
  }
  for (uint32_t o = threadIdx.x; o < c.D; o += kChainThreads) {
    uint64_t x = t0 + o;
    uint32_t k = 0;
    while (x < tend) {
      x += use_smem ? sj[x - t0] : c.jmp[x];
      ++k;
    }
    const uint64_t idx = (uint64_t)t * c.D + o;
    c.exit_[idx] = (x >= c.n) ? kChainEnd : (uint32_t)(x - (t0 + c.T));
    c.cnt[idx] = k;
  }
}

// The composition walks below follow dependent (tile, offset) lookups; each
// CTA first stages the rows it walks into shared memory (kChainStage bytes
// max) so a step is one LDS instead of an L2 round trip.
constexpr uint32_t kChainStage = 40 * 1024;

__global__ void __launch_bounds__(kChainThreads) chain_group_kernel(ChainArgs c) {
  extern __shared__ __align__(16) uint32_t sg[];
  const uint32_t g = blockIdx.x;
  const uint32_t tf = g * c.G;
  const uint32_t tl = (tf + c.G < c.ntiles) ? tf + c.G : c.ntiles;
  const uint64_t rows = (uint64_t)(tl - tf) * c.D;
  const bool staged = rows * 8 <= kChainStage;
  const uint32_t* cnt = c.cnt + (uint64_t)tf * c.D;
  const uint32_t* ex = c.exit_ + (uint64_t)tf * c.D;
  if (staged) {
    for (uint32_t i = threadIdx.x; i < rows; i += kChainThreads) {
      sg[i] = cnt[i];
      sg[rows + i] = ex[i];
    }
    __syncthreads();
    cnt = sg;
    ex = sg + rows;
  }
  for (uint32_t o = threadIdx.x; o < c.D; o += kChainThreads) {
    uint32_t off = o, total = 0;
    for (uint32_t t = 0; t < tl - tf && off != kChainEnd; ++t) {
      const uint64_t idx = (uint64_t)t * c.D + off;
      total += cnt[idx];
      off = ex[idx];
    }
    c.gexit[(uint64_t)g * c.D + o] = off;
    c.gcnt[(uint64_t)g * c.D + o] = total;
  }
}

__global__ void __launch_bounds__(1024) chain_top_kernel(ChainArgs c) {
  extern __shared__ __align__(16) uint32_t sg[];
  const uint64_t rows = (uint64_t)c.ngroups * c.D;
  const bool staged = rows * 8 <= kChainStage;
  const uint32_t* gcnt = c.gcnt;
  const uint32_t* gex = c.gexit;
  if (staged) {
    for (uint32_t i = threadIdx.x; i < rows; i += blockDim.x) {
      sg[i] = c.gcnt[i];
      sg[rows + i] = c.gexit[i];
    }
    __syncthreads();
    gcnt = sg;
    gex = sg + rows;
  }
  if (threadIdx.x != 0) return;
  uint32_t off = 0, total = 0;
  for (uint32_t g = 0; g < c.ngroups; ++g) {
    c.gentry[g] = off;
    c.gbase[g] = total;
    if (off == kChainEnd) continue;
    const uint64_t idx = (uint64_t)g * c.D + off;
    total += gcnt[idx];
    off = gex[idx];
  }
  *c.nnodes = total;
}

// Entry offset and first node index of every tile: CTA per group, its G
// tile rows staged in shared memory, one thread walks them (the tile maps
// compose along the true chain).
__global__ void __launch_bounds__(kChainThreads) chain_tile_entry_kernel(ChainArgs c, uint32_t* tentry,
                                                                          uint32_t* tbase) {
  extern __shared__ __align__(16) uint32_t sg[];
  const uint32_t g = blockIdx.x;
  const uint32_t tf = g * c.G;
  const uint32_t tl = (tf + c.G < c.ntiles) ? tf + c.G : c.ntiles;
  const uint64_t rows = (uint64_t)(tl - tf) * c.D;
  const bool staged = rows * 8 <= kChainStage;
  const uint32_t* cnt = c.cnt + (uint64_t)tf * c.D;
  const uint32_t* ex = c.exit_ + (uint64_t)tf * c.D;
  if (staged) {
    for (uint32_t i = threadIdx.x; i < rows; i += kChainThreads) {
      sg[i] = cnt[i];
      sg[rows + i] = ex[i];
    }
    __syncthreads();
    cnt = sg;
    ex = sg + rows;
  }
  if (threadIdx.x != 0) return;
  uint32_t off = c.gentry[g], base = c.gbase[g];
  for (uint32_t u = 0; u < tl - tf; ++u) {
    tentry[tf + u] = off;
    tbase[tf + u] = base;
    if (off == kChainEnd) continue;
    const uint64_t idx = (uint64_t)u * c.D + off;
    base += cnt[idx];
    off = ex[idx];
  }
}

// Walk each tile's true chain from its entry over the tile's jumps staged in
// shared memory (one dependent LDS per node instead of a global load).
__global__ void __launch_bounds__(kChainThreads) chain_emit_kernel(ChainArgs c, const uint32_t* tentry,
                                                                   const uint32_t* tbase) {
  extern __shared__ __align__(16) uint32_t sj[];
  const uint32_t t = blockIdx.x;
  const uint32_t off = tentry[t];
  if (off == kChainEnd) return;
  const uint64_t t0 = (uint64_t)t * c.T;
  const uint64_t tend = t0 + c.T < c.n ? t0 + c.T : c.n;
  const bool use_smem = c.T <= 12288;
  if (use_smem) {
    for (uint64_t x = t0 + threadIdx.x; x < tend; x += kChainThreads) sj[x - t0] = c.jmp[x];
    __syncthreads();
  }
  if (threadIdx.x != 0) return;
  uint64_t x = t0 + off;
  uint32_t k = tbase[t];
  while (x < tend) {
    c.nodes[k++] = (uint32_t)x;
    x += use_smem ? sj[x - t0] : c.jmp[x];
  }
}

// ---- block descriptors + exclusive prefix of sizes ----------------------------------
// Var jobs: index entry size of every block (varint(K) ∥ last key ∥ u32 ∥ u32,
// sst.py:67-76) with K the block's last internal key length.
template <int W>
__global__ void index_entry_size_kernel(const Rec<W>* rec, const uint32_t* blk_first, const uint32_t* blk_n,
                                        uint32_t nb, uint32_t* isz) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nb) return;
  const uint32_t K = rec_ulen(rec[(uint64_t)blk_first[k] + blk_n[k] - 1], true, 0) + 8;
  isz[k] = varint_size(K) + K + 8;
}

__global__ void block_desc_kernel(const uint32_t* nodes, uint32_t nb, const uint32_t* jmp, const uint32_t* bsz,
                                  uint32_t* blk_first, uint32_t* blk_n, uint32_t* blk_size) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nb) return;
  const uint32_t s = nodes[k];
  blk_first[k] = s;
  blk_n[k] = jmp[s];
  blk_size[k] = bsz[s];
}

// Single-pass exclusive scan (u64 out) of a u32 or u64 array with decoupled
// look-back; out[n] = total.
constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
template <typename T>
__global__ void __launch_bounds__(kScanThreads) scan_excl_kernel(const T* in, uint64_t n, uint64_t* out,
                                                                 uint64_t* lb, unsigned int* tile_ctr) {
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_warp[kScanThreads / 32];
  __shared__ uint64_t s_base;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t i0 = tile * (kScanThreads * kScanItems) + threadIdx.x * kScanItems;
  uint64_t v[kScanItems];
  uint64_t sum = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = (i0 + k < n) ? (uint64_t)in[i0 + k] : 0;
    sum += v[k];
  }
  const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
  const uint64_t incl = warp_incl_scan<uint64_t>(sum);
  if (lane == 31) s_warp[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    const uint64_t w = lane < kScanThreads / 32 ? s_warp[lane] : 0;
    const uint64_t wi = warp_incl_scan<uint64_t>(w);
    if (lane < kScanThreads / 32) s_warp[lane] = wi - w;
    const uint64_t total = __shfl_sync(0xFFFFFFFFu, wi, 31);
    if (lane == 0) lb_publish(lb, tile, kLbAgg, total);
    const uint64_t ex = lb_exclusive(lb, tile);
    if (lane == 0) {
      lb_publish(lb, tile, kLbInc, ex + total);
      s_base = ex;
      const uint64_t ntile = (n + kScanThreads * kScanItems - 1) / (kScanThreads * kScanItems);
      if (tile + 1 == ntile || n == 0) out[n] = ex + total;
    }
  }
  __syncthreads();
  uint64_t run = s_base + s_warp[wid] + incl - sum;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (i0 + k < n) out[i0 + k] = run;
    run += v[k];
  }
}

// ---- SST layout ----------------------------------------------------------------------
struct SstLayoutArgs {
  const uint32_t* sst_first_blk;  // chain nodes [nsst]
  uint32_t nsst;
  uint32_t nblk;
  const uint32_t* blk_first;
  const uint64_t* blk_pos;        // [nblk+1]
  uint64_t n_entries;
  uint32_t K;
  uint32_t bits_per_key;
  uint64_t* sst_size;             // out [nsst]
  uint64_t* sst_data;             // out: data bytes
  uint64_t* sst_nent;             // out: entries
  uint32_t* sst_last_blk;         // out: one past last block
  const uint64_t* blk_ipos;       // var jobs: exclusive prefix of index-entry sizes [nblk+1], else nullptr
};

__global__ void sst_layout_kernel(SstLayoutArgs a) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= a.nsst) return;
  const uint32_t fb = a.sst_first_blk[s];
  const uint32_t eb = (s + 1 < a.nsst) ? a.sst_first_blk[s + 1] : a.nblk;
  const uint64_t fe = a.blk_first[fb];
  const uint64_t ee = (eb < a.nblk) ? a.blk_first[eb] : a.n_entries;
  const uint64_t ne = ee - fe;
  const uint64_t data = a.blk_pos[eb] - a.blk_pos[fb];
  uint64_t nbits = ne * a.bits_per_key;
  if (nbits < 64) nbits = 64;
  nbits = (nbits + 7) & ~7ull;
  const uint64_t flen = nbits / 8 + 1 + 4;
  const uint64_t ilen = (a.blk_ipos ? a.blk_ipos[eb] - a.blk_ipos[fb] : (uint64_t)(eb - fb) * (varint_size(a.K) + a.K + 8)) + 8;
  a.sst_size[s] = data + flen + ilen + 24;
  a.sst_data[s] = data;
  a.sst_nent[s] = ne;
  a.sst_last_blk[s] = eb;
}

}  // namespace luda
