// luda_merge.cuh — k-way merge of sorted runs + version resolution.
//
// Replaces the reference's host-side cooperative sort (the
// composition is heapq.merge on keys.sort_key over per-file runs, keep the
// first (= newest) entry of every user key, drop it if it is a Delete and
// Version.covers_below is false — SPEC D12, version.py:122-128).
//
// Runs are merged pairwise by MERGE PATH: a partition kernel places every
// merge_tile_n<W>()-output tile boundary on the merge diagonal by binary search (ties
// go to the earlier run, so the merge is stable like heapq.merge over runs in
// priority order); each CTA loads its A and B slices into shared memory,
// every thread merges merge_items<W>() outputs after a local diagonal search, and
// the merged permutation is written back coalesced. The last pass fuses
// version resolution: keep flags (new user key, tombstone rule, optional key
// range) are scanned across the CTA and the tile's survivors are written
// compacted into the tile's own segment; a scan of the tile counts and
// merge_densify_kernel then pack the segments (no dependency between tiles).
// Every loaded slice is also checked for strict ascending order (keys.py
// order); violations are reported as the run position so the host can raise
// OrderingError.
#pragma once
#include "luda_rec.cuh"

namespace luda {

#ifndef LUDA_MERGE_THREADS
#define LUDA_MERGE_THREADS 256
#endif
#ifndef LUDA_MERGE_ITEMS
#define LUDA_MERGE_ITEMS 6
#endif
constexpr int kMergeThreads = LUDA_MERGE_THREADS;
// Outputs per thread: fewer for the long var records so a tile still fits
// shared memory (272-byte records).
template <int W>
__host__ __device__ constexpr int merge_items() {
  return W > kVarW ? 2 : LUDA_MERGE_ITEMS;
}
template <int W>
__host__ __device__ constexpr int merge_tile_n() {
  return kMergeThreads * merge_items<W>();
}

struct KeyBound {
  uint64_t k[kVarWLong];
  uint32_t incl;
  uint32_t present;
};

template <int W>
__device__ __forceinline__ int cmp_user(const Rec<W>& r, const KeyBound& b) {
#pragma unroll
  for (int i = 0; i < W; ++i)
    if (r.k[i] != b.k[i]) return r.k[i] < b.k[i] ? -1 : 1;
  return 0;
}

template <int W>
__device__ __forceinline__ bool above_lo(const Rec<W>& r, const KeyBound& lo) {
  if (!lo.present) return true;
  const int c = cmp_user(r, lo);
  return lo.incl ? c >= 0 : c > 0;
}

template <int W>
__device__ __forceinline__ bool below_hi(const Rec<W>& r, const KeyBound& hi) {
  if (!hi.present) return true;
  const int c = cmp_user(r, hi);
  return hi.incl ? c <= 0 : c < 0;
}

struct ResolveArgs {
  const KeyBound* deeper;  // pairs (lo, hi) of closed user-key intervals below the target
  uint32_t n_deeper;
  KeyBound range_lo, range_hi;  // subcompaction range [lo, hi)
  bool resolve;                 // final pass
};

template <int W>
__device__ __forceinline__ bool covered_below(const Rec<W>& r, const ResolveArgs& ra) {
  for (uint32_t i = 0; i < ra.n_deeper; ++i)
    if (above_lo(r, ra.deeper[2 * i]) && below_hi(r, ra.deeper[2 * i + 1])) return true;
  return false;
}

// A sorted run as seen by the merge: dense (`lo` == nullptr: element i at
// base[off + i]) or SEGMENTED — the decoder's layout (luda_decode.cuh), where
// logical record g lives in the segment s with lo[s] <= g < lo[s+1], at
// physical index s * cap + (g - lo[s]).
template <int W>
struct RunView {
  const Rec<W>* base;
  const uint64_t* lo;  // [nseg+1] logical segment starts, or nullptr (dense)
  uint64_t cap;
  uint32_t nseg;
  uint64_t off;        // logical index of the run's element 0
  __device__ __forceinline__ uint32_t seg(uint64_t g) const {
    uint32_t l = 0, h = nseg;
    while (h - l > 1) {
      const uint32_t mid = (l + h) >> 1;
      if (lo[mid] <= g) l = mid;
      else h = mid;
    }
    return l;
  }
  // segment of logical g starting from a nearby segment (the merge partition
  // stores each tile's starting segments, so CTAs never binary-search)
  __device__ __forceinline__ uint32_t seg_near(uint64_t g, uint32_t s) const {
    if (s >= nseg) s = nseg - 1;
    while (s > 0 && lo[s] > g) --s;
    while (s + 1 < nseg && lo[s + 1] <= g) ++s;
    return s;
  }
  __device__ __forceinline__ const Rec<W>& at_near(uint64_t i, uint32_t s) const {
    if (!lo) return base[off + i];
    const uint64_t g = off + i;
    s = seg_near(g, s);
    return base[(uint64_t)s * cap + (g - lo[s])];
  }
  __device__ __forceinline__ uint64_t phys(uint64_t i) const {
    if (!lo) return off + i;
    const uint64_t g = off + i;
    const uint32_t s = seg(g);
    return (uint64_t)s * cap + (g - lo[s]);
  }
  __device__ __forceinline__ const Rec<W>& operator[](uint64_t i) const { return base[phys(i)]; }
  // f(physical pointer, count, destination offset) over the contiguous pieces of [i0, i1)
  template <typename F>
  __device__ __forceinline__ void pieces(uint64_t i0, uint64_t i1, F f, uint32_t hint = ~0u) const {
    if (i0 >= i1) return;
    if (!lo) {
      f(base + off + i0, i1 - i0, 0ull);
      return;
    }
    uint64_t g = off + i0;
    const uint64_t g1 = off + i1;
    uint32_t s = hint == ~0u ? seg(g) : seg_near(g, hint);
    uint64_t done = 0;
    while (g < g1) {
      const uint64_t e = lo[s + 1] < g1 ? lo[s + 1] : g1;
      if (e > g) {
        f(base + (uint64_t)s * cap + (g - lo[s]), e - g, done);
        done += e - g;
        g = e;
      }
      ++s;
    }
  }
};

// Merge-path split: number of A elements among the first `diag` outputs.
template <int W>
__device__ __forceinline__ uint64_t merge_split(const RunView<W>& A, uint64_t na, const RunView<W>& B, uint64_t nb,
                                                uint64_t diag) {
  uint64_t lo = diag > nb ? diag - nb : 0;
  uint64_t hi = diag < na ? diag : na;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (rec_le(A[mid], B[diag - 1 - mid])) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Merge-path split by one WARP per diagonal: 32-ary search rounds (each lane
// tests one candidate; the predicate is monotone, so the ballot's popcount
// brackets the split), ~log32 instead of log2 dependent steps — every step
// resolves two segmented-view records (a segment binary search each).
template <int W>
__device__ __forceinline__ uint64_t merge_split_warp(const RunView<W>& A, uint64_t na, const RunView<W>& B, uint64_t nb,
                                                     uint64_t diag) {
  const uint32_t lane = threadIdx.x & 31u;
  uint64_t lo = diag > nb ? diag - nb : 0;
  uint64_t hi = diag < na ? diag : na;
  while (hi > lo) {
    const uint64_t span = hi - lo;
    const bool last = span <= 32;
    const uint64_t m = last ? lo + lane : lo + ((uint64_t)(lane + 1) * span) / 33;
    const bool p = (!last || lane < span) && rec_le(A[m], B[diag - 1 - m]);
    const uint32_t c = __popc(__ballot_sync(0xFFFFFFFFu, p));  // P holds on a prefix of the candidates
    if (last) return lo + c;
    const uint64_t lo0 = lo;
    if (c > 0) lo = lo0 + ((uint64_t)c * span) / 33 + 1;
    if (c < 32) hi = lo0 + ((uint64_t)(c + 1) * span) / 33;
  }
  return lo;
}

// warp_mode: a warp per diagonal (few tiles: latency-bound small jobs), else
// a thread per diagonal (many tiles: the 32-ary rounds would cost more loads).
template <int W>
__global__ void merge_partition_kernel(RunView<W> A, uint64_t na, RunView<W> B, uint64_t nb, uint64_t ntiles,
                                       uint64_t* split, bool warp_mode) {
  const uint64_t gt = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t t = warp_mode ? gt >> 5 : gt;
  if (t > ntiles) return;  // warp-uniform in warp mode
  uint64_t diag = t * (uint64_t)merge_tile_n<W>();
  if (diag > na + nb) diag = na + nb;
  const uint64_t a = warp_mode ? merge_split_warp(A, na, B, nb, diag) : merge_split(A, na, B, nb, diag);
  if (!warp_mode || (threadIdx.x & 31u) == 0) {
    split[t] = a;
    // starting segments of the tile's A / B slices (segmented views)
    split[(ntiles + 1) + t] = A.lo ? A.seg(A.off + a) : 0u;
    split[2 * (ntiles + 1) + t] = B.lo ? B.seg(B.off + (diag - a)) : 0u;
  }
}

// Level-run file seams, checked before any merge pass: the last record of
// file f-1 against the first record of file f, for every file f that is not
// the first of its run. A violated seam makes that run per-file runs (the
// reference merges per-file runs); order violations inside
// a file are OrderingErrors raised by the merge.
//   first_of_run[f]: index of the first file of f's run
template <int W>
__global__ void seam_check_kernel(RunView<W> v, const uint64_t* fbase, const uint32_t* first_of_run, uint32_t nfiles,
                                  uint32_t* bad) {
  const uint32_t f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nfiles) return;
  uint32_t b = 0;
  const uint64_t g = fbase[f];
  if (first_of_run[f] != f && g < fbase[f + 1] && g > fbase[first_of_run[f]]) b = rec_cmp(v[g - 1], v[g]) >= 0;
  bad[f] = b;
}

template <int W>
struct MergeArgs {
  RunView<W> A;
  uint64_t na;
  RunView<W> B;
  uint64_t nb;
  const uint64_t* split;  // [3][ntiles+1]: A elements before each tile, then A / B starting segments
  uint64_t ntiles;
  Rec<W>* out;            // plain pass: out[0 .. na+nb); resolve pass: survivors
  uint64_t a_run_base, b_run_base;  // record index of A[0] / B[0] in the decoded array
  unsigned long long* err_order;    // min(position in decoded array of the later element)
  // resolve pass only
  ResolveArgs ra;
  uint32_t* tile_cnt;     // resolve pass: survivors of each tile, written at out + tile * merge_tile_n<W>()
};

// Shared-memory tile layout: 16 bytes of padding after every 8 records. A
// thread's heads sit ~8 records (256 B) from its neighbours'; unpadded, all
// threads of a phase hit the same banks (ncu: 79% excess wavefronts).
constexpr uint32_t kMergePad = 16;
template <int W>
__host__ __device__ constexpr uint32_t mrg_off(uint32_t i) {
  return i * (uint32_t)sizeof(Rec<W>) + (i >> 3) * kMergePad;
}
template <int W>
__host__ __device__ constexpr uint32_t mrg_bytes(uint32_t n) {
  return mrg_off<W>(n) + kMergePad;
}

template <int W>
__global__ void __launch_bounds__(kMergeThreads) merge_kernel(MergeArgs<W> m) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* Sb = smem_raw;
  auto SR = [&](uint32_t i) -> const Rec<W>& { return *reinterpret_cast<const Rec<W>*>(Sb + mrg_off<W>(i)); };
  uint16_t* perm = reinterpret_cast<uint16_t*>(smem_raw + mrg_bytes<W>(merge_tile_n<W>()));
  uint16_t* comp = perm;  // the resolve pass compacts from registers into the same array
  __shared__ uint32_t s_warp[kMergeThreads / 32];
  __shared__ unsigned long long s_base;
  __shared__ uint32_t s_total;
  const uint32_t tid = threadIdx.x;
  const uint64_t tile = blockIdx.x;
  if (tile >= m.ntiles) return;
  const uint64_t d0 = tile * merge_tile_n<W>();
  const uint64_t d1 = (d0 + merge_tile_n<W>() < m.na + m.nb) ? d0 + merge_tile_n<W>() : m.na + m.nb;
  uint64_t a0 = m.split[tile], a1 = m.split[tile + 1];
  uint64_t b0 = d0 - a0, b1 = d1 - a1;
  if (a1 < a0 || b1 < b0) {
    // Split points are monotone only over sorted runs: an unsorted run is an
    // OrderingError, never an out-of-bounds tile load. The tile is emptied (its
    // survivor count is 0).
    if (tid == 0) atomicMin(m.err_order, (unsigned long long)(m.a_run_base + a0));
    a1 = a0;
    b1 = b0;
  }
  const uint32_t na_t = (uint32_t)(a1 - a0), nb_t = (uint32_t)(b1 - b0);
  const uint32_t nt = na_t + nb_t;
  const uint32_t sa = (uint32_t)m.split[(m.ntiles + 1) + tile], sb = (uint32_t)m.split[2 * (m.ntiles + 1) + tile];
  // ---- load the A and B slices into the padded layout: per-thread async
  // 16-byte (8-byte) copies. (One bulk copy per 8-record group serialised on
  // the SM's TMA unit: ~256 copies per tile.)
  {
    constexpr uint32_t RS = (uint32_t)sizeof(Rec<W>);
    constexpr uint32_t CH = (RS % 16 == 0) ? 16u : 8u;
    constexpr uint32_t NC = RS / CH;  // chunks per record
    auto copy = [&](uint32_t dst0) {
      return [&, dst0](const Rec<W>* src, uint64_t cnt, uint64_t at) {
        const uint8_t* gs = reinterpret_cast<const uint8_t*>(src);
        const uint32_t r0 = dst0 + (uint32_t)at;
        for (uint32_t c = tid; c < (uint32_t)cnt * NC; c += kMergeThreads) {
          uint8_t* d = Sb + mrg_off<W>(r0 + c / NC) + CH * (c % NC);
          if (CH == 16) cp_async16(d, gs + 16ull * c);
          else cp_async8(d, gs + 8ull * c);
        }
      };
    };
    m.A.pieces(a0, a1, copy(0), sa);
    m.B.pieces(b0, b1, copy(na_t), sb);
    cp_async_wait_all();
    __syncthreads();
  }
  // Strict-order check of both slices: inside the tile, the merge loop below
  // compares every consumed element with the next one of its run (both in
  // registers); here only the seams to the previous tile.
  if (tid == 0) {
    if (na_t > 0 && a0 > 0 && rec_cmp(m.A.at_near(a0 - 1, sa), SR(0)) >= 0)
      atomicMin(m.err_order, (unsigned long long)(m.a_run_base + a0));
    if (nb_t > 0 && b0 > 0 && rec_cmp(m.B.at_near(b0 - 1, sb), SR(na_t)) >= 0)
      atomicMin(m.err_order, (unsigned long long)(m.b_run_base + b0));
  }
  // ---- per-thread merge of merge_items<W>() outputs (heads kept in registers) ----
  const uint32_t p0 = tid * merge_items<W>();
  uint32_t keep_bits = 0, cnt = 0;
  uint16_t my_perm[merge_items<W>()];
  if (p0 < nt) {
    uint32_t lo = p0 > nb_t ? p0 - nb_t : 0;
    uint32_t hi = p0 < na_t ? p0 : na_t;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (rec_le(SR(mid), SR(na_t + (p0 - 1 - mid)))) lo = mid + 1;
      else hi = mid;
    }
    uint32_t i = lo, j = p0 - lo;
    Rec<W> ha, hb;
    if (i < na_t) ha = SR(i);
    if (j < nb_t) hb = SR(na_t + j);
    // resolve: predecessor of output p0 in merge order
    Rec<W> prev;
    bool has_prev = false;
    if (m.ra.resolve) {
      if (p0 > 0) {
        // the element output just before p0 is the larger of SR(i-1) (A) and SR(na_t+j-1) (B)
        if (i > 0 && j > 0) {
          const Rec<W>& pa = SR(i - 1);
          const Rec<W>& pb = SR(na_t + j - 1);
          prev = rec_le(pa, pb) ? pb : pa;
        } else {
          prev = i > 0 ? SR(i - 1) : SR(na_t + j - 1);
        }
        has_prev = true;
      } else if (d0 > 0) {
        if (a0 > 0 && b0 > 0) {
          const Rec<W> pa = m.A.at_near(a0 - 1, sa), pb = m.B.at_near(b0 - 1, sb);
          prev = rec_le(pa, pb) ? pb : pa;
        } else {
          prev = a0 > 0 ? m.A.at_near(a0 - 1, sa) : m.B.at_near(b0 - 1, sb);
        }
        has_prev = true;
      }
    }
#pragma unroll
    for (int k = 0; k < merge_items<W>(); ++k) {
      const uint32_t p = p0 + k;
      if (p < nt) {
        bool takeA;
        if (i >= na_t) takeA = false;
        else if (j >= nb_t) takeA = true;
        else takeA = rec_le(ha, hb);
        const Rec<W> cur = takeA ? ha : hb;
        my_perm[k] = (uint16_t)(takeA ? i : na_t + j);
        if (!m.ra.resolve) perm[p] = my_perm[k];
        if (takeA) {
          ++i;
          if (i < na_t) {
            ha = SR(i);
            if (rec_cmp(cur, ha) >= 0) atomicMin(m.err_order, (unsigned long long)(m.a_run_base + a0 + i));
          }
        } else {
          ++j;
          if (j < nb_t) {
            hb = SR(na_t + j);
            if (rec_cmp(cur, hb) >= 0) atomicMin(m.err_order, (unsigned long long)(m.b_run_base + b0 + j));
          }
        }
        if (m.ra.resolve) {
          const bool first = !has_prev || !same_user(prev, cur);
          bool keep = first && above_lo(cur, m.ra.range_lo) && below_hi(cur, m.ra.range_hi);
          if (keep && is_tombstone(cur) && !covered_below(cur, m.ra)) keep = false;
          if (keep) {
            keep_bits |= 1u << k;
            ++cnt;
          }
          prev = cur;
          has_prev = true;
        }
      }
    }
  }
  __syncthreads();
  if (!m.ra.resolve) {
    constexpr int R16 = sizeof(Rec<W>) / 16;
    if (R16 * 16 == sizeof(Rec<W>)) {
      uint4* go = reinterpret_cast<uint4*>(m.out + d0);
      for (uint32_t i = tid; i < nt * R16; i += kMergeThreads)
        go[i] = *reinterpret_cast<const uint4*>(Sb + mrg_off<W>(perm[i / R16]) + 16 * (i % R16));
    } else {
      constexpr int RW = sizeof(Rec<W>) / 8;
      uint64_t* go = reinterpret_cast<uint64_t*>(m.out + d0);
      for (uint32_t i = tid; i < nt * RW; i += kMergeThreads)
        go[i] = *reinterpret_cast<const uint64_t*>(Sb + mrg_off<W>(perm[i / RW]) + 8 * (i % RW));
    }
    return;
  }
  // ---- CTA exclusive scan of keep counts; the tile's survivors go to its own
  // segment (out + tile * merge_tile_n<W>()) and merge_densify_kernel packs the
  // segments once every count is known — no look-back between tiles ----
  const uint32_t lane = lane_id(), wid = tid >> 5;
  const uint32_t incl = warp_incl_scan<uint32_t>(cnt);
  if (lane == 31) s_warp[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    const uint32_t v = lane < kMergeThreads / 32 ? s_warp[lane] : 0;
    const uint32_t vi = warp_incl_scan<uint32_t>(v);
    if (lane < kMergeThreads / 32) s_warp[lane] = vi - v;
    const uint32_t total = __shfl_sync(0xFFFFFFFFu, vi, 31);
    if (lane == 0) {
      s_base = tile * (uint64_t)merge_tile_n<W>();
      s_total = total;
      m.tile_cnt[tile] = total;
    }
  }
  __syncthreads();
  uint32_t w = s_warp[wid] + incl - cnt;
#pragma unroll
  for (int k = 0; k < merge_items<W>(); ++k)
    if (keep_bits & (1u << k)) comp[w++] = my_perm[k];
  __syncthreads();
  {
    const uint32_t tot = s_total;
    constexpr int R16 = sizeof(Rec<W>) / 16;
    if (R16 * 16 == sizeof(Rec<W>) && (s_base * sizeof(Rec<W>)) % 16 == 0) {
      uint4* go = reinterpret_cast<uint4*>(m.out + s_base);
      for (uint32_t i = tid; i < tot * R16; i += kMergeThreads)
        go[i] = *reinterpret_cast<const uint4*>(Sb + mrg_off<W>(comp[i / R16]) + 16 * (i % R16));
    } else {
      constexpr int RW = sizeof(Rec<W>) / 8;
      uint64_t* go = reinterpret_cast<uint64_t*>(m.out + s_base);
      for (uint32_t i = tid; i < tot * RW; i += kMergeThreads)
        go[i] = *reinterpret_cast<const uint64_t*>(Sb + mrg_off<W>(comp[i / RW]) + 8 * (i % RW));
    }
  }
}

// Packs the resolve pass's tile segments: tile t's cnt survivors (at
// seg + t * merge_tile_n<W>()) to out + lo[t] (lo: exclusive scan of the counts).
template <int W>
__global__ void __launch_bounds__(256) merge_densify_kernel(const Rec<W>* seg, const uint64_t* lo, uint64_t ntiles,
                                                            Rec<W>* out) {
  const uint64_t t = blockIdx.x;
  if (t >= ntiles) return;
  const uint64_t base = lo[t], cnt = lo[t + 1] - base;
  const Rec<W>* src = seg + t * (uint64_t)merge_tile_n<W>();
  constexpr int R16 = sizeof(Rec<W>) / 16;
  if (R16 * 16 == sizeof(Rec<W>) && (base * sizeof(Rec<W>)) % 16 == 0) {
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    uint4* d4 = reinterpret_cast<uint4*>(out + base);
    for (uint64_t i = threadIdx.x; i < cnt * R16; i += blockDim.x) d4[i] = s4[i];
  } else {
    constexpr int RW = sizeof(Rec<W>) / 8;
    const uint64_t* s8 = reinterpret_cast<const uint64_t*>(src);
    uint64_t* d8 = reinterpret_cast<uint64_t*>(out + base);
    for (uint64_t i = threadIdx.x; i < cnt * RW; i += blockDim.x) d8[i] = s8[i];
  }
}

}  // namespace luda
