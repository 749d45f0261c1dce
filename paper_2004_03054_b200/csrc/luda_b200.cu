// luda_b200.cu — C ABI (include/luda_b200.h) and the native job orchestrator.
//
// Single translation unit: every stage header is included here so device
// globals (CRC tables) need no relocatable device code.
//
// luda_compact(job) runs the fused compaction pipeline on one stream:
//   parse_files_a + crc_flat     footer/filter/index checks   (sst.py:284-310)
//   parse_files_c                data-block table
//   decode_kernel<W>             CRC verify + parse → records (blocks.py:130-165)
//   merge passes <W>             merge path + resolve + compaction (SPEC D12/D20)
//   block_jump + chain           exact SstBuilder block cut     (sst.py:138-162)
//   scan + sst_jump + chain      exact SST cut (SizeOverflowError rule)
//   encode_kernel<W>             data blocks (blocks.py:77-103)
//   sst_meta_kernel<W>           filter, index, footer          (bloom.py:71-88, sst.py:67-76, 206-208)
// Host syncs happen only where a count decides the next launch shape.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <stdlib.h>

#include <algorithm>
#include <mutex>
#include <cmath>
#include <string>
#include <vector>

#include "../../include/luda_b200.h"
#include "luda_common.cuh"
#include "luda_decode.cuh"
#include "luda_dispatch.cuh"
#include "luda_encode.cuh"
#include "luda_merge.cuh"
#include "luda_parse.cuh"
#include "luda_plan.cuh"
#include "luda_read.cuh"
#include "luda_rec.cuh"
#include "luda_tables.cuh"

using namespace luda;

namespace {

thread_local std::string g_err;
thread_local int64_t g_err_off = -1;
int g_device = -1;
int g_num_sms = 148;
uint32_t g_planner_tile = 8192;  // LUDA_OPT_PLANNER_TILE
uint32_t g_dec_ctas = 0;         // LUDA_OPT_DEC_CTAS (0: one per SM)
uint32_t g_dec_segs = 0;         // LUDA_OPT_DEC_SEGS (0: automatic)

int fail(int status, const std::string& msg, int64_t off = -1) {
  g_err = msg;
  g_err_off = off;
  return status;
}

#define CK(expr)                                                                       \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(LUDA_DEVICE, std::string(#expr " failed: ") + cudaGetErrorString(e_)); \
  } while (0)

// Persistent device workspace: a bump allocator over cudaMalloc'd chunks
// that is reset at the start of every job, so steady-state jobs do no device
// allocation at all (multi-GB scratch would otherwise be re-mapped per job).
struct Workspace {
  struct Chunk {
    char* p;
    uint64_t size, used;
  };
  std::vector<Chunk> chunks;
  void reset() {
    for (auto& c : chunks) c.used = 0;
  }
  void* get(uint64_t bytes) {
    bytes = (bytes + 255) & ~uint64_t(255);
    for (auto& c : chunks)
      if (c.size - c.used >= bytes) {
        void* p = c.p + c.used;
        c.used += bytes;
        return p;
      }
    const uint64_t sz = std::max<uint64_t>(bytes, 256ull << 20);
    void* p = nullptr;
    if (cudaMalloc(&p, sz) != cudaSuccess) return nullptr;
    chunks.push_back({reinterpret_cast<char*>(p), sz, bytes});
    return p;
  }
  void release_all() {
    for (auto& c : chunks) cudaFree(c.p);
    chunks.clear();
  }
};
Workspace g_ws;

// Output buffers handed to the caller (luda_job_result.out); recycled by
// luda_job_release.
struct OutCache {
  struct Buf {
    void* p;
    uint64_t size;
    bool used;
  };
  std::vector<Buf> bufs;
  void* get(uint64_t bytes) {
    Buf* best = nullptr;
    for (auto& b : bufs)
      if (!b.used && b.size >= bytes && (!best || b.size < best->size)) best = &b;
    if (best) {
      best->used = true;
      return best->p;
    }
    void* p = nullptr;
    const uint64_t sz = bytes + (bytes >> 3) + 4096;
    if (cudaMalloc(&p, sz) != cudaSuccess) return nullptr;
    bufs.push_back({p, sz, true});
    return p;
  }
  bool put(void* p) {
    for (auto& b : bufs)
      if (b.p == p) {
        b.used = false;
        return true;
      }
    return false;
  }
};
OutCache g_out;
std::mutex g_job_mu;  // one job at a time per process (shared workspace)

struct Scratch {
  cudaStream_t st;
  explicit Scratch(cudaStream_t s) : st(s) { g_ws.reset(); }
  template <typename T>
  T* get(uint64_t count, bool zero = false) {
    const uint64_t bytes = std::max<uint64_t>(count * sizeof(T), 16) + 256;
    void* p = g_ws.get(bytes);
    if (!p) return nullptr;
    if (zero) cudaMemsetAsync(p, 0, bytes, st);
    return reinterpret_cast<T*>(p);
  }
};

#define GET(var, T, count, zero)                                                  \
  T* var = scratch.get<T>((count), (zero));                                       \
  if (!var) return fail(LUDA_DEVICE, "device allocation failed (" #var ")");

struct JobPriv {
  std::vector<uint64_t> off, len;
  std::vector<uint8_t> keys;
  std::vector<uint32_t> klens;
  cudaStream_t st = nullptr;  // stream the output buffer was allocated on
};

// Event pairs bracketing single kernels (k_ms of luda_job_result).
struct KTimer {
  cudaEvent_t a[8], b[8];
  bool used[8] = {};
  KTimer() {
    for (int i = 0; i < 8; ++i) { cudaEventCreate(&a[i]); cudaEventCreate(&b[i]); }
  }
  ~KTimer() {
    for (int i = 0; i < 8; ++i) { cudaEventDestroy(a[i]); cudaEventDestroy(b[i]); }
  }
  void start(int i, cudaStream_t s) { cudaEventRecord(a[i], s); used[i] = true; }
  void stop(int i, cudaStream_t s) { cudaEventRecord(b[i], s); }
  void read(double* out) {
    for (int i = 0; i < 8; ++i) {
      float ms = 0;
      if (used[i] && cudaEventElapsedTime(&ms, a[i], b[i]) == cudaSuccess) out[i] = ms;
    }
  }
};
thread_local KTimer* g_kt = nullptr;
thread_local uint64_t g_launches = 0;
#define KT_START(i, s) do { if (g_kt) g_kt->start(i, s); } while (0)
#define KT_STOP(i, s) do { if (g_kt) g_kt->stop(i, s); } while (0)

const char* file_msg(uint32_t code) {
  switch (code) {
    case F_SHORT: return "file too short for footer";
    case F_FILTER_SHORT: return "filter block too short";
    case F_INDEX_SHORT: return "index block too short";
    case F_IDX_VARINT_TRUNC: return "truncated varint";
    case F_IDX_VARINT_LONG: return "varint too long";
    case F_IDX_TRUNC: return "truncated index entry";
    case F_IDX_TRAILING: return "trailing garbage in index block";
    default: return "format error";
  }
}

// Small pinned host slots for per-job D2H of counters / error words (a D2H
// into pageable memory would block the host at the copy).
struct PinnedSlots {
  unsigned long long* herr = nullptr;
  uint64_t* hm = nullptr;
  int init() {
    if (herr) return LUDA_OK;
    void* p = nullptr;
    if (cudaHostAlloc(&p, 64, cudaHostAllocDefault) != cudaSuccess) return fail(LUDA_DEVICE, "pinned alloc failed");
    herr = reinterpret_cast<unsigned long long*>(p);
    hm = reinterpret_cast<uint64_t*>(herr + 2);
    return LUDA_OK;
  }
};
PinnedSlots g_pin;

// Filter / index CRCs of a job's input files, computed on a side stream while
// the block table and the decode run (jobs are serialised by g_job_mu, so one
// instance serves every job). h: pinned, crc[2 nf] then stored[2 nf].
struct DeferredCrc {
  cudaStream_t side = nullptr;
  cudaEvent_t parsed = nullptr, done = nullptr;
  uint32_t* h = nullptr;
  uint64_t cap = 0;
  uint32_t nf = 0;
  bool pending = false;
  std::vector<FileInfo> info;
  int prepare(uint32_t n) {
    pending = false;
    if (!side) {
      if (cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&parsed, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&done, cudaEventDisableTiming) != cudaSuccess)
        return fail(LUDA_DEVICE, "side stream / event creation failed");
    }
    if (4ull * n > cap) {
      if (h) cudaFreeHost(h);
      cap = std::max<uint64_t>(4ull * n, 1024);
      if (cudaHostAlloc(&h, cap * 4, cudaHostAllocDefault) != cudaSuccess) {
        h = nullptr;
        cap = 0;
        return fail(LUDA_DEVICE, "pinned CRC staging allocation failed");
      }
    }
    nf = n;
    info.assign(n, FileInfo{});
    return LUDA_OK;
  }
};
DeferredCrc g_dcrc;

int check_parsed_file(const FileInfo& fi, const uint32_t* crc, const uint32_t* stored);

// The deferred filter / index CRC comparisons, files in job order (the
// structural checks of every file passed before the job went on).
int deferred_crc_check() {
  DeferredCrc& dc = g_dcrc;
  if (!dc.pending) return LUDA_OK;
  dc.pending = false;
  CK(cudaEventSynchronize(dc.done));
  for (uint32_t f = 0; f < dc.nf; ++f) {
    const int rc = check_parsed_file(dc.info[f], dc.h + 2 * f, dc.h + 2 * dc.nf + 2 * f);
    if (rc) return rc;
  }
  return LUDA_OK;
}

// Table.__init__ (sst.py:284-310) outcome of one parsed file, in the
// reference's check order: footer/magic/filter length, filter CRC, probe
// count, index length, index CRC, index entries. crc/stored: filter, index.
int check_parsed_file(const FileInfo& fi, const uint32_t* crc, const uint32_t* stored) {
  char buf[96];
  if (fi.code == F_MAGIC) {
    snprintf(buf, sizeof buf, "bad magic 0x%016llx", (unsigned long long)fi.magic);
    return fail(LUDA_FORMAT, buf);
  }
  if (fi.code) return fail(LUDA_FORMAT, file_msg(fi.code));
  if (crc[0] != stored[0]) return fail(LUDA_CORRUPT, "filter block checksum mismatch", (int64_t)fi.filter_off);
  if (fi.kbad) {
    snprintf(buf, sizeof buf, "bad probe count %u", fi.kbyte);
    return fail(LUDA_FORMAT, buf);
  }
  if (fi.icode == F_INDEX_SHORT) return fail(LUDA_FORMAT, file_msg(fi.icode));
  if (crc[1] != stored[1]) return fail(LUDA_CORRUPT, "index block checksum mismatch", (int64_t)fi.index_off);
  if (fi.icode) return fail(LUDA_FORMAT, file_msg(fi.icode));
  return LUDA_OK;
}

const char* block_msg(uint32_t code) {
  switch (code) {
    case B_SHORT: return "block too short";
    case B_CRC: return "data block checksum mismatch";
    case B_RESTART: return "bad restart array";
    case B_VARINT_TRUNC: return "truncated varint";
    case B_VARINT_LONG: return "varint too long";
    case B_TRUNC_ENTRY: return "truncated block entry";
    case B_TRAILING: return "trailing garbage in block entries";
    case B_KEYLEN: return "keys of differing lengths in one job are not supported by the b200 fast path";
    case B_VALUE_BIG: return "value longer than 16 MiB (or arena beyond 1 TiB) not supported by the b200 fast path";
    case B_KEYLONG: return "user keys longer than 71 bytes (or internal keys shorter than the 8-byte trailer) are not supported by the b200 path";
    default: return "block error";
  }
}

int sync(cudaStream_t st) {
  CK(cudaStreamSynchronize(st));
  CK(cudaGetLastError());
  return LUDA_OK;
}

double ev_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

// Host transform of a user-key bound into the padded L-byte comparison domain
// (see luda_merge.cuh). `lower` = bound is a lower bound (k >= b); `closed`
// selects <=/>= vs </>.
KeyBound make_bound(const uint8_t* key, uint32_t klen, uint32_t L, bool lower, bool closed) {
  // Comparisons are done on user keys zero-padded to L bytes (luda_merge.cuh).
  //   lower, closed (k >= key):  klen <= L → pad(k) >= pad(key); klen > L → pad(k) > pad(key[:L])
  //   upper, closed (k <= key):  klen == L → <=;  klen < L → <;  klen > L → <= pad(key[:L])
  //   upper, open   (k <  key):  klen <= L → <;   klen > L → <= pad(key[:L])
  KeyBound b{};
  b.present = 1;
  uint8_t pad[32] = {0};
  memcpy(pad, key, std::min(klen, L));
  for (int w = 0; w < 4; ++w) {
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v = (v << 8) | pad[8 * w + i];
    b.k[w] = v;
  }
  if (lower) b.incl = klen <= L;
  else if (closed) b.incl = klen >= L;
  else b.incl = klen > L;
  return b;
}

// Var jobs (luda_rec.cuh): the bound is represented exactly — padded to
// 8 W - 1 bytes plus its length byte — so comparisons are exact.
KeyBound make_bound_var(const uint8_t* key, uint32_t klen, bool lower, bool closed, uint32_t W) {
  KeyBound b{};
  b.present = 1;
  uint8_t pad[8 * kVarWLong] = {0};
  memcpy(pad, key, std::min<uint32_t>(klen, 8 * W - 1));
  pad[8 * W - 1] = (uint8_t)klen;
  for (uint32_t w = 0; w < W; ++w) {
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v = (v << 8) | pad[8 * w + i];
    b.k[w] = v;
  }
  b.incl = lower ? 1u : (closed ? 1u : 0u);
  return b;
}

struct RunSeg {
  uint64_t start, len;
};

// Merge sorted runs (logical record ranges) down to one, fusing version
// resolution into the last pass. Pass 1 reads the decoder's segmented array
// `X` through `seg`; later passes ping-pong between dense buffers (X is
// reused densely: its physical capacity >= the record count).
template <int W>
int merge_runs(cudaStream_t st, Scratch& scratch, Rec<W>* X, const RunView<W>& seg, Rec<W>* Y, Rec<W>* S,
               std::vector<RunSeg> runs, const ResolveArgs& ra_final, unsigned long long* d_err_order,
               unsigned long long* d_nout) {
  // drop empty runs
  std::vector<RunSeg> segs;
  for (auto& r : runs)
    if (r.len) segs.push_back(r);
  if (segs.empty()) {
    CK(cudaMemsetAsync(d_nout, 0, 8, st));
    return LUDA_OK;
  }
  bool first_pass = true;
  const size_t smem = mrg_bytes<W>(merge_tile_n<W>()) + 2 * merge_tile_n<W>();
  CK(cudaFuncSetAttribute(merge_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  Rec<W>* cur = X;
  Rec<W>* nxt = Y;
  auto view = [&](const RunSeg& r) {
    RunView<W> v = seg;
    if (!first_pass) v = RunView<W>{cur, nullptr, 0, 1, 0};
    v.off = r.start;
    return v;
  };
  auto launch = [&](const RunView<W>& A, uint64_t na, const RunView<W>& B, uint64_t nb, Rec<W>* out, uint64_t abase,
                    uint64_t bbase, bool resolve) -> int {
    const uint64_t ntiles = (na + nb + merge_tile_n<W>() - 1) / merge_tile_n<W>();
    GET(split, uint64_t, 3 * (ntiles + 1), false);
    const bool warp_mode = ntiles + 1 <= 32ull * g_num_sms;
    merge_partition_kernel<W><<<(unsigned)(warp_mode ? (ntiles + 1 + 7) / 8 : (ntiles + 1 + 255) / 256), 256, 0, st>>>(
        A, na, B, nb, ntiles, split, warp_mode);
    ++g_launches;
    MergeArgs<W> m{};
    m.A = A; m.na = na; m.B = B; m.nb = nb; m.split = split; m.ntiles = ntiles; m.out = out;
    m.a_run_base = abase; m.b_run_base = bbase;
    m.err_order = d_err_order;  // order errors are reported for original runs only
    m.ra.resolve = resolve;
    uint32_t* tile_cnt = nullptr;
    Rec<W>* seg_out = out;
    if (resolve) {
      m.ra = ra_final;
      m.ra.resolve = true;
      GET(tc, uint32_t, ntiles, false);
      tile_cnt = tc;
      m.tile_cnt = tc;
      seg_out = nxt;  // tile segments; the final pass never reads `nxt`
      m.out = seg_out;
    }
    if (!first_pass) {
      GET(sink, unsigned long long, 1, true);
      m.err_order = sink;
    }
    if (resolve) KT_START(1, st);
    merge_kernel<W><<<(unsigned)ntiles, kMergeThreads, smem, st>>>(m);
    ++g_launches;
    if (resolve) {
      // tile counts → segment bases → packed survivors in `out`; n_out = total
      GET(lo, uint64_t, ntiles + 1, false);
      const uint64_t nt = std::max<uint64_t>(1, (ntiles + kScanThreads * kScanItems - 1) / (kScanThreads * kScanItems));
      GET(lb, uint64_t, nt, true);
      GET(ctr, unsigned int, 1, true);
      scan_excl_kernel<uint32_t><<<(unsigned)nt, kScanThreads, 0, st>>>(tile_cnt, ntiles, lo, lb, ctr);
      merge_densify_kernel<W><<<(unsigned)ntiles, 256, 0, st>>>(seg_out, lo, ntiles, out);
      g_launches += 2;
      CK(cudaMemcpyAsync(d_nout, lo + ntiles, 8, cudaMemcpyDeviceToDevice, st));
      KT_STOP(1, st);
    }
    CK(cudaGetLastError());
    return LUDA_OK;
  };
  while (segs.size() > 2) {
    std::vector<RunSeg> next;
    for (size_t i = 0; i < segs.size(); i += 2) {
      if (i + 1 < segs.size()) {
        const RunSeg a = segs[i], b = segs[i + 1];
        int rc = launch(view(a), a.len, view(b), b.len, nxt + a.start, a.start, b.start, false);
        if (rc) return rc;
        next.push_back({a.start, a.len + b.len});
      } else {
        const RunSeg a = segs[i];
        if (first_pass) {  // still order-check the odd run (and densify it)
          int rc = launch(view(a), a.len, view(a), 0, nxt + a.start, a.start, a.start, false);
          if (rc) return rc;
        } else {
          CK(cudaMemcpyAsync(nxt + a.start, cur + a.start, a.len * sizeof(Rec<W>), cudaMemcpyDeviceToDevice, st));
        }
        next.push_back(a);
      }
    }
    segs = next;
    std::swap(cur, nxt);
    first_pass = false;
  }
  if (segs.size() == 2) return launch(view(segs[0]), segs[0].len, view(segs[1]), segs[1].len, S, segs[0].start,
                                      segs[1].start, true);
  return launch(view(segs[0]), segs[0].len, view(segs[0]), 0, S, segs[0].start, segs[0].start, true);
}

struct ChainBufs {
  uint32_t* nodes;
  uint32_t n_nodes;
};

// Greedy chain over jmp[0..n) with max jump D; returns nodes (device) + count.
int run_chain(cudaStream_t st, Scratch& scratch, const uint32_t* jmp, uint32_t n, uint32_t D, uint32_t T_min,
              ChainBufs& outb) {
  if (n == 0) {
    outb.n_nodes = 0;
    outb.nodes = nullptr;
    return LUDA_OK;
  }
  D = std::max<uint32_t>(D, 1);
  // Tile: T_min (default 8192) for large inputs, shrunk so that small ones still
  // spread over >= 2 tiles per SM — the map / emit kernels walk a tile serially
  // (c2: 21.6K survivors in 3 tiles of 8192 made the block chain ~0.2 ms).
  const uint32_t T_fill = (uint32_t)((n + 2ull * g_num_sms - 1) / (2ull * g_num_sms));
  uint32_t T = std::max<uint32_t>(std::min<uint32_t>(T_min, std::max<uint32_t>(T_fill, 256)), D);
  T = (T + 31) & ~31u;
  const uint32_t ntiles = (uint32_t)((n + (uint64_t)T - 1) / T);
  const uint32_t G = std::max<uint32_t>(1, (uint32_t)std::ceil(std::sqrt((double)ntiles)));
  const uint32_t ngroups = (ntiles + G - 1) / G;
  ChainArgs c{};
  c.jmp = jmp; c.n = n; c.T = T; c.D = D; c.ntiles = ntiles; c.G = G; c.ngroups = ngroups;
  GET(ex, uint32_t, (uint64_t)ntiles * D, false);
  GET(cn, uint32_t, (uint64_t)ntiles * D, false);
  GET(gex, uint32_t, (uint64_t)ngroups * D, false);
  GET(gcn, uint32_t, (uint64_t)ngroups * D, false);
  GET(gen, uint32_t, ngroups, false);
  GET(gba, uint32_t, ngroups, false);
  GET(nodes, uint32_t, n, false);
  GET(nn, uint32_t, 1, true);
  c.exit_ = ex; c.cnt = cn; c.gexit = gex; c.gcnt = gcn; c.gentry = gen; c.gbase = gba; c.nodes = nodes; c.nnodes = nn;
  const size_t sm = T <= 12288 ? (size_t)T * 4 : 0;
  if (sm > 48 * 1024) CK(cudaFuncSetAttribute(chain_map_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  chain_map_kernel<<<ntiles, kChainThreads, sm, st>>>(c);
  ++g_launches;
  chain_group_kernel<<<ngroups, kChainThreads, kChainStage, st>>>(c);
  ++g_launches;
  chain_top_kernel<<<1, 1024, kChainStage, st>>>(c);
  ++g_launches;
  GET(tentry, uint32_t, ntiles, false);
  GET(tbase, uint32_t, ntiles, false);
  chain_tile_entry_kernel<<<ngroups, kChainThreads, kChainStage, st>>>(c, tentry, tbase);
  ++g_launches;
  if (sm > 48 * 1024) CK(cudaFuncSetAttribute(chain_emit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  chain_emit_kernel<<<ntiles, kChainThreads, sm, st>>>(c, tentry, tbase);
  ++g_launches;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(&outb.n_nodes, nn, 4, cudaMemcpyDeviceToHost, st));
  int rc = sync(st);
  if (rc) return rc;
  outb.nodes = nodes;
  return LUDA_OK;
}

struct EmitParams {
  uint32_t K, block_size, ri, bpk;
  uint64_t sst_target;
  uint32_t min_entry;         // lower bound of one encoded entry (sizes the planner halo)
  uint64_t file_entries = 0;  // > 0: cut an SST every file_entries entries instead of by size
  bool var = false;           // generic-length keys (W = kVarW / kVarWLong records)
};

// Plan + encode the survivors `S[0..n)` whose values live in `varena`.
template <int W>
int plan_and_emit(cudaStream_t st, Scratch& scratch, const Rec<W>* S, uint64_t n, const uint8_t* varena,
                  const EmitParams& p, luda_job_result* res, cudaEvent_t* ev) {
  JobPriv* priv = new JobPriv();
  res->priv = priv;
  res->key_len = p.K;
  res->n_out = n;
  if (n == 0) {
    res->n_sst = 0;
    res->out = nullptr;
    res->out_bytes = 0;
    return LUDA_OK;
  }
  if (n >= 0xFFFFFFF0ull) return fail(LUDA_UNSUPPORTED, "more than 2^32 surviving entries in one job");
  // ---- block jumps ----
  const uint32_t max_entries = std::max<uint32_t>(1, (p.block_size > 8 ? (p.block_size - 8) / p.min_entry : 0) + 1);
  const uint32_t halo = ((max_entries + 1 + 31) / 32) * 32;
  if (halo > 8192) return fail(LUDA_UNSUPPORTED, "block_size too large for the b200 planner");
  GET(jmp, uint32_t, n, false);
  GET(bsz, uint32_t, n, false);
  GET(ctl, unsigned int, 4, true);  // jmax, overflow, jmax_sst
  // kJumpTile survivors per CTA; small jobs (c2: ~22 K survivors) use smaller
  // tiles so that >= 2 CTAs per SM still run (the halo is re-read per tile)
  const uint64_t fill = (n + 2ull * g_num_sms - 1) / (2ull * g_num_sms);
  const uint32_t jtile = (uint32_t)std::min<uint64_t>(
      kJumpTile, std::max<uint64_t>(kJumpThreads, (fill + kJumpThreads - 1) / kJumpThreads * kJumpThreads));
  BlockJumpArgs<W> ja{S, n, p.K, p.block_size, p.ri, halo, jmp, bsz, ctl, ctl + 1, p.file_entries, p.var, jtile};
  const size_t jsm = (2ull * (jtile + halo) + 1) * 4;
  CK(cudaFuncSetAttribute(block_jump_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)((2ull * (kJumpTile + 8192) + 1) * 4)));
  KT_START(2, st);
  block_jump_kernel<W><<<(unsigned)((n + jtile - 1) / jtile), kJumpThreads, jsm, st>>>(ja);
  ++g_launches;
  KT_STOP(2, st);
  CK(cudaGetLastError());
  unsigned int hctl[4];
  CK(cudaMemcpyAsync(hctl, ctl, 16, cudaMemcpyDeviceToHost, st));
  int rc = sync(st);
  if (rc) return rc;
  if (hctl[1]) return fail(LUDA_DEVICE, "block planner halo overflow");
  ChainBufs bch{};
  rc = run_chain(st, scratch, jmp, (uint32_t)n, hctl[0], g_planner_tile, bch);
  if (rc) return rc;
  const uint32_t nblk = bch.n_nodes;
  res->blocks_out = nblk;
  GET(blk_first, uint32_t, nblk, false);
  GET(blk_n, uint32_t, nblk, false);
  GET(blk_size, uint32_t, nblk, false);
  GET(blk_pos, uint64_t, nblk + 1, false);
  block_desc_kernel<<<(nblk + 255) / 256, 256, 0, st>>>(bch.nodes, nblk, jmp, bsz, blk_first, blk_n, blk_size);
  ++g_launches;
  {
    const uint64_t nt = std::max<uint64_t>(1, (nblk + kScanThreads * kScanItems - 1) / (kScanThreads * kScanItems));
    GET(lb, uint64_t, nt, true);
    GET(ctr, unsigned int, 1, true);
    scan_excl_kernel<uint32_t><<<(unsigned)nt, kScanThreads, 0, st>>>(blk_size, nblk, blk_pos, lb, ctr);
    ++g_launches;
  }
  // ---- SST cut ----
  GET(sjmp, uint32_t, nblk, false);
  if (p.file_entries)
    sst_jump_files_kernel<<<(nblk + 255) / 256, 256, 0, st>>>(blk_first, nblk, p.file_entries, sjmp, ctl + 2);
  else
    sst_jump_kernel<<<(nblk + 255) / 256, 256, 0, st>>>(blk_pos, nblk, p.sst_target, sjmp, ctl + 2);
  ++g_launches;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(hctl, ctl, 16, cudaMemcpyDeviceToHost, st));
  rc = sync(st);
  if (rc) return rc;
  ChainBufs sch{};
  rc = run_chain(st, scratch, sjmp, nblk, hctl[2], g_planner_tile, sch);
  if (rc) return rc;
  const uint32_t nsst = sch.n_nodes;
  GET(sst_size, uint64_t, nsst, false);
  GET(sst_data, uint64_t, nsst, false);
  GET(sst_nent, uint64_t, nsst, false);
  GET(sst_last, uint32_t, nsst, false);
  GET(sst_off, uint64_t, nsst + 1, false);
  uint64_t* blk_ipos = nullptr;  // var jobs: index entries differ in size
  if (p.var) {
    GET(isz, uint32_t, nblk, false);
    GET(ipos, uint64_t, nblk + 1, false);
    index_entry_size_kernel<W><<<(nblk + 255) / 256, 256, 0, st>>>(S, blk_first, blk_n, nblk, isz);
    ++g_launches;
    const uint64_t nt = std::max<uint64_t>(1, (nblk + kScanThreads * kScanItems - 1) / (kScanThreads * kScanItems));
    GET(lb, uint64_t, nt, true);
    GET(ctr, unsigned int, 1, true);
    scan_excl_kernel<uint32_t><<<(unsigned)nt, kScanThreads, 0, st>>>(isz, nblk, ipos, lb, ctr);
    ++g_launches;
    blk_ipos = ipos;
  }
  SstLayoutArgs la{sch.nodes, nsst, nblk, blk_first, blk_pos, n, p.K, p.bpk, sst_size, sst_data, sst_nent, sst_last,
                   blk_ipos};
  sst_layout_kernel<<<(nsst + 255) / 256, 256, 0, st>>>(la);
  ++g_launches;
  {
    const uint64_t nt = std::max<uint64_t>(1, (nsst + kScanThreads * kScanItems - 1) / (kScanThreads * kScanItems));
    GET(lb, uint64_t, nt, true);
    GET(ctr, unsigned int, 1, true);
    scan_excl_kernel<uint64_t><<<(unsigned)nt, kScanThreads, 0, st>>>(sst_size, nsst, sst_off, lb, ctr);
    ++g_launches;
  }
  priv->off.resize(nsst + 1);
  priv->len.resize(nsst);
  std::vector<uint64_t> nent(nsst);
  CK(cudaMemcpyAsync(priv->off.data(), sst_off, 8ull * (nsst + 1), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(priv->len.data(), sst_size, 8ull * nsst, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(nent.data(), sst_nent, 8ull * nsst, cudaMemcpyDeviceToHost, st));
  rc = sync(st);
  if (rc) return rc;
  for (uint32_t s = 0; s < nsst; ++s)  // footer / index offsets are u32 (sst.py:199-208 struct.pack '<IIIIQ')
    if (priv->len[s] > 0xFFFFFFFFull)
      return fail(LUDA_FORMAT, "output SST larger than 4 GiB: u32 footer/index offsets cannot address it");
  if (ev) CK(cudaEventRecord(ev[0], st));
  const uint64_t total = priv->off[nsst];
  // big-filter scratch
  std::vector<uint64_t> soff(nsst, ~0ull);
  uint64_t big_words = 0;
  for (uint32_t s = 0; s < nsst; ++s) {
    uint64_t nbits = std::max<uint64_t>(64, nent[s] * p.bpk);
    nbits = (nbits + 7) & ~7ull;
    if (nbits / 8 + 1 > (uint64_t)kMetaBuf) {
      soff[s] = big_words;
      big_words += (nbits / 8 + 1 + 3) / 4 + 8;
    }
  }
  void* outp = g_out.get(total + 256);
  if (!outp) return fail(LUDA_DEVICE, "output allocation failed");
  priv->st = st;
  res->out = reinterpret_cast<uint8_t*>(outp);
  res->out_bytes = total;
  GET(bigs, uint32_t, big_words + 16, true);
  GET(d_soff, uint64_t, nsst, false);
  CK(cudaMemcpyAsync(d_soff, soff.data(), 8ull * nsst, cudaMemcpyHostToDevice, st));
  const uint32_t key_slot = p.var ? 8 * W + 8 : p.K;
  GET(d_keys, uint8_t, 2ull * nsst * key_slot, false);
  GET(d_klen, uint32_t, 2ull * nsst, false);
  // ---- encode data blocks ----
  GET(blk_out, uint64_t, nblk, false);
  block_out_kernel<<<(nblk + 255) / 256, 256, 0, st>>>(blk_pos, nblk, sch.nodes, nsst, sst_off, blk_out);
  ++g_launches;
#ifdef LUDA_ABLATION
  const uint32_t s_edbg = getenv("LUDA_ENC_DBG") ? (uint32_t)atoi(getenv("LUDA_ENC_DBG")) : 0u;
#else
  const uint32_t s_edbg = 0;
#endif
  EncodeArgs<W> ea{varena, S, p.K, p.ri, nblk, blk_first, blk_n, blk_size, blk_pos, sch.nodes, nsst, sst_off,
                   blk_out, res->out, s_edbg, p.var};
  const size_t esm = sizeof(CrcSmem) + (size_t)kEncPairs * sizeof(EncPairSmem) + sizeof(EncCtaSmem);
  CK(cudaFuncSetAttribute(encode_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)esm));
  const unsigned egrid = (unsigned)std::min<uint64_t>((nblk + kEncPairs - 1) / kEncPairs, (uint64_t)g_num_sms);
  KT_START(3, st);
  encode_kernel<W><<<std::max(1u, egrid), kEncWarps * 32, esm, st>>>(ea);
  ++g_launches;
  KT_STOP(3, st);
  CK(cudaGetLastError());
  // ---- filter / index / footer ----
  const uint32_t kprobes = std::max(1, std::min(30, (int)std::lround(p.bpk * std::log(2.0))));
  MetaArgs<W> ma{S, p.K, p.bpk, kprobes, nsst, sch.nodes, sst_last, sst_off, sst_data, sst_nent, sst_size,
                 blk_first, blk_n, blk_size, blk_pos, res->out, bigs, d_soff, d_keys, d_klen, key_slot, p.var,
                 blk_ipos};
  CK(cudaFuncSetAttribute(sst_meta_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMetaSmem));
  KT_START(4, st);
  sst_meta_kernel<W><<<std::min<uint32_t>(nsst, (uint32_t)g_num_sms), kMetaThreads, kMetaSmem, st>>>(ma);
  ++g_launches;
  KT_STOP(4, st);
  CK(cudaGetLastError());
  if (ev) CK(cudaEventRecord(ev[1], st));
  priv->keys.resize(2ull * nsst * key_slot);
  priv->klens.resize(2ull * nsst);
  CK(cudaMemcpyAsync(priv->keys.data(), d_keys, priv->keys.size(), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(priv->klens.data(), d_klen, 4ull * priv->klens.size(), cudaMemcpyDeviceToHost, st));
  rc = sync(st);
  if (rc) return rc;
  res->n_sst = nsst;
  res->sst_off = priv->off.data();
  res->sst_len = priv->len.data();
  res->sst_keys = priv->keys.data();
  res->sst_key_len = priv->klens.data();
  res->key_len = key_slot;
  return LUDA_OK;
}

constexpr int kRetryVar = 100;   // internal: a fixed-K job met another key length → rerun as a var job
constexpr int kRetryLong = 101;  // internal: a var job met a user key > 71 bytes → rerun with kVarWLong records

constexpr uint64_t merge_tile_slack = 2048;  // >= merge_tile_n<W>() for every W

template <int W>
int compact_w(cudaStream_t st, Scratch& scratch, const luda_job_desc* jd, luda_job_result* res, uint32_t K,
              uint32_t nblk, const BlockTable& bt, const uint32_t* d_file_blk_base,
              cudaEvent_t* ev, bool var) {
  const uint32_t L = K - 8;
  res->blocks_in = nblk;
  // ---- decode ----
  GET(errs, unsigned long long, 2, false);
  const size_t dsm = sizeof(CrcSmem) + (size_t)kDecPairs * sizeof(DecPairSmem) + sizeof(DecCtaSmem);
  CK(cudaFuncSetAttribute(decode_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
  Rec<W>* X = nullptr;
  uint64_t n_in = 0;
  std::vector<uint64_t> fbase(jd->n_files + 1);
  // Single-pass decode into warp segments (luda_decode.cuh). Segment
  // capacity comes from the records-per-input-byte ratio of earlier jobs
  // (first job: 1 record per 48 bytes); a job whose largest segment does not
  // fit is decoded again with the exact capacity.
  // record segments = block chunks handed to the decode pairs dynamically
  // (kDecChunksPerPair per pair on big jobs; one per pair, as long as a
  // chunk would hold >= 8 blocks, on small ones)
  const uint32_t dec_ctas = g_dec_ctas ? std::min<uint32_t>(g_dec_ctas, (uint32_t)g_num_sms) : (uint32_t)g_num_sms;
  const uint32_t npairs = dec_ctas * kDecPairs;
  const uint32_t nw = std::max<uint32_t>(
      1u, std::min<uint32_t>(nblk, g_dec_segs ? g_dec_segs
                                              : std::max<uint32_t>(npairs, std::min<uint32_t>(npairs * kDecChunksPerPair,
                                                                                              nblk / 8))));
  uint64_t blk_bytes = 0;
  for (uint32_t f = 0; f < jd->n_files; ++f) blk_bytes += jd->file_len[f];
  static double s_ratio = 1.0 / 48.0;
  uint64_t seg_cap = (uint64_t)((double)blk_bytes / nw * s_ratio * 1.25) + 4ull * (nblk / nw + 1) + 64;
  GET(d_local, uint32_t, nblk, false);
  GET(d_count, uint64_t, nw, false);
  GET(d_lo, uint64_t, nw + 1, false);
  GET(d_max, uint64_t, 1, false);
  GET(d_ctr, unsigned int, 1, false);
  // file seams of every multi-file run, checked (with the file bases) right
  // after the decode, before any merge pass
  std::vector<uint32_t> run_first(jd->run_first_file, jd->run_first_file + jd->n_runs + 1);
  std::vector<uint32_t> first_of_run(jd->n_files, 0), seam_bad(jd->n_files, 0);
  for (uint32_t r = 0; r + 1 < run_first.size(); ++r)
    for (uint32_t f = run_first[r]; f < run_first[r + 1] && f < jd->n_files; ++f) first_of_run[f] = run_first[r];
  GET(d_fbase, uint64_t, jd->n_files + 1, false);
  GET(d_for, uint32_t, jd->n_files, false);
  GET(d_bad, uint32_t, jd->n_files, false);
  CK(cudaMemcpyAsync(d_for, first_of_run.data(), 4ull * jd->n_files, cudaMemcpyHostToDevice, st));
  for (int attempt = 0; attempt < 2; ++attempt) {
    X = scratch.get<Rec<W>>((uint64_t)nw * seg_cap + merge_tile_slack, false);
    if (!X) return fail(LUDA_DEVICE, "device allocation failed (records)");
    CK(cudaMemsetAsync(errs, 0xFF, 16, st));
    CK(cudaMemsetAsync(d_max, 0, 8, st));
    CK(cudaMemsetAsync(d_ctr, 0, 4, st));
#ifdef LUDA_ABLATION
    static const uint32_t s_dbg = getenv("LUDA_DEC_DBG") ? (uint32_t)atoi(getenv("LUDA_DEC_DBG")) : 0u;
#else
    const uint32_t s_dbg = 0;
#endif
    DecodeArgs<W> da{jd->arena, bt, nblk, K, X, seg_cap, d_local, d_count, nw, d_ctr, errs, errs + 1, s_dbg, var};
    KT_START(0, st);
    decode_kernel<W><<<dec_ctas, kDecWarps * 32, dsm, st>>>(da);
    ++g_launches;
    KT_STOP(0, st);
    CK(cudaGetLastError());
    seg_scan_kernel<<<1, 1024, 0, st>>>(d_count, nw, d_lo, d_max);
    ++g_launches;
    // file bases and file-seam checks ride on the same sync (meaningless if
    // the segment capacity overflowed: then they are recomputed)
    file_entry_base_kernel<<<(jd->n_files + 1 + 255) / 256, 256, 0, st>>>(d_local, d_lo, nblk, nw,
                                                                            d_file_blk_base, jd->n_files, d_fbase);
    ++g_launches;
    {
      const RunView<W> sv{X, d_lo, seg_cap, nw, 0};
      seam_check_kernel<W><<<(jd->n_files + 255) / 256, 256, 0, st>>>(sv, d_fbase, d_for, jd->n_files, d_bad);
      ++g_launches;
    }
    unsigned long long* herr = g_pin.herr;
    uint64_t* hm = g_pin.hm;
    CK(cudaMemcpyAsync(herr, errs, 16, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&hm[0], d_lo + nw, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&hm[1], d_max, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(fbase.data(), d_fbase, 8ull * (jd->n_files + 1), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(seam_bad.data(), d_bad, 4ull * jd->n_files, cudaMemcpyDeviceToHost, st));
    int rc = sync(st);
    if (rc) return rc;
    rc = deferred_crc_check();  // filter / index CRC errors come before any data-block error
    if (rc) return rc;
    if (herr[0] != ~0ull || herr[1] != ~0ull) {
      const bool ref = herr[0] != ~0ull;
      const unsigned long long e = ref ? herr[0] : herr[1];
      const uint32_t b = (uint32_t)(e >> 8), code = (uint32_t)(e & 0xFF);
      uint32_t foff = 0;
      CK(cudaMemcpy(&foff, bt.foff + b, 4, cudaMemcpyDeviceToHost));
      if (!ref && code == B_KEYLEN && !var) return kRetryVar;
      if (!ref && code == B_KEYLONG && W == kVarW) return kRetryLong;  // a user key of 72..255 bytes
      if (!ref) return fail(LUDA_UNSUPPORTED, block_msg(code));
      if (code == B_CRC) return fail(LUDA_CORRUPT, block_msg(code), foff);
      return fail(LUDA_FORMAT, block_msg(code));
    }
    n_in = hm[0];
    if (blk_bytes) s_ratio = std::max(s_ratio * 0.5, (double)n_in / (double)blk_bytes);
    if (hm[1] <= seg_cap) break;
    if (attempt == 1) return fail(LUDA_DEVICE, "decode record capacity overflow");
    seg_cap = hm[1];
  }
  const RunView<W> segview{X, d_lo, seg_cap, nw, 0};
  res->n_in = n_in;
  if (ev) CK(cudaEventRecord(ev[2], st));
  // ---- merge + resolve ----
  ResolveArgs ra{};
  std::vector<KeyBound> bounds;
  {
    const uint8_t* kp = jd->deeper_keys;
    for (uint32_t i = 0; i < jd->n_deeper; ++i) {
      const uint32_t llo = jd->deeper_lens[2 * i], lhi = jd->deeper_lens[2 * i + 1];
      if (var && (llo > var_maxlen<W>() || lhi > var_maxlen<W>())) {
        if (W == kVarW) return kRetryLong;
        return fail(LUDA_UNSUPPORTED, "key-range bound longer than 255 bytes");
      }
      bounds.push_back(var ? make_bound_var(kp, llo, true, true, W) : make_bound(kp, llo, L, true, true));
      kp += llo;
      bounds.push_back(var ? make_bound_var(kp, lhi, false, true, W) : make_bound(kp, lhi, L, false, true));
      kp += lhi;
    }
  }
  KeyBound* d_bounds = nullptr;
  if (!bounds.empty()) {
    d_bounds = scratch.get<KeyBound>(bounds.size(), false);
    if (!d_bounds) return fail(LUDA_DEVICE, "device allocation failed (bounds)");
    CK(cudaMemcpyAsync(d_bounds, bounds.data(), bounds.size() * sizeof(KeyBound), cudaMemcpyHostToDevice, st));
  }
  ra.deeper = d_bounds;
  ra.n_deeper = jd->n_deeper;
  if (var && ((jd->range_lo && jd->range_lo_len > var_maxlen<W>()) ||
              (jd->range_hi && jd->range_hi_len > var_maxlen<W>()))) {
    if (W == kVarW) return kRetryLong;
    return fail(LUDA_UNSUPPORTED, "key-range bound longer than 255 bytes");
  }
  if (jd->range_lo)
    ra.range_lo = var ? make_bound_var(jd->range_lo, jd->range_lo_len, true, true, W)
                      : make_bound(jd->range_lo, jd->range_lo_len, L, true, true);
  if (jd->range_hi)
    ra.range_hi = var ? make_bound_var(jd->range_hi, jd->range_hi_len, false, false, W)
                      : make_bound(jd->range_hi, jd->range_hi_len, L, false, false);
  ra.resolve = true;
  // runs in merge-priority order; a run with a violated file seam is split into per-file runs
  std::vector<RunSeg> runs;
  for (uint32_t r = 0; r + 1 < run_first.size(); ++r) {
    bool split = false;
    for (uint32_t f = run_first[r]; f < run_first[r + 1]; ++f) split |= seam_bad[f] != 0;
    if (split) {
      for (uint32_t f = run_first[r]; f < run_first[r + 1]; ++f) runs.push_back({fbase[f], fbase[f + 1] - fbase[f]});
    } else {
      runs.push_back({fbase[run_first[r]], fbase[run_first[r + 1]] - fbase[run_first[r]]});
    }
  }
  GET(Y, Rec<W>, n_in + merge_tile_slack, false);  // + a tile: the resolve pass writes whole tile segments
  GET(S, Rec<W>, n_in, false);
  GET(merr, unsigned long long, 2, false);
  uint64_t n_out = 0;
  {
    CK(cudaMemsetAsync(merr, 0xFF, 8, st));
    CK(cudaMemsetAsync(merr + 1, 0, 8, st));
    int rc = merge_runs<W>(st, scratch, X, segview, Y, S, runs, ra, merr, merr + 1);
    if (rc) return rc;
    unsigned long long hm[2];
    CK(cudaMemcpyAsync(hm, merr, 16, cudaMemcpyDeviceToHost, st));
    rc = sync(st);
    if (rc) return rc;
    if (hm[0] != ~0ull)
      return fail(LUDA_ORDERING, "input run not strictly ascending (decoded record " + std::to_string(hm[0]) + ")");
    n_out = hm[1];
  }
  if (ev) CK(cudaEventRecord(ev[3], st));
  // survivors have distinct user keys → LCP < L → unshared >= 9 → entry >= 12 B
  // fixed K: survivors have distinct user keys → LCP < L → unshared >= 9 → entry >= 12 B; var: >= 4 B
  EmitParams ep{K, jd->block_size, jd->restart_interval, jd->bits_per_key, jd->sst_size_target, var ? 4u : 12u, 0,
                var};
  return plan_and_emit<W>(st, scratch, S, n_out, jd->arena, ep, res, ev ? ev + 4 : nullptr);
}

template <int W>
__global__ void records_from_arrays_kernel(const uint8_t* keys, uint32_t L, const uint64_t* trailers,
                                           const uint64_t* voff, const uint32_t* vlen, uint64_t n, Rec<W>* out,
                                           unsigned long long* bad) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  Rec<W> r;
#pragma unroll
  for (int j = 0; j < W; ++j) {
    uint64_t v = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const uint32_t idx = 8 * j + b;
      v = (v << 8) | (idx < L ? keys[i * L + idx] : 0u);
    }
    r.k[j] = v;
  }
  r.t = ~trailers[i];
  if (vlen[i] > kMaxValueLen || voff[i] > kMaxValueOff) atomicMin(bad, 0ull);
  r.h = handle_pack(voff[i], vlen[i]);
  out[i] = r;
}

// Var records (luda_rec.cuh) from flat arrays of keys of any length <= 8W-1:
// key i = keys[koff[i] .. + klen[i]], zero padded, its length in byte 8W-1.
template <int W>
__global__ void records_from_var_arrays_kernel(const uint8_t* keys, const uint64_t* koff, const uint32_t* klen,
                                               const uint64_t* trailers, const uint64_t* voff, const uint32_t* vlen,
                                               uint64_t n, Rec<W>* out, unsigned long long* bad) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint8_t* k = keys + koff[i];
  const uint32_t L = klen[i];
  Rec<W> r;
  for (int j = 0; j < W; ++j) {
    uint64_t v = 0;
    for (int b = 0; b < 8; ++b) {
      const uint32_t idx = 8 * j + b;
      v = (v << 8) | (idx < L ? k[idx] : 0u);
    }
    r.k[j] = v;
  }
  r.k[W - 1] |= L;  // byte 8W-1: always padding (L <= 8W-1)
  r.t = ~trailers[i];
  if (vlen[i] > kMaxValueLen || voff[i] > kMaxValueOff) atomicMin(bad, 0ull);
  r.h = handle_pack(voff[i], vlen[i]);
  out[i] = r;
}

template <int W>
__global__ void check_sorted_kernel(const Rec<W>* r, uint64_t n, unsigned long long* bad) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x + 1;
  if (i < n && rec_cmp(r[i - 1], r[i]) >= 0) atomicMin(bad, (unsigned long long)i);
}

template <int W>
int build_var_w(cudaStream_t st, Scratch& scratch, const uint8_t* keys, const uint64_t* koff, const uint32_t* klen,
                const uint64_t* tr, const uint8_t* values, const uint64_t* voff, const uint32_t* vlen, uint64_t n,
                const EmitParams& ep, luda_job_result* res) {
  GET(R, Rec<W>, n, false);
  GET(bad, unsigned long long, 1, false);
  CK(cudaMemsetAsync(bad, 0xFF, 8, st));
  const unsigned g = (unsigned)((n + 255) / 256);
  records_from_var_arrays_kernel<W><<<g, 256, 0, st>>>(keys, koff, klen, tr, voff, vlen, n, R, bad);
  ++g_launches;
  check_sorted_kernel<W><<<g, 256, 0, st>>>(R, n, bad);
  ++g_launches;
  unsigned long long hb = 0;
  CK(cudaMemcpyAsync(&hb, bad, 8, cudaMemcpyDeviceToHost, st));
  int rc = sync(st);
  if (rc) return rc;
  if (hb == 0) return fail(LUDA_UNSUPPORTED, "value too large for the b200 record handle");
  if (hb != ~0ull) return fail(LUDA_ORDERING, "keys not strictly ascending");
  res->n_in = n;
  return plan_and_emit<W>(st, scratch, R, n, values, ep, res, nullptr);
}

template <int W>
int build_w(cudaStream_t st, Scratch& scratch, const uint8_t* keys, uint32_t L, const uint64_t* tr,
            const uint8_t* values, const uint64_t* voff, const uint32_t* vlen, uint64_t n, const EmitParams& ep,
            luda_job_result* res) {
  GET(R, Rec<W>, n, false);
  GET(bad, unsigned long long, 1, false);
  CK(cudaMemsetAsync(bad, 0xFF, 8, st));
  const unsigned g = (unsigned)((n + 255) / 256);
  records_from_arrays_kernel<W><<<g, 256, 0, st>>>(keys, L, tr, voff, vlen, n, R, bad);
  ++g_launches;
  check_sorted_kernel<W><<<g, 256, 0, st>>>(R, n, bad);
  ++g_launches;
  unsigned long long hb = 0;
  CK(cudaMemcpyAsync(&hb, bad, 8, cudaMemcpyDeviceToHost, st));
  int rc = sync(st);
  if (rc) return rc;
  if (hb == 0) return fail(LUDA_UNSUPPORTED, "value too large for the b200 record handle");
  if (hb != ~0ull) return fail(LUDA_ORDERING, "keys not strictly ascending");
  res->n_in = n;
  return plan_and_emit<W>(st, scratch, R, n, values, ep, res, nullptr);
}

}  // namespace

extern "C" {

int luda_abi_version(void) { return 2; }

int luda_set_option(int option, int64_t value) {
  switch (option) {
    case LUDA_OPT_PLANNER_TILE:
      if (value < 32 || value > (1 << 20)) return fail(LUDA_DEVICE, "planner tile must be in [32, 2^20]");
      g_planner_tile = (uint32_t)value;
      return LUDA_OK;
    case LUDA_OPT_DEC_CTAS:
      if (value < 0 || value > (1 << 16)) return fail(LUDA_DEVICE, "decode CTAs must be in [0, 2^16]");
      g_dec_ctas = (uint32_t)value;
      return LUDA_OK;
    case LUDA_OPT_DEC_SEGS:
      if (value < 0 || value > (1 << 24)) return fail(LUDA_DEVICE, "decode chunks must be in [0, 2^24]");
      g_dec_segs = (uint32_t)value;
      return LUDA_OK;
    default:
      return fail(LUDA_DEVICE, "unknown option");
  }
}

const char* luda_last_error(void) { return g_err.c_str(); }
int64_t luda_last_error_offset(void) { return g_err_off; }

int luda_init(int device_ordinal) {
  CK(cudaSetDevice(device_ordinal));
  if (g_device == device_ordinal) return LUDA_OK;
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device_ordinal));
  if (prop.major != 10) return fail(LUDA_DEVICE, std::string("not an sm_100 device: ") + prop.name);
  g_num_sms = prop.multiProcessorCount;
  if (upload_crc_tables()) return fail(LUDA_DEVICE, "CRC table upload failed");
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device_ordinal) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  g_device = device_ordinal;
  return LUDA_OK;
}

int luda_shutdown(void) {
  if (g_device >= 0) cudaDeviceSynchronize();
  {
    std::lock_guard<std::mutex> lock(g_job_mu);
    g_ws.release_all();
  }
  g_device = -1;
  return LUDA_OK;
}

int luda_region_alloc(uint64_t nbytes, void** dev_ptr) {
  // regions start zero-filled like the reference's shared-memory regions
  CK(cudaMalloc(dev_ptr, std::max<uint64_t>(nbytes, 1) + 512));
  // (cudaMemset may return before the fill lands, and the staging streams are
  // non-blocking: finish it before any stream can copy into the region)
  CK(cudaMemsetAsync(*dev_ptr, 0, std::max<uint64_t>(nbytes, 1) + 512, 0));
  CK(cudaStreamSynchronize(0));
  return LUDA_OK;
}
int luda_region_free(void* p) {
  CK(cudaFree(p));
  return LUDA_OK;
}
int luda_host_alloc(uint64_t nbytes, void** p) {
  CK(cudaHostAlloc(p, std::max<uint64_t>(nbytes, 1), cudaHostAllocDefault));
  return LUDA_OK;
}
int luda_host_free(void* p) {
  CK(cudaFreeHost(p));
  return LUDA_OK;
}
int luda_stream_create(void** s) {
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  *s = st;
  return LUDA_OK;
}
int luda_stream_destroy(void* s) {
  CK(cudaStreamDestroy((cudaStream_t)s));
  return LUDA_OK;
}
int luda_stream_sync(void* s) {
  CK(cudaStreamSynchronize((cudaStream_t)s));
  return LUDA_OK;
}
int luda_stage_in_async(void* dst, const void* src, uint64_t n, void* s) {
  if (n) CK(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, (cudaStream_t)s));
  return LUDA_OK;
}
int luda_stage_out_async(void* dst, const void* src, uint64_t n, void* s) {
  if (n) CK(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, (cudaStream_t)s));
  return LUDA_OK;
}
int luda_memcpy_d2d_async(void* dst, const void* src, uint64_t n, void* s) {
  if (n) CK(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToDevice, (cudaStream_t)s));
  return LUDA_OK;
}
int luda_event_create(void** e) {
  cudaEvent_t ev;
  CK(cudaEventCreate(&ev));
  *e = ev;
  return LUDA_OK;
}
int luda_event_record(void* e, void* s) {
  CK(cudaEventRecord((cudaEvent_t)e, (cudaStream_t)s));
  return LUDA_OK;
}
int luda_event_query(void* e) {
  cudaError_t r = cudaEventQuery((cudaEvent_t)e);
  if (r == cudaSuccess) return 1;
  if (r == cudaErrorNotReady) return 0;
  fail(LUDA_DEVICE, cudaGetErrorString(r));
  return -1;
}
int luda_event_wait(void* e) {
  CK(cudaEventSynchronize((cudaEvent_t)e));
  return LUDA_OK;
}
int luda_event_elapsed_ms(void* a, void* b, float* ms) {
  CK(cudaEventElapsedTime(ms, (cudaEvent_t)a, (cudaEvent_t)b));
  return LUDA_OK;
}
int luda_event_destroy(void* e) {
  CK(cudaEventDestroy((cudaEvent_t)e));
  return LUDA_OK;
}
int luda_stream_wait_event(void* s, void* e) {
  CK(cudaStreamWaitEvent((cudaStream_t)s, (cudaEvent_t)e, 0));
  return LUDA_OK;
}

int luda_crc32_batch(const void* data, const uint64_t* off, const uint32_t* len, uint32_t n, uint32_t* out,
                     void* stream) {
  if (n == 0) return LUDA_OK;
  // (range, pass) items: prefix of per-range pass counts, then warps over items
  // (stream-ordered scratch: concurrent callers on other streams never share it)
  uint32_t* s_pstart = nullptr;
  CK(cudaMallocAsync(reinterpret_cast<void**>(&s_pstart), ((uint64_t)n + 1) * sizeof(uint32_t),
                     (cudaStream_t)stream));
  crc_plan_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(len, n, s_pstart, out);
  const size_t sm = sizeof(CrcSmem) + kCrcFlatWarps * (kGroup + 192);
  CK(cudaFuncSetAttribute(crc_flat_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  crc_flat_kernel<<<g_num_sms, kCrcFlatWarps * 32, sm, (cudaStream_t)stream>>>((const uint8_t*)data, off, len, n,
                                                                              s_pstart, out);
  g_launches += 2;
  CK(cudaGetLastError());
  CK(cudaFreeAsync(s_pstart, (cudaStream_t)stream));
  return LUDA_OK;
}

int luda_crc32(const void* data, uint64_t n, uint32_t* out_crc, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  uint32_t* d = nullptr;
  CK(cudaMallocAsync(&d, 4, st));
  CK(cudaMemsetAsync(d, 0xFF, 4, st));
  if (n < 4) {
    uint64_t* o = nullptr;
    uint32_t* l = nullptr;
    CK(cudaMallocAsync(&o, 8, st));
    CK(cudaMallocAsync(&l, 4, st));
    const uint64_t z = 0;
    const uint32_t nn = (uint32_t)n;
    CK(cudaMemcpyAsync(o, &z, 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(l, &nn, 4, cudaMemcpyHostToDevice, st));
    int rc = luda_crc32_batch(data, o, l, 1, d, stream);
    if (rc) return rc;
    CK(cudaMemcpyAsync(out_crc, d, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    cudaFreeAsync(o, st);
    cudaFreeAsync(l, st);
  } else {
    const size_t sm = sizeof(CrcSmem) + kCrcWarps * (kGroup + 192);
    CK(cudaFuncSetAttribute(crc_big_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    const uint64_t np = (n + kGroup - 1) / kGroup;
    const unsigned grid = (unsigned)std::min<uint64_t>((np + kCrcWarps - 1) / kCrcWarps, 4ull * g_num_sms);
    crc_big_kernel<<<grid, kCrcWarps * 32, sm, st>>>((const uint8_t*)data, n, d);
    ++g_launches;
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out_crc, d, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  cudaFreeAsync(d, st);
  return LUDA_OK;
}

int luda_job_release(luda_job_result* r) {
  if (!r) return LUDA_OK;
  JobPriv* priv = reinterpret_cast<JobPriv*>(r->priv);
  if (r->out) {
    if (priv && priv->st) cudaStreamSynchronize(priv->st);
    if (!g_out.put(r->out)) cudaFree(r->out);
  }
  delete priv;
  memset(r, 0, sizeof(*r));
  return LUDA_OK;
}

int luda_build_from_sorted(const uint8_t* keys, uint32_t L, const uint64_t* trailers, const uint8_t* values,
                           const uint64_t* voff, const uint32_t* vlen, uint64_t n, uint32_t block_size,
                           uint32_t restart_interval, uint32_t bits_per_key, uint64_t sst_size_target,
                           luda_job_result* res, void* stream) {
  return luda_build_files_from_sorted(keys, L, trailers, values, voff, vlen, n, block_size, restart_interval,
                                      bits_per_key, sst_size_target, 0, res, stream);
}

int luda_build_files_from_sorted(const uint8_t* keys, uint32_t L, const uint64_t* trailers, const uint8_t* values,
                                 const uint64_t* voff, const uint32_t* vlen, uint64_t n, uint32_t block_size,
                                 uint32_t restart_interval, uint32_t bits_per_key, uint64_t sst_size_target,
                                 uint64_t entries_per_file, luda_job_result* res, void* stream) {
  if (g_device < 0) return fail(LUDA_DEVICE, "luda_init not called");
  std::lock_guard<std::mutex> lock(g_job_mu);
  memset(res, 0, sizeof(*res));
  if (L > 32) return fail(LUDA_UNSUPPORTED, "user keys longer than 32 bytes");
  if (restart_interval < 1) return fail(LUDA_DEVICE, "restart_interval must be >= 1");
  cudaStream_t st = (cudaStream_t)stream;
  Scratch scratch(st);
  // duplicates of a user key may share up to K-1 bytes → entry >= 4 B
  EmitParams ep{L + 8, block_size, restart_interval, bits_per_key, sst_size_target, 4, entries_per_file};
  const uint32_t W = std::max<uint32_t>(1, (L + 7) / 8);
  int rc;
  switch (W) {
    case 1: rc = build_w<1>(st, scratch, keys, L, trailers, values, voff, vlen, n, ep, res); break;
    case 2: rc = build_w<2>(st, scratch, keys, L, trailers, values, voff, vlen, n, ep, res); break;
    case 3: rc = build_w<3>(st, scratch, keys, L, trailers, values, voff, vlen, n, ep, res); break;
    default: rc = build_w<4>(st, scratch, keys, L, trailers, values, voff, vlen, n, ep, res); break;
  }
  if (rc) luda_job_release(res);
  return rc;
}

int luda_build_from_sorted_var(const uint8_t* keys, const uint64_t* key_off, const uint32_t* key_len,
                               uint32_t max_key_len, const uint64_t* trailers, const uint8_t* values,
                               const uint64_t* voff, const uint32_t* vlen, uint64_t n, uint32_t block_size,
                               uint32_t restart_interval, uint32_t bits_per_key, uint64_t sst_size_target,
                               luda_job_result* res, void* stream) {
  if (g_device < 0) return fail(LUDA_DEVICE, "luda_init not called");
  std::lock_guard<std::mutex> lock(g_job_mu);
  memset(res, 0, sizeof(*res));
  if (max_key_len > kVarMaxLenLong) return fail(LUDA_UNSUPPORTED, "user keys longer than 255 bytes");
  if (restart_interval < 1) return fail(LUDA_DEVICE, "restart_interval must be >= 1");
  cudaStream_t st = (cudaStream_t)stream;
  Scratch scratch(st);
  EmitParams ep{8 * kVarW + 8, block_size, restart_interval, bits_per_key, sst_size_target, 4, 0, true};
  int rc;
  if (max_key_len <= kVarMaxLen) {
    rc = build_var_w<kVarW>(st, scratch, keys, key_off, key_len, trailers, values, voff, vlen, n, ep, res);
  } else {
    ep.K = 8 * kVarWLong + 8;
    rc = build_var_w<kVarWLong>(st, scratch, keys, key_off, key_len, trailers, values, voff, vlen, n, ep, res);
  }
  if (rc) luda_job_release(res);
  return rc;
}

int luda_dispatch(int kind, const int64_t* items, uint32_t n_items, void* const* region_ptr,
                  const uint64_t* region_cap, uint32_t n_regions, int64_t* results, int64_t* fail_item,
                  void* stream) {
  static const uint32_t kCols[4] = {9, 6, 10, 7};
  static const uint32_t kRcols[4] = {4, 1, 2, 1};
  *fail_item = -1;
  if (g_device < 0) return fail(LUDA_DEVICE, "luda_init not called");
  if (kind < 0 || kind > 3) return fail(LUDA_DEVICE, "unknown kernel kind");
  if (n_items == 0) return LUDA_OK;
  std::lock_guard<std::mutex> lock(g_job_mu);
  cudaStream_t st = (cudaStream_t)stream;
  Scratch scratch(st);
  const uint32_t cols = kCols[kind], rcols = kRcols[kind];
  GET(d_items, int64_t, (uint64_t)n_items * cols, false);
  GET(d_ptr, uint8_t*, std::max<uint32_t>(n_regions, 1), false);
  GET(d_cap, uint64_t, std::max<uint32_t>(n_regions, 1), false);
  GET(d_res, int64_t, (uint64_t)n_items * rcols, true);
  GET(d_status, uint32_t, n_items, false);
  GET(d_msg, uint32_t, n_items, false);
  GET(d_off, int64_t, n_items, false);
  CK(cudaMemcpyAsync(d_items, items, 8ull * n_items * cols, cudaMemcpyHostToDevice, st));
  if (n_regions) {
    CK(cudaMemcpyAsync(d_ptr, region_ptr, sizeof(void*) * n_regions, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_cap, region_cap, 8ull * n_regions, cudaMemcpyHostToDevice, st));
  }
  DispatchArgs da{kind, d_items, n_items, cols, d_ptr, d_cap, n_regions, d_res, rcols, d_status, d_msg, d_off};
  const size_t sm = sizeof(CrcSmem) + (size_t)kDispWarps * (kDispStage + 256);
  CK(cudaFuncSetAttribute(dispatch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  const unsigned grid = (unsigned)std::min<uint64_t>((n_items + kDispWarps - 1) / kDispWarps, 2ull * g_num_sms);
  dispatch_kernel<<<grid, kDispWarps * 32, sm, st>>>(da);
  ++g_launches;
  CK(cudaGetLastError());
  std::vector<uint32_t> hst(n_items), hmsg(n_items);
  std::vector<int64_t> hoff(n_items);
  CK(cudaMemcpyAsync(results, d_res, 8ull * n_items * rcols, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(hst.data(), d_status, 4ull * n_items, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(hmsg.data(), d_msg, 4ull * n_items, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(hoff.data(), d_off, 8ull * n_items, cudaMemcpyDeviceToHost, st));
  int rc = sync(st);
  if (rc) return rc;
  static const char* kMsg[] = {"ok", "block too short", "data block checksum mismatch", "bad restart array",
                               "truncated varint", "varint too long", "truncated block entry",
                               "trailing garbage in block entries", "BufferError: pair slot overflow",
                               "BufferError: tuple slot overflow", "error: ushort format requires 0 <= number <= 65535",
                               "region range outside the dispatch's regions",
                               "ValueError: restart_interval must be >= 1", "BufferError: encode slot overflow",
                               "BufferError: filter slot overflow", "ValueError: bits_per_key must be >= 1",
                               "error: tuple runs past its region"};
  for (uint32_t i = 0; i < n_items; ++i) {
    if (hst[i] == D_OK) continue;
    *fail_item = i;  // first failing item in dispatch order (device.py:445-447, 589-591)
    const char* m = hmsg[i] < sizeof(kMsg) / sizeof(kMsg[0]) ? kMsg[hmsg[i]] : "error";
    if (hst[i] == D_CORRUPT) return fail(LUDA_CORRUPT, m, hoff[i]);
    return fail(LUDA_DEVICE, m);
  }
  return LUDA_OK;
}

int luda_compact(const luda_job_desc* jd, luda_job_result* res, void* stream) {
  if (g_device < 0) return fail(LUDA_DEVICE, "luda_init not called");
  std::lock_guard<std::mutex> lock(g_job_mu);
  memset(res, 0, sizeof(*res));
  cudaStream_t st = (cudaStream_t)stream;
  {
    const int prc = g_pin.init();
    if (prc) return prc;
  }
  KTimer kt;
  g_kt = &kt;
  g_launches = 0;
  struct KtGuard { ~KtGuard() { g_kt = nullptr; } } ktg;
  Scratch scratch(st);
  cudaEvent_t ev[8];
  for (auto& e : ev) CK(cudaEventCreate(&e));
  struct EvGuard {
    cudaEvent_t* e;
    ~EvGuard() { for (int i = 0; i < 8; ++i) cudaEventDestroy(e[i]); }
  } evg{ev};
  CK(cudaEventRecord(ev[0], st));
  const uint32_t nf = jd->n_files;
  if (nf == 0) return LUDA_OK;
  if (jd->restart_interval < 1) return fail(LUDA_DEVICE, "restart_interval must be >= 1");
  GET(d_faddr, uint64_t, nf, false);
  GET(d_fsize, uint64_t, nf, false);
  CK(cudaMemcpyAsync(d_faddr, jd->file_off, 8ull * nf, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_fsize, jd->file_len, 8ull * nf, cudaMemcpyHostToDevice, st));
  GET(info, FileInfo, nf, false);
  GET(caddr, uint64_t, 2ull * nf, false);
  GET(clen, uint32_t, 2ull * nf, false);
  GET(cstored, uint32_t, 2ull * nf, false);
  GET(ccrc, uint32_t, 2ull * nf, false);
  ParseArgs pa{jd->arena, d_faddr, d_fsize, nf, info, caddr, clen, cstored};
  parse_files_a<<<(nf * 32 + kParseAThreads - 1) / kParseAThreads, kParseAThreads, 0, st>>>(pa);
  ++g_launches;
  CK(cudaGetLastError());
  // Filter / index CRCs on the side stream, concurrently with the block table
  // and the decode: nothing but error reporting needs them, and the decode
  // sync (or the end of the job) checks them before any later error.
  DeferredCrc& dc = g_dcrc;
  int rc = dc.prepare(nf);
  if (rc) return rc;
  CK(cudaEventRecord(dc.parsed, st));
  CK(cudaStreamWaitEvent(dc.side, dc.parsed, 0));
  rc = luda_crc32_batch(jd->arena, caddr, clen, 2 * nf, ccrc, dc.side);
  if (rc) return rc;
  CK(cudaMemcpyAsync(dc.h, ccrc, 8ull * nf, cudaMemcpyDeviceToHost, dc.side));
  CK(cudaMemcpyAsync(dc.h + 2 * nf, cstored, 8ull * nf, cudaMemcpyDeviceToHost, dc.side));
  CK(cudaEventRecord(dc.done, dc.side));
#ifdef LUDA_SERIAL_SIDE_CRC  // experiment: the main stream waits for the side-stream CRCs
  CK(cudaStreamWaitEvent(st, dc.done, 0));
#endif
  std::vector<FileInfo>& hinfo = dc.info;
  CK(cudaMemcpyAsync(hinfo.data(), info, sizeof(FileInfo) * nf, cudaMemcpyDeviceToHost, st));
  rc = sync(st);
  if (rc) return rc;
  bool clean = true;
  for (uint32_t f = 0; f < nf; ++f) clean &= !hinfo[f].code && !hinfo[f].kbad && !hinfo[f].icode;
  if (!clean) {  // a structural error: its place in the reference order depends on the CRCs
    CK(cudaEventSynchronize(dc.done));
    for (uint32_t f = 0; f < nf; ++f) {
      rc = check_parsed_file(hinfo[f], dc.h + 2 * f, dc.h + 2 * nf + 2 * f);
      if (rc) return rc;
    }
  }
  dc.pending = true;
  // Reference order per file (Table.__init__), files in job order.
  uint32_t K = 0xFFFFFFFEu;
  bool mixed = false;
  std::vector<uint32_t> fbb(nf + 1, 0);
  for (uint32_t f = 0; f < nf; ++f) {
    const FileInfo& fi = hinfo[f];
    fbb[f + 1] = fbb[f] + fi.nblocks;
    if (fi.nblocks) {
      if (fi.klen == 0xFFFFFFFFu) mixed = true;
      else if (K == 0xFFFFFFFEu) K = fi.klen;
      else if (K != fi.klen) mixed = true;
    }
  }
  const uint32_t nblk = fbb[nf];
  if (nblk == 0) return deferred_crc_check();  // no data blocks: empty output
  if (nblk >= kDecEnd) return fail(LUDA_UNSUPPORTED, "more than 2^31 - 1 data blocks in one job");
  // Fixed-K records when every index key has one length <= 32 bytes; else
  // (mixed lengths, longer keys) the generic-length "var" records.
  bool var = mixed || K < 8 || K - 8 > 32;
  const uint32_t L = var ? 8 * kVarW : K - 8;
  GET(d_fbb, uint32_t, nf + 1, false);
  CK(cudaMemcpyAsync(d_fbb, fbb.data(), 4ull * (nf + 1), cudaMemcpyHostToDevice, st));
  BlockTable bt{};
  {
    GET(a_, uint64_t, nblk, false);
    GET(l_, uint32_t, nblk, false);
    GET(o_, uint32_t, nblk, false);
    GET(f_, uint32_t, nblk, false);
    bt = BlockTable{a_, l_, o_, f_};
  }
  uint32_t max_nb = 0;
  for (uint32_t f = 0; f < nf; ++f) max_nb = std::max(max_nb, hinfo[f].nblocks);
  parse_files_c<<<dim3(nf, std::max(1u, (max_nb + kParseChunk - 1) / kParseChunk)), kParseThreads, 0, st>>>(
      pa, d_fbb, bt);
  ++g_launches;
  CK(cudaGetLastError());
  const uint32_t W = std::max<uint32_t>(1, (L + 7) / 8);
  CK(cudaEventRecord(ev[1], st));
  cudaEvent_t* pev = ev;
  if (!var) {
    switch (W) {
      case 1: rc = compact_w<1>(st, scratch, jd, res, K, nblk, bt, d_fbb, pev, false); break;
      case 2: rc = compact_w<2>(st, scratch, jd, res, K, nblk, bt, d_fbb, pev, false); break;
      case 3: rc = compact_w<3>(st, scratch, jd, res, K, nblk, bt, d_fbb, pev, false); break;
      default: rc = compact_w<4>(st, scratch, jd, res, K, nblk, bt, d_fbb, pev, false); break;
    }
    if (rc == kRetryVar) {  // a data block holds another key length than the index keys
      luda_job_release(res);
      memset(res, 0, sizeof(*res));
      var = true;
    }
  }
  if (var) {
    rc = compact_w<kVarW>(st, scratch, jd, res, 8 * kVarW + 8, nblk, bt, d_fbb, pev, true);
    if (rc == kRetryLong) {
      luda_job_release(res);
      memset(res, 0, sizeof(*res));
      rc = compact_w<kVarWLong>(st, scratch, jd, res, 8 * kVarWLong + 8, nblk, bt, d_fbb, pev, true);
    }
  }
  {
    const int crc_rc = deferred_crc_check();  // a filter / index CRC error outranks every later error
    if (crc_rc) rc = crc_rc;
  }
  if (rc) {
    luda_job_release(res);
    return rc;
  }
  CK(cudaEventRecord(ev[7], st));
  CK(cudaEventSynchronize(ev[7]));
  // t_ms: [0] parse, [1] decode, [2] merge, [3] plan, [4] emit, [7] total
  if (res->n_out) {
    for (int i = 0; i < 5; ++i) res->t_ms[i] = ev_ms(ev[i], ev[i + 1]);
  }
  res->t_ms[7] = ev_ms(ev[0], ev[7]);
  kt.read(res->k_ms);
  res->launches = g_launches;
  return LUDA_OK;
}

#ifdef ENC_TIMING
// instrumentation build only: accumulated encode builder/CRC warp section cycles
int luda_dbg_enc_timing(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, luda::g_enc_t, 16 * sizeof(unsigned long long));
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(luda::g_enc_t, z, sizeof(z));
  }
  return 0;
}
#endif
}  // extern "C"

#include "luda_read_abi.inc"
#include "luda_io_abi.inc"
#include "luda_nccl_abi.inc"
