/*
 * luda_b200.h — C ABI of the B200-native LUDA compaction path.
 *
 * The reference (pure Python, /root/reference/pkg/src/luda) exposes its
 * compaction path through an offload-device plugin protocol
 * (device.py:253-627: make_device → alloc/free/stage_in/stage_out/dispatch/
 * stats/close) and a SPEC-level entry point run_compaction(job, device)
 * (SPEC.md:323-331). This header is the native seam those calls bind to.
 * Every entry point returns an int status (enum luda_status); the message of
 * the last failure on the calling thread is available from luda_last_error().
 *
 * No torch types cross this boundary: device buffers are plain pointers,
 * streams/events are opaque handles (cudaStream_t / cudaEvent_t).
 */
#ifndef LUDA_B200_H
#define LUDA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; mapped to the reference exception tree (errors.py:4-46) by
 * paper_2004_03054_b200/errors.py:from_status. */
enum luda_status {
  LUDA_OK = 0,
  LUDA_CORRUPT = 1,     /* CorruptionError(offset) — checksum mismatch        */
  LUDA_FORMAT = 2,      /* FormatError — malformed footer/filter/index/block  */
  LUDA_CAPACITY = 3,    /* CapacityError                                       */
  LUDA_ORDERING = 4,    /* OrderingError — input run not strictly ascending    */
  LUDA_DEVICE = 5,      /* DeviceError — CUDA failure / bad argument           */
  LUDA_UNSUPPORTED = 6  /* valid input outside the fast-path envelope          */
};

/* Kernel kinds of the reference KernelSpec (kernels.py:171-178). */
enum luda_kind { LUDA_KIND_UNPACK = 0, LUDA_KIND_SHARED_KEY = 1, LUDA_KIND_ENCODE = 2,
                 LUDA_KIND_FILTER = 3 };

/* ---- context ----------------------------------------------------------- */
/* Replaces make_device(DeviceConfig) bring-up (device.py:622-627). */
int luda_init(int device_ordinal);
int luda_shutdown(void);
const char* luda_last_error(void);
int64_t luda_last_error_offset(void); /* block offset of the last LUDA_CORRUPT, or -1 */
int luda_abi_version(void);

/* Process-wide options. LUDA_OPT_PLANNER_TILE: tile (items) of the greedy-chain
 * block/SST planner, default 8192 — smaller (floor 256) when an input would
 * span fewer than 2 tiles per SM, never below the longest jump. Outputs do not depend on it;
 * the parity tests set it to 32 so that small jobs exercise the planner's
 * multi-tile / multi-group composition. */
/* LUDA_OPT_DEC_CTAS: decode CTAs (0 = one per SM) and LUDA_OPT_DEC_SEGS: block
 * chunks handed out to the decode pairs (0 = automatic). Outputs do not depend
 * on them; the parity tests use 1 CTA and one block per chunk so that small
 * jobs exercise the pairs' chunk switching. */
enum luda_option { LUDA_OPT_PLANNER_TILE = 1, LUDA_OPT_DEC_CTAS = 2, LUDA_OPT_DEC_SEGS = 3 };
int luda_set_option(int option, int64_t value);

/* ---- regions: device arena + pinned host staging ------------------------ */
/* Replaces _DeviceBase.alloc/free (device.py:266-294). */
int luda_region_alloc(uint64_t nbytes, void** dev_ptr);
int luda_region_free(void* dev_ptr);
int luda_host_alloc(uint64_t nbytes, void** host_ptr);
int luda_host_free(void* host_ptr);

/* ---- streams, transfers, events ----------------------------------------- */
/* Replaces stage_in/stage_out on the named FIFO streams in_lower/in_upper/out
 * (device.py:298-333, 511-547): one CUDA stream per named stream. */
int luda_stream_create(void** stream);
int luda_stream_destroy(void* stream);
int luda_stream_sync(void* stream);
int luda_stage_in_async(void* dst_dev, const void* src_host, uint64_t nbytes, void* stream);
int luda_stage_out_async(void* dst_host, const void* src_dev, uint64_t nbytes, void* stream);
int luda_memcpy_d2d_async(void* dst_dev, const void* src_dev, uint64_t nbytes, void* stream);
int luda_event_create(void** event);
int luda_event_record(void* event, void* stream);
int luda_event_query(void* event); /* 1 = complete, 0 = pending, <0 = error */
int luda_event_wait(void* event);
int luda_event_elapsed_ms(void* start, void* stop, float* ms);
int luda_event_destroy(void* event);
int luda_stream_wait_event(void* stream, void* event);

/* ---- primitives --------------------------------------------------------- */
/* CRC-32/IEEE of a device buffer (checksum.py:12-13); synchronous. */
int luda_crc32(const void* dev_data, uint64_t nbytes, uint32_t* out_crc, void* stream);
/* Batched CRC: crc of [data+off[i], +len[i]) for i < n, written to dev out. */
int luda_crc32_batch(const void* dev_data, const uint64_t* dev_off, const uint32_t* dev_len,
                     uint32_t n, uint32_t* dev_out, void* stream);

/* ---- per-kind dispatch (reference KernelSpec semantics) ----------------- */
/* Replaces SerialDevice/HostParallelDevice.dispatch (device.py:435-456,
 * 566-607) for the four kinds of kernels.py:72-168.
 *   items      : host array, n_items rows of the kind's argument tuple as
 *                int64 (unpack 9, shared_key 6, encode 10, filter 7 columns)
 *   region_ptr : host array mapping region id → device pointer
 *   region_cap : host array mapping region id → capacity (bytes)
 *   results    : host out, n_items rows of the kind's result tuple as int64
 *                (unpack 4, shared_key 1, encode 2, filter 1 columns)
 *   fail_item  : index of the first failing item in dispatch order, or -1;
 *                its tag (status) is the return value, its message in
 *                luda_last_error() and corrupt offset in luda_last_error_offset().
 * Synchronous on `stream`. */
int luda_dispatch(int kind, const int64_t* items, uint32_t n_items,
                  void* const* region_ptr, const uint64_t* region_cap, uint32_t n_regions,
                  int64_t* results, int64_t* fail_item, void* stream);

/* ---- fused compaction job (run_compaction) ------------- */
typedef struct {
  const uint8_t* arena;         /* device: staged input files                     */
  uint64_t arena_bytes;
  uint32_t n_files;
  const uint64_t* file_off;     /* host[n_files]: file i at arena + file_off[i]    */
  const uint64_t* file_len;     /* host[n_files]                                   */
  const int64_t* file_offset_base; /* host[n_files] or NULL: added to error offsets */
  uint32_t n_runs;              /* sorted runs, in merge-priority order            */
  const uint32_t* run_first_file; /* host[n_runs+1]                               */
  uint32_t block_size;          /* StoreConfig.block_size (config.py:48)           */
  uint32_t restart_interval;    /* StoreConfig.restart_interval (config.py:49)     */
  uint32_t bits_per_key;        /* StoreConfig.bits_per_key (config.py:50)         */
  uint64_t sst_size_target;     /* StoreConfig.sst_size_target (config.py:47)      */
  /* Version.covers_below(target_level) as closed user-key intervals
   * (version.py:122-128): n_deeper pairs, keys packed back to back. */
  uint32_t n_deeper;
  const uint8_t* deeper_keys;   /* host: lo0 hi0 lo1 hi1 ...                       */
  const uint32_t* deeper_lens;  /* host[2*n_deeper]                                */
  /* Optional key-range restriction [range_lo, range_hi) on user keys
   * (subcompactions); NULL = unbounded on that side. */
  const uint8_t* range_lo; uint32_t range_lo_len;
  const uint8_t* range_hi; uint32_t range_hi_len;
} luda_job_desc;

typedef struct {
  uint8_t* out;                 /* device: output SSTs back to back (lib-owned)   */
  uint64_t out_bytes;
  uint32_t n_sst;
  uint64_t* sst_off;            /* host[n_sst] (lib-owned)                         */
  uint64_t* sst_len;            /* host[n_sst]                                     */
  uint32_t key_len;             /* internal key length K                           */
  uint8_t* sst_keys;            /* host[n_sst*2*K]: smallest ∥ largest per SST     */
  uint64_t n_in, n_out, blocks_in, blocks_out;
  double t_ms[8];               /* phases: parse, decode, merge, plan, emit, -, -, total */
  double k_ms[8];               /* kernels: decode, merge(final), block_jump, encode, meta, -, -, - */
  uint64_t launches;            /* kernels launched by this job                   */
  void* priv;
  uint32_t* sst_key_len;        /* host[n_sst*2]: internal key lengths of sst_keys;
                                   key_len is then the slot size per key           */
} luda_job_result;

int luda_compact(const luda_job_desc* job, luda_job_result* result, void* stream);
int luda_job_release(luda_job_result* result);

/* Build SSTs from already-sorted unique records (used by the bench to
 * synthesise inputs and by the L0-flush path): records are produced by
 * luda_records_from_keys from flat arrays. Outputs like luda_compact. */
int luda_build_from_sorted(const uint8_t* dev_user_keys, uint32_t user_key_len,
                           const uint64_t* dev_trailers, const uint8_t* dev_values,
                           const uint64_t* dev_value_off, const uint32_t* dev_value_len,
                           uint64_t n, uint32_t block_size, uint32_t restart_interval,
                           uint32_t bits_per_key, uint64_t sst_size_target,
                           luda_job_result* result, void* stream);

/* As luda_build_from_sorted for user keys of mixed lengths (any length <=
 * 255 bytes, max_key_len = the longest): key i = dev_user_keys[key_off[i] ..
 * + key_len[i]] (device arrays). The generic-length records of the compaction
 * path; L0 flush of a memtable whose keys differ in length. */
int luda_build_from_sorted_var(const uint8_t* dev_user_keys, const uint64_t* dev_key_off,
                               const uint32_t* dev_key_len, uint32_t max_key_len, const uint64_t* dev_trailers,
                               const uint8_t* dev_values, const uint64_t* dev_value_off,
                               const uint32_t* dev_value_len, uint64_t n, uint32_t block_size,
                               uint32_t restart_interval, uint32_t bits_per_key, uint64_t sst_size_target,
                               luda_job_result* result, void* stream);
/* As luda_build_from_sorted, but cut an output SST every `entries_per_file`
 * entries (the last SST may hold fewer; sst_size_target is then unused):
 * synthesises input levels whose file boundaries are known in advance
 * (bench_c5.py: BASELINE config 5's global job). 0 = size cut. */
int luda_build_files_from_sorted(const uint8_t* dev_user_keys, uint32_t user_key_len,
                                 const uint64_t* dev_trailers, const uint8_t* dev_values,
                                 const uint64_t* dev_value_off, const uint32_t* dev_value_len,
                                 uint64_t n, uint32_t block_size, uint32_t restart_interval,
                                 uint32_t bits_per_key, uint64_t sst_size_target,
                                 uint64_t entries_per_file, luda_job_result* result, void* stream);

/* ---- batched read path ------------------------------- */
/* A set of SSTs resident in device memory (host-staged files, or a job's
 * output buffer, zero-copy). Replaces, per file, Table.__init__
 * (sst.py:284-310: footer, magic, filter and index checks — the first failing
 * file's error is returned) and verifies every data block's CRC once
 * (Table._raw_block, sst.py:322-340); a block's outcome is raised only by a
 * lookup that reads it, as in the reference. */
typedef struct luda_tables luda_tables;
int luda_tables_open(const uint8_t* dev_arena, const uint64_t* file_off, const uint64_t* file_len,
                     uint32_t n_files, luda_tables** out, void* stream);
int luda_tables_close(luda_tables* t);
int luda_tables_info(luda_tables* t, uint32_t* n_tables, uint32_t* n_blocks);
/* Table.filter_rejects / Table.data_block_reads (sst.py:296-297), host[n_files] each. */
int luda_tables_counters(luda_tables* t, uint64_t* filter_rejects, uint64_t* block_reads);
/* The store's probe order for a get: the L0 tables newest
 * first, then per level >= 1 the one file whose [smallest, largest] user-key
 * range holds the key (binary search over ascending ranges); the first table
 * whose Table.get returns an entry answers. */
typedef struct {
  uint32_t n_l0;
  const uint32_t* l0;            /* host[n_l0]: table ids, newest first           */
  uint32_t n_levels;
  const uint32_t* level_first;   /* host[n_levels+1]: into level_tables           */
  const uint32_t* level_tables;  /* host: table ids, ascending ranges per level   */
  const uint8_t* range_keys;     /* host: smallest ∥ largest user key per entry   */
  const uint32_t* range_lens;    /* host[2 * entries]                             */
} luda_probe_plan;
int luda_tables_set_plan(luda_tables* t, const luda_probe_plan* plan, void* stream);
typedef struct {
  uint32_t n;
  const uint32_t* status;     /* host[n]: 0 = None, 1 = (key, value), >1 = error  */
  const uint32_t* table;      /* host[n]: table that answered                     */
  const uint32_t* key_len;    /* host[n]: internal key length of a found entry     */
  const uint32_t* value_len;  /* host[n]                                           */
  const uint64_t* pos;        /* host[n+1]: found entry i = packed[pos[i] ..]: key ∥ value */
  const uint8_t* packed;      /* host                                              */
  uint64_t packed_bytes;
  const int64_t* err_off;     /* host[n]: block offset of a CorruptionError, else -1 */
  int64_t fail_index;         /* first failing lookup (its error is the return value) or -1 */
  double t_ms[4];             /* H2D, lookup + scan, pack, D2H                     */
} luda_get_result;
/* Table.get (sst.py:342-368) for n keys (key i = keys[key_off[i] .. + key_len[i]],
 * host memory; key_off NULL: n keys of key_len[0] bytes back to back): on table
 * table_of_key[i], or in the plan's store order when table_of_key is NULL. Found keys longer than key_cap fail (LUDA_UNSUPPORTED).
 * Result arrays are owned by the table set and valid until its next get.
 * Synchronous on `stream`. */
int luda_tables_get(luda_tables* t, const uint8_t* keys, uint64_t keys_bytes, const uint64_t* key_off,
                    const uint32_t* key_len, uint32_t n, const uint32_t* table_of_key, uint32_t key_cap,
                    luda_get_result* result, void* stream);
/* The lookup kernel alone over device-resident keys (throughput measurement;
 * dev_key_off NULL: fixed-length keys as above); results stay on the device.
 * Asynchronous on `stream`. */
int luda_tables_lookup_dev(luda_tables* t, const uint8_t* dev_keys, const uint64_t* dev_key_off,
                           const uint32_t* dev_key_len, uint32_t n, const uint32_t* dev_table_of_key,
                           uint32_t key_cap, void* stream);
/* ---- storage <-> HBM ---------------- */
/* Read n files (file i's first len[i] bytes) into dev_dst + dst_off[i], or
 * write dev_src + src_off[i] .. + len[i] to file i (created / truncated),
 * without a caller-visible host copy: GPUDirect Storage through cuFile
 * (dlopen'ed; its compatibility mode where nvidia-fs is absent), else a
 * native multi-threaded pread/pwrite ↔ pinned double-buffer ↔ cudaMemcpyAsync
 * pipeline. mode: 0 auto (cuFile if LUDA_GDS=1 and its driver opens within
 * LUDA_CUFILE_OPEN_TIMEOUT_S, default 5 s), 1 cuFile only, 2 bounce only; *used_mode = 1
 * (cuFile) or 2 (bounce). Synchronous. Replaces the host file reads / writes
 * around run_compaction (Table file I/O, sst.py:284-340; build_sst writes). */
int luda_files_read(const char* const* paths, uint32_t n, void* dev_dst, const uint64_t* dst_off,
                    const uint64_t* len, int mode, int* used_mode);
int luda_files_write(const char* const* paths, uint32_t n, const void* dev_src, const uint64_t* src_off,
                     const uint64_t* len, int mode, int* used_mode);
/* 1 when the cuFile driver opened (message in why), else 0. */
int luda_gds_status(char* why, uint32_t cap);
/* ---- multi-GPU: the splitter all-gather -------- */
/* The only collective of the key-range-partitioned compaction: every rank's
 * fixed-size index-key sample array is all-gathered so all ranks pick the same
 * P - 1 splitters. NCCL over NVLink/NVSwitch; libnccl is dlopen'ed. The
 * reference is single-host (multi-device is a SPEC non-goal). */
typedef struct luda_comm luda_comm;
int luda_nccl_unique_id(uint8_t* out_128_bytes);  /* rank 0 creates, the launcher distributes */
int luda_nccl_init_rank(int nranks, int rank, const uint8_t* unique_id, luda_comm** comm); /* one process per GPU */
int luda_nccl_init_all(int ndev, const int* devices, luda_comm** comms);  /* one process, ndev GPUs (comms[ndev]) */
/* recv = the ranks' send buffers (bytes_per_rank each) in rank order; device
 * pointers, asynchronous on `stream`. Several communicators of one process:
 * bracket the calls with luda_nccl_group_start / _end. */
int luda_allgather_splitters(luda_comm* comm, const void* dev_send, void* dev_recv, uint64_t bytes_per_rank,
                             void* stream);
int luda_nccl_group_start(void);
int luda_nccl_group_end(void);
int luda_nccl_destroy(luda_comm* comm);
#ifdef __cplusplus
}
#endif
#endif /* LUDA_B200_H */
