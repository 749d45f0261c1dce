"""``run_compaction(job, device)`` — the SPEC entry point,
implemented as one fused device pipeline.

The reference specifies but does not ship this function; its composition
 is: open every input table (footer, filter CRC, index CRC),
decode every data block, merge the per-file runs on ``keys.sort_key``, keep
the newest entry per user key, drop tombstones that nothing below the target
level covers (SPEC D12, ``Version.covers_below`` version.py:122-128) and
re-build SSTs with ``SstBuilder`` cutting on ``SizeOverflowError``
(sst.py:105-217). Here the host only stages whole input files (two copy
streams, Fig. 5a of the paper), calls ``luda_compact`` (decode → merge →
resolve → plan → encode → filter/index/footer, all on the GPU; the tuples never
round-trip to the host) and copies the finished SST bytes back.
"""

from __future__ import annotations

import ctypes
import os
import time
from dataclasses import dataclass, field

from . import _native
from .config import StoreConfig
from .device import STREAM_IN_LOWER, STREAM_IN_UPPER, STREAM_OUT, B200Device, PinnedBuffer
from .errors import DeviceError
from .version import SstMeta, deeper_ranges, user_key_of

ARENA_ALIGN = 256
ARENA_PAD = 256


@dataclass
class JobStats:
    """SPEC.md:360 job-stats columns (+ device-side detail)."""

    job_id: int = 0
    source_level: int = 0
    input_files: int = 0
    input_bytes: int = 0
    output_files: int = 0
    output_bytes: int = 0
    t_stage_in: float = 0.0
    t_unpack: float = 0.0
    t_sort_host: float = 0.0   # device merge+resolve (no host sort exists here)
    t_pack: float = 0.0
    t_stage_out: float = 0.0
    overlap_ratio: float = 0.0
    n_in: int = 0
    n_out: int = 0
    blocks_in: int = 0
    blocks_out: int = 0
    t_device_ms: dict = field(default_factory=dict)

    CSV_COLUMNS = ("job_id", "source_level", "input_files", "input_bytes", "output_files", "output_bytes",
                   "t_stage_in", "t_unpack", "t_sort_host", "t_pack", "t_stage_out", "overlap_ratio")

    def csv_row(self) -> str:
        return ",".join(str(getattr(self, c)) for c in self.CSV_COLUMNS)


@dataclass
class PreparedJob:
    """Host-side description of a job's inputs (file order = run order)."""

    files: list                 # bytes-like per input file
    run_first_file: list        # [n_runs + 1]
    deeper: list                # [(lo_user, hi_user)]
    block_size: int = 4096
    restart_interval: int = 16
    bits_per_key: int = 10
    sst_size_target: int = 4 * 2**20
    range_lo: bytes | None = None
    range_hi: bytes | None = None


def _read_input(meta, inputs, directory):
    if inputs is not None:
        return inputs[meta.file_id]
    if directory is None:
        raise ValueError("run_compaction needs `inputs` (file_id -> bytes) or `directory`")
    with open(os.path.join(directory, f"{meta.file_id}.sst"), "rb") as f:
        return f.read()


def prepare(job, *, inputs=None, directory=None, config: StoreConfig | None = None,
            key_range=None) -> PreparedJob:
    """Gather input bytes and the run structure of a CompactionJob.

    Run rules: L0 files may overlap (each is its own run, newest first as in
    a Version); a level >= 1 file set is one sorted run (device-verified at
    every file seam, falling back to per-file runs if a seam is out of order).
    """
    cfg = config or StoreConfig()
    files, run_first = [], [0]
    lower = list(job.lower)
    upper = list(job.upper)
    if lower:
        if job.source_level == 0:
            for m in lower:
                files.append(_read_input(m, inputs, directory))
                run_first.append(len(files))
        else:
            for m in lower:
                files.append(_read_input(m, inputs, directory))
            run_first.append(len(files))
    if upper:
        for m in upper:
            files.append(_read_input(m, inputs, directory))
        run_first.append(len(files))
    lo, hi = (key_range or (None, None))
    return PreparedJob(files=files, run_first_file=run_first,
                       deeper=deeper_ranges(job.version, job.target_level),
                       block_size=cfg.block_size, restart_interval=cfg.restart_interval,
                       bits_per_key=cfg.bits_per_key, sst_size_target=cfg.sst_size_target,
                       range_lo=lo, range_hi=hi)


class JobRunner:
    """Keeps the pinned staging, device arena and output buffers of a device
    across jobs (so repeated jobs do not re-pin or re-allocate)."""

    def __init__(self, device: B200Device):
        self.device = device
        self.L = device._L
        self.pin_in = PinnedBuffer()
        self.pin_out = PinnedBuffer()
        self.arena = None
        self._keep = []

    def _arena(self, nbytes):
        if self.arena is None or self.arena.capacity < nbytes:
            if self.arena is not None:
                self.device.free(self.arena)
            self.arena = self.device.alloc(nbytes, label="job-arena")
        return self.arena

    def layout(self, files):
        offs, pos = [], ARENA_PAD
        for f in files:
            offs.append(pos)
            pos += (len(f) + ARENA_ALIGN - 1) // ARENA_ALIGN * ARENA_ALIGN
        return offs, pos + ARENA_PAD

    def stage(self, pj: PreparedJob, n_lower_files: int):
        """Copy inputs to pinned memory and H2D on in_lower / in_upper."""
        offs, total = self.layout(pj.files)
        self.pin_in.ensure(total)
        for f, o in zip(pj.files, offs):
            ctypes.memmove(self.pin_in.ptr + o, bytes(f) if not isinstance(f, bytes) else f, len(f))
        arena = self._arena(total)
        dev = self.device
        s_lo, s_up = dev.stream(STREAM_IN_LOWER), dev.stream(STREAM_IN_UPPER)
        s_cmp = dev.stream("compute")
        split = offs[n_lower_files] if n_lower_files < len(offs) else total
        _native.check(self.L.luda_stage_in_async(arena.dptr, self.pin_in.ptr, split, s_lo))
        if total > split:
            _native.check(self.L.luda_stage_in_async(arena.dptr + split, self.pin_in.ptr + split, total - split, s_up))
        for s in (s_lo, s_up):
            e = dev._event_on(s)
            _native.check(self.L.luda_stream_wait_event(s_cmp, e))
            _native.check(self.L.luda_event_destroy(e))  # released once the wait is satisfied
        return arena, offs, total

    def describe(self, pj: PreparedJob, arena, offs, total):
        n = len(pj.files)
        keep = []
        fo = (ctypes.c_uint64 * max(n, 1))(*offs)
        fl = (ctypes.c_uint64 * max(n, 1))(*[len(f) for f in pj.files])
        rf = (ctypes.c_uint32 * len(pj.run_first_file))(*pj.run_first_file)
        keep += [fo, fl, rf]
        d = _native.JobDesc()
        d.arena = arena.dptr
        d.arena_bytes = total
        d.n_files = n
        d.file_off = ctypes.cast(fo, _native.c_u64p)
        d.file_len = ctypes.cast(fl, _native.c_u64p)
        d.n_runs = len(pj.run_first_file) - 1
        d.run_first_file = ctypes.cast(rf, _native.c_u32p)
        d.block_size = pj.block_size
        d.restart_interval = pj.restart_interval
        d.bits_per_key = pj.bits_per_key
        d.sst_size_target = pj.sst_size_target
        if pj.deeper:
            blob = b"".join(lo + hi for lo, hi in pj.deeper)
            kb = (ctypes.c_uint8 * len(blob)).from_buffer_copy(blob)
            lens = (ctypes.c_uint32 * (2 * len(pj.deeper)))(*[len(x) for r in pj.deeper for x in r])
            keep += [kb, lens]
            d.n_deeper = len(pj.deeper)
            d.deeper_keys = ctypes.cast(kb, _native.c_u8p)
            d.deeper_lens = ctypes.cast(lens, _native.c_u32p)
        for name, key in (("range_lo", pj.range_lo), ("range_hi", pj.range_hi)):
            if key is not None:
                kb = (ctypes.c_uint8 * max(1, len(key))).from_buffer_copy(key or b"\0")
                keep.append(kb)
                setattr(d, name, ctypes.cast(kb, _native.c_u8p))
                setattr(d, name + "_len", len(key))
        return d, keep

    def fetch(self, res):
        """D2H the finished SSTs; returns [(bytes, smallest, largest)]."""
        n = res.out_bytes
        outs = []
        if res.n_sst == 0:
            return outs
        s_out = self.device.stream(STREAM_OUT)
        s_cmp = self.device.stream("compute")
        e = self.device._event_on(s_cmp)
        _native.check(self.L.luda_stream_wait_event(s_out, e))
        _native.check(self.L.luda_event_destroy(e))
        self.pin_out.ensure(n)
        _native.check(self.L.luda_stage_out_async(self.pin_out.ptr, res.out, n, s_out))
        _native.check(self.L.luda_stream_sync(s_out))
        raw = bytes(self.pin_out.view(n))
        for i, (sm, lg) in enumerate(_native.sst_key_pairs(res)):
            o, ln = res.sst_off[i], res.sst_len[i]
            outs.append((raw[o:o + ln], sm, lg))
        return outs

    def run(self, pj: PreparedJob, n_lower_files: int):
        t0 = time.perf_counter()
        arena, offs, total = self.stage(pj, n_lower_files)
        t1 = time.perf_counter()
        desc, keep = self.describe(pj, arena, offs, total)
        res = self.device.compact(desc)
        t2 = time.perf_counter()
        try:
            outs = self.fetch(res)
        finally:
            info = dict(n_in=res.n_in, n_out=res.n_out, blocks_in=res.blocks_in, blocks_out=res.blocks_out,
                        t_ms=list(res.t_ms))
            self.device.release(res)
        t3 = time.perf_counter()
        del keep
        self._keep.clear()
        return outs, info, (t0, t1, t2, t3)


_runners: dict = {}


def runner_for(device) -> JobRunner:
    r = _runners.get(id(device))
    if r is None or r.device is not device:
        r = _runners[id(device)] = JobRunner(device)
    return r


def file_id_allocator(job, new_file_id=None, *, stride: int = 1, offset: int = 0):
    """Callable handing out output file ids.

    ``new_file_id`` may be a callable, or an object with a ``new_file_id()``
    method (the reference's ``VersionSet``, version.py:299). Without one, ids
    count up from above EVERY file id of ``job.version`` and the job's inputs
    (files flushed meanwhile belong to the caller's VersionSet, which should
    then be passed). ``stride``/``offset`` interleave the ids of several
    ranks of one subcompacted job (rank r of G: stride G, offset r)."""
    if new_file_id is not None:
        return getattr(new_file_id, "new_file_id", new_file_id)
    ids = [m.file_id for m in list(job.lower) + list(job.upper)]
    for level in getattr(getattr(job, "version", None), "levels", None) or []:
        ids += [m.file_id for m in level]
    nxt = [max(ids + [0]) + 1 + offset]

    def alloc():
        v = nxt[0]
        nxt[0] += stride
        return v
    return alloc


def run_compaction(job, device, *, inputs=None, directory=None, config: StoreConfig | None = None,
                   new_file_id=None, key_range=None, job_id: int = 0):
    """Compact ``job`` on ``device``; returns ``(outputs, stats)`` where
    outputs is ``[(sst_bytes, SstMeta)]`` in key order.

    ``inputs`` maps file_id → bytes (else ``{directory}/{file_id}.sst`` is read).
    ``new_file_id`` is a callable (or a ``VersionSet``) producing output file
    ids (default: :func:`file_id_allocator`). ``key_range=(lo, hi)`` restricts the job to
    user keys in [lo, hi) (one subcompaction).
    """
    if not isinstance(device, B200Device):
        raise DeviceError("run_compaction needs the b200 device (make_device(DeviceConfig(backend='b200')))")
    pj = prepare(job, inputs=inputs, directory=directory, config=config, key_range=key_range)
    n_lower = len(job.lower)
    outs, info, (t0, t1, t2, t3) = runner_for(device).run(pj, n_lower)
    new_file_id = file_id_allocator(job, new_file_id)
    results = []
    for data, smallest, largest in outs:
        results.append((data, SstMeta(file_id=new_file_id(), file_size=len(data), smallest=smallest,
                                      largest=largest, level=job.target_level)))
    t = info["t_ms"]
    stats = JobStats(job_id=job_id, source_level=job.source_level, input_files=len(pj.files),
                     input_bytes=sum(len(f) for f in pj.files), output_files=len(results),
                     output_bytes=sum(len(d) for d, _ in results), t_stage_in=t1 - t0,
                     t_unpack=(t[0] + t[1]) / 1e3, t_sort_host=t[2] / 1e3, t_pack=(t[3] + t[4]) / 1e3,
                     t_stage_out=t3 - t2, n_in=info["n_in"], n_out=info["n_out"],
                     blocks_in=info["blocks_in"], blocks_out=info["blocks_out"],
                     t_device_ms={"parse": t[0], "decode": t[1], "merge": t[2], "plan": t[3], "emit": t[4],
                                  "total": t[7]})
    return results, stats


def compact_files(device, lower_files, upper_files=(), *, source_level=1, l0_runs=False, deeper=(),
                  config: StoreConfig | None = None, key_range=None):
    """Convenience: compact raw file bytes (lower = Li, upper = Li+1).

    Returns [(sst_bytes, smallest, largest)] like the oracle's reference_compact.
    """
    cfg = config or StoreConfig()
    files = list(lower_files) + list(upper_files)
    run_first = [0]
    if lower_files:
        if l0_runs or source_level == 0:
            for i in range(len(lower_files)):
                run_first.append(i + 1)
        else:
            run_first.append(len(lower_files))
    if upper_files:
        run_first.append(len(files))
    lo, hi = key_range or (None, None)
    pj = PreparedJob(files=files, run_first_file=run_first, deeper=list(deeper), block_size=cfg.block_size,
                     restart_interval=cfg.restart_interval, bits_per_key=cfg.bits_per_key,
                     sst_size_target=cfg.sst_size_target, range_lo=lo, range_hi=hi)
    outs, info, _ = runner_for(device).run(pj, len(lower_files))
    return outs
