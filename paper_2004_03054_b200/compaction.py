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
    staged: object = None       # StagedInput holding `files` in pinned memory (no host copy)
    io_mode: int | None = None  # files are FileRefs read by luda_files_read in this mode


class FileRef:
    """An input SST on storage that ``luda_files_read`` stages straight into
    the job's device arena (GPUDirect Storage / native bounce; no host copy
    by the caller). Sized like the bytes it stands for."""

    __slots__ = ("path", "size")

    def __init__(self, path):
        self.path = os.fspath(path)
        self.size = os.path.getsize(self.path)

    def __len__(self):
        return self.size


IO_MODES = {"auto": 0, "gds": 1, "bounce": 2}  # luda_files_read / luda_files_write mode


def _read_input(meta, inputs, directory, io=None):
    if inputs is not None:
        return inputs[meta.file_id]
    if directory is None:
        raise ValueError("run_compaction needs `inputs` (file_id -> bytes) or `directory`")
    path = os.path.join(directory, f"{meta.file_id}.sst")
    if io is not None:
        return FileRef(path)
    with open(path, "rb") as f:
        return f.read()


def prepare(job, *, inputs=None, directory=None, config: StoreConfig | None = None,
            key_range=None, staged=None, io=None) -> PreparedJob:
    """Gather input bytes and the run structure of a CompactionJob.

    Run rules: L0 files may overlap (each is its own run, newest first as in
    a Version); a level >= 1 file set is one sorted run (device-verified at
    every file seam, falling back to per-file runs if a seam is out of order).
    """
    cfg = config or StoreConfig()
    files, run_first = [], [0]
    lower = list(job.lower)
    upper = list(job.upper)
    if staged is not None:  # the job's files, lower then upper, already in pinned memory
        if len(staged.views) != len(lower) + len(upper):
            raise ValueError("staged input does not hold the job's files")
        seq = iter(staged.views)
        inputs = {m.file_id: next(seq) for m in lower + upper}
    if lower:
        if job.source_level == 0:
            for m in lower:
                files.append(_read_input(m, inputs, directory, io))
                run_first.append(len(files))
        else:
            for m in lower:
                files.append(_read_input(m, inputs, directory, io))
            run_first.append(len(files))
    if upper:
        for m in upper:
            files.append(_read_input(m, inputs, directory, io))
        run_first.append(len(files))
    lo, hi = (key_range or (None, None))
    return PreparedJob(files=files, run_first_file=run_first,
                       deeper=deeper_ranges(job.version, job.target_level),
                       block_size=cfg.block_size, restart_interval=cfg.restart_interval,
                       bits_per_key=cfg.bits_per_key, sst_size_target=cfg.sst_size_target,
                       range_lo=lo, range_hi=hi, staged=staged, io_mode=IO_MODES[io] if io else None)


_COPY_POOL = None


def _host_copy_in(dst, files, offs):
    """Copy bytes-like files into pinned staging at dst + offs[i]. ctypes
    calls release the GIL, so large jobs are copied by several threads."""
    def one(f, o):
        if isinstance(f, bytes):
            ctypes.memmove(dst + o, f, len(f))
            return
        mv = memoryview(f).cast("B")
        if mv.readonly:
            ctypes.memmove(dst + o, bytes(mv), len(mv))
        else:
            ctypes.memmove(dst + o, (ctypes.c_char * len(mv)).from_buffer(mv), len(mv))
    total = sum(len(f) for f in files)
    if total < (64 << 20) or len(files) < 4:
        for f, o in zip(files, offs):
            one(f, o)
        return
    global _COPY_POOL
    if _COPY_POOL is None:
        from concurrent.futures import ThreadPoolExecutor
        _COPY_POOL = ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1))
    list(_COPY_POOL.map(lambda fo: one(*fo), zip(files, offs)))


class StagedInput:
    """A job's input files already in PINNED host memory, laid out as the
    device arena (``JobRunner.layout``): staging them is one H2D per stream,
    no host copy. Fill ``views[i]`` (writable memoryviews), e.g. with
    ``fileobj.readinto(view)``, then pass ``staged=`` to run_compaction(s)."""

    def __init__(self, sizes):
        self.sizes = list(sizes)
        self.offs, self.total = JobRunner.layout_sizes(self.sizes)
        self.buf = PinnedBuffer()
        self.buf.ensure(self.total)
        raw = memoryview(self.buf.view(self.total)).cast("B")
        self.views = [raw[o:o + n] for o, n in zip(self.offs, self.sizes)]

    def free(self):
        self.views = []
        self.buf.free()


class JobRunner:
    """Double-buffered job pipeline of one device (SPEC.md:632 A7).

    Job k is staged (H2D of its files on the in_lower / in_upper streams, from
    pinned host memory) into device arena k % 2 while job k-1 compacts on the
    compute stream and job k-2's outputs stream back on the out stream into
    pinned output buffer (k-2) % 2. Inputs given as bytes-like objects are
    first copied into pinned staging (one host copy); a ``StagedInput`` is
    staged as is. Outputs are returned as memoryviews into the pinned output
    buffer: valid until the pipeline advances past the next job (copy with
    ``bytes()`` to keep them longer)."""

    def __init__(self, device: B200Device):
        self.device = device
        self.L = device._L
        self.pin_in = [PinnedBuffer(), PinnedBuffer()]
        self.pin_out = [PinnedBuffer(), PinnedBuffer()]
        self.arena = [None, None]
        self.in_events = []

    def _arena(self, k, nbytes):
        a = self.arena[k]
        if a is None or a.capacity < nbytes:
            if a is not None:
                self.device.free(a)
            a = self.arena[k] = self.device.alloc(nbytes, label=f"job-arena-{k}")
        return a

    @staticmethod
    def layout_sizes(sizes):
        offs, pos = [], ARENA_PAD
        for n in sizes:
            offs.append(pos)
            pos += (n + ARENA_ALIGN - 1) // ARENA_ALIGN * ARENA_ALIGN
        return offs, pos + ARENA_PAD

    def layout(self, files):
        return self.layout_sizes([len(f) for f in files])

    def stage(self, pj: PreparedJob, n_lower_files: int, k: int, after=None):
        """Pinned staging (unless pre-staged) + H2D into arena k on in_lower /
        in_upper; the compute stream waits for both copies. ``after``: events
        the copies wait for (the pipeline's first job gets PCIe to itself)."""
        if pj.io_mode is not None:  # storage → HBM directly (luda_files_read)
            offs, total = self.layout(pj.files)
            arena = self._arena(k, total)
            n = len(pj.files)
            paths = (ctypes.c_char_p * max(1, n))(*[f.path.encode() for f in pj.files])
            used = ctypes.c_int()
            _native.check(self.L.luda_files_read(paths, n, arena.dptr, (ctypes.c_uint64 * max(1, n))(*offs),
                                                 (ctypes.c_uint64 * max(1, n))(*[len(f) for f in pj.files]),
                                                 pj.io_mode, ctypes.byref(used)))
            self.last_io = {1: "gds", 2: "bounce"}[used.value]
            self.in_events = []  # synchronous: nothing to wait for
            return arena, offs, total, []
        staged = getattr(pj, "staged", None)
        if staged is not None:
            offs, total, src = staged.offs, staged.total, staged.buf.ptr
        else:
            offs, total = self.layout(pj.files)
            self.pin_in[k].ensure(total)
            src = self.pin_in[k].ptr
            _host_copy_in(src, pj.files, offs)
        arena = self._arena(k, total)
        dev = self.device
        s_lo, s_up = dev.stream(STREAM_IN_LOWER), dev.stream(STREAM_IN_UPPER)
        split = offs[n_lower_files] if n_lower_files < len(offs) else total
        for e in after or ():
            for s in (s_lo, s_up):
                _native.check(self.L.luda_stream_wait_event(s, e))
        _native.check(self.L.luda_stage_in_async(arena.dptr, src, split, s_lo))
        if total > split:
            _native.check(self.L.luda_stage_in_async(arena.dptr + split, src + split, total - split, s_up))
        # completion events of both copies: the compute stream waits on them right
        # before THIS job's compaction (wait_in), not now — a wait queued now would
        # also hold back the previous job, whose compaction is enqueued later
        self.in_events = [dev._event_on(s) for s in (s_lo, s_up)]
        return arena, offs, total, self.in_events

    def wait_in(self, events):
        """The compute stream waits for a staged job's copies; events released."""
        s_cmp = self.device.stream("compute")
        for e in events:
            _native.check(self.L.luda_stream_wait_event(s_cmp, e))
            _native.check(self.L.luda_event_destroy(e))

    def describe(self, pj: PreparedJob, arena, offs, total):
        n = len(pj.files)
        keep = []
        lens = pj.staged.sizes if getattr(pj, "staged", None) is not None else [len(f) for f in pj.files]
        fo = (ctypes.c_uint64 * max(n, 1))(*offs)
        fl = (ctypes.c_uint64 * max(n, 1))(*lens)
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

    def _fetch_async(self, res, k):
        """D2H of a finished job's SSTs into pinned output buffer k on the out
        stream (after the job's kernels). Returns the completion event."""
        dev = self.device
        s_out, s_cmp = dev.stream(STREAM_OUT), dev.stream("compute")
        e = dev._event_on(s_cmp)
        _native.check(self.L.luda_stream_wait_event(s_out, e))
        _native.check(self.L.luda_event_destroy(e))
        if res.out_bytes:
            self.pin_out[k].ensure(res.out_bytes)
            _native.check(self.L.luda_stage_out_async(self.pin_out[k].ptr, res.out, res.out_bytes, s_out))
        return dev._event_on(s_out)

    def _finish(self, res, k, ev, pj, t_issue):
        """Wait for job k's D2H; outputs as memoryviews into pin_out[k]."""
        _native.check(self.L.luda_event_wait(ev))
        _native.check(self.L.luda_event_destroy(ev))
        outs = []
        if res.n_sst:
            raw = memoryview(self.pin_out[k].view(res.out_bytes)).cast("B")
            for i, (sm, lg) in enumerate(_native.sst_key_pairs(res)):
                o, ln = res.sst_off[i], res.sst_len[i]
                outs.append((raw[o:o + ln], sm, lg))
        info = dict(n_in=res.n_in, n_out=res.n_out, blocks_in=res.blocks_in, blocks_out=res.blocks_out,
                    t_ms=list(res.t_ms), launches=res.launches, input_bytes=sum(
                        pj.staged.sizes if getattr(pj, "staged", None) is not None else [len(f) for f in pj.files]),
                    t_wall=time.perf_counter() - t_issue)
        self.device.release(res)
        return outs, info

    def run_many(self, jobs):
        """Generator over (PreparedJob, n_lower_files) pairs yielding
        (outputs, info) per job, in order, through the double-buffered
        pipeline (class docstring)."""
        it = iter(jobs)
        cur = next(it, None)
        if cur is None:
            return
        k = 0
        t0 = time.perf_counter()
        staged = self.stage(cur[0], cur[1], k)
        prev = None  # (res, k, event, pj, t)
        while cur is not None:
            nxt = next(it, None)
            nxt_staged = None
            if nxt is not None:
                # arena / staging buffer (k+1)%2 were last used by job k-1, whose compaction has returned.
                # Job k+1's copies start when BOTH of job k's have landed: on two streams, the half that
                # finishes first would otherwise start job k+1's copy and share PCIe with the other half,
                # delaying job k (whose compaction waits for both) by up to a whole transfer.
                nxt_staged = self.stage(nxt[0], nxt[1], (k + 1) % 2, after=staged[3])
            self.wait_in(staged[3])
            desc, keep = self.describe(cur[0], *staged[:3])
            res = self.device.compact(desc)
            del keep
            ev = self._fetch_async(res, k % 2)
            if prev is not None:
                yield self._finish(*prev)
            prev = (res, k % 2, ev, cur[0], t0)
            t0 = time.perf_counter()
            cur, staged, k = nxt, nxt_staged, k + 1
        yield self._finish(*prev)

    def run_to_files(self, pj: PreparedJob, n_lower_files: int, alloc, out_directory, io_mode: int):
        """One job whose output SSTs go from device memory straight to
        ``{out_directory}/{file_id}.sst`` (luda_files_write); returns
        ([(path, size, smallest, largest, file_id)], info)."""
        t0 = time.perf_counter()
        arena, offs, total, evs = self.stage(pj, n_lower_files, 0)
        self.wait_in(evs)
        desc, keep = self.describe(pj, arena, offs, total)
        res = self.device.compact(desc)
        del keep
        try:
            pairs = _native.sst_key_pairs(res)
            ids = [alloc() for _ in range(res.n_sst)]
            paths = [os.path.join(out_directory, f"{i}.sst") for i in ids]
            n = res.n_sst
            t_w = time.perf_counter()
            if n:
                used = ctypes.c_int()
                _native.check(self.L.luda_files_write((ctypes.c_char_p * n)(*[p.encode() for p in paths]), n,
                                                      res.out, res.sst_off, res.sst_len, io_mode,
                                                      ctypes.byref(used)))
                self.last_io_out = {1: "gds", 2: "bounce"}[used.value]
            outs = [(paths[i], res.sst_len[i], pairs[i][0], pairs[i][1], ids[i]) for i in range(n)]
            info = dict(n_in=res.n_in, n_out=res.n_out, blocks_in=res.blocks_in, blocks_out=res.blocks_out,
                        t_ms=list(res.t_ms), launches=res.launches, input_bytes=sum(len(f) for f in pj.files),
                        t_wall=time.perf_counter() - t0, t_write=time.perf_counter() - t_w)
        finally:
            self.device.release(res)
        return outs, info

    def run(self, pj: PreparedJob, n_lower_files: int):
        """One job; outputs copied to bytes (independent of the pipeline buffers)."""
        t0 = time.perf_counter()
        outs, info = next(self.run_many([(pj, n_lower_files)]))
        outs = [(bytes(d), sm, lg) for d, sm, lg in outs]
        return outs, info, (t0, t0, t0 + info["t_wall"], time.perf_counter())


_runners: dict = {}


def close_runner(device):
    """Release the pinned buffers of a device's job pipeline (B200Device.close)."""
    r = _runners.pop(id(device), None)
    if r is not None:
        for b in r.pin_in + r.pin_out:
            b.free()


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


def _job_stats(job, pj, outs_meta, info, job_id, t_stage_in=0.0, t_stage_out=0.0):
    t = info["t_ms"]
    return JobStats(job_id=job_id, source_level=job.source_level, input_files=len(pj.files),
                    input_bytes=info["input_bytes"], output_files=len(outs_meta),
                    output_bytes=sum(len(d) for d, _ in outs_meta), t_stage_in=t_stage_in,
                    t_unpack=(t[0] + t[1]) / 1e3, t_sort_host=t[2] / 1e3, t_pack=(t[3] + t[4]) / 1e3,
                    t_stage_out=t_stage_out, n_in=info["n_in"], n_out=info["n_out"],
                    blocks_in=info["blocks_in"], blocks_out=info["blocks_out"],
                    t_device_ms={"parse": t[0], "decode": t[1], "merge": t[2], "plan": t[3], "emit": t[4],
                                 "total": t[7]})


def _metas(job, outs, alloc):
    return [(data, SstMeta(file_id=alloc(), file_size=len(data), smallest=smallest, largest=largest,
                           level=job.target_level)) for data, smallest, largest in outs]


def run_compaction(job, device, *, inputs=None, directory=None, config: StoreConfig | None = None,
                   new_file_id=None, key_range=None, job_id: int = 0, staged=None, io=None,
                   out_directory=None):
    """Compact ``job`` on ``device``; returns ``(outputs, stats)`` where
    outputs is ``[(sst_bytes, SstMeta)]`` in key order.

    ``inputs`` maps file_id → bytes-like (else ``{directory}/{file_id}.sst`` is
    read); ``staged`` (a :class:`StagedInput` holding the job's files, lower
    then upper, in pinned memory) skips the host copy. ``new_file_id`` is a
    callable (or a ``VersionSet``) producing output file ids (default:
    :func:`file_id_allocator`). ``key_range=(lo, hi)`` restricts the job to
    user keys in [lo, hi) (one subcompaction).

    ``io="auto" | "gds" | "bounce"`` reads the inputs from ``directory``
    straight into device memory (luda_files_read: GPUDirect Storage through
    cuFile, or the native pinned-bounce pipeline) instead of through Python
    bytes. ``out_directory`` writes every output SST from device memory to
    ``{out_directory}/{file_id}.sst`` the same way; outputs are then
    ``[(path, SstMeta)]``.
    """
    if not isinstance(device, B200Device):
        raise DeviceError("run_compaction needs the b200 device (make_device(DeviceConfig(backend='b200')))")
    pj = prepare(job, inputs=inputs, directory=directory, config=config, key_range=key_range, staged=staged,
                 io=io)
    if out_directory is not None:
        outs, info = runner_for(device).run_to_files(pj, len(job.lower), file_id_allocator(job, new_file_id),
                                                     out_directory, IO_MODES[io or "auto"])
        results = [(path, SstMeta(file_id=fid, file_size=size, smallest=sm, largest=lg, level=job.target_level))
                   for path, size, sm, lg, fid in outs]
        stats = _job_stats(job, pj, [(range(m.file_size), m) for _, m in results], info, job_id,
                           t_stage_out=info["t_write"])
        return results, stats
    outs, info, (t0, t1, t2, t3) = runner_for(device).run(pj, len(job.lower))
    results = _metas(job, outs, file_id_allocator(job, new_file_id))
    return results, _job_stats(job, pj, results, info, job_id, t_stage_out=t3 - t2)


def run_compactions(jobs, device, *, inputs=None, directory=None, config: StoreConfig | None = None,
                    new_file_id=None, first_job_id: int = 0):
    """Pipelined ``run_compaction`` over many jobs (SPEC.md:632 A7): while
    job k compacts, job k+1's inputs are already streaming in and job k-1's
    outputs streaming out (``JobRunner``). ``jobs`` yields CompactionJobs or
    ``(CompactionJob, StagedInput)`` pairs. Yields ``(outputs, stats)`` per
    job in order; outputs are ``[(memoryview, SstMeta)]`` into pinned memory,
    valid until the generator advances (copy with ``bytes()`` to keep)."""
    if not isinstance(device, B200Device):
        raise DeviceError("run_compactions needs the b200 device")
    pending = []

    def prepared():
        for j in jobs:
            job, staged = j if isinstance(j, tuple) else (j, None)
            pj = prepare(job, inputs=inputs, directory=directory, config=config, staged=staged)
            pending.append((job, pj))
            yield pj, len(job.lower)
    shared = [0]

    def alloc_for(job):
        if new_file_id is not None:
            return file_id_allocator(job, new_file_id)
        base = file_id_allocator(job)()  # above every file of this job's Version
        shared[0] = max(shared[0], base)

        def alloc():  # one counter across the sequence: ids never repeat between jobs
            v = shared[0]
            shared[0] += 1
            return v
        return alloc
    for k, (outs, info) in enumerate(runner_for(device).run_many(prepared())):
        job, pj = pending.pop(0)
        results = _metas(job, outs, alloc_for(job))
        yield results, _job_stats(job, pj, results, info, first_job_id + k)


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
