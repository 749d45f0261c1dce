"""BASELINE config 5 — key-range-partitioned bulk compaction of one global
job across the GPUs of one box, synthesised on the devices.

The global job (default ~256 GB of input, 16-byte keys / 128-byte values):
  * Li+1: one sorted run of N1 keys (90 % of the entries), cut into input
    SSTs of ``file_keys`` entries each;
  * Li:   N0 = 10 % of the entries — 90 % fresh keys uniform over the same
    key space, 10 % overwrites of Li+1 keys — also cut every ``file_keys``;
  * the target level is the bottom (no tombstones here; values 128 B).
Keys live in NB generation buckets (bucket = top 12 bits of the key); bucket
b's keys, membership and values are a pure function of (seed, b), so any
rank can synthesise any input file without the rest of the job: the global
job is identical for every GPU count.

Schedule (§8e):
  1. rank r samples the files i ≡ r (mod G) — 64 evenly spaced keys of each
     (the keys an index block would give) — and the first key of each of its
     Li+1 files;
  2. the fixed-size sample arrays are all-gathered over NCCL (the only
     collective; ``subcompact.allgather_bytes``);
  3. every rank picks the same P − 1 splitters snapped to Li+1 file
     boundaries (``subcompact.choose_splitters``), P fixed (64) for every G;
  4. ranges are dealt contiguously (``subcompact.ranges_of_rank``); a rank
     runs its ranges in WAVES: synthesise exactly the input files the range
     needs on the device (the Li+1 files inside it, the Li files overlapping
     it), then ``luda_compact`` with ``range_lo/range_hi``.
Timing: CUDA events around each wave's compaction (synthesis is not timed);
a rank's time is the sum over its waves; the job time is the max over ranks.
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass

BYTES_PER_ENTRY = 157.6  # 16 B / 128 B entry in an SST


@dataclass
class C5Spec:
    total_gb: float = 256.0
    klen: int = 16
    vlen: int = 128
    upper_frac: float = 0.9
    overwrite_frac: float = 0.1
    file_keys: int = 26000
    nbuckets: int = 4096
    nranges: int = 64
    samples_per_file: int = 64
    seed: int = 0xC5

    def __post_init__(self):
        n_total = int(self.total_gb * 1e9 / BYTES_PER_ENTRY)
        nb = self.nbuckets
        self.up_per_bucket = max(1, int(n_total * self.upper_frac) // nb)
        lo_total = max(1, n_total - self.up_per_bucket * nb)
        self.lo_per_bucket = max(1, lo_total // nb)
        self.ow_per_bucket = int(self.lo_per_bucket * self.overwrite_frac)
        self.fresh_per_bucket = self.lo_per_bucket - self.ow_per_bucket
        self.n_up = self.up_per_bucket * nb
        self.n_lo = self.lo_per_bucket * nb
        self.n_up_files = math.ceil(self.n_up / self.file_keys)
        self.n_lo_files = math.ceil(self.n_lo / self.file_keys)


class Bucket:
    """Keys of one generation bucket: Li+1 keys (sorted) and Li entries
    (sorted), as (hi, lo) int64 word pairs in unsigned-order-preserving form
    (hi XOR 2^63 sorts like the unsigned big-endian key)."""


def gen_bucket(spec: C5Spec, b: int, device):
    import torch
    g = torch.Generator(device=device)
    g.manual_seed((spec.seed * 1000003 + b) & 0x7FFFFFFFFFFFFFFF)
    n_up, n_fresh, n_ow = spec.up_per_bucket, spec.fresh_per_bucket, spec.ow_per_bucket
    n = n_up + n_fresh
    while True:
        # unsigned key prefix = b << 52 | rand52, held sign-flipped so signed order == unsigned order
        r52 = torch.randint(0, 1 << 52, (n,), generator=g, device=device, dtype=torch.int64)
        top = (b << 52) ^ (1 << 63)            # bucket prefix, sign-flipped, as a signed 64-bit value
        hi = r52 | (top - (1 << 64) if top >= 1 << 63 else top)
        lo = torch.randint(-(1 << 63), (1 << 63) - 1, (n,), generator=g, device=device, dtype=torch.int64)
        hi, order = torch.sort(hi)
        lo = lo[order]
        if bool((hi[1:] != hi[:-1]).all()):
            break
    is_up = torch.zeros(n, dtype=torch.bool, device=device)
    is_up[torch.randperm(n, generator=g, device=device)[:n_up]] = True
    up_idx = torch.nonzero(is_up).flatten()
    fresh_idx = torch.nonzero(~is_up).flatten()
    ow_idx = up_idx[torch.randperm(n_up, generator=g, device=device)[:n_ow]]
    lo_idx, _ = torch.sort(torch.cat([fresh_idx, ow_idx]))
    bk = Bucket()
    bk.up_hi, bk.up_lo = hi[up_idx], lo[up_idx]
    bk.lo_hi, bk.lo_lo = hi[lo_idx], lo[lo_idx]
    return bk


def key_bytes(hi, lo):
    """(hi sign-flipped, lo) int64 pairs -> n x 16 big-endian key bytes (uint8, flat)."""
    import torch
    words = torch.stack([hi ^ (-(1 << 63)), lo], 1).contiguous()
    return words.view(torch.uint8).view(-1, 2, 8).flip(2).reshape(-1).contiguous()


class Synth:
    """Bucket cache + global-index → key lookups for one rank."""

    def __init__(self, spec: C5Spec, device):
        self.spec = spec
        self.device = device
        self.cache = {}

    def bucket(self, b):
        bk = self.cache.get(b)
        if bk is None:
            if len(self.cache) > 64:
                self.cache.clear()
            bk = self.cache[b] = gen_bucket(self.spec, b, self.device)
        return bk

    def keys(self, level: str, i0: int, i1: int):
        """(hi, lo) of global entries [i0, i1) of a level ('up' or 'lo')."""
        import torch
        per = self.spec.up_per_bucket if level == "up" else self.spec.lo_per_bucket
        his, los = [], []
        i = i0
        while i < i1:
            b, off = divmod(i, per)
            take = min(i1 - i, per - off)
            bk = self.bucket(b)
            h, l_ = (bk.up_hi, bk.up_lo) if level == "up" else (bk.lo_hi, bk.lo_lo)
            his.append(h[off:off + take])
            los.append(l_[off:off + take])
            i += take
        return torch.cat(his), torch.cat(los)

    def n(self, level):
        return self.spec.n_up if level == "up" else self.spec.n_lo

    def file_span(self, level, f):
        F = self.spec.file_keys
        return f * F, min((f + 1) * F, self.n(level))


def gather_keys(synth: Synth, idx_up, idx_lo):
    """16-byte keys of global entry indices of both levels, generating every
    bucket once: returns (n_up x 16, n_lo x 16) uint8 numpy arrays in the
    order of the given indices."""
    import numpy as np
    import torch
    spec = synth.spec
    idx_up = np.asarray(idx_up, dtype=np.int64)
    idx_lo = np.asarray(idx_lo, dtype=np.int64)
    out_up = np.zeros((idx_up.size, 16), dtype=np.uint8)
    out_lo = np.zeros((idx_lo.size, 16), dtype=np.uint8)
    bu = idx_up // spec.up_per_bucket
    bl = idx_lo // spec.lo_per_bucket
    for b in np.union1d(np.unique(bu), np.unique(bl)):
        bk = gen_bucket(spec, int(b), synth.device)
        for idx, bsel, per, h, l_, out in ((idx_up, bu, spec.up_per_bucket, bk.up_hi, bk.up_lo, out_up),
                                           (idx_lo, bl, spec.lo_per_bucket, bk.lo_hi, bk.lo_lo, out_lo)):
            m = np.nonzero(bsel == b)[0]
            if m.size:
                t = torch.from_numpy(idx[m] - b * per).to(h.device)
                out[m] = key_bytes(h[t], l_[t]).view(-1, 16).cpu().numpy()
    return out_up, out_lo


def metadata(spec: C5Spec, synth: Synth, world: int, rank: int):
    """One pass over the generation buckets: (first, last) user key of every
    input file of both levels, and this rank's index-style samples (files
    i ≡ rank mod world of each level, `samples_per_file` evenly spaced keys)."""
    import numpy as np
    S, F = spec.samples_per_file, spec.file_keys
    idx = {}
    for level, nf, n in (("up", spec.n_up_files, spec.n_up), ("lo", spec.n_lo_files, spec.n_lo)):
        f = np.arange(nf, dtype=np.int64)
        a, e = f * F, np.minimum((f + 1) * F, n)
        mine = f[rank::world]
        smp = (a[mine][:, None] + (np.arange(S)[None, :] * (e[mine] - a[mine])[:, None]) // S).reshape(-1)
        idx[level] = (nf, mine.size, np.concatenate([a, e - 1, smp]))
    ku, kl = gather_keys(synth, idx["up"][2], idx["lo"][2])
    out = {}
    for level, keys in (("up", ku), ("lo", kl)):
        nf, nm, _ = idx[level]
        kb = [bytes(r) for r in keys]
        out[level] = ([(kb[f], kb[nf + f]) for f in range(nf)], kb[2 * nf:2 * nf + nm * S], nm)
    return out


def plan(spec: C5Spec, synth: Synth, world: int, rank: int, group=None, meta=None):
    """§8e steps 1-4 (samples of this rank's files, all-gather, splitters
    snapped to Li+1 file boundaries, contiguous deal). Returns (ranges, my
    range indices, plan wall ms, sample count, file bounds per level)."""
    from paper_2004_03054_b200 import subcompact as SC
    t0 = time.perf_counter()
    meta = meta or metadata(spec, synth, world, rank)
    S = spec.samples_per_file
    local = meta["up"][1] + meta["lo"][1]
    firsts = [meta["up"][1][q * S] for q in range(meta["up"][2])]
    per_rank = lambda nf: (nf + world - 1) // world  # noqa: E731 — files of the most loaded rank
    rows = (per_rank(spec.n_up_files) + per_rank(spec.n_lo_files)) * S
    samples = [k for gth in SC.allgather_bytes(SC.encode_samples(local, rows), world, group)
               for k in SC.decode_samples(gth)]
    bounds = [k for gth in SC.allgather_bytes(SC.encode_samples(firsts, per_rank(spec.n_up_files)), world, group)
              for k in SC.decode_samples(gth)]
    bounds = sorted(bounds)[1:]  # smallest user key of every Li+1 file but the first
    spl = SC.choose_splitters(samples, bounds, spec.nranges)
    ranges = SC.ranges_from_splitters(spl)
    mine = SC.ranges_of_rank(len(ranges), world, rank)
    return ranges, mine, (time.perf_counter() - t0) * 1e3, len(samples), (meta["up"][0], meta["lo"][0])


def file_bounds(spec: C5Spec, synth: Synth, level: str):
    """[(first user key, last user key)] of every input file of a level."""
    return metadata(spec, synth, 1, 0)[level][0]


def build_files(L, synth: Synth, level: str, f0: int, f1: int, stream, values_pool):
    """Input files [f0, f1) of a level, built on the device in ONE call
    (luda_build_files_from_sorted: an SST every file_keys entries)."""
    import torch
    from paper_2004_03054_b200 import _native
    spec = synth.spec
    F = spec.file_keys
    a, e = f0 * F, min(f1 * F, synth.n(level))
    n = e - a
    hi, lo = synth.keys(level, a, e)
    keys = key_bytes(hi, lo)
    idx = torch.arange(a, e, device=hi.device, dtype=torch.int64)
    seq = idx + 1 if level == "up" else idx + spec.n_up + 1
    tr = (seq << 8) | 1
    # value of entry i: a window of one shared random pool chosen by (level, i) — deterministic
    span = values_pool.numel() - spec.vlen
    voff = (idx * (2654435761 if level == "up" else 40503) + (0 if level == "up" else 7)) % span
    vl = torch.full((n,), spec.vlen, dtype=torch.int32, device=hi.device)
    # the builder runs on its own stream: torch's producers of keys/tr/voff/vl must be done
    torch.cuda.current_stream(hi.device).synchronize()
    res = _native.JobResult()
    _native.check(L.luda_build_files_from_sorted(keys.data_ptr(), spec.klen, tr.data_ptr(), values_pool.data_ptr(),
                                                 voff.data_ptr(), vl.data_ptr(), n, 4096, 16, 10, 1 << 31, F,
                                                 ctypes.byref(res), stream))
    assert res.n_sst == f1 - f0, (res.n_sst, f0, f1)
    return res


def values_pool_for(spec, device):
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(spec.seed ^ 0x5A5A)
    return torch.empty(1 << 24, dtype=torch.uint8, device=device).random_(0, 256, generator=g)


def stage_range(L, synth, bounds_up, bounds_lo, lo_key, hi_key, stream, pool, device):
    """Build the input files of one range (Li files overlapping [lo, hi),
    Li+1 files inside it) and lay them out in one device arena. Returns
    (arena, file_off, file_len, n_lower, arena bytes, bytes owned by the
    range: Li+1 files plus the Li files whose first key lies in it)."""
    import torch
    from paper_2004_03054_b200 import _native

    def overlapping(bounds):
        fs = [f for f, (s, l) in enumerate(bounds)
              if (hi_key is None or s < hi_key) and (lo_key is None or l >= lo_key)]
        return (fs[0], fs[-1] + 1) if fs else (0, 0)
    (l0, l1), (u0, u1) = overlapping(bounds_lo), overlapping(bounds_up)
    parts = []
    if l1 > l0:
        parts.append(("lo", l0, build_files(L, synth, "lo", l0, l1, stream, pool)))
    if u1 > u0:
        parts.append(("up", u0, build_files(L, synth, "up", u0, u1, stream, pool)))
    total = sum(r.out_bytes for _, _, r in parts) + 4096
    arena = torch.empty(total, dtype=torch.uint8, device=device)
    torch.cuda.current_stream(device).synchronize()  # (the block may come from a tensor torch just freed)
    offs, lens, at, owned = [], [], 0, 0
    for level, f0, r in parts:
        _native.check(L.luda_memcpy_d2d_async(arena.data_ptr() + at, r.out, r.out_bytes, stream))
        bnd = bounds_lo if level == "lo" else bounds_up
        for i in range(r.n_sst):
            offs.append(at + r.sst_off[i])
            lens.append(r.sst_len[i])
            first = bnd[f0 + i][0]
            if level == "up" or ((lo_key is None or first >= lo_key) and (hi_key is None or first < hi_key)):
                owned += r.sst_len[i]
        at += r.out_bytes
    _native.check(L.luda_stream_sync(stream))
    for _, _, r in parts:
        L.luda_job_release(ctypes.byref(r))
    return arena, offs, lens, (l1 - l0), at, owned


def range_desc(arena, offs, lens, n_lower, lo_key, hi_key, nbytes):
    from paper_2004_03054_b200 import _native
    n = len(offs)
    fo = (ctypes.c_uint64 * max(n, 1))(*offs)
    fl = (ctypes.c_uint64 * max(n, 1))(*lens)
    rf = (ctypes.c_uint32 * 3)(0, n_lower, n)
    d = _native.JobDesc()
    d.arena, d.arena_bytes, d.n_files = arena.data_ptr(), nbytes, n
    d.file_off = ctypes.cast(fo, _native.c_u64p)
    d.file_len = ctypes.cast(fl, _native.c_u64p)
    d.n_runs = 2 if 0 < n_lower < n else 1
    if d.n_runs == 1:
        rf = (ctypes.c_uint32 * 2)(0, n)
    d.run_first_file = ctypes.cast(rf, _native.c_u32p)
    d.block_size, d.restart_interval, d.bits_per_key, d.sst_size_target = 4096, 16, 10, 4 * 2**20
    keep = [fo, fl, rf]
    for name, key in (("range_lo", lo_key), ("range_hi", hi_key)):
        if key is not None:
            kb = (ctypes.c_uint8 * len(key)).from_buffer_copy(key)
            keep.append(kb)
            setattr(d, name, ctypes.cast(kb, _native.c_u8p))
            setattr(d, name + "_len", len(key))
    return d, keep


def run(spec: C5Spec, device_index: int, world: int, rank: int, group=None, steps: int = 1, warmup: int = 1,
        e2e_waves: int = 2, collect=None):
    """Plan + waves on this rank. Each wave: synthesise the range's inputs
    (untimed), `warmup` untimed compactions, then `steps` timed ones (CUDA
    events on the job stream; the wave's time is their mean). The first
    `e2e_waves` waves are also run end to end: the staged inputs are copied
    to pinned host memory (untimed), then H2D of every input + the job + D2H
    of every output are timed on the host clock.
    ``collect(range_index, result, L, stream, arena, offs, lens, n_lower, lo,
    hi)`` (tests) sees every range's inputs and result before they are
    released. Returns this rank's totals."""
    import torch
    from paper_2004_03054_b200 import _native
    from paper_2004_03054_b200.device import PinnedBuffer
    L = _native.lib(device_index)
    device = torch.device("cuda", device_index)
    synth = Synth(spec, device)
    ranges, mine, plan_ms, nsamples, (bounds_up, bounds_lo) = plan(spec, synth, world, rank, group)
    t0 = time.perf_counter()
    pool = values_pool_for(spec, device)
    s = ctypes.c_void_p()
    _native.check(L.luda_stream_create(ctypes.byref(s)))
    ev0, ev1 = ctypes.c_void_p(), ctypes.c_void_p()
    _native.check(L.luda_event_create(ctypes.byref(ev0)))
    _native.check(L.luda_event_create(ctypes.byref(ev1)))
    tot = dict(ms=0.0, in_bytes=0, staged_bytes=0, out_bytes=0, n_in=0, n_out=0, ssts=0, waves=0, launches=0,
               plan_ms=plan_ms, samples=nsamples, ranges=len(ranges), mine=[mine[0], mine[-1] + 1] if mine else [],
               e2e_s=0.0, e2e_in_bytes=0, e2e_h2d=0, e2e_d2h=0, e2e_waves=0, splitters=[
                   (r[0] or b"").hex() for r in ranges[1:]][:3])
    pin_in, pin_out = PinnedBuffer(), PinnedBuffer()

    def job(desc):
        res = _native.JobResult()
        _native.check(L.luda_compact(ctypes.byref(desc), ctypes.byref(res), s.value))
        return res

    for r in mine:
        lo_key, hi_key = ranges[r]
        arena, offs, lens, n_lower, nbytes, owned = stage_range(L, synth, bounds_up, bounds_lo, lo_key, hi_key,
                                                                s.value, pool, device)
        if not offs:
            continue
        desc, keep = range_desc(arena, offs, lens, n_lower, lo_key, hi_key, nbytes)
        for _ in range(warmup):
            L.luda_job_release(ctypes.byref(job(desc)))
        wave_ms = 0.0
        for k in range(steps):
            _native.check(L.luda_event_record(ev0.value, s.value))
            res = job(desc)
            _native.check(L.luda_event_record(ev1.value, s.value))
            _native.check(L.luda_event_wait(ev1.value))
            ms = ctypes.c_float()
            _native.check(L.luda_event_elapsed_ms(ev0.value, ev1.value, ctypes.byref(ms)))
            wave_ms += ms.value
            if k + 1 < steps:
                L.luda_job_release(ctypes.byref(res))
        tot["ms"] += wave_ms / max(1, steps)
        tot["in_bytes"] += owned
        tot["staged_bytes"] += nbytes
        tot["out_bytes"] += res.out_bytes
        tot["n_in"] += res.n_in
        tot["n_out"] += res.n_out
        tot["ssts"] += res.n_sst
        tot["launches"] += res.launches
        tot["waves"] += 1
        if collect is not None:
            collect(r, res, L, s.value, arena, offs, lens, n_lower, lo_key, hi_key)
        out_bytes = res.out_bytes
        L.luda_job_release(ctypes.byref(res))
        if tot["e2e_waves"] < e2e_waves:
            pin_in.ensure(nbytes)
            pin_out.ensure(out_bytes + 4096)
            _native.check(L.luda_stage_out_async(pin_in.ptr, arena.data_ptr(), nbytes, s.value))
            _native.check(L.luda_stream_sync(s.value))
            t1 = time.perf_counter()
            _native.check(L.luda_stage_in_async(arena.data_ptr(), pin_in.ptr, nbytes, s.value))
            res = job(desc)
            _native.check(L.luda_stage_out_async(pin_out.ptr, res.out, res.out_bytes, s.value))
            _native.check(L.luda_stream_sync(s.value))
            tot["e2e_s"] += time.perf_counter() - t1
            tot["e2e_in_bytes"] += owned
            tot["e2e_h2d"] += nbytes
            tot["e2e_d2h"] += res.out_bytes
            tot["e2e_waves"] += 1
            L.luda_job_release(ctypes.byref(res))
        del arena, keep
    pin_in.free()
    pin_out.free()
    tot["wall_s"] = time.perf_counter() - t0
    _native.check(L.luda_stream_destroy(s.value))
    return tot
