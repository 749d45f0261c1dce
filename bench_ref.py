"""Reference arm of bench.py (``--impl reference``) and the CPU baseline.

Times the UNMODIFIED reference (``/root/reference/pkg`` pip-installed into
``baseline/_ref`` — git-ignored, shipped to the GPU box with the snapshot)
on the box's host cores. The reference ships no compaction entry point
(``run_compaction`` is SPEC-only), so a job is the
composition of its own public calls that SURVEY §3.2 pins as the reference
compaction (and that ``tests/golden/make_golden.py`` checked byte-identical
against the reference's own offload kernels):

    Table parse (``sst.decode_index_block``, ``bloom.FilterBlock.decode``,
    ``blocks.decode_data_block``) → ``heapq.merge`` on ``keys.sort_key`` →
    newest per user key → D12 tombstone drop → ``sst.SstBuilder`` cut on
    ``SizeOverflowError``.

A second leg runs the reference's OFFLOAD path on its own
``HostParallelDevice`` (``workers = cores - 2``, no modelled bandwidth or
latency): ``unpack`` items per input block, host tuple merge + resolve +
greedy block plan, ``shared_key`` / ``encode`` items per output block,
``filter`` items per output SST, host index + footer.

Inputs are c3- (N = 1) or c5-shaped (N > 1) samples built with the
reference's ``SstBuilder`` (untimed). Without ``baseline/_ref`` the oracle
restatement (``oracle/``, pinned to the reference's golden outputs) stands
in and the line says ``kind: "port"``.
"""

from __future__ import annotations

import heapq
import os
import random
import statistics
import struct
import sys
import time

REPO = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(REPO, "baseline", "_ref")
MIB4 = 4 * 2**20


def load_reference():
    """The installed reference package (``luda``) or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "luda")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import luda.blocks  # noqa: F401
    import luda.bloom  # noqa: F401
    import luda.config  # noqa: F401
    import luda.device  # noqa: F401
    import luda.errors  # noqa: F401
    import luda.keys  # noqa: F401
    import luda.kernels  # noqa: F401
    import luda.sst  # noqa: F401
    import luda
    return luda


# ------------------------------------------------------------------------------------------
# reference composition (inline)
# ------------------------------------------------------------------------------------------
def ref_build_split(R, pairs, sst_size_target=MIB4, block_size=4096, restart_interval=16, bits_per_key=10):
    outs = []

    def new():
        return R.sst.SstBuilder(block_size=block_size, restart_interval=restart_interval,
                                bits_per_key=bits_per_key, sst_size_target=sst_size_target)
    b = new()
    count = 0
    for k, v in pairs:
        try:
            b.add(k, v)
        except R.errors.SizeOverflowError:
            outs.append(b.finish())
            b = new()
            b.add(k, v)
        count += 1
    if count:
        outs.append(b.finish())
    return outs


def ref_open_scan(R, data: bytes):
    foff, flen, ioff, ilen, magic = struct.unpack_from("<IIIIQ", data, len(data) - 24)
    if magic != R.sst.MAGIC:
        raise R.errors.FormatError("bad magic")
    R.bloom.FilterBlock.decode(data[foff:foff + flen], offset=foff)
    index = R.sst.decode_index_block(data[ioff:ioff + ilen], offset=ioff)
    pairs = []
    for _, off, ln in index:
        pairs.extend(R.blocks.decode_data_block(data[off:off + ln], offset=off))
    return pairs


def ref_compact(R, files, deeper=(), **cfg):
    runs = [ref_open_scan(R, f) for f in files]
    merged = heapq.merge(*runs, key=lambda kv: R.keys.sort_key(kv[0]))

    def survivors():
        prev = None
        for k, v in merged:
            u = R.keys.user_key_of(k)
            if u == prev:
                continue
            prev = u
            if R.keys.kind_of(k) == R.keys.KIND_DELETE and not any(lo <= u <= hi for lo, hi in deeper):
                continue
            yield k, v
    return ref_build_split(R, survivors(), **cfg)


# ------------------------------------------------------------------------------------------
# reference offload composition on HostParallelDevice
# ------------------------------------------------------------------------------------------
def ref_offload_compact(R, dev, files, deeper=(), sst_size_target=MIB4, block_size=4096, restart_interval=16,
                        bits_per_key=10):
    """The reference's offload compaction, composed from its shipped device
    protocol and kernels. Returns the output SST bytes."""
    KS = R.device.KernelSpec
    K = R.kernels
    # stage inputs, decode every block on the device workers
    regions = []
    items = []
    blocks_per_file = []
    total_blocks = 0
    for f in files:
        foff, flen, ioff, ilen, _ = struct.unpack_from("<IIIIQ", f, len(f) - 24)
        R.bloom.FilterBlock.decode(f[foff:foff + flen], offset=foff)
        index = R.sst.decode_index_block(f[ioff:ioff + ilen], offset=ioff)
        src = dev.alloc(len(f))
        dev.stage_in(src, f, "in_lower").wait()
        regions.append(src)
        blocks_per_file.append(index)
        total_blocks += sum(ln for _, _, ln in index)
    cap = total_blocks * 4 + 64
    pairs = dev.alloc(cap)
    tups = dev.alloc(cap)
    slot = 0
    spans = []
    for src, index in zip(regions, blocks_per_file):
        fs = []
        for _, off, ln in index:
            items.append((src.region_id, off, ln, pairs.region_id, slot, 4 * ln, tups.region_id, slot, 4 * ln))
            fs.append(slot)
            slot += 4 * ln
        spans.append(fs)
    res = dev.dispatch(KS("unpack", tuple(items), reads=tuple(r.region_id for r in regions),
                          writes=(pairs.region_id, tups.region_id))).wait()
    # tuples back to the host; per-file runs
    ranges = [(items[i][7], res[i][1]) for i in range(len(items))]
    tbuf = dev.stage_out(tups, ranges, "out").wait()
    runs, pos, i = [], 0, 0
    for fs in spans:
        run = []
        for _ in fs:
            n = ranges[i][1]
            for key, v_off, v_len in K.parse_tuples(tbuf, pos, pos + n):
                run.append((key, v_off, v_len))
            pos += n
            i += 1
        runs.append(run)
    # host merge + resolve (SPEC cooperative sort: newest per user key, D12)
    merged = heapq.merge(*runs, key=lambda t: R.keys.sort_key(t[0]))
    surv = []
    prev = None
    for t in merged:
        u = R.keys.user_key_of(t[0])
        if u == prev:
            continue
        prev = u
        if R.keys.kind_of(t[0]) == R.keys.KIND_DELETE and not any(lo <= u <= hi for lo, hi in deeper):
            continue
        surv.append(t)
    # host block plan (must equal SstBuilder's cut, sst.py:138-162) + SST cut
    ssts, cur, blocks = [], [], []
    cur_bytes, data_bytes, n_in_block, prev_key = 0, 0, 0, None
    for t in surv:
        key, vl = t[0], t[2]
        sh = 0 if n_in_block % restart_interval == 0 else R.blocks.shared_prefix_len(prev_key, key)
        size_e = R.blocks.entry_encoded_size(sh, len(key) - sh, vl)
        if cur and cur_bytes + size_e + R.blocks.block_overhead(n_in_block + 1, restart_interval) - 4 > block_size:
            blocks.append(cur)
            data_bytes += cur_bytes + R.blocks.block_overhead(n_in_block, restart_interval)
            cur, cur_bytes, n_in_block = [], 0, 0
            sh = 0
            size_e = R.blocks.entry_encoded_size(0, len(key), vl)
            if data_bytes >= sst_size_target:
                ssts.append(blocks)
                blocks, data_bytes = [], 0
        cur.append(t)
        cur_bytes += size_e
        n_in_block += 1
        prev_key = key
    if cur:
        blocks.append(cur)
    if blocks:
        ssts.append(blocks)
    # shared_key + encode per output block, filter per SST, on the device workers
    wire = bytearray()
    blk_spans, sst_spans = [], []
    for blocks in ssts:
        s0 = len(wire)
        for blk in blocks:
            b0 = len(wire)
            for key, v_off, v_len in blk:
                wire += K.encode_tuple(key, v_off, v_len)
            blk_spans.append((b0, len(wire), len(blk)))
        sst_spans.append((s0, len(wire), len(blocks)))
    treg = dev.alloc(max(1, len(wire)))
    dev.stage_in(treg, bytes(wire), "in_upper").wait()
    lay = dev.alloc(8 * max(1, len(surv)))
    sk, enc, lay_off = [], [], 0
    out_cap = sum(block_size + 16 + sum(len(t[0]) + t[2] + 15 for t in blk) for blocks in ssts for blk in blocks)
    outb = dev.alloc(out_cap)
    o = 0
    for b0, b1, n in blk_spans:
        sk.append((treg.region_id, b0, b1, restart_interval, lay.region_id, lay_off))
        lay_off += 8 * n
    dev.dispatch(KS("shared_key", tuple(sk), reads=(treg.region_id,), writes=(lay.region_id,))).wait()
    lay_off = 0
    caps = []
    for (b0, b1, n), blk in zip(blk_spans, [b for blocks in ssts for b in blocks]):
        cap_b = block_size + 16 + sum(len(t[0]) + t[2] + 15 for t in blk)
        enc.append((treg.region_id, b0, b1, lay.region_id, lay_off, pairs.region_id, outb.region_id, o, cap_b,
                    restart_interval))
        caps.append((o, cap_b))
        o += cap_b
        lay_off += 8 * n
    er = dev.dispatch(KS("encode", tuple(enc), reads=(treg.region_id, lay.region_id, pairs.region_id),
                         writes=(outb.region_id,))).wait()
    fcap = sum(bits_per_key * (s1 - s0) // 8 + 4096 for s0, s1, _ in sst_spans)
    freg = dev.alloc(max(1, fcap))
    fi, fo = [], 0
    for s0, s1, _ in sst_spans:
        c = (s1 - s0) * bits_per_key // 8 + 4096  # wire bytes bound the key count
        fi.append((treg.region_id, s0, s1, bits_per_key, freg.region_id, fo, c))
        fo += c
    fr = dev.dispatch(KS("filter", tuple(fi), reads=(treg.region_id,), writes=(freg.region_id,))).wait()
    blk_bytes = dev.stage_out(outb, [(caps[i][0], er[i][0]) for i in range(len(enc))], "out").wait()
    flt_bytes = dev.stage_out(freg, [(fi[i][5], fr[i][0]) for i in range(len(fi))], "out").wait()
    # host: index + footer (sst.py:67-76, 199-208)
    outs = []
    bp = fp = bi = 0
    for si, blocks in enumerate(ssts):
        data = bytearray()
        index = []
        for blk in blocks:
            ln = er[bi][0]
            index.append((blk[-1][0], len(data), ln))
            data += blk_bytes[bp:bp + ln]
            bp += ln
            bi += 1
        flen = fr[si][0]
        foff = len(data)
        data += flt_bytes[fp:fp + flen]
        fp += flen
        ioff = len(data)
        iblk = R.sst.encode_index_block(index)
        data += iblk
        data += struct.pack("<IIIIQ", foff, flen, ioff, len(iblk), R.sst.MAGIC)
        outs.append(bytes(data))
    dev.free_all()
    return outs


# ------------------------------------------------------------------------------------------
# sample jobs (built with the reference's SstBuilder, untimed)
# ------------------------------------------------------------------------------------------
def _keys(rng, n, klen=16):
    s = set()
    while len(s) < n:
        s.add(rng.randbytes(klen))
    return sorted(s)


def sample_job(R, shape: str, n_keys: int, seed: int):
    """Input files of one c3- or c5-shaped job (16 B / 128 B, 4 MiB SSTs)."""
    rng = random.Random(seed)
    enc = R.keys.encode_key
    if shape == "c3":  # every key in both runs, 20 % of the Li versions deletes
        keys = _keys(rng, n_keys)
        upper = [(enc(k, 1 + i, 1), rng.randbytes(128)) for i, k in enumerate(keys)]
        lower = []
        for i, k in enumerate(keys):
            dele = rng.random() < 0.2
            lower.append((enc(k, n_keys + 1 + i, 0 if dele else 1), b"" if dele else rng.randbytes(128)))
    else:  # c5: Li = 10 % of the entries, 90 % fresh keys + 10 % overwrites
        n_lo = max(1, n_keys // 9)
        allk = _keys(rng, n_keys + n_lo)
        up_set = set(rng.sample(range(len(allk)), n_keys))
        upk = [allk[i] for i in sorted(up_set)]
        fresh = [allk[i] for i in range(len(allk)) if i not in up_set]
        low = sorted(fresh[:n_lo - n_lo // 10] + rng.sample(upk, n_lo // 10))
        upper = [(enc(k, 1 + i, 1), rng.randbytes(128)) for i, k in enumerate(upk)]
        lower = [(enc(k, n_keys + 1 + i, 1), rng.randbytes(128)) for i, k in enumerate(low)]
    return ref_build_split(R, lower) + ref_build_split(R, upper)


# ------------------------------------------------------------------------------------------
# pool workers
# ------------------------------------------------------------------------------------------
_FILES = None
_R = None


def _init(shape, n_keys, seed):
    global _FILES, _R
    import multiprocessing as mp
    ident = mp.current_process()._identity
    _R = load_reference()
    if _R is None:
        from oracle import jobgen
        from oracle import luda_oracle as O  # noqa: F401
        job = jobgen.c3(n=n_keys, seed=seed + (ident[0] if ident else 0), sst_target=MIB4)
        lo, up = jobgen.materialize(job)
        _FILES = lo + up
    else:
        _FILES = sample_job(_R, shape, n_keys, seed + (ident[0] if ident else 0))


def _compact(_):
    t0 = time.perf_counter()
    if _R is None:
        from oracle import luda_oracle as O
        O.reference_compact(_FILES)
    else:
        ref_compact(_R, _FILES)
    dt = time.perf_counter() - t0
    return sum(len(f) for f in _FILES), dt


def inline_throughput(shape, n_keys, workers, steps, warmup, seed=0xC3):
    """Reference compaction on `workers` processes (one sample job each):
    per step MB/s = all workers' input bytes / slowest worker. Returns
    (median MB/s, median entries/s, kind, per-step seconds)."""
    import multiprocessing as mp
    kind = "reference" if load_reference() is not None else "port"
    entries = 2 * n_keys if shape == "c3" else n_keys + max(1, n_keys // 9)
    vals, secs = [], []
    if workers <= 1:
        _init(shape, n_keys, seed)
        for i in range(warmup + steps):
            b, dt = _compact(0)
            if i >= warmup:
                vals.append((b / dt / 1e6, entries / dt))
                secs.append(dt)
    else:
        ctx = mp.get_context("fork")
        with ctx.Pool(workers, initializer=_init, initargs=(shape, n_keys, seed)) as pool:
            for i in range(warmup + steps):
                res = pool.map(_compact, range(workers), chunksize=1)
                t_max = max(r[1] for r in res)
                if i >= warmup:
                    vals.append((sum(r[0] for r in res) / t_max / 1e6, entries * workers / t_max))
                    secs.append(t_max)
    return statistics.median(v[0] for v in vals), statistics.median(v[1] for v in vals), kind, secs


def offload_throughput(shape, n_keys, steps, seed=0xC3):
    """The reference's offload path on its HostParallelDevice (cores - 2
    workers, bandwidth/latency model off). Returns (MB/s, entries/s, workers)."""
    R = load_reference()
    if R is None:
        return None
    files = sample_job(R, shape, n_keys, seed)
    cfg = R.config.DeviceConfig(backend="host_parallel", workers=0, bandwidth_bytes_per_sec=float("inf"),
                                latency_sec=0.0, region_capacity=1 << 40)
    dev = R.device.make_device(cfg)
    entries = 2 * n_keys if shape == "c3" else n_keys + max(1, n_keys // 9)
    try:
        want = ref_compact(R, files)
        got = ref_offload_compact(R, dev, files)
        assert got == want, "reference offload composition differs from the inline reference"
        ts = []
        for _ in range(steps):
            t0 = time.perf_counter()
            ref_offload_compact(R, dev, files)
            ts.append(time.perf_counter() - t0)
    finally:
        dev.close()
    dt = statistics.median(ts)
    return sum(len(f) for f in files) / dt / 1e6, entries / dt, cfg.effective_workers()
