"""Key-range subcompactions across the GPUs of one box.

The reference compacts a job in one piece (multi-device is a SPEC non-goal,
SPEC.md:437); a compaction is, however, independent per user-key range, so
the B200 build shards a job into P fixed ranges:

1. every rank samples user keys from the INDEX blocks (the last key of each
   data block, sst.py:67-76 — no data-block decode) of the input files it is
   assigned for sampling (file i → rank i mod G);
2. the fixed-size sample arrays are all-gathered — the only collective of the
   path (NCCL on GPUs, gloo in the CPU tests);
3. every rank sorts the union and picks P − 1 splitters snapped to Li+1 file
   boundaries (smallest user keys of the target-level files), so each Li+1
   file lands in exactly one range; P does not depend on G and the sample
   union is the same for every G, hence 1/2/4/8-GPU runs produce identical
   ranges and identical output bytes;
4. ranges are dealt to ranks contiguously; a rank compacts each of its ranges
   with ``run_compaction(..., key_range=(lo, hi))``: the Li+1 files inside
   the range and the Li files overlapping it are staged, and records outside
   [lo, hi) are dropped on the device. No KV data crosses NVLink.

Parity: for every G the outputs equal the concatenation of reference
compactions run independently per range (``tests/test_subcompact.py``).
"""

from __future__ import annotations

import ctypes

import struct
from dataclasses import dataclass

from . import _native, errors
from .version import CompactionJob, user_key_of

FOOTER = struct.Struct("<IIIIQ")
SAMPLE_KEY_CAP = 256  # bytes of a user key carried in a sample row (splitter choice only)


def _varint(buf, pos):
    v = shift = 0
    while True:
        b = buf[pos]
        pos += 1
        v |= (b & 0x7F) << shift
        if not b & 0x80:
            return v, pos
        shift += 7


def index_user_keys(sst: bytes) -> list:
    """User keys of the index entries of one SST (block last keys, sst.py:67-76).

    Host-side footer + index parse only; the device verifies every CRC when
    the file is compacted."""
    if len(sst) < FOOTER.size:
        return []
    _, _, ioff, ilen, _ = FOOTER.unpack_from(sst, len(sst) - FOOTER.size)
    body = sst[ioff:ioff + ilen]
    if len(body) < 8:
        return []
    n = struct.unpack_from("<I", body, len(body) - 8)[0]
    out, pos = [], 0
    try:
        for _ in range(n):
            klen, pos = _varint(body, pos)
            out.append(user_key_of(bytes(body[pos:pos + klen])))
            pos += klen + 8
    except IndexError:
        return out
    return out


def sample_file(sst: bytes, per_file: int) -> list:
    """Evenly spaced index keys of one file (deterministic)."""
    keys = index_user_keys(sst)
    if len(keys) <= per_file:
        return keys
    step = len(keys) / per_file
    return [keys[int(i * step)] for i in range(per_file)]


def encode_samples(keys, rows: int) -> bytes:
    """Fixed-size sample array: rows × (u16 len ∥ key[:SAMPLE_KEY_CAP]); len
    0xFFFF marks an empty row."""
    w = 2 + SAMPLE_KEY_CAP
    out = bytearray(b"\xff\xff" + bytes(SAMPLE_KEY_CAP)) * rows
    for i, k in enumerate(keys[:rows]):
        k = k[:SAMPLE_KEY_CAP]
        struct.pack_into("<H", out, i * w, len(k))
        out[i * w + 2:i * w + 2 + len(k)] = k
    return bytes(out)


def decode_samples(buf: bytes) -> list:
    w = 2 + SAMPLE_KEY_CAP
    out = []
    for i in range(len(buf) // w):
        (n,) = struct.unpack_from("<H", buf, i * w)
        if n != 0xFFFF:
            out.append(bytes(buf[i * w + 2:i * w + 2 + n]))
    return out


def choose_splitters(samples, boundaries, nranges: int) -> list:
    """P − 1 ascending splitters. With Li+1 files, each splitter is the Li+1
    file boundary (a file's smallest user key) closest in sample rank to the
    ideal quantile; without, the quantile sample itself."""
    samples = sorted(samples)
    if nranges <= 1 or not samples:
        return []
    quant = [samples[min(len(samples) - 1, (p * len(samples)) // nranges)] for p in range(1, nranges)]
    if not boundaries:
        cand = quant
    else:
        import bisect
        bnd = sorted(set(boundaries))
        ranks = [bisect.bisect_left(samples, b) for b in bnd]
        cand = []
        for p, q in enumerate(quant, start=1):
            target = (p * len(samples)) // nranges
            i = min(range(len(bnd)), key=lambda j: (abs(ranks[j] - target), j))
            cand.append(bnd[i])
    out = []
    for c in cand:  # strictly ascending, duplicates dropped
        if not out or c > out[-1]:
            out.append(c)
    return out


def ranges_from_splitters(splitters):
    """[(lo, hi)] with None for an open end; ranges are [lo, hi)."""
    edges = [None] + list(splitters) + [None]
    return [(edges[i], edges[i + 1]) for i in range(len(edges) - 1)]


def ranges_of_rank(nranges: int, world: int, rank: int) -> list:
    """Contiguous deal of range indices to ranks."""
    lo = (nranges * rank) // world
    hi = (nranges * (rank + 1)) // world
    return list(range(lo, hi))


def _overlaps(meta, lo, hi) -> bool:
    """File's user-key span intersects [lo, hi)."""
    s, l = user_key_of(meta.smallest), user_key_of(meta.largest)
    return (hi is None or s < hi) and (lo is None or l >= lo)


def range_job(job: CompactionJob, lo, hi) -> CompactionJob:
    """The sub-job of [lo, hi): overlapping Li files, Li+1 files inside."""
    return CompactionJob(source_level=job.source_level,
                         lower=[m for m in job.lower if _overlaps(m, lo, hi)],
                         upper=[m for m in job.upper if _overlaps(m, lo, hi)],
                         target_level=job.target_level, version=job.version,
                         grandparents=list(job.grandparents))


@dataclass
class SplitPlan:
    splitters: list
    ranges: list            # [(lo, hi)]
    mine: list              # range indices of this rank


_COMMS: dict = {}


def _luda_comm(L, world: int, group):
    """The C-ABI NCCL communicator of this process group (luda_nccl_init_rank;
    rank 0's unique id travels over the launcher's process group)."""
    import torch.distributed as dist
    key = (id(group), world)
    c = _COMMS.get(key)
    if c is None:
        rank = dist.get_rank(group)
        uid = (ctypes.c_uint8 * 128)()
        if rank == 0:
            _native.check(L.luda_nccl_unique_id(uid))
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=0, group=group)
        uid = (ctypes.c_uint8 * 128).from_buffer_copy(obj[0])
        h = ctypes.c_void_p()
        _native.check(L.luda_nccl_init_rank(world, rank, uid, ctypes.byref(h)))
        c = _COMMS[key] = h.value
    return c


def allgather_bytes(payload: bytes, world: int, group=None) -> list:
    """All-gather equal-length byte strings. On GPUs
    (NCCL process group) through the C ABI's ``luda_allgather_splitters``
    over NVLink; on CPU process groups (gloo: the multi-process tests) through
    torch.distributed."""
    if world <= 1:
        return [payload]
    import torch
    import torch.distributed as dist
    backend = dist.get_backend(group)
    if backend == "nccl":
        n = len(payload)
        send = torch.frombuffer(bytearray(payload), dtype=torch.uint8).cuda()
        try:
            L = _native.lib(torch.cuda.current_device())
            comm = _luda_comm(L, world, group)
            recv = torch.empty(world * n, dtype=torch.uint8, device="cuda")
            s = torch.cuda.current_stream()
            _native.check(L.luda_allgather_splitters(comm, send.data_ptr(), recv.data_ptr(), n, s.cuda_stream))
            s.synchronize()
            blob = recv.cpu().numpy().tobytes()
            return [blob[i * n:(i + 1) * n] for i in range(world)]
        except errors.DeviceError as exc:  # the same NCCL collective through the process group instead
            import warnings
            warnings.warn(f"luda_allgather_splitters unavailable ({exc}); all-gather via torch.distributed")
            outs = [torch.empty_like(send) for _ in range(world)]
            dist.all_gather(outs, send, group=group)
            return [bytes(o.cpu().numpy().tobytes()) for o in outs]
    t = torch.frombuffer(bytearray(payload), dtype=torch.uint8)
    outs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(outs, t, group=group)
    return [bytes(o.numpy().tobytes()) for o in outs]


def plan_ranges(job: CompactionJob, inputs, *, nranges: int = 64, per_file: int = 64, world: int = 1,
                rank: int = 0, group=None) -> SplitPlan:
    """Steps 1–4 above: sample, all-gather, choose splitters, deal ranges."""
    files = list(job.lower) + list(job.upper)
    mine_files = files[rank::world]
    rows = ((len(files) + world - 1) // world) * per_file
    local = []
    for m in mine_files:
        local += sample_file(inputs[m.file_id], per_file)
    gathered = allgather_bytes(encode_samples(local, max(rows, 1)), world, group)
    samples = [k for g in gathered for k in decode_samples(g)]
    boundaries = [user_key_of(m.smallest) for m in sorted(job.upper, key=lambda m: m.smallest)[1:]]
    spl = choose_splitters(samples, boundaries, nranges)
    rngs = ranges_from_splitters(spl)
    return SplitPlan(splitters=spl, ranges=rngs, mine=ranges_of_rank(len(rngs), world, rank))


def run_subcompactions(job: CompactionJob, device, *, inputs, config=None, nranges: int = 64, per_file: int = 64,
                       world: int = 1, rank: int = 0, group=None, compact=None, new_file_id=None):
    """Plan the ranges (one all-gather) and compact this rank's ranges.

    Returns (plan, [(range_index, outputs, stats)]). ``compact`` defaults to
    ``run_compaction``; it receives (sub_job, device, inputs=, config=,
    key_range=, new_file_id=). One file-id allocator is shared by all ranges
    of this rank; without ``new_file_id`` the ranks draw interleaved ids
    above every file of the job's Version (rank r of G: r, r + G, ...), so
    no two outputs of the job share an id."""
    from .compaction import file_id_allocator
    if compact is None:
        from .compaction import run_compaction as compact
    new_file_id = file_id_allocator(job, new_file_id, stride=max(1, world), offset=rank)
    plan = plan_ranges(job, inputs, nranges=nranges, per_file=per_file, world=world, rank=rank, group=group)
    results = []
    for r in plan.mine:
        lo, hi = plan.ranges[r]
        sub = range_job(job, lo, hi)
        if not sub.lower and not sub.upper:
            results.append((r, [], None))
            continue
        outs, stats = compact(sub, device, inputs=inputs, config=config, key_range=(lo, hi), new_file_id=new_file_id)
        results.append((r, outs, stats))
    return plan, results
