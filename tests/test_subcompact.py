"""Key-range subcompactions: splitter sampling, the sample
all-gather (gloo, world size 2, CPU), range planning, and partition parity
against the per-range reference compaction (the oracle)."""

import os
import socket

import pytest
import torch.multiprocessing as mp

from oracle import jobgen
from oracle import luda_oracle as O
from paper_2004_03054_b200 import subcompact as SC
from paper_2004_03054_b200.version import CompactionJob, SstMeta, Version


def job_with_inputs(n=4000, seed=0xE5, sst_target=48 * 1024):
    spec = jobgen.c3(n=n, seed=seed, sst_target=sst_target)
    lower, upper = jobgen.materialize(spec)
    inputs, metas, fid = {}, [], 1
    for level, files in ((1, lower), (2, upper)):
        ms = []
        for f in files:
            _, index = O.open_table(f)
            first = next(iter(O.scan_table(f, index)))[0]
            ms.append(SstMeta(file_id=fid, file_size=len(f), smallest=first, largest=index[-1][0], level=level))
            inputs[fid] = f
            fid += 1
        metas.append(ms)
    job = CompactionJob(source_level=1, lower=metas[0], upper=metas[1], target_level=2, version=Version.empty())
    return job, inputs


def oracle_compact(sub, device, *, inputs, config=None, key_range=None, new_file_id=None):
    files = [inputs[m.file_id] for m in sub.lower + sub.upper]
    return O.reference_compact(files, sst_size_target=64 * 1024, key_range=key_range), None


def survivors(outs):
    got = []
    for data, _, _ in outs:
        _, idx = O.open_table(data)
        got += list(O.scan_table(data, idx))
    return got


def test_partition_parity_with_oracle():
    job, inputs = job_with_inputs()
    plan, res = SC.run_subcompactions(job, None, inputs=inputs, nranges=8, compact=oracle_compact)
    assert len(plan.ranges) == len(plan.splitters) + 1 and len(plan.ranges) > 1
    # every Li+1 file lands in exactly one range
    for m in job.upper:
        assert sum(1 for lo, hi in plan.ranges if SC._overlaps(m, lo, hi)) == 1
    # concatenated per-range outputs hold exactly the global compaction's entries
    files = [inputs[m.file_id] for m in job.lower + job.upper]
    want = survivors(O.reference_compact(files, sst_size_target=64 * 1024))
    got = []
    for _, outs, _ in sorted(res):
        got += survivors(outs)
    assert got == want
    # and no output SST spans a splitter
    for r, outs, _ in res:
        lo, hi = plan.ranges[r]
        for _, smallest, largest in outs:
            assert (lo is None or O.ukey(smallest) >= lo) and (hi is None or O.ukey(largest) < hi)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        job, inputs = job_with_inputs()
        plan, res = SC.run_subcompactions(job, None, inputs=inputs, nranges=8, world=world, rank=rank,
                                          compact=oracle_compact)
        q.put((rank, plan.splitters, plan.mine, [(r, [o[0] for o in outs]) for r, outs, _ in res]))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_matches_world1():
    """Splitters do not depend on the GPU count: the world-size-2 run (sample
    all-gather over gloo) chooses the world-size-1 splitters, deals the ranges
    contiguously, and yields byte-identical per-range outputs."""
    job, inputs = job_with_inputs()
    plan1, res1 = SC.run_subcompactions(job, None, inputs=inputs, nranges=8, compact=oracle_compact)
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get() for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    got.sort()
    assert all(g[1] == plan1.splitters for g in got)
    mine = [r for g in got for r in g[2]]
    assert mine == list(range(len(plan1.ranges)))
    by_range = {r: outs for g in got for r, outs in g[3]}
    for r, outs, _ in res1:
        assert by_range[r] == [o[0] for o in outs]


def test_sample_array_roundtrip():
    keys = [b"a", b"", b"\x00" * 300, b"zz"]
    enc = SC.encode_samples(keys, 6)
    assert len(enc) == 6 * (2 + SC.SAMPLE_KEY_CAP)
    assert SC.decode_samples(enc) == [b"a", b"", b"\x00" * SC.SAMPLE_KEY_CAP, b"zz"]
    assert SC.ranges_of_rank(10, 4, 0) == [0, 1] and SC.ranges_of_rank(10, 4, 3) == [7, 8, 9]
