"""BASELINE config 5 planning (bench_c5.py) on CPU: the global
job's generator is range-decomposable and the plan — index-style samples of
each rank's files, all-gather (gloo, world size 2), splitters snapped to Li+1
file boundaries, contiguous deal — is identical for every world size."""

import os
import socket

import torch
import torch.multiprocessing as mp

import bench_c5 as C

SPEC = dict(total_gb=0.05, nbuckets=16, file_keys=2000, nranges=8)
ODD = dict(total_gb=0.02, nbuckets=8, file_keys=1500, nranges=6)  # odd file counts in both levels


def test_generator_files_sorted_and_disjoint():
    spec = C.C5Spec(**SPEC)
    sy = C.Synth(spec, torch.device("cpu"))
    for level in ("up", "lo"):
        b = C.file_bounds(spec, sy, level)
        assert all(f[0] <= f[1] for f in b)
        assert all(b[i][1] < b[i + 1][0] for i in range(len(b) - 1))
    # the same bucket regenerated is bit-identical (any rank can synthesise any file)
    b1 = C.gen_bucket(spec, 3, torch.device("cpu"))
    b2 = C.gen_bucket(spec, 3, torch.device("cpu"))
    assert torch.equal(b1.up_hi, b2.up_hi) and torch.equal(b1.lo_lo, b2.lo_lo)
    # Li overwrites are Li+1 keys; Li fresh keys are not
    up = set(zip(b1.up_hi.tolist(), b1.up_lo.tolist()))
    lo = list(zip(b1.lo_hi.tolist(), b1.lo_lo.tolist()))
    assert sum(k in up for k in lo) == spec.ow_per_bucket


def test_plan_every_upper_file_in_one_range():
    spec = C.C5Spec(**SPEC)
    sy = C.Synth(spec, torch.device("cpu"))
    ranges, mine, _, _, _ = C.plan(spec, sy, 1, 0)
    assert len(ranges) == spec.nranges and mine == list(range(spec.nranges))
    for s, l in C.file_bounds(spec, sy, "up"):
        assert sum(1 for lo, hi in ranges if (hi is None or s < hi) and (lo is None or l >= lo)) == 1


def _worker(rank, world, port, q, kw):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    spec = C.C5Spec(**kw)
    ranges, mine, _, _, _ = C.plan(spec, C.Synth(spec, torch.device("cpu")), world, rank)
    q.put((rank, [(a.hex() if a else None, b.hex() if b else None) for a, b in ranges], mine))
    dist.barrier()
    dist.destroy_process_group()


import pytest


@pytest.mark.parametrize("kw", [SPEC, ODD])
def test_plan_identical_for_world_1_and_2(kw):
    spec = C.C5Spec(**kw)
    r1, _, _, _, _ = C.plan(spec, C.Synth(spec, torch.device("cpu")), 1, 0)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q, kw)) for r in range(2)]
    for p in ps:
        p.start()
    got = sorted(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(60)
    want = [(a.hex() if a else None, b.hex() if b else None) for a, b in r1]
    assert got[0][1] == want and got[1][1] == want
    assert got[0][2] + got[1][2] == list(range(len(want)))
