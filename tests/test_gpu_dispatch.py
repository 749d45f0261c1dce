"""GPU parity of the per-kind dispatch path (kernels.py:72-168 on the
offload-device protocol, device.py:435-456): the CUDA work items through
``luda_dispatch`` vs the reference's SerialDevice digests (items.json) and
the oracle's restatement (``O.run_item``), bit-exact."""

import hashlib
import json
import os
import random

import pytest

from oracle import jobgen
from oracle import luda_oracle as O

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ITEMS = json.load(open(os.path.join(HERE, "golden", "items.json")))


def sha(b):
    return hashlib.sha256(bytes(b)).hexdigest()


@pytest.fixture(scope="module")
def dev():
    from paper_2004_03054_b200 import DeviceConfig, make_device
    d = make_device(DeviceConfig(backend="b200"))
    yield d
    d.close()


def region(dev, data=None, cap=None):
    r = dev.alloc(cap if cap is not None else len(data))
    if data is not None:
        dev.stage_in(r, data, "in_lower").wait()
    else:
        dev.stage_in(r, b"", "in_lower").wait()
    return r


def out(dev, r, n=None):
    return dev.stage_out(r, [(0, r.capacity if n is None else n)], "out").wait()


def test_dispatch_matches_reference_serial_device(dev):
    from paper_2004_03054_b200.device import KernelSpec
    job = jobgen.mixed(7, n_files=2, max_keys=300)
    files = [f for r in job.lower for f, _, _ in O.build_tables_split(r.pairs, sst_size_target=r.sst_target)]
    assert [sha(f) for f in files] == ITEMS["files"]
    d_unpack, d_sk, d_enc, d_filt = ITEMS["dispatches"]
    data = files[0]
    src = region(dev, data)
    gold_items = [tuple(x) for x in d_unpack["items"]]
    cap = sum(it[2] for it in gold_items) * 4
    pairs, tups = region(dev, cap=cap), region(dev, cap=cap)
    items = tuple((src.region_id, it[1], it[2], pairs.region_id, it[4], it[5], tups.region_id, it[7], it[8])
                  for it in gold_items)
    res = dev.dispatch(KernelSpec("unpack", items, reads=(src.region_id,),
                                  writes=(pairs.region_id, tups.region_id))).wait()
    assert [list(r) for r in res] == d_unpack["results"]
    assert sha(out(dev, pairs)) == d_unpack["pairs_sha"]
    assert sha(out(dev, tups)) == d_unpack["tuples_sha"]
    n = res[0][2]
    tb = res[0][1]
    lay = region(dev, cap=8 * n)
    sk = tuple((tups.region_id, x[1], x[2], x[3], lay.region_id, x[5]) for x in d_sk["items"])
    r2 = dev.dispatch(KernelSpec("shared_key", sk, reads=(tups.region_id,), writes=(lay.region_id,))).wait()
    assert [list(r) for r in r2] == d_sk["results"]
    assert sha(out(dev, lay)) == d_sk["out_sha"]
    outb = region(dev, cap=2 * 8192)
    enc = tuple((tups.region_id, x[1], x[2], lay.region_id, x[4], pairs.region_id, outb.region_id, x[7], x[8], x[9])
                for x in d_enc["items"])
    r3 = dev.dispatch(KernelSpec("encode", enc, reads=(tups.region_id, lay.region_id, pairs.region_id),
                                 writes=(outb.region_id,))).wait()
    assert [list(r) for r in r3] == d_enc["results"]
    assert sha(out(dev, outb)) == d_enc["out_sha"]
    fo = region(dev, cap=4096)
    r4 = dev.dispatch(KernelSpec("filter", ((tups.region_id, 0, tb, 10, fo.region_id, 0, 4096),),
                                 reads=(tups.region_id,), writes=(fo.region_id,))).wait()
    assert [list(r) for r in r4] == d_filt["results"]
    assert sha(out(dev, fo)) == d_filt["out_sha"]
    dev.free_all()


@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5])
def test_dispatch_random_jobs_vs_oracle(dev, seed):
    """All four kinds on random jobs (variable key/value lengths, odd restart
    intervals and bits-per-key), every region byte compared with the oracle."""
    from paper_2004_03054_b200.device import KernelSpec
    rng = random.Random(seed)
    job = jobgen.mixed(seed, n_files=1, max_keys=400)
    data = [f for r in job.lower for f, _, _ in O.build_tables_split(r.pairs, sst_size_target=r.sst_target)][0]
    _, index = O.open_table(data)
    cap = sum(ln for _, _, ln in index) * 4 + 64
    R = {}  # oracle regions by our region id
    src = region(dev, data)
    pairs, tups = region(dev, cap=cap), region(dev, cap=cap)
    R[src.region_id], R[pairs.region_id], R[tups.region_id] = bytearray(data), bytearray(cap), bytearray(cap)
    items, slot = [], 0
    for _, off, ln in index:
        items.append((src.region_id, off, ln, pairs.region_id, slot, 4 * ln, tups.region_id, slot, 4 * ln))
        slot += 4 * ln
    want = [O.run_item("unpack", it, R) for it in items]
    got = dev.dispatch(KernelSpec("unpack", tuple(items), reads=(src.region_id,),
                                  writes=(pairs.region_id, tups.region_id))).wait()
    assert [tuple(g) for g in got] == [tuple(w[1]) for w in want]
    assert out(dev, pairs) == bytes(R[pairs.region_id]) and out(dev, tups) == bytes(R[tups.region_id])
    # shared_key / encode / filter over each unpacked block's tuples, odd knobs
    ri = rng.choice([1, 3, 16, 5])
    bpk = rng.choice([1, 7, 10, 13])
    eslot = [2 * ln + 4096 for _, _, ln in index]
    fslot = [2 * ln + 4096 for _, _, ln in index]
    lay = region(dev, cap=cap)
    outb = region(dev, cap=sum(eslot))
    fo = region(dev, cap=sum(fslot) + 8)
    for r in (lay, outb, fo):
        R[r.region_id] = bytearray(r.capacity)
    sk, enc, flt = [], [], []
    eo = fo_ = 0
    for i, (it, w) in enumerate(zip(items, want)):
        t0, t1 = it[7], it[7] + w[1][1]
        sk.append((tups.region_id, t0, t1, ri, lay.region_id, t0 // 2))
        enc.append((tups.region_id, t0, t1, lay.region_id, t0 // 2, pairs.region_id, outb.region_id,
                    eo, eslot[i], ri))
        flt.append((tups.region_id, t0, t1, bpk, fo.region_id, fo_ + (i % 3), fslot[i] - 3))
        eo += eslot[i]
        fo_ += fslot[i]
    for kind, its, reads, writes in (("shared_key", sk, (tups.region_id,), (lay.region_id,)),
                                     ("encode", enc, (tups.region_id, lay.region_id, pairs.region_id),
                                      (outb.region_id,)),
                                     ("filter", flt, (tups.region_id,), (fo.region_id,))):
        want_k = [O.run_item(kind, x, R) for x in its]
        assert all(w[0] == "ok" for w in want_k)
        got_k = dev.dispatch(KernelSpec(kind, tuple(its), reads=reads, writes=writes)).wait()
        assert [tuple(g) for g in got_k] == [tuple(w[1]) for w in want_k], kind
        for rid in writes:
            r = [x for x in (lay, outb, fo) if x.region_id == rid][0]
            assert out(dev, r) == bytes(R[rid]), kind
    dev.free_all()


def test_dispatch_errors_first_item_wins(dev):
    from paper_2004_03054_b200 import CorruptionError, DeviceError
    from paper_2004_03054_b200.device import KernelSpec
    pairs_ = [(O.make_ikey(b"key%05d" % i, i + 1, 1), b"v" * 50) for i in range(300)]
    data = bytearray(O.build_table(pairs_))
    _, index = O.open_table(bytes(data))
    off2 = index[2][1]
    data[off2 + 5] ^= 0x10  # corrupt block 2
    src = region(dev, bytes(data))
    cap = sum(ln for _, _, ln in index) * 4
    p, t = region(dev, cap=cap), region(dev, cap=cap)
    items, slot = [], 0
    for _, off, ln in index:
        items.append((src.region_id, off, ln, p.region_id, slot, 4 * ln, t.region_id, slot, 4 * ln))
        slot += 4 * ln
    h = dev.dispatch(KernelSpec("unpack", tuple(items), reads=(src.region_id,), writes=(p.region_id, t.region_id)))
    with pytest.raises(CorruptionError) as ei:
        h.wait()
    assert ei.value.offset == off2
    assert all(r is not None for r in h.results[:2]) and h.results[2] is None
    # a slot overflow (BufferError in the reference) is a DeviceError
    small = ((src.region_id, index[0][1], index[0][2], p.region_id, 0, 10, t.region_id, 0, 4 * index[0][2]),)
    with pytest.raises(DeviceError):
        dev.dispatch(KernelSpec("unpack", small, reads=(src.region_id,), writes=(p.region_id, t.region_id))).wait()
    dev.free_all()


def test_dispatch_is_asynchronous_with_ordered_callbacks(dev):
    """HostParallelDevice semantics (device.py:566-607): dispatch returns a
    handle at once, a collector thread calls on_item in item order, done()
    turns true and wait() returns the per-item results; written regions are
    FILLING until completion, READY after; back-to-back dispatches run in
    submission order."""
    import threading

    from paper_2004_03054_b200.device import READY, KernelSpec
    job = jobgen.c3(n=2000, seed=0xA5, sst_target=64 * 1024)
    lower, _ = jobgen.materialize(job)
    data = lower[0]
    _, index = O.open_table(data)
    src = region(dev, data)
    cap = sum(ln for _, _, ln in index) * 4
    p, t = region(dev, cap=cap), region(dev, cap=cap)
    items, slot = [], 0
    for _, off, ln in index:
        items.append((src.region_id, off, ln, p.region_id, slot, 4 * ln, t.region_id, slot, 4 * ln))
        slot += 4 * ln
    seen, tids = [], set()

    def on_item(i, r):
        seen.append(i)
        tids.add(threading.get_ident())

    h1 = dev.dispatch(KernelSpec("unpack", tuple(items), reads=(src.region_id,),
                                 writes=(p.region_id, t.region_id)), on_item=on_item)
    res1 = h1.wait(timeout=60)
    assert h1.done()
    assert seen == list(range(len(items)))
    assert threading.get_ident() not in tids  # called from the collector thread
    assert all(r is not None for r in res1)
    assert p.state == READY and t.region_id in dev._regions
    # two dispatches in flight: results equal a sequential run
    h2 = dev.dispatch(KernelSpec("unpack", tuple(items), reads=(src.region_id,), writes=(p.region_id, t.region_id)))
    h3 = dev.dispatch(KernelSpec("unpack", tuple(items), reads=(src.region_id,), writes=(p.region_id, t.region_id)))
    assert h2.wait(timeout=60) == res1 and h3.wait(timeout=60) == res1
    dev.free_all()
