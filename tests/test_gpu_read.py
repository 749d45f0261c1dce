"""GPU parity of the batched read path (paper_2004_03054_b200.read, through the
C ABI) against the oracle's Table.get restatement and the reference-frozen
goldens (tests/golden/reads.json): every lookup's outcome — entry bytes, None,
or the exception class and offset — plus the per-table counters."""

import json
import os
import random

import pytest

from oracle import jobgen
from oracle import luda_oracle as O
from tests.golden import read_cases as RC

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "reads.json")))


@pytest.fixture(scope="module")
def dev():
    from paper_2004_03054_b200 import DeviceConfig, make_device
    d = make_device(DeviceConfig(backend="b200"))
    yield d
    d.close()


def dev_outcome(mode, r):
    """Device per-key result → read_cases.encode form."""
    if isinstance(r, Exception):
        from paper_2004_03054_b200.read import _MSG, STRUCT_ERROR
        name = type(r).__name__
        if name == "FormatError" and str(r).startswith(_MSG[STRUCT_ERROR]):
            name = "struct.error"
        return RC.encode(mode, ("E", name, getattr(r, "offset", None)))
    return RC.encode(mode, ("ok", r))


def run_device(dev, c):
    from paper_2004_03054_b200.read import DeviceTables
    with DeviceTables(c["files"], dev) as T:
        if c["mode"] == "table":
            got = T.multi_get([q for _, q in c["queries"]], [t for t, _ in c["queries"]], errors_mode="return")
        else:
            T.set_levels(c["l0"], c["levels"])
            got = T.store_get([q for _, q in c["queries"]], errors_mode="return")
        rej, rd = T.counters()
    return [dev_outcome(c["mode"], r) for r in got], [[a, b] for a, b in zip(rej, rd)]


def oracle_run(c):
    tables = [O.MemTable(f) for f in c["files"]]
    enc = []
    for t, q in c["queries"]:
        if c["mode"] == "table":
            o = RC.outcome(lambda: tables[t].get(q))
        else:
            o = RC.outcome(lambda: O.store_get(tables, c["l0"], c["levels"], q))
        enc.append(RC.encode(c["mode"], o))
    return enc, [[tb.filter_rejects, tb.data_block_reads] for tb in tables]


@pytest.mark.parametrize("name", RC.READ_CASES)
def test_read_path_matches_oracle_and_golden(dev, name):
    c = RC.build(name)
    want, want_ctr = oracle_run(c)
    got, got_ctr = run_device(dev, c)
    bad = [(i, c["queries"][i], w, g) for i, (w, g) in enumerate(zip(want, got)) if w != g]
    assert not bad, bad[:5]
    assert got_ctr == want_ctr
    assert RC.summary(got) == GOLD[name]["results"]
    assert got_ctr == GOLD[name]["counters"]


def test_first_failing_lookup_raises(dev):
    """errors_mode="raise": the first failing key's exception, as a
    sequential loop of Table.get calls raises (sst.py:322-340)."""
    from paper_2004_03054_b200 import CorruptionError
    from paper_2004_03054_b200.read import DeviceTables
    c = RC.build("corrupt")
    tables = [O.MemTable(f) for f in c["files"]]
    first = None
    for t, q in c["queries"]:
        try:
            tables[t].get(q)
        except Exception as e:  # noqa: BLE001
            first = e
            break
    assert isinstance(first, O.CorruptionError)
    with DeviceTables(c["files"], dev) as T:
        with pytest.raises(CorruptionError) as ei:
            T.multi_get([q for _, q in c["queries"]], [t for t, _ in c["queries"]])
    assert ei.value.offset == first.offset


def test_open_errors_follow_table_init(dev):
    """A bad footer / filter CRC fails the open like Table.__init__ (sst.py:284-310)."""
    from paper_2004_03054_b200 import CorruptionError, FormatError
    from paper_2004_03054_b200.read import DeviceTables
    lower, _ = jobgen.materialize(jobgen.c3(n=800, seed=0x0E, sst_target=16 * 1024))
    bad = bytearray(lower[1])
    bad[-1] ^= 0xFF  # magic
    with pytest.raises(FormatError, match="bad magic"):
        DeviceTables([lower[0], bytes(bad)], dev)
    bad = bytearray(lower[0])
    foff = O.FOOTER.unpack_from(bytes(bad), len(bad) - 24)[0]
    bad[foff + 1] ^= 1
    with pytest.raises(CorruptionError) as ei:
        DeviceTables([bytes(bad)], dev)
    assert ei.value.offset == foff


def test_read_path_over_compaction_output_in_place(dev):
    """Open a GPU compaction's output buffer without copying and look up
    every survivor plus absent keys; compare with the oracle over the same
    bytes."""
    from paper_2004_03054_b200 import _native
    from paper_2004_03054_b200.read import DeviceTables
    job = jobgen.c3(n=20000, seed=0x3EAD, sst_target=64 * 1024)
    lower, upper = jobgen.materialize(job)
    files = lower + upper
    import ctypes
    L = dev._L
    sizes = [len(f) for f in files]
    offs, o = [], 0
    for s in sizes:
        offs.append(o)
        o += s
    region = dev.alloc(o + 64)
    blob = b"".join(files)
    buf = (ctypes.c_uint8 * len(blob)).from_buffer_copy(blob)
    st = dev.stream("rp")
    _native.check(L.luda_stage_in_async(region.dptr, buf, len(blob), st))
    jd = _native.JobDesc()
    jd.arena, jd.arena_bytes, jd.n_files = region.dptr, o, len(files)
    fo = (ctypes.c_uint64 * len(files))(*offs)
    fl = (ctypes.c_uint64 * len(files))(*sizes)
    jd.file_off, jd.file_len = fo, fl
    runs = (ctypes.c_uint32 * 3)(0, len(lower), len(files))
    jd.n_runs, jd.run_first_file = 2, runs
    jd.block_size, jd.restart_interval, jd.bits_per_key, jd.sst_size_target = 4096, 16, 10, 96 * 1024
    res = dev.compact(jd, stream="rp")
    try:
        host = (ctypes.c_uint8 * res.out_bytes)()
        _native.check(L.luda_stage_out_async(host, res.out, res.out_bytes, st))
        _native.check(L.luda_stream_sync(st))
        blob_out = bytes(host)
        outs = [blob_out[res.sst_off[i]:res.sst_off[i] + res.sst_len[i]] for i in range(res.n_sst)]
        mems = [O.MemTable(f) for f in outs]
        rng = random.Random(5)
        keys = []
        n_present = 0
        for t, f in enumerate(outs):
            _, index = O.open_table(f)
            ks = [k[:-8] for k, _ in O.scan_table(f, index)]
            keys += [(t, k) for k in rng.sample(ks, min(200, len(ks)))]
            n_present += min(200, len(ks))
            keys += [(t, rng.randbytes(16)) for _ in range(50)]
        with DeviceTables.from_job(dev, res) as T:
            got = T.multi_get([k for _, k in keys], [t for t, _ in keys])
        want = [mems[t].get(k) for t, k in keys]
        assert got == want
        assert sum(1 for g in got if g is not None) >= n_present
    finally:
        dev.release(res)
        dev.free(region)


def test_read_path_randomized_configs(dev):
    """Table.get over 120 random table sets (SPEC-A1 and mixed-length-key
    files under random block size / restart interval / bits per key), with
    present, absent, near-miss and prefix queries: every result equal to the
    oracle's, and the per-table counters too."""
    from paper_2004_03054_b200.read import DeviceTables
    rng = random.Random(0x6E7)
    for s in range(120):
        job = jobgen.spec_a1(3000 + s) if s % 2 == 0 else jobgen.varkey(500 + s, max_len=48, n_space=200)
        cfg = dict(block_size=rng.choice([256, 1024, 4096]), restart_interval=rng.choice([1, 2, 5, 16]),
                   bits_per_key=rng.choice([1, 4, 10, 16]))
        lower, upper = jobgen.materialize(job, **cfg)
        files = lower + upper
        c = {"files": files, "mode": "table"}
        qs = []
        for t, f in enumerate(files):
            qs += [(t, q) for q in RC._queries(rng, RC._user_keys(f), 40)]
        c["queries"] = qs
        want, want_ctr = oracle_run(c)
        got, got_ctr = run_device(dev, c)
        assert got == want, (s, cfg)
        assert got_ctr == want_ctr, (s, cfg)
