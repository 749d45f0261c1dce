"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle.

Bit-exact comparisons only (all of this is integer/byte work)."""

import ctypes
import hashlib
import json
import os
import random
import zlib

import pytest

from oracle import jobgen
from oracle import luda_oracle as O
from tests.golden.cases import ALL_CASES, CASES, EDGE_CASES, FULL_CASES, SPEC_A1_CASES, VARKEY_CASES

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "compaction.json")))


def sha(b):
    return hashlib.sha256(bytes(b)).hexdigest()


@pytest.fixture(scope="module")
def dev():
    from paper_2004_03054_b200 import DeviceConfig, make_device
    d = make_device(DeviceConfig(backend="b200"))
    yield d
    d.close()


@pytest.fixture(scope="module")
def native():
    from paper_2004_03054_b200 import _native
    return _native.lib(0)


def gpu_crc(native, data: bytes, pad_front=0):
    p = ctypes.c_void_p()
    assert native.luda_region_alloc(len(data) + pad_front + 64, ctypes.byref(p)) == 0
    try:
        buf = ctypes.create_string_buffer(bytes(pad_front) + data, len(data) + pad_front)
        assert native.luda_stage_in_async(p.value, buf, len(data) + pad_front, None) == 0
        out = ctypes.c_uint32()
        assert native.luda_crc32(p.value + pad_front, len(data), ctypes.byref(out), None) == 0
        return out.value
    finally:
        native.luda_region_free(p.value)


def test_crc32_kat_and_random(native):
    assert gpu_crc(native, b"123456789") == 0xCBF43926
    assert gpu_crc(native, b"") == 0
    rng = random.Random(7)
    for n in (1, 2, 3, 4, 5, 7, 8, 131, 132, 133, 263, 264, 265, 1000, 4095, 4096, 4223, 4224, 4225, 8448,
              4607, 4608, 4609, 9216, 13824,
              10025, 65537, 1 << 20, (1 << 22) + 3):
        for pad in (0, 1, 3, 13):
            b = rng.randbytes(n)
            assert gpu_crc(native, b, pad) == zlib.crc32(b), (n, pad)


def test_crc32_batch_many_ranges(native):
    """luda_crc32_batch ((range, pass) work items over all warps) vs zlib on
    ranges of every size class, unaligned offsets, empty and 1-3 byte ranges."""
    import numpy as np
    rng = random.Random(11)
    lens = [0, 1, 2, 3, 4, 5, 9, 4607, 4608, 4609, 9216, 33000, 34011, 100003] + \
        [rng.randrange(0, 70000) for _ in range(300)]
    blob = bytearray()
    offs = []
    for n in lens:
        blob += bytes(rng.randrange(0, 16))  # misalign the next range
        offs.append(len(blob))
        blob += rng.randbytes(n)
    p = ctypes.c_void_p()
    assert native.luda_region_alloc(len(blob) + 64, ctypes.byref(p)) == 0
    try:
        buf = ctypes.create_string_buffer(bytes(blob), len(blob))
        assert native.luda_stage_in_async(p.value, buf, len(blob), None) == 0
        import torch
        d_off = torch.tensor(offs, dtype=torch.int64, device="cuda")
        d_len = torch.tensor(lens, dtype=torch.int32, device="cuda")
        d_out = torch.zeros(len(lens), dtype=torch.int32, device="cuda")
        torch.cuda.synchronize()
        c_u64p, c_u32p = ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint32)
        assert native.luda_crc32_batch(p.value, ctypes.cast(d_off.data_ptr(), c_u64p),
                                       ctypes.cast(d_len.data_ptr(), c_u32p), len(lens),
                                       ctypes.cast(d_out.data_ptr(), c_u32p), None) == 0
        torch.cuda.synchronize()
        got = d_out.cpu().numpy().astype(np.uint32).tolist()
        want = [zlib.crc32(bytes(blob[o:o + n])) for o, n in zip(offs, lens)]
        assert got == want
    finally:
        native.luda_region_free(p.value)


def build(name):
    mk, out_cfg = {n: (m, c) for n, m, c in ALL_CASES}[name]
    job = mk()
    blk = {k: out_cfg[k] for k in ("block_size", "restart_interval") if k in out_cfg}
    lower, upper = jobgen.materialize(job, **blk)
    return job, lower, upper, out_cfg


def gpu_compact(dev, job, lower, upper, out_cfg, **kw):
    from paper_2004_03054_b200.compaction import compact_files
    from paper_2004_03054_b200.config import StoreConfig
    cfg = StoreConfig(**{k: out_cfg[k] for k in ("block_size", "restart_interval", "sst_size_target",
                                                 "bits_per_key") if k in out_cfg})
    return compact_files(dev, lower, upper, source_level=job.source_level, deeper=job.deeper, config=cfg, **kw)


def check_case(dev, name):
    job, lower, upper, out_cfg = build(name)
    want = O.reference_compact(lower + upper, deeper=job.deeper, **out_cfg)
    got = gpu_compact(dev, job, lower, upper, out_cfg)
    assert len(got) == len(want)
    for (gb, gs, gl), (wb, ws, wl) in zip(got, want):
        assert gs == ws and gl == wl
        assert gb == wb
    assert [sha(b) for b, _, _ in got] == [o["sha256"] for o in GOLD[name]["outputs"]]


FIXED_KEY_CASES = CASES + FULL_CASES + EDGE_CASES + SPEC_A1_CASES


@pytest.mark.parametrize("name", [n for n, _, _ in FIXED_KEY_CASES])
def test_compaction_matches_oracle_and_golden(dev, name):
    check_case(dev, name)


@pytest.fixture
def small_planner_tiles(native):
    """Greedy-chain planner tiles of 32 items (LUDA_OPT_PLANNER_TILE): every
    job's block cut and SST cut then compose over many tiles and groups."""
    from paper_2004_03054_b200 import _native
    _native.check(native.luda_set_option(_native.OPT_PLANNER_TILE, 32))
    yield
    _native.check(native.luda_set_option(_native.OPT_PLANNER_TILE, 8192))


@pytest.mark.parametrize("name", [n for n, _, _ in CASES + FULL_CASES + EDGE_CASES[2:] + SPEC_A1_CASES[:40]])
def test_compaction_multitile_planner(dev, small_planner_tiles, name):
    check_case(dev, name)


@pytest.fixture(params=[(1, 1 << 24), (1, 3), (2, 7)], ids=["1cta-1blk", "1cta-3chunks", "2cta-7chunks"])
def decode_chunks(request, native):
    """Decode work distribution forced small (LUDA_OPT_DEC_CTAS / _SEGS): one
    CTA with one block per chunk makes each of its 12 pairs switch chunks
    many times on a small job; 3 or 7 long chunks leave most pairs idle."""
    from paper_2004_03054_b200 import _native
    ctas, segs = request.param
    _native.check(native.luda_set_option(_native.OPT_DEC_CTAS, ctas))
    _native.check(native.luda_set_option(_native.OPT_DEC_SEGS, segs))
    yield
    _native.check(native.luda_set_option(_native.OPT_DEC_CTAS, 0))
    _native.check(native.luda_set_option(_native.OPT_DEC_SEGS, 0))


@pytest.mark.parametrize("name", [n for n, _, _ in CASES + EDGE_CASES + VARKEY_CASES[:6] + SPEC_A1_CASES[:12]])
def test_compaction_decode_chunking(dev, decode_chunks, name):
    check_case(dev, name)


def test_flush_builder_matches_oracle(native):
    from paper_2004_03054_b200.flush import build_ssts
    rng = random.Random(11)
    keys = sorted({rng.randbytes(16) for _ in range(5000)})
    pairs = []
    seq = 1
    for k in keys:
        for _ in range(rng.choice((1, 1, 1, 2, 3))):  # several versions per user key
            pairs.append((O.make_ikey(k, seq, O.KIND_PUT if rng.random() < 0.9 else O.KIND_DELETE),
                          rng.randbytes(rng.randint(0, 300))))
            seq += 1
    pairs.sort(key=lambda kv: O.order_key(kv[0]))
    for cfg in (dict(sst_size_target=64 * 1024), dict(sst_size_target=2**31, block_size=1024, restart_interval=3)):
        want = O.build_tables_split(pairs, **cfg)
        got = build_ssts(pairs, **cfg)
        assert [g[0] for g in got] == [w[0] for w in want]
        assert [(g[1], g[2]) for g in got] == [(w[1], w[2]) for w in want]


@pytest.mark.parametrize("max_len", [64, 200])
def test_flush_builder_generic_key_lengths(native, max_len):
    """The L0 flush builder for a memtable whose user keys differ in length
    (0..max_len bytes, prefix-rich; several versions per key) and for fixed
    keys longer than 32 bytes: byte-identical to SstBuilder."""
    from paper_2004_03054_b200.flush import build_ssts
    rng = random.Random(max_len)
    job = jobgen.varkey(max_len, max_len=max_len, n_space=600, n_files=3)
    pairs = sorted((kv for r in job.lower for kv in r.pairs), key=lambda kv: O.order_key(kv[0]))
    for cfg in (dict(sst_size_target=16 * 1024), dict(sst_size_target=2**31, block_size=1024, restart_interval=3)):
        want = O.build_tables_split(pairs, **cfg)
        got = build_ssts(pairs, **cfg)
        assert [g[0] for g in got] == [w[0] for w in want]
        assert [(g[1], g[2]) for g in got] == [(w[1], w[2]) for w in want]
    fixed = sorted(((O.make_ikey(rng.randbytes(48), i + 1, O.KIND_PUT), rng.randbytes(50)) for i in range(2000)),
                   key=lambda kv: O.order_key(kv[0]))
    want = O.build_tables_split(fixed, sst_size_target=32 * 1024)
    assert [g[0] for g in build_ssts(fixed, sst_size_target=32 * 1024)] == [w[0] for w in want]


def _corrupt_case():
    job = jobgen.c3(n=2000, seed=5, sst_target=32 * 1024)
    lower, upper = jobgen.materialize(job)
    return job, lower, upper


def test_corruption_reports_block_offset(dev):
    from paper_2004_03054_b200 import CorruptionError
    job, lower, upper = _corrupt_case()
    _, index = O.open_table(upper[1])
    off = index[3][1]
    bad = bytearray(upper[1])
    bad[off + 7] ^= 0x40
    upper = list(upper)
    upper[1] = bytes(bad)
    with pytest.raises(O.CorruptionError) as want:
        O.reference_compact(lower + upper)
    with pytest.raises(CorruptionError) as got:
        gpu_compact(dev, job, lower, upper, {})
    assert got.value.offset == want.value.offset == off


@pytest.mark.parametrize("mutate,exc", [
    (lambda f: f[:-1] + bytes([f[-1] ^ 1]), "FormatError"),          # bad magic
    (lambda f: f[:10], "FormatError"),                                 # too short
])
def test_format_errors(dev, mutate, exc):
    import paper_2004_03054_b200 as P
    job, lower, upper = _corrupt_case()
    lower = list(lower)
    lower[0] = mutate(lower[0])
    with pytest.raises(getattr(O, exc)):
        O.reference_compact(lower + upper)
    with pytest.raises(getattr(P, exc)):
        gpu_compact(dev, job, lower, upper, {})


def test_subcompactions_match_per_range_oracle(dev):
    """Key-range subcompactions on the GPU vs the per-range
    reference compaction, byte for byte, range by range."""
    from paper_2004_03054_b200 import subcompact as SC
    from paper_2004_03054_b200.config import StoreConfig
    from tests.test_subcompact import job_with_inputs
    job, inputs = job_with_inputs()
    cfg = StoreConfig(sst_size_target=64 * 1024)
    plan, res = SC.run_subcompactions(job, dev, inputs=inputs, config=cfg, nranges=8)
    assert len(res) == len(plan.ranges) > 1
    for r, outs, _ in res:
        lo, hi = plan.ranges[r]
        sub = SC.range_job(job, lo, hi)
        want = O.reference_compact([inputs[m.file_id] for m in sub.lower + sub.upper],
                                   sst_size_target=64 * 1024, key_range=(lo, hi))
        assert [o[0] for o in outs] == [w[0] for w in want], r


def _unchecked_table(pairs, **cfg):
    """An SST whose entries are NOT in order: the oracle builder with its
    ascending check bypassed (the reference's SstBuilder would refuse)."""
    b = O.TableBuilder(**cfg)
    for k, v in pairs:
        b.last_order = None
        b.add(k, v)
    return b.finish()


def test_level_run_with_overlapping_files_merges_per_file(dev):
    """A level >= 1 run whose files overlap (every file seam out of order),
    each file spanning many merge tiles: the seams are found before merging
    and the run is merged per file, like the reference's per-file heap merge."""
    rng = random.Random(0x5EA)
    files = []
    seq = 1
    for f in range(3):
        keys = sorted({rng.randbytes(16) for _ in range(6000)})
        pairs = []
        for k in keys:
            pairs.append((O.make_ikey(k, seq, O.KIND_PUT), rng.randbytes(rng.randint(0, 64))))
            seq += 1
        files.append(O.build_table(pairs, sst_size_target=2**31))
    files.reverse()  # newest first
    want = O.reference_compact(files, sst_size_target=256 * 1024)
    from paper_2004_03054_b200.compaction import compact_files
    from paper_2004_03054_b200.config import StoreConfig
    got = compact_files(dev, files, [], source_level=1, config=StoreConfig(sst_size_target=256 * 1024))
    assert [g[0] for g in got] == [w[0] for w in want]


@pytest.mark.parametrize("where", ["start", "middle", "end"])
def test_unsorted_file_raises_ordering_error(dev, where):
    """Order violations inside a file (many merge tiles) are OrderingErrors,
    never out-of-bounds tile loads (merge-path splits are monotone only over
    sorted runs)."""
    from paper_2004_03054_b200 import OrderingError
    from paper_2004_03054_b200.compaction import compact_files
    rng = random.Random({"start": 1, "middle": 2, "end": 3}[where])
    keys = sorted({rng.randbytes(16) for _ in range(20000)})
    pairs = [(O.make_ikey(k, i + 1, O.KIND_PUT), rng.randbytes(20)) for i, k in enumerate(keys)]
    i = {"start": 10, "middle": 9000, "end": len(pairs) - 30}[where]
    pairs[i:i + 20] = pairs[i:i + 20][::-1]
    bad = _unchecked_table(pairs, sst_size_target=2**31)
    other = O.build_table(sorted(((O.make_ikey(rng.randbytes(16), 10**6 + j, O.KIND_PUT), b"x")
                                  for j in range(5000)), key=lambda kv: O.order_key(kv[0])), sst_size_target=2**31)
    with pytest.raises(O.OrderingError):
        O.reference_compact([bad, other])
    with pytest.raises(OrderingError):
        compact_files(dev, [bad], [other], source_level=1)
    with pytest.raises(OrderingError):
        compact_files(dev, [other, bad], [], source_level=0)
    # the device stays usable afterwards
    job, lower, upper, out_cfg = build("c3_small")
    got = gpu_compact(dev, job, lower, upper, out_cfg)
    assert [sha(b) for b, _, _ in got] == [o["sha256"] for o in GOLD["c3_small"]["outputs"]]


def _reseal_block(f: bytes, block_index: int, mutate) -> bytes:
    """Mutate one data block's payload and recompute its CRC (blocks.py:99-103),
    so the block passes verification and reaches the entry parser."""
    import struct
    _, index = O.open_table(f)
    _, off, ln = index[block_index]
    body = bytearray(f[off:off + ln - 4])
    mutate(body)
    out = bytearray(f)
    out[off:off + ln - 4] = body
    struct.pack_into("<I", out, off + ln - 4, zlib.crc32(bytes(body)))
    return bytes(out)


@pytest.mark.parametrize("kind", ["filter", "index"])
def test_filter_and_index_crc_corruption(dev, kind):
    """Table.__init__ checks (sst.py:293-306): a flipped bit in the filter or
    the index block is a CorruptionError at that block's offset."""
    from paper_2004_03054_b200 import CorruptionError
    job, lower, upper = _corrupt_case()
    f = bytearray(upper[2])
    foff, flen, ioff, ilen, _ = O.FOOTER.unpack_from(f, len(f) - O.FOOTER_SIZE)
    pos = foff + 5 if kind == "filter" else ioff + 3
    f[pos] ^= 0x10
    upper = list(upper)
    upper[2] = bytes(f)
    with pytest.raises(O.CorruptionError) as want:
        O.reference_compact(lower + upper)
    with pytest.raises(CorruptionError) as got:
        gpu_compact(dev, job, lower, upper, {})
    assert got.value.offset == want.value.offset == (foff if kind == "filter" else ioff)


def _damage_block(body, damage):
    import struct
    n = len(body)
    n_restarts = struct.unpack_from("<I", body, n - 4)[0]
    entries_end = n - 4 - 4 * n_restarts
    shared, p = O.varint_read(body, 0)
    unshared, p = O.varint_read(body, p)
    vstart = p
    vlen, p = O.varint_read(body, p)
    first_end = p + unshared + vlen
    if damage == "varint_long":        # an 11-byte varint: shift > 63 (varint.py:42-43)
        body[0:11] = b"\x80" * 10 + b"\x01"
    elif damage == "entry_trunc":      # value runs past the entries region
        body[vstart:vstart + 2] = O.varint_bytes(16000)
    elif damage == "shared_too_long":  # second entry shares more than the previous key's length
        body[first_end] = 60
    elif damage == "restarts_zero":    # n_restarts must be >= 1
        struct.pack_into("<I", body, n - 4, 0)
    else:                              # restart array larger than the block
        struct.pack_into("<I", body, n - 4, n)


@pytest.mark.parametrize("damage", ["varint_long", "entry_trunc", "shared_too_long", "restarts_zero", "restarts_huge"])
def test_block_entry_format_errors(dev, damage):
    """Structural errors inside a CRC-valid data block (blocks.py:137-164,
    varint.py:28-43) are FormatErrors with the reference's message. (The
    'truncated varint' and 'trailing garbage' branches of decode_data_block
    cannot fire on a block whose restart count is valid: the count's high
    byte would have to be >= 0x80.)"""
    import paper_2004_03054_b200 as P
    job, lower, upper = _corrupt_case()
    upper = list(upper)
    upper[1] = _reseal_block(upper[1], 2, lambda body: _damage_block(body, damage))
    with pytest.raises((O.FormatError, O.CorruptionError)) as want:
        O.reference_compact(lower + upper)
    with pytest.raises((P.FormatError, P.CorruptionError)) as got:
        gpu_compact(dev, job, lower, upper, {})
    assert type(got.value).__name__ == type(want.value).__name__, (got.value, want.value)
    assert str(want.value) in str(got.value)


@pytest.mark.parametrize("name", [n for n, _, _ in VARKEY_CASES])
def test_generic_key_lengths(dev, name):
    """Mixed user-key lengths (0..64 B, prefixes of each other, bytes that
    collide with trailer bytes) and fixed lengths > 32 B: the generic-length
    record path (luda_rec.cuh kVarW) vs the oracle and the reference goldens."""
    check_case(dev, name)


@pytest.mark.parametrize("ext", [b"\x00", b"\x01", b"\x00\x00"])
def test_var_key_prefix_extension(dev, ext):
    """A user key followed by its extension (shorter prefix sorts first,
    keys.py:60-63), for every pair of key lengths that fits a var record: the
    record padding past the key length must be zero (a leaked byte made
    key ∥ 00 compare below key at L = 58, 66)."""
    from paper_2004_03054_b200.compaction import compact_files
    from paper_2004_03054_b200.config import StoreConfig
    base = bytes(range(1, 80))
    for L in range(0, 72 - len(ext)):  # user keys up to kVarMaxLen = 71 bytes
        keys = [base[:L], base[:L] + ext]
        pairs = [(O.make_ikey(k, 100 + i, O.KIND_PUT), b"v" * 7) for i, k in enumerate(keys)]
        # a third key of another length: mixed lengths force the generic-length records
        f = O.build_table(pairs + [(O.make_ikey(b"\xff" * 3, 1, O.KIND_PUT), b"z")], sst_size_target=1 << 20)
        want = O.reference_compact([f], sst_size_target=1 << 20)
        got = compact_files(dev, [f], [], source_level=0, config=StoreConfig(sst_size_target=1 << 20))
        assert [g[0] for g in got] == [w[0] for w in want], f"L={L}"


@pytest.mark.parametrize("name", [n for n, _, _ in VARKEY_CASES[:6]])
def test_generic_key_lengths_multitile_planner(dev, small_planner_tiles, name):
    check_case(dev, name)


def test_index_keys_one_length_data_keys_mixed(dev):
    """Index keys (block last keys) all of one length but data keys of others:
    the fixed-length decode meets another length and the job is re-run on the
    generic-length path."""
    from paper_2004_03054_b200.compaction import compact_files
    from paper_2004_03054_b200.config import StoreConfig
    rng = random.Random(0x71)
    files = []
    seq = 1
    for f in range(3):
        keys = sorted({bytes([f]) + rng.randbytes(rng.randint(0, 14)) for _ in range(12)})
        keys = [k for k in keys if len(k) < 16][:10] + [bytes([f]) + b"\xff" * 15]
        pairs = []
        for k in keys:
            pairs.append((O.make_ikey(k, seq, O.KIND_PUT), rng.randbytes(8)))
            seq += 1
        files.append(O.build_table(pairs, sst_size_target=2**31))
        assert len(O.open_table(files[-1])[1]) == 1  # one block: the index holds only the 16-byte last key
    want = O.reference_compact(files[::-1])
    got = compact_files(dev, files[::-1], [], source_level=0, config=StoreConfig())
    assert [g[0] for g in got] == [w[0] for w in want]
    assert [(g[1], g[2]) for g in got] == [(w[1], w[2]) for w in want]


@pytest.mark.parametrize("klen", [72, 80, 200, 255])
def test_user_keys_longer_than_71_bytes(dev, klen):
    """Keys past the 71-byte var record re-run on the long records (<= 255
    bytes), byte-identical to the oracle."""
    from paper_2004_03054_b200.compaction import compact_files
    rng = random.Random(0x72 + klen)
    pairs = sorted(((O.make_ikey(rng.randbytes(klen), i + 1, O.KIND_PUT), b"v" * (i % 7)) for i in range(300)),
                   key=lambda kv: O.order_key(kv[0]))
    f = O.build_table(pairs, block_size=1024)
    short = O.build_table([(O.make_ikey(b"\x01" * 5, 900, O.KIND_PUT), b"s")])  # mixed lengths in the job
    want = O.reference_compact([short, f], sst_size_target=64 * 1024)
    from paper_2004_03054_b200.config import StoreConfig
    got = compact_files(dev, [short, f], [], source_level=0, config=StoreConfig(sst_size_target=64 * 1024))
    assert [g[0] for g in got] == [w[0] for w in want]
    assert [(g[1], g[2]) for g in got] == [(w[1], w[2]) for w in want]


def test_user_keys_longer_than_255_bytes_unsupported(dev):
    from paper_2004_03054_b200 import UnsupportedInputError
    from paper_2004_03054_b200.compaction import compact_files
    rng = random.Random(0x73)
    pairs = sorted(((O.make_ikey(rng.randbytes(300), i + 1, O.KIND_PUT), b"v") for i in range(50)),
                   key=lambda kv: O.order_key(kv[0]))
    f = O.build_table(pairs)
    O.reference_compact([f])  # the reference accepts them
    with pytest.raises(UnsupportedInputError):
        compact_files(dev, [f], [], source_level=0)


@pytest.mark.parametrize("ext", [b"\x00", b"\xff"])
def test_long_var_key_prefix_extension(dev, ext):
    """Prefix / extension pairs on the long records (lengths 72..254)."""
    from paper_2004_03054_b200.compaction import compact_files
    from paper_2004_03054_b200.config import StoreConfig
    base = bytes((i * 7 + 1) & 0xFF for i in range(260))
    for L in list(range(70, 90)) + [120, 127, 128, 129, 200, 247, 248, 253]:
        keys = [base[:L], base[:L] + ext]
        pairs = [(O.make_ikey(k, 100 + i, O.KIND_PUT), b"v" * 7) for i, k in enumerate(keys)]
        f = O.build_table(pairs + [(O.make_ikey(b"\xff" * 3, 1, O.KIND_PUT), b"z")], sst_size_target=1 << 20)
        want = O.reference_compact([f], sst_size_target=1 << 20)
        got = compact_files(dev, [f], [], source_level=0, config=StoreConfig(sst_size_target=1 << 20))
        assert [g[0] for g in got] == [w[0] for w in want], f"L={L}"


def test_crc_error_outranks_later_data_errors(dev):
    """The filter / index CRCs are checked on a side stream while the decode
    runs; their errors still come first: Table.__init__ of every input file
    precedes the data-block decode, so a bad filter CRC in
    a later file outranks a corrupt data block in an earlier one."""
    from paper_2004_03054_b200 import CorruptionError
    job, lower, upper = _corrupt_case()
    lower = list(lower)
    _, index = O.open_table(lower[0])
    bad = bytearray(lower[0])
    bad[index[1][1] + 9] ^= 0x20  # data block 1 of the first file
    lower[0] = bytes(bad)
    f = bytearray(upper[2])
    foff = O.FOOTER.unpack_from(f, len(f) - O.FOOTER_SIZE)[0]
    f[foff + 2] ^= 0x04  # filter of a later file
    upper = list(upper)
    upper[2] = bytes(f)
    with pytest.raises(O.CorruptionError) as want:
        O.reference_compact(lower + upper)
    assert want.value.offset == foff
    with pytest.raises(CorruptionError) as got:
        gpu_compact(dev, job, lower, upper, {})
    assert got.value.offset == foff


def test_structural_error_before_later_crc_error(dev):
    """A structural filter error (bad probe count, CRC recomputed so the filter
    CRC itself passes) in the first file outranks a filter CRC error in a later
    file — the synchronous check path."""
    import struct

    from paper_2004_03054_b200 import FormatError
    job, lower, upper = _corrupt_case()
    lower = list(lower)
    f = bytearray(lower[0])
    foff, flen, _, _, _ = O.FOOTER.unpack_from(f, len(f) - O.FOOTER_SIZE)
    f[foff + flen - 5] = 40  # probe count k > 30
    struct.pack_into("<I", f, foff + flen - 4, zlib.crc32(bytes(f[foff:foff + flen - 4])))
    lower[0] = bytes(f)
    g = bytearray(upper[1])
    goff = O.FOOTER.unpack_from(g, len(g) - O.FOOTER_SIZE)[0]
    g[goff + 1] ^= 0x01
    upper = list(upper)
    upper[1] = bytes(g)
    with pytest.raises(O.FormatError, match="bad probe count"):
        O.reference_compact(lower + upper)
    with pytest.raises(FormatError, match="bad probe count"):
        gpu_compact(dev, job, lower, upper, {})


def test_spec_a1_randomized_configs(dev):
    """SPEC A1: 800 more random jobs (with the 200 golden ones:
    1,000) — 1-6 L0 SSTs, 64 B - 4 KiB values, 0-20 % tombstones — each under a
    random store configuration (block size, restart interval, bits per key, SST
    target), byte-compared with the oracle."""
    rng = random.Random(0x5EC1A)
    bad = []
    for s in range(1000, 1800):
        job = jobgen.spec_a1(s)
        cfg = dict(block_size=rng.choice([512, 1024, 4096, 8192]), restart_interval=rng.choice([1, 2, 3, 16, 32]),
                   bits_per_key=rng.choice([1, 7, 10, 13]),
                   sst_size_target=rng.choice([8, 32, 128, 1024, 4096]) * 1024)
        blk = {k: cfg[k] for k in ("block_size", "restart_interval")}
        lower, upper = jobgen.materialize(job, **blk)
        want = O.reference_compact(lower + upper, deeper=job.deeper, **cfg)
        got = gpu_compact(dev, job, lower, upper, cfg)
        if [g[0] for g in got] != [w[0] for w in want] or [g[1:] for g in got] != [w[1:] for w in want]:
            bad.append((s, cfg))
    assert not bad, bad[:5]


def test_varkey_randomized_configs(dev):
    """Generic-length keys (0-64 B mixed in one job, prefix-rich) under random
    store configurations: 150 jobs byte-compared with the oracle."""
    rng = random.Random(0x7A57)
    bad = []
    for s in range(100, 250):
        job = jobgen.varkey(s, max_len=64, n_space=rng.randint(50, 400))
        cfg = dict(block_size=rng.choice([512, 1024, 4096]), restart_interval=rng.choice([1, 3, 16]),
                   bits_per_key=rng.choice([7, 10, 13]), sst_size_target=rng.choice([4, 16, 64]) * 1024)
        blk = {k: cfg[k] for k in ("block_size", "restart_interval")}
        lower, upper = jobgen.materialize(job, **blk)
        want = O.reference_compact(lower + upper, deeper=job.deeper, **cfg)
        got = gpu_compact(dev, job, lower, upper, cfg)
        if [g[0] for g in got] != [w[0] for w in want] or [g[1:] for g in got] != [w[1:] for w in want]:
            bad.append((s, cfg))
    assert not bad, bad[:5]


def _var_many_blocks(klen_fn, n=3000, seed=0x91):
    rng = random.Random(seed)
    keys = sorted({rng.randbytes(klen_fn(rng)) for _ in range(n)})
    pairs = sorted(((O.make_ikey(k, i + 1, O.KIND_PUT), b"v" * (i % 5)) for i, k in enumerate(keys)),
                   key=lambda kv: O.order_key(kv[0]))
    return O.build_table(pairs, block_size=256)


def _reseal_index(f: bytes, mutate) -> bytes:
    """Mutate the index payload (entries ∥ count) and recompute its CRC so the
    damage reaches decode_index_block (sst.py:79-102) instead of the CRC check."""
    import struct
    foff, flen, ioff, ilen, magic = O.FOOTER.unpack_from(f, len(f) - O.FOOTER_SIZE)
    payload = bytearray(f[ioff:ioff + ilen - 4])
    mutate(payload)
    out = bytearray(f[:ioff]) + payload + struct.pack("<I", zlib.crc32(bytes(payload)))
    ilen2 = len(payload) + 4
    foff2 = foff if foff < ioff else foff + (ilen2 - ilen)
    return bytes(out) + bytes(f[ioff + ilen:len(f) - O.FOOTER_SIZE]) + O.FOOTER.pack(foff2, flen, ioff, ilen2, magic)


def _index_entry_starts(payload):
    import struct
    n = struct.unpack_from("<I", payload, len(payload) - 4)[0]
    pos, starts = 0, []
    for _ in range(n):
        starts.append(pos)
        kl, pos = O.varint_read(payload, pos)
        pos += kl + 8
    return starts


@pytest.mark.parametrize("damage", ["count_minus", "count_plus", "klen_big", "klen_cont", "klen_long_varint",
                                    "klen_short", "count_ff"])
def test_index_parse_errors_multi_window(dev, damage):
    """decode_index_block errors (varint truncated / too long, truncated entry,
    trailing bytes) at entries far past the first staged window of the warp
    walk, on a mixed-length index (no fixed stride): same exception class and
    message as the reference's Table.__init__."""
    import struct
    from paper_2004_03054_b200.compaction import compact_files
    f = _var_many_blocks(lambda r: r.randint(8, 60))

    def mut(p):
        starts = _index_entry_starts(p)
        n = len(starts)
        late = starts[int(n * 0.8)]
        if damage == "count_minus":
            struct.pack_into("<I", p, len(p) - 4, n - 1)
        elif damage == "count_plus":
            struct.pack_into("<I", p, len(p) - 4, n + 1)
        elif damage == "klen_big":
            p[late] = 0x7F
        elif damage == "klen_cont":
            p[late] = p[late] | 0x80
        elif damage == "klen_long_varint":
            p[late:late + 11] = b"\xff" * 11
        elif damage == "klen_short":
            p[late] = max(0, p[late] - 3)
        elif damage == "count_ff":  # the walk runs into the count: varint truncated
            struct.pack_into("<I", p, len(p) - 4, 0xFFFFFFFF)
    g = _reseal_index(f, mut)
    with pytest.raises(Exception) as want:
        O.reference_compact([g])
    with pytest.raises(Exception) as got:
        compact_files(dev, [g], [], source_level=0)
    assert type(got.value).__name__ == type(want.value).__name__
    assert str(got.value) == str(want.value)


@pytest.mark.parametrize("klen", [1000, 2100, 5000])
def test_index_keys_longer_than_the_walk_window(dev, klen):
    """Index entries whose keys exceed the warp walk's 2 KB window parse
    (off/len read past the window); the job is then unsupported (keys > 255 B)."""
    from paper_2004_03054_b200 import UnsupportedInputError
    from paper_2004_03054_b200.compaction import compact_files
    rng = random.Random(klen)
    pairs = sorted(((O.make_ikey(rng.randbytes(klen), i + 1, O.KIND_PUT), b"v") for i in range(40)),
                   key=lambda kv: O.order_key(kv[0]))
    f = O.build_table(pairs, block_size=256)
    O.reference_compact([f])
    with pytest.raises(UnsupportedInputError):
        compact_files(dev, [f], [], source_level=0)


@pytest.mark.parametrize("seed", range(3))
def test_var_many_blocks_multi_window_index(dev, seed):
    """A mixed-length job whose indexes span many walk windows: byte-identical."""
    from paper_2004_03054_b200.compaction import compact_files
    from paper_2004_03054_b200.config import StoreConfig
    a = _var_many_blocks(lambda r: r.randint(8, 70), seed=seed)
    b = _var_many_blocks(lambda r: r.choice([8, 9, 40, 70, 71]), n=2000, seed=seed + 100)
    want = O.reference_compact([a, b], sst_size_target=128 * 1024)
    got = compact_files(dev, [a, b], [], source_level=0, config=StoreConfig(sst_size_target=128 * 1024))
    assert [g[0] for g in got] == [w[0] for w in want]
