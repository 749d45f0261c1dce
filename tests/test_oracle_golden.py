"""Pin the CPU oracle (oracle/luda_oracle.py) against golden vectors frozen from
the real reference by tests/golden/make_golden.py. CPU-only."""

import hashlib
import json
import os
import random
import struct

import pytest

from oracle import jobgen
from oracle import luda_oracle as O
from tests.golden.cases import ALL_CASES as CASES

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "compaction.json")))
KAT = json.load(open(os.path.join(HERE, "golden", "kat.json")))
ITEMS = json.load(open(os.path.join(HERE, "golden", "items.json")))


def sha(b):
    return hashlib.sha256(bytes(b)).hexdigest()


def build_case(name):
    mk, out_cfg = {n: (m, c) for n, m, c in CASES}[name]
    job = mk()
    blk = {k: out_cfg[k] for k in ("block_size", "restart_interval") if k in out_cfg}
    lower, upper = jobgen.materialize(job, **blk)
    return job, lower, upper, out_cfg


@pytest.mark.parametrize("name", [n for n, _, _ in CASES])
def test_compaction_matches_reference(name):
    job, lower, upper, out_cfg = build_case(name)
    g = GOLD[name]
    assert [sha(f) for f in lower] == g["inputs_lower"]
    assert [sha(f) for f in upper] == g["inputs_upper"]
    outs = O.reference_compact(lower + upper, deeper=job.deeper, **out_cfg)
    got = [{"sha256": sha(f), "size": len(f), "smallest": s.hex(), "largest": l.hex()}
           for f, s, l in outs]
    assert got == g["outputs"]


def test_crc_kats():
    assert O.crc32(b"123456789") == KAT["crc_check"] == 0xCBF43926
    assert O.crc32(b"") == KAT["crc_empty"] == 0
    rng = random.Random(KAT["crc_random_seed"])
    for hexed, digest, n, crc in KAT["crc_random"]:
        b = rng.randbytes(n)
        assert sha(b) == digest
        assert O.crc32(b) == crc


def test_codec_kats():
    assert [list(x) for x in O.block_layouts([b"apple", b"applet", b"apply"], 16)] == KAT["layouts_apple"]
    a = O.make_ikey(b"ab", 5, 1)
    b = O.make_ikey(b"ab\x01", 5, 1)
    assert O.common_prefix(a, b) == KAT["prefix_into_trailer"] == 3  # shared prefix runs into the trailer
    pairs = [(O.make_ikey(b"k%03d" % i, 100 + i, 1), bytes([i]) * 100) for i in range(3)]
    assert O.build_table(pairs).hex() == KAT["three_pairs_sst_hex"]
    for v, hexed in KAT["varints"]:
        assert O.varint_bytes(v).hex() == hexed
        assert O.varint_read(bytes.fromhex(hexed), 0) == (v, len(hexed) // 2)
    assert O.filter_block(*O.bloom_bits([], 10)).hex() == KAT["bloom_empty"]


def test_bloom_and_oversized_kats():
    rng = random.Random(KAT["crc_random_seed"])
    for _, _, n, _ in KAT["crc_random"]:
        rng.randbytes(n)
    keys = [rng.randbytes(16) for _ in range(200)]
    assert [k.hex() for k in keys] == KAT["bloom200"]["keys"]
    assert O.filter_block(*O.bloom_bits(keys, 10)).hex() == KAT["bloom200"]["encoded"]
    bits, k = O.bloom_bits(keys, 10)
    assert all(O.bloom_may_contain(bits, k, x) for x in keys)
    big = (O.make_ikey(b"x" * 16, 7, 1), rng.randbytes(10000))
    blk = O.build_block([big[0]], [big[1]], O.block_layouts([big[0]], 16), 16)
    assert len(blk) == KAT["oversized_block_len"]
    assert sha(blk) == KAT["oversized_block_hex_sha"]


def test_item_kernels_match_reference():
    """Dispatch-level parity of the four kernel kinds (kernels.py) vs the reference SerialDevice."""
    job = jobgen.mixed(7, n_files=2, max_keys=300)
    files = [f for r in job.lower for f, _, _ in O.build_tables_split(r.pairs, sst_size_target=r.sst_target)]
    assert [sha(f) for f in files] == ITEMS["files"]
    d_unpack, d_sk, d_enc, d_filt = ITEMS["dispatches"]
    data = files[0]
    items = [tuple(x) for x in d_unpack["items"]]
    cap = sum(it[2] for it in items) * 4
    regions = {items[0][0]: bytearray(data), items[0][3]: bytearray(cap), items[0][6]: bytearray(cap)}
    res = [O.run_item("unpack", it, regions) for it in items]
    assert [list(r[1]) for r in res] == d_unpack["results"]
    assert sha(regions[items[0][3]]) == d_unpack["pairs_sha"]
    assert sha(regions[items[0][6]]) == d_unpack["tuples_sha"]
    sk_items = [tuple(x) for x in d_sk["items"]]
    n = res[0][1][2]
    regions[sk_items[0][4]] = bytearray(8 * n)
    assert [list(O.run_item("shared_key", it, regions)[1]) for it in sk_items] == d_sk["results"]
    assert sha(regions[sk_items[0][4]]) == d_sk["out_sha"]
    enc_items = [tuple(x) for x in d_enc["items"]]
    regions[enc_items[0][6]] = bytearray(2 * 8192)
    assert [list(O.run_item("encode", it, regions)[1]) for it in enc_items] == d_enc["results"]
    assert sha(regions[enc_items[0][6]]) == d_enc["out_sha"]
    tb = res[0][1][1]
    fo = max(regions) + 1
    regions[fo] = bytearray(4096)
    r = O.run_item("filter", (items[0][6], 0, tb, 10, fo, 0, 4096), regions)
    assert [list(r[1])] == d_filt["results"]
    assert sha(regions[fo]) == d_filt["out_sha"]


def test_corruption_and_format_errors():
    pairs = [(O.make_ikey(b"key%05d" % i, i + 1, 1), b"v" * 50) for i in range(200)]
    data = bytearray(O.build_table(pairs))
    _, index = O.open_table(bytes(data))
    off = index[1][1]
    data[off + 5] ^= 0x10
    with pytest.raises(O.CorruptionError) as ei:
        list(O.scan_table(bytes(data), index))
    assert ei.value.offset == off
    bad = bytearray(O.build_table(pairs))
    bad[-1] ^= 1
    with pytest.raises(O.FormatError):
        O.open_table(bytes(bad))
    with pytest.raises(O.OrderingError):
        list(O.merge_resolve([[(O.make_ikey(b"b", 2, 1), b""), (O.make_ikey(b"a", 1, 1), b"")]]))


def test_merge_example_from_spec():
    a5, b2 = O.make_ikey(b"a", 5, 1), O.make_ikey(b"b", 2, 1)
    a3, c1 = O.make_ikey(b"a", 3, 1), O.make_ikey(b"c", 1, 1)
    got = [k for k, _ in O.merge_resolve([[(a5, b""), (b2, b"")], [(a3, b""), (c1, b"")]])]
    assert got == [a5, b2, c1]
    x7 = O.make_ikey(b"x", 7, 0)
    assert list(O.merge_resolve([[(x7, b"")]])) == []
    assert [k for k, _ in O.merge_resolve([[(x7, b"")]], deeper=[(b"a", b"z")])] == [x7]
