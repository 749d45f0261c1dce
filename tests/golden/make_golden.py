"""Freeze golden vectors from the REAL reference (run in the build container only).

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_golden.py

For every case in ``CASES`` this script
  1. generates the seeded job with ``oracle/jobgen.py`` (data only),
  2. cuts each run into SST files with the reference's ``SstBuilder``
     (sst.py:105-217) using the SizeOverflowError → finish → new builder rule,
  3. compacts them with a composition of reference calls only:
     ``FilterBlock.decode`` / ``decode_index_block`` / ``decode_data_block``,
     ``heapq.merge`` on ``keys.sort_key``, first-per-user-key, D12 tombstone
     drop, ``SstBuilder`` with the same cut rule,
and writes SHA-256 digests of every input and output file (plus smallest /
largest keys) to ``tests/golden/compaction.json``. It also writes known-answer
vectors (``kat.json``) and dispatch-level item results of the reference's
``kernels.py`` run on its ``SerialDevice`` (``items.json``).

The reference tree is never needed at test time: the oracle restatement is
checked against these digests (tests/test_oracle_golden.py) and the CUDA path
against the oracle.
"""

from __future__ import annotations

import hashlib
import heapq
import json
import os
import random
import struct
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from luda import blocks as R_blocks  # noqa: E402
from luda import bloom as R_bloom  # noqa: E402
from luda import checksum as R_crc  # noqa: E402
from luda import keys as R_keys  # noqa: E402
from luda import kernels as R_kernels  # noqa: E402
from luda import sst as R_sst  # noqa: E402
from luda.config import DeviceConfig as R_DeviceConfig  # noqa: E402
from luda.device import KernelSpec as R_KernelSpec, make_device as R_make_device  # noqa: E402
from luda.errors import SizeOverflowError as R_SizeOverflow  # noqa: E402

from oracle import jobgen  # noqa: E402


def sha(b: bytes) -> str:
    return hashlib.sha256(bytes(b)).hexdigest()


def ref_build_split(pairs, sst_size_target=4 * 2**20, block_size=4096, restart_interval=16, bits_per_key=10):
    outs = []

    def new():
        return R_sst.SstBuilder(block_size=block_size, restart_interval=restart_interval,
                                bits_per_key=bits_per_key, sst_size_target=sst_size_target)
    b = new()
    count = 0
    for k, v in pairs:
        try:
            b.add(k, v)
        except R_SizeOverflow:
            outs.append((b.finish(), b.smallest, b.largest))
            b = new()
            b.add(k, v)
        count += 1
    if count:
        outs.append((b.finish(), b.smallest, b.largest))
    return outs


def ref_open_scan(data: bytes):
    """Table.__init__ + Table.scan over an in-memory file, via reference calls."""
    foff, flen, ioff, ilen, magic = struct.unpack_from("<IIIIQ", data, len(data) - 24)
    assert magic == R_sst.MAGIC
    R_bloom.FilterBlock.decode(data[foff:foff + flen], offset=foff)
    index = R_sst.decode_index_block(data[ioff:ioff + ilen], offset=ioff)
    pairs = []
    for _, off, ln in index:
        pairs.extend(R_blocks.decode_data_block(data[off:off + ln], offset=off))
    return pairs


def ref_compact(files, deeper, out_cfg):
    runs = [ref_open_scan(f) for f in files]
    merged = heapq.merge(*runs, key=lambda kv: R_keys.sort_key(kv[0]))

    def survivors():
        prev = None
        for k, v in merged:
            u = R_keys.user_key_of(k)
            if u == prev:
                continue
            prev = u
            if R_keys.kind_of(k) == R_keys.KIND_DELETE and not any(lo <= u <= hi for lo, hi in deeper):
                continue
            yield k, v
    return ref_build_split(survivors(), **out_cfg)


from tests.golden.cases import ALL_CASES as CASES  # noqa: E402


def make_compaction_goldens():
    out = {}
    for name, mk, out_cfg in CASES:
        job = mk()
        blk = {k: out_cfg[k] for k in ("block_size", "restart_interval") if k in out_cfg}
        lower = [f for r in job.lower for f, _, _ in ref_build_split(r.pairs, r.sst_target, **blk)]
        upper = [f for r in job.upper for f, _, _ in ref_build_split(r.pairs, r.sst_target, **blk)]
        deeper = [(lo, hi) for lo, hi in job.deeper]
        outs = ref_compact(lower + upper, deeper, out_cfg)
        out[name] = {
            "out_cfg": out_cfg,
            "inputs_lower": [sha(f) for f in lower],
            "inputs_upper": [sha(f) for f in upper],
            "input_sizes": [len(f) for f in lower + upper],
            "outputs": [{"sha256": sha(f), "size": len(f), "smallest": s.hex(), "largest": l.hex()}
                        for f, s, l in outs],
        }
        print(f"{name}: {len(lower)}+{len(upper)} inputs -> {len(outs)} outputs", flush=True)
    return out


def make_kats():
    rng = random.Random(0x5EED)
    kat = {}
    kat["crc_check"] = R_crc.crc32(b"123456789")
    kat["crc_empty"] = R_crc.crc32(b"")
    bufs = [rng.randbytes(n) for n in (1, 3, 4, 15, 16, 17, 127, 128, 129, 1000, 4096, 4100, 10025, 65537)]
    kat["crc_random"] = [[b.hex() if len(b) <= 64 else None, sha(b), len(b), R_crc.crc32(b)] for b in bufs]
    kat["crc_random_seed"] = 0x5EED
    kat["layouts_apple"] = R_blocks.compute_layouts([b"apple", b"applet", b"apply"], 16)
    kat["prefix_into_trailer"] = R_blocks.shared_prefix_len(
        R_keys.encode_key(b"ab", 5, 1), R_keys.encode_key(b"ab\x01", 5, 1))
    pairs = [(R_keys.encode_key(b"k%03d" % i, 100 + i, 1), bytes([i]) * 100) for i in range(3)]
    data, meta = R_sst.build_sst(pairs)
    kat["three_pairs_sst_hex"] = data.hex()
    keys = [rng.randbytes(16) for _ in range(200)]
    f = R_bloom.build_filter(keys, 10)
    kat["bloom200"] = {"seed_note": "keys = [Random(0x5EED) after crc bufs].randbytes(16) x200",
                       "keys": [k.hex() for k in keys], "encoded": f.encode().hex()}
    kat["bloom_empty"] = R_bloom.build_filter([], 10).encode().hex()
    kat["varints"] = [[v, __import__("luda.varint", fromlist=["x"]).encode(v).hex()]
                      for v in (0, 1, 127, 128, 300, 16383, 16384, 2**32, 2**63 - 1)]
    big = (R_keys.encode_key(b"x" * 16, 7, 1), rng.randbytes(10000))
    kat["oversized_block_hex_sha"] = sha(R_blocks.encode_data_block([big]))
    kat["oversized_block_len"] = len(R_blocks.encode_data_block([big]))
    return kat


def make_item_goldens():
    """Run the reference's four kernel kinds on its SerialDevice; digest regions + results."""
    job = jobgen.mixed(7, n_files=2, max_keys=300)
    files = [f for r in job.lower for f, _, _ in ref_build_split(r.pairs, r.sst_target)]
    dev = R_make_device(R_DeviceConfig(backend="serial"))
    res = {"files": [sha(f) for f in files], "dispatches": []}
    try:
        data = files[0]
        foff, flen, ioff, ilen, _ = struct.unpack_from("<IIIIQ", data, len(data) - 24)
        index = R_sst.decode_index_block(data[ioff:ioff + ilen])
        src = dev.alloc(len(data))
        dev.stage_in(src, data, "in_lower").wait()
        cap = sum(ln for _, _, ln in index) * 4
        pairs = dev.alloc(cap)
        tups = dev.alloc(cap)
        items = []
        slot = 0
        for _, off, ln in index:
            items.append((src.region_id, off, ln, pairs.region_id, slot, 4 * ln,
                          tups.region_id, slot, 4 * ln))
            slot += 4 * ln
        h = dev.dispatch(R_KernelSpec("unpack", tuple(items), reads=(src.region_id,),
                                      writes=(pairs.region_id, tups.region_id)))
        results = h.wait()
        res["dispatches"].append({"kind": "unpack", "items": items, "results": results,
                                  "pairs_sha": sha(dev.stage_out(pairs, [(0, cap)], "out").wait()),
                                  "tuples_sha": sha(dev.stage_out(tups, [(0, cap)], "out").wait())})
        # shared_key + encode + filter over the first block's tuples, in 2 blocks.
        _, tb, n, _ = results[0]
        all_t = R_kernels.parse_tuples(dev._regions[tups.region_id].buf, 0, tb)
        cut = 0
        pos = 0
        for t in all_t[: max(1, n // 2)]:
            pos += R_kernels.tuple_wire_size(len(t[0]))
        cut = pos
        lay = dev.alloc(8 * n)
        sk_items = ((tups.region_id, 0, cut, 16, lay.region_id, 0),
                    (tups.region_id, cut, tb, 16, lay.region_id, 8 * max(1, n // 2)))
        r2 = dev.dispatch(R_KernelSpec("shared_key", sk_items, reads=(tups.region_id,),
                                       writes=(lay.region_id,))).wait()
        outb = dev.alloc(2 * 8192)
        enc_items = ((tups.region_id, 0, cut, lay.region_id, 0, pairs.region_id, outb.region_id, 0, 8192, 16),
                     (tups.region_id, cut, tb, lay.region_id, 8 * max(1, n // 2), pairs.region_id,
                      outb.region_id, 8192, 8192, 16))
        r3 = dev.dispatch(R_KernelSpec("encode", enc_items, reads=(tups.region_id, lay.region_id, pairs.region_id),
                                       writes=(outb.region_id,))).wait()
        fo = dev.alloc(4096)
        r4 = dev.dispatch(R_KernelSpec("filter", ((tups.region_id, 0, tb, 10, fo.region_id, 0, 4096),),
                                       reads=(tups.region_id,), writes=(fo.region_id,))).wait()
        res["dispatches"].append({"kind": "shared_key", "items": sk_items, "results": r2,
                                  "out_sha": sha(dev.stage_out(lay, [(0, 8 * n)], "out").wait())})
        res["dispatches"].append({"kind": "encode", "items": enc_items, "results": r3,
                                  "out_sha": sha(dev.stage_out(outb, [(0, 2 * 8192)], "out").wait())})
        res["dispatches"].append({"kind": "filter", "results": r4,
                                  "out_sha": sha(dev.stage_out(fo, [(0, 4096)], "out").wait())})
    finally:
        dev.close()
    return res


def make_read_goldens():
    """Read-path goldens: the reference SstBuilder's files opened with the
    reference Table (files in a temp dir, no block cache) and probed with
    Table.get (sst.py:342-368) — per table, or in SPEC store order."""
    import tempfile
    from tests.golden import read_cases as RC
    out = {}
    for name in RC.READ_CASES:
        c = RC.build(name, builder=lambda pairs, sst_size_target, **cfg: ref_build_split(pairs, sst_size_target, **cfg))
        with tempfile.TemporaryDirectory() as d:
            tables = []
            for i, f in enumerate(c["files"]):
                p = os.path.join(d, f"{i}.sst")
                with open(p, "wb") as fh:
                    fh.write(f)
                tables.append(R_sst.open_sst(p))
            enc = []
            for t, q in c["queries"]:
                if c["mode"] == "table":
                    o = RC.outcome(lambda: tables[t].get(q))
                else:
                    o = RC.outcome(lambda: O_store_get(tables, c["l0"], c["levels"], q))
                enc.append(RC.encode(c["mode"], o))
            counters = [[tb.filter_rejects, tb.data_block_reads] for tb in tables]
            for tb in tables:
                tb.close()
        out[name] = {"files": [sha(f) for f in c["files"]], "results": RC.summary(enc), "counters": counters}
        print(f"{name}: {len(c['files'])} files, {RC.summary(enc)}", flush=True)
    return out


def O_store_get(tables, l0, levels, q):
    from oracle import luda_oracle as O
    return O.store_get(tables, l0, levels, q)  # SPEC-order composition over the REFERENCE Table objects


def main():
    if sys.argv[1:] == ["reads"]:
        with open(os.path.join(HERE, "reads.json"), "w") as f:
            json.dump(make_read_goldens(), f, indent=1, sort_keys=True)
        return
    with open(os.path.join(HERE, "reads.json"), "w") as f:
        json.dump(make_read_goldens(), f, indent=1, sort_keys=True)
    gold = make_compaction_goldens()
    with open(os.path.join(HERE, "compaction.json"), "w") as f:
        json.dump(gold, f, indent=1, sort_keys=True)
    with open(os.path.join(HERE, "kat.json"), "w") as f:
        json.dump(make_kats(), f, indent=1, sort_keys=True)
    with open(os.path.join(HERE, "items.json"), "w") as f:
        json.dump(make_item_goldens(), f, indent=1, sort_keys=True, default=list)


if __name__ == "__main__":
    main()
