"""Read-path golden cases, shared by make_golden.py
(reference side: reference SstBuilder + reference Table.get on files written to
a temp dir) and the tests (oracle MemTable / the device table set).

A case is a set of SST files plus a query list:
* mode "table": queries are (table id, user key) — Table.get (sst.py:342-368);
* mode "store": queries are user keys probed in the SPEC store order
   over ``l0`` (newest first) and ``levels``.
Queries mix present keys, absent keys of the same length, near misses (last
byte +-1), prefixes / extensions of present keys, the empty key and keys
past both ends. ``corrupt`` flips bytes inside chosen data blocks after the
files are built, so lookups that read those blocks raise CorruptionError.
"""

from __future__ import annotations

import random
import struct

from oracle import jobgen
from oracle import luda_oracle as O


def _user_keys(data):
    """All user keys of one SST, in file order (oracle scan)."""
    _, index = O.open_table(data)
    return [k[:-8] for k, _ in O.scan_table(data, index)]


def _ranges(files):
    out = []
    for f in files:
        ks = _user_keys(f)
        out.append((min(ks), max(ks)))
    return out


def _queries(rng, pool, n, klen=None):
    """n query keys: 50% present, rest absent / near-miss / prefix / extension."""
    out = []
    pool = list(pool)
    for _ in range(n):
        r = rng.random()
        k = rng.choice(pool)
        if r < 0.5:
            q = k
        elif r < 0.65:
            q = rng.randbytes(klen if klen is not None else len(k))
        elif r < 0.8 and k:
            b = k[-1]
            q = k[:-1] + bytes([(b + rng.choice((1, 255))) & 0xFF])
        elif r < 0.9:
            q = k[:rng.randint(0, len(k))]
        else:
            q = k + bytes([rng.choice((0, 1, 0x80, 0xFF))])
        out.append(q)
    out += [b"", b"\x00" * (klen or 16), b"\xff" * (klen or 16)]
    return out


def _files(job, builder, **cfg):
    lower, upper = jobgen.materialize(job, builder=builder, **cfg)
    return lower, upper


def _corrupt(files, targets):
    """Flip one byte in the middle of data block `blk` of file `fi` (the block
    CRC then fails; filter, index and footer stay intact)."""
    files = [bytearray(f) for f in files]
    offs = []
    for fi, blk in targets:
        _, index = O.open_table(bytes(files[fi]))
        _, off, ln = index[blk % len(index)]
        files[fi][off + ln // 2] ^= 0x5A
        offs.append((fi, off))
    return [bytes(f) for f in files], offs


def build(name, builder=O.build_tables_split):
    """(files, mode, queries, l0, levels) of a read case."""
    rng = random.Random(sum(name.encode()) * 7919)
    if name == "c3_tables":
        lower, upper = _files(jobgen.c3(n=6000, sst_target=96 * 1024), builder)
        files = lower + upper
        qs = []
        for t, f in enumerate(files):
            for q in _queries(rng, _user_keys(f), 120, klen=16):
                qs.append((t, q))
        return dict(files=files, mode="table", queries=qs)
    if name == "ri4_bs1024":
        lower, upper = _files(jobgen.c3(n=2500, seed=0xAB, sst_target=40 * 1024), builder,
                              block_size=1024, restart_interval=4)
        files = lower + upper
        qs = [(t, q) for t, f in enumerate(files) for q in _queries(rng, _user_keys(f), 150, klen=16)]
        return dict(files=files, mode="table", queries=qs)
    if name == "c4_tables":
        lower, _ = _files(jobgen.c4(n_per_file=700, files=3), builder)
        qs = [(t, q) for t, f in enumerate(lower) for q in _queries(rng, _user_keys(f), 200, klen=24)]
        return dict(files=lower, mode="table", queries=qs)
    if name == "varkey_long":
        job = jobgen.varkey(77, max_len=250, n_space=300)
        for r in job.lower:
            r.sst_target = 24 * 1024
        lower, _ = _files(job, builder)
        qs = [(t, q) for t, f in enumerate(lower) for q in _queries(rng, _user_keys(f), 150)]
        return dict(files=lower, mode="table", queries=qs)
    if name.startswith("varkey"):
        job = jobgen.varkey(int(name[6:]), max_len=64)
        for r in job.lower:
            r.sst_target = 6 * 1024
        lower, _ = _files(job, builder)
        qs = [(t, q) for t, f in enumerate(lower) for q in _queries(rng, _user_keys(f), 150)]
        return dict(files=lower, mode="table", queries=qs)
    if name == "values_4k_12k":
        lower, upper = _files(jobgen.values_job(n=120), builder)
        files = lower + upper
        qs = [(t, q) for t, f in enumerate(files) for q in _queries(rng, _user_keys(f), 60, klen=16)]
        return dict(files=files, mode="table", queries=qs)
    if name == "bpk1":
        lower, upper = _files(jobgen.c3(n=3000, seed=0xB1, sst_target=64 * 1024), builder, bits_per_key=1)
        files = lower + upper
        qs = [(t, q) for t, f in enumerate(files) for q in _queries(rng, _user_keys(f), 100, klen=16)]
        return dict(files=files, mode="table", queries=qs)
    if name == "corrupt":
        lower, upper = _files(jobgen.c3(n=3000, seed=0xC0, sst_target=48 * 1024), builder)
        files, _ = _corrupt(lower + upper, [(0, 2), (1, 0), (len(lower), 5)])
        # key pool from the clean files; queries reach every block of the corrupted tables
        qs = [(t, q) for t, f in enumerate(lower + upper) for q in _queries(rng, _user_keys(f), 80, klen=16)]
        return dict(files=files, mode="table", queries=qs)
    if name == "store":
        # L0: the files of a mixed job's runs (overlapping, newest first);
        # L1 / L2: the lower and upper runs of a c3 job (disjoint files per level)
        mix = jobgen.mixed(5, n_files=4, max_keys=500, key_space=900)
        l0_files = [f for r in mix.lower for f, _, _ in builder(r.pairs, sst_size_target=16 * 1024)]
        lo1, lo2 = _files(jobgen.c3(n=4000, seed=0x5707, sst_target=48 * 1024), builder)
        files = l0_files + lo1 + lo2
        l0 = list(range(len(l0_files)))
        levels = []
        base = len(l0_files)
        for run in (lo1, lo2):
            rs = _ranges(run)
            levels.append([(base + i, lo, hi) for i, (lo, hi) in enumerate(rs)])
            base += len(run)
        pool = [k for f in files for k in _user_keys(f)]
        qs = [(None, q) for q in _queries(rng, pool, 3000, klen=16)]
        return dict(files=files, mode="store", queries=qs, l0=l0, levels=levels)
    if name == "malformed":
        f, qs = _malformed()
        return dict(files=[f], mode="table", queries=qs)
    raise KeyError(name)


def _malformed():
    """One SST whose data blocks carry VALID CRCs over malformed contents, so
    every DataBlockReader / _entry_at error path of the reference is reached
    (blocks.py:175-218, sst.py:322-340): bad restart arrays, restart offsets
    past the block, truncated and over-long varints, keys shorter than the
    trailer, clamped keys and values, shared > len(prev), 4-byte and 2-byte
    blocks, and a block past the end of the file (short read)."""
    V = O.varint_bytes
    U = O.U32.pack

    def ik(i, seq=5):
        return O.make_ikey(b"key-%02d" % i + b"." * 9, seq, 1)

    def blk(payload):
        return payload + U(O.crc32(payload))

    def entry(shared, unshared_bytes, value, unshared=None):
        u = len(unshared_bytes) if unshared is None else unshared
        return V(shared) + V(u) + V(len(value)) + unshared_bytes + value

    good0 = entry(0, ik(0), b"v0")
    blocks = [
        blk(good0 + U(0) + U(1)),                                   # 0 valid
        blk(U(0)),                                                  # 1 n_restarts = 0
        blk(U(5)),                                                  # 2 entries_end < 0
        blk(entry(0, ik(3), b"v3") + U(0) + U(200) + U(2)),         # 3 restart offset past the block
        blk(b"\x80\x80" + U(0) + U(1)),                             # 4 varint runs into the restart array
        blk(b"\xff" * 10 + U(0) + U(1)),                             # 5 varint too long
        blk(entry(0, b"abc", b"") + U(0) + U(1)),                   # 6 key shorter than the trailer
        blk(entry(0, ik(7)[:4], b"", unshared=60) + U(0) + U(1)),    # 7 unshared clamps at the block end
        blk(entry(0, ik(8), b"", ) + entry(40, ik(8)[-3:], b"xyz") + U(0) + U(1)),  # 8 shared > len(prev)
        blk(entry(0, ik(9), b"v9" * 3)[:-2] + U(0) + U(1)),          # 9 value clamped (runs into restarts)
        blk(b""),                                                   # 10 4-byte block (crc only)
        b"\x00\x00",                                                 # 11 2-byte block
        blk(entry(0, ik(12, 9), b"a") + entry(16, ik(12, 3)[16:], b"b") + entry(0, ik(12, 1), b"c")
            + U(0) + U(2 + len(entry(0, ik(12, 9), b"a")) + len(entry(16, ik(12, 3)[16:], b"b")) - 2) + U(2)),
    ]
    data = bytearray()
    index = []
    for i, b in enumerate(blocks):
        index.append((ik(i, 0), len(data), len(b)))
        data += b
    index.append((ik(len(blocks), 0), len(data) + 10 ** 6, 100))  # short read: past the end of the file
    foff = len(data)
    filt = O.filter_block(b"\xff" * 8, 1)
    data += filt
    ioff = len(data)
    idx = O.index_block(index)
    data += idx
    data += O.FOOTER.pack(foff, len(filt), ioff, len(idx), O.MAGIC)
    qs = []
    for i in range(len(index)):
        for q in (b"key-%02d" % i + b"." * 9, b"key-%02d" % i + b"." * 8, b"key-%02d" % i):
            qs.append((0, q))
    return bytes(data), qs


READ_CASES = ["c3_tables", "ri4_bs1024", "c4_tables", "varkey0", "varkey1", "varkey_long", "values_4k_12k", "bpk1",
              "corrupt", "store", "malformed"]


def outcome(fn):
    """Run fn(); ('ok', result) or ('E', exception class name, offset)."""
    try:
        return ("ok", fn())
    except struct.error:
        return ("E", "struct.error", None)
    except Exception as e:  # noqa: BLE001 — classes compared by name with the reference's
        return ("E", type(e).__name__, getattr(e, "offset", None))


def encode(mode, out):
    """JSON-able form of one outcome: None | [table, sha(key, value)] | ["E", class, offset]."""
    import hashlib
    if out[0] == "E":
        return ["E", out[1], out[2]]
    r = out[1]
    if r is None:
        return None
    t, (k, v) = r if mode == "store" else (None, r)
    h = hashlib.sha256(len(k).to_bytes(4, "little") + k + v).hexdigest()[:16]
    return [t, h]


def digest(encoded):
    import hashlib
    import json
    return hashlib.sha256(json.dumps(encoded).encode()).hexdigest()


def summary(encoded):
    found = sum(1 for e in encoded if e is not None and e[0] != "E")
    errs = sum(1 for e in encoded if e is not None and e[0] == "E")
    return {"n": len(encoded), "found": found, "errors": errs, "sha": digest(encoded)}
