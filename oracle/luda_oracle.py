"""CPU oracle for the LUDA compaction path — TEST INFRASTRUCTURE ONLY.

This module is a restatement, in plain Python + zlib + numpy, of the
reference's algorithm for the compaction hot path (the reference is pure
Python: ``/root/reference/pkg/src/luda``). It exists to CHECK the CUDA path.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it; the product
(``paper_2004_03054_b200``) never does.

Parity pinning: ``tests/golden/make_golden.py`` imports the real reference
(in the build container only) and freezes SHA-256 digests of its outputs for
seeded jobs into ``tests/golden/*.json``; ``tests/test_oracle_golden.py``
checks this restatement against them on every CPU test run.

Each function cites the reference ``file:line`` it restates. The compaction
composition (``reference_compact``) is absent from the reference and is
composed exactly as SURVEY.md §8(c) describes: open tables (footer, filter
CRC, index CRC), decode every data block in file order, heap-merge per-file
runs on ``sort_key``, keep the newest entry per user key, drop tombstones
not covered below the target level (SPEC D12), and feed ``SstBuilder`` with
``SizeOverflowError`` → ``finish`` → new builder.
"""

from __future__ import annotations

import heapq
import math
import struct
import zlib

import numpy as np

from paper_2004_03054_b200.errors import (
    CorruptionError,
    FormatError,
    OrderingError,
    SizeOverflowError,
)

U32 = struct.Struct("<I")
U64 = struct.Struct("<Q")
FOOTER = struct.Struct("<IIIIQ")
FOOTER_SIZE = FOOTER.size
MAGIC = 0x4C55444153535431  # sst.py:42
KIND_DELETE, KIND_PUT = 0, 1  # keys.py:16-17
TRAILER = 8


# --------------------------------------------------------------------------
# L1 primitives
# --------------------------------------------------------------------------

def crc32(data) -> int:
    """CRC-32/IEEE, zlib flavour (checksum.py:12-13)."""
    return zlib.crc32(data) & 0xFFFFFFFF


def varint_bytes(v: int) -> bytes:
    """Unsigned LEB128 (varint.py:6-17)."""
    if v < 0:
        raise ValueError("varint cannot encode negative values")
    out = bytearray()
    while v >= 0x80:
        out.append((v & 0x7F) | 0x80)
        v >>= 7
    out.append(v)
    return bytes(out)


def varint_len(v: int) -> int:
    """Encoded size (varint.py:20-25)."""
    n = 1
    while v >= 0x80:
        v >>= 7
        n += 1
    return n


def varint_read(buf, pos: int):
    """Decode one varint; FormatError on truncation / >63-bit shift (varint.py:28-43)."""
    value = 0
    shift = 0
    end = len(buf)
    while True:
        if pos >= end:
            raise FormatError("truncated varint")
        b = buf[pos]
        pos += 1
        value |= (b & 0x7F) << shift
        if b < 0x80:
            return value, pos
        shift += 7
        if shift > 63:
            raise FormatError("varint too long")


def make_ikey(user_key: bytes, seq: int, kind: int) -> bytes:
    """user_key ∥ u64le((seq<<8)|kind) (keys.py:25-34)."""
    if not 0 <= seq < (1 << 56):
        raise ValueError("seq out of 56-bit range")
    if kind not in (KIND_DELETE, KIND_PUT):
        raise ValueError("bad kind")
    return user_key + U64.pack((seq << 8) | kind)


def order_key(ikey: bytes):
    """(user_key asc, trailer desc) — keys.py:60-63."""
    return ikey[:-TRAILER], -U64.unpack_from(ikey, len(ikey) - TRAILER)[0]


def ukey(ikey: bytes) -> bytes:
    return ikey[:-TRAILER]


def kind_of(ikey: bytes) -> int:
    return ikey[-TRAILER]


# --------------------------------------------------------------------------
# L2 data-block codec (blocks.py)
# --------------------------------------------------------------------------

def common_prefix(a: bytes, b: bytes) -> int:
    """blocks.py:33-38."""
    n = min(len(a), len(b))
    i = 0
    while i < n and a[i] == b[i]:
        i += 1
    return i


def block_layouts(keys, restart_interval: int):
    """(shared, unshared) per entry, shared vs the PREVIOUS key, 0 at i%ri==0 (blocks.py:41-58)."""
    if restart_interval < 1:
        raise ValueError("restart_interval must be >= 1")
    out = []
    prev = b""
    for i, k in enumerate(keys):
        s = 0 if i % restart_interval == 0 else common_prefix(prev, k)
        out.append((s, len(k) - s))
        prev = k
    return out


def entry_size(shared: int, unshared: int, vlen: int) -> int:
    """blocks.py:61-68."""
    return varint_len(shared) + varint_len(unshared) + varint_len(vlen) + unshared + vlen


def tail_overhead(n_entries: int, restart_interval: int) -> int:
    """Restart array + count + crc (blocks.py:71-74)."""
    return 4 * ((n_entries + restart_interval - 1) // restart_interval) + 8


def build_block(keys, values, layouts, restart_interval: int) -> bytes:
    """entries ∥ u32 restarts ∥ u32 n_restarts ∥ u32 crc (blocks.py:77-103)."""
    body = bytearray()
    restarts = []
    for i, (k, v) in enumerate(zip(keys, values)):
        s, u = layouts[i]
        if i % restart_interval == 0:
            restarts.append(len(body))
        body += varint_bytes(s) + varint_bytes(u) + varint_bytes(len(v))
        body += k[s:]
        body += v
    for r in restarts:
        body += U32.pack(r)
    body += U32.pack(len(restarts))
    return bytes(body) + U32.pack(crc32(body))


def decode_block(data, offset=None):
    """Verify crc then parse sequentially, ignoring restart offsets (blocks.py:130-165)."""
    if len(data) < 12:
        raise FormatError("block too short")
    data = bytes(data)
    payload = data[:-4]
    if crc32(payload) != U32.unpack_from(data, len(data) - 4)[0]:
        raise CorruptionError("data block checksum mismatch", offset=offset)
    nres = U32.unpack_from(payload, len(payload) - 4)[0]
    end = len(payload) - 4 - 4 * nres
    if nres < 1 or end < 0:
        raise FormatError("bad restart array")
    pairs = []
    pos = 0
    prev = b""
    while pos < end:
        s, pos = varint_read(payload, pos)
        u, pos = varint_read(payload, pos)
        vl, pos = varint_read(payload, pos)
        if s > len(prev) or pos + u + vl > end:
            raise FormatError("truncated block entry")
        key = prev[:s] + payload[pos:pos + u]
        pos += u
        pairs.append((key, payload[pos:pos + vl]))
        pos += vl
        prev = key
    if pos != end:
        raise FormatError("trailing garbage in block entries")
    return pairs


# --------------------------------------------------------------------------
# Bloom filter (bloom.py)
# --------------------------------------------------------------------------

def bloom_probes(bits_per_key: int) -> int:
    """k = round(bpk·ln2) clamped to [1,30] (bloom.py:24-25)."""
    return max(1, min(30, round(bits_per_key * math.log(2))))


def bloom_bits(user_keys, bits_per_key: int):
    """(bits, k) — double hashing in 64-bit without wrap (bloom.py:71-88)."""
    if bits_per_key < 1:
        raise ValueError("bits_per_key must be >= 1")
    user_keys = list(user_keys)
    if not user_keys:
        return b"\x00", 1
    k = bloom_probes(bits_per_key)
    nbits = max(64, len(user_keys) * bits_per_key)
    nbits = (nbits + 7) & ~7
    h = np.array([crc32(x) for x in user_keys], dtype=np.uint64)
    delta = ((h >> np.uint64(17)) | (h << np.uint64(15))) & np.uint64(0xFFFFFFFF)
    bits = np.zeros(nbits // 8, dtype=np.uint8)
    for j in range(k):
        p = (h + np.uint64(j) * delta) % np.uint64(nbits)
        np.bitwise_or.at(bits, (p >> np.uint64(3)).astype(np.int64),
                         np.left_shift(np.uint8(1), (p & np.uint64(7)).astype(np.uint8)))
    return bits.tobytes(), k


def filter_block(bits: bytes, k: int) -> bytes:
    """bits ∥ u8 k ∥ u32 crc (bloom.py:53-55)."""
    body = bits + bytes([k])
    return body + U32.pack(crc32(body))


def parse_filter(data, offset=None):
    """bloom.py:57-68."""
    if len(data) < 6:
        raise FormatError("filter block too short")
    body = data[:-4]
    if crc32(body) != U32.unpack_from(data, len(data) - 4)[0]:
        raise CorruptionError("filter block checksum mismatch", offset=offset)
    k = body[-1]
    if not 1 <= k <= 30:
        raise FormatError(f"bad probe count {k}")
    return bytes(body[:-1]), k


def bloom_may_contain(bits: bytes, k: int, key: bytes) -> bool:
    """bloom.py:91-102 (read path; used by tests only)."""
    n = 8 * len(bits)
    h = crc32(key)
    d = ((h >> 17) | (h << 15)) & 0xFFFFFFFF
    for _ in range(k):
        p = h % n
        if not bits[p >> 3] & (1 << (p & 7)):
            return False
        h = (h + d) & 0xFFFFFFFFFFFFFFFF
    return True


# --------------------------------------------------------------------------
# Index block, SST builder, table parse (sst.py)
# --------------------------------------------------------------------------

def index_block(entries) -> bytes:
    """(varint klen ∥ key ∥ u32 off ∥ u32 len)* ∥ u32 n ∥ u32 crc (sst.py:67-76)."""
    body = bytearray()
    for key, off, ln in entries:
        body += varint_bytes(len(key)) + key + U32.pack(off) + U32.pack(ln)
    body += U32.pack(len(entries))
    return bytes(body) + U32.pack(crc32(body))


def parse_index(data, offset=None):
    """sst.py:79-102."""
    if len(data) < 8:
        raise FormatError("index block too short")
    body = bytes(data[:-4])
    if crc32(body) != U32.unpack_from(data, len(data) - 4)[0]:
        raise CorruptionError("index block checksum mismatch", offset=offset)
    n = U32.unpack_from(body, len(body) - 4)[0]
    end = len(body) - 4
    pos = 0
    out = []
    for _ in range(n):
        klen, pos = varint_read(body, pos)
        if pos + klen + 8 > end:
            raise FormatError("truncated index entry")
        key = body[pos:pos + klen]
        pos += klen
        out.append((key, U32.unpack_from(body, pos)[0], U32.unpack_from(body, pos + 4)[0]))
        pos += 8
    if pos != end:
        raise FormatError("trailing garbage in index block")
    return out


class TableBuilder:
    """Greedy block cut + SST-size signal, restating SstBuilder (sst.py:105-217)."""

    def __init__(self, block_size=4096, restart_interval=16, bits_per_key=10,
                 sst_size_target=4 * 2**20):
        self.block_size = block_size
        self.ri = restart_interval
        self.bpk = bits_per_key
        self.target = sst_size_target
        self.out = bytearray()
        self.keys = []
        self.vals = []
        self.cur_bytes = 0
        self.index = []
        self.user_keys = []
        self.smallest = None
        self.largest = None
        self.last_order = None
        self.done = False

    def _size_with(self, key: bytes, vlen: int) -> int:
        # sst.py:138-151 — pre-checksum size if `key` joined the open block.
        i = len(self.keys)
        s = 0 if i % self.ri == 0 else common_prefix(self.keys[-1], key)
        return self.cur_bytes + entry_size(s, len(key) - s, vlen) + tail_overhead(i + 1, self.ri) - 4

    def add(self, key: bytes, value: bytes):
        # sst.py:153-177
        if self.done:
            raise RuntimeError("builder already finished")
        ok = order_key(key)
        if self.last_order is not None and ok <= self.last_order:
            raise OrderingError(f"keys not strictly ascending at {key!r}")
        if self.keys and self._size_with(key, len(value)) > self.block_size:
            self._flush()
        if self.out and len(self.out) >= self.target:
            raise SizeOverflowError("table exceeds size target; split required")
        self.last_order = ok
        if self.smallest is None:
            self.smallest = key
        self.largest = key
        i = len(self.keys)
        s = 0 if i % self.ri == 0 else common_prefix(self.keys[-1], key)
        self.cur_bytes += entry_size(s, len(key) - s, len(value))
        self.keys.append(key)
        self.vals.append(value)
        self.user_keys.append(ukey(key))

    def _flush(self):
        # sst.py:179-189
        blk = build_block(self.keys, self.vals, block_layouts(self.keys, self.ri), self.ri)
        self.index.append((self.keys[-1], len(self.out), len(blk)))
        self.out += blk
        self.keys, self.vals, self.cur_bytes = [], [], 0

    def finish(self) -> bytes:
        # sst.py:191-209
        if self.done:
            raise RuntimeError("builder already finished")
        if self.keys:
            self._flush()
        if not self.index:
            raise ValueError("cannot build an empty table")
        self.done = True
        bits, k = bloom_bits(self.user_keys, self.bpk)
        fblk = filter_block(bits, k)
        foff = len(self.out)
        self.out += fblk
        ioff = len(self.out)
        iblk = index_block(self.index)
        self.out += iblk
        self.out += FOOTER.pack(foff, len(fblk), ioff, len(iblk), MAGIC)
        return bytes(self.out)


def build_table(pairs, **cfg) -> bytes:
    """build_sst without the meta (sst.py:220-246)."""
    b = TableBuilder(**cfg)
    for k, v in pairs:
        b.add(k, v)
    return b.finish()


def build_tables_split(pairs, **cfg):
    """Stream pairs through builders, cutting on SizeOverflowError."""
    outs = []
    b = TableBuilder(**cfg)
    n = 0
    for k, v in pairs:
        try:
            b.add(k, v)
        except SizeOverflowError:
            outs.append((b.finish(), b.smallest, b.largest))
            b = TableBuilder(**cfg)
            b.add(k, v)
        n += 1
    if b.keys or b.index:
        outs.append((b.finish(), b.smallest, b.largest))
    return outs


def _pread(data, length, offset):
    """os.pread semantics on an in-memory file: short reads past EOF."""
    if offset >= len(data):
        return b""
    return bytes(data[offset:offset + length])


def open_table(data):
    """Footer, magic, filter crc, index crc — Table.__init__ (sst.py:284-310)."""
    if len(data) < FOOTER_SIZE:
        raise FormatError("file too short for footer")
    foff, flen, ioff, ilen, magic = FOOTER.unpack_from(data, len(data) - FOOTER_SIZE)
    if magic != MAGIC:
        raise FormatError(f"bad magic 0x{magic:016x}")
    filt = parse_filter(_pread(data, flen, foff), offset=foff)
    index = parse_index(_pread(data, ilen, ioff), offset=ioff)
    return filt, index


def scan_table(data, index):
    """Table.scan (sst.py:370-375) over an in-memory file."""
    for _, off, ln in index:
        yield from decode_block(_pread(data, ln, off), offset=off)


# --------------------------------------------------------------------------
# Read path: Table.get over an in-memory file
# --------------------------------------------------------------------------

SEEK_TRAILER = (((1 << 56) - 1) << 8) | KIND_PUT  # seek_key (keys.py:66-68)


def _sort_key(ikey):
    """keys.py:60-63 (struct.error on keys shorter than the trailer, as there)."""
    trailer = U64.unpack_from(ikey, len(ikey) - TRAILER)[0]
    return (ikey[:-TRAILER], -trailer)


class BlockReader:
    """DataBlockReader (blocks.py:168-226) over a checksum-verified raw block."""

    def __init__(self, data: bytes):
        self.data = data
        payload_len = len(data) - 4
        n_restarts = U32.unpack_from(data, payload_len - 4)[0]
        self.entries_end = payload_len - 4 - 4 * n_restarts
        if n_restarts < 1 or self.entries_end < 0:
            raise FormatError("bad restart array")
        self.restarts = [U32.unpack_from(data, self.entries_end + 4 * i)[0] for i in range(n_restarts)]

    def entry_at(self, pos: int, prev_key: bytes):
        """blocks.py:188-196: prefix slices and value slices clamp silently."""
        d = self.data
        shared, pos = varint_read(d, pos)
        unshared, pos = varint_read(d, pos)
        vlen, pos = varint_read(d, pos)
        key = prev_key[:shared] + d[pos:pos + unshared]
        pos += unshared
        return key, d[pos:pos + vlen], pos + vlen

    def seek(self, target):
        """blocks.py:202-218: rightmost restart <= target, then one interval."""
        lo, hi = 0, len(self.restarts) - 1
        while lo < hi:
            mid = (lo + hi + 1) // 2
            if _sort_key(self.entry_at(self.restarts[mid], b"")[0]) <= target:
                lo = mid
            else:
                hi = mid - 1
        pos = self.restarts[lo]
        prev = b""
        while pos < self.entries_end:
            key, value, pos = self.entry_at(pos, prev)
            if _sort_key(key) >= target:
                return key, value
            prev = key
        return None


class MemTable:
    """Table (sst.py:284-368) over SST bytes held in memory, no block cache:
    the same checks at open, the same counters, the same get."""

    def __init__(self, data):
        self.data = bytes(data)
        (bits, self.k), self.index = open_table(self.data)
        self.bits = bits
        self.index_sort_keys = [_sort_key(k) for k, _, _ in self.index]  # sst.py:309
        self.filter_rejects = 0
        self.data_block_reads = 0

    def raw_block(self, offset: int, length: int) -> bytes:
        """sst.py:322-340 without a cache."""
        data = _pread(self.data, length, offset)
        if len(data) != length:
            raise FormatError("short block read")
        self.data_block_reads += 1
        stored = U32.unpack_from(data, length - 4)[0]
        if crc32(data[:-4]) != stored:
            raise CorruptionError("data block checksum mismatch", offset=offset)
        return data

    def get(self, user_key: bytes):
        """sst.py:342-368."""
        if not bloom_may_contain(self.bits, self.k, user_key):
            self.filter_rejects += 1
            return None
        target = (user_key, -SEEK_TRAILER)
        lo, hi = 0, len(self.index)
        while lo < hi:
            mid = (lo + hi) // 2
            if self.index_sort_keys[mid] < target:
                lo = mid + 1
            else:
                hi = mid
        if lo == len(self.index):
            return None
        _, off, ln = self.index[lo]
        found = BlockReader(self.raw_block(off, ln)).seek(target)
        if found is None or found[0][:-TRAILER] != user_key:
            return None
        return found


def store_get(tables, l0, levels, user_key: bytes):
    """SPEC.md:185-189 over SSTs only: ``l0`` table ids newest first, then
    ``levels`` = [[(table id, smallest user key, largest user key)] ascending]
    — the one file whose range holds the key; the first table whose get
    returns an entry answers (its kind decides Put vs not-found upstream)."""
    for t in l0:
        r = tables[t].get(user_key)
        if r is not None:
            return t, r
    for files in levels:
        lo, hi = 0, len(files)
        while lo < hi:
            mid = (lo + hi) // 2
            if files[mid][2] < user_key:
                lo = mid + 1
            else:
                hi = mid
        if lo == len(files) or files[lo][1] > user_key:
            continue
        t = files[lo][0]
        r = tables[t].get(user_key)
        if r is not None:
            return t, r
    return None


# --------------------------------------------------------------------------
# Kernel work items (kernels.py) — used for dispatch-level parity tests
# --------------------------------------------------------------------------

TUP_HEAD = struct.Struct("<H")
TUP_TAIL = struct.Struct("<QI")


def tuple_bytes(key: bytes, v_off: int, v_len: int) -> bytes:
    """u16 klen ∥ key ∥ u64 v_off ∥ u32 v_len (kernels.py:35-36)."""
    return TUP_HEAD.pack(len(key)) + key + TUP_TAIL.pack(v_off, v_len)


def tuples_in(buf, start: int, end: int):
    """kernels.py:39-51."""
    out = []
    pos = start
    while pos < end:
        (kl,) = TUP_HEAD.unpack_from(buf, pos)
        pos += 2
        key = bytes(buf[pos:pos + kl])
        pos += kl
        vo, vl = TUP_TAIL.unpack_from(buf, pos)
        pos += 12
        out.append((key, vo, vl))
    return out


def pair_bytes(key: bytes, value: bytes) -> bytes:
    """varint klen ∥ key ∥ value (kernels.py:54-55)."""
    return varint_bytes(len(key)) + key + value


def pair_value(buf, v_off: int, v_len: int) -> bytes:
    """kernels.py:58-61."""
    kl, pos = varint_read(buf, v_off)
    pos += kl
    return bytes(buf[pos:pos + v_len])


def item_unpack(args, regions):
    """kernels.py:72-104."""
    (src, boff, blen, prid, poff, pcap, trid, toff, tcap) = args
    pairs = decode_block(bytes(regions[src][boff:boff + blen]), offset=boff)
    pbuf, tbuf = regions[prid], regions[trid]
    pp, tp, vb = poff, toff, 0
    for k, v in pairs:
        rec = pair_bytes(k, v)
        tup = tuple_bytes(k, pp, len(v))
        if pp + len(rec) > poff + pcap:
            raise BufferError("pair slot overflow")
        if tp + len(tup) > toff + tcap:
            raise BufferError("tuple slot overflow")
        pbuf[pp:pp + len(rec)] = rec
        tbuf[tp:tp + len(tup)] = tup
        pp += len(rec)
        tp += len(tup)
        vb += len(v)
    return (pp - poff, tp - toff, len(pairs), vb)


def item_shared_key(args, regions):
    """kernels.py:107-117."""
    trid, ts, te, ri, lrid, loff = args
    keys = [t[0] for t in tuples_in(regions[trid], ts, te)]
    lay = block_layouts(keys, ri)
    out = regions[lrid]
    pos = loff
    for s, u in lay:
        struct.pack_into("<II", out, pos, s, u)
        pos += 8
    return (len(lay),)


def item_encode(args, regions):
    """kernels.py:120-155."""
    (trid, ts, te, lrid, loff, prid, orid, ooff, ocap, ri) = args
    tups = tuples_in(regions[trid], ts, te)
    lbuf = regions[lrid]
    lay = [struct.unpack_from("<II", lbuf, loff + 8 * i) for i in range(len(tups))]
    pbuf = regions[prid]
    keys = [t[0] for t in tups]
    vals = [pair_value(pbuf, vo, vl) for _, vo, vl in tups]
    blk = build_block(keys, vals, lay, ri)
    if len(blk) > ocap:
        raise BufferError("encode slot overflow")
    regions[orid][ooff:ooff + len(blk)] = blk
    return (len(blk), sum(vl for _, _, vl in tups))


def item_filter(args, regions):
    """kernels.py:158-168."""
    trid, ts, te, bpk, orid, ooff, ocap = args
    uks = [k[:-8] for k, _, _ in tuples_in(regions[trid], ts, te)]
    enc = filter_block(*bloom_bits(uks, bpk))
    if len(enc) > ocap:
        raise BufferError("filter slot overflow")
    regions[orid][ooff:ooff + len(enc)] = enc
    return (len(enc),)


ITEMS = {"unpack": item_unpack, "shared_key": item_shared_key,
         "encode": item_encode, "filter": item_filter}


def run_item(kind, args, regions):
    """run_item_safe tagging (kernels.py:185-192)."""
    try:
        return ("ok", ITEMS[kind](args, regions))
    except CorruptionError as exc:
        return ("corrupt", str(exc), exc.offset)
    except Exception as exc:  # noqa: BLE001
        return ("err", f"{type(exc).__name__}: {exc}")


# --------------------------------------------------------------------------
# Compaction composition (SPEC reference_compact)
# --------------------------------------------------------------------------

def covered(user_key: bytes, ranges) -> bool:
    """Version.covers_below over pre-extracted closed user-key ranges (version.py:122-128)."""
    for lo, hi in ranges:
        if lo <= user_key <= hi:
            return True
    return False


def merge_resolve(runs, deeper=()):
    """heapq merge on order_key, newest per user key, D12 tombstone drop."""
    for r, run in enumerate(runs):
        for a, b in zip(run, run[1:]):
            if order_key(a[0]) >= order_key(b[0]):
                raise OrderingError(f"input run {r} not strictly ascending")
    merged = heapq.merge(*runs, key=lambda kv: order_key(kv[0]))
    prev_user = None
    for k, v in merged:
        u = ukey(k)
        if u == prev_user:
            continue
        prev_user = u
        if kind_of(k) == KIND_DELETE and not covered(u, deeper):
            continue
        yield k, v


def reference_compact(files, *, deeper=(), block_size=4096, restart_interval=16,
                      bits_per_key=10, sst_size_target=4 * 2**20, key_range=None):
    """Compact input files (bytes, lower first then upper) into output SSTs.

    Returns a list of (sst_bytes, smallest_ikey, largest_ikey) in key order.
    ``key_range=(lo, hi)`` (None = open end) keeps user keys in [lo, hi): the
    per-range reference of a subcompaction.
    """
    opened = [open_table(f) for f in files]          # all footers/filters/indexes first
    runs = [list(scan_table(f, idx)) for f, (_, idx) in zip(files, opened)]
    survivors = merge_resolve(runs, deeper)
    if key_range is not None:
        lo, hi = key_range
        survivors = (kv for kv in survivors
                     if (lo is None or ukey(kv[0]) >= lo) and (hi is None or ukey(kv[0]) < hi))
    return build_tables_split(survivors, block_size=block_size,
                              restart_interval=restart_interval,
                              bits_per_key=bits_per_key, sst_size_target=sst_size_target)
