"""Batched read path over HBM-resident SSTs.

Mirrors the reference's ``Table`` (sst.py:281-375) for many keys at once:
``DeviceTables(files, device)`` opens every file like ``Table.__init__``
(footer, magic, filter CRC, index CRC — the first failing file raises the
reference's exception) and keeps the files in device memory;
``get(t, key)`` / ``multi_get(keys, tables)`` are ``Table.get`` (bloom probe →
index binary search → block CRC → restart binary search → one interval scan);
``store_get(keys)`` probes in the SPEC store order over the
levels given to ``set_levels``. ``filter_rejects`` / ``data_block_reads``
are the reference's per-table counters.

``DeviceTables.from_job(device, result)`` opens a compaction's output buffer
in place (no copy): the read path consumes what the GPU compaction wrote.
There is no CPU fallback: every call goes through ``libluda_b200.so``.
"""

from __future__ import annotations

import ctypes

from . import _native, errors

KEY_CAP = 264  # bytes reserved per found internal key: user keys up to 256 bytes (longer: UnsupportedInputError)

# luda_read.cuh GetStatus → reference exception class
_ERR = {2: errors.FormatError, 3: errors.CorruptionError, 4: errors.FormatError, 5: errors.FormatError,
        6: errors.FormatError, 7: errors.FormatError, 8: errors.UnsupportedInputError}
_MSG = {2: "short block read", 3: "data block checksum mismatch", 4: "bad restart array", 5: "truncated varint",
        6: "varint too long", 7: "fixed-width field past the end of its buffer (struct.error in the reference)",
        8: "found key longer than the result slot"}
STRUCT_ERROR = 7


ProbePlan = _native.ProbePlan
GetResult = _native.GetResult


def _u32(xs):
    return (ctypes.c_uint32 * max(1, len(xs)))(*xs)


def _u64(xs):
    return (ctypes.c_uint64 * max(1, len(xs)))(*xs)


def _pack_keys(keys):
    keys = [bytes(k) for k in keys]
    blob = b"".join(keys)
    offs, o = [], 0
    for k in keys:
        offs.append(o)
        o += len(k)
    return blob, offs, [len(k) for k in keys]


class DeviceTables:
    """A set of SSTs resident in device memory with batched ``Table.get``."""

    def __init__(self, files=None, device=None, *, stream: str = "read", _attach=None):
        if device is None:
            raise errors.DeviceError("DeviceTables needs a b200 device (no CPU fallback)")
        self.device = device
        self._L = device._L
        self._stream = device.stream(stream)
        self._region = None
        self._owner = None
        if _attach is not None:
            arena, offs, lens, self._owner = _attach
        else:
            files = [memoryview(f).cast("B") for f in files]
            offs, o = [], 0
            for f in files:
                offs.append(o)
                o += (len(f) + 15) & ~15
            self._region = device.alloc(max(o, 16), label="tables")
            arena = self._region.dptr
            for f, off in zip(files, offs):
                if len(f):
                    buf = (ctypes.c_uint8 * len(f)).from_buffer_copy(f)
                    _native.check(self._L.luda_stage_in_async(arena + off, buf, len(f), self._stream))
                    _native.check(self._L.luda_stream_sync(self._stream))
            lens = [len(f) for f in files]
        self.n = len(offs)
        h = ctypes.c_void_p()
        try:
            _native.check(self._L.luda_tables_open(arena, _u64(offs), _u64(lens), self.n, ctypes.byref(h),
                                                   self._stream))
        except Exception:
            self._free_region()
            raise
        self._h = h.value
        self._has_plan = False

    @classmethod
    def from_job(cls, device, result, *, stream: str = "read"):
        """Open the output SSTs of a ``luda_compact`` result in place; the
        result must stay alive (not released) while the table set is used."""
        offs = [result.sst_off[i] for i in range(result.n_sst)]
        lens = [result.sst_len[i] for i in range(result.n_sst)]
        return cls(None, device, stream=stream, _attach=(result.out, offs, lens, result))

    # -- lifecycle -------------------------------------------------------------
    def _free_region(self):
        if self._region is not None:
            self.device.free(self._region)
            self._region = None

    def close(self):
        if getattr(self, "_h", None):
            self._L.luda_tables_close(self._h)
            self._h = None
        self._free_region()
        self._owner = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __len__(self):
        return self.n

    # -- counters (sst.py:296-297) ----------------------------------------------
    def counters(self):
        rej = (ctypes.c_uint64 * max(1, self.n))()
        rd = (ctypes.c_uint64 * max(1, self.n))()
        _native.check(self._L.luda_tables_counters(self._h, rej, rd))
        return list(rej)[:self.n], list(rd)[:self.n]

    @property
    def filter_rejects(self):
        return self.counters()[0]

    @property
    def data_block_reads(self):
        return self.counters()[1]

    # -- store order ----------------------------------------------------------
    def set_levels(self, l0, levels):
        """``l0``: table ids newest first; ``levels``: per level >= 1 a list of
        (table id, smallest user key, largest user key), ascending."""
        first, tabs, rk, rl = [0], [], [], []
        for files in levels:
            for t, lo, hi in files:
                tabs.append(t)
                rk += [bytes(lo), bytes(hi)]
                rl += [len(lo), len(hi)]
            first.append(len(tabs))
        blob = b"".join(rk)
        keybuf = (ctypes.c_uint8 * max(1, len(blob))).from_buffer_copy(blob + b"\0")
        plan = ProbePlan(len(l0), _u32(l0), len(levels), _u32(first), _u32(tabs), keybuf, _u32(rl))
        _native.check(self._L.luda_tables_set_plan(self._h, ctypes.byref(plan), self._stream))
        self._has_plan = True

    # -- lookups ----------------------------------------------------------------
    def _run(self, keys, tables):
        n = len(keys)
        blob, offs, lens = _pack_keys(keys)
        kb = (ctypes.c_uint8 * max(1, len(blob))).from_buffer_copy(blob + b"\0")
        res = GetResult()
        qt = _u32(tables) if tables is not None else None
        fixed = len(set(lens)) == 1  # one key length: no per-key offsets / lengths to ship
        st = self._L.luda_tables_get(self._h, kb, len(blob), None if fixed else _u64(offs),
                                     _u32(lens[:1] if fixed else lens), n, qt, KEY_CAP, ctypes.byref(res),
                                     self._stream)
        return st, res

    def _decode(self, st, res, n, store, errors_mode):
        if st != 0 and res.n != n:  # failed before any lookup ran
            _native.check(st)
        packed = ctypes.string_at(res.packed, res.packed_bytes) if res.packed_bytes else b""
        out = []
        for i in range(n):
            s = res.status[i]
            if s == 0:
                out.append(None)
                continue
            if s == 1:
                p, kl, vl = res.pos[i], res.key_len[i], res.value_len[i]
                kv = (packed[p:p + kl], packed[p + kl:p + kl + vl])
                out.append((res.table[i], kv) if store else kv)
                continue
            if errors_mode == "raise":
                _native.check(st)  # the first failing key's error (sequential get semantics)
            off = res.err_off[i]
            out.append(_ERR[s](_MSG[s], offset=off) if s == 3 else _ERR[s](_MSG[s]))
        if errors_mode == "raise" and st != 0:
            _native.check(st)
        return out

    def multi_get(self, keys, tables, *, errors_mode: str = "raise"):
        """``Table.get(key)`` of ``tables[i]`` (or one table id for all keys)
        for every key. ``errors_mode="raise"``: raise the first failing key's
        error, as a sequential loop of gets would; ``"return"``: per-key
        exception objects in place of results."""
        keys = list(keys)
        if isinstance(tables, int):
            tables = [tables] * len(keys)
        tables = list(tables)
        if len(tables) != len(keys):
            raise ValueError("one table id per key")
        if not keys:
            return []
        st, res = self._run(keys, tables)
        return self._decode(st, res, len(keys), False, errors_mode)

    def get(self, table: int, user_key: bytes):
        """Table.get (sst.py:342-368) on one table."""
        return self.multi_get([user_key], [table])[0]

    def store_get(self, keys, *, errors_mode: str = "raise"):
        """SPEC store-order lookups over the SST levels set
        by ``set_levels``: (table id, (internal key, value)) of the first
        table that returns an entry, or None. The caller applies the kind
        (Delete → not found) and consults its memtables first."""
        if not self._has_plan:
            raise errors.DeviceError("set_levels() first")
        keys = list(keys)
        if not keys:
            return []
        st, res = self._run(keys, None)
        return self._decode(st, res, len(keys), True, errors_mode)

    # -- device-resident lookups (throughput) ---------------------------------------
    def lookup_dev(self, dkeys, dkoff, dklen, n, dtables=None, stream=None):
        """The lookup kernel alone over device buffers (pointers); async."""
        _native.check(self._L.luda_tables_lookup_dev(self._h, dkeys, dkoff, dklen, n, dtables, KEY_CAP,
                                                     stream if stream is not None else self._stream))
