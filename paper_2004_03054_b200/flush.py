"""Build SSTs on the GPU from sorted (internal_key, value) pairs.

This is the L0 producer of SURVEY §8(f) rank 1 (memtable flush → ``build_sst``,
sst.py:220-246) and the bench's input synthesiser. It reuses the compaction
back half unchanged (block planner, encoder, filter/index/footer kernels), so
the bytes equal ``SstBuilder`` output with the SizeOverflowError cut rule.
"""

from __future__ import annotations

import ctypes
import struct

import numpy as np

from . import _native

_TR = struct.Struct("<Q")


class DeviceArrays:
    """Device copies of flat key / trailer / value arrays (luda_region_alloc).
    ``key_lens`` (generic-length keys): per-key user-key lengths."""

    def __init__(self, L, keys: bytes, trailers: np.ndarray, values: bytes, voff: np.ndarray, vlen: np.ndarray,
                 stream, key_lens=None):
        self.L = _native.load()
        self.ptrs = []
        self.n = len(trailers)
        self.keys = self._put(keys, stream)
        self.trailers = self._put(trailers.astype(np.uint64).tobytes(), stream)
        self.values = self._put(b"\0" * 64 + values + b"\0" * 64, stream) + 64
        self.voff = self._put(voff.astype(np.uint64).tobytes(), stream)
        self.vlen = self._put(vlen.astype(np.uint32).tobytes(), stream)
        self.klen = L
        self.max_key_len = 0
        if key_lens is not None:
            kl = np.asarray(key_lens, dtype=np.uint32)
            ko = np.zeros(len(kl), dtype=np.uint64)
            if len(kl) > 1:
                ko[1:] = np.cumsum(kl[:-1], dtype=np.uint64)
            self.key_off = self._put(ko.tobytes(), stream)
            self.key_len = self._put(kl.tobytes(), stream)
            self.max_key_len = int(kl.max()) if len(kl) else 0

    def _put(self, data: bytes, stream):
        p = ctypes.c_void_p()
        _native.check(self.L.luda_region_alloc(max(1, len(data)), ctypes.byref(p)))
        self.ptrs.append(p.value)
        if data:
            buf = ctypes.create_string_buffer(data, len(data))
            _native.check(self.L.luda_stage_in_async(p.value, buf, len(data), stream))
            _native.check(self.L.luda_stream_sync(stream))
        return p.value

    def free(self):
        for p in self.ptrs:
            self.L.luda_region_free(p)
        self.ptrs.clear()


def pack_pairs(pairs):
    """(ikey, value) list → (L, keys, trailers, values, voff, vlen); L = None
    when the user keys differ in length or are longer than 32 bytes (the
    generic-length builder; keys then carry their own offsets / lengths)."""
    if not pairs:
        raise ValueError("cannot build an empty table")
    L = len(pairs[0][0]) - 8
    if any(len(k) < 8 for k, _ in pairs):
        raise ValueError("internal keys are at least 8 bytes (keys.py:39)")
    if L > 32 or any(len(k) - 8 != L for k, _ in pairs):
        L = None
    keys = b"".join(k[:-8] for k, _ in pairs)
    trailers = np.array([_TR.unpack_from(k, len(k) - 8)[0] for k, _ in pairs], dtype=np.uint64)
    vlen = np.array([len(v) for _, v in pairs], dtype=np.uint32)
    voff = np.zeros(len(pairs), dtype=np.uint64)
    if len(pairs) > 1:
        voff[1:] = np.cumsum(vlen[:-1], dtype=np.uint64)
    values = b"".join(v for _, v in pairs)
    return L, keys, trailers, values, voff, vlen


def build_from_device(arrs: DeviceArrays, *, stream, block_size=4096, restart_interval=16, bits_per_key=10,
                      sst_size_target=4 * 2**20):
    """Run luda_build_from_sorted; returns the (device-owned) JobResult."""
    L = _native.load()
    res = _native.JobResult()
    if arrs.klen is None:  # generic-length keys
        _native.check(L.luda_build_from_sorted_var(arrs.keys, arrs.key_off, arrs.key_len, arrs.max_key_len,
                                                   arrs.trailers, arrs.values, arrs.voff, arrs.vlen, arrs.n,
                                                   block_size, restart_interval, bits_per_key, sst_size_target,
                                                   ctypes.byref(res), stream))
        return res
    _native.check(L.luda_build_from_sorted(arrs.keys, arrs.klen, arrs.trailers, arrs.values, arrs.voff, arrs.vlen,
                                           arrs.n, block_size, restart_interval, bits_per_key, sst_size_target,
                                           ctypes.byref(res), stream))
    return res


def result_files(res, stream):
    """D2H all SSTs of a JobResult → [(bytes, smallest, largest)] and release it."""
    L = _native.load()
    try:
        if res.n_sst == 0:
            return []
        buf = ctypes.create_string_buffer(res.out_bytes)
        _native.check(L.luda_stage_out_async(buf, res.out, res.out_bytes, stream))
        _native.check(L.luda_stream_sync(stream))
        raw = buf.raw
        out = []
        for i, (sm, lg) in enumerate(_native.sst_key_pairs(res)):
            o, n = res.sst_off[i], res.sst_len[i]
            out.append((raw[o:o + n], sm, lg))
        return out
    finally:
        L.luda_job_release(ctypes.byref(res))


def build_ssts(pairs, *, device_ordinal=0, block_size=4096, restart_interval=16, bits_per_key=10,
               sst_size_target=4 * 2**20):
    """Sorted pairs → [(sst_bytes, smallest, largest)], byte-identical to
    SstBuilder with the SizeOverflowError → finish → new builder rule."""
    L = _native.lib(device_ordinal)
    s = ctypes.c_void_p()
    _native.check(L.luda_stream_create(ctypes.byref(s)))
    packed = pack_pairs(pairs)
    arrs = DeviceArrays(*packed, s.value, key_lens=[len(k) - 8 for k, _ in pairs] if packed[0] is None else None)
    try:
        res = build_from_device(arrs, stream=s.value, block_size=block_size, restart_interval=restart_interval,
                                bits_per_key=bits_per_key, sst_size_target=sst_size_target)
        return result_files(res, s.value)
    finally:
        arrs.free()
        L.luda_stream_destroy(s.value)
