"""Full-size (BASELINE c3: 2 x 2^25 keys, 9.6 GB in) parity through
size-independent properties, all through the C ABI:

* entry accounting: n_in = 2 x keys; survivors = keys minus the Li run's
  deletes (tombstones are dropped at the bottom level, SPEC D12);
* idempotence: the output SSTs, compacted again as one bottom-level run, come
  back byte-identical (same block cuts, same SST cuts — the SizeOverflowError
  rule of sst.py:161-162 —, same filters, indexes, footers and metas), which
  re-verifies every output CRC, footer, filter and index on the way in.

The oracle cannot run at this size; the small-size byte-for-byte parity is
tests/test_gpu_parity.py."""

import ctypes
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _host(L, ptr, n, stream):
    from paper_2004_03054_b200 import _native
    from paper_2004_03054_b200.device import PinnedBuffer
    pin = PinnedBuffer()
    pin.ensure(max(n, 1))
    _native.check(L.luda_stage_out_async(pin.ptr, ptr, n, stream))
    _native.check(L.luda_stream_sync(stream))
    out = np.ctypeslib.as_array((ctypes.c_uint8 * n).from_address(pin.ptr)).copy()
    pin.free()
    return out


def test_c3_full_size_accounting_and_recompaction_identity():
    import bench
    from paper_2004_03054_b200 import _native
    import torch
    torch.cuda.set_device(0)
    L = _native.lib(0)
    keys = int(os.environ.get("LUDA_FULL_KEYS", 1 << 25))
    w = bench.synth_c3(keys, seed=0xC3, device_index=0)
    desc, keep = bench.job_desc(w, w.arena.data_ptr())
    res = _native.JobResult()
    _native.check(L.luda_compact(ctypes.byref(desc), ctypes.byref(res), w.stream))
    try:
        assert res.n_in == 2 * keys
        assert res.n_out == w.n_out_expected, (res.n_out, w.n_out_expected)
        n = res.n_sst
        offs = [res.sst_off[i] for i in range(n)]
        lens = [res.sst_len[i] for i in range(n)]
        assert offs[0] == 0 and all(offs[i] + lens[i] == offs[i + 1] for i in range(n - 1))
        # the outputs as the input of a second (bottom-level, single-run) compaction
        fo = (ctypes.c_uint64 * n)(*offs)
        fl = (ctypes.c_uint64 * n)(*lens)
        rf = (ctypes.c_uint32 * 2)(0, n)
        d2 = _native.JobDesc()
        d2.arena, d2.arena_bytes, d2.n_files = res.out, res.out_bytes, n
        d2.file_off = ctypes.cast(fo, _native.c_u64p)
        d2.file_len = ctypes.cast(fl, _native.c_u64p)
        d2.n_runs = 1
        d2.run_first_file = ctypes.cast(rf, _native.c_u32p)
        d2.block_size, d2.restart_interval, d2.bits_per_key, d2.sst_size_target = desc.block_size, \
            desc.restart_interval, desc.bits_per_key, desc.sst_size_target
        res2 = _native.JobResult()
        _native.check(L.luda_compact(ctypes.byref(d2), ctypes.byref(res2), w.stream))
        try:
            assert res2.n_in == res.n_out and res2.n_out == res.n_out
            assert res2.n_sst == n and [res2.sst_len[i] for i in range(n)] == lens
            K = res.key_len
            k1 = bytes((ctypes.c_uint8 * (2 * n * K)).from_address(ctypes.addressof(res.sst_keys.contents)))
            k2 = bytes((ctypes.c_uint8 * (2 * n * K)).from_address(ctypes.addressof(res2.sst_keys.contents)))
            assert k1 == k2  # smallest / largest internal key of every output SST
            a = _host(L, res.out, res.out_bytes, w.stream)
            b = _host(L, res2.out, res2.out_bytes, w.stream)
            assert a.size == b.size and np.array_equal(a, b)
        finally:
            L.luda_job_release(ctypes.byref(res2))
    finally:
        L.luda_job_release(ctypes.byref(res))
