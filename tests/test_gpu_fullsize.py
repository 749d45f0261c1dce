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

from oracle import luda_oracle as O

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


TARGET = 4 * 2**20


def _index_last(sst: bytes):
    """(data bytes, last block length) of one SST from its footer + index (sst.py:67-76)."""
    foff, flen, ioff, ilen, _ = O.FOOTER.unpack_from(sst, len(sst) - O.FOOTER_SIZE)
    idx = O.parse_index(sst[ioff:ioff + ilen])
    return foff, idx[-1][2]


def check_sst_cuts(out: np.ndarray, offs, lens, target=TARGET):
    """The SST cut rule (sst.py:161-162) over EVERY output:
    a non-last SST closes right after the first block whose flush makes its
    data bytes >= target."""
    for i, (o, ln) in enumerate(zip(offs, lens)):
        data, last = _index_last(out[o:o + ln].tobytes())
        if i + 1 < len(offs):
            assert data >= target and data - last < target, (i, data, last)
        else:
            assert data - last < target or data < target, (i, data, last)


def check_rebuild(out: np.ndarray, offs, lens, picks, target=TARGET):
    """Each sampled SST, decoded and rebuilt by the oracle's SstBuilder at the
    same target, comes back as exactly one byte-identical SST: its block cuts,
    restarts, shared prefixes, CRCs, filter, index and footer are the
    reference's. Returns the decoded entries per pick."""
    got = {}
    for i in picks:
        sst = out[offs[i]:offs[i] + lens[i]].tobytes()
        _, index = O.open_table(sst)
        pairs = list(O.scan_table(sst, index))
        rebuilt = O.build_tables_split(pairs, sst_size_target=target)
        assert len(rebuilt) == 1 and rebuilt[0][0] == sst, i
        got[i] = pairs
    return got


def test_c3_full_size_accounting_and_recompaction_identity():
    import bench
    from paper_2004_03054_b200 import _native
    import torch
    torch.cuda.set_device(0)
    L = _native.lib(0)
    keys = int(os.environ.get("LUDA_FULL_KEYS", 1 << 25))
    w = bench.synth_c3(keys, seed=0xC3, device_index=0, keep_truth=True)
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
            check_sst_cuts(a, offs, lens)
            picks = sorted({0, 1, n // 3, n // 2, n - 2, n - 1})
            decoded = check_rebuild(a, offs, lens, picks)
            check_against_generator(w, keys, decoded)
        finally:
            L.luda_job_release(ctypes.byref(res2))
    finally:
        L.luda_job_release(ctypes.byref(res))


def check_against_generator(w, n, decoded):
    """Survivors of the sampled SSTs vs the generator (bench.synth_c3): every
    entry is the Li (newest) version of its key — seq n + 1 + index, a Put
    whose value is the generator's bytes — and its key was not deleted; the
    SSTs' entries are consecutive surviving keys."""
    import torch
    keys_d, values_d, voff_lo, is_del = w.truth
    kh = keys_d.view(-1, 16)[:, :8].cpu().numpy().copy().view(">u8").reshape(-1).astype(np.uint64)
    alive = (~is_del).cpu().numpy()
    for i, pairs in decoded.items():
        uk = np.frombuffer(b"".join(k[:8] for k, _ in pairs), dtype=">u8").astype(np.uint64)
        idx = np.searchsorted(kh, uk)
        assert (idx < n).all() and (kh[idx] == uk).all(), i
        full = keys_d.view(-1, 16)[torch.from_numpy(idx).to(keys_d.device)].cpu().numpy()
        assert [bytes(r) for r in full] == [k[:16] for k, _ in pairs], i
        tr = [int.from_bytes(k[16:], "little") for k, _ in pairs]
        assert [t >> 8 for t in tr] == (idx + n + 1).tolist(), i
        assert all(t & 0xFF == O.KIND_PUT for t in tr) and alive[idx].all(), i
        # consecutive survivors: no live key between two neighbours of one SST
        live_rank = np.cumsum(alive) - 1
        assert (np.diff(live_rank[idx]) == 1).all(), i
        offs = voff_lo[torch.from_numpy(idx).to(voff_lo.device)]
        cols = torch.arange(128, device=offs.device)
        vals = values_d[(offs[:, None] + cols[None, :]).reshape(-1)].view(-1, 128).cpu().numpy()
        assert [bytes(r) for r in vals] == [v for _, v in pairs], i


def _desc(_native, arena_ptr, arena_bytes, offs, lens, run_first):
    fo = (ctypes.c_uint64 * len(offs))(*offs)
    fl = (ctypes.c_uint64 * len(lens))(*lens)
    rf = (ctypes.c_uint32 * len(run_first))(*run_first)
    d = _native.JobDesc()
    d.arena, d.arena_bytes, d.n_files = arena_ptr, arena_bytes, len(offs)
    d.file_off = ctypes.cast(fo, _native.c_u64p)
    d.file_len = ctypes.cast(fl, _native.c_u64p)
    d.n_runs = len(run_first) - 1
    d.run_first_file = ctypes.cast(rf, _native.c_u32p)
    d.block_size, d.restart_interval, d.bits_per_key, d.sst_size_target = 4096, 16, 10, 4 * 2**20
    return d, (fo, fl, rf)


def test_c4_scaled_eight_runs_accounting_and_recompaction_identity():
    """c4 scaled: 8 fully overlapping L0 runs x 2^22 keys (24-byte keys, W = 3
    records, 256-byte values, 3 merge passes) → every entry survives, outputs
    sorted into 4 MiB SSTs; re-compacting them is the identity."""
    from paper_2004_03054_b200 import _native
    import torch
    torch.cuda.set_device(0)
    L = _native.lib(0)
    n = int(os.environ.get("LUDA_C4_KEYS", 1 << 22))
    s = ctypes.c_void_p()
    _native.check(L.luda_stream_create(ctypes.byref(s)))
    import bench
    arena, offs, lens = bench.synth_c4(L, 8, n, 0xC4, s.value)
    desc, keep = _desc(_native, arena.data_ptr(), arena.numel(), offs, lens, list(range(9)))
    res = _native.JobResult()
    _native.check(L.luda_compact(ctypes.byref(desc), ctypes.byref(res), s.value))
    try:
        assert res.n_in == 8 * n and res.n_out == 8 * n
        m = res.n_sst
        o1 = [res.sst_off[i] for i in range(m)]
        l1 = [res.sst_len[i] for i in range(m)]
        d2, keep2 = _desc(_native, res.out, res.out_bytes, o1, l1, [0, m])
        res2 = _native.JobResult()
        _native.check(L.luda_compact(ctypes.byref(d2), ctypes.byref(res2), s.value))
        try:
            assert res2.n_out == res.n_out and res2.n_sst == m
            assert [res2.sst_len[i] for i in range(m)] == l1
            a = _host(L, res.out, res.out_bytes, s.value)
            b = _host(L, res2.out, res2.out_bytes, s.value)
            assert np.array_equal(a, b)
            check_sst_cuts(a, o1, l1)
            check_rebuild(a, o1, l1, sorted({0, m // 2, m - 1}))
        finally:
            L.luda_job_release(ctypes.byref(res2))
    finally:
        L.luda_job_release(ctypes.byref(res))
        L.luda_stream_destroy(s.value)
