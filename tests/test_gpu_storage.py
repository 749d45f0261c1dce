"""Storage ↔ HBM staging: run_compaction reading its input
SSTs from a directory straight into device memory (luda_files_read) and
writing its outputs from device memory to files (luda_files_write), through
cuFile (GPUDirect Storage, compatibility mode where nvidia-fs is absent) and
through the native pinned-bounce pipeline. Output files must be byte-identical
to the oracle's compaction."""

import ctypes
import os

import pytest

from oracle import jobgen
from oracle import luda_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    from paper_2004_03054_b200 import DeviceConfig, make_device
    d = make_device(DeviceConfig(backend="b200"))
    yield d
    d.close()


def _job_on_disk(tmp_path, n=6000, seed=0xC3):
    from paper_2004_03054_b200 import CompactionJob, SstMeta, Version
    job = jobgen.c3(n=n, seed=seed, sst_target=96 * 1024)
    lower = O.build_tables_split(job.lower[0].pairs, sst_size_target=96 * 1024)
    upper = O.build_tables_split(job.upper[0].pairs, sst_size_target=96 * 1024)
    fid = 1
    metas = {1: [], 2: []}
    for level, outs in ((1, lower), (2, upper)):
        for data, sm, lg in outs:
            (tmp_path / f"{fid}.sst").write_bytes(data)
            metas[level].append(SstMeta(file_id=fid, file_size=len(data), smallest=sm, largest=lg, level=level))
            fid += 1
    v = Version([[], metas[1], metas[2]] + [[] for _ in range(4)])
    cj = CompactionJob(source_level=1, lower=metas[1], upper=metas[2], target_level=2, version=v)
    want = O.reference_compact([f for f, _, _ in lower + upper], sst_size_target=128 * 1024)
    return cj, want


def gds_mode(dev):
    buf = ctypes.create_string_buffer(256)
    return dev._L.luda_gds_status(buf, 256), buf.value.decode()


@pytest.mark.parametrize("io", ["auto", "bounce", "gds"])
def test_run_compaction_storage_to_storage(dev, tmp_path, io):
    from paper_2004_03054_b200 import UnsupportedInputError, run_compaction
    from paper_2004_03054_b200.compaction import runner_for
    from paper_2004_03054_b200.config import StoreConfig
    ok, why = gds_mode(dev)
    if io == "gds" and not ok:
        job, _ = _job_on_disk(tmp_path)
        with pytest.raises(UnsupportedInputError):
            run_compaction(job, dev, directory=str(tmp_path), io="gds", out_directory=str(tmp_path / "o"),
                           config=StoreConfig(sst_size_target=128 * 1024))
        return
    job, want = _job_on_disk(tmp_path)
    out_dir = tmp_path / "out"
    out_dir.mkdir()
    results, stats = run_compaction(job, dev, directory=str(tmp_path), io=io, out_directory=str(out_dir),
                                    config=StoreConfig(sst_size_target=128 * 1024))
    assert len(results) == len(want)
    for (path, meta), (data, sm, lg) in zip(results, want):
        assert open(path, "rb").read() == data
        assert meta.file_size == len(data) and meta.smallest == sm and meta.largest == lg
        assert os.path.basename(path) == f"{meta.file_id}.sst"
    r = runner_for(dev)
    if io == "bounce":
        assert r.last_io == "bounce" and r.last_io_out == "bounce"
    if io == "gds":
        assert r.last_io == "gds" and r.last_io_out == "gds"
    print(f"io={io}: in {r.last_io}, out {r.last_io_out}; cuFile: {why}")


def test_files_read_large_and_unaligned(dev, tmp_path):
    """Files larger than one bounce chunk (8 MiB) and odd sizes / destination
    offsets, both paths, byte-exact after a D2H."""
    from paper_2004_03054_b200 import _native
    L = dev._L
    rng = __import__("random").Random(9)
    sizes = [1, 4095, 8 << 20, (8 << 20) + 3, 20_000_001, 0, 77]
    blobs = [rng.randbytes(s) for s in sizes]
    paths = []
    for i, b in enumerate(blobs):
        p = tmp_path / f"f{i}"
        p.write_bytes(b)
        paths.append(str(p).encode())
    offs, o = [], 5
    for s in sizes:
        offs.append(o)
        o += s + 3
    region = dev.alloc(o + 16)
    n = len(sizes)
    try:
        for mode in (2, 0):
            used = ctypes.c_int()
            _native.check(L.luda_files_read((ctypes.c_char_p * n)(*paths), n, region.dptr,
                                            (ctypes.c_uint64 * n)(*offs), (ctypes.c_uint64 * n)(*sizes), mode,
                                            ctypes.byref(used)))
            host = (ctypes.c_uint8 * (o + 16))()
            st = dev.stream("io-test")
            _native.check(L.luda_stage_out_async(host, region.dptr, o + 16, st))
            _native.check(L.luda_stream_sync(st))
            got = bytes(host)
            for b, off in zip(blobs, offs):
                assert got[off:off + len(b)] == b, (mode, used.value, len(b))
            # and back out through luda_files_write
            outp = [str(tmp_path / f"w{mode}_{i}").encode() for i in range(n)]
            _native.check(L.luda_files_write((ctypes.c_char_p * n)(*outp), n, region.dptr,
                                             (ctypes.c_uint64 * n)(*offs), (ctypes.c_uint64 * n)(*sizes), mode,
                                             ctypes.byref(used)))
            for b, p in zip(blobs, outp):
                assert open(p, "rb").read() == b
    finally:
        dev.free(region)


def test_missing_input_file_fails_loudly(dev, tmp_path):
    from paper_2004_03054_b200 import DeviceError
    from paper_2004_03054_b200 import _native
    L = dev._L
    region = dev.alloc(64)
    try:
        p = (ctypes.c_char_p * 1)(str(tmp_path / "nope.sst").encode())
        with pytest.raises(DeviceError, match="open failed"):
            _native.check(L.luda_files_read(p, 1, region.dptr, (ctypes.c_uint64 * 1)(0), (ctypes.c_uint64 * 1)(10),
                                            2, None))
    finally:
        dev.free(region)
