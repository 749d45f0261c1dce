"""Probe the storage <-> HBM paths on the GPU box step by step (each step
flushed, so a hang shows where): luda_gds_status (cuFileDriverOpen), a bounce
read, a cuFile read. Run under `timeout`."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2004_03054_b200 import _native  # noqa: E402

L = _native.lib(0)
p = "/tmp/gds_probe.bin"
data = os.urandom(3 << 20)
open(p, "wb").write(data)
dev = ctypes.c_void_p()
_native.check(L.luda_region_alloc(len(data) + 64, ctypes.byref(dev)))
paths = (ctypes.c_char_p * 1)(p.encode())
off = (ctypes.c_uint64 * 1)(0)
ln = (ctypes.c_uint64 * 1)(len(data))
used = ctypes.c_int()
steps = sys.argv[1:] or ["bounce", "status", "gds"]
for s in steps:
    t = time.perf_counter()
    print("step", s, flush=True)
    if s == "status":
        buf = ctypes.create_string_buffer(256)
        r = L.luda_gds_status(buf, 256)
        print("  gds_status", r, buf.value.decode(), flush=True)
    else:
        rc = L.luda_files_read(paths, 1, dev.value, off, ln, 2 if s == "bounce" else 1, ctypes.byref(used))
        print("  rc", rc, used.value, L.luda_last_error().decode(), flush=True)
    print("  %.3f s" % (time.perf_counter() - t), flush=True)
