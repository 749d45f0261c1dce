"""c2 (1 L1 + 10 L2 SSTs of 2 MB, 16 B keys / 1 KB values) phase breakdown
(experiment): median over jobs of the device phase times luda_compact
records with events (res.t_ms) and of the call's host wall time."""
import ctypes
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2004_03054_b200 import _native  # noqa: E402

L = _native.lib(0)
st = ctypes.c_void_p()
_native.check(L.luda_stream_create(ctypes.byref(st)))
arena, offs, lens, nlow = bench.synth_c2(L, st.value)
total = offs[-1] + lens[-1]
desc, keep = bench.make_desc(arena.data_ptr(), total, offs, lens, [0, nlow, len(offs)])
rows, wall = [], []
for i in range(60):
    t0 = time.perf_counter()
    res = bench.compact_once(L, desc, st.value)
    wall.append((time.perf_counter() - t0) * 1e3)
    rows.append([res.t_ms[k] for k in range(8)])
    L.luda_job_release(ctypes.byref(res))
rows, wall = rows[10:], wall[10:]
med = [statistics.median(r[k] for r in rows) for k in range(8)]
print("c2 device ms (median): parse %.3f decode %.3f merge %.3f plan %.3f emit %.3f | t5 %.3f t6 %.3f total %.3f"
      % tuple(med))
print("c2 host wall ms (median) %.3f" % statistics.median(wall))
