"""c2 (latency-bound BASELINE config) job under ncu: python profiles/c2_launches.py
(run as `ncu --metrics gpu__time_duration.sum --csv ... python profiles/c2_launches.py`);
without ncu it prints per-phase device times of one job."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2004_03054_b200 import _native  # noqa: E402

L = _native.lib(0)
st = ctypes.c_void_p()
_native.check(L.luda_stream_create(ctypes.byref(st)))
arena, offs, lens, nlow = bench.synth_c2(L, st.value)
total = offs[-1] + lens[-1]
desc, keep = bench.make_desc(arena.data_ptr(), total, offs, lens, [0, nlow, len(offs)])
for i in range(3):
    res = bench.compact_once(L, desc, st.value)
    print("job", i, "t_ms", [round(x, 3) for x in res.t_ms], "launches", res.launches, flush=True)
    L.luda_job_release(ctypes.byref(res))
