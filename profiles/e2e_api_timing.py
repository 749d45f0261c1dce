"""Host timeline of the public-API e2e pipeline (run_compactions over the c3
job with StagedInput): wall-clock stamps around every JobRunner stage /
compact / fetch / finish call, to locate host time between steps. Usage:
python profiles/e2e_api_timing.py [steps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2004_03054_b200 import compaction as C  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
w = bench.synth_c3(1 << 25, seed=0xC3, device_index=0)
T0 = [time.perf_counter()]
log = []


def wrap(obj, name):
    f = getattr(obj, name)

    def g(*a, **k):
        t = time.perf_counter()
        r = f(*a, **k)
        log.append((name, round((t - T0[0]) * 1e3, 1), round((time.perf_counter() - t) * 1e3, 1)))
        return r
    setattr(obj, name, g)


for n in ("stage", "describe", "_fetch_async", "_finish"):
    wrap(C.JobRunner, n)
orig_compact = C.B200Device.compact


def compact(self, desc, stream="compute"):
    t = time.perf_counter()
    r = orig_compact(self, desc, stream)
    log.append(("compact", round((t - T0[0]) * 1e3, 1), round((time.perf_counter() - t) * 1e3, 1)))
    return r


C.B200Device.compact = compact
orig_prepare = C.prepare


def prepare(*a, **k):
    t = time.perf_counter()
    r = orig_prepare(*a, **k)
    log.append(("prepare", round((t - T0[0]) * 1e3, 1), round((time.perf_counter() - t) * 1e3, 1)))
    return r


C.prepare = prepare
import types  # noqa: E402

orig_api = bench.e2e_public_api
# time the timed loop only: reset T0 when the timed run_compactions starts
orig_rc = C.run_compactions
calls = [0]


def rc(*a, **k):
    calls[0] += 1
    if calls[0] == 2:
        T0[0] = time.perf_counter()
        log.clear()
    return orig_rc(*a, **k)


import paper_2004_03054_b200 as P  # noqa: E402

P.run_compactions = lambda jobs, device, **kw: rc(jobs, device, **kw)
r = bench.e2e_public_api(w, steps)
print(r["value"], r["ms_per_step"])
for e in log:
    print(*e)
