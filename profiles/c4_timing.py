"""Timing of the fused job on the BASELINE c4 (scaled) shape: 8 fully overlapping L0 runs x 2^22
24-byte keys, 256-byte values, one SST per run (experiment; per-phase ms from luda_compact)."""
import ctypes, sys, os, json
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO); sys.path.insert(0, os.path.join(REPO, "tests"))
import torch
from paper_2004_03054_b200 import _native
import test_gpu_fullsize as T
torch.cuda.set_device(0)
L = _native.lib(0)
s = ctypes.c_void_p(); _native.check(L.luda_stream_create(ctypes.byref(s)))
n = 1 << 22
arena, offs, lens = T._synth_c4_runs(L, 8, n, 0xC4, s.value)
desc, keep = T._desc(_native, arena.data_ptr(), arena.numel(), offs, lens, list(range(9)))
ts = []
for i in range(5):
    res = _native.JobResult()
    _native.check(L.luda_compact(ctypes.byref(desc), ctypes.byref(res), s.value))
    ts.append((res.t_ms[7], [round(res.t_ms[k], 3) for k in range(5)], [round(res.k_ms[k], 3) for k in range(5)]))
    L.luda_job_release(ctypes.byref(res))
print(json.dumps({"s_in": sum(lens), "n_in": 8 * n, "runs": ts[2:]}))
