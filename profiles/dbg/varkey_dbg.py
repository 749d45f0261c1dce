"""Debug: the generic-length-key golden cases on the GPU, in isolation and in sequence."""
import os
import sys
sys.path.insert(0, os.getcwd())
from oracle import luda_oracle as O  # noqa: E402
from paper_2004_03054_b200 import DeviceConfig, make_device  # noqa: E402
from tests.golden.cases import VARKEY_CASES  # noqa: E402
from tests.test_gpu_parity import build, gpu_compact  # noqa: E402

order = sys.argv[1].split(",") if len(sys.argv) > 1 else [n for n, _, _ in VARKEY_CASES]
dev = make_device(DeviceConfig(backend="b200"))
for name in order:
    job, lower, upper, out_cfg = build(name)
    want = O.reference_compact(lower + upper, deeper=job.deeper, **out_cfg)
    try:
        got = gpu_compact(dev, job, lower, upper, out_cfg)
        ok = [g[0] for g in got] == [w[0] for w in want]
        print(name, "OK" if ok else "MISMATCH", len(got), len(want), flush=True)
    except Exception as e:  # noqa: BLE001
        print(name, "ERR", type(e).__name__, e, flush=True)
dev.close()
