"""Var-key vs fixed-key compaction time at a moderate size (experiment): two
sorted runs of N entries (the newer one overwriting half the keys), 100-byte
values, built on the GPU by the flush builders, then compacted by luda_compact.
Prints device ms per job for mixed-length (8..40 B) and fixed 24-byte keys."""
import os
import random
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import luda_oracle as O  # noqa: E402
from paper_2004_03054_b200 import DeviceConfig, make_device  # noqa: E402
from paper_2004_03054_b200.compaction import PreparedJob, runner_for  # noqa: E402
from paper_2004_03054_b200.config import StoreConfig  # noqa: E402
from paper_2004_03054_b200.flush import build_ssts  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 400000
dev = make_device(DeviceConfig(backend="b200"))
for label, lens in (("fixed24", lambda r: 24), ("mixed8_40", lambda r: r.randint(8, 40))):
    rng = random.Random(1)
    keys = sorted({rng.randbytes(lens(rng)) for _ in range(N)})
    up = [(O.make_ikey(k, i + 1, O.KIND_PUT), rng.randbytes(100)) for i, k in enumerate(keys)]
    lo = [(O.make_ikey(k, N + 1 + i, O.KIND_PUT), rng.randbytes(100)) for i, k in enumerate(keys[::2])]
    up.sort(key=lambda kv: O.order_key(kv[0]))
    lo.sort(key=lambda kv: O.order_key(kv[0]))
    cfg = dict(sst_size_target=4 << 20)
    upper = [f for f, _, _ in build_ssts(up, **cfg)]
    lower = [f for f, _, _ in build_ssts(lo, **cfg)]
    files = lower + upper
    pj = PreparedJob(files=files, run_first_file=[0, len(lower), len(files)], deeper=[],
                     sst_size_target=cfg["sst_size_target"])
    for i in range(3):
        outs, info, _ = runner_for(dev).run(pj, len(lower))
    t = info["t_ms"]
    print(label, len(keys) + len(keys[::2]), "entries in;", len(files), "files; device ms: parse %.2f decode %.2f "
          "merge %.2f plan %.2f emit %.2f total %.2f" % (t[0], t[1], t[2], t[3], t[4], t[7]), flush=True)
dev.close()
