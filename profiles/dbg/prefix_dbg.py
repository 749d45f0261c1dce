"""Debug: one-file var jobs of a key followed by its one-byte extension."""
import os
import sys
sys.path.insert(0, os.getcwd())
from oracle import luda_oracle as O  # noqa: E402
from paper_2004_03054_b200 import DeviceConfig, make_device  # noqa: E402
from paper_2004_03054_b200.compaction import compact_files  # noqa: E402
from paper_2004_03054_b200.config import StoreConfig  # noqa: E402

dev = make_device(DeviceConfig(backend="b200"))
cfg = StoreConfig(sst_size_target=1 << 20)


def run(tag, keys, kinds=None):
    kinds = kinds or [O.KIND_PUT] * len(keys)
    pairs = [(O.make_ikey(k, 100 + i, kinds[i]), b"v" * 7) for i, k in enumerate(keys)]
    # a third key of another length forces the var path
    f = O.build_table(pairs + [(O.make_ikey(b"\xff" * 3, 1, O.KIND_PUT), b"z")], sst_size_target=1 << 20)
    want = O.reference_compact([f], sst_size_target=1 << 20)
    try:
        got = compact_files(dev, [f], [], source_level=0, config=cfg)
        r = "OK" if [g[0] for g in got] == [w[0] for w in want] else "MISMATCH"
    except Exception as e:  # noqa: BLE001
        r = f"ERR {e}"
    print(tag, r, flush=True)


base = bytes(range(1, 80))
for L in list(range(0, 71)):
    run(f"L={L} +00", [base[:L], base[:L] + b"\x00"])
for L in (7, 8, 15, 16, 57, 58):
    run(f"L={L} +01", [base[:L], base[:L] + b"\x01"])
    run(f"L={L} +00 del", [base[:L], base[:L] + b"\x00"], [O.KIND_DELETE, O.KIND_PUT])
    run(f"L={L} +0000", [base[:L], base[:L] + b"\x00\x00"])
dev.close()
