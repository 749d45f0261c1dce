import os, sys
sys.path.insert(0, os.getcwd())
from oracle import luda_oracle as O
from paper_2004_03054_b200 import DeviceConfig, make_device
from paper_2004_03054_b200.compaction import compact_files
from paper_2004_03054_b200.config import StoreConfig
dev = make_device(DeviceConfig(backend="b200"))
base = bytes(range(1, 80))
for L in (57, 58):
    keys = [base[:L], base[:L] + b"\x00"]
    pairs = [(O.make_ikey(k, 100 + i, O.KIND_PUT), b"v" * 7) for i, k in enumerate(keys)]
    f = O.build_table(pairs + [(O.make_ikey(b"\xff" * 3, 1, O.KIND_PUT), b"z")], sst_size_target=1 << 20)
    print("L", L, f[:160].hex(), flush=True)
    try:
        compact_files(dev, [f], [], source_level=0, config=StoreConfig(sst_size_target=1 << 20))
        print("ok", flush=True)
    except Exception as e:
        print("ERR", e, flush=True)
dev.close()
