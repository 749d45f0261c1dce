"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv`) of `bench.py --steps 1 --warmup 1`: the launches of
the LAST compaction step (from its last parse_files_a), with share of kernel time.
    python profiles/launch_summary.py launches.csv > summary.txt"""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
L = OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        k = int(d["ID"])
        e = L.setdefault(k, {"name": d["Kernel Name"]})
        v = float(d["Metric Value"].replace(",", ""))
        u = d["Metric Unit"]
        scale = {"ns": 1e-3, "us": 1, "ms": 1e3, "byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1}.get(u, 1)
        e[d["Metric Name"]] = v * scale
ids = [k for k, e in L.items() if e["name"].startswith("luda::parse_files_a")]
step = [e for k, e in L.items() if k >= ids[-1]]
tot = sum(e.get("gpu__time_duration.sum", 0) for e in step)
print(f"ncu launch list, last c3 compaction step (64M entries, 9.64 GB in), launches {ids[-1]}.. of "
      "`bench.py --steps 1 --warmup 1`")
print("cold-cache, serialised (compare shares, not absolutes); DRAM bytes per launch")
print(f"{'kernel':64s} {'us':>8s} {'share':>6s} {'rd GB':>7s} {'wr GB':>7s} {'GB/s':>7s}")
for e in step:
    t = e.get("gpu__time_duration.sum", 0)
    rd, wr = e.get("dram__bytes_read.sum", 0), e.get("dram__bytes_write.sum", 0)
    print(f"{e['name'][:64]:64s} {t:8.1f} {100 * t / tot:5.1f}% {rd:7.3f} {wr:7.3f} {(rd + wr) / (t * 1e-6) if t else 0:7.0f}")
print(f"total kernel time {tot / 1e3:.3f} ms over {len(step)} launches")
