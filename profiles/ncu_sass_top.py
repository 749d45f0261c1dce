"""Top SASS instructions by warp-stall samples from an `ncu --page source --csv
--print-source=cuda,sass` export, with the CUDA line they belong to and the
dominant stall reasons.   python profiles/ncu_sass_top.py src.csv[.gz] [top]"""
import csv
import gzip
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
f = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
rows = list(csv.reader(f))
hdr = None
cur = ("", "")
items = []
tot = 0
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < 6:
        continue
    if r[0]:
        cur = (f"{fname}:{r[0]}", r[1][:60])
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        continue
    tot += s
    stalls = sorted(((int(v), k) for k, v in d.items() if k.startswith("stall_") or "Stall" in k and k not in (
        "Warp Stall Sampling (All Samples)", "Warp Stall Sampling (Not-issued Samples)") and v.isdigit()),
        reverse=True)[:3]
    items.append((s, r[3].strip()[:60], cur[0], cur[1], stalls))
items.sort(key=lambda x: -x[0])
print(f"total samples {tot}")
for s, sass, loc, src, st in items[:top]:
    print(f"{100 * s / max(tot, 1):5.1f}%  {sass:60s} {loc:28s} {src}")
