"""Summarise an `ncu --page source --csv --print-source=cuda,sass` export per
CUDA source line: warp-stall samples and instructions executed (top N)."""
import csv
import sys
from collections import defaultdict


def main(path, kernel_filter="", top=25):
    rows = list(csv.reader(open(path)))
    cur_file, cur_fn = "", ""
    agg = defaultdict(lambda: [0, 0, ""])
    tot_s = tot_i = 0
    hdr = None
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if len(r) == 2 and r[0] == "Function Name":
            cur_fn = r[1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if not hdr or not r or not r[0] or kernel_filter not in cur_fn:
            continue
        d = dict(zip(hdr, r))
        try:
            s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
            i = int(d.get("Instructions Executed", "0") or 0)
        except ValueError:
            continue
        k = (cur_file, int(r[0]))
        agg[k][0] += s
        agg[k][1] += i
        agg[k][2] = r[1][:90]
        tot_s += s
        tot_i += i
    print(f"total samples {tot_s}  instructions {tot_i}")
    for (f, ln), (s, i, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{s / max(tot_s, 1) * 100:5.1f}% smp {i / max(tot_i, 1) * 100:5.1f}% ins  {f}:{ln:<4} {src}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "", int(sys.argv[3]) if len(sys.argv) > 3 else 25)
