"""Per-source-line shared-memory wavefronts (actual vs ideal) from an
`ncu --page source --csv --print-source=cuda,sass` export."""
import csv
import sys
from collections import defaultdict


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    hdr = None
    cur = ""
    agg = defaultdict(lambda: [0.0, 0.0, ""])
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            iw, ii = hdr.index("L1 Wavefronts Shared"), hdr.index("L1 Wavefronts Shared Ideal")
            continue
        if hdr and len(r) == len(hdr) and r[0].isdigit():
            try:
                w, idl = float(r[iw] or 0), float(r[ii] or 0)
            except ValueError:
                continue
            k = (cur, int(r[0]))
            agg[k][0] += w
            agg[k][1] += idl
            agg[k][2] = r[1][:90]
    tot = sum(v[0] for v in agg.values())
    print("total shared wavefronts", tot)
    for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{100 * v[0] / tot:5.1f}% ideal {100 * v[1] / tot:5.1f}%  {k[0]}:{k[1]}  {v[2]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
