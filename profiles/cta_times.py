"""Summarise decode per-CTA timestamps (LUDA_DEC_CTA_TIMES build) per launch
(experiment): launch span, CTA start spread, CTA duration min / max, SMs."""
import sys
rows = []
for line in open(sys.argv[1]):
    if line.startswith("CTAT "):
        b, sm, t0, t1 = map(int, line.split()[1:5])
        rows.append((t0, t1, b, sm))
rows.sort()
launches, cur = [], []
for r in rows:
    if cur and r[0] - cur[-1][0] > 2_000_000:  # > 2 ms after the previous CTA start: a new launch
        launches.append(cur)
        cur = []
    cur.append(r)
if cur:
    launches.append(cur)
for L in launches:
    t0 = min(r[0] for r in L)
    t1 = max(r[1] for r in L)
    starts = sorted(r[0] - t0 for r in L)
    durs = sorted(r[1] - r[0] for r in L)
    sms = len(set(r[3] for r in L))
    late = [r for r in L if r[0] - t0 > 100_000]
    print("ctas %d sms %d span %.3f ms start spread %.3f ms dur min %.3f med %.3f max %.3f late(>0.1ms) %d"
          % (len(L), sms, (t1 - t0) / 1e6, starts[-1] / 1e6, durs[0] / 1e6, durs[len(durs) // 2] / 1e6,
             durs[-1] / 1e6, len(late)))
