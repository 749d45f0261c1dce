"""Print the key ncu --set full metrics (per kernel) of a report: python profiles/ncu_summary.py rep.ncu-rep"""
import csv, io, subprocess, sys
WANT = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'Compute (SM) Throughput', 'Achieved Occupancy',
        'Registers Per Thread', 'L1/TEX Hit Rate', 'L2 Hit Rate', 'Executed Ipc Active', 'Issue Slots Busy',
        'Eligible Warps Per Scheduler', 'Warp Cycles Per Issued Instruction', 'Theoretical Occupancy',
        'L1/TEX Cache Throughput', 'L2 Cache Throughput']
out = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'details', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]; idx = {h: i for i, h in enumerate(hdr)}
last = None
for r in rows[1:]:
    k = r[idx['Kernel Name']].split('(')[0]; m = r[idx['Metric Name']]
    if m in WANT:
        if k != last: print(f"== {k}"); last = k
        print(f"  {m:38s} {r[idx['Metric Value']]:>10s} {r[idx['Metric Unit']]}")
raw = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
h = rr[0]
for r in rr[2:]:
    d = dict(zip(h, r))
    print(f"  dram bytes read {d.get('dram__bytes_read.sum','?')}  write {d.get('dram__bytes_write.sum','?')}  "
          f"(units: {rr[1][h.index('dram__bytes_read.sum')] if 'dram__bytes_read.sum' in h else '?'})")
