"""Summarise an .ncu-rep: key metrics per kernel + top SASS stall hotspots."""
import csv, io, subprocess, sys

rep = sys.argv[1]
want = ('Duration', 'DRAM Throughput', 'Compute (SM) Throughput', 'Achieved Occupancy',
        'Theoretical Occupancy', 'Registers Per Thread', 'Issue Slots Busy',
        'Executed Ipc Active', 'L2 Hit Rate', 'Eligible Warps Per Scheduler',
        'Active Warps Per Scheduler', 'Warp Cycles Per Issued Instruction',
        'Grid Size', 'Block Size', 'Dynamic Shared Memory Per Block')
out = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True,
                     text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[0]
ki, mi, vi, ui = (h.index(k) for k in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit'))
ii = h.index('ID')
last = None
for x in r[1:]:
    if x[mi] in want:
        key = (x[ii], x[ki])
        if key != last:
            print('==', x[ii], x[ki][:60])
            last = key
        print('   ', x[mi], x[vi], x[ui])
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True,
                     text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, rows = r[0], r[2:]
ki = h.index('Kernel Name')
for row in rows:
    d = dict(zip(h, row))
    st = []
    for k, v in d.items():
        if k.startswith('smsp__average_warp_latency_issue_stalled') or \
           (k.startswith('smsp__warp_issue_stalled') and k.endswith('per_warp_active.pct')):
            try:
                st.append((float(v.replace(',', '')), k))
            except ValueError:
                pass
    print('==', row[ki][:50], 'inst', d.get('smsp__inst_executed.sum'),
          'sm active avg/max', d.get('sm__cycles_active.avg'), d.get('sm__cycles_active.max'))
    for v, k in sorted(st, reverse=True)[:8]:
        print('    ', k, v)
