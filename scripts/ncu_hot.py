"""Top stalled SASS instructions of one kernel in an .ncu-rep (needs -lineinfo)."""
import csv, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '-k', 'regex:' + kre,
                      '--print-source', 'sass,cuda'], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
# find header rows
hdr = None
rows = []
for x in r:
    if x and x[0] == 'Address':
        hdr = x
        continue
    if hdr and x and x[0].startswith('0x'):
        rows.append(dict(zip(hdr, x)))
    if len(rows) > 0 and x and x[0].startswith('Kernel Name') and rows:
        break
f = lambda v: float(v) if v not in ('', '-') else 0.0
tot = sum(f(d['Warp Stall Sampling (All Samples)']) for d in rows)
print('samples', tot, 'sass', len(rows))
top = sorted(rows, key=lambda d: -f(d['Warp Stall Sampling (All Samples)']))[:n]
for d in top:
    print(f"{100*f(d['Warp Stall Sampling (All Samples)'])/tot:5.1f}%  {d['Source'][:70]}")
