"""Hot SASS of one kernel (first instance) with 3 lines of context.
usage: ncu_sass_hot.py rep kernel_regex [threshold_pct]"""
import csv, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 1.5
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '-k', 'regex:' + kre,
                      '--print-source', 'sass'], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
hdr = r[1]
rows = [dict(zip(hdr, x)) for x in r[2:] if x and x[0].startswith('0x')]
seen, rr = set(), []
for d in rows:
    if d['Address'] in seen:
        break
    seen.add(d['Address'])
    rr.append(d)
f = lambda v: float(v) if v not in ('', '-') else 0.0
key = 'Warp Stall Sampling (All Samples)'
tot = sum(f(d[key]) for d in rr)
print('samples', tot, 'sass', len(rr))
for i, d in enumerate(rr):
    s = f(d[key])
    if s / tot * 100 >= thr:
        for j in range(max(0, i - 3), i):
            print('        ', j, rr[j]['Source'].strip()[:90])
        print(f"{100 * s / tot:5.1f}% {i} {d['Source'].strip()[:90]}  (exec {d['Instructions Executed']})")
