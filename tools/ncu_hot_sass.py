"""Top SASS instructions by warp-stall samples from an ncu report (source page)."""
import csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
si = h.index('Warp Stall Sampling (All Samples)')
reasons = [c for c in h if c.startswith('stall_') and 'Not Issued' not in c]
data = []
for r in rows[2:]:
    if len(r) <= si or not r[si].strip(): continue
    try: n = float(r[si])
    except ValueError: continue
    rs = {c: float(r[h.index(c)] or 0) for c in reasons}
    data.append((n, r[0], r[1], rs))
tot = sum(d[0] for d in data)
agg = {}
for d in data:
    for k, v in d[3].items(): agg[k] = agg.get(k, 0) + v
print('total samples', tot)
print('by reason:', ', '.join(f'{k[6:]}={v/tot:.1%}' for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
for n, addr, src, rs in sorted(data, key=lambda x: -x[0])[:top]:
    main = sorted(rs.items(), key=lambda x: -x[1])[:2]
    print(f'{n/tot:6.1%} {addr:>6s} {src[:70]:70s} ' + ' '.join(f'{k[6:]}:{v:.0f}' for k, v in main))
