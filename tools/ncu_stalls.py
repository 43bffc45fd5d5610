"""Per-kernel warp-stall breakdown (raw smsp__pcsamp_warps_issue_stalled_* counters)."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
cols = [i for i, c in enumerate(h) if c.startswith('smsp__pcsamp_warps_issue_stalled_') and not c.endswith('_not_issued')]
for v in rows[2:]:
    name = v[h.index('Kernel Name')][:50]
    vals = []
    for i in cols:
        try: vals.append((float(v[i].replace(',', '')), h[i][len('smsp__pcsamp_warps_issue_stalled_'):]))
        except ValueError: pass
    tot = sum(x for x, _ in vals) or 1
    print('==', name, ' '.join(f'{n}={x/tot:.1%}' for x, n in sorted(vals, reverse=True)[:8]))
