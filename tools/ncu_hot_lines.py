"""Top CUDA source lines by warp-stall samples (ncu source page, cuda+sass correlation)."""
import csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
kern = sys.argv[3] if len(sys.argv) > 3 else None
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass'] + (['-k', 'regex:' + kern] if kern else []),
                     capture_output=True, text=True).stdout
fname = None; rows = []
for r in csv.reader(out.splitlines()):
    if len(r) == 2 and r[0] == 'File Path': fname = r[1].split('/')[-1]; continue
    if len(r) > 4 and r[0] not in ('', 'Line No') and r[2] == '-':
        try: rows.append((float(r[4]), fname, r[0], r[1]))
        except ValueError: pass
tot = sum(x[0] for x in rows)
for n, f, ln, src in sorted(rows, reverse=True)[:top]:
    print(f'{n/tot:6.1%} {f}:{ln:5s} {src.strip()[:90]}')
