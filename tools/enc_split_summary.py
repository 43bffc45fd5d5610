"""Summarise tools/enc_split.sh output: per encode launch (pass) time, DRAM, instructions."""
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; idx = {n: i for i, n in enumerate(h)}
rec = {}
for r in rows[1:]:
    key = (int(r[idx['ID']]), r[idx['Kernel Name']].split('(')[0].split('::')[-1])
    rec.setdefault(key, {})[r[idx['Metric Name']]] = float(r[idx['Metric Value']])
tot = {}
for (i, k), m in sorted(rec.items()):
    t = m.get('gpu__time_duration.sum', 0) / 1e6
    print(f"{i:3d} {k:28s} {t:7.3f} ms  dram {(m.get('dram__bytes_read.sum',0)+m.get('dram__bytes_write.sum',0))/1e9:6.2f} GB"
          f"  inst {m.get('smsp__inst_executed.sum',0)/1e6:7.1f} M  L2hit {m.get('lts__t_sector_hit_rate.pct',0):5.1f}%"
          f"  reds {m.get('lts__t_requests_srcunit_tex_op_red.sum',0)/1e6:6.1f} M  LTS {m.get('lts__throughput.avg.pct_of_peak_sustained_elapsed',0):4.1f}%")
    tot[k] = tot.get(k, 0) + t
print({k: round(v, 3) for k, v in tot.items()})
