"""Per-kernel totals and shares from an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

src, dst = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else None)
SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
rows = list(csv.reader(open(src)))
h, agg = None, collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        h = r
        continue
    if not h or len(r) < len(h) or r[h.index("Metric Name")] != "gpu__time_duration.sum":
        continue
    ms = float(r[h.index("Metric Value")].replace(",", "")) * SCALE.get(r[h.index("Metric Unit")], 1e-6)
    k = r[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("dg::<unnamed>::", "")[:60]
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += ms
tot = sum(v[1] for v in agg.values())
out = [f"{'kernel':62s} {'launches':>8s} {'total_ms':>9s} {'share':>6s}   (ncu launch list: {src})"]
for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
    out.append(f"{k:62s} {n:8d} {ms:9.3f} {ms / tot:6.1%}")
text = "\n".join(out) + "\n"
print(text)
if dst:
    open(dst, "w").write(text)
