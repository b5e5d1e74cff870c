"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import csv, collections, sys
lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.reader(lines))
h = rows[0]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[1:]:
    name = r[ik].split("(")[0].replace("void ", "").strip()
    v = float(r[iv].replace(",", ""))
    v *= {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(r[iu], 1.0)
    tot[name] += v
    cnt[name] += 1
S = sum(tot.values())
print(f"{'kernel':40s} {'launches':>8s} {'total ms':>10s} {'avg ms':>9s} {'share':>6s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:40s} {cnt[k]:8d} {v:10.3f} {v / cnt[k]:9.4f} {100 * v / S:5.1f}%")
