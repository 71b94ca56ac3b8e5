"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]; ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
agg = collections.defaultdict(lambda: [0, 0.0]); tot = 0.0
for r in rows[hi + 1:]:
    if len(r) <= vi: continue
    ms = float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
    a = agg[r[ki][:80]]; a[0] += 1; a[1] += ms; tot += ms
for k, (c, ms) in sorted(agg.items(), key=lambda x: -x[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{ms:9.2f} ms {c:5d}  {k}")
print(f"total {tot:.2f} ms")
