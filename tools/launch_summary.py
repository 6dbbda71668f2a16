"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel name."""
import collections, csv, sys

agg = collections.defaultdict(lambda: [0, 0.0])
hdr = None
for r in csv.reader(open(sys.argv[1])):
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            k = d["Kernel Name"][: int(sys.argv[2]) if len(sys.argv) > 2 else 70]
            agg[k][0] += 1
            agg[k][1] += float(d["Metric Value"].replace(",", ""))
tot = sum(t for _, t in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:6d} {t / 1e3:10.1f} us {100 * t / tot:5.1f}%  avg {t / n / 1e3:8.2f} us  {k}")
print(f"total {tot / 1e3:.1f} us")
