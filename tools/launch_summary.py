"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) by kernel:
count, total, share, average (cold-cache, serialised per-launch times)."""
import collections
import csv
import sys


def main(path, out=None):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    for d in data:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
                 "nsecond": 1e-3}.get(d["Metric Unit"], 1.0)
        a = agg.setdefault(d["Kernel Name"][:110], [0, 0.0])
        a[0] += 1
        a[1] += float(d["Metric Value"]) * scale
    tot = sum(v[1] for v in agg.values())
    lines = []
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{c:6d} {t:11.1f} us {100 * t / tot:5.1f}%  avg {t / c:9.2f} us  {k}")
    lines.append(f"total {tot:.1f} us over {sum(v[0] for v in agg.values())} launches")
    text = "\n".join(lines) + "\n"
    if out:
        open(out, "w").write(text)
    print(text)


if __name__ == "__main__":
    main(*sys.argv[1:])
