"""ncu --csv launch list (gpu__time_duration.sum) -> markdown share table (dev tool).

    python tools/launch_summary.py launches.csv "title" > profiles/rXX_launches_summary.md
"""
import collections, csv, sys

rows = list(csv.reader(open(sys.argv[1])))
title = sys.argv[2] if len(sys.argv) > 2 else "launch list"
hdr, agg = None, collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        v *= {"ms": 1e3, "us": 1.0, "ns": 1e-3, "s": 1e6}.get(d.get("Metric Unit", "us"), 1.0)
        a = agg.setdefault(d["Kernel Name"], [0.0, 0])
        a[0] += v
        a[1] += 1
tot = sum(v[0] for v in agg.values())
print(f"# {title}\n")
print("ncu serialises and cold-starts every launch: compare SHARES, not absolutes.\n")
print(f"total {tot:.1f} us over {sum(v[1] for v in agg.values())} launches\n")
print("| share | total us | launches | kernel |\n|---|---|---|---|")
for k, (t, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    if t / tot < 0.001:
        continue
    name = k.replace("|", "/")[:110]
    print(f"| {100 * t / tot:5.1f}% | {t:10.1f} | {n} | `{name}` |")
