"""Summarise an ncu --csv metrics log of one bench step: per kernel name the
launches, device time, DRAM bytes / GB/s (vs MEASURED_PEAKS hbm_gbs), tensor-pipe
utilisation and issue activity.  Dev tool: python tools/ncu_summary_step.py <csv>"""
import csv
import json
import os
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr = None
data = []
for r in rows:
    if r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
peak = 6552.6
pp = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
if os.path.exists(pp):
    peak = json.load(open(pp))["hbm_gbs"]
k = OrderedDict()
for d in data:
    name = d["Kernel Name"].split("(")[0].replace("void ", "")
    e = k.setdefault((d["ID"], name), {})
    v = d["Metric Value"].replace(",", "")
    try:
        v = float(v)
    except ValueError:
        continue
    unit = d["Metric Unit"]
    if unit == "ms":
        v *= 1e3
    elif unit == "ns":
        v *= 1e-3
    elif unit == "Kbyte":
        v *= 1e3
    elif unit == "Mbyte":
        v *= 1e6
    elif unit == "Gbyte":
        v *= 1e9
    e[d["Metric Name"]] = v
agg = OrderedDict()
for (lid, name), e in k.items():
    a = agg.setdefault(name, {"launches": 0, "us": 0.0, "dram": 0.0, "imma": [], "tensor": [],
                              "dmma": [], "issue": [], "dram_pct": []})
    a["launches"] += 1
    a["us"] += e.get("gpu__time_duration.sum", 0.0)
    a["dram"] += e.get("dram__bytes_read.sum", 0.0) + e.get("dram__bytes_write.sum", 0.0)
    for key, m in (("imma", "sm__pipe_tensor_subpipe_imma_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"),
                   ("tensor", "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"),
                   ("dmma", "smsp__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed"),
                   ("issue", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                   ("dram_pct", "dram__throughput.avg.pct_of_peak_sustained_elapsed")):
        if m in e:
            a[key].append(e[m])
tot = sum(a["us"] for a in agg.values())
print(f"| share | us | launches | kernel | DRAM MB | DRAM GB/s | % of {peak:.0f} | dram% (ncu) | tensor% | imma% | dmma% | issue% |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|")
mean = lambda l: sum(l) / len(l) if l else float("nan")  # noqa: E731
for name, a in sorted(agg.items(), key=lambda kv: -kv[1]["us"]):
    gbs = a["dram"] / (a["us"] * 1e-6) / 1e9 if a["us"] else 0.0
    print(f"| {100 * a['us'] / tot:5.1f}% | {a['us']:9.1f} | {a['launches']} | `{name}` | {a['dram'] / 1e6:8.1f} | "
          f"{gbs:7.0f} | {100 * gbs / peak:5.1f}% | {mean(a['dram_pct']):5.1f} | {mean(a['tensor']):5.1f} | "
          f"{mean(a['imma']):5.1f} | {mean(a['dmma']):5.1f} | {mean(a['issue']):5.1f} |")
print(f"\ntotal {tot:.1f} us")
