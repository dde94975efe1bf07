"""Per-source-line aggregation of an arbitrary source-page metric."""
import csv, collections, sys, subprocess
rep, metric = sys.argv[1], sys.argv[2]; top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = None; stats = collections.defaultdict(lambda: [0, ""]); mi = None
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur = r[1].split('/')[-1]; continue
    if r[0] == "Function Name": continue
    if r[0] == "Line No": mi = r.index(metric); continue
    if r[0] and r[0].isdigit():
        k = (cur, int(r[0])); stats[k][1] = r[1][:80]
        try: stats[k][0] += float(r[mi] or 0)
        except Exception: pass
tot = sum(v[0] for v in stats.values())
print(metric, "total", tot)
for k, v in sorted(stats.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k[0]:12s}{k[1]:5d} {v[0]/max(tot,1):6.1%} | {v[1]}")
