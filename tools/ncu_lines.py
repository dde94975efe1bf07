"""Aggregate an ncu source-page CSV (cuda,sass) per CUDA source line."""
import csv, collections, sys, subprocess
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur_file = None; stats = collections.defaultdict(lambda: [0, 0, ""]); ie = ss = None
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur_file = r[1].split('/')[-1]; continue
    if r[0] == "Function Name": continue
    if r[0] == "Line No": ie = r.index("Instructions Executed"); ss = r.index("Warp Stall Sampling (All Samples)"); continue
    if r[0] and r[0].isdigit():
        k = (cur_file, int(r[0])); stats[k][2] = r[1][:80]
        try: stats[k][0] += int(r[ie] or 0); stats[k][1] += int(r[ss] or 0)
        except Exception: pass
ti = sum(v[0] for v in stats.values()); ts = sum(v[1] for v in stats.values())
print("total warp instr", ti, "stall samples", ts)
for k, v in sorted(stats.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{k[0]:12s}{k[1]:5d} instr {v[0]/ti:6.1%} stall {v[1]/max(ts,1):6.1%} | {v[2]}")
