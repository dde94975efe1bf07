"""BASELINE configs[3]: patch-size sweep (T 3..65, N=16) and bin-count sweep
(N 8..256, T=9) at 1024x1024 textures (512 x 128^2 WRN features), QFCA.

Prints one JSON object: per setting the scoring kernel version picked, the
device time of detect_batch per image (CUDA events, after warm-up) and the
ratio to the T=3 / N=8 point (the constant-time pooling check: <= 1.5x across
T).  Dev tool; `python tools/sweep.py [--batch B]`.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2510_15602_b200 as Q
from paper_2510_15602_b200 import _native as N
import workloads

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--force", type=int, default=0, help="force a scoring kernel version (0: auto)")
a = ap.parse_args()
x, _ = workloads.make_features(a.batch, 1024, seed=7)
N.call("qfca_set_score_kernel", a.force)
b, c, h, w = x.shape
L = N.lib()


def run(n, t):
    cfg = Q.PipelineConfig(n_bins=n, patch_size=t)
    ver = L.qfca_score_version(h, w, n, t, c, b, N.PAD_CODES[cfg.pad], cfg.sample_budget, 0)
    if a.force and ver < 0:
        return {"n_bins": n, "patch_size": t, "kernel": -1, "ms_per_image": float("nan")}
    if ver < 0:
        ver = L.qfca_score_version(h, w, n, t, c, b, N.PAD_CODES[cfg.pad], cfg.sample_budget, 1)
    Q.detect_batch(x, cfg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        Q.detect_batch(x, cfg)
    e1.record()
    torch.cuda.synchronize()
    return {"n_bins": n, "patch_size": t, "kernel": ver,
            "ms_per_image": e0.elapsed_time(e1) / a.reps / b}


res = {"workload": f"QFCA, {b} x 1024^2 textures, WRN50-2 random-init 512 x 128^2",
       "forced_kernel": a.force,
       "patch_sweep": [run(16, t) for t in (3, 5, 7, 9, 11, 13, 15, 17, 33, 65)],
       "bin_sweep": [run(n, 9) for n in (8, 16, 32, 64, 128, 256)]}
base_t = res["patch_sweep"][0]["ms_per_image"]
base_n = res["bin_sweep"][0]["ms_per_image"]
for r in res["patch_sweep"]:
    r["vs_T3"] = r["ms_per_image"] / base_t
for r in res["bin_sweep"]:
    r["vs_N8"] = r["ms_per_image"] / base_n
res["patch_flatness_max_ratio"] = max(r["vs_T3"] for r in res["patch_sweep"])
print(json.dumps(res, indent=1))
