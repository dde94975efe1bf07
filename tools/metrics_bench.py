"""Time the GPU evaluation metrics (paper_2510_15602_b200.metrics) on one class
of B maps of HxW (device-resident fp64 maps + bool masks), and the oracle's
NumPy/SciPy restatement of metrics.py on the host for the same class.

    python tools/metrics_bench.py [--images 64] [--size 1024] [--reps 5] [--cpu-images 8]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2510_15602_b200 import metrics as M  # noqa: E402


def make(b, h, w, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    sc = torch.randn((b, h, w), generator=g, device="cuda", dtype=torch.float64)
    sc = torch.nn.functional.avg_pool2d(sc[:, None], 9, 1, 4)[:, 0]
    mk = torch.zeros((b, h, w), dtype=torch.bool, device="cuda")
    rng = np.random.default_rng(seed)
    for i in range(b):
        if i % 4 == 3:
            continue
        for _ in range(rng.integers(1, 6)):
            y, x = rng.integers(0, h), rng.integers(0, w)
            ry, rx = rng.integers(4, h // 10), rng.integers(4, w // 10)
            mk[i, max(0, y - ry):y + ry, max(0, x - rx):x + rx] = True
    sc += mk * 0.3
    # anomaly maps reach evaluation upsampled: float32 values held in fp64
    sc = sc.float().double()
    return sc, mk


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--images", type=int, default=64)
    ap.add_argument("--size", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--cpu-images", type=int, default=8)
    a = ap.parse_args()
    sc, mk = make(a.images, a.size, a.size)
    samples = [M.EvalSample(scores=sc[i], mask=mk[i], image_label=bool(mk[i].any()), border=4)
               for i in range(a.images)]
    rep = M.MetricReport()
    rep.add_class("warm", samples)
    torch.cuda.synchronize()
    times = []
    for r in range(a.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        row = M.MetricReport().add_class("c", samples)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    gpu_ms = 1e3 * float(np.median(times))
    out = {"images": a.images, "size": a.size, "gpu_ms_per_class": gpu_ms,
           "gpu_mpix_per_s": a.images * a.size ** 2 / gpu_ms / 1e3, "row": row}
    # stage split (device-resident pool)
    p = M._Pool(samples)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); p.rank(); torch.cuda.synchronize(); t1 = time.perf_counter()
    thr = M._pro_thresholds(p); torch.cuda.synchronize(); t2 = time.perf_counter()
    M._pro_curve(p, thr); torch.cuda.synchronize(); t3 = time.perf_counter()
    out["stages_ms"] = {"sort+rank": 1e3 * (t1 - t0), "quantiles": 1e3 * (t2 - t1),
                        "components+pro": 1e3 * (t3 - t2)}
    if a.cpu_images > 0:
        from oracle import qfca_oracle as O
        k = a.cpu_images
        hs = [(sc[i].cpu().numpy(), mk[i].cpu().numpy(), bool(mk[i].any()), 4) for i in range(k)]
        t0 = time.perf_counter()
        s_, l_ = O.metrics_pooled(hs)
        O.pro_at_fpr(hs), O.rank_auroc(s_, l_), O.f1_optimal(s_, l_), O.auroc_image(hs)
        cpu = time.perf_counter() - t0
        out["cpu_oracle_s"] = cpu
        out["cpu_images"] = k
        out["cpu_mpix_per_s"] = k * a.size ** 2 / cpu / 1e6
        ev = [M.EvalSample(scores=torch.from_numpy(x[0]).cuda(), mask=torch.from_numpy(x[1]).cuda(),
                           image_label=x[2], border=4) for x in hs]
        g = M.MetricReport().add_class("c", ev)
        out["cpu_subset_row"] = {"pro": O.pro_at_fpr(hs), "auroc_s": O.rank_auroc(s_, l_),
                                 "f1": O.f1_optimal(s_, l_), "auroc_c": O.auroc_image(hs)}
        out["gpu_subset_row"] = g
    print(json.dumps(out))


if __name__ == "__main__":
    main()
