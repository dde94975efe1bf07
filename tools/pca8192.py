"""Time QFCA+ on one 8192^2 texture (512 x 1024^2 features) on one GPU via
sharding.detect_pca_sharded (world size 1): pixel-sharded mean + centred Gram
(exact int8 blocks), top-k eigh, residual, channel-sharded scoring.

    python tools/pca8192.py [--size 1024] [--channels 512] [--reps 3]
"""
import argparse, json, os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_15602_b200 as Q  # noqa: E402
from paper_2510_15602_b200.sharding import detect_pca_sharded, pca_fit_sharded  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, default=1024)
ap.add_argument("--channels", type=int, default=512)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
g = torch.Generator(device="cuda").manual_seed(0)
c, n = a.channels, a.size
u = torch.linalg.qr(torch.randn((c, 10), generator=g, device="cuda"))[0]
z = torch.randn((10, n * n), generator=g, device="cuda") * torch.linspace(6, 2, 10, device="cuda")[:, None]
x = (u @ z + 0.5 * torch.randn((c, n * n), generator=g, device="cuda")).clamp(min=0).reshape(c, n, n)
cfg = Q.PipelineConfig(pca_components=10)
detect_pca_sharded(x, cfg)
torch.cuda.synchronize()
ts, tp = [], []
for _ in range(a.reps):
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record(); pca_fit_sharded(x, 10); e1.record()
    final, img, _ = detect_pca_sharded(x, cfg); e2.record()
    torch.cuda.synchronize()
    tp.append(e0.elapsed_time(e1)); ts.append(e1.elapsed_time(e2))
print(json.dumps({"workload": f"QFCA+ one {8 * n}^2 texture ({c} x {n}^2 features), 1 GPU",
                  "pca_fit_ms": sorted(tp)[len(tp) // 2], "detect_ms": sorted(ts)[len(ts) // 2],
                  "images_per_s": 1e3 / sorted(ts)[len(ts) // 2], "image_score": float(img)}))
