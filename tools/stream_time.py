"""Dev: event-timed streaming stages of configs[1] (64 x 512 ch x 64^2 WRN
features): covariance (k_cov_digits + k_cov_i8), residual, quantize, and the
configs[2] upsample; bytes are the compulsory DRAM traffic of each stage."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2510_15602_b200 as Q
from paper_2510_15602_b200 import features, quantize
import workloads


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


with torch.no_grad():
    x, _ = workloads.make_features(64, 512, seed=3)
b, c, h, w = x.shape
n = b * c * h * w
mean, comps, _ = features.pca_fit_batch(x, 10)
res = features.pca_residual_batch(x, mean, comps)
rows = []
ms = timed(lambda: features.covariance_exact(x, None))
rows.append(("covariance (digits + int8 MMA)", ms, 4 * n))
ms = timed(lambda: features.pca_residual_batch(x, mean, comps, res))
rows.append(("pca_residual", ms, 8 * n))
ms = timed(lambda: quantize.quantize_dev(res.view(b * c, h * w), b * c, h * w, 16))
rows.append(("quantize (K1+K2)", ms, 5 * n))
s = torch.rand(64, 128, 128, dtype=torch.float64, device="cuda")
ms = timed(lambda: Q.upsample_batch(s, 1024, 1024))
rows.append(("upsample 64 x 1024^2", ms, 64 * 1024 * 1024 * 4 + s.numel() * 8))
for name, ms, by in rows:
    print(f"{name:34s} {ms:7.3f} ms  {by / ms / 1e9:6.2f} TB/s  ({100 * by / ms / 1e9 / 6.5526:4.1f}% of 6553 GB/s)")
