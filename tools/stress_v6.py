"""Dev stress: v6 vs v3 partials on several shapes, repeated."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from test_score6 import _partials
from paper_2510_15602_b200 import quantize
bad = 0
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    for (images, C, h, n, t, pad) in [(2, 12, 128, 16, 9, 1), (1, 8, 128, 16, 9, 2), (1, 6, 256, 16, 9, 1),
                                     (2, 6, 128, 16, 3, 1), (1, 4, 40, 16, 9, 1)]:
        rng = np.random.default_rng(it * 100 + C + h + t)
        x = np.maximum(rng.standard_normal((images, C, h, 128)) + 0.3, 0).astype(np.float32)
        x[0, 1] = 0.5
        xd = torch.from_numpy(x).cuda().reshape(images * C, h * 128)
        lo, hi, _ = quantize.minmax_dev(xd, images * C, h * 128)
        bins = quantize.bins_dev(xd, lo, hi, images * C, h * 128, n)
        p3 = _partials(3, bins, lo, hi, None, images, C, h, n, t, pad, 2)
        p6 = _partials(6, bins, lo, hi, None, images, C, h, n, t, pad, 2)
        eq = np.array_equal(p3, p6)
        bad += not eq
        print(it, (images, C, h, n, t, pad), "equal" if eq else f"DIFF max {np.abs(p3 - p6).max()}", flush=True)
print("bad", bad)
