"""Dev: detect_batch time per 1024^2 image at large T with N > 16."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2510_15602_b200 as Q
import workloads
x, _ = workloads.make_features(2, 1024, seed=7)
for n, t in ((16, 33), (32, 33), (32, 17), (64, 33)):
    cfg = Q.PipelineConfig(n_bins=n, patch_size=t)
    Q.detect_batch(x[:1], cfg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    Q.detect_batch(x, cfg)
    e1.record()
    torch.cuda.synchronize()
    print(n, t, round(e0.elapsed_time(e1) / 2, 2), "ms per image")
