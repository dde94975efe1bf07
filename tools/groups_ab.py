"""Dev: K4 channel groups per image (CTAs = images x groups) on configs[2]."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2510_15602_b200 as Q
import workloads
x, _ = workloads.make_features(64, 1024, seed=7)
cfg = Q.PipelineConfig()
for g in (0, 16, 37, 74, 8):
    for _ in range(2):
        Q.detect_batch(x, cfg, groups=g)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        Q.detect_batch(x, cfg, groups=g)
    e1.record()
    torch.cuda.synchronize()
    print("groups", g, round(e0.elapsed_time(e1) / 5, 3), "ms per 64 images")
