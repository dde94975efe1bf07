"""Dev: detect_batch time on the configurations the fused kernels do not take
(zero padding, finite sigma_p, quan-* / mean-quan references), 8 x 512 x 128^2."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2510_15602_b200 as Q
import workloads
x, _ = workloads.make_features(8, 1024, seed=7)
for kw in ({}, {"pad": "zero"}, {"sigma_p": 2.0}, {"reference_mode": "quan-median"},
           {"reference_mode": "mean-quan"}):
    cfg = Q.PipelineConfig(**kw)
    Q.detect_batch(x[:1], cfg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    Q.detect_batch(x, cfg)
    e1.record()
    torch.cuda.synchronize()
    print(kw or "default", round(e0.elapsed_time(e1) / 8, 3), "ms per image")
