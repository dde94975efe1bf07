"""Dev ncu target: detect_batch on configs[1] residual-shaped inputs (8 x 512 x 64^2)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2510_15602_b200 as Q
import workloads
x, _ = workloads.make_features(8, 512, seed=7)
cfg = Q.PipelineConfig()
for _ in range(2):
    Q.detect_batch(x, cfg)
torch.cuda.synchronize()
print("ok")
