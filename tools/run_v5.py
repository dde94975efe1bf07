"""One detect_batch at 1024^2 (8 images) with patch size T (v5 for T >= 17): ncu target."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_15602_b200 as Q
import workloads
t = int(sys.argv[1]) if len(sys.argv) > 1 else 33
x, _ = workloads.make_features(8, 1024, seed=7)
cfg = Q.PipelineConfig(patch_size=t)
for _ in range(2):
    Q.detect_batch(x, cfg)
torch.cuda.synchronize()
