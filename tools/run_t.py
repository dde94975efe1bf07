"""Dev: one detect_batch at 1024^2 for a given patch size (ncu target)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2510_15602_b200 as Q
import workloads
t = int(sys.argv[1]); n = int(sys.argv[2]) if len(sys.argv) > 2 else 16
x, _ = workloads.make_features(8, 1024, seed=7)
cfg = Q.PipelineConfig(patch_size=t, n_bins=n)
for _ in range(2):
    Q.detect_batch(x, cfg)
torch.cuda.synchronize()
print("ok")
