"""Dev ncu target: pca_residual_batch on configs[1] features (64 x 512 x 64^2)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2510_15602_b200 import features
import workloads
with torch.no_grad():
    x, _ = workloads.make_features(64, 512, seed=3)
mean, comps, _ = features.pca_fit_batch(x, 10)
for _ in range(2):
    r = features.pca_residual_batch(x, mean, comps)
torch.cuda.synchronize()
