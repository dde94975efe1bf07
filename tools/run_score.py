"""Run the fused detect on WRN features (profiling target)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_15602_b200 as Q
import workloads
ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, default=1024)
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--n", type=int, default=16)
ap.add_argument("--t", type=int, default=9)
a = ap.parse_args()
x, _ = workloads.make_features(a.batch, a.size, seed=3)
cfg = Q.PipelineConfig(n_bins=a.n, patch_size=a.t)
for _ in range(a.reps):
    r = Q.detect_batch(x, cfg)
torch.cuda.synchronize()
print("ok", float(r.image_scores[0]))
