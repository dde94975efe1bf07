import sys, os, torch
sys.path.insert(0, os.getcwd())
import paper_2510_15602_b200 as Q, workloads
x, _ = workloads.make_features(8, 1024, seed=7)
cfg = Q.PipelineConfig(n_bins=16, patch_size=17)
Q.detect_batch(x, cfg); torch.cuda.synchronize()
Q.detect_batch(x, cfg); torch.cuda.synchronize()
