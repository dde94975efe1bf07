"""Per-stage device times of the QFCA path (dev tool; CUDA events)."""
import argparse, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_15602_b200 as Q
from paper_2510_15602_b200 import features as F, _native as N
import workloads

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, default=512)
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--pca", type=int, default=10)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
x, _ = workloads.make_features(a.batch, a.size, seed=5)
b, c, h, w = x.shape
def ev():
    e = torch.cuda.Event(enable_timing=True); e.record(); return e
res = {}
for rep in range(a.reps + 1):
    t = {}
    e0 = ev()
    if a.pca:
        hw = h * w
        e1 = ev()
        cov, mean = F.covariance_exact(x, None)  # means + covariance, one pass over x
        e2 = ev()
        evals, vecs = F.topk_eigh(cov, a.pca)
        e3 = ev()
        idx = torch.arange(c - 1, c - 1 - a.pca, -1, device=x.device)
        comps = vecs.transpose(1, 2).contiguous()
        r = F.pca_residual_batch(x, mean, comps)
        e4 = ev()
    else:
        r = x; e1 = e2 = e3 = e4 = e0
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(); s1.record()
    cfg = Q.PipelineConfig()
    out = Q.detect_batch(r, cfg, score_events=(s0, s1))
    e5 = ev()
    up = Q.upsample_batch(out.scores, a.size, a.size)
    e6 = ev()
    torch.cuda.synchronize()
    t = {"mean": e0.elapsed_time(e1), "cov": e1.elapsed_time(e2), "eigh": e2.elapsed_time(e3),
         "residual": e3.elapsed_time(e4), "quant+ref": e4.elapsed_time(s0), "score": s0.elapsed_time(s1),
         "finalize": s1.elapsed_time(e5), "upsample": e5.elapsed_time(e6), "total": e0.elapsed_time(e6)}
    if rep:
        for k, v in t.items(): res.setdefault(k, []).append(v)
print(json.dumps({k: round(min(v), 3) for k, v in res.items()}))
print("per image ms:", json.dumps({k: round(min(v) / b, 4) for k, v in res.items()}))
