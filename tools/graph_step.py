"""Eager vs CUDA-graph-captured bench step (dev tool)."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_15602_b200 as Q
import workloads
size = int(sys.argv[1]) if len(sys.argv) > 1 else 512
pca = int(sys.argv[2]) if len(sys.argv) > 2 else 10
feats, _ = workloads.make_features(64, size, seed=1000, device="cuda")
cfg = Q.PipelineConfig(pca_components=pca)
def step():
    res = Q.detect_batch(feats, cfg)
    return res, Q.upsample_batch(res.scores, size, size)
for _ in range(3): step()
torch.cuda.synchronize()
def timeit(f, n=30):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); t0 = time.perf_counter(); e0.record()
    for _ in range(n): f()
    e1.record(); t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    return e0.elapsed_time(e1) / n, (t1 - t0) / n * 1e3, (t2 - t0) / n * 1e3
eager = [timeit(step) for _ in range(3)]
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(2): step()
torch.cuda.current_stream().wait_stream(s)
with torch.cuda.graph(g):
    out = step()
graph = [timeit(g.replay) for _ in range(3)]
ref = step()
torch.cuda.synchronize()
g.replay(); torch.cuda.synchronize()
same = bool(torch.equal(out[0].scores, ref[0].scores))
print(json.dumps({"eager_ms(dev,host_enqueue,wall)": eager, "graph_ms": graph, "graph_matches_eager": same}))
