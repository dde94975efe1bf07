"""Batch split over two CUDA streams (latency-bound eigensolver of one half
overlapping the throughput-bound stages of the other) vs one stream (dev tool)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_15602_b200 as Q
import workloads
size = int(sys.argv[1]) if len(sys.argv) > 1 else 512
pca = int(sys.argv[2]) if len(sys.argv) > 2 else 10
nsplit = int(sys.argv[3]) if len(sys.argv) > 3 else 2
feats, _ = workloads.make_features(64, size, seed=1000, device="cuda")
cfg = Q.PipelineConfig(pca_components=pca)
streams = [torch.cuda.Stream() for _ in range(nsplit)]
def step1():
    res = Q.detect_batch(feats, cfg)
    return Q.upsample_batch(res.scores, size, size)
def stepn():
    main = torch.cuda.current_stream()
    outs = []
    chunk = feats.shape[0] // nsplit
    for k, s in enumerate(streams):
        s.wait_stream(main)
        with torch.cuda.stream(s):
            x = feats[k * chunk:(k + 1) * chunk]
            r = Q.detect_batch(x, cfg)
            outs.append(Q.upsample_batch(r.scores, size, size))
    for s in streams:
        main.wait_stream(s)
    return outs
def timeit(f, n=20):
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
a = [timeit(step1) for _ in range(2)]
b = [timeit(stepn) for _ in range(2)]
ref = step1(); got = stepn(); torch.cuda.synchronize()
same = bool(torch.equal(torch.cat(got), ref))
print(json.dumps({"one_stream_ms": a, f"{nsplit}_streams_ms": b, "identical": same}))
