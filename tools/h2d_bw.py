"""Dev: pinned host -> device copy bandwidth, one stream vs several (chunked)."""
import torch
n = 2 << 30
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    chunk = n // ns
    for _ in range(2):
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        evs = []
        for i, s in enumerate(streams):
            s.wait_event(e0) if False else None
            with torch.cuda.stream(s):
                d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
    for s in streams:
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{ns} stream(s): {5 * n / ms / 1e6:.1f} GB/s")
