import torch, time, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_15602_b200 import features as F
x = torch.relu(torch.randn(64, 512, 4096, device="cuda"))
x = x - x.mean(-1, keepdim=True)
def t(f, n=3):
    f(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / n * 1e3
ref = F.covariance_dev(x, precise="fp64")
for mode in ("fp32", "fp64", "3xtf32"):
    for ch in (512, 1024, 4096):
        c = F.covariance_dev(x, chunk=ch, precise=mode)
        err = ((c - ref).abs().max() / ref.abs().max()).item()
        print(mode, ch, "ms %.3f" % t(lambda: F.covariance_dev(x, chunk=ch, precise=mode)), "err %.2e" % err)
