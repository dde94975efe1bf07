"""Stage times of the top-k eigensolver on the bench workload's covariances (dev tool)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_15602_b200  # noqa: F401
from paper_2510_15602_b200 import features as F, _native as N
import workloads

x, _ = workloads.make_features(64, 512, seed=5)
cov, _ = F.covariance_exact(x, None)
b, c, _ = cov.shape
def timed(f, n=5):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
n = F.LANCZOS_DIM
q0 = F._start_block(c, F.LANCZOS_BW, cov.device).contiguous()
basis = torch.empty((b, n, c), dtype=torch.float64, device="cuda")
h = torch.empty((b, n, n), dtype=torch.float64, device="cuda")
lz = lambda: N.call("qfca_lanczos", cov.data_ptr(), b, c, F.LANCZOS_PASSES, q0.data_ptr(),
                    basis.data_ptr(), h.data_ptr(), None, None, None, N.stream())
lz()
hs = torch.triu(h) + torch.triu(h, 1).mT
p = 32
x0 = F._start_block(n, p, cov.device).contiguous()
xo = torch.empty((b, n, p), dtype=torch.float64, device="cuda")
hm = torch.empty((b, p, p), dtype=torch.float64, device="cuda")
rz = lambda: N.call("qfca_ritz", h.data_ptr(), b, n, x0.data_ptr(), 15, xo.data_ptr(),
                    hm.data_ptr(), N.stream())
res = {"lanczos_kernel": timed(lz), "ritz_kernel": timed(rz),
       "sym_eig": timed(lambda: F.sym_eig(hm)),
       "small_topk": timed(lambda: F.topk_eigh(hs, 10, lanczos=False)),
       "lanczos_total": timed(lambda: F.topk_eigh(cov, 10)),
       "subspace_total": timed(lambda: F.topk_eigh(cov, 10, lanczos=False))}
print(json.dumps({k: round(v, 3) for k, v in res.items()}))
