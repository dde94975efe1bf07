"""Launch the block-Lanczos kernel alone on 64 synthetic 512 x 512 covariances (ncu target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_15602_b200  # noqa: F401
from paper_2510_15602_b200 import features as F, _native as N
b, c = 64, 512
g = torch.Generator(device="cuda").manual_seed(0)
a = torch.randn(b, c, 1024, device="cuda", dtype=torch.float64, generator=g)
cov = a @ a.mT / 1024
n = F.LANCZOS_DIM
q0 = F._start_block(c, F.LANCZOS_BW, cov.device).contiguous()
basis = torch.empty((b, n, c), dtype=torch.float64, device="cuda")
h = torch.empty((b, n, n), dtype=torch.float64, device="cuda")
for _ in range(3):
    N.call("qfca_lanczos", cov.data_ptr(), b, c, F.LANCZOS_PASSES, q0.data_ptr(),
           basis.data_ptr(), h.data_ptr(), None, None, None, N.stream())
torch.cuda.synchronize()
