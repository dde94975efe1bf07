"""PCA-stage micro-benchmark on the bench workload (dev tool, CUDA events).

Covariance variants (accuracy vs an fp64 GEMM, time) and the pieces of the
top-k eigensolver.
"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_15602_b200 import features as F, _native as N
import workloads

B = int(os.environ.get("B", 64))
x, _ = workloads.make_features(B, 512, seed=5)
b, c, h, w = x.shape
hw = h * w


def timed(f, n=5):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        out = f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n, out


mean = torch.empty((b, c), dtype=torch.float64, device="cuda")
N.call("qfca_plane_mean", x.data_ptr(), b * c, hw, mean.data_ptr(), N.stream())
xc = torch.empty((b, c, hw), dtype=torch.float32, device="cuda")
t_center, _ = timed(lambda: N.call("qfca_center", x.data_ptr(), b * c, hw, mean.data_ptr(),
                                   xc.data_ptr(), N.stream()))
xd_ = x.reshape(b, c, hw).double() - mean[:, :, None]
ref = torch.bmm(xd_, xd_.mT) / hw
del xd_
res = {"center_ms": t_center}


def err(cv):
    return float(((cv - ref).abs().amax(dim=(1, 2)) / ref.abs().amax(dim=(1, 2))).max())


for name, fn in [("fp32_chunk1024", lambda: F.covariance_dev(xc)),
                 ("fp32_chunk4096", lambda: F.covariance_dev(xc, chunk=4096))]:
    t, cv = timed(fn)
    res[name] = {"ms": t, "relerr": err(cv)}


def split3(v):
    a = v.to(torch.bfloat16)
    r = v - a.float()
    bb = r.to(torch.bfloat16)
    cc = (r - bb.float()).to(torch.bfloat16)
    return a, bb, cc


def bf16x6(chunk):
    a, bb, cc = split3(xc)
    nk = hw // chunk

    def blk(t):
        return t.reshape(b, c, nk, chunk).permute(0, 2, 1, 3).reshape(b * nk, c, chunk)
    a, bb, cc = blk(a), blk(bb), blk(cc)
    f32 = torch.float32
    s = torch.bmm(a, a.mT, out_dtype=f32)
    m1 = torch.bmm(a, bb.mT, out_dtype=f32)
    m1 += torch.bmm(a, cc.mT, out_dtype=f32)
    s += torch.bmm(bb, bb.mT, out_dtype=f32)
    s += m1
    s += m1.mT
    return s.reshape(b, nk, c, c).sum(dim=1, dtype=torch.float64) / hw


covs = {}
for chunk in (1024, 4096):
    try:
        t, cv = timed(lambda: bf16x6(chunk))
        res[f"bf16x6_chunk{chunk}"] = {"ms": t, "relerr": err(cv)}
        covs[f"bf16x6_chunk{chunk}"] = cv
    except Exception as e:  # noqa
        res[f"bf16x6_chunk{chunk}"] = str(e)[:200]
def fp64cov():
    xd = x.reshape(b, c, hw).double() - mean[:, :, None]
    return torch.bmm(xd, xd.mT) / hw


t, cv = timed(lambda: F.covariance_exact(x, mean))
res["i8_exact"] = {"ms": t, "relerr": err(cv)}
covs["i8_exact"] = cv
t, cv = timed(fp64cov)
res["fp64_direct"] = {"ms": t, "relerr": err(cv)}
covs["fp64_direct"] = cv
def ozaki(ndig, min_cls):
    """Emulated int8 digit scheme: balanced base-256 digits of the per-channel
    fixed-point xc, pairs with k + l >= min_cls, exact products (fp64 GEMM of
    small integers)."""
    xd = x.reshape(b, c, hw).double() - mean[:, :, None]
    mx = xd.abs().amax(dim=2)
    e = torch.where(mx > 0, torch.floor(torch.log2(mx.clamp_min(1e-300))) + 3, 0.0)  # max|xc| <= 2^(e-2)
    bits = 8 * ndig
    N = torch.round(xd * torch.exp2(bits - e)[:, :, None])  # |N| <= 2^(bits-2)
    digs = []
    r = N
    for k in range(ndig):
        d = torch.remainder(r, 256.0)
        d = torch.where(d >= 128, d - 256, d)
        digs.append(d)
        r = (r - d) / 256.0
    S = torch.zeros((b, c, c), dtype=torch.float64, device="cuda")
    for k in range(ndig):
        for l in range(ndig):
            if k + l >= min_cls:
                S += torch.bmm(digs[k], digs[l].mT) * (256.0 ** (k + l))
    sc = torch.exp2(e - bits)
    return S * sc[:, :, None] * sc[:, None, :] / hw


for nd, mc in ((4, 2),):
    cv = ozaki(nd, mc)
    res[f"ozaki_{nd}d_cls{mc}"] = {"relerr": err(cv)}
    covs[f"ozaki_{nd}d_cls{mc}"] = cv
covs["fp32_chunk1024"] = F.covariance_dev(xc)
covs["fp32_chunk4096"] = F.covariance_dev(xc, chunk=4096)

# map error of each covariance variant against the fp64-covariance pipeline
import paper_2510_15602_b200 as Q


def maps(cv):
    ev, vec = F.topk_eigh(cv, 10)
    comps = vec.transpose(1, 2).contiguous()
    arg = comps.abs().argmax(dim=2, keepdim=True)
    comps = comps * torch.where(torch.gather(comps, 2, arg) < 0, -1.0, 1.0)
    r = F.pca_residual_batch(x, mean, comps)
    return Q.detect_batch(r, Q.PipelineConfig()).scores


m_ref = maps(ref)
for k, cv in covs.items():
    m = maps(cv)
    e = ((m - m_ref).abs().amax(dim=(1, 2)) / m_ref.abs().amax(dim=(1, 2)))
    res[k]["map_err_max"] = float(e.max())
    res[k]["map_err_median"] = float(e.median())

cov = F.covariance_dev(xc)
t, _ = timed(lambda: F.topk_eigh(cov, 10))
res["topk_eigh_ms"] = t
X32 = F._start_block(c, 32, cov.device).expand(b, c, 32)
sqm = cov @ cov
t, Y32 = timed(lambda: sqm @ X32)
res["it_SX_ms"] = t
t, G32 = timed(lambda: Y32.mT @ Y32)
res["it_gram_ms"] = t
t, R32 = timed(lambda: F.chol_rinv(G32))
res["it_chol_rinv_ms"] = t
t, _ = timed(lambda: Y32 @ R32)
res["it_YR_ms"] = t
t, _ = timed(lambda: F.sym_eig(G32))
res["sym_eig_gram_ms"] = t
xs = X32.contiguous()
for _ in range(15):
    xs = F._cholqr_inplace(sqm @ xs)
hm_ = xs.mT @ (cov @ xs)
t, _ = timed(lambda: F.sym_eig(hm_))
res["sym_eig_rr_ms"] = t
t, _ = timed(lambda: F._cholqr_inplace(sqm @ xs))
res["iteration_fused_ms"] = t


def one_iter():
    y = sqm @ X32
    return y @ F.chol_rinv(y.mT @ y)


t, _ = timed(one_iter, n=20)
res["iteration_ms"] = t
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    gout = F.topk_eigh(cov, 10)
t, _ = timed(lambda: g.replay())
res["topk_eigh_graph_ms"] = t
Xs = F._cholqr(torch.randn(b, c, 32, dtype=torch.float64, device="cuda"))


def rr():
    hm = Xs.mT @ (cov @ Xs)
    hm = 0.5 * (hm + hm.mT)
    w_, u = torch.linalg.eigh(hm)
    return Xs @ u[..., -10:].flip(-1)


t, _ = timed(rr)
res["rayleigh_ritz_ms"] = t
hm = Xs.mT @ (cov @ Xs)
t, _ = timed(lambda: torch.linalg.eigh(hm))
res["eigh32_ms"] = t
sq = cov @ cov
t, _ = timed(lambda: cov @ cov)
res["covsq_ms"] = t
X = F._cholqr(torch.randn(b, c, 32, dtype=torch.float64, device="cuda"))
t, Y = timed(lambda: sq @ X)
res["SX_ms"] = t
t, _ = timed(lambda: F._cholqr(Y))
res["cholqr_ms"] = t
t, _ = timed(lambda: Y.mT @ Y)
res["gram_ms"] = t
G = Y.mT @ Y
t, L = timed(lambda: torch.linalg.cholesky(G))
res["chol32_ms"] = t
t, _ = timed(lambda: torch.linalg.solve_triangular(L.mT, Y, upper=True, left=False))
res["trsm_ms"] = t
t, _ = timed(lambda: Y @ L)
res["YL_ms"] = t
t, _ = timed(lambda: F.pca_residual_batch(x, mean, torch.randn(b, 10, c, dtype=torch.float64,
                                                                device="cuda")))
res["residual_ms"] = t
print(json.dumps(res, indent=1))
