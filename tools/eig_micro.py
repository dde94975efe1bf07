import torch, time
torch.manual_seed(0)
B, C, p = 64, 512, 48
A = torch.randn(B, C, C, dtype=torch.float64, device="cuda"); cov = A @ A.mT / C
X = torch.randn(B, C, p, dtype=torch.float64, device="cuda")
def t(f, n=5):
    f(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / n * 1e3
G = X.mT @ X
L = torch.linalg.cholesky(G)
print("bmm", t(lambda: cov @ X))
print("gram", t(lambda: X.mT @ X))
print("chol", t(lambda: torch.linalg.cholesky(G)))
print("trsm", t(lambda: torch.linalg.solve_triangular(L.mT, X, upper=True, left=False)))
H = G + G.mT
print("eigh48", t(lambda: torch.linalg.eigh(H)))
H32 = H[:, :32, :32].contiguous()
print("eigh32", t(lambda: torch.linalg.eigh(H32)))
print("eigh512", t(lambda: torch.linalg.eigh(cov[:4]), n=1))
