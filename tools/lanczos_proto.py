"""Block-Lanczos prototype (numpy): how many passes of an 8-column block over the
covariance put the top-10 eigenvectors in the Krylov space, and how many
subspace-iteration steps on the small projection H recover them (dev tool;
reads cov6.npy = covariances of six WRN50-2 workload images, see mkcov in
git history / tools/eig_time.py for the GPU version)."""
import numpy as np
cov = np.load("cov6.npy")
k = 10
def cholqr(W):
    G = W.T @ W
    L = np.linalg.cholesky(G)
    return W @ np.linalg.inv(L.T)
def lanczos_H(S, b, P, seed=0):
    C = S.shape[0]
    rng = np.random.default_rng(seed)
    Q = cholqr(cholqr(rng.standard_normal((C, b))))
    n = P * b
    B = np.zeros((C, n)); H = np.zeros((n, n))
    B[:, :b] = Q
    for j in range(P):
        W = S @ B[:, j*b:(j+1)*b]
        cols = (j+1)*b
        C1 = B[:, :cols].T @ W
        H[:cols, j*b:(j+1)*b] = C1
        W = W - B[:, :cols] @ C1
        C2 = B[:, :cols].T @ W
        W = W - B[:, :cols] @ C2
        if j + 1 < P:
            B[:, cols:cols+b] = cholqr(cholqr(W))
    # symmetrize: take upper
    Hs = np.triu(H) + np.triu(H, 1).T
    return B, Hs
def topk_small(H, k, p=32, iters=15, seed=1):
    n = H.shape[0]
    rng = np.random.default_rng(seed)
    X = cholqr(rng.standard_normal((n, p)))
    H2 = H @ H
    for _ in range(iters):
        X = cholqr(H2 @ X)
    Hm = X.T @ H @ X
    w, u = np.linalg.eigh(Hm)
    return w[::-1][:k], X @ u[:, ::-1][:, :k]
for i in range(cov.shape[0]):
    S = cov[i]
    wr, vr = np.linalg.eigh(S); wr = wr[::-1][:k]; vr = vr[:, ::-1][:, :k]
    for b, P in ((4, 18), (4, 21), (4, 24), (8, 11), (8, 13), (2, 40)):
        B, H = lanczos_H(S, b, P)
        for iters in (10, 15):
            w, u = topk_small(H, k, iters=iters)
            V = B @ u
            Pe = np.abs(V @ V.T - vr @ vr.T).max()
            print(i, b, P, b*P, iters, f"proj {Pe:.1e} eval {np.abs(w-wr).max()/wr[0]:.1e}")
print("----")
for i in range(cov.shape[0]):
    S = cov[i]
    wr, vr = np.linalg.eigh(S); wr = wr[::-1][:k]; vr = vr[:, ::-1][:, :k]
    for b, P in ((8, 14), (8, 15), (8, 16), (6, 18), (6, 20), (16, 9), (16,10)):
        B, H = lanczos_H(S, b, P)
        w, u = topk_small(H, k, iters=15)
        V = B @ u
        Pe = np.abs(V @ V.T - vr @ vr.T).max()
        print(i, b, P, b*P, f"proj {Pe:.1e} eval {np.abs(w-wr).max()/wr[0]:.1e}")
