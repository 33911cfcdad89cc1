import torch, time
def t(f, r=5):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    best = 1e9
    for _ in range(r):
        e0.record(); f(); e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    return best
for N in (4096, 8192, 16384):
    a = torch.randn(N, N, dtype=torch.float64, device="cuda"); b = torch.randn_like(a)
    ms = t(lambda: a @ b)
    print(f"dgemm {N}: {ms:.2f} ms {2*N**3/ms/1e9:.1f} TF/s")
N = 16641
A = torch.randn(N, N, dtype=torch.float64, device="cuda"); A = A @ A.T / N + torch.eye(N, dtype=torch.float64, device="cuda")
ms = t(lambda: torch.linalg.cholesky(A), 3)
print(f"potrf {N}: {ms:.2f} ms {N**3/3/ms/1e9:.1f} TF/s")
k = 2048
C = torch.randn(N - k, N - k, dtype=torch.float64, device="cuda"); P = torch.randn(N - k, k, dtype=torch.float64, device="cuda")
ms = t(lambda: C.addmm_(P, P.T, alpha=-1.0))
print(f"update {N-k}x{k}: {ms:.2f} ms {2*(N-k)**2*k/ms/1e9:.1f} TF/s")
