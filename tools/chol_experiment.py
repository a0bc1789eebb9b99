"""Cholesky alternatives for the GRF LDL^T step (5130 x 5130 f64) vs cuSOLVER potrf:
recursive / right-looking blocked over cuBLAS TRSM + GEMM, and the MAGMA backend.
Measured slower; kept as the record of that experiment."""
import time, torch
n=5130
torch.manual_seed(0)
x = torch.randn(n, n, dtype=torch.float64, device="cuda")
a = x @ x.T + n * torch.eye(n, dtype=torch.float64, device="cuda")
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t0=time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter()-t0)/reps*1e3
for lib in ("cusolver", "magma", "cusolver"):
    torch.backends.cuda.preferred_linalg_library(lib)
    print(lib, "cholesky_ex %.2f ms" % t(lambda: torch.linalg.cholesky_ex(a)))

def rchol(A, nb):
    n = A.shape[-1]
    if n <= nb:
        return torch.linalg.cholesky_ex(A)[0]
    n1 = n // 2
    L11 = rchol(A[:n1, :n1], nb)
    L21 = torch.linalg.solve_triangular(L11, A[n1:, :n1].T, upper=False).T
    A22 = torch.addmm(A[n1:, n1:], L21, L21.T, beta=1.0, alpha=-1.0)
    L22 = rchol(A22, nb)
    L = torch.zeros_like(A)
    L[:n1, :n1] = L11; L[n1:, :n1] = L21; L[n1:, n1:] = L22
    return L

def bchol(A, nb):
    """right-looking blocked, in place on a copy: panel potrf + trsm + gemm update of the trailing lower part"""
    A = A.clone()
    n = A.shape[-1]
    for k in range(0, n, nb):
        e = min(k + nb, n)
        A[k:e, k:e] = torch.linalg.cholesky_ex(A[k:e, k:e])[0]
        if e < n:
            Lkk = A[k:e, k:e]
            A[e:, k:e] = torch.linalg.solve_triangular(Lkk, A[e:, k:e].T, upper=False).T
            P = A[e:, k:e]
            A[e:, e:] -= P @ P.T
    return torch.tril(A)
torch.backends.cuda.preferred_linalg_library("cusolver")
ref = torch.linalg.cholesky_ex(a)[0]
for nb in (256, 512, 1024):
    L = rchol(a, nb)
    print("rchol nb", nb, "%.2f ms" % t(lambda: rchol(a, nb)), "maxrel", float(((L-ref).abs().max()/ref.abs().max())))
for nb in (512, 1024):
    L = bchol(a, nb)
    print("bchol nb", nb, "%.2f ms" % t(lambda: bchol(a, nb)), "maxrel", float(((L-ref).abs().max()/ref.abs().max())))
print("trsm 2565: %.2f ms" % t(lambda: torch.linalg.solve_triangular(ref[:2565,:2565], a[2565:, :2565].T.contiguous(), upper=False)))
y = a[2565:, :2565].contiguous()
print("gemm 2565: %.2f ms" % t(lambda: y @ y.T))
