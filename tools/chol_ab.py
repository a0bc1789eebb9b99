"""Hand-written batched Cholesky (sfb_chol_batch) vs cuSOLVER potrf on the
acceptance-11 batch (4 x 5130^2): time and agreement (measurement scaffolding)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2201_06604_b200 as sf  # noqa: E402

big = sf.GridSpec(90, 57, 1.0)
batch = [sf.MaternParams(1.0, 8.0, 1.0), sf.MaternParams(1.5, 12.0, 2.0, 2.0, 0.5),
         sf.MaternParams(0.5, 6.0, 1.5), sf.MaternParams(2.0, 10.0, 1.0, 1.5, 1.0)]


def ev(fn, reps=3):
    out = None
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        out = fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    return out, min(ts)


cov = sf.matern_cov(batch, big)
n, B = cov.n, cov.batch_count
a = cov.device().reshape(B, n, n)


def cusolver():
    c = torch.stack([torch.linalg.cholesky_ex(a[b])[0] for b in range(B)])
    d = torch.diagonal(c, dim1=1, dim2=2)
    lm = c / d.unsqueeze(1)
    lm.diagonal(dim1=1, dim2=2).fill_(1.0)
    return lm, d * d


(lref, dref), t_ref = ev(cusolver)
(lm, dg), t_new = ev(lambda: sf.chol_batch(cov))
l_new = lm.device().reshape(B, n, n)
err_l = ((l_new - lref).abs().max() / lref.abs().max()).item()
err_d = ((dg.device() - dref).abs() / dref.abs()).max().item()
print(f"n={n} B={B}: cuSOLVER potrf path {t_ref:.2f} ms, hand-written {t_new:.2f} ms "
      f"({B * n**3 / 3 / (t_new * 1e-3) / 1e12:.1f} TFLOP/s); max |dL|/max|L| {err_l:.2e}, "
      f"max rel dD {err_d:.2e}")
z = torch.randn(B * n, 2, dtype=torch.float64, device="cuda")
ref_mul, t_mref = ev(lambda: torch.matmul(lref, torch.sqrt(dref).unsqueeze(2) * z.reshape(B, n, 2)))
out, t_mul = ev(lambda: sf.multiply_lower_diag_batch(lm, dg, z))
err_m = ((out.device().reshape(B, n, 2) - ref_mul).abs().max() / ref_mul.abs().max()).item()
print(f"L D^1/2 Z (R=2): cuBLAS {t_mref:.3f} ms, hand-written {t_mul:.3f} ms "
      f"({B * n * n * 8 / 2 / (t_mul * 1e-3) / 1e9:.0f} GB/s of L), rel err {err_m:.2e}")
