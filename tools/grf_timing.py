"""Component timing of the GRF pipeline on the acceptance-11 batch (4 x 5130^2)."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2201_06604_b200 as sf  # noqa: E402

big = sf.GridSpec(90, 57, 1.0)
batch = [sf.MaternParams(1.0, 8.0, 1.0), sf.MaternParams(1.5, 12.0, 2.0, 2.0, 0.5),
         sf.MaternParams(0.5, 6.0, 1.5), sf.MaternParams(2.0, 10.0, 1.0, 1.5, 1.0)]


def t(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return r, (time.perf_counter() - t0) * 1e3


for rep in range(3):
    cov, a = t(lambda: sf.matern_cov(batch, big))
    (lm, dg), b = t(lambda: sf.chol_batch(cov))
    st = sf.create_streams(sf.set_base_creator(), 64)[0]
    f, c = t(lambda: sf.simulate_grf(batch, big, 2, st, sf.WorkGrid(8, 8)))
    print(f"matern_cov {a:.1f} ms, chol_batch {b:.1f} ms, simulate_grf total {c:.1f} ms")
rng = __import__("numpy").random.default_rng(7)
coords = rng.uniform(0, 100, size=(5130, 2))
_, d = t(lambda: sf.matern_cov(batch, coords))
_, d = t(lambda: sf.matern_cov(batch, coords))
print(f"matern_cov arbitrary coords (4 x 5130^2 pairs) {d:.1f} ms")

# batched vs per-matrix Cholesky (cuSOLVER)
a = cov.device().reshape(4, 5130, 5130)
for rep in range(2):
    _, e = t(lambda: torch.linalg.cholesky_ex(a))
    _, f = t(lambda: [torch.linalg.cholesky_ex(a[b]) for b in range(4)])
    print(f"cholesky_ex batched {e:.1f} ms, per-matrix loop {f:.1f} ms")
x = torch.randn(5130, 5130, dtype=torch.float64, device="cuda")
_, g = t(lambda: x @ x)
_, g = t(lambda: x @ x)
print(f"DGEMM 5130^3: {g:.2f} ms = {2 * 5130 ** 3 / g / 1e9:.1f} TFLOP/s")

# per-matrix potrf on concurrent streams (each potrf alone leaves SMs idle in
# its panel phases)
def chol_streams(a, nstreams=4):
    cur = torch.cuda.current_stream()
    ss = [torch.cuda.Stream() for _ in range(nstreams)]
    out = torch.empty_like(a)
    info = torch.empty(a.shape[0], dtype=torch.int32, device="cuda")
    for b in range(a.shape[0]):
        s = ss[b % nstreams]
        s.wait_stream(cur)
        with torch.cuda.stream(s):
            torch.linalg.cholesky_ex(a[b], out=(out[b], info[b]))
    for s in ss:
        cur.wait_stream(s)
    return out, info


for rep in range(3):
    _, h = t(lambda: chol_streams(a, 4))
    _, h2 = t(lambda: chol_streams(a, 2))
    _, f = t(lambda: [torch.linalg.cholesky_ex(a[b]) for b in range(4)])
    print(f"cholesky per-matrix on 4 streams {h:.1f} ms, 2 streams {h2:.1f} ms, serial {f:.1f} ms")
