"""Live cost of one step of the Cholesky factorisation chain (measurement
scaffolding): sfb_chol_batch on batch-4 SPD blocks of n = 64 t for small t,
where the trailing updates are tiny and the call is the serial chain
(diag -> panel solve -> next column's update); the slope in t is the live
per-step chain latency.  Also the acceptance size for reference."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2201_06604_b200 import _lib  # noqa: E402


def spd(n, b):
    g = torch.Generator(device="cuda").manual_seed(1)
    m = torch.randn(b, n, n, dtype=torch.float64, device="cuda", generator=g) / n ** 0.5
    return m @ m.transpose(1, 2) + torch.eye(n, dtype=torch.float64, device="cuda")


def time_chol(n, b=4, reps=20):
    a = spd(n, b)
    lm = torch.empty_like(a)
    d = torch.empty(b, n, dtype=torch.float64, device="cuda")
    info = torch.empty(b, dtype=torch.int32, device="cuda")
    lib = _lib.lib()
    st = _lib.stream_handle()

    def call():
        _lib.check(lib.sfb_chol_batch(_lib.dptr(a), n, b, _lib.dptr(lm), _lib.dptr(d),
                                      _lib.dptr(info), st))
    for _ in range(3):
        call()
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        call()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    assert int(info.abs().sum()) == 0
    return ts[len(ts) // 2]


if __name__ == "__main__":
    pts = []
    for t in (1, 2, 4, 8, 12, 16):
        ms = time_chol(64 * t)
        pts.append((t, ms))
        print(f"t={t:3d} n={64 * t:5d}: {ms * 1e3:8.1f} us")
    (t0, m0), (t1, m1) = pts[2], pts[-1]
    print(f"chain slope {(m1 - m0) / (t1 - t0) * 1e3:.1f} us per 64-column step (t {t0}..{t1})")
