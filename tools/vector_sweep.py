"""The reference's default use: a 1 x 1e8 vector on the default 64 x 8 grid (8 active
streams; generic kernel): chunk-size sweep, every kind, and the write probes."""
import os, sys, json, torch
sys.path.insert(0, "/root/repo")
import paper_2201_06604_b200 as sf
from paper_2201_06604_b200.grid import launch_fill
def timeit(fn, reps=20):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3): fn()
    torch.cuda.synchronize(); s.record()
    for _ in range(reps): fn()
    e.record(); e.synchronize()
    return s.elapsed_time(e) / reps
st = sf.create_streams(sf.set_base_creator(), 512)[0]
cur = st.device_current()
n = 10 ** 8
out = torch.empty((1, n), dtype=torch.float64, device="cuda")
for ch in (512, 128, 256, 1024, 2048, 4096, 16384, 512):
    os.environ["SFB_GENERIC_CHUNK"] = str(ch)
    ms = timeit(lambda: launch_fill("uniform", cur, st.count, out, 1, n, n, 64, 8))
    print(json.dumps({"chunk": ch, "ms": round(ms, 4), "TBs": round(n*8/ms/1e9, 3)}), flush=True)
for kind, dt in (("normal", torch.float64), ("normal", torch.float32), ("exponential", torch.float64),
                 ("uniform-integer", torch.int64)):
    o2 = torch.empty((1, n), dtype=dt, device="cuda")
    for ch in (512, 128, 256, 1024):
        os.environ["SFB_GENERIC_CHUNK"] = str(ch)
        ms = timeit(lambda: launch_fill(kind, cur, st.count, o2, 1, n, n, 64, 8))
        print(json.dumps({"vector": kind, "dtype": str(dt), "chunk": ch, "ms": round(ms, 4),
                          "TBs": round(n * o2.element_size() / ms / 1e9, 3)}), flush=True)
    del o2
os.environ.pop("SFB_GENERIC_CHUNK")
probe = torch.empty(n * 8, dtype=torch.uint8, device="cuda")
from paper_2201_06604_b200 import _lib
for v in (0, 1, 2):
    ms = timeit(lambda: _lib.lib().sfb_probe_write(probe.data_ptr(), n * 8, v, _lib.stream_handle()))
    print(json.dumps({"probe": v, "ms": round(ms, 4), "TBs": round(n*8/ms/1e9, 3)}), flush=True)
