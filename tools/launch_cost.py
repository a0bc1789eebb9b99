"""Host-side cost of the Fisher launch path: Python wrapper vs raw ctypes enqueue,
the stream-handle query, and the count readback variants."""
import sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2201_06604_b200 as sf
from paper_2201_06604_b200 import _lib
from paper_2201_06604_b200.fisher import launch_fisher, plan_fisher
T4 = np.array([[5, 9, 5, 7], [9, 5, 9, 7], [8, 6, 2, 6], [10, 8, 8, 8]])
g = sf.WorkGrid(256, 64)
st = sf.create_streams(sf.set_base_creator(), g.size)[0]
plan = plan_fisher(T4, 10**6, st, g)
cur = st.device_current()
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
for _ in range(20): launch_fisher(plan, cur, st.count, cnt)
torch.cuda.synchronize()
N = 300
t0 = time.perf_counter()
for _ in range(N): launch_fisher(plan, cur, st.count, cnt)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host enqueue per launch {1e6*(t1-t0)/N:.1f} us; device per launch {1e6*(t2-t0)/N:.1f} us")
# raw ctypes call cost with prebuilt args
rm, cm, lf = plan.c_args()
L = _lib.lib(); f = L.sfb_fisher_replicates
args = (cur.data_ptr(), st.count, rm, 4, cm, 4, lf, len(plan.lf), plan.kernel_threshold, plan.reps, 0, g.size, None, None, cnt.data_ptr(), 1, _lib.stream_handle())
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(N): f(*args)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"raw ctypes enqueue {1e6*(t1-t0)/N:.1f} us")

import timeit
dev = torch.cuda.current_device()
print("current_stream().cuda_stream %.2f us" % (timeit.timeit(lambda: torch.cuda.current_stream().cuda_stream, number=20000) / 20000 * 1e6))
print("_cuda_getCurrentRawStream %.2f us" % (timeit.timeit(lambda: torch._C._cuda_getCurrentRawStream(dev), number=20000) / 20000 * 1e6))
print("current_device %.2f us" % (timeit.timeit(lambda: torch.cuda.current_device(), number=20000) / 20000 * 1e6))
print("data_ptr %.2f us" % (timeit.timeit(lambda: cur.data_ptr(), number=20000) / 20000 * 1e6))
print("torch.empty(1) cuda %.2f us" % (timeit.timeit(lambda: torch.empty(1, dtype=torch.int64, device="cuda"), number=20000) / 20000 * 1e6))
print("count.item %.2f us" % (timeit.timeit(lambda: cnt.item(), number=2000) / 2000 * 1e6))
from paper_2201_06604_b200 import _lib as L2
print("_lib.stream_handle %.2f us" % (timeit.timeit(L2.stream_handle, number=20000) / 20000 * 1e6))
assert L2.stream_handle() == torch.cuda.current_stream().cuda_stream
s2 = torch.cuda.Stream()
with torch.cuda.stream(s2):
    assert L2.stream_handle() == s2.cuda_stream
print("stream_handle follows torch.cuda.stream contexts")
hp = torch.zeros(1, dtype=torch.int64, pin_memory=True)
def b():
    hp.copy_(cnt, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return int(hp[0])
def c():
    hp.copy_(cnt, non_blocking=True)
    torch.cuda.synchronize()
    return int(hp[0])
def d():
    hp.copy_(cnt)
    return int(hp[0])
for name, fn in (("item", lambda: cnt.item()), ("pinned+stream sync", b), ("pinned+device sync", c), ("pinned blocking copy", d)):
    print("%s %.2f us" % (name, timeit.timeit(fn, number=3000) / 3000 * 1e6))
