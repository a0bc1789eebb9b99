"""T4 (configs[2]) chunking / memo-staging sweep: SFB_FISHER_TARGET_Q x SFB_FISHER_MEMO_SMEM_KB."""
import os, sys, json, numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tools")
import paper_2201_06604_b200 as sf
from paper_2201_06604_b200.fisher import launch_fisher, plan_fisher

def timeit(fn, reps=10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / reps
T4 = [[5, 9, 5, 7], [9, 5, 9, 7], [8, 6, 2, 6], [10, 8, 8, 8]]
grid = sf.WorkGrid(256, 64)
st = sf.create_streams(sf.set_base_creator(), grid.size)[0]
plan = plan_fisher(np.asarray(T4), 10**6, st, grid)
cur = st.device_current()
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
for q in (4, 1, 2, 3, 6, 8, 4):
    for smem in (48, 0):
        os.environ["SFB_FISHER_TARGET_Q"] = str(q)
        os.environ["SFB_FISHER_MEMO_SMEM_KB"] = str(smem)
        ms = timeit(lambda: launch_fisher(plan, cur, st.count, cnt), reps=20)
        print(json.dumps({"q": q, "memo_smem_kb": smem, "ms": round(ms, 4)}), flush=True)
