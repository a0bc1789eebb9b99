"""Run one small Fisher launch (E2x2 table, grid g0 x g1) and save counts,
per-item counts and statistics to gpurun_out/<tag>.npz, to compare a plain
run with one under compute-sanitizer.

    python tools/fisher_repeat_detail.py tag g0 g1 [n]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2201_06604_b200 as sf  # noqa: E402
from paper_2201_06604_b200.fisher import launch_fisher, plan_fisher  # noqa: E402

tag, g0, g1 = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
n = int(sys.argv[4]) if len(sys.argv) > 4 else 3000
t = np.array([[3, 7], [6, 2]])
g = sf.WorkGrid(g0, g1)
st = sf.create_streams(sf.set_base_creator(), g.size)[0]
plan = plan_fisher(t, n, st, g)
cur = st.device_current()
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
ic = torch.zeros(g.size, dtype=torch.int64, device="cuda")
stats = torch.empty(plan.sim_num, dtype=torch.float64, device="cuda")
launch_fisher(plan, cur, st.count, cnt, item_counts_dev=ic, stats_dev=stats)
torch.cuda.synchronize()
os.makedirs("gpurun_out", exist_ok=True)
np.savez(f"gpurun_out/{tag}.npz", count=cnt.cpu().numpy(), ic=ic.cpu().numpy(),
         stats=stats.cpu().numpy(), cur=cur.cpu().numpy(), reps=plan.reps)
print(tag, int(cnt.item()), plan.reps)
