import os, sys, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_2201_06604_b200 as sf
from paper_2201_06604_b200.fisher import launch_fisher, plan_fisher
T4 = [[5, 9, 5, 7], [9, 5, 9, 7], [8, 6, 2, 6], [10, 8, 8, 8]]
for n in (16384, 10**6):
    grid = sf.WorkGrid(256, 64)
    st = sf.create_streams(sf.set_base_creator(), grid.size)[0]
    plan = plan_fisher(np.asarray(T4), n, st, grid)
    cur = st.device_current(); cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    for i in range(3):
        launch_fisher(plan, cur, st.count, cnt)
    torch.cuda.synchronize()
