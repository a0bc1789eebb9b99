"""Fisher kernel timing under tuning knobs (measurement scaffolding).

    python tools/fisher_time.py "SFB_X=1,SFB_Y=2" "SFB_X=0" ...

Each config runs in its own process (memo tables are cached per process).
Per workload: CUDA-event time of single launches, L2 flushed before each
(as bench.py does), median of N; the fixed-state launch repeats the same
tables so counts are comparable across configs.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, os, sys, statistics
import numpy as np, torch
sys.path.insert(0, ROOT)
import paper_2201_06604_b200 as sf
from paper_2201_06604_b200.fisher import launch_fisher, plan_fisher
T4 = [[5, 9, 5, 7], [9, 5, 9, 7], [8, 6, 2, 6], [10, 8, 8, 8]]
G = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))
A = np.load(os.path.join(ROOT, "tests", "golden", "golden.npz"))
scratch = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def case(name, table, n, g, reps):
    grid = sf.WorkGrid(*g)
    st = sf.create_streams(sf.set_base_creator(), grid.size)[0]
    plan = plan_fisher(np.asarray(table), n, st, grid)
    cur = st.device_current(); cur0 = cur.clone()
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    ts = []
    for i in range(reps + 3):
        cur.copy_(cur0)
        if os.environ.get("SLEEP"): torch.cuda._sleep(int(os.environ["SLEEP"]))  # warm L2, host launch hidden
        elif not os.environ.get("NOFLUSH"): scratch.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); launch_fisher(plan, cur, st.count, cnt); e.record(); e.synchronize()
        if i >= 3: ts.append(s.elapsed_time(e))
    ms = statistics.median(ts)
    return name, dict(ms=ms, tables_per_s=plan.sim_num / (ms / 1e3), counts=int(cnt.item()))
out = {}
CASES = os.environ.get("CASES", "T4,T10,month,week").split(",")
for name, table, n, g, reps in [c for c in [("T4", T4, 10**6, (256, 64), 60),
                                ("T4x10", T4, 10**7, (256, 64), 20),
                                ("T4n16k", T4, 16384, (256, 64), 60),
                                ("T4n64k", T4, 65536, (256, 64), 60),
                                ("T4n256k", T4, 262144, (256, 64), 60),
                                ("T4x4", T4, 4 * 10**6, (256, 64), 20),
                                ("T10", G["T10"], (1 << 21) * 8, (2048, 1024), 8),
                                ("T10c4", G["T10"], (1 << 21) * 477, (2048, 1024), 3),
                                ("month", A["month"], 10**6, (256, 64), 10),
                                ("week", A["week"], 10**6, (256, 64), 10)] if c[0] in CASES]:
    k, v = case(name, table, n, g, reps); out[k] = v
print(json.dumps(out))
'''


def main():
    for cfg in sys.argv[1:] or [""]:
        env = dict(os.environ)
        for kv in filter(None, cfg.split(",")):
            k, v = kv.split("=")
            env[k] = v
        r = subprocess.run([sys.executable, "-c", "ROOT=%r\n" % ROOT + CHILD], env=env,
                           capture_output=True, text=True)
        if r.returncode:
            print(cfg, "FAILED", r.stderr[-1500:])
            continue
        d = json.loads(r.stdout.strip().splitlines()[-1])
        print(f"{cfg or 'default':40s} " + "  ".join(
            f"{k} {v['ms']:.4f} ms {v['tables_per_s']:.3e}/s" for k, v in d.items()), flush=True)


if __name__ == "__main__":
    main()
