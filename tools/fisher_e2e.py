"""End-to-end fisher_sim with host-resident states (the C3 e2e leg of
bench.py): tables/s over repeated calls, per library build.

    python tools/fisher_e2e.py "" "SFB_LIB=ab/libsfb_head.so"
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, time, numpy as np
sys.path.insert(0, ROOT)
import paper_2201_06604_b200 as sf
T4 = [[5, 9, 5, 7], [9, 5, 9, 7], [8, 6, 2, 6], [10, 8, 8, 8]]
grid = sf.WorkGrid(256, 64)
st = sf.create_streams(sf.set_base_creator(), grid.size)[0]
r = sf.fisher_sim(T4, 10**6, st, grid=grid)
best = 0
for rep in range(5):
    t0 = time.perf_counter()
    for _ in range(50):
        _ = st.current
        r = sf.fisher_sim(T4, 10**6, st, grid=grid)
    best = max(best, r.sim_num * 50 / (time.perf_counter() - t0))
print(best, r.counts, int(st.current[0, 0]))
'''


def main():
    for cfg in sys.argv[1:] or [""]:
        env = dict(os.environ)
        for kv in filter(None, cfg.split(",")):
            k, v = kv.split("=")
            env[k] = v
        out = subprocess.run([sys.executable, "-c", "ROOT=%r\n" % ROOT + CHILD], env=env,
                             capture_output=True, text=True)
        print(f"{cfg or 'default':36s}", out.stdout.strip() or out.stderr[-800:], flush=True)


if __name__ == "__main__":
    main()
