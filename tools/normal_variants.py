"""Time the configs[1] float32 normal fill (C2 shape) under SFB_NORMAL_VARIANT
values given on the command line (measurement scaffolding).

    python tools/normal_variants.py 10 42 74 ...

Each value runs in the same process (the knob is read per launch); the first
value is the reference for a bit-equality check of the outputs.
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2201_06604_b200 as sf  # noqa: E402
from paper_2201_06604_b200.grid import launch_fill  # noqa: E402


def main():
    vs = [int(v, 0) for v in sys.argv[1:]] or [10]
    st = sf.create_streams(sf.set_base_creator(), 1 << 18)[0]
    cur0 = st.device_current().clone()
    cur = cur0.clone()
    out = torch.empty((31250, 32000), dtype=torch.float32, device="cuda")
    ref = None
    for rep in range(2):
        for v in vs:
            os.environ["SFB_NORMAL_VARIANT"] = str(v)
            ts = []
            for i in range(8):
                cur.copy_(cur0)
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                launch_fill("normal", cur, st.count, out, 31250, 32000, 32000, 512, 512)
                e.record()
                e.synchronize()
                if i >= 2:
                    ts.append(s.elapsed_time(e))
            ts.sort()
            if ref is None:
                ref = out.clone()
                same = "ref"
            else:
                same = int((out != ref).sum().item())
            print(f"variant {v:#x}: {ts[len(ts) // 2]:.4f} ms  ({1e9 / ts[len(ts) // 2] / 1e6:.3e} normals/s)"
                  f"  cells differing from first: {same}", flush=True)


if __name__ == "__main__":
    main()
