"""Full-size parity runs that are too slow for the test suite (run on the GPU box):

    python tools/validate_full.py normal     # configs[1]: 1e9 float32 normals vs float32(oracle)

Prints one JSON line with the cell counts that differ and the largest difference
in float32 ulps, plus whether the final stream states match bit for bit.
"""

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2201_06604_b200 as sf  # noqa: E402
from oracle import oracle as orc  # noqa: E402


def normal_full():
    shape, g, n = (31250, 32000), (512, 512), 1 << 18
    st = sf.create_streams(sf.set_base_creator(), n)[0]
    t0 = time.time()
    got = sf.fill_normal(st, sf.FillRequest(shape=shape, grid=sf.WorkGrid(*g),
                                            dtype=np.float32)).values
    t_gpu = time.time() - t0
    ref_st, _ = orc.create_streams(sf.DEFAULT_SEED, n)
    ref = np.zeros(shape, np.float32)
    t0 = time.time()
    orc.fill_normal(ref_st, ref.ravel(), shape[0], shape[1], shape[1], g[0], g[1])
    t_cpu = time.time() - t0
    diff = got != ref
    nd = int(diff.sum())
    ulps = 0.0
    if nd:
        a = got[diff].astype(np.float64)
        b = ref[diff].astype(np.float64)
        ulps = float((np.abs(a - b) / np.spacing(np.abs(ref[diff])).astype(np.float64)).max())
    return {"check": "configs[1] float32 normals vs float32(oracle)", "cells": int(got.size),
            "cells_differing": nd, "max_ulp_f32": ulps,
            "states_equal": bool(np.array_equal(st.current, ref_st)),
            "gpu_api_s": t_gpu, "oracle_s": t_cpu, "oracle_threads": orc.max_threads()}


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "normal"
    if what == "normal":
        print(json.dumps(normal_full()), flush=True)
