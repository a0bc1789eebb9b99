"""Determinism of the chunked launches (several threads per stream): Fisher
with one table per thread, and fills with tiny chunks (generic, quad and
normal kernels).  `save` records a plain run's outputs and final stream
states; `compare` repeats every case and compares each run with the record.
Run `compare` under `compute-sanitizer --tool synccheck`, which perturbs block
scheduling: a kernel whose result depends on block order shows up there.

    python tools/determinism_check.py save gpurun_out/det.npz
    compute-sanitizer --tool synccheck python tools/determinism_check.py compare gpurun_out/det.npz 5
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2201_06604_b200 as sf  # noqa: E402

mode, path = sys.argv[1], sys.argv[2]
runs = int(sys.argv[3]) if len(sys.argv) > 3 else 5
os.environ["SFB_GENERIC_CHUNK"] = "1"  # generic kernels: one draw per chunk


def fisher_case():
    st = sf.create_streams(sf.set_base_creator(), 16)[0]
    r = sf.fisher_sim(np.array([[3, 7], [6, 2]]), 3000, st, grid=sf.WorkGrid(4, 4),
                      return_stats=True)
    return r.statistics.tobytes() + st.current.tobytes()


def fill_case(kind, shape, g, dtype=None):
    def run():
        st = sf.create_streams(sf.set_base_creator(), g[0] * g[1])[0]
        req = sf.FillRequest(shape=shape, grid=sf.WorkGrid(*g),
                             **({"dtype": dtype} if dtype else {}))
        fill = {"uniform": sf.fill_uniform, "normal": sf.fill_normal}[kind]
        return fill(st, req).data.tobytes() + st.current.tobytes()
    return run


cases = {"fisher_E2x2_grid4x4": fisher_case,
         "uniform_generic_odd_g1": fill_case("uniform", (300, 301), (3, 5)),
         "uniform_quad_many_row_chunks": fill_case("uniform", (8192, 64), (2, 8)),
         "normal_generic_vector": fill_case("normal", 20000, (1, 8), np.float32)}
if mode == "save":
    np.savez(path, **{k: np.frombuffer(fn(), np.uint8) for k, fn in cases.items()})
    print("saved", path)
    sys.exit(0)
ref = np.load(path)
bad_total = 0
for name, fn in cases.items():
    want = ref[name].tobytes()
    bad = sum(fn() != want for _ in range(runs))
    bad_total += bad
    print(f"{name}: {bad} of {runs} runs differ from the plain run", flush=True)
print("DETERMINISTIC" if bad_total == 0 else "NONDETERMINISTIC")
