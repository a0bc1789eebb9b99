#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
python -m pytest tests/test_grf.py -m gpu -x -q > gpurun_out/grf_tests.txt 2>&1; tail -1 gpurun_out/grf_tests.txt
for r in 1 2; do
for P in 0 1; do echo EARLY=$P; SFB_CHOL_EARLY=$P python tools/chol_ab.py 2>&1 | head -1 | sed 's/.*hand-written//'; done; done
for P in 0 1; do echo EARLY=$P; SFB_CHOL_EARLY=$P python tools/chol_chain.py 2>&1 | tail -1; done
