#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
python -m pytest tests/test_grf.py -m gpu -x -q > gpurun_out/grf_tests.txt 2>&1; tail -2 gpurun_out/grf_tests.txt
for r in 1 2; do
for B in 0 1; do echo SPLIT_B=$B; SFB_CHOL_SPLIT_B=$B python tools/chol_ab.py 2>&1 | head -1 | sed 's/.*hand-written//'; done; done
for W in 6 10 12; do echo W=$W; SFB_CHOL_PANEL=$W python tools/chol_ab.py 2>&1 | head -1 | sed 's/.*hand-written//'; done
