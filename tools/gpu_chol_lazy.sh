#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
python -m pytest tests/test_grf.py -m gpu -x -q > gpurun_out/grf_tests.txt 2>&1; tail -2 gpurun_out/grf_tests.txt
for r in 1 2; do
for cfg in "2 3" "3 2" "3 1"; do set -- $cfg; echo STAGES=$1 BULK=$2; SFB_CHOL_STAGES=$1 SFB_CHOL_BULK_CTAS=$2 python tools/chol_ab.py 2>&1 | head -1 | sed 's/.*hand-written//'; done; done
