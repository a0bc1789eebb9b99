#!/bin/bash
# GRF Cholesky: GPU tests, the chain-step latency, the acceptance timing
# (and, when ab/libsfb_dbg.so exists, the chol_diag phase clocks)
cd "${GRAFT_REPO_ROOT:-.}"
python -m pytest tests/test_grf.py -m gpu -x -q > gpurun_out/grf_tests.txt 2>&1; tail -3 gpurun_out/grf_tests.txt
python tools/chol_chain.py 2>&1 | tail -1
for i in 1 2 3; do python tools/chol_ab.py 2>&1 | head -1 | sed 's/.*hand-written//'; done
if [ -f ab/libsfb_dbg.so ]; then SFB_LIB=$PWD/ab/libsfb_dbg.so python tools/chol_chain.py 2>&1 | grep "diag k=5" | head -2; fi
