#!/bin/bash
# GRF Cholesky: GPU tests, the chain-step latency, the acceptance timing and
# the per-kernel launch breakdown (one gpurun call)
cd "${GRAFT_REPO_ROOT:-.}"
python -m pytest tests/test_grf.py -m gpu -x -q > gpurun_out/grf_tests.txt 2>&1; tail -3 gpurun_out/grf_tests.txt
python tools/chol_chain.py 2>&1 | tail -3
for i in 1 2; do python tools/chol_ab.py 2>&1 | head -2; done
WS=8 bash tools/gpu_chol_prof.sh 2>&1 | tail -7
