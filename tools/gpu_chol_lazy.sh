#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
for r in 1 2; do
for D in 0 160 200; do echo DIAG_KB=$D; SFB_CHOL_DIAG_KB=$D python tools/chol_ab.py 2>&1 | head -1 | sed 's/.*hand-written//'; done; done
