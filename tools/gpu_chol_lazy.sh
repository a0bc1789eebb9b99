#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
for r in 1 2; do
for W in 6 8 10; do echo W=$W; SFB_CHOL_PANEL=$W python tools/chol_ab.py 2>&1 | head -1 | sed 's/.*hand-written//'; done; done
