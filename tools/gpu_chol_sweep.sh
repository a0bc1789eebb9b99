#!/bin/bash
# Cholesky super-panel width x bulk-CTA cap sweep (tools/chol_ab.py per setting)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for W in ${WS:-4 8 16}; do for C in ${CS:-2 3}; do
  r=$(SFB_CHOL_BULK_CTAS=$C SFB_CHOL_PANEL=$W python tools/chol_ab.py 2>&1 | head -1)
  echo "W=$W C=$C $r"
done; done | tee gpurun_out/chol_sweep.txt
