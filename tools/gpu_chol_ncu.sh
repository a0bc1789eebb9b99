#!/bin/bash
# ncu --set full of the first 40 chol_update launches of one hand-written
# factorisation (the bulk, K = 512, launches are the 296-CTA ones)
cd "${GRAFT_REPO_ROOT:-.}"
ncu --set full --clock-control none --import-source on ${NCU_EXTRA} -k regex:"${KREGEX:-chol_update}" -c ${COUNT:-40} \
    -o gpurun_out/prof_chol_${TAG:-upd} -f python tools/chol_ab.py > gpurun_out/chol_ncu.log 2>&1
tail -3 gpurun_out/chol_ncu.log
