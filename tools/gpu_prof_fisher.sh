#!/bin/bash
# one gpurun call: ncu --set full of the Fisher kernel under tuning knobs
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${TAG:-r2}
for K in ${KERNELS:-fisher4 fisher10}; do
  for cfg in ${FISHER_CFGS:-"SFB_FISHER_MEMO_INT=1" "SFB_FISHER_MEMO_INT=0"}; do
    name=$(echo "$cfg" | tr '=' '_' | tr ' ' '_')
    env $cfg timeout 600 ncu --set full --clock-control none --import-source on \
        -k regex:fisher_kernel -s 1 -c 1 -f -o gpurun_out/prof_${K}_${name}_$TAG \
        python tools/prof_driver.py $K > gpurun_out/ncu_${K}_${name}.txt 2>&1
  done
done
ls gpurun_out
