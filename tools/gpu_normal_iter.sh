#!/bin/bash
# one gpurun call while iterating on the normal fill: parity tests, variant
# sweep, ncu --set full of the float32 fast kernel
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "normal or rsqrt or box_muller" -s \
    > gpurun_out/pytest_normal.txt 2>&1
grep -E "rsqrt|variant|passed|failed|Error" gpurun_out/pytest_normal.txt | tail
timeout 600 python tools/tune.py normal > gpurun_out/tune_normal.txt 2>&1
cat gpurun_out/tune_normal.txt
if [ -z "$NO_NCU" ]; then
  SFB_NORMAL_VARIANT=${NCU_VARIANT:-0} timeout 600 ncu --set full --clock-control none \
      --import-source on -k regex:fill_normal_fast -s 1 -c 1 -f -o gpurun_out/prof_normal_${TAG:-it} \
      python tools/prof_driver.py normal > gpurun_out/ncu_normal.txt 2>&1
  tail -2 gpurun_out/ncu_normal.txt
fi
