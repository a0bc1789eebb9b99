#!/bin/bash
# racecheck over the parity tests the full-suite run did not reach in its time
# limit (tests 93+ of tools/gpu_sanitize.sh's selection), one file at a time
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
K='not c5_full and not c4_full and not beyond and not large_vs and not exponential_big and not configs1 and not c5'
for f in tests/test_gpu_parity.py tests/test_gpu_random_layouts.py; do
  start=$(date +%s)
  name=$(basename $f .py)
  timeout ${SAN_TIMEOUT:-1700} compute-sanitizer --tool racecheck --print-limit 10 python -m pytest \
      $f -q -k "$K" --deselect tests/test_gpu_parity.py::test_fisher_walk_forms_bit_exact \
      > gpurun_out/san_race_$name.txt 2>&1
  echo "racecheck $name exit $? ($(( $(date +%s) - start )) s)" >> gpurun_out/san_race_$name.txt
  echo "== $name"; grep -E "passed|failed|RACECHECK SUMMARY|exit" gpurun_out/san_race_$name.txt | tail -3
done
