#!/bin/bash
# compute-sanitizer over the GRF tests (hand-written Cholesky / multiply kernels)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for t in ${TOOLS:-memcheck initcheck synccheck racecheck}; do
  start=$(date +%s)
  timeout ${SAN_TIMEOUT:-1200} compute-sanitizer --tool $t --print-limit 10 python -m pytest \
      tests/test_grf.py -q -x -k "${K:-not simulate_grf_reference_properties}" > gpurun_out/san_grf_$t.txt 2>&1
  echo "$t exit $? ($(( $(date +%s) - start )) s)" >> gpurun_out/san_grf_$t.txt
  echo "== $t"; grep -E "passed|failed|ERROR SUMMARY|RACECHECK SUMMARY|exit" gpurun_out/san_grf_$t.txt | tail -4
done
