#!/bin/bash
# compute-sanitizer (memcheck, initcheck, synccheck, racecheck) over the GPU
# parity suite minus the multi-GB cases (one gpurun call; summaries in gpurun_out/)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
K='not c5_full and not c4_full and not beyond and not large_vs and not exponential_big and not configs1 and not c5'
for t in ${TOOLS:-memcheck initcheck synccheck racecheck}; do
  start=$(date +%s)
  timeout ${SAN_TIMEOUT:-1500} compute-sanitizer --tool $t --print-limit 10 python -m pytest \
      tests/test_gpu_parity.py tests/test_gpu_random_layouts.py tests/test_grf.py -q -x -k "$K" \
      > gpurun_out/san_$t.txt 2>&1
  echo "$t exit $? ($(( $(date +%s) - start )) s)" >> gpurun_out/san_$t.txt
  echo "== $t"; grep -E "passed|failed|ERROR SUMMARY|RACECHECK SUMMARY|exit" gpurun_out/san_$t.txt | tail -4
done
