#!/bin/bash
# racecheck / memcheck of the concurrent-host-threads test (concurrent kernels
# from four host threads), with and without serialised launches
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
T=tests/test_gpu_parity.py::test_concurrent_host_threads_match_serial
timeout 900 compute-sanitizer --tool racecheck --print-limit 3 python -m pytest $T -q > gpurun_out/diag_race.txt 2>&1
CUDA_LAUNCH_BLOCKING=1 timeout 900 compute-sanitizer --tool racecheck --print-limit 3 python -m pytest $T -q > gpurun_out/diag_race_blocking.txt 2>&1
timeout 600 compute-sanitizer --tool memcheck --print-limit 3 python -m pytest $T -q > gpurun_out/diag_memcheck.txt 2>&1
for f in diag_race diag_race_blocking diag_memcheck; do echo "== $f"; grep -E "passed|failed|nvalid|SUMMARY|load_desc" gpurun_out/$f.txt | head -6; done
