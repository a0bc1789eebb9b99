#!/bin/bash
# one gpurun call: environment facts, GPU parity tests, smoke, short bench
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
{ nvidia-smi; free -g; nproc; lscpu | grep -E "Model name|Socket|Thread"; } > gpurun_out/env.txt 2>&1
timeout ${PYTEST_TIMEOUT:-900} python -m pytest tests -m gpu -q ${PYTEST_ARGS:--k "not c5_full"} \
    > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.txt
timeout ${BENCH_TIMEOUT:-600} python bench.py ${BENCH_ARGS:---steps 5 --warmup 3} \
    > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench exit $?" >> gpurun_out/bench.err
tail -5 gpurun_out/pytest_gpu.txt; cat gpurun_out/smoke.txt | tail -3; tail -3 gpurun_out/bench.err
