#!/bin/bash
# one gpurun call: parity tests + bench + ncu launch list + ncu --set full of
# the hot kernels (reports land in gpurun_out/, summaries are copied to profiles/)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${TAG:-r1}
timeout ${PYTEST_TIMEOUT:-900} python -m pytest tests -m gpu -q ${PYTEST_ARGS:--k "not c5_full"} \
    > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.txt
timeout ${BENCH_TIMEOUT:-600} python bench.py ${BENCH_ARGS:---steps 10 --warmup 3} \
    > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench exit $?" >> gpurun_out/bench.err
if [ -z "$NO_REF" ]; then
  timeout 900 python bench.py --impl reference --steps 3 --warmup 1 \
      > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
  echo "reference exit $?" >> gpurun_out/bench_reference.err
fi
if [ -z "$NO_NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
      --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 4 --warmup 3 --no-cpu \
      > gpurun_out/ncu_bench_stdout.txt 2>&1
  for K in ${KERNELS:-uniform exponential normal fisher4 fisher10}; do
    case $K in
      uniform|exponential) RX="fill_uniform_";;
      normal) RX="fill_normal_fast";;
      fisher4|fisher10) RX="fisher_kernel";;
    esac
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$RX -s 1 -c 1 \
        -f -o gpurun_out/prof_${K}_$TAG python tools/prof_driver.py $K \
        > gpurun_out/ncu_${K}.txt 2>&1
  done
fi
tail -3 gpurun_out/pytest_gpu.txt; tail -2 gpurun_out/bench.err; ls gpurun_out
