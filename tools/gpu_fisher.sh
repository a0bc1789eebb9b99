#!/bin/bash
# one gpurun call: Fisher parity tests + Fisher bench under tuning knobs
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
if [ -z "$NO_TESTS" ]; then
timeout 900 python -m pytest tests -m gpu -q -x -k "${TEST_K:-fisher or rcont2 or concurrent or held}" \
    > gpurun_out/pytest_fisher.txt 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_fisher.txt
tail -3 gpurun_out/pytest_fisher.txt
fi
for cfg in ${FISHER_CFGS:-"SFB_FISHER_MEMO_INT=1" "SFB_FISHER_MEMO_INT=0"}; do
    name=$(echo "$cfg" | tr '=,' '__')
    env $(echo $cfg | tr ',' ' ') timeout 300 python bench.py --only fisher --steps 10 --warmup 3 --no-cpu \
        > gpurun_out/bench_fisher_$name.json 2> gpurun_out/bench_fisher_$name.err
    python - "$name" "$cfg" <<'PY'
import json, sys
try:
    d = json.loads(open(f"gpurun_out/bench_fisher_{sys.argv[1]}.json").read().strip().splitlines()[-1])
    w = d["workloads"]
    print(sys.argv[2], "T4 %.3e (%.4f ms)" % (w["fisher_T4_1e6"]["value"], w["fisher_T4_1e6"]["ms_per_step"]),
          "T10 %.3e" % w["fisher_T10"]["value"], "T4 e2e %.3e" % w["fisher_T4_1e6"]["e2e"]["value"])
except Exception as e:
    print(sys.argv[2], "failed", e, open(f"gpurun_out/bench_fisher_{sys.argv[1]}.err").read()[-2000:])
PY
done
