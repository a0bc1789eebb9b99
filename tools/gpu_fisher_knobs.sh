#!/bin/bash
# Fisher kernel timing under tuning knobs (tools/fisher_time.py; one gpurun call)
cd "${GRAFT_REPO_ROOT:-.}"
CASES=${CASES:-T4,T4x10} python tools/fisher_time.py ${CFGS:-""}
