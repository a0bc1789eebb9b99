#!/bin/bash
# A/B timing of the Fisher kernel: ab/libsfb_head.so (previous build) vs the tree's build,
# then the Fisher GPU parity tests of the tree's build
cd "${GRAFT_REPO_ROOT:-.}"
python tools/fisher_time.py "SFB_LIB=ab/libsfb_head.so" "" "SFB_LIB=ab/libsfb_head.so" ""
if [ -z "$NO_TESTS" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x -k "fisher or rcont2 or concurrent or held" 2>&1 | tail -2
fi
