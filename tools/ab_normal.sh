#!/bin/bash
# A/B timing of the configs[1] normal fill: ab/libsfb_head.so (previous build) vs the tree's build
cd "${GRAFT_REPO_ROOT:-.}"
for i in 1 2; do
  echo "head:"; SFB_LIB=ab/libsfb_head.so python tools/normal_variants.py 10 | tail -1
  echo "new:";  python tools/normal_variants.py 10 | tail -1
done
