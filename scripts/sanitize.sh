#!/bin/bash
# compute-sanitizer evidence: memcheck, racecheck (shared-memory
# hazards), synccheck (barrier misuse) and initcheck on the small cases of
# scripts/sanitize_cases.py.  Run on the GPU box:
#   bash scripts/sanitize.sh > gpurun_out/sanitize.log 2>&1
cd "$(dirname "$0")/.."
CS=/usr/local/cuda/bin/compute-sanitizer
for c in persist plain1d refined1d cocg2d cocg3d pencil; do
  for tool in memcheck racecheck synccheck; do
    echo "=== $tool $c"
    timeout 900 $CS --tool $tool --error-exitcode 99 --print-limit 20 python scripts/sanitize_cases.py $c 2>&1 | tail -6
    echo "rc=${PIPESTATUS[0]}"
  done
done
