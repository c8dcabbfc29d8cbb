#!/bin/bash
# compute-sanitizer over the SYRK tile policies added in round 2: split-K
# clusters (DSMEM reduction) and 128 x 256 tiles, auto and forced.
# Usage: gpurun --timeout 1800 -- 'bash tools/sanitize_syrk.sh <tag>'
set -u
TAG=${1:-san_syrk}
OUT=gpurun_out/$TAG; mkdir -p $OUT
CS="compute-sanitizer --target-processes all --print-limit 50 --error-exitcode 99"
run() { echo "== $*" >> $OUT/log.txt; "$@" >> $OUT/log.txt 2>&1; echo "rc=$?" >> $OUT/log.txt; }
for tool in memcheck racecheck synccheck; do
  run timeout 900 $CS --tool $tool python -m pytest -q -x tests/test_syrk_splitk_gpu.py -k "deterministic or accumulate"
done
for env in PF_KSPLIT=8 PF_KSPLIT=4 PF_SYRK_WIDE=2; do
  for tool in memcheck racecheck; do
    run env $env timeout 600 $CS --tool $tool python tools/probe/syrk_small.py
  done
done
echo finished >> $OUT/log.txt
