#!/bin/bash
# compute-sanitizer over the GPU parity tests (memcheck: out-of-bounds /
# misaligned global and shared accesses; synccheck: barrier misuse; racecheck:
# shared-memory hazards).  Usage (from this container):
#   gpurun --timeout 3000 -- 'bash tools/sanitize.sh <tag>'
# Reports land in gpurun_out/<tag>/.
set -u
TAG=${1:-san}
OUT=gpurun_out/$TAG; mkdir -p $OUT
CS="compute-sanitizer --target-processes all --print-limit 50 --error-exitcode 99"
SMALL="tests/test_kfac_gpu.py tests/test_cholesky_gpu.py tests/test_slice_gpu.py"
run() { echo "== $*" >> $OUT/log.txt; "$@" >> $OUT/log.txt 2>&1; echo "rc=$?" >> $OUT/log.txt; }
# memcheck: every parity test of the kernels (graph capture included), the
# baseline-size cases too; the persistent GEMM's cross-CTA tickets included
run timeout 2400 $CS --tool memcheck python -m pytest -q -x $SMALL tests/test_bert_golden_gpu.py tests/test_switches_gpu.py
# synccheck / racecheck: the small and odd sizes (tails, n < 128, ragged K)
run timeout 1200 $CS --tool synccheck python -m pytest -q -x $SMALL -k "not baseline and not bert_shapes and not 4096 and not 2048"
run timeout 1800 $CS --tool racecheck --racecheck-report hazard python -m pytest -q -x tests/test_kfac_gpu.py -k "matches_oracle and not baseline"
echo finished >> $OUT/log.txt
