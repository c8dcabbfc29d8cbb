#!/bin/bash
# Full GPU evidence pass: tests, bench, launch list, ncu --set full of the
# SYRK, the largest digit GEMM (precondition) and the leaf kernel.
set -u
TAG=${1:-r01}
OUT=gpurun_out/$TAG; mkdir -p $OUT
run() { echo "== $*" >> $OUT/log.txt; "$@" >> $OUT/log.txt 2>&1; echo "rc=$?" >> $OUT/log.txt; }
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
run timeout 900 python -m pytest tests -m gpu -x -q
run timeout 600 python bench.py --steps 10 --warmup 3
grep '^{' $OUT/log.txt | tail -1 > $OUT/bench.json
run timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches.csv python tools/prof_phase.py step 2
run timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:umma_gemm_kernel -s 0 -c 1 -o $OUT/syrk python tools/prof_phase.py curvature 1
run timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:umma_gemm_kernel -s 0 -c 2 -o $OUT/prec python tools/prof_phase.py precondition 1
run timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:leaf -s 0 -c 1 -o $OUT/leaf python tools/prof_phase.py inversion 1
echo finished >> $OUT/log.txt
