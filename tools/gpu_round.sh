#!/bin/bash
# One gpurun call: GPU tests, a bench line, the ncu launch list and one
# `ncu --profile-from-start off --set full` capture per hot kernel.  Usage (from this container):
#   gpurun --timeout 2400 -- 'bash tools/gpu_round.sh [tag]'
# Everything lands in gpurun_out/<tag>/.
set -u
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi > "$OUT/nvidia-smi.txt" 2>&1
nproc > "$OUT/host.txt"; lscpu | grep -E 'Model name|^CPU\(s\)' >> "$OUT/host.txt"

run() { echo "== $*" >> "$OUT/log.txt"; "$@" >> "$OUT/log.txt" 2>&1; echo "rc=$?" >> "$OUT/log.txt"; }

[ "${SKIP_TESTS:-0}" = 1 ] || run timeout 900 python -m pytest tests -m gpu -x -q
run timeout 600 python bench.py --steps 10 --warmup 3
grep '^{' "$OUT/log.txt" | tail -1 > "$OUT/bench.json"
run timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file "$OUT/launches.csv" python tools/prof_phase.py step 2
if [ "${SKIP_FULL:-0}" != 1 ]; then
  run timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:umma_gemm_kernel -s 0 -c 1 -o "$OUT/syrk" python tools/prof_phase.py curvature 1
  run timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:umma_gemm -s 0 -c 2 -o "$OUT/prec" python tools/prof_phase.py precondition 1
fi
echo finished >> "$OUT/log.txt"
