#!/bin/bash
# Round-2 evidence pass: bench line, launch list of one layer step, and one
# `ncu --set full` capture of every kernel class of the layer step (SYRK,
# persistent digit GEMM, the three split widths of the short-K digit GEMM,
# leaf, short / long slicer, damp).  Usage:
#   gpurun --timeout 3000 -- 'bash tools/gpu_profiles_r02.sh <tag>'
set -u
TAG=${1:-r02}
OUT=gpurun_out/$TAG; mkdir -p $OUT
run() { echo "== $*" >> $OUT/log.txt; "$@" >> $OUT/log.txt 2>&1; echo "rc=$?" >> $OUT/log.txt; }
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
nproc > $OUT/host.txt; lscpu | grep -E 'Model name|^CPU\(s\)' >> $OUT/host.txt
[ "${SKIP_TESTS:-0}" = 1 ] || run timeout 900 python -m pytest tests -m gpu -x -q
run timeout 900 python bench.py --steps 20 --warmup 5
grep '^{' $OUT/log.txt | tail -1 > $OUT/bench.json
run timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches.csv python tools/prof_phase.py step 2
cap() {  # name phase kernel-regex skip   (CAPS="name ..." limits the captures: gpurun copies back <= 64 MiB)
  if [ -n "${CAPS:-}" ] && ! echo " $CAPS " | grep -q " $1 "; then return; fi
  run timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base mangled \
      -k "regex:$3" -s ${4:-0} -c 1 -o $OUT/$1 python tools/prof_phase.py $2 1
}
cap syrk curvature 'umma_gemm_kernelILi1ELi256'
# split-K SYRK (single d = 1024 factor: 2-CTA clusters), from the SYRK probe
if [ -z "${CAPS:-}" ] || echo " $CAPS " | grep -q " syrk_splitk "; then
run timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k "regex:umma_gemm_kernelILi1ELi128" -s 6 -c 1 -o $OUT/syrk_splitk python tools/probe/syrk_small.py
fi
cap prec precondition 'umma_gemm_persist_kernelILb0'
cap gemm32 inversion 'umma_gemm_kernelILi3ELi32E' 20
cap gemm64 inversion 'umma_gemm_kernelILi3ELi64E' 10
cap gemm128 inversion 'umma_gemm_kernelILi3ELi128ELb0' 10
cap leaf inversion 'leaf_chol' 10
cap slice_short inversion 'slice_short' 20
cap slice_long inversion 'slice_long'
cap damp inversion 'damp_kernel'
cap lauum inversion 'umma_gemm_persist_kernelILb1'
echo finished >> $OUT/log.txt
