set -u
OUT=gpurun_out/${1:-r01c}; mkdir -p $OUT
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:leaf -s 0 -c 1 -o $OUT/leaf python tools/prof_phase.py inversion 1 >> $OUT/log.txt 2>&1
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:umma_gemm -s 0 -c 2 -o $OUT/gemm3 python tools/prof_phase.py inversion 1 >> $OUT/log.txt 2>&1
