set -x
mkdir -p gpurun_out/wd
timeout 900 python -m pytest tests/test_syrk_splitk_gpu.py tests/test_kfac_gpu.py tests/test_bert_golden_gpu.py -x -q > gpurun_out/wd/tests.txt 2>&1; echo rc=$? >> gpurun_out/wd/tests.txt
for w in 0 1; do PF_UB_PER_GRAPH=20 PF_SYRK_WIDE=$w timeout 300 python tools/ubench_syrk.py > gpurun_out/wd/ub20_w$w.txt 2>&1; done
timeout 300 ncu --set full --clock-control none -k regex:umma_gemm_kernelILi1ELi256 -s 2 -c 1 -o gpurun_out/wd/syrk_wide python tools/probe/syrk_small.py > gpurun_out/wd/ncu.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/wd/bench.json 2> gpurun_out/wd/bench.err
echo finished
