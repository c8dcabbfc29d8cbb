mkdir -p gpurun_out/wd2
timeout 900 python -m pytest tests/test_syrk_splitk_gpu.py -x -q > gpurun_out/wd2/tests.txt 2>&1; echo rc=$? >> gpurun_out/wd2/tests.txt
PF_UB_PER_GRAPH=20 timeout 300 python tools/ubench_syrk.py > gpurun_out/wd2/ub20.txt 2>&1
for i in 1 2; do timeout 600 python bench.py --steps 20 --warmup 5 --no-pipeline --no-cpu-baseline > gpurun_out/wd2/b$i.json 2> gpurun_out/wd2/b$i.err; done
echo finished
