set -x
mkdir -p gpurun_out/sk3
timeout 900 python -m pytest tests/test_syrk_splitk_gpu.py tests/test_kfac_gpu.py tests/test_bert_golden_gpu.py -x -q > gpurun_out/sk3/tests.txt 2>&1; echo rc=$? >> gpurun_out/sk3/tests.txt
for ks in 1 0; do PF_UB_PER_GRAPH=20 PF_KSPLIT=$ks timeout 300 python tools/ubench_syrk.py > gpurun_out/sk3/ub20_$ks.txt 2>&1; done
PF_KSPLIT=0 timeout 300 python tools/ubench_syrk.py > gpurun_out/sk3/ub1_0.txt 2>&1
timeout 900 python tools/kernel_sweep.py > gpurun_out/sk3/sweep.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/sk3/bench.json 2> gpurun_out/sk3/bench.err
echo finished
