mkdir -p gpurun_out/dag
timeout 600 python bench.py --steps 20 --warmup 5 --no-pipeline --no-cpu-baseline > gpurun_out/dag/on.json 2> gpurun_out/dag/on.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-pipeline --no-cpu-baseline --no-dag > gpurun_out/dag/off.json 2> gpurun_out/dag/off.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-pipeline --no-cpu-baseline > gpurun_out/dag/on2.json 2>> gpurun_out/dag/on.err
echo finished
