mkdir -p gpurun_out/rdy
timeout 1200 python -m pytest tests/test_switches_gpu.py tests/test_kfac_gpu.py tests/test_cholesky_gpu.py -x -q > gpurun_out/rdy/tests.txt 2>&1; echo rc=$? >> gpurun_out/rdy/tests.txt
for i in 1 2; do
  for f in 1 0; do PF_READY_FLAGS=$f timeout 600 python bench.py --steps 20 --warmup 5 --no-pipeline --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/rdy/b${f}_$i.json; done
done
CS="compute-sanitizer --target-processes all --print-limit 20 --error-exitcode 99"
for tool in memcheck racecheck synccheck; do
  timeout 900 $CS --tool $tool python -m pytest -q -x tests/test_kfac_gpu.py -k "inverse and not baseline and not 4096" > gpurun_out/rdy/san_$tool.txt 2>&1; echo rc=$? >> gpurun_out/rdy/san_$tool.txt
done
echo finished
