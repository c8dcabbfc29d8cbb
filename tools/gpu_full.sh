mkdir -p gpurun_out/full
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/full/tests.txt 2>&1; echo rc=$? >> gpurun_out/full/tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full/smoke.txt 2>&1; echo rc=$? >> gpurun_out/full/smoke.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/full/bench.json 2> gpurun_out/full/bench.err
echo finished
