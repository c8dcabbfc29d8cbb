OUT=gpurun_out/r01j; mkdir -p $OUT
timeout 900 python -m pytest tests/test_engine_gpu.py -x -q > $OUT/test_engine.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > $OUT/tests.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/bench.txt 2>&1
