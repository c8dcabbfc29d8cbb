OUT=gpurun_out/${TAG:-sp}; mkdir -p $OUT
python tools/ubench_inv.py > $OUT/ub_spine.txt 2>&1
PF_TRTRI_SPINE=0 python tools/ubench_inv.py > $OUT/ub_nospine.txt 2>&1
PF_TL_DUMP=270:330 python tools/timeline.py 4096:1 > $OUT/tl.txt 2>&1
python -m pytest -q -x tests/test_switches_gpu.py tests/test_kfac_gpu.py > $OUT/tests.txt 2>&1
